#!/bin/bash
# NEXT-row measurements and the large workloads (run under gpurun, 1 GPU)
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python bench.py --vote --workload C2 --steps 3 --warmup 1 > gpurun_out/vote_C2_$TAG.json 2>&1
timeout 600 python bench.py --levels 3 --iters 200 --no-cpu-baseline > gpurun_out/ml_C2_$TAG.json 2>&1
timeout 600 python bench.py --model tvl1 > gpurun_out/tvl1_C2_$TAG.json 2>&1
timeout 600 python bench.py --model tvl1 --schedule split --no-cpu-baseline --no-e2e > gpurun_out/tvl1_split_C2_$TAG.json 2>&1
timeout 600 python bench.py --out-of-core 2097152 --levels 3 --steps 3 --warmup 1 > gpurun_out/ooc_C2_$TAG.json 2>&1
timeout 1200 python bench.py --workload C3 --steps 2 --warmup 1 > gpurun_out/C3_$TAG.json 2>&1
timeout 1200 python bench.py --workload C4 --iters 20 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/C4_$TAG.json 2>&1
timeout 900 python bench.py --vote --workload C4 --steps 2 --warmup 1 > gpurun_out/vote_C4_$TAG.json 2>&1
timeout 1200 python bench.py --workload C4 --out-of-core 268435456 --levels 3 --steps 1 --warmup 1 > gpurun_out/ooc_C4_$TAG.json 2>&1
