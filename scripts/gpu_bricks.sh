#!/bin/bash
# NEXT-3 block-sparse brick sets on one GPU: tests, C5 benches (in core, parts, SPLIT), ncu evidence.
#   usage (from this container): gpurun --timeout 2400 -- 'bash scripts/gpu_bricks.sh [tag]'
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_bricks.py tests/test_gpu_brick_levels.py -q -x > gpurun_out/pytest_bricks_$TAG.log 2>&1
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 > gpurun_out/bench_C5_$TAG.json 2> gpurun_out/bench_C5_$TAG.err
timeout 900 python bench.py --workload C5 --schedule split --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_split_$TAG.json 2>&1
timeout 900 python bench.py --workload C5 --parts 8 --steps 3 --warmup 3 > gpurun_out/bench_C5_parts8_$TAG.json 2>&1
bash scripts/gpu_bricks_prof.sh $TAG
