#!/bin/bash
# NEXT-3 block-sparse brick sets on one GPU: tests, C5 bench, ncu evidence.
#   usage (from this container): gpurun --timeout 1800 -- 'bash scripts/gpu_bricks.sh [tag]'
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 700 python -m pytest tests/test_gpu_bricks.py tests/test_gpu_brick_levels.py -q -x > gpurun_out/pytest_bricks_$TAG.log 2>&1
timeout 900 python bench.py --workload C5 --steps 3 --warmup 3 > gpurun_out/bench_C5_$TAG.json 2> gpurun_out/bench_C5_$TAG.err
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1400 --csv \
  --log-file gpurun_out/launches_C5_$TAG.csv python bench.py --workload C5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
  > gpurun_out/launches_C5_bench_$TAG.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"brick_(dual|primal)" -s 1210 -c 2 \
  -o gpurun_out/prof_bricks_$TAG python bench.py --workload C5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
  > gpurun_out/prof_bricks_bench_$TAG.log 2>&1
ls -la gpurun_out | tail -20
