#!/bin/bash
# ncu evidence for the bench workload (run under gpurun, 1 GPU).
#   launch list: every launch's device time (cold-cache, serialised)
#   full capture: --set full of the fused kernel and of the split dual/primal kernels
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1200 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/launches_bench_$TAG.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"fused" -s 5 -c 2 \
  -o gpurun_out/prof_fused_$TAG python bench.py --steps 1 --warmup 0 --iters 12 --no-cpu-baseline --no-e2e \
  > gpurun_out/prof_fused_bench_$TAG.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"split" -s 10 -c 2 \
  -o gpurun_out/prof_split_$TAG python bench.py --steps 1 --warmup 0 --iters 12 --schedule split --no-cpu-baseline --no-e2e \
  > gpurun_out/prof_split_bench_$TAG.log 2>&1
ls -la gpurun_out
