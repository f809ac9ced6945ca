#!/bin/bash
# ncu --set full of one kernel of the bench workload. usage: gpu_prof_one.sh TAG REGEX [extra bench args]
TAG=$1; RX=$2; shift 2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 5 -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 0 --iters 10 --no-cpu-baseline --no-e2e "$@" \
  > gpurun_out/prof_$TAG.log 2>&1
