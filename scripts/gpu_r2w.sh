#!/bin/bash
# Round-2 pass w: ncu --set full with source counters of the brick fused sweep on C5's finest level.
set -x
T=${1:-r2w}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1200 /usr/local/cuda/bin/ncu --set full --import-source on -k regex:"brick_fused" -s 6 -c 1 --clock-control none \
    -o gpurun_out/${T}_brick_fused_C5 python bench.py --workload C5 --steps 1 --warmup 0 --iters 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu.log 2>&1
ls -la gpurun_out
