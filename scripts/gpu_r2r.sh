#!/bin/bash
# Round-2 pass r: NEXT-3 lines on the final code: C5 with its finest level as a 2:1 mixed set (FUSED), C5 in 8 parts.
set -x
T=${1:-r2r}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1200 python bench.py --workload C5 --mixed --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_c5_mixed.json 2> gpurun_out/${T}_c5_mixed.err
timeout 1200 python bench.py --workload C5 --parts 8 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_c5_parts8.json 2> gpurun_out/${T}_c5_parts8.err
ls -la gpurun_out
