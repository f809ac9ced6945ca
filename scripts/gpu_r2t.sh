#!/bin/bash
# Round-2 pass t: brick contexts on the stream-ordered memory pool (parts probe, C5 parts bench, brick tests),
# mixed C5 FUSED vs SPLIT on one box.
set -x
T=${1:-r2t}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bricks.py tests/test_gpu_mixed.py tests/test_gpu_brick_levels.py -q -m gpu -x > gpurun_out/${T}_pytest_bricks.log 2>&1
timeout 900 python scripts/dev/parts_probe.py > gpurun_out/${T}_parts_probe.log 2>&1
timeout 1200 python bench.py --workload C5 --parts 8 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_c5_parts8.json 2> gpurun_out/${T}_c5_parts8.err
for sc in fused split; do
  timeout 1200 python bench.py --workload C5 --mixed --schedule $sc --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c5_mixed_$sc.json 2> gpurun_out/${T}_c5_mixed_$sc.err
done
timeout 900 python bench.py --workload C5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err
ls -la gpurun_out
