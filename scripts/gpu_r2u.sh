#!/bin/bash
# Round-2 pass u: pinned part read-back, mixed default SPLIT: brick tests, C5 parts and mixed lines.
set -x
T=${1:-r2u}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bricks.py tests/test_gpu_mixed.py tests/test_gpu_brick_levels.py -q -m gpu -x > gpurun_out/${T}_pytest_bricks.log 2>&1
timeout 1200 python bench.py --workload C5 --parts 8 --steps 2 --warmup 1 > gpurun_out/${T}_c5_parts8.json 2> gpurun_out/${T}_c5_parts8.err
timeout 1200 python bench.py --workload C5 --mixed --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_c5_mixed.json 2> gpurun_out/${T}_c5_mixed.err
ls -la gpurun_out
