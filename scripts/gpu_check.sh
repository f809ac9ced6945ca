#!/bin/bash
# One gpurun session: build, GPU tests, smoke, bench (both schedules).
# usage (from this container):  gpurun --timeout 1800 -- 'bash scripts/gpu_check.sh [tag]'
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi_$TAG.txt 2>&1
timeout 300 TGV_BUILD_INCREMENTAL=1 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1 || exit 1
timeout 900 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
TGV_FUSED_IMPL=regs timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_regs_$TAG.json 2>&1
timeout 600 python bench.py --schedule split --no-cpu-baseline --no-e2e > gpurun_out/bench_split_$TAG.json 2> gpurun_out/bench_split_$TAG.err
