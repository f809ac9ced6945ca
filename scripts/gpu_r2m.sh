#!/bin/bash
# Round-2 pass m: full GPU suite (energy sweep fixed, lock-step round sync on, CUDA-graph iterate),
# energy A/B, band-major schedule knob, C4 default bench, C5 bench, C4 launch list + energy ncu capture.
set -x
T=${1:-r2m}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
TGV_BUILD_INCREMENTAL=1 timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "energy or knobs or graph or c1_full or one_iteration" > gpurun_out/${T}_pytest_quick.log 2>&1
timeout 600 python scripts/dev/energy_probe.py > gpurun_out/${T}_energy_ab.log 2>&1
timeout 900 python scripts/dev/knob_probe.py TGV_SCHED_BANDS 0 1 0 1 > gpurun_out/${T}_bands.log 2>&1
timeout 1500 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --workload C5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -c 400 --csv --log-file gpurun_out/${T}_c4_launches.csv \
    python bench.py --workload C4 --steps 1 --warmup 0 --iters 6 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on -k regex:"energy_tma" --clock-control none -c 1 \
    -o gpurun_out/${T}_energy_tma_C4 python bench.py --workload C4 --steps 1 --warmup 0 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 2700 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${T}_pytest.log 2>&1
ls -la gpurun_out
