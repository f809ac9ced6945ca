#!/bin/bash
# Round-2 pass k: full GPU suite on the current head, then the L2 eviction-hint knob sweep (pass j) with ncu DRAM bytes per hint.
set -x
T=${1:-r2k}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
TGV_BUILD_INCREMENTAL=1 timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 2700 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${T}_pytest.log 2>&1
timeout 900 python scripts/dev/knob_probe.py TGV_L2_HINTS 0 1 2 3 0 1 3 > gpurun_out/${T}_hints.log 2>&1
for h in 0 1 3; do
  TGV_L2_HINTS=$h timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    -k regex:"fused" --clock-control none -c 6 --csv --log-file gpurun_out/${T}_c4_launches_h$h.csv \
    python bench.py --workload C4 --steps 1 --warmup 0 --iters 6 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
ls -la gpurun_out
