#!/bin/bash
# Round-2 pass n: energy sweeps A/B (regs / tma / tma2, round sync), fused chunk size under the round
# sync, TV-L1 round sync A/B on C4, C4 launch list (DRAM bytes of the round-synced sweep), full GPU suite.
set -x
T=${1:-r2n}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
TGV_BUILD_INCREMENTAL=1 timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "energy or knobs or graph or round_sync or c1_full or one_iteration" > gpurun_out/${T}_pytest_quick.log 2>&1
timeout 600 python scripts/dev/energy_probe.py > gpurun_out/${T}_energy_ab.log 2>&1
timeout 900 python scripts/dev/knob_probe.py TGV_FUSED_ZC 128 64 256 128 64 256 > gpurun_out/${T}_zc.log 2>&1
for rs in 1 0; do
  TGV_ROUND_SYNC=$rs timeout 900 python bench.py --model tvl1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_tvl1_rs$rs.json 2>> gpurun_out/${T}_tvl1.err
done
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -c 400 --csv --log-file gpurun_out/${T}_c4_launches.csv \
    python bench.py --workload C4 --steps 1 --warmup 0 --iters 6 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 2700 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${T}_pytest.log 2>&1
ls -la gpurun_out
