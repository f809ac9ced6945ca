#!/bin/bash
# Round-2 pass l: TMA-staged energy sweep (parity, A/B vs the register sweep, ncu DRAM bytes) and the
# DEEP x ring of the fused sweep (bitwise test, knob A/B on C4 / C2, ncu DRAM bytes).
set -x
T=${1:-r2l}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
TGV_BUILD_INCREMENTAL=1 timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "energy or deep or knobs or c1_full or ragged or group or one_iteration" > gpurun_out/${T}_pytest.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bricks.py tests/test_gpu_mixed.py -q -m gpu -x > gpurun_out/${T}_pytest_bricks.log 2>&1
for ch in 1 8 1 8; do
  TGV_BRICK_CHAIN=$ch timeout 900 python bench.py --workload C5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c5_chain$ch.json 2>> gpurun_out/${T}_c5.err
  mv gpurun_out/${T}_c5_chain$ch.json gpurun_out/${T}_c5_chain${ch}_$(date +%s).json
done
timeout 600 python scripts/dev/energy_probe.py > gpurun_out/${T}_energy_ab.log 2>&1
timeout 900 python scripts/dev/knob_probe.py TGV_FUSED_DEEP 0 1 0 1 > gpurun_out/${T}_deep.log 2>&1
timeout 900 python scripts/dev/knob_probe.py TGV_ROUND_SYNC 0 1 0 1 > gpurun_out/${T}_rsync.log 2>&1
for d in 0 1 2; do
  TGV_FUSED_DEEP=$((d == 1)) TGV_ROUND_SYNC=$((d == 2)) timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    -k regex:"fused|energy" --clock-control none -c 8 --csv --log-file gpurun_out/${T}_c4_launches_deep$d.csv \
    python bench.py --workload C4 --steps 1 --warmup 0 --iters 6 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on -k regex:"energy_tma" --clock-control none -c 1 \
    -o gpurun_out/${T}_energy_tma_C4 python bench.py --workload C4 --steps 1 --warmup 0 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out
