#!/bin/bash
# Round-2 pass p: brick sweep row-warp cp.async ring (TGV_BRICK_RING): bitwise tests, C5 A/B, ncu DRAM bytes.
set -x
T=${1:-r2p}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
TGV_BUILD_INCREMENTAL=1 timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bricks.py tests/test_gpu_mixed.py -q -m gpu -x > gpurun_out/${T}_pytest_bricks.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "energy" > gpurun_out/${T}_pytest_energy.log 2>&1
for rg in 0 1 0 1; do
  TGV_BRICK_RING=$rg timeout 900 python bench.py --workload C5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c5_ring${rg}_$(date +%s).json 2>> gpurun_out/${T}_c5.err
done
for rg in 0 1; do
  TGV_BRICK_RING=$rg timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    -k regex:"brick_fused" --clock-control none -c 12 --csv --log-file gpurun_out/${T}_c5_fused_ring$rg.csv \
    python bench.py --workload C5 --steps 1 --warmup 0 --iters 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
ls -la gpurun_out
