#!/bin/bash
# Round-2 pass o: TMA L2 promotion probe, C4 launch list (all of our kernels but the mip pyramid, which ncu
# fails to profile), fused-sweep ncu --set full capture on C4, C2 bench.
set -x
T=${1:-r2o}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
TGV_BUILD_INCREMENTAL=1 timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "energy or c1_full" > gpurun_out/${T}_pytest_quick.log 2>&1
timeout 600 python scripts/dev/energy_probe.py > gpurun_out/${T}_energy_ab.log 2>&1
for k in 1 2; do
  timeout 900 python bench.py --model tvl1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_tvl1_$k.json 2>> gpurun_out/${T}_tvl1.err
done
timeout 1200 python scripts/dev/promo_probe.py 3 1 0 2 3 1 > gpurun_out/${T}_promo.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    -k regex:'^(?!pyramid).*' --clock-control none -c 400 --csv --log-file gpurun_out/${T}_c4_launches.csv \
    python bench.py --workload C4 --steps 1 --warmup 0 --iters 6 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_list.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on -k regex:"fused_tma" -s 3 -c 1 --clock-control none \
    -o gpurun_out/${T}_fused_C4 python bench.py --workload C4 --steps 1 --warmup 0 --iters 6 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_full.log 2>&1
timeout 900 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
ls -la gpurun_out
