#!/bin/bash
# Round-2 pass f: energy-kernel parity after the per-plane barrier, default bench (C4, with the CPU baseline), C2 bench,
# pad probes at 128-plane chunks, ncu launch list and a full capture of the C4 energy kernel.
set -x
T=${1:-r2f}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py tests/test_gpu_multislab.py -q -m gpu -x -k "not c2_full_grid_full" > gpurun_out/${T}_pytest.log 2>&1
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
for pad in 131072 524288 131072 524288; do
  TGV_FIELD_PAD=$pad timeout 300 python scripts/dev/c4_probe.py 1024 0 20 2>&1 | grep -v Warn | sed "s/^/pad=$pad /" >> gpurun_out/${T}_probe.log
done
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  -k regex:"fused|energy" --clock-control none -c 12 --csv --log-file gpurun_out/${T}_c4_launches.csv \
  python bench.py --workload C4 --steps 1 --warmup 0 --iters 8 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4_launches.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"energy_partial" -c 1 \
  -o gpurun_out/${T}_energy_C4 python bench.py --workload C4 --steps 1 --warmup 0 --iters 2 --no-cpu-baseline --no-e2e > gpurun_out/${T}_energy_prof.log 2>&1
ls -la gpurun_out
