#!/bin/bash
# Round-2 pass b: new energy kernel + gap parity tests, default (C4) bench line, C4 footprint / pad / chunk probes,
# ncu launch list of the C4 fused + energy kernels.
set -x
T=${1:-r2b}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
nproc > gpurun_out/${T}_host.txt; free -g >> gpurun_out/${T}_host.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x --durations=30 -k "not stated_count" > gpurun_out/${T}_pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for spec in "512 0" "512 75" "1024 0" "256 0" "256 115"; do
  timeout 300 python scripts/dev/c4_probe.py $spec >> gpurun_out/${T}_probe.log 2>&1
done
for pad in 0 262144 524288 1048576 3145728; do
  TGV_FIELD_PAD=$pad timeout 300 python scripts/dev/c4_probe.py 1024 0 20 2>&1 | sed "s/^/pad=$pad /" >> gpurun_out/${T}_probe.log
done
for zc in 128 512 1024; do
  TGV_FUSED_ZC=$zc timeout 300 python scripts/dev/c4_probe.py 1024 0 20 2>&1 | sed "s/^/zc=$zc /" >> gpurun_out/${T}_probe.log
done
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  -k regex:"fused|energy" --clock-control none -c 12 --csv --log-file gpurun_out/${T}_c4_launches.csv \
  python bench.py --workload C4 --steps 1 --warmup 0 --iters 8 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4_launches.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  -k regex:"fused|energy" --clock-control none -c 60 --csv --log-file gpurun_out/${T}_c2_launches.csv \
  python bench.py --workload C2 --steps 1 --warmup 0 --iters 40 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c2_launches.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"energy_partial" -c 1 \
  -o gpurun_out/${T}_energy_C2 python bench.py --workload C2 --steps 1 --warmup 0 --iters 4 --no-cpu-baseline --no-e2e > gpurun_out/${T}_energy_prof.log 2>&1
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"fused_tma" -s 2 -c 1 \
  -o gpurun_out/${T}_fused_C4 python bench.py --workload C4 --steps 1 --warmup 0 --iters 4 --no-cpu-baseline --no-e2e > gpurun_out/${T}_fused_prof.log 2>&1
ls -la gpurun_out
