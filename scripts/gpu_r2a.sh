#!/bin/bash
# Round-2 first GPU pass: tests, smoke, C2 and C4 bench lines, C4 footprint probes, C4 ncu launch list.
set -x
T=${1:-r2a}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${T}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --durations=25 > gpurun_out/${T}_pytest.log 2>&1
timeout 600 python bench.py --workload C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
timeout 900 python bench.py --workload C4 --steps 2 --warmup 1 --iters 30 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err
for spec in "512 0" "512 75" "1024 0" "256 0" "256 115"; do
  timeout 300 python scripts/dev/c4_probe.py $spec >> gpurun_out/${T}_probe.log 2>&1
done
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -c 60 --csv --log-file gpurun_out/${T}_c4_launches.csv \
  python bench.py --workload C4 --steps 1 --warmup 0 --iters 12 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4_launches.log 2>&1
ls -la gpurun_out
