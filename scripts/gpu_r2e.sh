#!/bin/bash
# Round-2 pass e: full GPU suite (C3 + C4 goldens, mixed sets, sanitizers), C5 mixed bench, C4 energy launch list.
set -x
T=${1:-r2e}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 2700 python -m pytest tests -q -m gpu --durations=40 > gpurun_out/${T}_pytest.log 2>&1
timeout 900 python bench.py --workload C5 --mixed --no-cpu-baseline --steps 3 --warmup 1 > gpurun_out/${T}_c5_mixed.json 2> gpurun_out/${T}_c5_mixed.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  -k regex:"fused|energy" --clock-control none -c 12 --csv --log-file gpurun_out/${T}_c4_launches.csv \
  python bench.py --workload C4 --steps 1 --warmup 0 --iters 8 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4_launches.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"mixed|brick" --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/${T}_c5_mixed_launches.csv \
  python bench.py --workload C5 --mixed --steps 1 --warmup 0 --iters 6 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c5_mixed_launches.log 2>&1
ls -la gpurun_out
