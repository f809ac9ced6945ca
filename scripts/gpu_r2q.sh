#!/bin/bash
# Round-2 pass q (round check): full GPU suite, default bench (C4), C2 / C3 / C5 / TV-L1 bench lines,
# C4 launch list and the energy sweep's ncu capture.
set -x
T=${1:-r2q}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 2700 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${T}_pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
timeout 1200 python bench.py --workload C3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_c3.json 2> gpurun_out/${T}_c3.err
timeout 900 python bench.py --workload C5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err
timeout 900 python bench.py --model tvl1 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_tvl1.json 2> gpurun_out/${T}_tvl1.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    -k regex:'^(?!pyramid).*' --clock-control none -c 60 --csv --log-file gpurun_out/${T}_c4_launches.csv \
    python bench.py --workload C4 --steps 1 --warmup 0 --iters 6 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_list.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on -k regex:"energy_tma" -c 1 --clock-control none \
    -o gpurun_out/${T}_energy_C4 python bench.py --workload C4 --steps 1 --warmup 0 --iters 2 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_energy.log 2>&1
ls -la gpurun_out
