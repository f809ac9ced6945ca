#!/bin/bash
# Round-2 pass d: C4 goldens (host, background), full GPU suite, default bench (C4, zc 128), C5 (+ mixed), TV-L1 C4,
# slab chunk probes, ncu launch list of C4 and a full capture of the fp32 energy kernel.
set -x
T=${1:-r2d}
export PYTHONPATH=$PWD
mkdir -p gpurun_out/goldens
python -c "import oracle, synth; oracle.build(); synth.build()"
nohup python scripts/make_goldens.py C4 --out gpurun_out/goldens > gpurun_out/${T}_goldens.log 2>&1 &
GP=$!
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x --durations=30 -k "not C4-170" > gpurun_out/${T}_pytest.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --workload C5 --no-cpu-baseline --steps 3 --warmup 1 > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err
timeout 900 python bench.py --workload C5 --mixed --no-cpu-baseline --steps 3 --warmup 1 > gpurun_out/${T}_c5_mixed.json 2> gpurun_out/${T}_c5_mixed.err
timeout 900 python bench.py --workload C4 --model tvl1 --no-cpu-baseline --no-e2e --steps 3 --warmup 1 > gpurun_out/${T}_tvl1_c4.json 2> gpurun_out/${T}_tvl1_c4.err
for spec in "512 128" "512 256" "512 128" "512 256"; do
  set -- $spec
  TGV_FUSED_ZC=$2 timeout 300 python scripts/dev/c4_probe.py $1 0 20 2>&1 | grep -v Warn | sed "s/^/zc=$2 /" >> gpurun_out/${T}_probe.log
done
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  -k regex:"fused|energy" --clock-control none -c 12 --csv --log-file gpurun_out/${T}_c4_launches.csv \
  python bench.py --workload C4 --steps 1 --warmup 0 --iters 8 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4_launches.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"energy_partial" -c 1 \
  -o gpurun_out/${T}_energy_C2 python bench.py --workload C2 --steps 1 --warmup 0 --iters 4 --no-cpu-baseline --no-e2e > gpurun_out/${T}_energy_prof.log 2>&1
wait $GP
ls -la gpurun_out gpurun_out/goldens
