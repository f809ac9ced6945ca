#!/bin/bash
# Round-2 pass h: the fused sweep with a 3-plane x ring (counts by plain loads, one suv buffer, 36-wide p / q boxes):
# correctness (parity, bitwise schedules, slabs, peer IPC, leaves, sanitizers), A/B against the previous build, bench.
set -x
T=${1:-r2h}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
TGV_BUILD_INCREMENTAL=1 timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multislab.py tests/test_gpu_peer_ipc.py tests/test_gpu_leaves.py tests/test_gpu_sanitizer.py tests/test_gpu_multilevel.py tests/test_gpu_full_size.py -q -m gpu -k "not c2_full_grid_full" > gpurun_out/${T}_pytest.log 2>&1
bash scripts/dev/ab_probe.sh gpurun_out/${T}_ab.log paper_2107_14790_b200/lib/libtgv.so paper_2107_14790_b200/lib/libtgv_prev.so
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  -k regex:"fused|energy" --clock-control none -c 12 --csv --log-file gpurun_out/${T}_c4_launches.csv \
  python bench.py --workload C4 --steps 1 --warmup 0 --iters 8 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c4_launches.log 2>&1
ls -la gpurun_out
