#!/bin/bash
# ncu evidence for the C5 brick-set bench (run under gpurun, 1 GPU):
#   launch list of every brick solve kernel of one step, and --set full captures of
#   the finest level's fused sweep, frozen-face dual, and (SPLIT) dual / primal kernels
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --workload C5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"brick_(dual|primal|fused|energy|prolong|init)|energy_final" -c 3000 --csv \
  --log-file gpurun_out/launches_C5_$TAG.csv $B > gpurun_out/launches_C5_bench_$TAG.log 2>&1
# fused: 200 launches per level, finest level from launch 400; frozen faces: levels 1 and 0 (200 each)
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"brick_fused" -s 500 -c 1 \
  -o gpurun_out/prof_brick_fused_$TAG $B > gpurun_out/prof_brick_fused_bench_$TAG.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"brick_dual" -s 300 -c 1 \
  -o gpurun_out/prof_brick_faces_$TAG $B > gpurun_out/prof_brick_faces_bench_$TAG.log 2>&1
ls -la gpurun_out | tail
