python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_bricks.py -q -x -k "fused or ragged or random" 2>&1 | tail -1
for cfg in "0 1" "0 0"; do set -- $cfg
  TGV_BRICK_MORTON=$1 TGV_BRICK_FOLD_X=$2 timeout 600 python bench.py --workload C5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ab_m$1_x$2.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_m$1_x$2.json').readlines()[-1]); print('morton=$1 foldx=$2', round(d['value']/1e9,2), round(d['ms_per_step']), {k: round(v) for k,v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done
