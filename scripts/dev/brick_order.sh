python -c "import __graft_entry__ as g; g.build()" || exit 1
for o in 0 2 0 2; do
  TGV_BRICK_ORDER=$o timeout 600 python bench.py --workload C5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/order$o.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/order$o.json').readlines()[-1]); print('order=$o', round(d['value']/1e9,2), round(d['ms_per_step']), {k: round(v) for k,v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done
