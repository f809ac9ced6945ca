python -c "import __graft_entry__ as g; g.build()" || exit 1
for i in 1 2 3; do
timeout 600 python bench.py --workload C5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/rep$i.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/rep$i.json').readlines()[-1]); print('C5 rep$i', round(d['value']/1e9,2), round(d['ms_per_step']), {k: round(v) for k,v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'], d['clocks']['power_w_max'])"
done
