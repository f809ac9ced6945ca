python -c "import __graft_entry__ as g; g.build()" || exit 1
for sch in split fused split fused; do
TGV_PARTS_SCHEDULE=$sch timeout 900 python bench.py --workload C5 --parts 8 --steps 2 --warmup 2 > gpurun_out/pab_$sch.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/pab_$sch.json').readlines()[-1]); print('parts $sch', round(d['value']/1e9,2), round(d['ms_per_step']), d['clocks']['sm_mhz'])"
done
