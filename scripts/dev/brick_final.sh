python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_bricks.py tests/test_gpu_brick_levels.py -q -x 2>&1 | tail -1
for sch in fused split fused; do
timeout 600 python bench.py --workload C5 --schedule $sch --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/fin_$sch.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/fin_$sch.json').readlines()[-1]); print('C5 $sch', round(d['value']/1e9,2), round(d['ms_per_step']), {k: round(v) for k,v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done
