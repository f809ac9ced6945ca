python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_bricks.py -q -x 2>&1 | tail -1
timeout 600 python bench.py --workload C5 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/quick.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/quick.json').readlines()[-1]); print('C5', round(d['value']/1e9,2), round(d['ms_per_step']), {k: round(v) for k,v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"
