python -c "import __graft_entry__ as g; g.build()" || exit 1
TGV_BRICK_XDEPTH=2 timeout 600 python -m pytest tests/test_gpu_bricks.py -q -x -k fused 2>&1 | tail -1
for d in 1 2 1 2; do
TGV_BRICK_XDEPTH=$d timeout 600 python bench.py --workload C5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/xd$d.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/xd$d.json').readlines()[-1]); print('C5 xdepth=$d', round(d['value']/1e9,2), round(d['ms_per_step']), {k: round(v) for k,v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done
