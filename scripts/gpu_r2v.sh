#!/bin/bash
# Round-2 pass v (final check): full GPU suite, default bench (C4), C5 bench (pinned e2e), C5 mixed default.
set -x
T=${1:-r2v}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 2700 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${T}_pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --workload C5 --steps 2 --warmup 1 > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err
timeout 1200 python bench.py --workload C5 --mixed --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${T}_c5_mixed.json 2> gpurun_out/${T}_c5_mixed.err
ls -la gpurun_out
