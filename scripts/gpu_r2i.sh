#!/bin/bash
# Round-2 pass i: full GPU suite, default bench (C4, pipelined e2e), C2 bench.
set -x
T=${1:-r2i}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 2700 python -m pytest tests -q -m gpu --durations=20 > gpurun_out/${T}_pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
ls -la gpurun_out
