#!/bin/bash
# Round-2 pass z (final round check): full GPU suite, default bench (C4), C2 line, C4 out-of-core 3-level line.
set -x
T=${1:-r2z}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 2700 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${T}_pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
timeout 1500 python bench.py --workload C4 --levels 3 --out-of-core 268435456 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_c4_ooc.json 2> gpurun_out/${T}_c4_ooc.err
ls -la gpurun_out
