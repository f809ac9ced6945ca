#!/bin/bash
# Round-2 pass ad (final round check after the round-sync refactor): the give-up test first, then the full GPU
# suite and the default bench.
set -x
T=${1:-r2ad}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "gives_up" > gpurun_out/${T}_giveup.log 2>&1
timeout 2700 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${T}_pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
ls -la gpurun_out
