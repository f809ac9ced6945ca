#!/bin/bash
# Round-2 pass g: L2-prefetch distance sweeps (dense TMA sweep on C4 / C2, brick sweep on C5).
set -x
T=${1:-r2g}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
TGV_BUILD_INCREMENTAL=1 timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python scripts/dev/pf_probe.py dense > gpurun_out/${T}_pf_dense.log 2>&1
timeout 1200 python scripts/dev/pf_probe.py bricks > gpurun_out/${T}_pf_bricks.log 2>&1
ls -la gpurun_out
