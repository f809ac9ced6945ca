#!/bin/bash
# Round-2 pass x: peer-IPC / multislab / multirank tests after the UUID record change; C2 energy chunk probe.
set -x
T=${1:-r2x}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer_ipc.py tests/test_gpu_multislab.py tests/test_gpu_multirank.py tests/test_gpu_leaves.py -q -m gpu > gpurun_out/${T}_pytest.log 2>&1
timeout 600 python scripts/dev/energy_zc_probe.py > gpurun_out/${T}_energy_zc.log 2>&1
ls -la gpurun_out
