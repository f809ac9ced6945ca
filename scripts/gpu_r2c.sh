#!/bin/bash
# Round-2 pass c: C3 oracle goldens on the host (background), mixed-level GPU tests, sustained-rate probes, zc probes.
set -x
T=${1:-r2c}
export PYTHONPATH=$PWD
mkdir -p gpurun_out/goldens
python -c "import oracle, synth; oracle.build(); synth.build()"
nohup python scripts/make_goldens.py C3 --out gpurun_out/goldens > gpurun_out/${T}_goldens.log 2>&1 &
GP=$!
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_brick_levels.py tests/test_gpu_bricks.py -q -x -m gpu > gpurun_out/${T}_pytest.log 2>&1
SMI_OUT=gpurun_out/${T}_smi_sustain.csv timeout 600 python scripts/dev/sustain_probe.py 1024 300 > gpurun_out/${T}_sustain.log 2>&1
for zc in 64 96 128 256 128 256; do
  TGV_FUSED_ZC=$zc timeout 300 python scripts/dev/c4_probe.py 1024 0 20 2>&1 | grep -v Warn | sed "s/^/zc=$zc /" >> gpurun_out/${T}_probe.log
done
TGV_FUSED_ZC=128 SMI_OUT=gpurun_out/${T}_smi_sustain128.csv timeout 600 python scripts/dev/sustain_probe.py 1024 300 > gpurun_out/${T}_sustain128.log 2>&1
wait $GP
ls -la gpurun_out gpurun_out/goldens
