"""Quick timing sweep of the fused kernel over env knobs (dev tool, not the bench)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2107_14790_b200 import Solver  # noqa: E402

wl = synth.workload(sys.argv[1] if len(sys.argv) > 1 else "C2")
h = synth.make_histograms(wl.name)
knob = sys.argv[2] if len(sys.argv) > 2 else "TGV_FUSED_ZC"
vals = sys.argv[3].split(",") if len(sys.argv) > 3 else ["0"]
sched = sys.argv[4] if len(sys.argv) > 4 else "fused"
for v in vals:
    os.environ[knob] = v
    s = Solver(wl.shape, list(wl.centers)).set_schedule(sched).load(h)
    s.iterate(20)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.iterate(200)
    el = time.perf_counter() - t0
    info = s.info()
    print(f"{knob}={v} zc={info['fused_zc']} tma={info['fused_tma']}: {el / 200 * 1e3:.4f} ms/it "
          f"{wl.nvox * 200 / el / 1e9:.2f} G vox-it/s", flush=True)
    s.close()
