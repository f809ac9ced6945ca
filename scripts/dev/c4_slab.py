"""Per-GPU efficiency of one C4 z-slab (dev tool): 1024 x 1024 x Z planes of C4
(GPU-voted counts of global planes [0, Z)) as its own grid; fused iterations timed
with CUDA events."""
import sys
import time
import torch
import synth
from paper_2107_14790_b200 import Solver

Z = int(sys.argv[1]) if len(sys.argv) > 1 else 128
IT = int(sys.argv[2]) if len(sys.argv) > 2 else 40
wl = synth.workload("C4")
cams = [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
         "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]
depths = synth.render_depths(wl)
kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
s = Solver((1024, 1024, Z), list(wl.centers), **kw)
s.vote(cams, depths, voxel_radius=wl.voxel_radius)
info = s.info()
s.iterate(5)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
s.iterate(IT)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / IT
nv = 1024 * 1024 * Z
print(f"Z={Z} zc={info['fused_zc']} count_bytes={info['count_bytes']}: {ms:.3f} ms/it, "
      f"{nv / ms / 1e6:.2f} G vox-it/s, {info['bytes_fused'] * nv / ms / 1e6:.0f} GB/s")
