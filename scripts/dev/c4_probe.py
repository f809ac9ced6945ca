"""C4 footprint probe (dev tool): the fused sweep on a 1024 x 1024 x Z slab of C4 as its own
grid, with BALLAST GB of unrelated device memory allocated first (does the per-launch rate
depend on the total footprint?).  usage: c4_probe.py Z BALLAST_GB [iters]"""
import sys

import torch

import synth
from paper_2107_14790_b200 import Solver

Z = int(sys.argv[1])
BG = float(sys.argv[2])
IT = int(sys.argv[3]) if len(sys.argv) > 3 else 30
ballast = torch.empty(int(BG * 2 ** 30), dtype=torch.uint8, device="cuda") if BG > 0 else None
if ballast is not None:
    ballast.fill_(1)
wl = synth.workload("C4")
cams = [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
         "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]
depths = synth.render_depths(wl)
kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
s = Solver((1024, 1024, Z), list(wl.centers), **kw)
s.vote(cams, depths, voxel_radius=wl.voxel_radius)
info = s.info()
s.iterate(5)
for rep in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.iterate(IT)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / IT
    nv = 1024 * 1024 * Z
    print(f"Z={Z} ballast={BG:.0f}GB state={info['device_bytes'] / 1e9:.1f}GB zc={info['fused_zc']} rep{rep}: "
          f"{ms:.3f} ms/it, {nv / ms / 1e6:.2f} G vox-it/s, {info['bytes_fused'] * nv / ms / 1e6:.0f} GB/s", flush=True)
s.close()
