"""TMA L2 sector promotion (TGV_TMA_PROMO, read when a context builds its tensor maps) on the
fused sweep of C4 (1024^3) and C2: a fresh context per value, voted on the GPU, timed with the
library's per-launch CUDA events (dev tool).  usage: promo_probe.py [values...]"""
import os
import sys

import synth
from paper_2107_14790_b200 import Solver

vals = sys.argv[1:] or ["3", "1", "0", "2", "3", "1"]


def cams_of(wl):
    return [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
             "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]


for name, n in (("C4", 20), ("C2", 200)):
    wl = synth.workload(name)
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
    depths = synth.render_depths(wl)
    out = []
    for v in vals:
        os.environ["TGV_TMA_PROMO"] = v
        s = Solver(wl.shape, list(wl.centers), **kw)
        s.vote(cams_of(wl), depths, voxel_radius=wl.voxel_radius)
        s.iterate(2)
        s.set_timing(True)
        s.iterate(n)
        t = s.timing()
        s.close()
        out.append(f"{v}:{t['fused_ms'] / max(1, t['fused_launches']):.3f}")
        print(f"{name} TGV_TMA_PROMO ms per fused launch: " + " ".join(out), flush=True)
