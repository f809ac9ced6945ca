"""Sweep one library env knob (read at every launch) on the fused dense sweep of C4 (1024^3)
and C2 in one process, timing each value with the library's per-launch CUDA events (dev tool).
usage: knob_probe.py VAR v1 v2 ...   e.g.  knob_probe.py TGV_L2_HINTS 0 1 2 3 0 1 3"""
import os
import sys

import synth
from paper_2107_14790_b200 import Solver

var, vals = sys.argv[1], sys.argv[2:]


def cams_of(wl):
    return [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
             "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]


for name, n in (("C4", 20), ("C2", 200)):
    wl = synth.workload(name)
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
    s = Solver(wl.shape, list(wl.centers), **kw)
    s.vote(cams_of(wl), synth.render_depths(wl), voxel_radius=wl.voxel_radius)
    for rep in range(2):
        out = []
        for v in vals:
            os.environ[var] = v
            s.iterate(2)
            s.set_timing(True)
            s.iterate(n)
            t = s.timing()
            s.set_timing(False)
            out.append(f"{v}:{t['fused_ms'] / max(1, t['fused_launches']):.3f}")
        print(f"{name} rep{rep} {var} ms per fused launch:", " ".join(out), flush=True)
    s.close()
