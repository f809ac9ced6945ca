"""L2-prefetch distance sweep (dev tool): the fused TMA sweep on C4 (1024^3) and C2, and the
fused brick sweep on C5's finest level, timed per launch with the library's CUDA events for
each TGV_L2_PREFETCH / TGV_BRICK_L2_PREFETCH value (read by the library at every launch).
usage: pf_probe.py [dense|bricks]"""
import os
import sys

import synth
from paper_2107_14790_b200 import Solver

which = sys.argv[1] if len(sys.argv) > 1 else "dense"


def cams_of(wl):
    return [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
             "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]


def sweep(s, var, vals, n, label):
    out = []
    for v in vals:
        os.environ[var] = str(v)
        s.iterate(2)
        s.set_timing(True)
        s.iterate(n)
        t = s.timing()
        s.set_timing(False)
        ms = t["fused_ms"] / max(1, t["fused_launches"])
        out.append(f"{v}:{ms:.3f}")
    print(f"{label} {var} ms per fused launch:", " ".join(out), flush=True)


if which == "dense":
    for name, n in (("C4", 20), ("C2", 200)):
        wl = synth.workload(name)
        kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
        s = Solver(wl.shape, list(wl.centers), **kw)
        s.vote(cams_of(wl), synth.render_depths(wl), voxel_radius=wl.voxel_radius)
        for rep in range(2):
            sweep(s, "TGV_L2_PREFETCH", [0, 1, 2, 3, 4, 6], n, f"{name} rep{rep}")
        s.close()
else:
    from paper_2107_14790_b200.brick_levels import BrickLevels
    wl = synth.workload("C5")
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma, centers=list(wl.centers))
    bl = BrickLevels(wl.shape, cams_of(wl), synth.render_depths(wl), levels=3, edge=32, voxel_radius=wl.voxel_radius,
                     **kw)
    f = bl.solvers[0]
    for rep in range(2):
        sweep(f, "TGV_BRICK_L2_PREFETCH", [0, 2, 3, 4, 6], 10, f"C5 finest rep{rep}")
    bl.close()
