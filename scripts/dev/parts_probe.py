"""Time the phases of the C5 parts solve (bench --parts 8) one by one on one GPU (dev tool):
context creation, H2D load, prolongation, 200 iterations, u read-back, destroy, per part."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2107_14790_b200.brick_levels import BrickLevels, PartSolver  # noqa: E402
from paper_2107_14790_b200.bricks import BrickSolver  # noqa: E402

wl = bench.load_workload("C5")
kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma, centers=list(wl.centers))
bl = BrickLevels(wl.shape, bench.cams_of(wl), bench.render_shared(wl, 0, 1), levels=3, edge=32,
                 voxel_radius=wl.voxel_radius, resident_finest=False, device=0, **kw)
ps = PartSolver(bl, 8, pinned=True, schedule="fused")
s = bl.solvers[2].reset().iterate(200)
f = bl.solvers[1]
f.prolong_from(s)
f.iterate(200)
s = f


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(2):
    tot = {}
    for p in ps.mine:
        c, fr, cnt = ps.sets[p]
        t0 = t()
        b = BrickSolver(32, c, fr, **ps.kw)
        b.set_schedule("fused")
        t1 = t()
        b.load(cnt)
        t2 = t()
        b.prolong_from(s)
        t3 = t()
        b.iterate(200)
        t4 = t()
        nA = int((~fr).sum())
        u = b.read_u()[:nA]
        t5 = t()
        b.close()
        t6 = t()
        ph = dict(create=t1 - t0, load=t2 - t1, prolong=t3 - t2, iterate=t4 - t3, read=t5 - t4, close=t6 - t5)
        for k, v in ph.items():
            tot[k] = tot.get(k, 0) + v
        print(f"rep{rep} part {p} ({len(c)} bricks): " + " ".join(f"{k} {v * 1e3:.1f}" for k, v in ph.items()) + " ms",
              flush=True)
    print(f"rep{rep} totals: " + " ".join(f"{k} {v * 1e3:.0f}" for k, v in tot.items()) + " ms", flush=True)
