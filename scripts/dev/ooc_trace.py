"""Per-call host time of the out-of-core driver on C2 (dev tool): which calls block."""
import sys
import time
import collections
import numpy as np
import torch
import synth
from paper_2107_14790_b200 import out_of_core
from paper_2107_14790_b200.tgv import Solver

leaf_voxels = int(sys.argv[1]) if len(sys.argv) > 1 else 2097152
wl = synth.workload("C2")
counts = torch.from_numpy(synth.make_histograms("C2")).pin_memory().numpy()
kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
T = collections.defaultdict(float)
N = collections.defaultdict(int)
for name in ("load_coarsened", "prolong_slab", "iterate", "read_u", "get_into", "rebind"):
    f = getattr(Solver, name)
    def wrap(self, *a, _f=f, _n=name, **k):
        t = time.perf_counter()
        r = _f(self, *a, **k)
        lev = self.shape[0]
        T[(lev, _n)] += time.perf_counter() - t
        N[(lev, _n)] += 1
        return r
    setattr(Solver, name, wrap)
ooc = out_of_core.OutOfCore(wl.shape, list(wl.centers), levels=3, iters=200, leaf_voxels=leaf_voxels, **kw)
ooc.solve(counts)
T.clear(); N.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
ooc.solve(counts)
torch.cuda.synchronize()
print("total ms", (time.perf_counter() - t0) * 1e3)
for k in sorted(T):
    print(k, N[k], round(T[k] * 1e3, 2))
