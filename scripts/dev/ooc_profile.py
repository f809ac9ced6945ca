"""Breakdown of the out-of-core driver's per-leaf costs on C2 (dev tool)."""
import time
import numpy as np
import torch
import synth
from paper_2107_14790_b200 import Solver
from paper_2107_14790_b200.multilevel import level_shapes

wl = synth.workload("C2")
counts = synth.make_histograms("C2")
pinned = torch.from_numpy(counts).pin_memory().numpy()
kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
shape = wl.shape
C = list(wl.centers)
T = {}
def tic(): torch.cuda.synchronize(); return time.perf_counter()
def add(k, t0): torch.cuda.synchronize(); T[k] = T.get(k, 0) + time.perf_counter() - t0
for src_name, src in (("pageable", counts), ("pinned", pinned)):
    T.clear()
    z0, z1 = 0, 32
    for rep in range(3):
        t = tic(); leaf = Solver.leaf(shape, C, 32, 64, **kw); add("create", t)
        t = tic(); leaf.load_coarsened(src[32:64], shape, 1); add("load", t)
        pu = np.zeros((18, 128, 128), np.float32); pv = np.zeros((3, 18, 128, 128), np.float32)
        t = tic(); leaf.prolong_slab(pu, pv, 15); add("prolong", t)
        t = tic(); leaf.iterate(200); add("iterate200", t)
        u = np.empty((32, 256, 256), np.float32); v = np.empty((3, 32, 256, 256), np.float32)
        t = tic(); leaf.read_u(u); leaf.get_into("v", v); add("read", t)
        t = tic(); leaf.close(); add("close", t)
    print(src_name, {k: round(v / 3 * 1e3, 2) for k, v in T.items()})
