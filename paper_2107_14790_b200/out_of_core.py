"""NEXT-3 (z-slab leaves): out-of-core coarse-to-fine TGV with frozen leaf borders
(§4.5 and Fig. 9: "we update the indicator for all cubes inside the
current leaf's border (set A) while the indicator for neighboring cubes outside of
the border (set B) is frozen and is equal to indicator values of their parenting
cubes"; PAPER.md:431-433 coarse-to-fine; R23).

The device holds one leaf at a time (plus the next one being staged); the levels'
u and v live in host memory, the histogram counts of the finest level too.  Each
leaf is a z-slab of a level: a libtgv leaf context (tgv_create_leaf) whose counts
are the fine counts summed on the device (tgv_load_histograms_coarsened), whose
state and frozen borders are prolongated on the device from the parent level's
host u, v (tgv_prolong_slab), then `iters` fused iterations.  Levels that fit in one
leaf are solved whole (the paper's batching of the treetop leaves).

Orchestration only: every arithmetic step runs in libtgv.so's kernels.  While leaf
k iterates on its stream, leaf k+1 is created, loaded and prolongated on its own,
so the host<->device traffic of one leaf hides behind the iterations of the other.
"""
from __future__ import annotations

import numpy as np

from .multilevel import level_shapes
from .tgv import Solver


def leaf_cuts(shape, leaf_voxels: int):
    """z-cuts of one level: consecutive slabs of max(1, leaf_voxels // (nx ny)) planes
    from z = 0; a level of at most leaf_voxels voxels is one leaf."""
    nx, ny, nz = shape
    planes = nz if nx * ny * nz <= leaf_voxels else max(1, leaf_voxels // (nx * ny))
    cuts = list(range(0, nz, planes)) + [nz]
    return cuts


def _parents(z0, z1, nz, cnz):
    """Coarse planes [c0, c1) holding the parents of fine planes z0-1 .. z1 (those that exist)."""
    lo = max(z0 - 1, 0) // 2
    hi = min(z1, nz - 1) // 2 + 1
    return lo, min(hi, cnz)


def solve(shape, counts, centers, levels=3, iters=200, leaf_voxels=1 << 24, device=0, stats=None, **params):
    """Out-of-core coarse-to-fine solve.  counts: host uint32 [nz, ny, nx, nbins] of the
    finest grid.  Returns host (u [nz, ny, nx], v [3, nz, ny, nx]) of the finest level.
    `stats` (a dict) receives the leaf counts per level."""
    counts = np.ascontiguousarray(counts, dtype=np.uint32)
    shapes = level_shapes(shape, levels)
    if np.prod(shapes[-1]) > leaf_voxels:
        raise ValueError(f"the coarsest level {shapes[-1]} must fit in one leaf ({leaf_voxels} voxels)")
    prev = None
    for lev in range(levels - 1, -1, -1):
        sx, sy, sz = shapes[lev]
        factor = 1 << lev
        u = np.empty((sz, sy, sx), np.float32)
        v = np.empty((3, sz, sy, sx), np.float32)
        cuts = leaf_cuts(shapes[lev], leaf_voxels)
        if stats is not None:
            stats.setdefault("leaves", []).append(len(cuts) - 1)

        def stage(z0, z1):
            leaf = Solver.leaf(shapes[lev], centers, z0, z1, device=device, **params)
            f0, f1 = z0 * factor, min(z1 * factor, shape[2])
            leaf.load_coarsened(counts[f0:f1], shape, factor)
            if prev is not None:
                pu, pv = prev
                c0, c1 = _parents(z0, z1, sz, pu.shape[0])
                leaf.prolong_slab(pu[c0:c1], pv[:, c0:c1], c0)
            return leaf

        nxt = stage(cuts[0], cuts[1])
        for k in range(len(cuts) - 1):
            cur = nxt
            cur.iterate(iters)  # asynchronous on the leaf's stream
            nxt = stage(cuts[k + 1], cuts[k + 2]) if k + 2 < len(cuts) else None
            z0, z1 = cuts[k], cuts[k + 1]
            cur.read_u(u[z0:z1])
            cur.get_into("v", v[:, z0:z1])
            cur.close()
        prev = (u, v)
    return prev
