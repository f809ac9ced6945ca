"""NEXT-3 (z-slab leaves): out-of-core coarse-to-fine TGV with frozen leaf borders
(§4.5 and Fig. 9: "we update the indicator for all cubes inside the
current leaf's border (set A) while the indicator for neighboring cubes outside of
the border (set B) is frozen and is equal to indicator values of their parenting
cubes"; PAPER.md:431-433 coarse-to-fine; R23).

The levels' u and v live in host memory (pinned), and so do the finest counts; the
device holds a pool of leaf contexts (two per leaf size: one iterating while the
other is read back and restaged).  Each leaf is a z-slab of a level: a libtgv leaf
context (tgv_create_leaf, moved between slabs with tgv_leaf_rebind) whose counts are
the fine counts summed on the device (tgv_load_histograms_coarsened), whose state
and frozen borders are prolongated on the device from the parent level's host u, v
(tgv_prolong_slab), then `iters` fused iterations.  A level that fits in one leaf is
solved whole (the paper's batching of the treetop leaves).

Orchestration only: every arithmetic step runs in libtgv.so's kernels.  The counts
of leaf k+1 (the next level's first leaf included) are loaded while leaf k iterates,
and leaf k is read back while leaf k+1 iterates, so most host<->device traffic hides
behind the iterations.
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
    return list(range(0, nz, planes)) + [nz]


def _parents(z0, z1, nz, cnz):
    """Coarse planes [c0, c1) holding the parents of fine planes z0-1 .. z1 (those that exist)."""
    lo = max(z0 - 1, 0) // 2
    hi = min(z1, nz - 1) // 2 + 1
    return lo, min(hi, cnz)


def _host_empty(shape, pinned):
    if pinned:
        try:
            import torch
            return torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()
        except Exception:  # no CUDA-capable torch: pageable memory
            pass
    return np.empty(shape, np.float32)


class OutOfCore:
    """Out-of-core coarse-to-fine solver over z-slab leaves of <= leaf_voxels voxels.

    solve(counts) returns (u, v) of the finest level as views of this object's host
    buffers (overwritten by the next solve).  With keep_pool the leaf contexts stay
    allocated between solves; otherwise each level's pool is freed when it is done
    (device memory bounded by two leaves)."""

    def __init__(self, shape, centers, levels=3, iters=200, leaf_voxels=1 << 24, device=0, keep_pool=True,
                 pinned=True, **params):
        self.shape = tuple(int(n) for n in shape)
        self.centers, self.iters, self.device, self.params = list(centers), int(iters), device, params
        self.shapes = level_shapes(self.shape, levels)
        if int(np.prod(self.shapes[-1])) > leaf_voxels:
            raise ValueError(f"the coarsest level {self.shapes[-1]} must fit in one leaf ({leaf_voxels} voxels)")
        self.cuts = [leaf_cuts(sh, leaf_voxels) for sh in self.shapes]
        self.keep_pool = keep_pool
        self.pool = {}  # (level, planes) -> free leaf Solvers
        self.u = [_host_empty(sh[::-1], pinned) for sh in self.shapes]
        self.v = [_host_empty((3,) + sh[::-1], pinned) for sh in self.shapes]

    @property
    def leaves(self):
        """Leaves per level, finest first."""
        return [len(c) - 1 for c in self.cuts]

    def _leaf(self, lev, z0, z1):
        free = self.pool.setdefault((lev, z1 - z0), [])
        if free:
            return free.pop().rebind(z0, z1)
        return Solver.leaf(self.shapes[lev], self.centers, z0, z1, device=self.device, **self.params)

    def _load(self, lev, z0, z1, counts):
        leaf = self._leaf(lev, z0, z1)
        factor = 1 << lev
        leaf.load_coarsened(counts[z0 * factor:min(z1 * factor, self.shape[2])], self.shape, factor)
        return leaf

    def _prolong(self, lev, leaf, z0, z1):
        if lev + 1 < len(self.shapes):
            pu, pv = self.u[lev + 1], self.v[lev + 1]
            c0, c1 = _parents(z0, z1, self.shapes[lev][2], pu.shape[0])
            leaf.prolong_slab(pu[c0:c1], pv[:, c0:c1], c0)

    def _retire(self, lev, leaf, z0, z1):
        leaf.read_u(self.u[lev][z0:z1])  # waits for the leaf's iterations
        leaf.get_into("v", self.v[lev][:, z0:z1])
        self.pool[(lev, z1 - z0)].append(leaf)

    def solve(self, counts):
        """counts: host uint8 / uint16 / uint32 [nz, ny, nx, nbins] of the finest grid
        (narrow types move fewer bytes; pinned memory overlaps the copies)."""
        counts = np.asarray(counts)
        if counts.dtype not in (np.uint8, np.uint16, np.uint32):
            counts = counts.astype(np.uint32)
        counts = np.ascontiguousarray(counts)
        # every leaf of every level, coarsest level first.  A leaf's counts do not
        # depend on other leaves, so leaf j+1 is loaded while leaf j iterates; its
        # prolongation needs the whole parent level, read back before it.
        items = [(lev, self.cuts[lev][k], self.cuts[lev][k + 1]) for lev in range(len(self.shapes) - 1, -1, -1)
                 for k in range(len(self.cuts[lev]) - 1)]
        pending = None
        nxt = self._load(*items[0], counts)
        for j, (lev, z0, z1) in enumerate(items):
            cur = nxt
            if pending is not None and pending[0] != lev:  # the parent level is complete first
                self._retire(*pending)
                self._free_level(pending[0])
                pending = None
            self._prolong(lev, cur, z0, z1)
            cur.iterate_async(self.iters)  # enqueued on the leaf's stream
            if pending is not None:
                self._retire(*pending)
            pending = (lev, cur, z0, z1)
            nxt = self._load(*items[j + 1], counts) if j + 1 < len(items) else None
        self._retire(*pending)
        self._free_level(pending[0])
        return self.u[0], self.v[0]

    def _free_level(self, lev):
        if not self.keep_pool:
            for key in [k for k in self.pool if k[0] == lev]:
                for leaf in self.pool.pop(key):
                    leaf.close()

    def close(self):
        for leaves in self.pool.values():
            for leaf in leaves:
                leaf.close()
        self.pool = {}

    def __del__(self):
        self.close()


def solve(shape, counts, centers, levels=3, iters=200, leaf_voxels=1 << 24, device=0, stats=None, **params):
    """One out-of-core solve (see OutOfCore); returns copies of the finest (u, v).
    `stats` (a dict) receives the leaf counts per level, coarsest first."""
    ooc = OutOfCore(shape, centers, levels, iters, leaf_voxels, device, keep_pool=False, pinned=False, **params)
    try:
        u, v = ooc.solve(counts)
        if stats is not None:
            stats["leaves"] = ooc.leaves[::-1]
        return u.copy(), v.copy()
    finally:
        ooc.close()
