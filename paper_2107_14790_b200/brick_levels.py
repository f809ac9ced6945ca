"""Block-sparse brick levels, coarse to fine (NEXT-3 + NEXT-1 + NEXT-2 on brick sets;
BASELINE.json configs[4]; reading R24).

Host logic only (which bricks exist, which are frozen); every arithmetic step -- the
Alg. 1 votes, the refinement flags, the prolongation, the iterations, the energy --
runs in libtgv.so through include/tgv_bricks.h.

How a level's bricks are chosen (R25): the paper refines its octree where the depth
samples are (§4.1) and solves each level over the cubes that exist
(PAPER.md:431-461).  Here:
  * the coarsest level is every brick of its grid, all solved;
  * a level's solved set A is every octant (a finer brick) of the coarser level's
    solved bricks that holds at least `min_votes` votes outside the free-space bin
    (tgv_bricks_refine_flags), i.e. where the surface samples of that level are;
  * its frozen set B is the rest of A's 26-neighbourhood inside the grid: the cubes
    "outside of the border" whose values come from the parent level
    (PAPER.md:449-453), by prolongation (R19, tgv_bricks_prolong_from).
Every brick of a finer level then has a parent brick in the coarser level (the
parent of a 26-neighbour of a child of A is in A or its 26-neighbourhood).
"""
from __future__ import annotations

import numpy as np

from .bricks import BrickSolver

_OCT = np.array([(o & 1, o >> 1 & 1, o >> 2) for o in range(8)], dtype=np.int64)
_N26 = np.array([(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)
                 if (dx, dy, dz) != (0, 0, 0)], dtype=np.int64)


def brick_grid(extent, edge, level):
    """Bricks per axis at `level` (voxel size 2^level) covering extent (x, y, z) voxels."""
    s = edge << level
    return tuple((int(n) + s - 1) // s for n in extent)


def _key(c):
    c = np.asarray(c, dtype=np.int64)
    return c[:, 0] | c[:, 1] << 21 | c[:, 2] << 42


def children(coords, flags, grid):
    """Finer bricks of the flagged octants, inside the finer grid, sorted (z, y, x)."""
    b, o = np.nonzero(np.asarray(flags))
    ch = 2 * np.asarray(coords, np.int64)[b] + _OCT[o]
    ch = ch[np.all(ch < np.asarray(grid), axis=1)]
    return _sorted(ch)


def shell(coords, grid):
    """The 26-neighbourhood of `coords` inside `grid`, minus `coords`, sorted."""
    c = np.asarray(coords, np.int64)
    if len(c) == 0:
        return c.reshape(0, 3)
    nb = (c[:, None, :] + _N26[None, :, :]).reshape(-1, 3)
    nb = nb[np.all((nb >= 0) & (nb < np.asarray(grid)), axis=1)]
    nb = _sorted(nb)
    return nb[~np.isin(_key(nb), _key(c))]


def _sorted(c):
    c = np.unique(np.asarray(c, np.int64).reshape(-1, 3), axis=0)
    return c[np.lexsort((c[:, 0], c[:, 1], c[:, 2]))]


_FACES = np.array([(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)], np.int64)


def mixed_border(A, grid):
    """A 2:1 mixed-level set around the level-0 bricks A (R27): A solved; frozen, every
    face neighbour of A inside `grid` as a level-0 brick when its parent cube holds a
    brick of A, else as that parent cube (level 1, deduplicated).  Levels 0 and 1 only,
    so the set is 2:1 balanced, and no level-1 brick contains a level-0 brick.
    Returns (coords int32 [n, 3] in each brick's level units, levels uint8, frozen bool)."""
    A = _sorted(A)
    nb = (A[:, None, :] + _FACES[None]).reshape(-1, 3)
    nb = _sorted(nb[np.all((nb >= 0) & (nb < np.asarray(grid)), axis=1)])
    nb = nb[~np.isin(_key(nb), _key(A))]
    fine = np.isin(_key(nb >> 1), _key(A >> 1))
    B0 = nb[fine]
    B1 = _sorted(nb[~fine] >> 1)
    coords = np.concatenate([A, B0, B1]).astype(np.int32)
    levels = np.concatenate([np.zeros(len(A) + len(B0), np.uint8), np.ones(len(B1), np.uint8)])
    frozen = np.concatenate([np.zeros(len(A), bool), np.ones(len(B0) + len(B1), bool)])
    return coords, levels, frozen


class BrickLevels:
    """Brick sets of `levels` levels (index 0 = finest) built from the depth maps, with
    their counts resident on the GPU; `solve` runs the coarse-to-fine TGV solve."""

    def __init__(self, extent, cams, depths, levels=3, edge=32, grid_origin=(0.0, 0.0, 0.0), voxel_size=1.0,
                 voxel_radius=0.5, min_votes=2, centers=None, lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25,
                 device=0, resident_finest=True):
        """resident_finest=False: the finest level's bricks are chosen (from level 1's
        flags) but no context is created for it -- PartSolver solves it part by part."""
        kw = dict(centers=centers, lam=lam, alpha0=alpha0, alpha1=alpha1, tau=tau, sigma=sigma, device=device)
        self.kw = kw
        self.extent = tuple(int(n) for n in extent)
        self.edge, self.levels = edge, levels
        self.solvers = [None] * levels
        self.coords = [None] * levels
        self.frozen = [None] * levels
        top = levels - 1
        g = brick_grid(extent, edge, top)
        allc = _sorted(np.stack(np.meshgrid(*[np.arange(n) for n in g], indexing="ij"), -1).reshape(-1, 3))
        self._add(top, allc, np.zeros(len(allc), bool), cams, depths, grid_origin, voxel_size, voxel_radius, kw)
        for lev in range(top - 1, -1, -1):
            g = brick_grid(extent, edge, lev)
            up = self.solvers[lev + 1]
            A = children(self.coords[lev + 1], up.refine_flags(min_votes), g)
            B = shell(A, g)
            c = np.concatenate([A, B]).astype(np.int32)
            fr = np.concatenate([np.zeros(len(A), bool), np.ones(len(B), bool)])
            self._add(lev, c, fr, cams, depths, grid_origin, voxel_size, voxel_radius, kw,
                      create=resident_finest or lev > 0)
        self.vote_args = (cams, depths, grid_origin, voxel_size, voxel_radius)

    def _add(self, lev, coords, frozen, cams, depths, origin, h, r, kw, create=True):
        s = None
        if create:
            s = BrickSolver(self.edge, coords, frozen, **kw)
            s.vote(cams, depths, grid_origin=origin, voxel_size=h * (1 << lev), voxel_radius=r * (1 << lev))
        self.solvers[lev], self.coords[lev], self.frozen[lev] = s, np.asarray(coords), np.asarray(frozen)

    def bricks(self):
        """(solved, frozen) brick counts per level, finest first."""
        return [(int((~f).sum()), int(f.sum())) for f in self.frozen]

    def voxels(self):
        return [len(c) * self.edge ** 3 for c in self.coords]

    def solve(self, iters):
        """Coarsest level from its votes (R9), each finer level prolongated from the
        coarser one (R19) with its frozen bricks held at the parent values; `iters`
        iterations per level (R20).  Returns the finest level's BrickSolver."""
        top = self.levels - 1
        s = self.solvers[top].reset().iterate(iters)
        for lev in range(top - 1, -1, -1):
            f = self.solvers[lev]
            f.prolong_from(s)
            f.iterate(iters)
            s = f
        return s

    def mixed_finest(self):
        """The finest level as a 2:1 mixed-level set (R27):
        its solved bricks A (level 0) with a frozen border B of face neighbours -- a
        level-0 brick where the parent cube also holds a brick of A, else the parent
        cube itself (a level-1 brick).  Returns (coords, levels, frozen); the solve
        prolongates every brick from level 1 (R19; a level-1 brick keeps its own u, v / 2)."""
        return mixed_border(self.coords[0][~self.frozen[0]], brick_grid(self.extent, self.edge, 0))

    def build_mixed(self):
        """Create and vote the finest level's mixed-level context (see mixed_finest)."""
        coords, levels, frozen = self.mixed_finest()
        cams, depths, origin, h, r = self.vote_args
        m = BrickSolver(self.edge, coords, frozen, levels=levels, **self.kw)
        m.vote(cams, depths, grid_origin=origin, voxel_size=h, voxel_radius=r)
        self.mixed = (m, coords, levels, frozen)
        return m

    def solve_mixed(self, iters):
        """solve(), with the finest level replaced by its mixed-level set."""
        top = self.levels - 1
        s = self.solvers[top].reset().iterate(iters)
        for lev in range(top - 1, 0, -1):
            f = self.solvers[lev]
            f.prolong_from(s)
            f.iterate(iters)
            s = f
        m = self.mixed[0]
        m.prolong_from(s)
        m.iterate(iters)
        return m

    def close(self):
        for s in self.solvers:
            if s is not None:
                s.close()
        self.solvers = []
        if getattr(self, "mixed", None):
            self.mixed[0].close()
            self.mixed = None


# ---------------------------------------------------------------------------
# Parts of the finest level: the treetop leaves of PAPER.md:370-388 / :446-461.
# A part is a Morton-contiguous run of the finest level's solved bricks; its frozen
# shell is the rest of its 26-neighbourhood (other parts' solved bricks included),
# held at the parent level's values -- the borders of Fig. 9, so parts need no
# exchange: they can be streamed through one GPU (memory bounded by the part) or
# spread over several GPUs (R26).
# ---------------------------------------------------------------------------
def _spread(v):
    v = np.asarray(v, np.uint64) & np.uint64(0x1FFFFF)
    v = (v | v << np.uint64(32)) & np.uint64(0x1F00000000FFFF)
    v = (v | v << np.uint64(16)) & np.uint64(0x1F0000FF0000FF)
    v = (v | v << np.uint64(8)) & np.uint64(0x100F00F00F00F00F)
    v = (v | v << np.uint64(4)) & np.uint64(0x10C30C30C30C30C3)
    v = (v | v << np.uint64(2)) & np.uint64(0x1249249249249249)
    return v


def morton(coords):
    c = np.asarray(coords, np.int64)
    return _spread(c[:, 0]) | _spread(c[:, 1]) << np.uint64(1) | _spread(c[:, 2]) << np.uint64(2)


def split_parts(solved, nparts):
    """Morton-ordered solved bricks cut into nparts contiguous runs of near-equal size."""
    s = np.asarray(solved, np.int64)
    s = s[np.argsort(morton(s), kind="stable")]
    return [_sorted(p) for p in np.array_split(s, nparts) if len(p)]


class PartSolver:
    """The finest level of a BrickLevels solved part by part: out of core (one part's
    bricks on the GPU at a time, its counts in host memory, voted once per part at
    set-up) or only the parts `mine` (a rank's share on several GPUs).  The coarser
    levels stay resident in `levels`."""

    def __init__(self, levels: BrickLevels, nparts, mine=None, pinned=False, schedule=None):
        """schedule: the parts' iteration schedule, "fused" (default; 32^3 bricks) or
        "split" (TGV_PARTS_SCHEDULE overrides the default).  On C5's 8 parts the fused
        sweep measured 21.7-22.7 G solved vox-it/s against SPLIT's 13.6-17.5 G on the
        same box."""
        import os
        sched = (schedule or os.environ.get("TGV_PARTS_SCHEDULE") or "fused").strip().lower()
        if sched not in ("fused", "split"):
            raise ValueError(f"PartSolver schedule must be 'fused' or 'split', got {sched!r}")
        if sched == "fused" and levels.edge != 32:
            sched = "split"  # the fused brick sweep is built for 32^3 bricks only
        self.schedule = sched
        self.bl, self.E = levels, levels.edge
        self.grid = brick_grid(levels.extent, levels.edge, 0)
        A = levels.coords[0][~levels.frozen[0]]
        self.parts = split_parts(A, nparts)
        self.mine = list(range(len(self.parts))) if mine is None else [p for p in mine if p < len(self.parts)]
        cams, depths, origin, h, r = levels.vote_args
        self.kw = levels.kw
        self.sets = {}
        self.ubufs = {}
        for p in self.mine:
            Ap = self.parts[p]
            Bp = shell(Ap, self.grid)
            c = np.concatenate([Ap, Bp]).astype(np.int32)
            fr = np.concatenate([np.zeros(len(Ap), bool), np.ones(len(Bp), bool)])
            ps = BrickSolver(self.E, c, fr, **self.kw).vote(cams, depths, grid_origin=origin, voxel_size=h,
                                                            voxel_radius=r)
            cnt = ps.read_counts()
            if cnt.max() <= 255:
                cnt = cnt.astype(np.uint8)
            ps.close()
            ubuf = None
            if pinned:  # pinned counts (H2D) and a pinned u buffer per part (D2H at full link speed)
                import torch
                cnt = torch.from_numpy(cnt).pin_memory().numpy()
                ubuf = torch.empty(len(c) * self.E ** 3, dtype=torch.float32).pin_memory().numpy()
            self.sets[p] = (c, fr, cnt)
            self.ubufs[p] = ubuf

    def solve(self, iters, pool=None):
        """Coarse levels (resident), then every owned part: H2D of its counts,
        prolongation from the next coarser level, iterations, D2H of its solved bricks'
        u.  pool (dict): keep each part's context between solves (allocation outside
        the solve).  Returns {part: (coords of its solved bricks, u [n, E, E, E])}; with
        pinned=True each u is a view of the part's pinned buffer, rewritten by the next solve."""
        bl = self.bl
        top = bl.levels - 1
        s = bl.solvers[top].reset().iterate(iters)
        for lev in range(top - 1, 0, -1):
            f = bl.solvers[lev]
            f.prolong_from(s)
            f.iterate(iters)
            s = f
        out = {}
        for p in self.mine:
            c, fr, cnt = self.sets[p]
            ps = pool.get(p) if pool is not None else None
            if ps is None:
                ps = BrickSolver(self.E, c, fr, **self.kw)
                ps.set_schedule(self.schedule)
                if pool is not None:
                    pool[p] = ps
            ps.load(cnt).prolong_from(s).iterate(iters)
            nA = int((~fr).sum())
            out[p] = (c[:nA], ps.read_u(self.ubufs[p])[:nA])
            if pool is None:
                ps.close()
        return out

    def solved_voxels(self):
        return sum(len(self.parts[p]) for p in self.mine) * self.E ** 3

    def part_voxels(self):
        return {p: len(self.sets[p][0]) * self.E ** 3 for p in self.mine}
