"""NEXT-3 2:1 mixed-level brick sets -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu legs may import
this module; it never imports the product and shares no code with it.

What it follows.  The paper discretises on an adaptive octree whose cubes reach their
neighbours through stored references, 2:1 balanced "leading to the point when each
cube has only 4 or less neighbors over each face" (§3.3); a part's
border cubes are frozen at "indicator values of their parenting cubes" (PAPER.md:446-453,
§4.5, Fig. 9).  It never writes the stencil across a level change.  DESIGN.md reading
R27 (this file is its plain statement):

  * a mixed set is a list of bricks of E^3 voxels, brick b at level l_b (voxel edge
    h = 2^l in finest-level units) and integer brick coordinates c_b of that level, so
    voxel (x, y, z) of b is the cube h (E c_b + (x, y, z)) + [0, h)^3; bricks are
    disjoint and 2:1 balanced: face-adjacent voxels differ by at most one level;
  * the +k face neighbours N+_k(i) of voxel i are the voxels whose cubes share a
    piece of i's +k face: none (Neumann, reading R11), one voxel of the same or the
    next coarser level, or the four voxels of the next finer level that tile the face;
  * the forward difference takes the face-area-weighted mean of u over N+_k(i) (the
    face-area averaging of SPEC.md:325) over the centre-to-centre distance along k,
    d = (h_i + h_n) / 2:
        D+_k u(i) = (mean_{n in N+_k(i)} u(n) - u(i)) / d      (0 if N+_k(i) is empty)
    on a one-level set with h = 1 this is reading R6's D+ exactly;
  * every term of the functional is integrated over the cells, so the inner products
    are weighted by the cell volumes H = diag(h^3) (Eq. 2's integral):
        E(u, v) = sum_i h_i^3 [alpha1 |grad u - v| + alpha0 |E v|_F + lambda sum_b h_b |u - c_b|];
    D-_k = -(D+_k)^* is the adjoint in that inner product, D-_k = -H^-1 (D+_k)^T H,
    and grad, E, div = -grad^*, div2 = -E^* are reading R6's formulas with these D+, D-;
  * Chambolle-Pock in the weighted spaces is the unweighted scheme of SURVEY.md §8
    (a1)-(a3) with these operators: the h^3 cancels in the per-cell projections and in
    the per-cell prox of the data term;
  * solved (A) / frozen (B) bricks, S, and the restricted dual are reading R24's, with
    every sum weighted by h^3:
        D_V = sum_A h^3 [min_{u in [-1,1]} (G(u) - u div p) - V |p + div2 q|_1]
            + sum_B h^3 [-u div p - v.(p + div2 q)].

The state is a vector per field over all voxels, brick-major (z, y, x inside a brick);
the operators are sparse matrices built voxel by voxel from the brick geometry (the one
place with loops); everything else is a matrix-vector product or elementwise.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import default_centers
from .bricks import QIDX, data_term, proj, prox


def _voxel_lo(E, levels, coords):
    """[nvox, 3] integer lower corner (x, y, z) of every voxel in its own level's units,
    and [nvox] level; voxel order brick-major, z, y, x inside a brick."""
    z, y, x = np.meshgrid(np.arange(E), np.arange(E), np.arange(E), indexing="ij")
    off = np.stack([x.ravel(), y.ravel(), z.ravel()], 1)  # [E^3, 3]
    lo = (np.asarray(coords, np.int64)[:, None, :] * E + off[None]).reshape(-1, 3)
    lev = np.repeat(np.asarray(levels, np.int64), E ** 3)
    return lo, lev


def neighbours(E, levels, coords):
    """For every voxel and axis k the +k face neighbour set: a list per axis of
    (kind [nvox] in {0 none, 1 same, 2 coarser, 3 finer}, idx [nvox, 4] (-1 padded))."""
    lo, lev = _voxel_lo(E, levels, coords)
    cell = {}
    for i, (p, l) in enumerate(zip(map(tuple, lo), lev)):
        cell[(int(l),) + p] = i
    out = []
    for k in range(3):
        ek = np.eye(3, dtype=np.int64)[k]
        kind = np.zeros(len(lo), np.int8)
        idx = np.full((len(lo), 4), -1, np.int64)
        lat = [a for a in range(3) if a != k]
        for i in range(len(lo)):
            l, p = int(lev[i]), lo[i]
            q = p + ek
            j = cell.get((l,) + tuple(int(t) for t in q))
            if j is not None:
                kind[i], idx[i, 0] = 1, j
                continue
            j = cell.get((l + 1,) + tuple(int(t) for t in (q // 2)))
            if j is not None:
                kind[i], idx[i, 0] = 2, j
                continue
            fine = []
            for a in (0, 1):
                for b in (0, 1):
                    f = 2 * q
                    f[lat[0]] += a
                    f[lat[1]] += b
                    fine.append(cell.get((l - 1,) + tuple(int(t) for t in f)))
            if any(f is not None for f in fine):
                if any(f is None for f in fine):
                    raise ValueError("a face is partly covered by finer voxels (not a brick-aligned 2:1 set)")
                kind[i], idx[i] = 3, fine
        out.append((kind, idx))
    return out


def check_balanced(E, levels, coords):
    """Bricks disjoint (no voxel of one inside another) and 2:1 at every face."""
    lo, lev = _voxel_lo(E, levels, coords)
    h = 2 ** lev
    lo_f = lo * h[:, None]  # finest units
    lmax = int(lev.max())
    occ = {}
    for i in range(len(lo)):
        hh = int(h[i])
        # claim the finest-unit cells of this voxel at the coarsest granularity that is exact
        key = tuple(int(t) for t in lo_f[i])
        for dz in range(hh):
            for dy in range(hh):
                for dx in range(hh):
                    c = (key[0] + dx, key[1] + dy, key[2] + dz)
                    if c in occ:
                        raise ValueError("bricks overlap")
                    occ[c] = i
    del lmax
    for kind, idx in neighbours(E, levels, coords):
        pass  # neighbours() raises on a face that is partly covered by finer voxels
    # a voxel's face neighbour two or more levels finer / coarser would be seen as "none"
    # by neighbours(); detect it from the finest-unit occupancy
    for k in range(3):
        ek = np.eye(3, dtype=np.int64)[k]
        for i in range(len(lo)):
            hh = int(h[i])
            f = lo_f[i] + hh * ek
            for dy in range(hh):
                for dx in range(hh):
                    c = f.copy()
                    lat = [a for a in range(3) if a != k]
                    c[lat[0]] += dx
                    c[lat[1]] += dy
                    j = occ.get(tuple(int(t) for t in c))
                    if j is not None and abs(int(lev[j]) - int(lev[i])) > 1:
                        raise ValueError("not 2:1 balanced")


def dplus_matrix(E, levels, coords, nb=None):
    """D+_k as a sparse [nvox, nvox] matrix per axis (reading R27)."""
    lo, lev = _voxel_lo(E, levels, coords)
    h = (2.0 ** lev).astype(np.float64)
    nb = neighbours(E, levels, coords) if nb is None else nb
    mats = []
    n = len(lo)
    for k in range(3):
        kind, idx = nb[k]
        rows, cols, vals = [], [], []
        for i in range(n):
            if kind[i] == 0:
                continue
            if kind[i] == 1:
                d = h[i]
                rows += [i, i]
                cols += [int(idx[i, 0]), i]
                vals += [1.0 / d, -1.0 / d]
            elif kind[i] == 2:
                d = 0.5 * (h[i] + 2.0 * h[i])
                rows += [i, i]
                cols += [int(idx[i, 0]), i]
                vals += [1.0 / d, -1.0 / d]
            else:
                d = 0.5 * (h[i] + 0.5 * h[i])
                for j in idx[i]:
                    rows.append(i)
                    cols.append(int(j))
                    vals.append(0.25 / d)
                rows.append(i)
                cols.append(i)
                vals.append(-1.0 / d)
        mats.append(sp.csr_matrix((vals, (rows, cols)), shape=(n, n)))
    return mats, h


class MixedOracle:
    """fp64 state of one 2:1 mixed-level brick set (R27).

    levels [nbricks] (0 = finest), coords [nbricks, 3] in each brick's own level units,
    frozen [nbricks] bool.  Arrays exchanged with the caller are brick-major like
    oracle/bricks.py: u [nbricks, E, E, E], v [nbricks, 3, E, E, E], counts [..., nbins]."""

    def __init__(self, edge_, levels, coords, frozen=None, lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25,
                 centers=None, V=2.0):
        self.E = int(edge_)
        self.levels = np.asarray(levels, np.int64).reshape(-1)
        self.coords = np.asarray(coords, np.int64).reshape(-1, 3)
        nbk = len(self.coords)
        self.frozen = np.zeros(nbk, bool) if frozen is None else np.asarray(frozen, bool).reshape(nbk)
        self.c = default_centers(8) if centers is None else np.asarray(centers, np.float64)
        self.lam, self.alpha0, self.alpha1, self.tau, self.sigma, self.V = lam, alpha0, alpha1, tau, sigma, V
        check_balanced(self.E, self.levels, self.coords)
        self.nb = neighbours(self.E, self.levels, self.coords)
        self.Dp, self.h = dplus_matrix(self.E, self.levels, self.coords, self.nb)
        self.w = self.h ** 3  # cell volumes (the inner-product weights)
        W, Wi = sp.diags(self.w), sp.diags(1.0 / self.w)
        self.Dm = [(-(Wi @ D.T @ W)).tocsr() for D in self.Dp]
        n = len(self.h)
        self.act = np.repeat(~self.frozen, self.E ** 3)
        self.om = np.ones(n, bool)
        # S = A + the frozen voxels with a face neighbour in A (either side, any level)
        near = np.zeros(n, bool)
        for D in self.Dp:
            adj = (D != 0).astype(np.int8)
            near |= (adj @ self.act.astype(np.int8)) > 0       # a + neighbour in A
            near |= (adj.T @ self.act.astype(np.int8)) > 0     # a - neighbour in A
        self.S = self.act | near
        self.u, self.ubar = np.zeros(n), np.zeros(n)
        self.v, self.vbar, self.p, self.q = np.zeros((3, n)), np.zeros((3, n)), np.zeros((3, n)), np.zeros((6, n))
        self.hist = np.zeros((n, len(self.c)))

    # ---- operators (reading R6's formulas with R27's D+, D-)
    def grad(self, u):
        return np.stack([D @ u for D in self.Dp])

    def symgrad(self, v):
        e = np.zeros((6, v.shape[1]))
        for k in range(3):
            for l in range(k, 3):
                e[QIDX[k][l]] = 0.5 * (self.Dm[l] @ v[k] + self.Dm[k] @ v[l])
        return e

    def div(self, p):
        return self.Dm[0] @ p[0] + self.Dm[1] @ p[1] + self.Dm[2] @ p[2]

    def div2(self, q):
        return np.stack([self.Dp[0] @ q[QIDX[k][0]] + self.Dp[1] @ q[QIDX[k][1]] + self.Dp[2] @ q[QIDX[k][2]]
                         for k in range(3)])

    # ---- brick-major views
    def _flat(self, a, lead):
        a = np.asarray(a, np.float64)
        nbk, E = len(self.coords), self.E
        if lead == 0:
            return a.reshape(nbk * E ** 3)
        return a.reshape(nbk, lead, E ** 3).transpose(1, 0, 2).reshape(lead, nbk * E ** 3)

    def _bricks(self, a):
        nbk, E = len(self.coords), self.E
        if a.ndim == 1:
            return a.reshape(nbk, E, E, E)
        lead = a.shape[0]
        return a.reshape(lead, nbk, E, E, E).transpose(1, 0, 2, 3, 4).copy()

    def load(self, counts):
        """Histograms of every brick (frozen bricks' are ignored) and reading R9 on A."""
        c = np.asarray(counts, np.float64).reshape(len(self.h), len(self.c))
        self.hist = np.where(self.act[:, None], c, 0.0)
        W = self.hist.sum(-1)
        m = self.hist @ self.c
        u0 = np.where(W > 0, m / np.where(W > 0, W, 1.0), 0.0)
        self.u = np.where(self.act, u0, 0.0)
        self.ubar = self.u.copy()
        self.v[:] = 0.0
        self.vbar[:] = 0.0
        self.p[:] = 0.0
        self.q[:] = 0.0
        return self

    def set_primal(self, u, v=None):
        """u, v on every brick, a restart (ubar = u, vbar = v, p = q = 0; B keeps them)."""
        self.u = self._flat(u, 0).copy()
        self.v = np.zeros((3, len(self.h))) if v is None else self._flat(v, 3).copy()
        self.ubar, self.vbar = self.u.copy(), self.v.copy()
        self.p[:] = 0.0
        self.q[:] = 0.0
        return self

    def set(self, name, a):
        lead = {"u": 0, "ubar": 0, "v": 3, "vbar": 3, "p": 3, "q": 6}[name]
        setattr(self, name, self._flat(a, lead).copy())

    def get(self, name):
        return self._bricks(getattr(self, name))

    def dual(self):
        """(a1) on S; the operators see every voxel (the frozen values around S)."""
        pn = self.p + self.sigma * (self.grad(self.ubar) - self.vbar)
        pn = proj(pn, self.alpha1, pn[0] ** 2 + pn[1] ** 2 + pn[2] ** 2)
        qn = self.q + self.sigma * self.symgrad(self.vbar)
        n2 = qn[0] ** 2 + qn[1] ** 2 + qn[2] ** 2 + 2.0 * (qn[3] ** 2 + qn[4] ** 2 + qn[5] ** 2)
        qn = proj(qn, self.alpha0, n2)
        self.p = np.where(self.S, pn, 0.0)
        self.q = np.where(self.S, qn, 0.0)

    def primal(self):
        """(a2) + (a3) on A; B unchanged."""
        A = self.act
        un = prox(self.u + self.tau * self.div(self.p), self.tau * self.lam, self.hist, self.c)
        vn = self.v + self.tau * (self.p + self.div2(self.q))
        un = np.where(A, un, self.u)
        vn = np.where(A, vn, self.v)
        self.ubar = 2.0 * un - self.u
        self.vbar = 2.0 * vn - self.v
        self.u, self.v = un, vn

    def iterate(self, n):
        for _ in range(int(n)):
            self.dual()
            self.primal()
        return self

    def energy(self):
        """{E, alpha1, alpha0, data, gap, vmax, dual}, every term weighted by h^3."""
        A, w = self.act, self.w
        a = self.grad(self.u) - self.v
        t1 = self.alpha1 * np.sqrt(a[0] ** 2 + a[1] ** 2 + a[2] ** 2)
        e = self.symgrad(self.v)
        t0 = self.alpha0 * np.sqrt(e[0] ** 2 + e[1] ** 2 + e[2] ** 2 + 2.0 * (e[3] ** 2 + e[4] ** 2 + e[5] ** 2))
        td = data_term(self.hist, self.c, self.lam, self.u)
        d = self.div(self.p)
        wq = self.p + self.div2(self.q)
        cand = [-1.0] + list(self.c) + [1.0]
        best = np.min(np.stack([data_term(self.hist, self.c, self.lam, np.full(len(w), uu)) - uu * d
                                for uu in cand]), axis=0)
        dA = best - self.V * (np.abs(wq[0]) + np.abs(wq[1]) + np.abs(wq[2]))
        dB = -self.u * d - (self.v[0] * wq[0] + self.v[1] * wq[1] + self.v[2] * wq[2])
        T1, T0 = float(np.sum((w * t1)[self.S])), float(np.sum((w * t0)[self.S]))
        TD = float(np.sum((w * td)[A]))
        D = float(np.sum((w * dA)[A]) + np.sum((w * dB)[~A]))
        E = T1 + T0 + TD
        vmax = float(np.max(np.abs(self.v[:, A]))) if A.any() else 0.0
        return {"E": E, "alpha1": T1, "alpha0": T0, "data": TD, "gap": E - D, "vmax": vmax, "dual": D}

    def op_norm2(self, iters=200, seed=0):
        """||K||^2 in the weighted norms, K(u, v) = (grad u - v, E v), by power iteration
        on K^* K (K^* (p, q) = (-div p, -p - div2 q))."""
        rng = np.random.default_rng(seed)
        n = len(self.h)
        u, v = rng.normal(size=n), rng.normal(size=(3, n))
        lam_ = 0.0
        for _ in range(iters):
            p = self.grad(u) - v
            q = self.symgrad(v)
            u2, v2 = -self.div(p), -p - self.div2(q)
            nrm = np.sqrt(np.sum(self.w * u2 ** 2) + np.sum(self.w * v2 ** 2))
            lam_ = nrm / np.sqrt(np.sum(self.w * u ** 2) + np.sum(self.w * v ** 2))
            u, v = u2 / nrm, v2 / nrm
        return lam_
