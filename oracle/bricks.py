"""NEXT-3 block-sparse brick sets -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu legs may import
this module; it never imports the product and shares no code with it.

What it follows.  The paper solves each level over the cubes of an octree, part by
part: "we update the indicator for all cubes inside the current leaf's border (set A)
while the indicator for neighboring cubes outside of the border (set B) is frozen"
(§4.5, Fig. 9), and cubes reach their neighbours through stored
neighbour references (§4.2).  DESIGN.md reading R24 turns this into
a block-sparse level:

  * a level is a list of bricks, edge E voxels, at integer brick coordinates
    (bx, by, bz); each brick is either solved (set A) or frozen (set B);
  * the domain Omega is the union of the bricks' voxels; voxels outside Omega do not
    exist (Neumann / zero flux across the boundary of Omega, reading R11);
  * the difference operators are those of reading R6 restricted to Omega:
        D+_k w[x] = w[x + e_k] - w[x]    if x + e_k in Omega, else 0
        D-_k w[x] = [x + e_k in Omega] w[x] - [x - e_k in Omega] w[x - e_k]
    so that D-_k = -(D+_k)^T on Omega (pinned by tests/test_oracle_bricks.py); on a
    box-shaped Omega they are the dense grid's operators;
  * S = A plus the frozen voxels with a face neighbour in A (dB).  The terms of the
    functional at a voxel x involve u(x), u(x + e_k), v(x), v(x - e_k) only, so the
    terms at voxels outside S are constants of the solve, and the only duals the
    primal step on A reads are those on S (p at x - e_k, q at x + e_l);
  * one iteration is the scheme of oracle/tgv_oracle.c:
    the dual step on the voxels of S (the duals elsewhere stay 0), the primal step
    (prox, clamp, v update, over-relaxation) on the voxels of A only; on B, u and v
    keep the values they were given (ubar = u, vbar = v), as in reading R23's frozen
    leaf borders (whose recomputed halo duals are exactly dB's);
  * the energy is the functional restricted to what the solve changes: the
    regulariser over S and the data term over A.  The restricted dual value follows
    from the saddle-point form sum_S [<grad u - v, p> + <E v, q>] + G(u_A) with the
    duals zero outside S, i.e. sum_Omega [-u div p - v.(p + div2 q)] + G(u_A):
        D_V = sum_A [min_{u in [-1,1]} (G(u) - u div p) - V |p + div2 q|_1]
            + sum_B [-u div p - v.(p + div2 q)]
    and gap = E - D_V >= 0 whenever the minimiser has |v_A| <= V (reading R14).

The state is embedded in the dense bounding box of the bricks (numpy fp64 arrays,
[z, y, x]); the masks do the rest.  Every array operation is elementwise or a shift by
one voxel, written out per axis.
"""
from __future__ import annotations

import numpy as np

from . import default_centers

AX = {0: 2, 1: 1, 2: 0}  # operator axis k (x, y, z) -> numpy axis of a [z, y, x] array
QIDX = ((0, 3, 4), (3, 1, 5), (4, 5, 2))  # symmetric tensor storage xx, yy, zz, xy, xz, yz


def _next(a, k):
    """a[x + e_k], zero beyond the box."""
    ax = AX[k]
    out = np.zeros_like(a)
    src = [slice(None)] * a.ndim
    dst = [slice(None)] * a.ndim
    src[ax] = slice(1, None)
    dst[ax] = slice(0, -1)
    out[tuple(dst)] = a[tuple(src)]
    return out


def _prev(a, k):
    """a[x - e_k], zero before the box."""
    ax = AX[k]
    out = np.zeros_like(a)
    src = [slice(None)] * a.ndim
    dst = [slice(None)] * a.ndim
    src[ax] = slice(0, -1)
    dst[ax] = slice(1, None)
    out[tuple(dst)] = a[tuple(src)]
    return out


def edge(om, k):
    """[x in Omega and x + e_k in Omega]: the forward difference along k exists at x."""
    return om & _next(om, k)


def dplus(w, om, k):
    m = edge(om, k)
    return np.where(m, _next(w, k) - w, 0.0)


def dminus(w, om, k):
    m = edge(om, k)
    a = np.where(m, w, 0.0)
    return np.where(om, a - _prev(a, k), 0.0)


def grad(u, om):
    return np.stack([dplus(u, om, k) for k in range(3)])


def symgrad(v, om):
    e = np.zeros((6,) + v.shape[1:])
    for k in range(3):
        for l in range(k, 3):
            e[QIDX[k][l]] = 0.5 * (dminus(v[k], om, l) + dminus(v[l], om, k))
    return e


def div(p, om):
    return dminus(p[0], om, 0) + dminus(p[1], om, 1) + dminus(p[2], om, 2)


def div2(q, om):
    out = np.zeros((3,) + q.shape[1:])
    for k in range(3):
        out[k] = dplus(q[QIDX[k][0]], om, 0) + dplus(q[QIDX[k][1]], om, 1) + dplus(q[QIDX[k][2]], om, 2)
    return out


def data_term(h, c, lam, u):
    """lambda sum_b h_b |u - c_b| (readings R1-R3); h [..., nb]."""
    return lam * np.sum(h * np.abs(u[..., None] - c), axis=-1)


def prox(ut, t, h, c):
    """argmin_{u in [-1, 1]} 1/2 (u - ut)^2 + t sum_b h_b |u - c_b|, elementwise.
    Same plain definition as oracle_prox (oracle/tgv_oracle.c): the objective is a
    convex quadratic on each interval between breakpoints; minimise each piece, clip
    to its interval, keep the best (first on ties)."""
    nb = len(c)
    best_u = np.zeros_like(ut)
    best_f = np.full_like(ut, np.inf)
    for j in range(nb + 1):
        lo = -1.0 if j == 0 else max(c[j - 1], -1.0)
        hi = 1.0 if j == nb else min(c[j], 1.0)
        if lo > hi:
            continue
        below = h[..., :j].sum(-1)
        above = h[..., j:].sum(-1)
        s = np.clip(ut - t * (below - above), lo, hi)
        f = 0.5 * (s - ut) ** 2 + t * np.sum(h * np.abs(s[..., None] - c), axis=-1)
        better = f < best_f
        best_u = np.where(better, s, best_u)
        best_f = np.where(better, f, best_f)
    return best_u


def proj(x, a, n2):
    """x / max(1, |x| / a) with |x|^2 = n2 (reading R5)."""
    n = np.sqrt(n2)
    return x * np.where(n > a, a / np.where(n > 0, n, 1.0), 1.0)


class BrickOracle:
    """fp64 state of one block-sparse level (R24).

    coords [nbricks, 3] integer brick coordinates (bx, by, bz); frozen [nbricks] bool
    (True = set B).  Arrays exchanged with the caller are brick-major:
    u [nbricks, E, E, E] (z, y, x inside a brick), v [nbricks, 3, E, E, E],
    counts [nbricks, E, E, E, nbins]."""

    def __init__(self, edge_, coords, frozen=None, lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25,
                 centers=None, V=2.0):
        self.E = int(edge_)
        self.coords = np.asarray(coords, dtype=np.int64).reshape(-1, 3)
        nbk = len(self.coords)
        if len({tuple(c) for c in self.coords}) != nbk:
            raise ValueError("duplicate brick coordinates")
        self.frozen = np.zeros(nbk, bool) if frozen is None else np.asarray(frozen, bool).reshape(nbk)
        self.c = default_centers(8) if centers is None else np.asarray(centers, np.float64)
        self.lam, self.alpha0, self.alpha1, self.tau, self.sigma, self.V = lam, alpha0, alpha1, tau, sigma, V
        self.lo = self.coords.min(0)
        ext = (self.coords.max(0) - self.lo + 1) * self.E  # (x, y, z) extents of the bounding box
        self.box = (int(ext[2]), int(ext[1]), int(ext[0]))  # [z, y, x]
        self.om = np.zeros(self.box, bool)
        self.act = np.zeros(self.box, bool)
        for b in range(nbk):
            self.om[self._sl(b)] = True
            self.act[self._sl(b)] = not self.frozen[b]
        # S = A + the frozen voxels with a face neighbour in A
        near = np.zeros(self.box, bool)
        for k in range(3):
            near |= _next(self.act, k) | _prev(self.act, k)
        self.S = self.act | (self.om & near)
        z = lambda *lead: np.zeros(lead + self.box)  # noqa: E731
        self.u, self.ubar = z(), z()
        self.v, self.vbar, self.p, self.q = z(3), z(3), z(3), z(6)
        self.h = np.zeros(self.box + (len(self.c),))

    def _sl(self, b):
        o = (self.coords[b] - self.lo) * self.E
        E = self.E
        return (slice(o[2], o[2] + E), slice(o[1], o[1] + E), slice(o[0], o[0] + E))

    # ---- brick-major <-> dense box
    def _scatter(self, dst, src, lead):
        for b in range(len(self.coords)):
            dst[(Ellipsis,) + self._sl(b)] = src[b] if lead == 0 else src[b].reshape((lead,) + (self.E,) * 3)

    def _gather(self, src, lead):
        shp = (len(self.coords),) + ((lead,) if lead else ()) + (self.E,) * 3
        out = np.zeros(shp)
        for b in range(len(self.coords)):
            out[b] = src[(Ellipsis,) + self._sl(b)]
        return out

    def load(self, counts):
        """Histograms of the bricks (frozen bricks' entries are ignored) and the
        initialisation of reading R9 on A; B holds 0 until set_primal."""
        counts = np.asarray(counts, dtype=np.float64).reshape((len(self.coords),) + (self.E,) * 3 + (len(self.c),))
        self.h[:] = 0.0
        for b in range(len(self.coords)):
            if not self.frozen[b]:
                self.h[self._sl(b)] = counts[b]
        W = self.h.sum(-1)
        m = np.sum(self.h * self.c, axis=-1)
        u0 = np.where(W > 0, m / np.where(W > 0, W, 1.0), 0.0)
        self.u = np.where(self.act, u0, 0.0)
        self.ubar = self.u.copy()
        self.v[:] = 0.0
        self.vbar[:] = 0.0
        self.p[:] = 0.0
        self.q[:] = 0.0
        return self

    def set_primal(self, u, v=None):
        """u, v on every brick (A and B), a restart: ubar = u, vbar = v, p = q = 0
        (the prolongation restart of reading R19; B keeps these values frozen)."""
        self._scatter(self.u, np.asarray(u, np.float64), 0)
        self.v[:] = 0.0
        if v is not None:
            self._scatter(self.v, np.asarray(v, np.float64), 3)
        self.ubar = self.u.copy()
        self.vbar = self.v.copy()
        self.p[:] = 0.0
        self.q[:] = 0.0
        return self

    def dual(self):
        """(a1) on the voxels of S: p <- P_a1(p + s(grad ubar - vbar)), q <- P_a0(q + s E(vbar));
        the operators still see every voxel of Omega (the frozen values around S)."""
        om = self.om
        pn = self.p + self.sigma * (grad(self.ubar, om) - self.vbar)
        pn = proj(pn, self.alpha1, pn[0] ** 2 + pn[1] ** 2 + pn[2] ** 2)
        qn = self.q + self.sigma * symgrad(self.vbar, om)
        n2 = qn[0] ** 2 + qn[1] ** 2 + qn[2] ** 2 + 2.0 * (qn[3] ** 2 + qn[4] ** 2 + qn[5] ** 2)
        qn = proj(qn, self.alpha0, n2)
        self.p = np.where(self.S, pn, 0.0)
        self.q = np.where(self.S, qn, 0.0)

    def primal(self):
        """(a2) + (a3) on A: u+ = clamp(prox(u + t div p)), v+ = v + t(p + div2 q),
        ubar = 2u+ - u, vbar = 2v+ - v; B unchanged (ubar = u, vbar = v)."""
        om, A = self.om, self.act
        un = prox(self.u + self.tau * div(self.p, om), self.tau * self.lam, self.h, self.c)
        vn = self.v + self.tau * (self.p + div2(self.q, om))
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

    def get(self, name):
        a = getattr(self, name)
        return self._gather(a, 0 if a.ndim == 3 else a.shape[0])

    def energy(self):
        """{E, alpha1, alpha0, data, gap, vmax, dual}: regulariser over S, data over A,
        restricted dual D_V of the module docstring, vmax over A."""
        om, A = self.om, self.act
        a = grad(self.u, om) - self.v
        t1 = self.alpha1 * np.sqrt(a[0] ** 2 + a[1] ** 2 + a[2] ** 2)
        e = symgrad(self.v, om)
        t0 = self.alpha0 * np.sqrt(e[0] ** 2 + e[1] ** 2 + e[2] ** 2 + 2.0 * (e[3] ** 2 + e[4] ** 2 + e[5] ** 2))
        td = data_term(self.h, self.c, self.lam, self.u)
        d = div(self.p, om)
        w = self.p + div2(self.q, om)
        cand = [-1.0] + list(self.c) + [1.0]
        best = np.min(np.stack([data_term(self.h, self.c, self.lam, np.full(self.box, uu)) - uu * d for uu in cand]),
                      axis=0)
        dA = best - self.V * (np.abs(w[0]) + np.abs(w[1]) + np.abs(w[2]))
        dB = -self.u * d - (self.v[0] * w[0] + self.v[1] * w[1] + self.v[2] * w[2])
        T1, T0 = float(np.sum(t1[self.S])), float(np.sum(t0[self.S]))
        TD = float(np.sum(td[A]))
        D = float(np.sum(dA[A]) + np.sum(dB[om & ~A]))
        E = T1 + T0 + TD
        vmax = float(np.max(np.abs(self.v[:, A]))) if A.any() else 0.0
        return {"E": E, "alpha1": T1, "alpha0": T0, "data": TD, "gap": E - D, "vmax": vmax, "dual": D}


# ---------------------------------------------------------------------------
# Level companions on brick sets (R24 with R18-R22)
# ---------------------------------------------------------------------------
def vote(coords, E, cams, depths, grid_origin=(0.0, 0.0, 0.0), voxel_size=1.0, r=0.5):
    """Alg. 1 counts of every brick: the oracle's dense vote of the
    brick's box, voxel (x, y, z) of brick (bx, by, bz) at grid_origin + h (E b + (x, y, z)).
    The dense oracle places voxel x at origin + h x, so the brick's box is voted from
    origin + h E (bx, by, 0) with planes [E bz, E bz + E): identical coordinates whenever
    those sums are exact in fp64 (the tests use origins and voxel sizes that are)."""
    from . import alg1_vote
    out = []
    for bx, by, bz in np.asarray(coords, np.int64):
        o = (grid_origin[0] + voxel_size * E * bx, grid_origin[1] + voxel_size * E * by, grid_origin[2])
        out.append(alg1_vote(cams, depths, E, E, E * bz, E * bz + E, origin=o, voxel_size=voxel_size, r=r))
    return np.stack(out)


def refine_flags(counts, frozen, min_votes):
    """flags [nbricks, 8]: octant o = (x >= E/2) + 2 (y >= E/2) + 4 (z >= E/2) of a solved
    brick holds a voxel with >= min_votes votes outside the last (free-space) bin."""
    c = np.asarray(counts)
    nb, E = c.shape[0], c.shape[1]
    surf = c[..., :-1].sum(-1) >= min_votes  # [nb, z, y, x]
    h = E // 2
    flags = np.zeros((nb, 8), np.uint8)
    for o in range(8):
        ox, oy, oz = o & 1, o >> 1 & 1, o >> 2
        blk = surf[:, oz * h:(oz + 1) * h, oy * h:(oy + 1) * h, ox * h:(ox + 1) * h]
        flags[:, o] = blk.reshape(nb, -1).any(1)
    flags[np.asarray(frozen, bool)] = 0
    return flags


def prolong(coarse, fine_coords):
    """Reading R19 on brick sets: fine voxel p of brick b takes u and v / 2 of the coarse
    voxel floor((E b + p) / 2), which lies in coarse brick floor(b / 2).
    coarse: BrickOracle; returns (u [nb, E, E, E], v [nb, 3, E, E, E]) fp64."""
    E = coarse.E
    cu, cv = coarse.get("u"), coarse.get("v")
    index = {tuple(int(a) for a in c): i for i, c in enumerate(coarse.coords)}
    fc = np.asarray(fine_coords, np.int64)
    u = np.zeros((len(fc), E, E, E))
    v = np.zeros((len(fc), 3, E, E, E))
    for i, (bx, by, bz) in enumerate(fc):
        pb = index[(int(bx) // 2, int(by) // 2, int(bz) // 2)]
        iz = (E * (bz % 2) + np.arange(E)) // 2
        iy = (E * (by % 2) + np.arange(E)) // 2
        ix = (E * (bx % 2) + np.arange(E)) // 2
        u[i] = cu[pb][np.ix_(iz, iy, ix)]
        for d in range(3):
            v[i, d] = 0.5 * cv[pb, d][np.ix_(iz, iy, ix)]
    return u, v
