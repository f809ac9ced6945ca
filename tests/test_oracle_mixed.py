"""Pins of the 2:1 mixed-level brick oracle (oracle/mixed.py; reading R27;
PAPER.md:221-225 "4 or less neighbors over each face", :446-453 frozen parent cubes).

Each pin is something other than the oracle's own formula:
  * a one-level set is the (independently pinned) block-sparse oracle of R24 bit for bit;
  * D+ of a linear field: exact on same-level and coarse-to-fine faces (the mean of the
    four fine centres sits on the coarse voxel's axis), exact along k on fine-to-coarse
    faces for fields that vary along k only -- a wrong distance or weight fails it;
  * D- written out case by case by hand (the weighted adjoint of each kind of face)
    equals the oracle's -H^-1 (D+)^T H;
  * ||K||^2 < 16 on mixed sets (the step-size bound of R7 carries over);
  * the scheme reaches the minimum of the weighted functional found by SLSQP on the
    second-order-cone form, on a 9-cell set with faces of both kinds;
  * 2:1 violations and overlaps are rejected; the gap closes on a set with frozen bricks.
"""
import numpy as np
import pytest
from scipy.optimize import minimize

from oracle import bricks as ob
from oracle import mixed as om

KW = dict(lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25)


def two_level_set():
    """E = 4: one level-1 brick with level-0 bricks across its +x, -y and +z faces (the
    four fine bricks that tile each face), and a same-level fine neighbour chain; some
    frozen.  Coordinates in each brick's own level units."""
    levels, coords = [1], [(1, 1, 1)]  # coarse brick: fine units [8, 16)^3 (E = 4, h = 2)
    for a in (0, 1):
        for b in (0, 1):
            levels.append(0)
            coords.append((4, 2 + a, 2 + b))  # +x face of the coarse brick (fine x in [16, 20))
            levels.append(0)
            coords.append((2 + a, 1, 2 + b))  # -y face (fine y in [4, 8))
            levels.append(0)
            coords.append((2 + a, 2 + b, 4))  # +z face
    levels.append(0)
    coords.append((5, 2, 2))  # same-level neighbour of a fine brick
    levels.append(1)
    coords.append((1, 1, 0))  # a coarse neighbour below (-z) of the coarse brick
    return np.array(levels), np.array(coords)


def test_one_level_set_is_the_brick_oracle():
    rng = np.random.default_rng(1)
    E = 4
    coords = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 0, 1), (2, 1, 0), (1, 1, 1)])
    frozen = np.array([0, 1, 0, 0, 1, 0], bool)
    h = rng.integers(0, 5, (len(coords), E, E, E, 8))
    a = ob.BrickOracle(E, coords, frozen, **KW).load(h)
    b = om.MixedOracle(E, np.zeros(len(coords), int), coords, frozen, **KW).load(h)
    u0 = rng.uniform(-1, 1, (len(coords), E, E, E))
    v0 = rng.normal(0, 0.3, (len(coords), 3, E, E, E))
    a.set_primal(u0, v0)
    b.set_primal(u0, v0)
    a.iterate(25)
    b.iterate(25)
    for f in ("u", "v", "p", "q"):
        np.testing.assert_allclose(b.get(f), a.get(f), rtol=0, atol=1e-12, err_msg=f)
    ea, eb = a.energy(), b.energy()
    for k in ("E", "alpha1", "alpha0", "data", "gap", "vmax"):
        assert abs(ea[k] - eb[k]) <= 1e-10 * max(1.0, abs(ea["E"])), k


def _centres(E, levels, coords):
    lo, lev = om._voxel_lo(E, levels, coords)
    h = 2.0 ** lev
    return (lo + 0.5) * h[:, None], lev


def test_forward_difference_of_linear_fields():
    E = 4
    levels, coords = two_level_set()
    x, lev = _centres(E, levels, coords)
    nb = om.neighbours(E, levels, coords)
    D, _ = om.dplus_matrix(E, levels, coords, nb)
    a = np.array([0.3, -1.7, 2.2])
    u = x @ a
    seen = set()
    for k in range(3):
        kind, _ = nb[k]
        g = D[k] @ u
        exact = (kind == 1) | (kind == 3)
        np.testing.assert_allclose(g[exact], a[k], rtol=0, atol=1e-12)
        assert np.all(g[kind == 0] == 0.0)
        # fine -> coarse: exact for a field varying along k only
        gk = D[k] @ (x[:, k] * a[k])
        np.testing.assert_allclose(gk[kind == 2], a[k], rtol=0, atol=1e-12)
        seen |= set(int(t) for t in np.unique(kind))
    assert seen == {0, 1, 2, 3}  # every kind of face occurs


def test_backward_difference_written_out_by_hand():
    """D-_k p at voxel j = b_j p_j - (contributions of j's -k neighbours), by case:
    b_j = 1/h (same-level + neighbour), 1/(1.5 h) (coarser), 1/(0.75 h) (finer), 0 (none);
    a same-level -k neighbour i adds p_i / h, each of four finer ones p_i / (6 h)
    (weight h_i^3 / h_j^3 = 1/8 over its distance 0.75 h), a coarser one 4 p_i / (3 h)
    (weight 8, its share 1/4 over its distance 1.5 h)."""
    E = 4
    levels, coords = two_level_set()
    x, lev = _centres(E, levels, coords)
    h = 2.0 ** lev
    nb = om.neighbours(E, levels, coords)
    mo = om.MixedOracle(E, levels, coords, **KW)
    rng = np.random.default_rng(3)
    p = rng.normal(size=len(h))
    for k in range(3):
        kind, idx = nb[k]
        want = np.zeros(len(h))
        for j in range(len(h)):
            b = {0: 0.0, 1: 1.0 / h[j], 2: 1.0 / (1.5 * h[j]), 3: 1.0 / (0.75 * h[j])}[int(kind[j])]
            want[j] += b * p[j]
        for i in range(len(h)):  # i's + neighbours receive i's p
            if kind[i] == 1:
                j = idx[i, 0]
                want[j] -= p[i] / h[j]
            elif kind[i] == 2:  # i fine, j coarser: j has i among its 4 finer -k neighbours
                j = idx[i, 0]
                want[j] -= p[i] / (6.0 * h[j])
            elif kind[i] == 3:  # i coarse, its 4 finer + neighbours j
                for j in idx[i]:
                    want[j] -= 4.0 * p[i] / (3.0 * h[j])
        np.testing.assert_allclose(mo.Dm[k] @ p, want, rtol=0, atol=1e-13)


def test_operator_norm_below_the_step_bound():
    E = 4
    levels, coords = two_level_set()
    mo = om.MixedOracle(E, levels, coords, **KW)
    n2 = mo.op_norm2(iters=300)
    assert 12.0 < n2 < 16.0, n2


def test_unbalanced_and_overlapping_sets_are_rejected():
    with pytest.raises(ValueError):  # level 2 next to level 0
        om.MixedOracle(2, [2, 0], [(0, 0, 0), (4, 0, 0)])
    with pytest.raises(ValueError):  # overlap
        om.MixedOracle(2, [1, 0], [(0, 0, 0), (1, 1, 1)])
    with pytest.raises(ValueError):  # a coarse face only partly covered by finer voxels
        om.MixedOracle(1, [1, 0], [(0, 0, 0), (2, 0, 0)])


def _socp_minimum(mo, H, lam=0.5, alpha0=2.0, alpha1=1.0):
    """The weighted functional of R27 as a cone program, solved by SLSQP from the
    oracle's operator matrices (probed column by column), without the scheme."""
    n = len(mo.h)
    c = mo.c
    G = np.zeros((3 * n, n))
    Es = np.zeros((6 * n, 3 * n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        G[:, j] = mo.grad(e).reshape(-1)
    for j in range(3 * n):
        e = np.zeros(3 * n)
        e[j] = 1.0
        Es[:, j] = mo.symgrad(e.reshape(3, n)).reshape(-1)
    Wf = np.array([1, 1, 1, 2, 2, 2.0])[:, None]
    w = mo.w

    def split(z):
        return z[:n], z[n:4 * n], z[4 * n:5 * n], z[5 * n:6 * n], z[6 * n:].reshape(n, 8)

    def obj(z):
        _, _, t1, t0, ww = split(z)
        return np.sum(w * (alpha1 * t1 + alpha0 * t0 + lam * (H * ww).sum(1)))

    def cons(z):
        u, v, t1, t0, ww = split(z)
        g = (G @ u - v).reshape(3, n)
        e = (Es @ v).reshape(6, n)
        d = u[:, None] - c[None, :]
        return np.concatenate([t1 - np.sqrt((g ** 2).sum(0) + 1e-18), t0 - np.sqrt((Wf * e ** 2).sum(0) + 1e-18),
                               (ww - d).ravel(), (ww + d).ravel()])

    gobj = np.concatenate([np.zeros(4 * n), alpha1 * w, alpha0 * w, (lam * w[:, None] * H).ravel()])

    def cons_jac(z):  # analytic Jacobian of cons (rows: t1, t0, w - d, w + d; columns: u, v, t1, t0, w)
        u, v, t1, t0, ww = split(z)
        g = (G @ u - v).reshape(3, n)
        e = (Es @ v).reshape(6, n)
        ng = np.sqrt((g ** 2).sum(0) + 1e-18)
        ne = np.sqrt((Wf * e ** 2).sum(0) + 1e-18)
        J = np.zeros((18 * n, 14 * n))
        Gr = G.reshape(3, n, n)
        J[:n, :n] = -np.einsum("ki,kij->ij", g / ng, Gr)
        for k in range(3):
            J[np.arange(n), n + k * n + np.arange(n)] = g[k] / ng
        J[np.arange(n), 4 * n + np.arange(n)] = 1.0
        Er = Es.reshape(6, n, 3 * n)
        J[n:2 * n, n:4 * n] = -np.einsum("mi,mij->ij", Wf * e / ne, Er)
        J[n + np.arange(n), 5 * n + np.arange(n)] = 1.0
        rows = np.arange(8 * n)
        J[2 * n + rows, 6 * n + rows] = 1.0
        J[10 * n + rows, 6 * n + rows] = 1.0
        J[2 * n + rows, rows // 8] = -1.0
        J[10 * n + rows, rows // 8] = 1.0
        return J

    z0 = np.concatenate([np.zeros(4 * n), np.full(2 * n, 3.0), (np.abs(c)[None, :] + np.ones((n, 8))).ravel()])
    r = minimize(obj, z0, jac=lambda z: gobj, method="SLSQP",
                 constraints=[{"type": "ineq", "fun": cons, "jac": cons_jac}],
                 bounds=[(-1.0, 1.0)] * n + [(None, None)] * (13 * n), options={"maxiter": 4000, "ftol": 1e-15})
    u, v, _, _, _ = split(r.x)
    u = np.clip(u, -1.0, 1.0)
    g = (G @ u - v).reshape(3, n)
    e = (Es @ v).reshape(6, n)
    return float(np.sum(w * (alpha1 * np.sqrt((g ** 2).sum(0)) + alpha0 * np.sqrt((Wf * e ** 2).sum(0))
                             + lam * (H * np.abs(u[:, None] - c[None, :])).sum(1))))


def test_scheme_reaches_the_socp_minimum_on_a_mixed_set():
    # E = 1 (one voxel per brick): a level-1 cell at fine x [2, 4) with the four fine
    # cells that tile its -x face (fine -> coarse) and the four that tile its +x face
    # (coarse -> fine)
    levels = [1] + [0] * 8
    coords = [(1, 0, 0)] + [(1, y, z) for y in (0, 1) for z in (0, 1)] + [(4, y, z) for y in (0, 1) for z in (0, 1)]
    rng = np.random.default_rng(11)
    H = rng.integers(0, 4, (9, 8)).astype(np.float64)
    H[0] = [0, 0, 3, 0, 0, 0, 1, 0]
    mo = om.MixedOracle(1, levels, coords, **KW)
    assert mo.op_norm2() < 16.0
    f_socp = _socp_minimum(mo, H)
    mo.load(H.reshape(9, 1, 1, 1, 8)).iterate(20000)
    en = mo.energy()
    assert en["E"] <= f_socp + 1e-9 * f_socp, (en["E"], f_socp)
    assert en["E"] >= f_socp - 1e-6 * f_socp, (en["E"], f_socp)
    assert en["gap"] <= 1e-7 * en["E"]


def test_gap_closes_with_frozen_coarse_neighbours():
    """A fine part (solved) whose border cubes are frozen coarse parents (the paper's B,
    PAPER.md:446-453): the restricted gap of the weighted functional closes."""
    E = 2
    levels, coords = [], []
    for x in range(2):
        for y in range(2):
            for z in range(2):
                levels.append(0)
                coords.append((2 + x, 2 + y, 2 + z))  # the fine part: fine units [4, 8)^3
    for c in [(0, 1, 1), (3, 1, 1), (1, 0, 1), (1, 3, 1), (1, 1, 0), (1, 1, 3)]:
        levels.append(1)
        coords.append(c)  # coarse face neighbours, frozen
    frozen = np.array([False] * 8 + [True] * 6)
    rng = np.random.default_rng(5)
    h = rng.integers(0, 4, (14, E, E, E, 8))
    mo = om.MixedOracle(E, levels, coords, frozen, **KW).load(h)
    u0 = np.zeros((14, E, E, E))
    u0[8:] = rng.uniform(-1, 1, (6, 1, 1, 1))
    mo.set_primal(u0, np.zeros((14, 3, E, E, E)))
    assert mo.S.sum() > 8 * E ** 3  # frozen coarse voxels next to the part are in S
    e0 = mo.energy()
    mo.iterate(8000)
    e1 = mo.energy()
    assert e1["E"] < e0["E"]
    assert 0 <= e1["gap"] <= 1e-5 * e1["E"], e1
    np.testing.assert_array_equal(mo.get("u")[8:], u0[8:])  # B stays frozen
