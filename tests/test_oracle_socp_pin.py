"""Pin of the whole 3-D scheme to the minimum of the functional found by an independent
optimiser (DESIGN.md §3 "whole scheme, 3-D").

The TGV-hist functional of Eq. 2 with the readings R1-R8 (PAPER.md:150-157, :239-240,
:130-131) is a second-order-cone program: minimise
    sum_x alpha1 t1_x + alpha0 t0_x + lambda sum_b h_xb w_xb
subject to t1_x >= |(grad u - v)_x|_2, t0_x >= |E(v)_x|_F, w_xb >= |u_x - c_b|, -1 <= u <= 1.
scipy's SLSQP solves it on a tiny 3-D grid from the operators of the oracle (probed with
unit vectors; the operators themselves are pinned in test_oracle_operators.py), with no
part of the primal-dual scheme (no prox, projection, step sizes or over-relaxation).
The oracle's iterate after 20 000 Chambolle-Pock iterations must reach the same minimum
value; the minimiser itself need not be unique (L1 data term), the value is.
"""
import numpy as np
import pytest
from scipy.optimize import minimize

import oracle

KW = dict(lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25)


def _socp_minimum(shape, h, lam=0.5, alpha0=2.0, alpha1=1.0):
    nx, ny, nz = shape
    n = nx * ny * nz
    c = oracle.default_centers(8)
    G = np.zeros((3 * n, n))
    Es = np.zeros((6 * n, 3 * n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        G[:, j] = oracle.grad(e.reshape(nz, ny, nx)).reshape(-1)
    for j in range(3 * n):
        e = np.zeros(3 * n)
        e[j] = 1.0
        Es[:, j] = oracle.symgrad(e.reshape(3, nz, ny, nx)).reshape(-1)
    Wf = np.array([1, 1, 1, 2, 2, 2.0])[:, None]  # Frobenius weights of xx yy zz xy xz yz (R5)
    H = h.reshape(n, 8).astype(np.float64)

    def split(z):
        u, v = z[:n], z[n:4 * n]
        t1, t0 = z[4 * n:5 * n], z[5 * n:6 * n]
        return u, v, t1, t0, z[6 * n:].reshape(n, 8)

    def obj(z):
        _, _, t1, t0, w = split(z)
        return alpha1 * t1.sum() + alpha0 * t0.sum() + lam * (H * w).sum()

    def cons(z):
        u, v, t1, t0, w = split(z)
        g = (G @ u - v).reshape(3, n)
        e = (Es @ v).reshape(6, n)
        d = u[:, None] - c[None, :]
        return np.concatenate([t1 - np.sqrt((g ** 2).sum(0) + 1e-18), t0 - np.sqrt((Wf * e ** 2).sum(0) + 1e-18),
                               (w - d).ravel(), (w + d).ravel()])

    u0 = np.zeros(n)
    z0 = np.concatenate([u0, np.zeros(3 * n), np.full(n, 3.0), np.full(n, 3.0), (np.abs(u0[:, None] - c) + 1).ravel()])
    bounds = [(-1.0, 1.0)] * n + [(None, None)] * (13 * n)
    r = minimize(obj, z0, method="SLSQP", constraints=[{"type": "ineq", "fun": cons}], bounds=bounds,
                 options={"maxiter": 3000, "ftol": 1e-15})
    # the functional at SLSQP's (u, v) itself (its epigraph variables may violate their
    # constraints by the solver's tolerance): an upper bound of the minimum
    u, v, _, _, _ = split(r.x)
    u = np.clip(u, -1.0, 1.0)
    g = (G @ u - v).reshape(3, n)
    e = (Es @ v).reshape(6, n)
    return (alpha1 * np.sqrt((g ** 2).sum(0)).sum() + alpha0 * np.sqrt((Wf * e ** 2).sum(0)).sum()
            + lam * (H * np.abs(u[:, None] - c[None, :])).sum())


@pytest.mark.parametrize("shape,seed", [((2, 2, 2), 3), ((1, 2, 3), 4)])
def test_scheme_reaches_the_socp_minimum_in_3d(shape, seed):
    rng = np.random.default_rng(seed)
    nx, ny, nz = shape
    h = rng.integers(0, 4, (nz, ny, nx, 8)).astype(np.uint32)
    f_socp = _socp_minimum(shape, h)
    o = oracle.Oracle(shape, **KW).load(h).iterate(20000)
    en = o.energy()
    # the scheme's value is no worse than the independent optimiser's point, and within
    # 1e-6 of it (SLSQP's own accuracy on this non-smooth cone program)
    assert en["E"] <= f_socp + 1e-9 * f_socp, (en["E"], f_socp)
    assert en["E"] >= f_socp - 1e-6 * f_socp, (en["E"], f_socp)
    assert en["gap"] <= 1e-7 * en["E"]
