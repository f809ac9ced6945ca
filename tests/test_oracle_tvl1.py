"""Pins of the oracle's NEXT-4 TV-L1 model (Eq. 1; R21)."""
import numpy as np
from scipy.optimize import linprog

import oracle
import synth

C = oracle.default_centers(8)


def lp_tvl1_1d(h, lam, alpha1, c):
    """min_{u in [-1,1]^N} alpha1 sum |D+ u| + lam sum_ib h_ib |u_i - c_b| as an LP."""
    N, nb = h.shape
    nv = 2 * N + N * nb
    cost = np.zeros(nv)
    cost[N:2 * N] = alpha1
    cost[2 * N:] = lam * h.reshape(-1)
    A, b = [], []
    for i in range(N):
        for sgn in (1, -1):
            row = np.zeros(nv)
            if i < N - 1:
                row[i + 1] += sgn
                row[i] -= sgn
            row[N + i] = -1
            A.append(row)
            b.append(0)
        for k in range(nb):
            for sgn in (1, -1):
                row = np.zeros(nv)
                row[i] = sgn
                row[2 * N + i * nb + k] = -1
                A.append(row)
                b.append(sgn * c[k])
    res = linprog(cost, A_ub=np.array(A), b_ub=np.array(b),
                  bounds=[(-1, 1)] * N + [(0, None)] * (N + N * nb), method="highs")
    return res.fun


def test_tvl1_1d_reaches_lp_optimum():
    N = 14
    rng = np.random.default_rng(8)
    h = rng.integers(0, 4, size=(N, 8)).astype(np.uint32) * (rng.uniform(size=(N, 8)) < 0.35)
    h[: N // 2, 0] += 2
    h[N // 2:, 7] += 2
    Estar = lp_tvl1_1d(h.astype(float), 0.5, 1.0, C)
    o = oracle.Oracle((1, 1, N), model="tvl1").load(h.reshape(N, 1, 1, 8)).iterate(20000)
    e = o.energy()
    assert abs(e["E"] - Estar) <= 1e-8 * Estar
    assert -1e-9 * Estar <= e["gap"] <= 1e-6 * Estar
    assert e["alpha0"] == 0.0 and e["vmax"] == 0.0


def test_tvl1_keeps_v_q_zero_and_differs_from_tgv():
    shape = (9, 8, 7)
    h = synth.random_histograms(shape, 2)
    t = oracle.Oracle(shape, model="tvl1").load(h).iterate(40)
    assert np.all(t.get("v") == 0) and np.all(t.get("q") == 0)
    g = oracle.Oracle(shape).load(h).iterate(40)
    assert np.max(np.abs(t.u - g.u)) > 1e-3


def test_tvl1_gap_nonincreasing_on_checkpoints():
    shape = (6, 5, 4)
    o = oracle.Oracle(shape, model="tvl1").load(synth.random_histograms(shape, 4))
    it, gaps = 0, []
    for ck in (8, 16, 32, 64, 128, 256):
        o.iterate(ck - it)
        it = ck
        gaps.append(o.energy()["gap"])
    assert np.all(np.diff(gaps) <= 0) and gaps[-1] >= -1e-12
