"""Pins of the oracle's whole iteration (SURVEY.md §8(c) "Whole scheme").

* special cases with closed forms: zero histograms, constant histograms
  (weighted-median limit), 1x1x1 prox-point sequence (golden fixture);
* exact optimum: on 1x1xN grids the TGV-L1-histogram functional is a linear
  program; scipy's HiGHS solves it independently and the oracle's long-run
  energy must reach the LP optimum, with the restricted gap closing;
* 3-D behaviour (reading R15): restricted gap non-increasing on
  power-of-two checkpoints from 8, E(N) <= E(8), gap >= 0 while max|v| <= V;
* energy closed form for u = 0, constant v;
* u in [-1, 1]; thread-count invariance (Jacobi sweeps).
"""
import json
import os

import numpy as np
import pytest
from scipy.optimize import linprog

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
C = oracle.default_centers(8)


def test_zero_histograms_keep_u_zero():
    shape = (5, 4, 6)
    o = oracle.Oracle(shape).load(np.zeros((6, 4, 5, 8), np.uint32)).iterate(50)
    assert np.all(o.u == 0.0)
    assert np.all(o.get("v") == 0.0)


def test_constant_histograms_reach_weighted_median():
    # h = [3,0,1,0,0,2,5,1]: W = 12, cumulative counts 3,3,4,4,4,6 -> the median
    # interval is [c_5, c_6] = [0.375, 0.625]; u0 = 1.75/12 lies below it, so the
    # prox-point iteration stops at its left end 0.375.
    h = np.array([3, 0, 1, 0, 0, 2, 5, 1], np.uint32)
    shape = (4, 3, 5)
    counts = np.broadcast_to(h, (5, 3, 4, 8)).copy()
    o = oracle.Oracle(shape).load(counts)
    np.testing.assert_allclose(o.u, 1.75 / 12, rtol=0, atol=1e-15)
    o.iterate(3)
    assert np.all(o.u == 0.375)
    o.iterate(40)
    assert np.all(o.u == 0.375)
    assert np.all(o.get("v") == 0.0) and np.all(o.get("p") == 0.0)


def test_even_split_stays_at_projection_onto_median_interval():
    # h = e_2 + e_5: median interval [c_2, c_5] = [-0.375, 0.375]; u0 = 0 inside it
    h = np.zeros(8, np.uint32)
    h[2] = h[5] = 4
    counts = np.broadcast_to(h, (3, 3, 3, 8)).copy()
    o = oracle.Oracle((3, 3, 3)).load(counts).iterate(30)
    assert np.all(o.u == 0.0)


def test_prox_point_sequence_1x1x1_golden():
    g = json.load(open(os.path.join(GOLD, "prox_point_1x1x1.json")))
    counts = np.array(g["counts"], np.uint32).reshape(1, 1, 1, 8)
    o = oracle.Oracle((1, 1, 1), lam=g["lambda"], alpha0=g["alpha0"], alpha1=g["alpha1"], tau=g["tau"],
                      sigma=g["sigma"]).load(counts)
    seq = [float(o.u.ravel()[0])]
    for _ in range(len(g["u_after_k_iterations_numerator_over_24"]) - 1):
        o.iterate(1)
        seq.append(float(o.u.ravel()[0]))
    np.testing.assert_allclose(seq, np.array(g["u_after_k_iterations_numerator_over_24"]) / 24.0, rtol=0, atol=1e-15)


# ---------------------------------------------------------------------------
# exact LP optimum on 1x1xN grids
# ---------------------------------------------------------------------------
def lp_optimum_1d(h, lam, alpha0, alpha1, c):
    """min over u in [-1,1]^N, w in R^N of
         alpha1 sum_i |(D+ u)_i - w_i| + alpha0 sum_i |(D- w)_i| + lam sum_ib h_ib |u_i - c_b|
    (the 1x1xN reduction: v_x = v_y = 0 at the optimum).  Variables
    x = [u (N), w (N), a (N), b (N), d (N*nb)]."""
    N, nb = h.shape
    nv = 4 * N + N * nb
    iu, iw, ia, ib, idd = 0, N, 2 * N, 3 * N, 4 * N
    cost = np.zeros(nv)
    cost[ia:ia + N] = alpha1
    cost[ib:ib + N] = alpha0
    cost[idd:] = lam * h.reshape(-1)
    rows, rhs = [], []

    def add(coefs, r):
        row = np.zeros(nv)
        for k, val in coefs:
            row[k] += val
        rows.append(row)
        rhs.append(r)

    for i in range(N):
        # D+ u_i = u_{i+1} - u_i (i < N-1), 0 at N-1
        dp = [(iu + i + 1, 1.0), (iu + i, -1.0)] if i < N - 1 else []
        e = dp + [(iw + i, -1.0)]
        add(e + [(ia + i, -1.0)], 0.0)
        add([(k, -v) for k, v in e] + [(ia + i, -1.0)], 0.0)
        # D- w_i = wt_i - wt_{i-1}, wt_m = w_m for m < N-1 else 0
        dm = []
        if i < N - 1:
            dm.append((iw + i, 1.0))
        if i > 0:
            dm.append((iw + i - 1, -1.0))
        add(dm + [(ib + i, -1.0)], 0.0)
        add([(k, -v) for k, v in dm] + [(ib + i, -1.0)], 0.0)
        for b in range(nb):
            add([(iu + i, 1.0), (idd + i * nb + b, -1.0)], c[b])
            add([(iu + i, -1.0), (idd + i * nb + b, -1.0)], -c[b])
    bounds = [(-1, 1)] * N + [(None, None)] * N + [(0, None)] * (2 * N + N * nb)
    res = linprog(cost, A_ub=np.array(rows), b_ub=np.array(rhs), bounds=bounds, method="highs")
    assert res.status == 0
    return res.fun, res.x[:N]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_1d_energy_reaches_lp_optimum(seed):
    N = 12
    rng = np.random.default_rng(seed)
    h = np.zeros((N, 8), np.uint32)
    # a 1-D slab: votes at -1 on one side, +1 on the other, noisy transition
    for i in range(N):
        if i < N // 2 - 1:
            h[i, 0] = rng.integers(1, 4)
        elif i > N // 2:
            h[i, 7] = rng.integers(1, 4)
        h[i] += rng.integers(0, 2, size=8).astype(np.uint32) * (rng.uniform(size=8) < 0.3)
    lam, a0, a1 = 0.5, 2.0, 1.0
    Estar, _ = lp_optimum_1d(h.astype(np.float64), lam, a0, a1, C)
    o = oracle.Oracle((1, 1, N), lam=lam, alpha0=a0, alpha1=a1).load(h.reshape(N, 1, 1, 8))
    o.iterate(20000)
    e = o.energy()
    assert abs(e["E"] - Estar) <= 1e-8 * abs(Estar), (e["E"], Estar)
    assert -1e-9 * Estar <= e["gap"] <= 1e-6 * Estar
    u = o.u.ravel()
    assert u[0] < 0 < u[-1]


# ---------------------------------------------------------------------------
# 3-D behaviour (reading R15)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(6))
def test_gap_nonincreasing_on_checkpoints(seed):
    shape = (6, 5, 4)
    o = oracle.Oracle(shape).load(synth.random_histograms(shape, seed))
    it, gaps, Es = 0, [], []
    for ck in [8, 16, 32, 64, 128, 256, 512]:
        o.iterate(ck - it)
        it = ck
        e = o.energy()
        gaps.append(e["gap"])
        Es.append(e["E"])
        assert e["vmax"] <= 2.0
        assert e["gap"] >= -1e-9 * e["E"]
        assert np.all(np.abs(o.u) <= 1.0)
    assert np.all(np.diff(gaps) <= 0.0), gaps
    assert Es[-1] <= Es[0]
    assert gaps[-1] <= 1e-2 * Es[-1]


def test_energy_closed_form_constant_v():
    # u = 0, v = (a, 0, 0), h = 0 on an n^3 grid (n >= 2):
    #   alpha1 term = alpha1 n^3 |a|
    #   E(v): E_xx = a at x=0, -a at x=n-1; E_xy = +-a/2 on y-boundary planes;
    #         E_xz = +-a/2 on z-boundary planes  ->  |E v|_F^2 = a^2 (bx + by/2 + bz/2)
    #   where bk = 1 on the two boundary planes of axis k; D_V with p = q = 0 is 0.
    n, a = 5, 0.3
    o = oracle.Oracle((n, n, n), alpha0=2.0, alpha1=1.0).load(np.zeros((n, n, n, 8), np.uint32))
    v = np.zeros((3, n, n, n))
    v[0] = a
    o.set("v", v)
    e = o.energy()
    cnt = {0: n - 2, 1: 2}
    s = sum(cnt[bx] * cnt[by] * cnt[bz] * np.sqrt(bx + by / 2 + bz / 2)
            for bx in (0, 1) for by in (0, 1) for bz in (0, 1))
    assert abs(e["alpha1"] - 1.0 * n ** 3 * a) < 1e-12
    assert abs(e["alpha0"] - 2.0 * a * s) < 1e-12
    assert e["data"] == 0.0 and e["dual"] == 0.0
    assert abs(e["vmax"] - a) < 1e-15


def test_energy_data_term_closed_form():
    # u = u0 = weighted mean; v = 0; only the data term and the alpha1 |grad u| term
    h = np.array([1, 0, 0, 2, 0, 0, 0, 1], np.uint32)
    counts = np.broadcast_to(h, (2, 2, 2, 8)).copy()
    o = oracle.Oracle((2, 2, 2), lam=0.5).load(counts)
    u0 = (-0.875 - 0.25 + 0.875) / 4
    e = o.energy()
    expect = 8 * 0.5 * (abs(u0 + 0.875) + 2 * abs(u0 + 0.125) + abs(u0 - 0.875))
    assert abs(e["data"] - expect) < 1e-14
    assert e["alpha1"] == 0.0 and e["alpha0"] == 0.0


def test_thread_count_invariance_and_range():
    shape = (12, 10, 9)
    h = synth.random_histograms(shape, 5)
    a = oracle.Oracle(shape).load(h).iterate(30, threads=1)
    b = oracle.Oracle(shape).load(h).iterate(30, threads=4)
    for f in ("u", "v", "p", "q", "ubar", "vbar"):
        assert np.array_equal(a.get(f), b.get(f)), f
    assert np.all(np.abs(a.u) <= 1.0)


@pytest.mark.parametrize("shape", [(1, 1, 24), (6, 5, 24)])
def test_opposite_votes_give_a_jump_with_closed_form_energy(shape):
    """SPEC.md:346 idea ("a slab with strong bin votes at -1 on one side and +1 on the
    other -> a monotone transition crossing 0; energy at 200 within 1 % of a long run";
    E(200) <= E(10), :347).  With 3 votes per voxel (data slope lambda * 3 = 1.5 > alpha1)
    the minimiser is the step u = c_0 below the middle, c_7 above, v = 0, so
    E* = alpha1 |c_7 - c_0| per column = 1.75 nx ny (TV of one jump, no data cost)."""
    nx, ny, nz = shape
    h = np.zeros((nz, ny, nx, 8), np.uint32)
    h[:nz // 2, ..., 0] = 3
    h[nz // 2:, ..., 7] = 3
    energies = {}
    for n in (10, 200, 5000):
        o = oracle.Oracle(shape).load(h).iterate(n)
        energies[n] = o.energy()["E"]
    u = o.u
    assert abs(energies[5000] - 1.75 * nx * ny) <= 1e-9 * 1.75 * nx * ny
    assert np.max(np.abs(u[:nz // 2] + 0.875)) <= 1e-9 and np.max(np.abs(u[nz // 2:] - 0.875)) <= 1e-9
    assert np.all(np.diff(u, axis=0) >= -1e-12)  # monotone along z, crossing 0 between the halves
    assert energies[200] <= 1.01 * energies[5000]
    assert energies[200] <= energies[10]
