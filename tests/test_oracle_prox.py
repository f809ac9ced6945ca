"""Pins of the oracle's histogram-L1 prox (SURVEY.md §8(c) "Prox (a2)").

oracle.prox(ut, t, h, c) = argmin_{u in [-1,1]} 1/2 (u-ut)^2 + t sum_b h_b |u-c_b|
(data term of Eq. 2, written through the histogram of §3.4,
PAPER.md:239-240; readings R1-R3, R8 in DESIGN.md).

The pins do not reuse the oracle's per-interval construction:
  * a dense grid search of the objective (step 1e-5);
  * the Li-Osher median formula of the EXPANDED multiset (each centre c_b
    repeated h_b times, plus the W+1 shifted points ut + t(W - 2k));
  * closed-form special cases.
"""
import numpy as np
import pytest

import oracle

C = oracle.default_centers(8)


def objective(u, ut, t, h, c):
    u = np.asarray(u)[..., None]
    return 0.5 * (u[..., 0] - ut) ** 2 + t * np.sum(h * np.abs(u - c), axis=-1)


def li_osher(ut, t, h, c):
    """Li & Osher median formula for prox of t*sum_i |u - f_i| over the multiset f."""
    f = np.repeat(c, h.astype(np.int64))
    W = len(f)
    shifted = ut + t * (W - 2.0 * np.arange(W + 1))
    allv = np.sort(np.concatenate([f, shifted]))
    med = allv[W]  # 2W+1 elements
    return min(1.0, max(-1.0, med))


def test_default_centers_are_bin_midpoints():
    # Alg. 1 bins a in [-1,1] into floor((a+1)/2*8): bin b covers [-1+b/4, -1+(b+1)/4)
    np.testing.assert_array_equal(C, [-0.875, -0.625, -0.375, -0.125, 0.125, 0.375, 0.625, 0.875])


def test_zero_histogram_is_clamp():
    h = np.zeros(8)
    for ut in [-3.0, -1.0, -0.3, 0.0, 0.7, 1.0, 2.5]:
        assert oracle.prox(ut, 0.2, h, C) == min(1.0, max(-1.0, ut))


@pytest.mark.parametrize("ut", [0.125, 0.0, 0.3, -0.2, 0.5])
def test_single_vote_in_bin4(ut):
    # hist = e_4, t >= |ut - 0.125| -> c_4 = 0.125
    h = np.zeros(8)
    h[4] = 1
    t = abs(ut - 0.125) + 0.01
    assert oracle.prox(ut, t, h, C) == 0.125
    # and a small step moves only by t towards c_4
    t = 0.5 * abs(ut - 0.125)
    if t > 0:
        expect = ut - t * np.sign(ut - 0.125)
        assert abs(oracle.prox(ut, t, h, C) - expect) < 1e-15


def test_grid_search():
    rng = np.random.default_rng(11)
    grid = np.linspace(-1.0, 1.0, 200001)
    for _ in range(300):
        ut = rng.uniform(-1.6, 1.6)
        t = rng.uniform(0.0, 0.4)
        h = rng.integers(0, 7, size=8).astype(np.float64)
        h[rng.uniform(size=8) < 0.4] = 0
        p = oracle.prox(ut, t, h, C)
        fg = objective(grid, ut, t, h, C)
        g = grid[np.argmin(fg)]
        assert abs(p - g) <= 1.0001e-5, (ut, t, h, p, g)
        # the oracle's point is no worse than the best grid point
        assert objective(np.array([p]), ut, t, h, C)[0] <= fg.min() + 1e-12


def test_li_osher_expanded_median():
    rng = np.random.default_rng(12)
    for _ in range(10000):
        ut = rng.uniform(-2.0, 2.0)
        t = rng.choice([0.0, 0.125, rng.uniform(0, 0.5)])
        h = rng.integers(0, 9, size=8)
        h[rng.uniform(size=8) < 0.5] = 0
        p = oracle.prox(ut, t, h.astype(np.float64), C)
        assert abs(p - li_osher(ut, t, h, C)) <= 1e-12, (ut, t, h)


def test_nonuniform_centres_and_nbins():
    rng = np.random.default_rng(13)
    for nb in [1, 2, 3, 5, 16]:
        for _ in range(300):
            c = np.sort(rng.uniform(-1, 1, size=nb))
            h = rng.integers(0, 5, size=nb)
            ut, t = rng.uniform(-1.5, 1.5), rng.uniform(0, 0.3)
            assert abs(oracle.prox(ut, t, h.astype(np.float64), c) - li_osher(ut, t, h, c)) <= 1e-12


def test_prox_is_monotone_and_nonexpansive():
    rng = np.random.default_rng(14)
    for _ in range(200):
        h = rng.integers(0, 6, size=8).astype(np.float64)
        t = rng.uniform(0, 0.3)
        uts = np.sort(rng.uniform(-1.5, 1.5, size=20))
        ps = np.array([oracle.prox(x, t, h, C) for x in uts])
        assert np.all(np.diff(ps) >= -1e-15)
        assert np.all(np.diff(ps) <= np.diff(uts) + 1e-15)
