"""Pins of the oracle's NEXT-1 coarse-to-fine pieces (R18-R20)."""
import numpy as np

import oracle
import synth


def test_restriction_conserves_votes_and_sums_children():
    h = synth.random_histograms((7, 6, 5), 3)  # odd and even extents
    c = oracle.restrict_counts(h)
    assert c.shape == (3, 3, 4, 8)
    assert np.array_equal(c.sum(axis=(0, 1, 2)), h.sum(axis=(0, 1, 2), dtype=np.uint64))
    # hand check: coarse (0,0,0) = the 8 fine voxels x,y,z in {0,1}; coarse x=3 (fine x=6) has only
    # children with x = 6 (nx = 7)
    assert np.array_equal(c[0, 0, 0], h[0:2, 0:2, 0:2].sum(axis=(0, 1, 2)))
    assert np.array_equal(c[2, 2, 3], h[4:5, 4:6, 6:7].sum(axis=(0, 1, 2)))


def test_prolongation_values():
    co = oracle.Oracle((2, 2, 2)).load(np.zeros((2, 2, 2, 8), np.uint32))
    co.set("u", np.arange(8, dtype=float).reshape(2, 2, 2) / 10)
    co.set("v", np.stack([np.full((2, 2, 2), 0.4), np.full((2, 2, 2), -0.2), np.zeros((2, 2, 2))]))
    fi = oracle.Oracle((3, 4, 3)).load(np.zeros((3, 4, 3, 8), np.uint32))
    oracle.prolong_into(fi, co)
    u = fi.get("u")
    assert u[2, 3, 2] == co.get("u")[1, 1, 1] and u[0, 1, 1] == co.get("u")[0, 0, 0]
    assert np.all(fi.get("v")[0] == 0.2) and np.all(fi.get("v")[1] == -0.1)
    assert np.array_equal(fi.get("ubar"), u) and np.array_equal(fi.get("vbar"), fi.get("v"))
    assert np.all(fi.get("p") == 0) and np.all(fi.get("q") == 0)


def test_coarse_to_fine_reaches_the_fine_optimum_1d():
    """A coarse start changes the path, not the limit: the 1x1xN LP optimum is still reached."""
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle_scheme import lp_optimum_1d
    N = 16
    rng = np.random.default_rng(5)
    h = np.zeros((N, 8), np.uint32)
    h[: N // 2, 0] = rng.integers(1, 4, N // 2)
    h[N // 2:, 7] = rng.integers(1, 4, N - N // 2)
    Estar, _ = lp_optimum_1d(h.astype(np.float64), 0.5, 2.0, 1.0, oracle.default_centers(8))
    o = oracle.coarse_to_fine((1, 1, N), h.reshape(N, 1, 1, 8), levels=3, iters=20000)
    assert abs(o.energy()["E"] - Estar) <= 1e-7 * Estar


def test_coarse_start_lowers_early_energy():
    """On the C1 sphere, 3 levels x 50 iterations end below a cold 50-iteration fine solve
    (the coarse-to-fine motivation)."""
    wl = synth.workload("C1")
    h = synth.make_histograms("C1")
    cold = oracle.Oracle(wl.shape).load(h).iterate(50, threads=oracle.max_threads()).energy()["E"]
    warm = oracle.coarse_to_fine(wl.shape, h, levels=3, iters=50, threads=oracle.max_threads()).energy()["E"]
    assert warm < cold
