"""The input generator: Alg. 1 conformance
and partition invariance of the generated histograms."""
import math

import numpy as np
import pytest

import synth


def test_alg1_bins():
    r = 0.5  # delta = 3, eta = 9 (PAPER.md:118 with r = h/2)
    assert synth.alg1_bin(10.0, 10.0, r) == 4            # a = 0 -> floor(0.5*8) = 4
    assert synth.alg1_bin(13.0, 10.0, r) == 7            # a = delta -> floor(8) = 8 -> clamped to 7
    assert synth.alg1_bin(100.0, 10.0, r) == 7           # far in front: clamp
    assert synth.alg1_bin(10.0, 13.0, r) == 0            # a = -delta -> bin 0
    assert synth.alg1_bin(10.0, 19.0, r) == 0            # a = -eta: still observed
    assert synth.alg1_bin(10.0, 19.0001, r) == -1        # a < -eta: no vote


def test_alg1_fuzz_matches_transliteration():
    rng = np.random.default_rng(0)
    for _ in range(20000):
        r = rng.uniform(0.1, 2.0)
        dep, dist = rng.uniform(0, 50), rng.uniform(0, 50)
        d, e = 6 * r, 18 * r
        a = dep - dist
        if a < -e:
            want = -1
        else:
            a = max(-1.0, min(1.0, a / d))
            want = min(int(math.floor((a + 1.0) / 2.0 * 8.0)), 7)
        assert synth.alg1_bin(dep, dist, r) == want


def test_c1_histograms_and_partition_invariance():
    full = synth.make_histograms("C1")
    assert full.shape == (32, 32, 32, 8) and full.dtype == np.uint32
    W = full.sum(-1)
    assert W.max() <= 16  # 16 cameras, vote weight 1
    assert 0.1 < (W == 0).mean() < 0.5
    # slabs generated independently equal the monolithic planes
    part = synth.make_histograms("C1", 5, 17)
    assert np.array_equal(part, full[5:17])
    # voxels on the sphere surface: of their near-surface votes (bins 1..6) most land in the
    # two central bins (|a| < delta/4); the rest are bin 0 (seen from behind) or 7
    c = 15.5
    z, y, x = np.meshgrid(np.arange(32), np.arange(32), np.arange(32), indexing="ij")
    rr = np.sqrt((x - c) ** 2 + (y - c) ** 2 + (z - c) ** 2)
    shell = np.abs(rr - 10.0) < 0.4
    assert full[shell][:, 3:5].sum() > full[shell][:, [1, 2, 5, 6]].sum()
    outside = rr > 14.0
    # free space: all votes in bin 7 except a few behind silhouettes (nearest-pixel lookup)
    assert full[outside][:, 7].sum() >= 0.999 * full[outside].sum()


def test_generator_is_seed_deterministic():
    wl = synth.workload("C1")
    d1 = synth.render_depths(wl)
    d2 = synth.render_depths(wl)
    for a, b in zip(d1, d2):
        assert np.array_equal(a, b, equal_nan=True)


def test_random_histograms_structure():
    h = synth.random_histograms((8, 7, 6), 0)
    assert h.shape == (6, 7, 8, 8)
    W = h.sum(-1)
    assert (W == 0).any() and ((h[..., 7] == W) & (W > 0)).any()


def test_vote_box_is_the_cropped_full_vote():
    """synth.vote_box (the golden windows of scripts/make_goldens.py) votes exactly the
    full-plane vote cropped to the box."""
    full = synth.make_histograms("C1", 3, 29)
    for box in [(2, 30, 5, 17, 3, 29), (0, 32, 0, 32, 10, 11), (31, 32, 0, 1, 3, 29)]:
        x0, x1, y0, y1, z0, z1 = box
        got = synth.make_histograms_box("C1", box)
        assert np.array_equal(got, full[z0 - 3:z1 - 3, y0:y1, x0:x1])
