"""Pins of the NEXT-3 leaf oracle (oracle.leaf_step / leaf_from_parent / out_of_core;
PAPER.md:446-458 §4.5 Fig. 9; R23).

- a degenerate partition (every level one leaf) is the in-core coarse-to-fine solve,
  bit for bit ("octree fitting in one group at all levels -> identical
  result to a monolithic in-core solve");
- one leaf iteration from a global state reproduces the global iteration on the
  leaf's planes bit for bit (the leaf's update of A is the scheme's own; only B
  differs, and B is read-only within one iteration);
- the indicator of B stays frozen bit for bit over many iterations (Fig. 9);
- with >= 8 leaves the solution stays close to the single-leaf solve: mean |du| <=
  0.05 and the same sign at >= 99% of the voxels (exact equality is not
  expected because borders freeze).
"""
import numpy as np

import oracle
import synth

KW = dict(lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25)


def test_single_leaf_partition_is_the_in_core_solve():
    shape = (13, 11, 10)
    h = synth.random_histograms(shape, 3)
    u, v = oracle.out_of_core(shape, h, levels=2, iters=20, leaf_voxels=10 ** 9, **KW)
    o = oracle.coarse_to_fine(shape, h, levels=2, iters=20, **KW)
    assert np.array_equal(u, o.u)
    assert np.array_equal(v, o.get("v"))


def test_one_leaf_iteration_is_the_global_iteration():
    shape = (9, 7, 12)
    h = synth.random_histograms(shape, 5)
    g = oracle.Oracle(shape, **KW).load(h).iterate(6)
    zb, ze = 4, 8
    leaf = oracle.Oracle(shape, zb=zb, ze=ze, **KW).load(h[zb:ze])
    for name in ("u", "ubar", "v", "vbar", "p", "q"):
        a = g.get(name)
        leaf.set(name, a[..., zb:ze, :, :])
        for comp in range(len(oracle.FIELDS[name])):
            for z in (zb - 1, ze):
                leaf.set_plane(name, comp, z, a[z] if a.ndim == 3 else a[comp, z])
    oracle.leaf_step(leaf)
    g.iterate(1)
    for name in ("u", "v", "p", "q", "ubar", "vbar"):
        assert np.array_equal(leaf.get(name), g.get(name)[..., zb:ze, :, :]), name
    # the border duals the leaf recomputed are the global ones
    for comp in range(3):
        assert np.array_equal(leaf.get_plane("p", comp, zb - 1), g.get("p")[comp, zb - 1])
    for comp in range(6):
        assert np.array_equal(leaf.get_plane("q", comp, ze), g.get("q")[comp, ze])


def test_border_indicator_stays_frozen():
    shape = (10, 9, 16)
    h = synth.random_histograms(shape, 7)
    cshape = tuple((n + 1) // 2 for n in shape)
    rng = np.random.default_rng(1)
    pu = rng.uniform(-1, 1, cshape[::-1])
    pv = rng.uniform(-0.3, 0.3, (3,) + cshape[::-1])
    zb, ze = 5, 11
    o = oracle.leaf_from_parent(shape, zb, ze, h[zb:ze], pu, pv, **KW)
    before = {(n, c, z): o.get_plane(n, c, z) for n in ("u", "ubar", "v", "vbar")
              for c in range(len(oracle.FIELDS[n])) for z in (zb - 1, ze)}
    u0 = o.u.copy()
    for _ in range(25):
        oracle.leaf_step(o)
    for key, plane in before.items():
        assert np.array_equal(o.get_plane(*key), plane), key
    # border values are the parents' (u) and half the parents' (v)
    assert np.array_equal(before[("u", 0, zb - 1)], np.repeat(np.repeat(pu[(zb - 1) // 2], 2, 0), 2, 1)[:9, :10])
    assert np.array_equal(before[("v", 2, ze)],
                          np.repeat(np.repeat(pv[2, ze // 2], 2, 0), 2, 1)[:9, :10] * 0.5)
    assert not np.array_equal(o.u, u0)  # A did move


def test_many_leaves_stay_close_to_the_single_leaf_solve():
    wl = synth.workload("C1")
    h = synth.make_histograms("C1")
    nx, ny, nz = wl.shape
    leaf_voxels = nx * ny * 2  # 16 leaves on the finest level, 2 on the next, 1 on the coarsest
    u, _ = oracle.out_of_core(wl.shape, h, levels=3, iters=200, leaf_voxels=leaf_voxels,
                              threads=oracle.max_threads(), **KW)
    ref = oracle.coarse_to_fine(wl.shape, h, levels=3, iters=200, threads=oracle.max_threads(), **KW).u
    assert np.mean(np.abs(u - ref)) <= 0.05
    assert np.mean(np.sign(u) == np.sign(ref)) >= 0.99
