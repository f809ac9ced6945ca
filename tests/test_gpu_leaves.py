"""NEXT-3 z-slab leaves with frozen borders on the GPU (R23;
PAPER.md:446-458 §4.5 Fig. 9).

- coarsened loading is bit-exact against the oracle's restriction (integers);
- tgv_prolong_slab of a whole grid equals tgv_prolong_from (bit for bit);
- one leaf iteration equals the slab group's iteration on the same planes, bit for
  bit (same arithmetic, same inputs);
- the out-of-core solve (16 leaves on the finest level) matches the oracle's
  out-of-core solve within the north-star tolerance;
- with >= 8 leaves it stays close to the in-core solve.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
C8 = [-0.875 + 0.25 * b for b in range(8)]


def test_coarsened_load_is_bit_exact():
    from paper_2107_14790_b200 import Solver
    shape = (37, 22, 19)
    h = synth.random_histograms(shape, 4)
    for factor in (1, 2, 4):
        ref = h
        for _ in range({1: 0, 2: 1, 4: 2}[factor]):
            ref = oracle.restrict_counts(ref)
        cs = tuple((n + factor - 1) // factor for n in shape)
        # whole grid, and a leaf slab of it
        s = Solver(cs, C8).load_coarsened(h, shape, factor)
        assert np.array_equal(s.read_counts(), ref)
        z0, z1 = 1, cs[2] - 1
        leaf = Solver.leaf(cs, C8, z0, z1).load_coarsened(h[z0 * factor:z1 * factor], shape, factor)
        assert np.array_equal(leaf.read_counts(), ref[z0:z1])
        for narrow in (np.uint8, np.uint16):  # narrow host counts, the same sums
            assert h.max() <= 255
            leaf.load_coarsened(h[z0 * factor:z1 * factor].astype(narrow), shape, factor)
            assert np.array_equal(leaf.read_counts(), ref[z0:z1])


def test_prolong_slab_equals_prolong_from():
    from paper_2107_14790_b200 import Solver
    shape = (37, 22, 19)
    cs = tuple((n + 1) // 2 for n in shape)
    h = synth.random_histograms(shape, 4)
    coarse = Solver(cs, C8).load(oracle.restrict_counts(h)).iterate(9)
    a = Solver(shape, C8).load(h).prolong_from(coarse)
    b = Solver(shape, C8).load(h).prolong_slab(coarse.read_u(), coarse.get("v"), 0)
    for f in ("u", "v", "ubar", "vbar", "p", "q"):
        assert np.array_equal(a.get(f), b.get(f)), f
    a.iterate(5)
    b.iterate(5)
    assert np.array_equal(a.read_u(), b.read_u())


@pytest.mark.parametrize("impl", ["tma", "regs"])
def test_leaf_iteration_equals_group_iteration(impl, monkeypatch):
    from paper_2107_14790_b200 import Group, Solver
    if impl == "regs":
        monkeypatch.setenv("TGV_FUSED_IMPL", "regs")
    shape = (45, 33, 24)
    h = synth.random_histograms(shape, 6)
    cuts = [0, 7, 16, 24]
    grp = Group(shape, cuts, C8).load(h)
    z0, z1 = 7, 16
    leaf = Solver.leaf(shape, C8, z0, z1).load(h[z0:z1])
    # the group's initial state is u_0 = u_-1 (ubar = u), v = p = q = 0: the border
    # planes are the group's neighbouring planes
    u = grp.read_u()
    leaf.set_border(0, u=u[z0 - 1]).set_border(1, u=u[z1])
    grp.iterate(1)
    leaf.iterate(1)
    for f in ("u", "v", "p", "q"):
        assert np.array_equal(leaf.get(f), grp.get(f)[..., z0:z1, :, :]), f


@pytest.mark.parametrize("impl", ["tma", "regs"])
def test_leaf_from_parent_matches_oracle_leaf(impl, monkeypatch):
    from paper_2107_14790_b200 import Solver
    if impl == "regs":
        monkeypatch.setenv("TGV_FUSED_IMPL", "regs")
    shape = (41, 30, 26)
    cs = tuple((n + 1) // 2 for n in shape)
    h = synth.random_histograms(shape, 8)
    rng = np.random.default_rng(3)
    pu = rng.uniform(-1, 1, cs[::-1]).astype(np.float32)
    pv = rng.uniform(-0.2, 0.2, (3,) + cs[::-1]).astype(np.float32)
    for z0, z1 in ((0, 9), (9, 17), (17, 26)):
        leaf = Solver.leaf(shape, C8, z0, z1).load(h[z0:z1])
        c0, c1 = max(z0 - 1, 0) // 2, min(z1, shape[2] - 1) // 2 + 1
        leaf.prolong_slab(pu[c0:c1], pv[:, c0:c1], c0).iterate(60)
        o = oracle.leaf_from_parent(shape, z0, z1, h[z0:z1], pu, pv)
        for _ in range(60):
            oracle.leaf_step(o)
        assert np.max(np.abs(leaf.read_u().astype(np.float64) - o.u)) <= 1e-4, (z0, z1)
        assert np.max(np.abs(leaf.get("p").astype(np.float64) - o.get("p"))) <= 1e-4, (z0, z1)


def test_out_of_core_matches_oracle_out_of_core():
    from paper_2107_14790_b200 import out_of_core
    wl = synth.workload("C1")
    h = synth.make_histograms("C1")
    nx, ny, _ = wl.shape
    stats = {}
    u, v = out_of_core.solve(wl.shape, h, C8, levels=3, iters=200, leaf_voxels=nx * ny * 2, stats=stats,
                             lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
    assert stats["leaves"] == [1, 2, 16]
    uo, vo = oracle.out_of_core(wl.shape, h, levels=3, iters=200, leaf_voxels=nx * ny * 2,
                                threads=oracle.max_threads(), lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1,
                                tau=wl.tau, sigma=wl.sigma)
    assert np.max(np.abs(u.astype(np.float64) - uo)) <= 1e-4
    assert np.max(np.abs(v.astype(np.float64) - vo)) <= 1e-4


def test_pooled_leaves_are_reproducible():
    """Leaves moved between slabs (tgv_leaf_rebind) give the freshly created leaves'
    result bit for bit, solve after solve."""
    from paper_2107_14790_b200 import out_of_core
    shape = (40, 36, 45)
    h = synth.random_histograms(shape, 9)
    kw = dict(levels=3, iters=40, leaf_voxels=40 * 36 * 4)
    ref_u, ref_v = out_of_core.solve(shape, h, C8, **kw)
    ooc = out_of_core.OutOfCore(shape, C8, keep_pool=True, **kw)
    assert ooc.leaves == [12, 2, 1]  # 45 planes by 4 and 23 by 16 (ragged last leaves), 12 in one
    for counts in (h, h.astype(np.uint8)):
        u, v = ooc.solve(counts)
        assert np.array_equal(u, ref_u) and np.array_equal(v, ref_v)
    ooc.close()


def test_many_leaves_stay_close_to_in_core():
    from paper_2107_14790_b200 import out_of_core
    from paper_2107_14790_b200.multilevel import coarse_to_fine
    wl = synth.workload("C2")
    h = synth.make_histograms("C2")
    nx, ny, nz = wl.shape
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
    stats = {}
    u, _ = out_of_core.solve(wl.shape, h, C8, levels=3, iters=200, leaf_voxels=nx * ny * nz // 8, stats=stats, **kw)
    assert stats["leaves"][-1] >= 8
    ref = coarse_to_fine(wl.shape, h, C8, levels=3, iters=200, **kw).read_u()
    assert np.mean(np.abs(u - ref)) <= 0.05
    assert np.mean(np.sign(u) == np.sign(ref)) >= 0.99


def test_leaf_errors():
    from paper_2107_14790_b200 import Solver, tgv
    shape = (16, 16, 16)
    h = synth.random_histograms(shape, 1)
    leaf = Solver.leaf(shape, C8, 4, 12).load(h[4:12])
    for call in (lambda: leaf.set_schedule("split"), lambda: leaf.set_model("tvl1")):
        with pytest.raises(tgv.TgvError) as ei:
            call()
        assert ei.value.status == tgv.TGV_EINVAL
    with pytest.raises(tgv.TgvError) as ei:  # parents of planes 3..12 are coarse planes 1..6
        leaf.prolong_slab(np.zeros((3, 8, 8), np.float32), np.zeros((3, 3, 8, 8), np.float32), 2)
    assert ei.value.status == tgv.TGV_EINVAL
    with pytest.raises(tgv.TgvError) as ei:  # a leaf keeps its plane count
        leaf.rebind(0, 9)
    assert ei.value.status == tgv.TGV_EINVAL
    whole = Solver(shape, C8).load(h)
    for call in (lambda: whole.set_border(0), lambda: whole.rebind(0, 16)):
        with pytest.raises(tgv.TgvError) as ei:
            call()
        assert ei.value.status == tgv.TGV_ESTATE
    with pytest.raises(tgv.TgvError) as ei:  # leaves do not take part in restrict / prolong_from
        Solver((8, 8, 8), C8).restrict_from(leaf)
    assert ei.value.status == tgv.TGV_EINVAL
