"""GPU parity of the NEXT-3 block-sparse brick sets (include/tgv_bricks.h; DESIGN.md
R24) against the brick-set oracle (oracle/bricks.py, pinned in test_oracle_bricks.py),
through the C ABI.  Gates: max|u_gpu - u_cpu| <= 1e-4, |dE|/E <= 1e-5 (north star).

- random sparse sets with frozen bricks, brick edges 4, 8, 16, 32, and a ragged
  L-shaped set of 32^3 bricks (the bench's brick edge);
- a box of solved bricks is the dense SPLIT schedule bit for bit (same expressions);
- frozen bricks keep their values bit for bit; u16 counts and 3 / 16 bins;
- brick order does not matter (bitwise); error paths.
"""
import numpy as np
import pytest

import synth
from oracle import bricks as ob

pytestmark = pytest.mark.gpu

KW = dict(lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25)


def _rand_set(rng, n, span):
    cells = set()
    while len(cells) < n:
        cells.add(tuple(int(a) for a in rng.integers(0, span, 3)))
    return np.array(sorted(cells), dtype=np.int32)


def _counts(nb, E, seed, nbins=8, max_count=12):
    h = synth.random_histograms((E, E, nb * E), seed, max_count=max_count)  # [nb*E, E, E, 8]
    h = h.reshape(nb, E, E, E, 8)
    if max_count > 255:
        h[0, 0, 0, 0, 3] = 1000  # u16 storage
    if nbins != 8:
        rng = np.random.default_rng(seed)
        h = rng.integers(0, max_count, (nb, E, E, E, nbins)).astype(np.uint32)
    return h


def _frozen_state(rng, nb, E):
    return rng.uniform(-0.9, 0.9, (nb, E, E, E)), rng.uniform(-0.3, 0.3, (nb, 3, E, E, E))


def _run_pair(E, coords, frozen, h, iters, centers=None, primal=None):
    from paper_2107_14790_b200.bricks import BrickSolver
    s = BrickSolver(E, coords, frozen, centers=centers, **KW).load(h)
    o = ob.BrickOracle(E, coords, frozen, centers=centers, **KW).load(h)
    if primal is not None:
        u0, v0 = primal
        # A keeps the loaded initialisation, B gets the frozen values (a prolongation-like restart)
        ua = np.where(frozen[:, None, None, None], u0, o.get("u"))
        va = v0 * frozen[:, None, None, None, None]
        s.set_primal(ua.astype(np.float32), va.astype(np.float32))
        o.set_primal(ua.astype(np.float32).astype(np.float64), va.astype(np.float32).astype(np.float64))
    s.iterate(iters)
    o.iterate(iters)
    return s, o


def _check(s, o, tol_u=1e-4):
    du = float(np.max(np.abs(s.read_u().astype(np.float64) - o.get("u"))))
    eg, eo = s.energy(), o.energy()
    assert du <= tol_u, du
    assert abs(eg["E"] - eo["E"]) <= 1e-5 * abs(eo["E"]), (eg, eo)
    assert abs(eg["gap"] - eo["gap"]) <= 1e-5 * abs(eo["E"]), (eg, eo)
    assert abs(eg["vmax"] - eo["vmax"]) <= 1e-4
    # duals: equal on S, exactly 0 elsewhere (R24)
    for name in ("p", "q"):
        g, r = s.get(name), o.get(name)
        assert float(np.max(np.abs(g - r))) <= 1e-4, name
        assert not np.any(g[r == 0.0]) or float(np.max(np.abs(g[r == 0.0]))) <= 1e-4
    return du


@pytest.mark.parametrize("E,n,span,iters,seed", [(4, 40, 5, 60, 0), (8, 14, 3, 50, 1), (16, 6, 3, 30, 2)])
def test_random_sets_with_frozen_bricks_match_oracle(E, n, span, iters, seed):
    rng = np.random.default_rng(seed)
    coords = _rand_set(rng, n, span)
    frozen = rng.random(len(coords)) < 0.3
    h = _counts(len(coords), E, 100 + seed)
    s, o = _run_pair(E, coords, frozen, h, iters, primal=_frozen_state(rng, len(coords), E))
    _check(s, o)
    # B is frozen bit for bit at the values given
    assert np.array_equal(s.read_u()[frozen], o.get("u")[frozen].astype(np.float32))
    assert s.info()["s_voxels"] == int(o.S.sum())


def test_ragged_set_of_32_cubed_bricks_matches_oracle():
    coords = np.array([(0, 0, 0), (1, 0, 0), (2, 0, 0), (2, 1, 0), (2, 1, 1), (0, 1, 1), (1, 2, 1)], dtype=np.int32)
    frozen = np.array([0, 0, 0, 0, 0, 1, 1], bool)
    rng = np.random.default_rng(3)
    h = _counts(len(coords), 32, 7)
    s, o = _run_pair(32, coords, frozen, h, 25, primal=_frozen_state(rng, len(coords), 32))
    _check(s, o)


def test_box_of_solved_bricks_is_the_dense_split_schedule_bitwise():
    from paper_2107_14790_b200 import Solver, tgv
    from paper_2107_14790_b200.bricks import BrickSolver
    E, nbx, nby, nbz = 16, 3, 2, 2
    shape = (nbx * E, nby * E, nbz * E)
    h = synth.random_histograms(shape, 9)  # [nz, ny, nx, 8]
    coords = np.array([(bx, by, bz) for bz in range(nbz) for by in range(nby) for bx in range(nbx)], dtype=np.int32)
    hb = np.stack([h[bz * E:(bz + 1) * E, by * E:(by + 1) * E, bx * E:(bx + 1) * E] for bx, by, bz in coords])
    s = BrickSolver(E, coords, **KW).load(hb).iterate(40)
    d = Solver(shape, [-0.875 + 0.25 * b for b in range(8)], **KW)
    d.set_schedule(tgv.SCHEDULE_SPLIT)
    d.load(h).iterate(40)
    for name in ("u", "v", "p", "q"):
        a = d.get(name)
        b = s.get(name)
        lead = () if a.ndim == 3 else (slice(None),)
        for i, (bx, by, bz) in enumerate(coords):
            blk = a[lead + (slice(bz * E, (bz + 1) * E), slice(by * E, (by + 1) * E), slice(bx * E, (bx + 1) * E))]
            assert np.array_equal(b[i], blk), (name, i)
    # the dense energy kernel forms fp32 per-voxel terms (fp64 sums), the brick kernel fp64 ones
    assert s.energy()["E"] == pytest.approx(d.energy()["E"], rel=1e-6)
    d.close()


def test_u16_counts_and_other_bin_counts():
    rng = np.random.default_rng(4)
    coords = _rand_set(rng, 9, 3)
    frozen = np.zeros(len(coords), bool)
    h = _counts(len(coords), 8, 11, max_count=300)
    h[0, 0, 0, 0, 3] = 1000  # forces u16 storage
    s, o = _run_pair(8, coords, frozen, h, 30)
    inf = s.info()
    assert inf["count_bytes"] == 2 and inf["nfrozen"] == 0 and inf["s_voxels"] == inf["solved_voxels"]
    _check(s, o)
    for centers in ([-0.6, 0.1, 0.7], list(np.linspace(-0.95, 0.95, 16))):
        h = _counts(len(coords), 8, 12, nbins=len(centers))
        s, o = _run_pair(8, coords, frozen, h, 30, centers=centers)
        _check(s, o)


def test_brick_order_does_not_matter_bitwise():
    from paper_2107_14790_b200.bricks import BrickSolver
    rng = np.random.default_rng(5)
    coords = _rand_set(rng, 12, 3)
    frozen = rng.random(len(coords)) < 0.25
    h = _counts(len(coords), 8, 13)
    u0, v0 = _frozen_state(rng, len(coords), 8)
    perm = rng.permutation(len(coords))
    a = BrickSolver(8, coords, frozen, **KW).load(h).set_primal(u0.astype(np.float32), v0.astype(np.float32))
    b = BrickSolver(8, coords[perm], frozen[perm], **KW).load(h[perm])
    b.set_primal(u0[perm].astype(np.float32), v0[perm].astype(np.float32))
    a.iterate(20)
    b.iterate(20)
    assert np.array_equal(a.read_u()[perm], b.read_u())
    assert np.array_equal(a.get("q")[perm], b.get("q"))


def test_error_paths_and_timing():
    from paper_2107_14790_b200 import tgv
    from paper_2107_14790_b200.bricks import BrickSolver
    s = BrickSolver(8, [(0, 0, 0), (0, 0, 1)], **KW)
    with pytest.raises(tgv.TgvError) as ei:
        s.iterate(1)
    assert ei.value.status == tgv.TGV_ESTATE
    s.load(_counts(2, 8, 1))
    with pytest.raises(tgv.TgvError) as ei:
        s.read(tgv.FIELD_UBAR)
    assert ei.value.status == tgv.TGV_EINVAL
    with pytest.raises(tgv.TgvError) as ei:
        s.load(np.zeros(5, np.uint32))
    assert ei.value.status == tgv.TGV_EINVAL
    big = _counts(2, 8, 1)
    big[0, 0, 0, 0, 0] = 70000
    with pytest.raises(tgv.TgvError) as ei:
        s.load(big)
    assert ei.value.status == tgv.TGV_ERANGE
    s.load(_counts(2, 8, 1))
    s.set_timing(True)
    s.iterate(3)
    t = s.timing()
    assert t["dual_launches"] == 3 and t["primal_launches"] == 3 and t["dual_ms"] > 0


@pytest.mark.parametrize("seed,nbins,big", [(0, 8, False), (1, 8, True), (2, 3, False), (3, 16, False)])
def test_fused_schedule_equals_split_bitwise(seed, nbins, big):
    """The single-sweep brick kernel (FUSED, default for 32^3 bricks) and the SPLIT
    schedule agree bit for bit on u, v, p, q: random sparse sets with frozen bricks,
    u8 / u16 counts, 3 bins; and the fused run matches the oracle."""
    from paper_2107_14790_b200.bricks import BrickSolver
    rng = np.random.default_rng(seed)
    coords = _rand_set(rng, 16, 3)
    frozen = rng.random(len(coords)) < 0.3
    frozen[0] = False
    centers = {8: None, 3: [-0.6, 0.1, 0.7], 16: list(np.linspace(-0.95, 0.95, 16))}[nbins]
    h = _counts(len(coords), 32, 40 + seed, nbins=nbins, max_count=300 if big else 12)
    u0, v0 = _frozen_state(rng, len(coords), 32)
    runs = {}
    for sched in ("fused", "split"):
        s = BrickSolver(32, coords, frozen, centers=centers, **KW).set_schedule(sched).load(h)
        assert s.info()["schedule"] == (0 if sched == "fused" else 1)
        ua = np.where(frozen[:, None, None, None], u0, s.read_u()).astype(np.float32)
        s.set_primal(ua, (v0 * frozen[:, None, None, None, None]).astype(np.float32))
        s.iterate(7)
        runs[sched] = {n: s.get(n) for n in ("u", "v", "p", "q")}
        runs[sched]["E"] = s.energy()["E"]
        if big:
            assert s.info()["count_bytes"] == 2
        s.close()
    for n in ("u", "v", "p", "q"):
        assert np.array_equal(runs["fused"][n], runs["split"][n]), n
    assert runs["fused"]["E"] == runs["split"]["E"]


def test_fused_schedule_only_for_32_cubed_bricks():
    from paper_2107_14790_b200 import tgv
    from paper_2107_14790_b200.bricks import BrickSolver
    s = BrickSolver(16, [(0, 0, 0)], **KW)
    assert s.info()["schedule"] == 1
    with pytest.raises(tgv.TgvError) as ei:
        s.set_schedule("fused")
    assert ei.value.status == tgv.TGV_EINVAL


def test_fused_schedule_edge_sets():
    """A single brick (every neighbour outside Omega), a line of bricks with frozen ends,
    and a set with no solved brick: FUSED = SPLIT bitwise, frozen values untouched."""
    from paper_2107_14790_b200.bricks import BrickSolver
    rng = np.random.default_rng(7)
    cases = [(np.array([(3, 2, 1)]), np.array([False])),
             (np.array([(x, 0, 0) for x in range(5)]), np.array([True, False, False, False, True])),
             (np.array([(0, 0, 0), (0, 1, 0)]), np.array([True, True]))]
    for coords, frozen in cases:
        h = _counts(len(coords), 32, 60 + len(coords))
        u0, v0 = _frozen_state(rng, len(coords), 32)
        out = {}
        for sched in ("fused", "split"):
            s = BrickSolver(32, coords, frozen, **KW).set_schedule(sched).load(h)
            s.set_primal(np.where(frozen[:, None, None, None], u0, s.read_u()).astype(np.float32),
                         (v0 * frozen[:, None, None, None, None]).astype(np.float32))
            s.iterate(5)
            out[sched] = (s.read_u(), s.get("q"))
            s.close()
        assert np.array_equal(out["fused"][0], out["split"][0])
        assert np.array_equal(out["fused"][1], out["split"][1])
        assert np.array_equal(out["fused"][0][frozen], u0[frozen].astype(np.float32))


