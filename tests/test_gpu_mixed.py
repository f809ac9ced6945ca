"""GPU parity of 2:1 mixed-level brick sets (tgv_bricks_create_mixed, R27)
against oracle/mixed.py ("4 or less neighbors over each face",
:446-453 frozen parent cubes): one iteration from a random state with every kind of
face, the scheme over many iterations (u within 1e-4, energy 1e-5, gap, max|v|), a
one-level set equal to the uniform SPLIT brick schedule bit for bit, Alg. 1 votes per
level bit-exact, prolongation into a mixed set exact, S and the error paths."""
import numpy as np
import pytest

import synth
from oracle import bricks as ob
from oracle import mixed as om

pytestmark = pytest.mark.gpu

KW = dict(lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25)


def BS():
    from paper_2107_14790_b200.bricks import BrickSolver
    return BrickSolver


def two_level_set(E):
    """A level-1 brick with the level-0 bricks tiling its +x, -y and +z faces (one quadrant
    of the +x face left empty), a same-level fine neighbour, a coarse neighbour below, and
    a level-1 frozen brick beside a fine frozen brick."""
    levels, coords = [1], [(1, 1, 1)]
    for a in (0, 1):
        for b in (0, 1):
            if (a, b) != (1, 1):
                levels.append(0)
                coords.append((4, 2 + a, 2 + b))  # +x face of the coarse brick, one quadrant empty
            levels.append(0)
            coords.append((2 + a, 1, 2 + b))  # -y face
            levels.append(0)
            coords.append((2 + a, 2 + b, 4))  # +z face
    levels += [0, 1, 1]
    coords += [(5, 2, 2), (1, 1, 0), (2, 1, 0)]
    frozen = np.zeros(len(levels), bool)
    frozen[[2, 5, len(levels) - 2, len(levels) - 1]] = True
    del E
    return np.array(levels), np.array(coords), frozen


def pair(E, seed, frozen_values=True, nbins=8, scale=1):
    levels, coords, frozen = two_level_set(E)
    rng = np.random.default_rng(seed)
    nb = len(levels)
    c = None
    if nbins != 8:
        c = np.sort(rng.uniform(-0.95, 0.95, nbins)).astype(np.float32).astype(np.float64)
    h = (rng.integers(0, 6, (nb, E, E, E, nbins)) * scale).astype(np.uint32)
    o = om.MixedOracle(E, levels, coords, frozen, centers=c, **KW).load(h)
    s = BS()(E, coords, frozen.astype(np.uint8), levels=levels, centers=None if c is None else list(c), **KW).load(h)
    if frozen_values:
        u0 = np.where(frozen[:, None, None, None], rng.uniform(-1, 1, (nb, E, E, E)), o.get("u"))
        v0 = rng.normal(0, 0.2, (nb, 3, E, E, E)) * frozen[:, None, None, None, None]
        u0, v0 = u0.astype(np.float32), v0.astype(np.float32)
        o.set_primal(u0.astype(np.float64), v0.astype(np.float64))
        s.set_primal(u0, v0)
    return o, s, (levels, coords, frozen)


@pytest.mark.parametrize("E", [4, 8])
def test_one_iteration_from_a_random_primal(E):
    """Every kind of face (same level, coarser, four finer, a missing quadrant, none) and
    the frozen S faces in one dual + primal step from random u, v on every brick."""
    levels, coords, frozen = two_level_set(E)
    rng = np.random.default_rng(2)
    nb = len(levels)
    h = rng.integers(0, 6, (nb, E, E, E, 8)).astype(np.uint32)
    u0 = rng.uniform(-1, 1, (nb, E, E, E)).astype(np.float32)
    v0 = rng.normal(0, 0.5, (nb, 3, E, E, E)).astype(np.float32)
    o = om.MixedOracle(E, levels, coords, frozen, **KW).load(h).set_primal(u0.astype(np.float64), v0.astype(np.float64))
    s = BS()(E, coords, frozen.astype(np.uint8), levels=levels, **KW).load(h).set_primal(u0, v0)
    for it in range(2):
        o.iterate(1)
        s.iterate(1)
        for f in ("p", "q", "u", "v"):
            np.testing.assert_allclose(s.get(f), o.get(f), rtol=0, atol=3e-6, err_msg=f"{f} after {it + 1}")
    assert s.info()["s_voxels"] == int(o.S.sum())


@pytest.mark.parametrize("E,nbins,scale", [(4, 8, 1), (8, 8, 1), (16, 16, 100), (8, 3, 1)])
def test_mixed_set_matches_oracle(E, nbins, scale):
    """Also 16 bins with u16 counts (x100) and 3 non-uniform bins."""
    o, s, _ = pair(E, 5, nbins=nbins, scale=scale)
    if scale > 1:
        assert s.info()["count_bytes"] == 2
    o.iterate(60)
    s.iterate(60)
    du = float(np.max(np.abs(s.read_u().astype(np.float64) - o.get("u"))))
    eo, es = o.energy(), s.energy()
    assert du <= 1e-4, du
    assert abs(es["E"] - eo["E"]) <= 1e-5 * abs(eo["E"]), (es["E"], eo["E"])
    for k in ("alpha1", "alpha0", "data"):
        assert abs(es[k] - eo[k]) <= 1e-5 * abs(eo["E"]), k
    assert abs(es["gap"] - eo["gap"]) <= 1e-5 * abs(eo["E"]), (es["gap"], eo["gap"])
    assert abs(es["vmax"] - eo["vmax"]) <= 1e-4
    print(f"mixed E={E} x60: max|du| = {du:.2e}, rel dE = {abs(es['E'] - eo['E']) / eo['E']:.2e}")


def test_energy_of_a_shared_state_is_the_oracle_s():
    """tgv_bricks_energy on a mixed set after the same single step from the same random
    primal: every term within fp64 rounding of the oracle's (h^3 weights, S, the B term)."""
    E = 4
    levels, coords, frozen = two_level_set(E)
    rng = np.random.default_rng(9)
    nb = len(levels)
    h = rng.integers(0, 6, (nb, E, E, E, 8)).astype(np.uint32)
    u0 = rng.uniform(-1, 1, (nb, E, E, E)).astype(np.float32)
    v0 = rng.normal(0, 0.5, (nb, 3, E, E, E)).astype(np.float32)
    s = BS()(E, coords, frozen.astype(np.uint8), levels=levels, **KW).load(h).set_primal(u0, v0).iterate(1)
    o = om.MixedOracle(E, levels, coords, frozen, **KW).load(h)
    o.set_primal(s.read_u().astype(np.float64), s.get("v").astype(np.float64))  # the GPU's own fp32 state
    o.p, o.q = o._flat(s.get("p"), 3), o._flat(s.get("q"), 6)
    eo, es = o.energy(), s.energy()
    for k in ("E", "alpha1", "alpha0", "data", "gap"):
        assert abs(es[k] - eo[k]) <= 1e-10 * abs(eo["E"]), (k, es[k], eo[k])
    assert es["vmax"] == eo["vmax"]


@pytest.mark.parametrize("E", [4, 8])
def test_one_level_mixed_set_is_the_split_brick_schedule_bitwise(E):
    rng = np.random.default_rng(4)
    coords = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 0, 1), (2, 1, 0), (1, 1, 1), (3, 1, 0)])
    frozen = np.array([0, 1, 0, 0, 1, 0, 0], np.uint8)
    h = rng.integers(0, 6, (len(coords), E, E, E, 8)).astype(np.uint32)
    a = BS()(E, coords, frozen, **KW).set_schedule("split").load(h).iterate(23)
    b = BS()(E, coords, frozen, levels=np.zeros(len(coords), np.uint8), **KW).load(h).iterate(23)
    for f in ("u", "v", "p", "q"):
        assert np.array_equal(a.get(f), b.get(f)), f
    ea, eb = a.energy(), b.energy()
    assert abs(ea["E"] - eb["E"]) <= 1e-12 * abs(ea["E"]) and abs(ea["gap"] - eb["gap"]) <= 1e-9 * abs(ea["E"])
    assert a.info()["s_voxels"] == b.info()["s_voxels"]


def test_votes_per_level_bit_exact():
    """Alg. 1 into a mixed set: brick b voted at voxel size 2^l, radius 2^(l-1) equals the
    oracle's dense vote of that brick's box at its level (R22, R25)."""
    E = 8
    wl = synth.workload("C1")
    depths = synth.render_depths(wl)
    cams = [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
             "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]
    levels = np.array([1, 0, 0, 0, 0, 1])
    coords = np.array([(0, 0, 0), (2, 0, 0), (2, 1, 0), (2, 0, 1), (2, 1, 1), (0, 1, 0)])
    s = BS()(E, coords, None, levels=levels, **KW).vote(cams, depths, voxel_radius=0.5)
    got = s.read_counts()
    for b in range(len(coords)):
        hb = float(1 << int(levels[b]))
        want = ob.vote(coords[b:b + 1], E, cams, depths, voxel_size=hb, r=0.5 * hb)[0]
        assert np.array_equal(got[b], want), b
    assert got.sum() > 0


def test_prolongation_into_a_mixed_set():
    """Level-0 bricks take their parent voxel's u and v / 2 (R19); level-1 bricks copy the
    coarse brick at their own coordinates (u, v / 2: v in finest-level units)."""
    E = 4
    rng = np.random.default_rng(6)
    ccoords = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0)])
    h = rng.integers(0, 5, (4, E, E, E, 8)).astype(np.uint32)
    coarse = BS()(E, ccoords, **KW).set_schedule("split").load(h).iterate(7)
    cu, cv = coarse.read_u(), coarse.get("v")
    levels = np.array([1, 1, 0, 0, 0, 0])
    coords = np.array([(0, 0, 0), (0, 1, 0), (2, 0, 0), (2, 1, 0), (3, 0, 0), (3, 1, 0)])
    fh = rng.integers(0, 5, (6, E, E, E, 8)).astype(np.uint32)
    m = BS()(E, coords, np.ones(6, np.uint8), levels=levels, **KW).load(fh).prolong_from(coarse)
    u, v = m.read_u(), m.get("v")
    np.testing.assert_array_equal(u[0], cu[0])
    np.testing.assert_array_equal(u[1], cu[3])
    np.testing.assert_array_equal(v[0], np.float32(0.5) * cv[0])
    idx = (E * 1 + np.arange(E)) // 2  # brick (3, y, 0): parent (1, .) with x offset E
    for b, (cx, cy, _) in enumerate(coords[2:], start=2):
        pb = {(1, 0): 1, (1, 1): 2}[(cx // 2, cy // 2)]
        ix = (E * (cx % 2) + np.arange(E)) // 2
        iy = (E * (cy % 2) + np.arange(E)) // 2
        iz = np.arange(E) // 2
        np.testing.assert_array_equal(u[b], cu[pb][np.ix_(iz, iy, ix)])
        np.testing.assert_array_equal(v[b], np.float32(0.5) * cv[pb][:, iz][:, :, iy][:, :, :, ix])
    del idx


def test_mixed_error_paths():
    from paper_2107_14790_b200 import tgv
    with pytest.raises(tgv.TgvError):  # level 2 beside level 0
        BS()(4, [(0, 0, 0), (4, 0, 0)], levels=[2, 0])
    with pytest.raises(tgv.TgvError):  # overlap
        BS()(4, [(0, 0, 0), (1, 1, 1)], levels=[1, 0])
    s = BS()(32, [(0, 0, 0), (2, 0, 0)], levels=[1, 0])
    assert s.info()["schedule"] == tgv.SCHEDULE_SPLIT  # the default (measured faster on C5)
    s.set_schedule("fused")  # E = 32: the fused sweep where it applies
    assert s.info()["schedule"] == tgv.SCHEDULE_FUSED
    s = BS()(16, [(0, 0, 0), (2, 0, 0)], levels=[1, 0])
    assert s.info()["schedule"] == tgv.SCHEDULE_SPLIT
    with pytest.raises(tgv.TgvError):
        s.set_schedule("fused")


def test_mixed_finest_level_matches_oracle_hierarchy():
    """The C1 hierarchy (E = 4, 3 levels) with its finest level solved as a 2:1 mixed set:
    A at level 0, the frozen border made of level-0 bricks under A's parents and of the
    level-1 parent cubes elsewhere (R27); against the oracle solving the
    same coarse levels and the same mixed set (votes per level, prolongation from level 1:
    R19 for level-0 bricks, the parent's own u, v / 2 for level-1 bricks)."""
    from paper_2107_14790_b200.brick_levels import BrickLevels
    wl = synth.workload("C1")
    depths = synth.render_depths(wl)
    cams = [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
             "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]
    E, levels, iters = 4, 3, 40
    bl = BrickLevels((32, 32, 32), cams, depths, levels=levels, edge=E, min_votes=2, **KW)
    m = bl.build_mixed()
    _, coords, lv, fr = bl.mixed
    assert (lv == 1).any() and (lv == 0).sum() > (~fr).sum()  # both kinds of border brick
    s = bl.solve_mixed(iters)
    assert s is m
    # oracle: levels 2 and 1 (same sets as the GPU's), then the mixed set
    o = ob.BrickOracle(E, bl.coords[2], bl.frozen[2], **KW)
    o.load(ob.vote(bl.coords[2], E, cams, depths, voxel_size=4.0, r=2.0)).iterate(iters)
    o1 = ob.BrickOracle(E, bl.coords[1], bl.frozen[1], **KW)
    o1.load(ob.vote(bl.coords[1], E, cams, depths, voxel_size=2.0, r=1.0))
    o1.set_primal(*ob.prolong(o, bl.coords[1]))
    o1.iterate(iters)
    counts = np.concatenate([ob.vote(coords[b:b + 1], E, cams, depths, voxel_size=float(1 << int(lv[b])),
                                     r=0.5 * (1 << int(lv[b]))) for b in range(len(coords))])
    mo = om.MixedOracle(E, lv, coords, fr, **KW).load(counts)
    u0 = np.zeros((len(coords), E, E, E))
    v0 = np.zeros((len(coords), 3, E, E, E))
    fine = lv == 0
    pu, pv = ob.prolong(o1, coords[fine])
    u0[fine], v0[fine] = pu, pv
    idx = {tuple(int(t) for t in c): i for i, c in enumerate(bl.coords[1])}
    o1u, o1v = o1.get("u"), o1.get("v")
    for b in np.nonzero(~fine)[0]:
        j = idx[tuple(int(t) for t in coords[b])]
        u0[b], v0[b] = o1u[j], 0.5 * o1v[j]
    mo.set_primal(u0, v0).iterate(iters)
    du = float(np.max(np.abs(s.read_u().astype(np.float64) - mo.get("u"))))
    eg, eo = s.energy(), mo.energy()
    assert du <= 1e-4, du
    assert abs(eg["E"] - eo["E"]) <= 1e-5 * abs(eo["E"])
    assert abs(eg["gap"] - eo["gap"]) <= 1e-5 * abs(eo["E"])
    print(f"mixed finest level of C1: {len(coords)} bricks ({int((lv == 1).sum())} coarse), max|du| = {du:.2e}")
    bl.close()


def test_fused_schedule_of_a_mixed_set_equals_split_bitwise():
    """E = 32: the FUSED schedule of a mixed set (the fused brick sweep over the solved
    level-0 bricks whose 26-neighbourhood is level 0 or empty, the mixed kernels elsewhere)
    gives the SPLIT schedule's iterates bit for bit, with both kinds of brick present."""
    from paper_2107_14790_b200 import tgv
    E = 32
    # a 2 x 2 x 2 block of level-0 bricks (some far from any coarse brick), a level-1 brick on
    # the -x side of it, frozen bricks of both levels
    levels, coords = [], []
    for x in range(2, 6):
        for y in range(0, 2):
            for z in range(0, 2):
                levels.append(0)
                coords.append((x, y, z))
    levels += [1, 1]
    coords += [(0, 0, 0), (3, 0, 0)]  # level 1: fine x in [0, 64) and [192, 256)
    frozen = np.zeros(len(levels), np.uint8)
    frozen[[1, len(levels) - 1]] = 1
    rng = np.random.default_rng(12)
    h = rng.integers(0, 6, (len(levels), E, E, E, 8)).astype(np.uint32)
    u0 = rng.uniform(-1, 1, (len(levels), E, E, E)).astype(np.float32)
    v0 = rng.normal(0, 0.3, (len(levels), 3, E, E, E)).astype(np.float32)
    a = BS()(E, coords, frozen, levels=levels, **KW).set_schedule("fused").load(h).set_primal(u0, v0)
    assert a.info()["schedule"] == tgv.SCHEDULE_FUSED
    b = BS()(E, coords, frozen, levels=levels, **KW).set_schedule("split").load(h).set_primal(u0, v0)
    a.iterate(9)
    b.iterate(9)
    for f in ("u", "v", "p", "q"):
        assert np.array_equal(a.get(f), b.get(f)), (f, float(np.max(np.abs(a.get(f) - b.get(f)))))
    ea, eb = a.energy(), b.energy()
    assert ea["E"] == eb["E"] and ea["gap"] == eb["gap"]
    a.close()
    b.close()
