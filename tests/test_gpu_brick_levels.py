"""GPU parity of the brick-set level companions (include/tgv_bricks.h; R24 with
R18-R22) against oracle/bricks.py: Alg. 1 votes into bricks (bit-exact integer counts),
refinement flags (bit-exact), prolongation (exact), and the whole coarse-to-fine
block-sparse solve of paper_2107_14790_b200.brick_levels (u within 1e-4, energy 1e-5)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import bricks as ob

pytestmark = pytest.mark.gpu

KW = dict(lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25)


def cams_of(wl):
    return [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
             "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]


@pytest.mark.parametrize("E,h,r", [(8, 1.0, 0.5), (4, 2.0, 1.0)])
def test_brick_votes_and_refine_flags_bit_exact(E, h, r):
    from paper_2107_14790_b200.bricks import BrickSolver
    wl = synth.workload("C1")
    depths = synth.render_depths(wl)
    cams = cams_of(wl)
    n = int(32 / h) // E
    rng = np.random.default_rng(0)
    allc = np.array([(x, y, z) for z in range(n) for y in range(n) for x in range(n)], dtype=np.int32)
    coords = allc[rng.permutation(len(allc))[: max(4, len(allc) * 2 // 3)]]
    frozen = rng.random(len(coords)) < 0.2
    s = BrickSolver(E, coords, frozen, **KW).vote(cams, depths, voxel_size=h, voxel_radius=r)
    got = s.read_counts()
    ref = ob.vote(coords, E, cams, depths, voxel_size=h, r=r)
    assert np.array_equal(got, ref), int(np.sum(got != ref))
    assert got[..., :7].sum() > 0  # the surface is inside the set
    for mv in (1, 2, 5):
        assert np.array_equal(s.refine_flags(mv), ob.refine_flags(ref, frozen, mv))


def test_prolongation_is_exact():
    from paper_2107_14790_b200.bricks import BrickSolver
    E = 8
    rng = np.random.default_rng(1)
    cc = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 1)], dtype=np.int32)
    fine = np.array([(2 * x + a, 2 * y + b, 2 * z + c) for x, y, z in cc for a in (0, 1) for b in (0, 1) for c in (0, 1)
                     if rng.random() < 0.6], dtype=np.int32)
    frozen = rng.random(len(fine)) < 0.3
    cu = rng.uniform(-1, 1, (len(cc), E, E, E)).astype(np.float32)
    cv = rng.uniform(-0.5, 0.5, (len(cc), 3, E, E, E)).astype(np.float32)
    hc = rng.integers(0, 4, (len(cc), E, E, E, 8)).astype(np.uint32)
    hf = rng.integers(0, 4, (len(fine), E, E, E, 8)).astype(np.uint32)
    g = BrickSolver(E, cc, **KW).load(hc).set_primal(cu, cv)
    f = BrickSolver(E, fine, frozen, **KW).load(hf).prolong_from(g)
    o = ob.BrickOracle(E, cc, **KW).load(hc).set_primal(cu.astype(np.float64), cv.astype(np.float64))
    u_ref, v_ref = ob.prolong(o, fine)
    assert np.array_equal(f.read_u(), u_ref.astype(np.float32))
    assert np.array_equal(f.get("v"), v_ref.astype(np.float32))
    assert not np.any(f.get("p")) and not np.any(f.get("q"))
    # a brick whose parent is missing is rejected
    from paper_2107_14790_b200 import tgv
    orphan = BrickSolver(E, [(9, 9, 9)], **KW).load(np.zeros((1, E, E, E, 8), np.uint32))
    with pytest.raises(tgv.TgvError) as ei:
        orphan.prolong_from(g)
    assert ei.value.status == tgv.TGV_EINVAL


def test_coarse_to_fine_brick_levels_match_oracle():
    from paper_2107_14790_b200.brick_levels import BrickLevels
    wl = synth.workload("C1")
    depths = synth.render_depths(wl)
    cams = cams_of(wl)
    E, levels, iters = 4, 3, 40
    bl = BrickLevels((32, 32, 32), cams, depths, levels=levels, edge=E, min_votes=2, **KW)
    # the oracle rebuilds the same hierarchy from its own votes and flags
    top = levels - 1
    o = ob.BrickOracle(E, bl.coords[top], bl.frozen[top], **KW)
    o.load(ob.vote(bl.coords[top], E, cams, depths, voxel_size=4.0, r=2.0))
    assert not bl.frozen[top].any() and len(bl.coords[top]) == 8
    o.iterate(iters)
    for lev in range(top - 1, -1, -1):
        h = float(1 << lev)
        up_counts = ob.vote(bl.coords[lev + 1], E, cams, depths, voxel_size=2 * h, r=h)
        flags = ob.refine_flags(up_counts, bl.frozen[lev + 1], 2)
        b, oc = np.nonzero(flags)
        A = {tuple(int(t) for t in 2 * bl.coords[lev + 1][i] + (k & 1, k >> 1 & 1, k >> 2)) for i, k in zip(b, oc)}
        A = {a for a in A if max(a) < 32 // (E << lev)}
        got_A = {tuple(int(t) for t in c) for c, fr in zip(bl.coords[lev], bl.frozen[lev]) if not fr}
        assert got_A == A, lev
        f = ob.BrickOracle(E, bl.coords[lev], bl.frozen[lev], **KW)
        f.load(ob.vote(bl.coords[lev], E, cams, depths, voxel_size=h, r=0.5 * h))
        u, v = ob.prolong(o, bl.coords[lev])
        f.set_primal(u, v)
        f.iterate(iters)
        o = f
    s = bl.solve(iters)
    du = float(np.max(np.abs(s.read_u().astype(np.float64) - o.get("u"))))
    eg, eo = s.energy(), o.energy()
    assert du <= 1e-4, du
    assert abs(eg["E"] - eo["E"]) <= 1e-5 * abs(eo["E"])
    assert abs(eg["gap"] - eo["gap"]) <= 1e-5 * abs(eo["E"])
    assert sum(a for a, _ in bl.bricks()) < 8 ** 3  # block-sparse: fewer solved bricks than the dense finest grid
    # a second solve from the resident counts is bitwise the same
    u1 = s.read_u().copy()
    assert np.array_equal(bl.solve(iters).read_u(), u1)
    bl.close()


def test_finest_level_in_parts_matches_oracle_parts():
    """R26: the finest level solved in Morton-contiguous parts, each with its frozen
    shell held at the parent values: one part is the in-core solve
    bit for bit; three parts match the oracle solving the same parts."""
    from paper_2107_14790_b200.brick_levels import BrickLevels, PartSolver
    wl = synth.workload("C1")
    depths = synth.render_depths(wl)
    cams = cams_of(wl)
    E, levels, iters = 4, 3, 30
    bl = BrickLevels((32, 32, 32), cams, depths, levels=levels, edge=E, **KW)
    ref = bl.solve(iters).read_u()
    solved = bl.coords[0][~bl.frozen[0]]
    one = PartSolver(bl, 1).solve(iters)
    c1, u1 = one[0]
    assert np.array_equal(c1, solved) and np.array_equal(u1, ref[: len(solved)])
    ps = PartSolver(bl, 3)
    got = ps.solve(iters, pool={})
    assert len(got) == 3 and sum(len(c) for c, _ in got.values()) == len(solved)
    # oracle: the coarse levels, then each part with its own frozen shell
    o = ob.BrickOracle(E, bl.coords[2], bl.frozen[2], **KW).load(ob.vote(bl.coords[2], E, cams, depths, voxel_size=4.0, r=2.0))
    o.iterate(iters)
    o1 = ob.BrickOracle(E, bl.coords[1], bl.frozen[1], **KW).load(ob.vote(bl.coords[1], E, cams, depths, voxel_size=2.0, r=1.0))
    o1.set_primal(*ob.prolong(o, bl.coords[1]))
    o1.iterate(iters)
    differs = False
    for p, (c, u) in got.items():
        cp, fr, _ = ps.sets[p]
        op = ob.BrickOracle(E, cp, fr, **KW).load(ob.vote(cp, E, cams, depths, voxel_size=1.0, r=0.5))
        op.set_primal(*ob.prolong(o1, cp))
        op.iterate(iters)
        nA = int((~fr).sum())
        assert float(np.max(np.abs(u.astype(np.float64) - op.get("u")[:nA]))) <= 1e-4
        # frozen borders: near part borders the parts differ from the single-set solve
        idx = {tuple(int(t) for t in x): i for i, x in enumerate(solved)}
        rows = [idx[tuple(int(t) for t in x)] for x in c]
        differs |= not np.array_equal(u, ref[rows])
    assert differs
    bl.close()


def test_parts_shared_by_ranks_equal_one_rank():
    """R26 on several GPUs: rank r solves parts r, r + N, ...; parts need no exchange, so
    the union of two ranks' shares (emulated in one process on one GPU) is the one-rank
    solve of all parts, bit for bit."""
    from paper_2107_14790_b200.brick_levels import BrickLevels, PartSolver
    wl = synth.workload("C1")
    depths = synth.render_depths(wl)
    E, iters = 4, 20
    bl = BrickLevels((32, 32, 32), cams_of(wl), depths, levels=3, edge=E, **KW)
    allp = PartSolver(bl, 4).solve(iters)
    shares = [PartSolver(bl, 4, mine=list(range(r, 4, 2))).solve(iters) for r in range(2)]
    merged = {**shares[0], **shares[1]}
    assert sorted(merged) == sorted(allp) == [0, 1, 2, 3]
    for p in allp:
        assert np.array_equal(merged[p][0], allp[p][0]) and np.array_equal(merged[p][1], allp[p][1])
    bl.close()


def test_parts_edge32_fused_one_part_bitwise_and_fused_equals_split():
    """R26 with the bench's 32^3 bricks (the fused brick sweep, large frozen shells, pooled
    contexts, pinned u8 counts): one part is the in-core finest level bit for bit, and
    three parts give the same u with the fused sweep and with SPLIT."""
    from paper_2107_14790_b200.brick_levels import BrickLevels, PartSolver
    wl = synth.workload("C2")
    depths = synth.render_depths(wl)
    iters = 20
    bl = BrickLevels(wl.shape, cams_of(wl), depths, levels=2, edge=32, voxel_radius=wl.voxel_radius, **KW)
    ref = bl.solve(iters).read_u()
    solved = bl.coords[0][~bl.frozen[0]]
    one = PartSolver(bl, 1, pinned=True, schedule="fused")
    assert one.schedule == "fused"
    c1, u1 = one.solve(iters, pool={})[0]
    assert np.array_equal(c1, solved) and np.array_equal(u1, ref[: len(solved)])
    fz = PartSolver(bl, 3, pinned=True, schedule="fused").solve(iters, pool={})
    sp = PartSolver(bl, 3, pinned=True, schedule="split").solve(iters)
    assert sorted(fz) == sorted(sp) == [0, 1, 2]
    for p in fz:
        assert np.array_equal(fz[p][0], sp[p][0])
        assert np.array_equal(fz[p][1], sp[p][1]), (p, float(np.max(np.abs(fz[p][1] - sp[p][1]))))
    with pytest.raises(ValueError):
        PartSolver(bl, 2, schedule="FAST")
    bl.close()
