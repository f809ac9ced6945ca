"""Pins of the NEXT-3 block-sparse brick-set oracle (oracle/bricks.py; PAPER.md:221-225
§4.2, :446-453 §4.5 Fig. 9; reading R24).  None of them re-types the oracle's
formulas: each pins it to something it must reduce to.

- adjointness of the masked operators on random brick sets (<D+ w, p> = -<w, D- p> on
  Omega; <grad u, p> = -<u, div p>; <E v, q>_F = -<v, div2 q>), and D+ of a linear
  field is its slope wherever the forward neighbour exists and 0 elsewhere;
- a box-shaped set of solved bricks is the dense grid: the C oracle (pinned in
  test_oracle_*.py) gives the same iterates and energy;
- bricks that touch only along an edge or a corner do not interact: each one is its
  own dense box;
- solved bricks between frozen bricks are the z-slab leaf of reading R23
  (oracle.leaf_from_parent / leaf_step, pinned in test_oracle_leaves.py);
- the restricted gap, including the frozen bricks' terms of the dual, closes on a
  non-box set with frozen bricks (a wrong or missing B term leaves a gap);
- the brick order does not matter.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import bricks as ob

KW = dict(lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25)


def _random_set(rng, n, span=3):
    cells = set()
    while len(cells) < n:
        cells.add(tuple(int(a) for a in rng.integers(0, span, 3)))
    return np.array(sorted(cells))


def _omega(coords, E):
    o = ob.BrickOracle(E, coords)
    return o.om


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_masked_operators_are_adjoint(seed):
    rng = np.random.default_rng(seed)
    E = 3
    om = _omega(_random_set(rng, 6 + seed), E)
    sh = om.shape
    w = rng.standard_normal(sh) * om
    for k in range(3):
        p = rng.standard_normal(sh) * om
        lhs = np.sum(ob.dplus(w, om, k) * p)
        rhs = -np.sum(w * ob.dminus(p, om, k))
        assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1.0)
    p3 = rng.standard_normal((3,) + sh) * om
    assert abs(np.sum(ob.grad(w, om) * p3) + np.sum(w * ob.div(p3, om))) <= 1e-11
    v = rng.standard_normal((3,) + sh) * om
    q = rng.standard_normal((6,) + sh) * om
    e = ob.symgrad(v, om)
    wt = np.array([1, 1, 1, 2, 2, 2.0])[:, None, None, None]  # off-diagonals counted twice (R5)
    lhs = np.sum(wt * e * q)
    rhs = -np.sum(v * ob.div2(q, om))
    assert abs(lhs - rhs) <= 1e-11 * (abs(lhs) + 1.0)


def test_forward_difference_of_a_linear_field():
    rng = np.random.default_rng(4)
    om = _omega(_random_set(rng, 9), 4)
    z, y, x = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in om.shape], indexing="ij")
    lin = 0.5 * x - 0.25 * y + 0.125 * z
    for k, slope in enumerate((0.5, -0.25, 0.125)):
        d = ob.dplus(lin, om, k)
        m = ob.edge(om, k)
        assert np.array_equal(d[m], np.full(int(m.sum()), slope))
        assert not np.any(d[~m])


def _dense_oracle(counts_box, box_xyz, iters):
    return oracle.Oracle(box_xyz, **KW).load(counts_box).iterate(iters)


def _brick_counts(coords, E, dense_counts, lo=(0, 0, 0)):
    out = np.zeros((len(coords), E, E, E, dense_counts.shape[-1]), np.uint32)
    for b, (bx, by, bz) in enumerate(coords):
        x0, y0, z0 = (bx - lo[0]) * E, (by - lo[1]) * E, (bz - lo[2]) * E
        out[b] = dense_counts[z0:z0 + E, y0:y0 + E, x0:x0 + E]
    return out


def test_box_of_solved_bricks_is_the_dense_grid():
    E, nb = 4, (3, 2, 2)  # bricks along x, y, z
    coords = np.array([(bx, by, bz) for bz in range(nb[2]) for by in range(nb[1]) for bx in range(nb[0])])
    rng = np.random.default_rng(0)
    coords = coords[rng.permutation(len(coords))]  # any order
    shape = (nb[0] * E, nb[1] * E, nb[2] * E)
    h = synth.random_histograms(shape, 11)
    bo = ob.BrickOracle(E, coords, **KW).load(_brick_counts(coords, E, h)).iterate(25)
    do = _dense_oracle(h, shape, 25)
    for name in ("u", "v", "p", "q"):
        assert np.max(np.abs(getattr(bo, name) - do.get(name))) <= 1e-12, name
    eb, ed = bo.energy(), do.energy()
    for k in ("E", "alpha1", "alpha0", "data", "gap", "vmax"):
        assert abs(eb[k] - ed[k]) <= 1e-10 * max(1.0, abs(ed[k])), k


def test_bricks_touching_at_an_edge_or_corner_do_not_interact():
    E = 4
    coords = np.array([(0, 0, 0), (1, 1, 0), (2, 2, 1)])  # (0,0,0)-(1,1,0) share an edge, (1,1,0)-(2,2,1) a corner
    hs = [synth.random_histograms((E, E, E), 20 + b) for b in range(3)]
    bo = ob.BrickOracle(E, coords, **KW).load(np.stack(hs)).iterate(20)
    u = bo.get("u")
    for b in range(3):
        do = _dense_oracle(hs[b], (E, E, E), 20)
        assert np.max(np.abs(u[b] - do.u)) <= 1e-12


def test_solved_bricks_between_frozen_bricks_are_the_slab_leaf():
    E = 4
    nx, ny, nz = 8, 4, 16  # bricks 2 x 1 x 4: z-bricks 1, 2 solved, 0 and 3 frozen
    shape = (nx, ny, nz)
    zb, ze = 4, 12
    coords = np.array([(bx, 0, bz) for bz in range(4) for bx in range(2)])
    frozen = coords[:, 2] % 3 == 0
    h = synth.random_histograms(shape, 13)
    rng = np.random.default_rng(2)
    cshape = (nx // 2, ny // 2, nz // 2)
    pu = rng.uniform(-1, 1, cshape[::-1])
    pv = rng.uniform(-0.3, 0.3, (3,) + cshape[::-1])
    leaf = oracle.leaf_from_parent(shape, zb, ze, h[zb:ze], pu, pv, **KW)

    def up(a):
        return np.repeat(np.repeat(np.repeat(a, 2, axis=-3), 2, axis=-2), 2, axis=-1)

    U, Vv = up(pu), up(pv) * 0.5
    bu =np.stack([U[bz * E:(bz + 1) * E, :, bx * E:(bx + 1) * E] for bx, _, bz in coords])
    bv = np.stack([Vv[:, bz * E:(bz + 1) * E, :, bx * E:(bx + 1) * E] for bx, _, bz in coords])
    bo = ob.BrickOracle(E, coords, frozen=frozen, **KW).load(_brick_counts(coords, E, h)).set_primal(bu, bv)
    for _ in range(15):
        oracle.leaf_step(leaf)
        bo.iterate(1)
    assert np.max(np.abs(bo.u[zb:ze] - leaf.u)) <= 1e-12
    assert np.max(np.abs(bo.v[:, zb:ze] - leaf.get("v"))) <= 1e-12
    # the frozen bricks kept their values
    assert np.array_equal(bo.get("u")[frozen], bu[frozen])


def test_gap_closes_with_frozen_bricks_on_a_non_box_set():
    E = 2
    coords = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (1, 1, 1), (2, 1, 1), (0, 1, 0)])
    frozen = np.array([False, False, False, False, True, True])
    rng = np.random.default_rng(5)
    h = rng.integers(0, 6, (len(coords), E, E, E, 8)).astype(np.uint32)
    fu = rng.uniform(-0.8, 0.8, (len(coords), E, E, E))
    fv = rng.uniform(-0.2, 0.2, (len(coords), 3, E, E, E))
    bo = ob.BrickOracle(E, coords, frozen=frozen, **KW).load(h)
    bo.set_primal(np.where(frozen[:, None, None, None], fu, bo.get("u")), fv * frozen[:, None, None, None, None])
    gaps = []
    for n in (8, 64, 512, 4096, 16384):
        bo.iterate(n - (0 if not gaps else prev))
        prev = n
        en = bo.energy()
        gaps.append(en["gap"])
        assert en["vmax"] <= 2.0
        assert en["gap"] >= -1e-9 * en["E"]
    assert gaps[-1] <= 1e-6 * bo.energy()["E"], gaps
    # dropping the frozen bricks' terms from the dual would leave a gap the size of
    # their stencil coupling: make sure that term is not negligible here
    om, A = bo.om, bo.act
    d = ob.div(bo.p, om)
    w = bo.p + ob.div2(bo.q, om)
    dB = -bo.u * d - np.sum(bo.v * w, axis=0)
    assert abs(np.sum(dB[om & ~A])) > 1e-3


def test_brick_order_does_not_matter():
    E = 3
    rng = np.random.default_rng(8)
    coords = _random_set(rng, 7)
    frozen = rng.random(len(coords)) < 0.3
    h = rng.integers(0, 5, (len(coords), E, E, E, 8)).astype(np.uint32)
    a = ob.BrickOracle(E, coords, frozen=frozen, **KW).load(h).iterate(12)
    perm = rng.permutation(len(coords))
    b = ob.BrickOracle(E, coords[perm], frozen=frozen[perm], **KW).load(h[perm]).iterate(12)
    assert np.array_equal(a.get("u")[perm], b.get("u"))
    assert np.array_equal(a.get("v")[perm], b.get("v"))


def test_solved_iterates_do_not_depend_on_duals_outside_S():
    """R24: the primal step on A reads duals only on S = A + frozen voxels face-adjacent
    to A, so updating the duals on every voxel of Omega leaves A's iterates unchanged."""
    E = 3
    rng = np.random.default_rng(9)
    coords = _random_set(rng, 10)
    frozen = rng.random(len(coords)) < 0.4
    frozen[0] = False
    h = rng.integers(0, 5, (len(coords), E, E, E, 8)).astype(np.uint32)
    fu = rng.uniform(-0.8, 0.8, (len(coords), E, E, E))
    fv = rng.uniform(-0.2, 0.2, (len(coords), 3, E, E, E))
    a = ob.BrickOracle(E, coords, frozen=frozen, **KW).load(h).set_primal(fu, fv)
    b = ob.BrickOracle(E, coords, frozen=frozen, **KW).load(h).set_primal(fu, fv)
    b.S = b.om.copy()  # duals everywhere
    assert (a.S != a.om).any()
    a.iterate(15)
    b.iterate(15)
    assert np.array_equal(a.u[a.act], b.u[b.act])
    assert np.array_equal(a.v[:, a.act], b.v[:, b.act])
    assert not np.any(a.p[:, ~a.S]) and not np.any(a.q[:, ~a.S])
