"""Host logic of the brick levels (paper_2107_14790_b200.brick_levels; R25,
R26), checked on CPU: which bricks a finer level gets, its frozen shell, and the
Morton parts of the finest level.  No device work (the module's GPU calls are not
made here)."""
import itertools

import numpy as np

from paper_2107_14790_b200 import brick_levels as blv


def _set(c):
    return {tuple(int(t) for t in x) for x in np.asarray(c).reshape(-1, 3)}


def test_brick_grid_rounds_up():
    assert blv.brick_grid((2048, 2048, 256), 32, 0) == (64, 64, 8)
    assert blv.brick_grid((2048, 2048, 256), 32, 2) == (16, 16, 2)
    assert blv.brick_grid((33, 32, 1), 32, 0) == (2, 1, 1)


def test_children_of_flagged_octants():
    coords = np.array([(0, 0, 0), (1, 2, 0)])
    flags = np.zeros((2, 8), np.uint8)
    flags[0, 0] = flags[0, 7] = 1  # octants (0,0,0) and (1,1,1)
    flags[1, 5] = 1                # octant (1,0,1)
    got = blv.children(coords, flags, (8, 8, 8))
    assert _set(got) == {(0, 0, 0), (1, 1, 1), (3, 4, 1)}
    # sorted z, then y, then x
    assert [tuple(x) for x in got] == sorted(_set(got), key=lambda t: (t[2], t[1], t[0]))
    # octants outside the finer grid are dropped
    assert _set(blv.children(coords, flags, (3, 8, 8))) == {(0, 0, 0), (1, 1, 1)}


def test_shell_is_the_26_neighbourhood_minus_the_set():
    rng = np.random.default_rng(0)
    grid = (6, 5, 4)
    A = {tuple(int(t) for t in rng.integers(0, g)) for g in [grid] * 1 for _ in range(12)}
    A = np.array(sorted(A))
    got = _set(blv.shell(A, grid))
    want = set()
    for a in _set(A):
        for d in itertools.product((-1, 0, 1), repeat=3):
            n = tuple(a[i] + d[i] for i in range(3))
            if all(0 <= n[i] < grid[i] for i in range(3)) and n not in _set(A):
                want.add(n)
    assert got == want
    # every shell brick's parent lies in the parent set or its 26-neighbourhood (R25)
    parents = _set(np.asarray(A) // 2)
    pshell = _set(blv.shell(np.array(sorted(parents)), tuple((g + 1) // 2 for g in grid)))
    for b in got:
        assert tuple(t // 2 for t in b) in parents | pshell


def test_morton_parts_partition_the_solved_bricks():
    rng = np.random.default_rng(1)
    cells = {tuple(int(t) for t in rng.integers(0, 16, 3)) for _ in range(300)}
    A = np.array(sorted(cells))
    for n in (1, 3, 8):
        parts = blv.split_parts(A, n)
        assert len(parts) == n
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1
        allp = [x for p in parts for x in _set(p)]
        assert len(allp) == len(A) and set(allp) == _set(A)  # disjoint cover
        # Morton-contiguous: the parts' code ranges do not interleave
        rngs = sorted((int(blv.morton(p).min()), int(blv.morton(p).max())) for p in parts)
        for (a0, a1), (b0, b1) in zip(rngs, rngs[1:]):
            assert a1 < b0


def test_morton_code_interleaves_bits():
    c = np.array([(1, 0, 0), (0, 1, 0), (0, 0, 1), (3, 0, 0), (0, 0, 2), (5, 3, 6)])
    m = blv.morton(c)
    assert list(m[:5]) == [1, 2, 4, 9, 32]
    x, y, z = 5, 3, 6
    ref = sum(((x >> i & 1) << (3 * i)) | ((y >> i & 1) << (3 * i + 1)) | ((z >> i & 1) << (3 * i + 2)) for i in range(8))
    assert int(m[5]) == ref


def test_mixed_border_is_a_balanced_disjoint_set_around_A():
    """R27 host logic: the mixed finest level (A plus its frozen face border, level-0 where
    the parent cube holds A, else the parent cube) is disjoint and 2:1 balanced (the oracle's
    own checks), covers every face neighbour of A, and has only face neighbours of A (or
    their parents) in B."""
    from oracle import mixed as om
    from paper_2107_14790_b200.brick_levels import mixed_border
    rng = np.random.default_rng(3)
    grid = (8, 8, 6)
    A = np.unique(rng.integers(0, [8, 8, 6], (40, 3)), axis=0)
    coords, levels, frozen = mixed_border(A, grid)
    om.check_balanced(2, levels, coords)  # E = 2: the smallest brick-aligned geometry
    fine = {tuple(c) for c, l in zip(coords, levels) if l == 0}
    coarse = {tuple(c) for c, l in zip(coords, levels) if l == 1}
    assert {tuple(a) for a in A} <= fine and not frozen[:len(A)].any() and frozen[len(A):].all()
    for a in A:
        for d in ([1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]):
            n = a + np.array(d)
            if np.any(n < 0) or np.any(n >= grid):
                continue
            assert tuple(n) in fine or tuple(n >> 1) in coarse
    for c, l in zip(coords[len(A):], levels[len(A):]):
        kids = [np.array(c)] if l == 0 else [2 * np.array(c) + np.array(o) for o in np.ndindex(2, 2, 2)]
        assert any(np.abs(k - a).sum() == 1 for k in kids for a in A)
