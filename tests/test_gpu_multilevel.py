"""NEXT-1 coarse-to-fine on the GPU vs the oracle (R18-R20):
restriction bit-exact (integers), prolongation exact, and a full 3-level solve
within the north-star tolerances."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
C8 = [-0.875 + 0.25 * b for b in range(8)]


def test_restriction_bit_exact_and_prolongation_exact():
    from paper_2107_14790_b200 import Solver
    shape = (37, 22, 19)
    h = synth.random_histograms(shape, 4)
    fine = Solver(shape, C8).load(h).iterate(7)
    cshape = tuple((n + 1) // 2 for n in shape)
    coarse = Solver(cshape, C8).restrict_from(fine)
    hc = oracle.restrict_counts(h)
    # the GPU restricted counts start the coarse state exactly like loading hc would
    ref = Solver(cshape, C8).load(hc)
    assert np.array_equal(coarse.read_u(), ref.read_u())
    coarse.iterate(5)
    ref.iterate(5)
    for f in ("u", "v", "p", "q"):
        assert np.array_equal(coarse.get(f), ref.get(f)), f
    # prolongation: parent u, v / 2; duals zero
    fine.prolong_from(coarse)
    u, v = fine.get("u"), fine.get("v")
    up = lambda a: np.repeat(np.repeat(np.repeat(a, 2, -3), 2, -2), 2, -1)[..., :19, :22, :37]
    assert np.array_equal(u, up(coarse.get("u")))
    assert np.array_equal(v, up(coarse.get("v")) * np.float32(0.5))
    assert np.array_equal(fine.get("ubar"), u) and np.array_equal(fine.get("vbar"), v)
    assert np.all(fine.get("p") == 0) and np.all(fine.get("q") == 0)


@pytest.mark.parametrize("schedule", ["fused", "split"])
def test_coarse_to_fine_c1_matches_oracle(schedule):
    from paper_2107_14790_b200.multilevel import coarse_to_fine
    wl = synth.workload("C1")
    h = synth.make_histograms("C1")
    s = coarse_to_fine(wl.shape, h, C8, levels=3, iters=200, schedule=schedule)
    o = oracle.coarse_to_fine(wl.shape, h, levels=3, iters=200, threads=oracle.max_threads())
    du = np.max(np.abs(s.read_u().astype(np.float64) - o.u))
    es, eo = s.energy()["E"], o.energy()["E"]
    assert du <= 1e-4, du
    assert abs(es - eo) / eo <= 1e-5


def test_restrict_errors():
    from paper_2107_14790_b200 import Solver, tgv
    fine = Solver((16, 16, 16), C8).load(synth.random_histograms((16, 16, 16), 1))
    with pytest.raises(tgv.TgvError) as ei:
        Solver((9, 8, 8), C8).restrict_from(fine)
    assert ei.value.status == tgv.TGV_EINVAL
