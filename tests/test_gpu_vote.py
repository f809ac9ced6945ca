"""NEXT-2 GPU histogram voting (Alg. 1) vs the oracle: bit-exact integer counts
(R22), then the voted histograms through the solver."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
C8 = [-0.875 + 0.25 * b for b in range(8)]


def cams_of(wl):
    return [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
             "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_vote_bit_exact(name):
    from paper_2107_14790_b200 import Solver
    wl = synth.workload(name)
    depths = synth.render_depths(wl)
    cams = cams_of(wl)
    s = Solver(wl.shape, C8).vote(cams, depths)
    got = s.read_counts()
    nx, ny, nz = wl.shape
    ref = oracle.alg1_vote(cams, depths, nx, ny, 0, nz)
    assert np.array_equal(got, ref), int(np.sum(got != ref))
    # the state is initialised from the voted histograms exactly as by a host load
    t = Solver(wl.shape, C8).load(ref)
    assert np.array_equal(s.read_u(), t.read_u())


def test_vote_hand_cases_and_weights():
    from paper_2107_14790_b200 import Solver
    yy, xx = np.mgrid[0:64, 0:64]
    depths = [np.full((64, 64), 50.0, np.float32), np.where((xx + yy) % 2 == 0, 40.0, 60.0).astype(np.float32)]
    cams = [{"origin": (0.0, 0.0, 0.0), "rot": np.eye(3), "fx": f, "fy": f, "cx": 32.5, "cy": 32.5, "width": 64,
             "height": 64, "vote_weight": wgt} for f, wgt in ((100.0, 1), (60.0, 5))]
    shape = (3, 4, 25)
    s = Solver(shape, C8).vote(cams, depths, grid_origin=(-1.0, -2.0, 40.0))
    ref = oracle.alg1_vote(cams, depths, 3, 4, 0, 25, origin=(-1.0, -2.0, 40.0))
    assert np.array_equal(s.read_counts(), ref)


def test_vote_then_solve_matches_oracle():
    from paper_2107_14790_b200 import Solver
    wl = synth.workload("C1")
    depths = synth.render_depths(wl)
    cams = cams_of(wl)
    s = Solver(wl.shape, C8).vote(cams, depths).iterate(wl.iters)
    nx, ny, nz = wl.shape
    o = oracle.Oracle(wl.shape).load(oracle.alg1_vote(cams, depths, nx, ny, 0, nz)).iterate(wl.iters)
    assert np.max(np.abs(s.read_u() - o.u)) <= 1e-4


def test_vote_errors():
    from paper_2107_14790_b200 import Solver, tgv
    s = Solver((8, 8, 8), [-0.5, 0.5])
    cam = {"origin": (0.0, 0.0, 0.0), "rot": np.eye(3), "fx": 10.0, "fy": 10.0, "cx": 4.0, "cy": 4.0, "width": 8,
           "height": 8}
    with pytest.raises(tgv.TgvError) as ei:
        s.vote([cam], [np.ones((8, 8), np.float32)])  # 2 bins: Alg. 1 needs 8
    assert ei.value.status == tgv.TGV_EINVAL
