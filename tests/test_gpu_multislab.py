"""Multi-slab decomposition on the GPU (reading R12):
an in-process group of z-slab contexts exchanging one-plane halos with the same
plans as the NCCL path must equal one context over the whole grid BITWISE, for
both schedules, and match the oracle.  (NCCL itself needs one GPU per rank; the
halo plans are shared and are pinned on CPU by tests/test_slab_gloo.py.)"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
C8 = [-0.875 + 0.25 * b for b in range(8)]


@pytest.mark.parametrize("schedule", ["fused", "split"])
@pytest.mark.parametrize("shape,cuts", [((45, 31, 26), [0, 13, 26]), ((37, 23, 30), [0, 1, 9, 10, 30]),
                                        ((64, 40, 48), [0, 7, 20, 33, 48])])
def test_group_equals_single_context_bitwise(shape, cuts, schedule):
    from paper_2107_14790_b200 import Group, Solver
    h = synth.random_histograms(shape, 21)
    one = Solver(shape, C8).set_schedule(schedule).load(h).iterate(33)
    grp = Group(shape, cuts, C8).set_schedule(schedule).load(h).iterate(33)
    for f in ("u", "v", "p", "q"):
        assert np.array_equal(grp.get(f), one.get(f)), f
    e1, eg = one.energy(), grp.energy()
    for k in ("E", "alpha1", "alpha0", "data", "gap"):
        assert abs(e1[k] - eg[k]) <= 1e-12 * max(1.0, abs(e1[k])), k
    assert e1["vmax"] == eg["vmax"]
    o = oracle.Oracle(shape).load(h).iterate(33, threads=oracle.max_threads())
    assert np.max(np.abs(grp.read_u() - o.u)) <= 1e-4


def test_group_fused_chunks_and_c1(monkeypatch):
    """Slab boundaries combined with fused z-chunks, on the C1 workload at its full count."""
    from paper_2107_14790_b200 import Group, Solver
    monkeypatch.setenv("TGV_FUSED_ZC", "5")
    wl = synth.workload("C1")
    h = synth.make_histograms("C1")
    one = Solver(wl.shape, C8).load(h).iterate(wl.iters)
    grp = Group(wl.shape, [0, 11, 16, 32], C8).load(h).iterate(wl.iters)
    assert np.array_equal(grp.read_u(), one.read_u())


def test_group_errors():
    from paper_2107_14790_b200 import Group, tgv
    shape = (16, 16, 16)
    with pytest.raises(tgv.TgvError):
        Group(shape, [0, 8, 15], C8)  # does not tile [0, nz)
    g = Group(shape, [0, 8, 16], C8)
    with pytest.raises(tgv.TgvError) as ei:
        g.iterate(1)  # not loaded
    assert ei.value.status == tgv.TGV_ESTATE
    g.load(synth.random_histograms(shape, 1))
    with pytest.raises(tgv.TgvError) as ei:
        tgv.tgv_iterate(g.ctxs[0], 1)  # members go through tgv_group_iterate
    assert ei.value.status == tgv.TGV_ESTATE
    g.iterate(2)


@pytest.mark.parametrize("peer", ["1", "0"])
def test_peer_halo_mode_replaces_the_exchange(peer, monkeypatch):
    """Peer halo mode: the fused kernel writes its boundary planes into the
    neighbours' halo planes and hands over with flags, so after the first iteration of a
    call no halo copy runs; TGV_PEER_HALO=0 keeps the per-iteration exchange.  Both are
    bitwise equal to one context."""
    from paper_2107_14790_b200 import Group, Solver, tgv
    monkeypatch.setenv("TGV_PEER_HALO", peer)
    shape, cuts, iters = (61, 35, 29), [0, 7, 8, 20, 29], 12
    h = synth.random_histograms(shape, 21)
    one = Solver(shape, C8).load(h).iterate(iters)
    grp = Group(shape, cuts, C8).load(h)
    for c in grp.ctxs:
        tgv.tgv_set_timing(c, True)
    grp.iterate(iters)
    exchanges = [tgv.tgv_get_timing(c)["halo_exchanges"] for c in grp.ctxs]
    assert np.array_equal(grp.read_u(), one.read_u())
    for f in ("v", "p", "q"):
        assert np.array_equal(grp.get(f), one.get(f)), f
    assert exchanges == ([1] * 4 if peer == "1" else [iters] * 4), exchanges
    # a state change outside iterate (reset) falls back to one exchange, then peer writes again
    for c in grp.ctxs:
        tgv.tgv_reset(c)
    grp.iterate(3)
    one.reset()
    one.iterate(3)
    assert np.array_equal(grp.read_u(), one.read_u())
    e1, eg = one.energy(), grp.energy()
    assert abs(e1["E"] - eg["E"]) <= 1e-12 * abs(e1["E"])
