"""GPU (libtgv.so through the C ABI) vs the fp64 CPU oracle on the same seeded
inputs (SURVEY.md §8(c) "GPU vs oracle parity"; north_star tolerances):

    max |u_gpu - u_cpu| <= 1e-4   and   |E_gpu - E_cpu| / |E_cpu| <= 1e-5

after the stated iteration count.  Sizes: the C1 workload at its full count,
ragged grids spanning several 32x8 tiles with partial tiles and size-1 axes,
a 64^3 window of the C2 workload at C2's full 500 iterations, and the full
256^3 C2 grid (the bench's launch configuration) at a truncated count plus
properties that hold at any size at the full count.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

U_TOL = 1e-4
E_RTOL = 1e-5
GAP_RTOL = 1e-5  # |gap_gpu - gap_cpu| / |E_cpu|
VMAX_TOL = 1e-4
NT = max(1, oracle.max_threads())


def solver_cls():
    from paper_2107_14790_b200 import Solver
    return Solver


def params(wl=None, **kw):
    p = dict(lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25)
    if wl is not None:
        p = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
    p.update(kw)
    return p


SCHEDULES = ["fused", "split"]


def pair(shape, counts, iters, centers=None, schedule="fused", **kw):
    c = oracle.default_centers(8) if centers is None else np.asarray(centers, np.float64)
    p = params(**kw)
    o = oracle.Oracle(shape, centers=c, **p).load(counts).iterate(iters, threads=NT)
    s = solver_cls()(shape, [float(x) for x in c], **p).set_schedule(schedule)
    s.load(np.ascontiguousarray(counts, np.uint32)).iterate(iters)
    return o, s


def assert_parity(o, s, u_tol=U_TOL, e_rtol=E_RTOL):
    du = np.max(np.abs(s.read_u().astype(np.float64) - o.u))
    eo, es = o.energy(), s.energy()
    rel = abs(es["E"] - eo["E"]) / max(abs(eo["E"]), 1e-300)
    assert du <= u_tol, f"max|du| = {du}"
    assert rel <= e_rtol, f"energy rel diff {rel} (gpu {es['E']}, cpu {eo['E']})"
    for k in ("alpha1", "alpha0", "data"):
        assert abs(es[k] - eo[k]) <= 1e-4 * max(1.0, abs(eo["E"])), k
    # (a4) the restricted gap E - D_V (R14) and max|v|: the fp32 iterates differ from the fp64
    # ones by ~1e-7, and every term of D_V is O(1)-Lipschitz in them
    dgap = abs(es["gap"] - eo["gap"])
    assert dgap <= GAP_RTOL * max(1.0, abs(eo["E"])), f"gap {es['gap']} vs {eo['gap']}"
    assert abs(es["vmax"] - eo["vmax"]) <= VMAX_TOL, f"max|v| {es['vmax']} vs {eo['vmax']}"
    return du, rel


def test_init_matches():
    shape = (37, 23, 19)
    h = synth.random_histograms(shape, 1)
    o, s = pair(shape, h, 0)
    np.testing.assert_allclose(s.read_u(), o.u, rtol=0, atol=6e-8)
    assert np.all(s.get("ubar") == s.read_u())
    for f in ("v", "vbar", "p", "q"):
        assert np.all(s.get(f) == 0)


@pytest.mark.parametrize("schedule", SCHEDULES)
@pytest.mark.parametrize("shape", [(37, 23, 19), (64, 16, 5), (1, 1, 9), (33, 1, 4), (2, 70, 3), (61, 29, 40)])
def test_one_iteration_from_random_state(shape, schedule):
    """Every stencil path (interior, all six boundary faces, projections active) in one step."""
    nx, ny, nz = shape
    rng = np.random.default_rng(7)
    h = synth.random_histograms(shape, 2)
    c = oracle.default_centers(8)
    o = oracle.Oracle(shape, **params()).load(h)
    s = solver_cls()(shape, list(c), **params()).set_schedule(schedule).load(h)
    st = {"u": rng.uniform(-1, 1, (nz, ny, nx)), "ubar": rng.uniform(-1.5, 1.5, (nz, ny, nx)),
          "v": rng.normal(0, 0.5, (3, nz, ny, nx)), "vbar": rng.normal(0, 0.5, (3, nz, ny, nx)),
          "p": rng.normal(0, 0.7, (3, nz, ny, nx)), "q": rng.normal(0, 1.0, (6, nz, ny, nx))}
    for k in ("u", "ubar", "v", "vbar", "p", "q"):  # u / v before ubar / vbar (tgv_write_field)
        a = st[k]
        a32 = a.astype(np.float32)
        s.set(k, a32)
        o.set(k, a32.astype(np.float64))
    o.iterate(1)
    s.iterate(1)
    for f in ("p", "q", "u", "ubar", "v", "vbar"):
        np.testing.assert_allclose(s.get(f), o.get(f), rtol=0, atol=3e-6, err_msg=f)


def random_state(shape, seed, model="tgv"):
    nx, ny, nz = shape
    rng = np.random.default_rng(seed)
    st = {"u": rng.uniform(-1, 1, (nz, ny, nx)), "p": rng.normal(0, 0.7, (3, nz, ny, nx))}
    if model == "tgv":
        st.update(v=rng.normal(0, 0.5, (3, nz, ny, nx)), q=rng.normal(0, 1.0, (6, nz, ny, nx)))
    return {k: a.astype(np.float32) for k, a in st.items()}


@pytest.mark.parametrize("model", ["tgv", "tvl1"])
@pytest.mark.parametrize("shape,nb,scale", [((37, 23, 19), 8, 1), ((64, 16, 5), 8, 1), ((1, 1, 9), 8, 1),
                                            ((33, 1, 4), 8, 1), ((70, 9, 21), 3, 1), ((29, 14, 12), 16, 1),
                                            ((40, 33, 17), 8, 100)])
def test_energy_terms_from_random_state(shape, nb, scale, model):
    """(a4) tgv_energy on a state both sides hold bit-identically (random u, v, p, q with every
    boundary face and large ||p + div2 q||_1): E, its three terms, the restricted gap E - D_V
    (R14, V = 2; TV-L1 V = 0) and max|v| equal the oracle's up to the kernel's fp32 per-voxel
    rounding (fp64 sums).  Counts up to 100x (u16), 3 / 8 / 16 bins with non-uniform centres."""
    nx, ny, nz = shape
    rng = np.random.default_rng(nb * 1000 + nx)
    if nb == 8:
        c = oracle.default_centers(8)
    else:
        c = np.sort(rng.uniform(-0.97, 0.97, nb)).astype(np.float32).astype(np.float64)
    h = (rng.integers(0, 6, size=(nz, ny, nx, nb)) * scale).astype(np.uint32)
    o = oracle.Oracle(shape, centers=c, model=model, **params()).load(h)
    s = solver_cls()(shape, [float(x) for x in c], **params()).set_model(model).load(h)
    st = random_state(shape, 40 + nx, model)
    for k in ("u", "v", "p", "q"):
        if k in st:
            s.set(k, st[k])
            o.set(k, st[k].astype(np.float64))
    for k in ("u", "v", "p", "q"):
        if k in st:
            assert np.array_equal(s.get(k), st[k]), k
    eo, es = o.energy(), s.energy()
    # the kernel forms each voxel's terms in fp32 from the (identical) fp32 state and sums
    # them in fp64: relative error ~1e-7 of the summed magnitudes |E| + |D_V|
    tol = 2e-6 * max(1.0, abs(eo["E"]), abs(eo["dual"]))
    for k in ("E", "alpha1", "alpha0", "data", "gap"):
        assert abs(es[k] - eo[k]) <= tol, (k, es[k], eo[k], tol)
    assert es["vmax"] == eo["vmax"]
    # the V term matters here: it moves the gap by far more than the tolerance
    assert model == "tvl1" or abs(o.energy(V=0.0)["gap"] - eo["gap"]) > 100 * tol


@pytest.mark.parametrize("shape,nb,scale", [((37, 23, 19), 8, 1), ((1, 1, 9), 8, 1), ((33, 1, 4), 8, 1),
                                            ((29, 14, 12), 16, 1), ((40, 33, 17), 8, 100), ((70, 9, 21), 16, 100),
                                            ((96, 45, 300), 8, 1), ((300, 450, 3), 8, 1), ((320, 140, 96), 8, 1)])
def test_energy_sweeps_agree(shape, nb, scale, monkeypatch):
    """(a4) the three energy sweeps -- TMA-staged with one CTA per SM (TGV_ENERGY_IMPL=tma) or
    two (=tma2, u8 counts and 8 bins; the default picks by grid size) and register-streaming
    (=regs) -- form the same fp32
    per-voxel terms and differ only in the order of the fp64 sums; max|v| is exact; each is
    deterministic.  Ragged tiles, size-1 axes, u8 / u16 counts, 8 / 16 bins, and a 300-plane
    grid (lock-step chunks, round sync, split remainder segments)."""
    nx, ny, nz = shape
    rng = np.random.default_rng(nb * 7 + nx)
    c = oracle.default_centers(nb)
    h = (rng.integers(0, 6, size=(nz, ny, nx, nb)) * scale).astype(np.uint32)
    s = solver_cls()(shape, [float(x) for x in c], **params()).load(h)
    for k, a in random_state(shape, 90 + nx, "tgv").items():
        s.set(k, a)
    ed = s.energy()  # default: the TMA sweep
    monkeypatch.setenv("TGV_ROUND_SYNC", "0")  # the round sync only orders the items
    assert s.energy() == ed
    monkeypatch.delenv("TGV_ROUND_SYNC")
    monkeypatch.setenv("TGV_ENERGY_IMPL", "regs")
    er = s.energy()
    for impl in ("tma", "tma2", None):
        if impl:
            monkeypatch.setenv("TGV_ENERGY_IMPL", impl)
        else:
            monkeypatch.delenv("TGV_ENERGY_IMPL")
        et = s.energy()
        assert s.energy() == et  # deterministic
        for k in ("E", "alpha1", "alpha0", "data", "gap"):
            assert abs(et[k] - er[k]) <= 1e-12 * max(1.0, abs(er["E"]), abs(er["gap"])), (impl, k, et[k], er[k])
        assert et["vmax"] == er["vmax"], impl
    assert et == ed


@pytest.mark.parametrize("schedule", SCHEDULES)
def test_c1_full_count(schedule):
    wl = synth.workload("C1")
    h = synth.make_histograms("C1")
    o, s = pair(wl.shape, h, wl.iters, schedule=schedule, **params(wl))
    du, rel = assert_parity(o, s)
    print(f"C1 x{wl.iters} ({schedule}): max|du| = {du:.3e}, rel dE = {rel:.3e}")


@pytest.mark.parametrize("schedule", SCHEDULES)
@pytest.mark.parametrize("shape,seed", [((37, 23, 19), 3), ((1, 1, 40), 4), ((33, 1, 7), 5), ((129, 9, 4), 6),
                                        ((1, 1, 1), 7), ((5, 64, 3), 8), ((91, 45, 70), 9)])
def test_ragged_shapes(shape, seed, schedule):
    h = synth.random_histograms(shape, seed)
    o, s = pair(shape, h, 60, schedule=schedule)
    assert_parity(o, s)


@pytest.mark.parametrize("schedule", SCHEDULES)
def test_nonuniform_centres_and_16_bins(schedule):
    shape = (21, 13, 11)
    rng = np.random.default_rng(9)
    for nb in (3, 16):
        c = np.sort(rng.uniform(-0.95, 0.95, nb)).astype(np.float32).astype(np.float64)
        h = rng.integers(0, 5, size=(11, 13, 21, nb)).astype(np.uint32)
        o, s = pair(shape, h, 40, centers=c, schedule=schedule)
        assert_parity(o, s)


def test_u16_counts_and_large_votes(monkeypatch):
    """Counts above 255 keep u16 storage; LIDAR-style vote weight 5."""
    shape = (33, 17, 9)
    h = synth.random_histograms(shape, 11) * np.uint32(5)
    h[2, 3, 4, 6] = 300
    for sched in SCHEDULES:
        o, s = pair(shape, h, 50, schedule=sched)
        assert s.info()["count_bytes"] == 2
        assert_parity(o, s)


def test_schedules_and_count_widths_agree_bitwise(monkeypatch):
    """FUSED and SPLIT evaluate the same fp32 expressions; u8 and u16 counts are the same integers."""
    shape = (67, 41, 23)
    h = synth.random_histograms(shape, 12)
    c = list(oracle.default_centers(8))
    outs = {}
    for sched, impl in (("fused", "tma"), ("fused", "regs"), ("split", "-")):
        for force16 in ("0", "1"):
            monkeypatch.setenv("TGV_FORCE_U16", force16)
            monkeypatch.setenv("TGV_FUSED_IMPL", impl)
            s = solver_cls()(shape, c).set_schedule(sched).load(h).iterate(37)
            assert s.info()["count_bytes"] == (2 if force16 == "1" else 1)
            if sched == "fused":
                assert s.info()["fused_tma"] == (impl == "tma")
            outs[(sched, impl, force16)] = {f: s.get(f) for f in ("u", "v", "p", "q")}
            s.close()
    ref = outs[("split", "-", "1")]
    for key, o in outs.items():
        for f in ("u", "v", "p", "q"):
            assert np.array_equal(o[f], ref[f]), (key, f, np.max(np.abs(o[f] - ref[f])))


@pytest.mark.parametrize("knobs", [{"TGV_ROUND_SYNC": "1"}])
@pytest.mark.parametrize("shape", [(256, 140, 43), (512, 150, 12), (45, 31, 26)])
def test_fused_schedule_knobs_equal_default_bitwise(monkeypatch, knobs, shape):
    """The lock-step round sync (TGV_ROUND_SYNC, default: CTAs wait for each round before the
    next) only orders the work: many rounds of (tile, short chunk) items plus remainder
    segments, bitwise the unsynchronised sweep, over launches in a row (the round counter
    resets at the end of each launch)."""
    monkeypatch.setenv("TGV_FUSED_ZC", "4" if shape[2] > 20 else "3")
    h = synth.random_histograms(shape, 15)
    c = list(oracle.default_centers(8))
    outs = []
    for on in (False, True):
        for k, v in knobs.items():
            monkeypatch.setenv(k, v if on else "0")
        s = solver_cls()(shape, c).load(h).iterate(7)
        outs.append({f: s.get(f) for f in ("u", "v", "p", "q")})
        s.close()
    for f in ("u", "v", "p", "q"):
        assert np.array_equal(outs[0][f], outs[1][f]), f


def test_tvl1_round_sync_equals_unsynchronised_bitwise(monkeypatch):
    """TV-L1's TMA sweep (two CTAs per SM) under the lock-step round sync: bitwise the
    unsynchronised sweep over many rounds of short chunks."""
    shape = (256, 140, 43)
    monkeypatch.setenv("TGV_FUSED_ZC", "2")
    h = synth.random_histograms(shape, 17)
    c = list(oracle.default_centers(8))
    outs = []
    for on in ("0", "1"):
        monkeypatch.setenv("TGV_ROUND_SYNC", on)
        s = solver_cls()(shape, c).set_model("tvl1").load(h).iterate(9)
        outs.append({f: s.get(f) for f in ("u", "p")})
        s.close()
    for f in ("u", "p"):
        assert np.array_equal(outs[0][f], outs[1][f]), f


@pytest.mark.parametrize("impl", ["tma", "regs"])
@pytest.mark.parametrize("zc", [1, 3, 7, 64])
def test_fused_chunk_sizes(monkeypatch, zc, impl):
    """z-chunk boundaries of the fused kernel (redundant halo planes) do not change the result."""
    monkeypatch.setenv("TGV_FUSED_ZC", str(zc))
    monkeypatch.setenv("TGV_FUSED_IMPL", impl)
    shape = (45, 31, 26)
    h = synth.random_histograms(shape, 13)
    o, s = pair(shape, h, 30, schedule="fused")
    assert s.info()["fused_zc"] == zc
    assert_parity(o, s)


def test_special_cases_exact():
    S = solver_cls()
    c = list(oracle.default_centers(8))
    s = S((9, 7, 5), c).load(np.zeros((5, 7, 9, 8), np.uint32)).iterate(20)
    assert np.all(s.read_u() == 0.0)
    h = np.array([3, 0, 1, 0, 0, 2, 5, 1], np.uint32)
    s = S((9, 7, 5), c).load(np.broadcast_to(h, (5, 7, 9, 8)).copy()).iterate(5)
    assert np.all(s.read_u() == 0.375)  # weighted-median limit (tests/test_oracle_scheme.py)


@pytest.mark.parametrize("schedule", SCHEDULES)
def test_c2_window_full_count(schedule):
    """A 64^3 window of the C2 workload (sphere + plane, noise, floaters) at C2's 500 iterations."""
    wl = synth.workload("C2")
    h = synth.make_histograms("C2", 118, 182)[:, 96:160, 96:160]
    h = np.ascontiguousarray(h)
    o, s = pair((64, 64, 64), h, wl.iters, schedule=schedule, **params(wl))
    du, rel = assert_parity(o, s)
    print(f"C2 window 64^3 x{wl.iters}: max|du| = {du:.3e}, rel dE = {rel:.3e}")


def test_c2_full_grid_truncated_count():
    """Full 256^3 C2 grid in the bench's launch configuration, every voxel compared."""
    wl = synth.workload("C2")
    h = synth.make_histograms("C2")
    o, s = pair(wl.shape, h, 6, schedule="fused", **params(wl))
    assert_parity(o, s)
    s.set_schedule("split")
    s.reset()
    s.iterate(6)
    assert_parity(o, s)


def test_c2_full_grid_full_count():
    """C2 (BASELINE configs[1]) as the bench runs it: the full 256^3 grid at its stated 500
    iterations, every voxel of u, E, its terms, the restricted gap and max|v| against the
    oracle solving the same full grid (north-star tolerances)."""
    wl = synth.workload("C2")
    h = synth.make_histograms("C2")
    o, s = pair(wl.shape, h, wl.iters, schedule="fused", **params(wl))
    du, rel = assert_parity(o, s)
    eo, es = o.energy(), s.energy()
    print(f"C2 256^3 x{wl.iters}: max|du| = {du:.3e}, rel dE = {rel:.3e}, gap {es['gap']:.6g} vs {eo['gap']:.6g}")


def test_c2_full_count_properties():
    wl = synth.workload("C2")
    h = synth.make_histograms("C2")
    s = solver_cls()(wl.shape, list(wl.centers), **params(wl)).load(h)
    it, gaps, Es = 0, [], []
    for ck in (8, 16, 32, 64, 128, 256, wl.iters):
        s.iterate(ck - it)
        it = ck
        e = s.energy()
        gaps.append(e["gap"])
        Es.append(e["E"])
        assert e["vmax"] <= 2.0 and e["gap"] >= -1e-6 * e["E"]
    u1 = s.read_u()
    assert np.all(np.abs(u1) <= 1.0)
    assert Es[-1] <= Es[0]
    assert all(b <= a * (1 + 1e-6) for a, b in zip(gaps, gaps[1:])), gaps
    s.reset()
    s.iterate(wl.iters)
    assert np.array_equal(s.read_u(), u1)  # deterministic


def test_error_paths():
    from paper_2107_14790_b200 import tgv
    S = solver_cls()
    c = list(oracle.default_centers(8))
    s = S((8, 8, 8), c)
    with pytest.raises(tgv.TgvError) as ei:
        s.iterate(1)
    assert ei.value.status == tgv.TGV_ESTATE
    with pytest.raises(tgv.TgvError) as ei:
        s.load(np.zeros((8, 8, 8, 7), np.uint32))
    assert ei.value.status == tgv.TGV_EINVAL
    h = np.zeros((8, 8, 8, 8), np.uint32)
    h[3, 4, 5, 2] = 70000
    with pytest.raises(tgv.TgvError) as ei:
        s.load(h)
    assert ei.value.status == tgv.TGV_ERANGE
    s.load(np.ones((8, 8, 8, 8), np.uint32))
    with pytest.raises(tgv.TgvError) as ei:
        s.iterate(-1)
    assert ei.value.status == tgv.TGV_EINVAL
    s.iterate(2)


# ---------------------------------------------------------------------------
# NEXT-4 TV-L1 model (Eq. 1; R21)
@pytest.mark.parametrize("schedule", ["fused", "split"])
@pytest.mark.parametrize("shape,iters", [((37, 23, 19), 60), ((1, 1, 40), 200), ((64, 64, 64), 500)])
def test_tvl1_matches_oracle(shape, iters, schedule):
    if shape == (64, 64, 64):
        h = np.ascontiguousarray(synth.make_histograms("C2", 118, 182)[:, 96:160, 96:160])
    else:
        h = synth.random_histograms(shape, 31)
    c = oracle.default_centers(8)
    o = oracle.Oracle(shape, model="tvl1").load(h).iterate(iters, threads=NT)
    s = solver_cls()(shape, list(c)).set_schedule(schedule).set_model("tvl1").load(h).iterate(iters)
    assert s.info()["model"] == 1
    du, rel = assert_parity(o, s)
    assert np.all(s.get("v") == 0) and np.all(s.get("q") == 0)
    assert abs(s.energy()["gap"] - o.energy()["gap"]) <= 1e-4 * o.energy()["E"]


@pytest.mark.parametrize("schedule", ["fused", "split"])
def test_tvl1_group_equals_single(schedule):
    from paper_2107_14790_b200 import Group
    shape = (40, 30, 27)
    h = synth.random_histograms(shape, 32)
    c = list(oracle.default_centers(8))
    one = solver_cls()(shape, c).set_schedule(schedule).set_model("tvl1").load(h).iterate(25)
    grp = Group(shape, [0, 9, 10, 20, 27], c).set_schedule(schedule).set_model("tvl1").load(h).iterate(25)
    assert np.array_equal(grp.read_u(), one.read_u())
    assert np.array_equal(grp.get("p"), one.get("p"))


@pytest.mark.parametrize("impl", ["tma", "regs"])
@pytest.mark.parametrize("zc", ["0", "1", "3", "7"])
def test_tvl1_fused_equals_split_bitwise(zc, impl, monkeypatch):
    """The NEXT-4 single sweeps (TMA and register kernels) do the two kernels'
    arithmetic expression for expression: bitwise equal for any z-chunking, u8 and
    u16 counts, 3 bins."""
    monkeypatch.setenv("TGV_FUSED_ZC", zc)
    if impl == "regs":
        monkeypatch.setenv("TGV_FUSED_IMPL", "regs")
    for shape, h, c in (((45, 31, 22), synth.random_histograms((45, 31, 22), 33), list(oracle.default_centers(8))),
                        ((33, 17, 9), synth.random_histograms((33, 17, 9), 34) * 40, list(oracle.default_centers(8))),
                        ((29, 14, 12), np.ascontiguousarray(synth.random_histograms((29, 14, 12), 35)[..., :3]), [-0.5, 0.1, 0.7])):
        a = solver_cls()(shape, c).set_schedule("fused").set_model("tvl1").load(h).iterate(17)
        b = solver_cls()(shape, c).set_schedule("split").set_model("tvl1").load(h).iterate(17)
        assert np.array_equal(a.read_u(), b.read_u())
        assert np.array_equal(a.get("p"), b.get("p"))


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.uint32])
def test_staged_load_and_async_read_equal_the_synchronous_path(dtype):
    """Pipelined host I/O (include/tgv.h tgv_stage_histograms / tgv_load_staged /
    tgv_read_u_async): staged counts of any width give the state tgv_load_histograms gives,
    bit for bit; a second staging while the first solve runs replaces it; the asynchronous u
    read returns the iterate it was ordered after."""
    import torch
    from paper_2107_14790_b200 import tgv
    shape = (45, 31, 22)
    c = list(oracle.default_centers(8))
    h1 = synth.random_histograms(shape, 51)
    h2 = synth.random_histograms(shape, 52)
    ref = []
    for h in (h1, h2):
        s = solver_cls()(shape, c).load(h).iterate(13)
        ref.append(s.read_u().copy())
        s.close()
    s = solver_cls()(shape, c)
    def pinned(a):  # page-locked host copy of any dtype (a uint8 torch buffer viewed as the array)
        buf = torch.empty(a.nbytes, dtype=torch.uint8).pin_memory().numpy()
        out_ = buf.view(a.dtype).reshape(a.shape)
        out_[...] = a
        return out_
    pin = [pinned(np.ascontiguousarray(h.astype(dtype))) for h in (h1, h2)]
    out = [torch.empty((shape[2], shape[1], shape[0]), dtype=torch.float32).pin_memory() for _ in range(2)]
    tgv.tgv_stage_histograms(s.ctx, pin[0])
    tgv.tgv_load_staged(s.ctx)
    tgv.tgv_stage_histograms(s.ctx, pin[1])  # overlaps the next solve
    s.iterate(13)
    tgv.tgv_read_u_async(s.ctx, out[0])
    tgv.tgv_load_staged(s.ctx)
    s.iterate(13)
    tgv.tgv_read_u_async(s.ctx, out[1])
    tgv.tgv_wait_io(s.ctx)
    assert np.array_equal(out[0].numpy(), ref[0])
    assert np.array_equal(out[1].numpy(), ref[1])
    with pytest.raises(tgv.TgvError) as ei:
        tgv.tgv_load_staged(s.ctx)  # nothing staged any more
    assert ei.value.status == tgv.TGV_ESTATE
    s.close()


@pytest.mark.parametrize("model,schedule", [("tgv", "fused"), ("tgv", "split"), ("tvl1", "fused"), ("tvl1", "split")])
def test_graph_replay_equals_direct_launches_bitwise(monkeypatch, model, schedule):
    """tgv_iterate replays a captured CUDA graph of 6 iterations (the buffer-rotation period)
    for long runs; the iterates equal plain launches bit for bit, from an unaligned k, across
    a schedule / model change between calls (re-capture, in-place graph update) and a reload."""
    shape = (45, 31, 26)
    h = synth.random_histograms(shape, 16)
    c = list(oracle.default_centers(8))
    outs = []
    for graph in ("0", "1"):
        monkeypatch.setenv("TGV_GRAPH", graph)
        s = solver_cls()(shape, c).set_model(model).set_schedule(schedule).load(h)
        s.iterate(5).iterate(40)
        s.set_schedule("split" if schedule == "fused" else "fused").iterate(23)
        s.set_schedule(schedule).load(h).iterate(31)
        outs.append({f: s.get(f) for f in ("u", "p")})
        outs[-1]["E"] = s.energy()["E"]
        s.close()
    for f in ("u", "p", "E"):
        assert np.array_equal(outs[0][f], outs[1][f]), f


@pytest.mark.parametrize("model", ["tgv", "tvl1"])
def test_round_sync_gives_up_when_the_grid_is_not_resident(monkeypatch, model):
    """TGV_PERSIST_OVERSUB=2 launches twice the persistent CTAs that can be resident, so the
    first wave's round waits can never be met: the bounded wait must give up (once per launch)
    and the sweep finish with the unsynchronised result bit for bit, in bounded time."""
    import time
    shape = (256, 140, 43)
    monkeypatch.setenv("TGV_FUSED_ZC", "4" if model == "tgv" else "2")
    h = synth.random_histograms(shape, 18)
    c = list(oracle.default_centers(8))
    outs, secs = [], []
    for sync, over in (("0", "1"), ("1", "2")):
        monkeypatch.setenv("TGV_ROUND_SYNC", sync)
        monkeypatch.setenv("TGV_PERSIST_OVERSUB", over)
        s = solver_cls()(shape, c).set_model(model).load(h)
        t0 = time.perf_counter()
        s.iterate(5)
        secs.append(time.perf_counter() - t0)
        outs.append(s.get("u"))
        s.close()
    assert np.array_equal(outs[0], outs[1])
    assert secs[1] < 5.0, secs  # one give-up per launch (~tens of ms), not one per round
