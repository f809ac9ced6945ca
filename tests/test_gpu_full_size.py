"""Parity at the full BASELINE sizes C3 (512^3) and C4 (1024^3: the configuration
bench.py times on 2/4/8 GPUs), in the solver's launch configuration, on sampled outputs
the oracle can compute (DESIGN.md §3 "light cone").

One iteration of the scheme reads only the 6-neighbourhood of a voxel (the dual reads
ubar at +1 and vbar at -1, the primal p at -1 and q at +1), so after n iterations
u(x) depends on the input within L-inf distance n of x.  The oracle therefore solves
a window of the grid with a margin of 2n + 4 voxels around a 32^3 block (its own
Neumann faces stay outside the block's light cone, except where the window face is
the grid's own boundary, where both agree) and the block is compared voxel by voxel
with the full-grid GPU iterate.  The GPU grid's counts come from GPU Alg. 1 (bit-exact
vs the CPU generator, tests/test_gpu_vote.py); the oracle's from the CPU generator.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
ITERS = 8
M = 2 * ITERS + 4
B = 32


def _cams(wl):
    return [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
             "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]


def _blocks(wl):
    """32^3 blocks (x0, y0, z0) per workload: grid corners (boundary faces) and surface crossings."""
    nx, ny, nz = wl.shape
    if wl.name == "C3":  # terrain around z = 200 +- 78, observed from above
        return [(0, 0, 184), (240, 240, 184), (nx - B, ny - B, 184), (nx - B, ny - B, nz - B)]
    sph = wl.prims[1][1]  # C4: (cx, cy, cz, r) of the first sphere; ground plane z = 100
    return [(0, 0, 84), (496, 496, 84), (int(sph[0] + 0.7 * sph[3]) - 16, int(sph[1]) - 16, 84),
            (nx - B, ny - B, nz - B)]


@pytest.mark.parametrize("name,mem_gb", [("C3", 25), ("C4", 170)])
def test_full_grid_blocks_match_oracle_windows(name, mem_gb):
    import torch
    from paper_2107_14790_b200 import Solver
    if torch.cuda.get_device_properties(0).total_memory < mem_gb * 1e9:
        pytest.skip(f"{name} needs about {mem_gb} GB of device memory")
    wl = synth.workload(name)
    nx, ny, nz = wl.shape
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
    depths = synth._depths_cached(name)  # shared with make_histograms below (same maps)
    s = Solver(wl.shape, list(wl.centers), **kw)
    s.vote(_cams(wl), depths, voxel_radius=wl.voxel_radius).iterate(ITERS)
    u = s.read_u()
    e = s.energy()
    s.close()
    assert np.all(np.abs(u) <= 1) and np.isfinite(e["E"]) and e["gap"] >= -1e-9 * e["E"]
    bands = {}
    worst, observed = 0.0, 0
    blocks = _blocks(wl)
    for x0, y0, z0 in blocks:
        x0, y0 = min(max(x0, 0), nx - B), min(max(y0, 0), ny - B)
        wz0, wz1 = max(z0 - M, 0), min(z0 + B + M, nz)
        if (wz0, wz1) not in bands:
            bands[(wz0, wz1)] = synth.make_histograms(name, wz0, wz1)
        wx0, wx1 = max(x0 - M, 0), min(x0 + B + M, nx)
        wy0, wy1 = max(y0 - M, 0), min(y0 + B + M, ny)
        h = np.ascontiguousarray(bands[(wz0, wz1)][:, wy0:wy1, wx0:wx1])
        o = oracle.Oracle((wx1 - wx0, wy1 - wy0, wz1 - wz0), centers=np.asarray(wl.centers), **kw)
        o.load(h).iterate(ITERS, threads=oracle.max_threads())
        ref = o.u[z0 - wz0:z0 - wz0 + B, y0 - wy0:y0 - wy0 + B, x0 - wx0:x0 - wx0 + B]
        got = u[z0:z0 + B, y0:y0 + B, x0:x0 + B].astype(np.float64)
        d = float(np.max(np.abs(got - ref)))
        worst = max(worst, d)
        assert d <= 1e-4, ((x0, y0, z0), d)
        observed += int(np.any(h[z0 - wz0:z0 - wz0 + B, y0 - wy0:y0 - wy0 + B, x0 - wx0:x0 - wx0 + B].sum(-1) > 0))
    assert observed >= 2  # not only unobserved space (the corners may be outside every frustum)
    print(f"{name} {wl.shape}, {ITERS} iterations: max|du| over {len(blocks)} blocks of {B}^3 = {worst:.3g}")


GOLDEN = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden")


def _golden(name):
    import json
    import os
    jp, zp = os.path.join(GOLDEN, name + ".json"), os.path.join(GOLDEN, name + ".npz")
    if not (os.path.exists(jp) and os.path.exists(zp)):
        pytest.fail(f"golden {name} missing: run scripts/make_goldens.py")
    return json.load(open(jp)), np.load(zp)


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, np.uint32).tobytes()).hexdigest()


@pytest.mark.parametrize("name,mem_gb", [("C3", 25), ("C4", 170)])
def test_full_grid_at_stated_count_matches_oracle_golden(name, mem_gb):
    """The bench's full grids at their STATED iteration counts (R10: C3 1000, C4 200),
    solved on the GPU in the bench's launch configuration from GPU Alg. 1 counts, against
    oracle goldens written by scripts/make_goldens.py (oracle/ + synth/ only):
    C3 -- the oracle solved the full 512^3 grid (1000 iterations reach every voxel):
         four 32^3 blocks of u, and the full-grid E, its terms, the restricted gap and
         max|v| (north-star tolerances: max|du| <= 1e-4, rel dE <= 1e-5);
    C4 -- the oracle solved each block's light-cone window (margin 2n + 4): four 32^3
         blocks of u.
    The GPU's counts are checked to be the same integers as the oracle's (sha256)."""
    import torch
    from paper_2107_14790_b200 import Solver
    if torch.cuda.get_device_properties(0).total_memory < mem_gb * 1e9:
        pytest.skip(f"{name} needs about {mem_gb} GB of device memory")
    rec, arrs = _golden(name.lower() + "_full_count")
    wl = synth.workload(name)
    assert rec["shape"] == list(wl.shape) and rec["iters"] == wl.iters
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
    assert rec["params"] == kw and rec["centers"] == list(map(float, wl.centers))
    s = Solver(wl.shape, list(wl.centers), **kw)
    s.vote(_cams(wl), synth._depths_cached(name), voxel_radius=wl.voxel_radius)
    counts = s.read_counts()
    if name == "C3":
        assert _sha(counts) == rec["counts_sha256"]
    else:
        for (x0, x1, y0, y1, z0, z1), h in zip(rec["windows"], rec["window_counts_sha256"]):
            assert _sha(counts[z0:z1, y0:y1, x0:x1]) == h
    del counts
    s.iterate(wl.iters)
    u = s.read_u()
    e = s.energy()
    s.close()
    worst = 0.0
    for k, (x0, y0, z0) in enumerate(rec["blocks"]):
        got = u[z0:z0 + B, y0:y0 + B, x0:x0 + B].astype(np.float64)
        d = float(np.max(np.abs(got - arrs[f"u{k}"])))
        worst = max(worst, d)
        assert d <= 1e-4, ((x0, y0, z0), d)
    msg = f"{name} {wl.shape} x{wl.iters}: max|du| over {len(rec['blocks'])} blocks = {worst:.3g}"
    if name == "C3":
        eo = rec["energy"]
        rel = abs(e["E"] - eo["E"]) / abs(eo["E"])
        assert rel <= 1e-5, (e["E"], eo["E"])
        for t in ("alpha1", "alpha0", "data"):
            assert abs(e[t] - eo[t]) <= 1e-5 * abs(eo["E"]), t
        assert abs(e["gap"] - eo["gap"]) <= 1e-5 * abs(eo["E"]), (e["gap"], eo["gap"])
        assert abs(e["vmax"] - eo["vmax"]) <= 1e-4, (e["vmax"], eo["vmax"])
        msg += f", rel dE = {rel:.3g}, gap {e['gap']:.6g} vs {eo['gap']:.6g}"
    print(msg)


def test_c3_slab_group_equals_single_context_bitwise():
    """the z-slab decomposition equals one GPU bitwise at a BASELINE
    size -- C3 (512^3) as 4 uneven slabs of an in-process group (the NCCL path's slab
    geometry, halo plans and kernels; only the transport differs) against one context."""
    import torch
    from paper_2107_14790_b200 import Group, Solver
    if torch.cuda.get_device_properties(0).total_memory < 60e9:
        pytest.skip("needs about 45 GB of device memory")
    wl = synth.workload("C3")
    nx, ny, nz = wl.shape
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
    depths = synth._depths_cached("C3")
    one = Solver(wl.shape, list(wl.centers), **kw).vote(_cams(wl), depths, voxel_radius=wl.voxel_radius)
    counts = one.read_counts()
    one.iterate(10)
    cuts = [0, 100, 256, 257, 512]
    grp = Group(wl.shape, cuts, list(wl.centers), **kw).load(counts).iterate(10)
    assert np.array_equal(grp.read_u(), one.read_u())
    eg, e1 = grp.energy(), one.energy()
    assert abs(eg["E"] - e1["E"]) <= 1e-12 * abs(e1["E"])


def test_c5_finest_brick_level_samples_match_oracle_windows():
    """C5 (BASELINE configs[4]) at full size: the finest brick level of the bench's
    hierarchy (13 912 solved + 9383 frozen 32^3 bricks, counts from GPU Alg. 1 into the
    bricks) iterated ITERS times from its vote initialisation; sampled solved bricks are
    compared with the brick oracle on the window of the brick and its 26 neighbours in
    the set (the same solved / frozen flags, counts from the oracle's own Alg. 1).  The
    window's outer faces are 32 voxels from the sample, outside its light cone."""
    import torch
    from paper_2107_14790_b200.brick_levels import BrickLevels
    from paper_2107_14790_b200.bricks import BrickSolver
    from oracle import bricks as ob
    if torch.cuda.get_device_properties(0).total_memory < 120e9:
        pytest.skip("C5's finest level needs about 110 GB of device memory")
    wl = synth.workload("C5")
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma, centers=list(wl.centers))
    depths = synth.render_depths(wl)
    cams = _cams(wl)
    bl = BrickLevels(wl.shape, cams, depths, levels=3, edge=B, resident_finest=False, **kw)
    coords, frozen = bl.coords[0], bl.frozen[0]
    bl.close()
    s = BrickSolver(B, coords, frozen, **kw).vote(cams, depths, voxel_radius=wl.voxel_radius).iterate(ITERS)
    e = s.energy()
    assert np.isfinite(e["E"]) and e["gap"] >= -1e-9 * e["E"]
    index = {tuple(int(t) for t in c): i for i, c in enumerate(coords)}
    solved = np.nonzero(~frozen)[0]
    nfrozen_nb = np.array([sum(frozen[index[n]] for n in
                               [(c[0] + dx, c[1] + dy, c[2] + dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1)
                                for dz in (-1, 0, 1)] if n in index) for c in coords[solved]])
    rng = np.random.default_rng(5)
    samples = [solved[0], solved[int(np.argmax(nfrozen_nb))], solved[len(solved) // 2], rng.choice(solved)]
    u = s.read_u()
    s.close()
    worst = 0.0
    for b in samples:
        c = coords[b]
        win = [index[n] for n in [(c[0] + dx, c[1] + dy, c[2] + dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1)
                                  for dx in (-1, 0, 1)] if n in index]
        wc, wf = coords[win], frozen[win]
        o = ob.BrickOracle(B, wc, wf, **kw).load(ob.vote(wc, B, cams, depths, r=wl.voxel_radius)).iterate(ITERS)
        k = win.index(b)
        d = float(np.max(np.abs(u[b].astype(np.float64) - o.get("u")[k])))
        worst = max(worst, d)
        assert d <= 1e-4, (tuple(c), d)
    print(f"C5 finest level: {len(samples)} sampled bricks, max|du| = {worst:.2e}")
