"""Benchmark of the TGV primal-dual hot path (BASELINE.json metric:
"TGV voxel-iterations/sec at 1/2/4/8 B200; achieved HBM GB/s vs peak").

A step is one full solve of the workload: reset the state from the resident
histograms, `iters` iterations of (dual + primal/over-relaxation), and one
energy/gap evaluation (all SURVEY.md §8(a) rows).  value = voxels x iters x
steps / time, over all ranks.  Inputs are synthetic (synth/, seeded).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2] [--iters I]
  python bench.py --impl reference ...   # the fp64 CPU oracle as the reference arm
  python bench.py --workload C5          # NEXT-3 block-sparse brick levels (BASELINE configs[4])

Multi-GPU (torchrun, one rank per GPU): the grid is split in z-slabs across
ranks (strong scaling of the same workload); NCCL halo exchange inside the
library; the step time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "TGV voxel-iterations/sec"
UNIT = "vox-it/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C4",
                    help="default C4 (BASELINE configs[3]: 1024^3, z-slabs across the ranks) at every N, so the "
                         "1/2/4/8-GPU lines are one workload; C2 / C3 (configs[1] / [2]) and C5 on request")
    ap.add_argument("--iters", type=int, default=None, help="iterations per step (default: the workload's)")
    ap.add_argument("--schedule", default="fused", choices=["fused", "split"])
    ap.add_argument("--model", default="tgv", choices=["tgv", "tvl1"], help="tvl1: NEXT-4 (Eq. 1)")
    ap.add_argument("--levels", type=int, default=1,
                    help="NEXT-1: coarse-to-fine levels (a step = the whole multilevel solve, iters per level)")
    ap.add_argument("--out-of-core", type=int, default=0, metavar="LEAF_VOXELS",
                    help="NEXT-3: out-of-core coarse-to-fine over z-slab leaves of <= LEAF_VOXELS voxels "
                         "(host-resident counts and levels; a step = the whole solve, --levels levels)")
    ap.add_argument("--mixed", action="store_true",
                    help="C5: solve the finest brick level as a 2:1 mixed-level set (R27: frozen border of level-0 "
                         "bricks or level-1 parent cubes); its own default schedule (SPLIT) unless --schedule is given")
    ap.add_argument("--parts", type=int, default=0,
                    help="C5: solve the finest brick level in this many Morton parts with frozen shells (R26); "
                         "streamed through one GPU, or shared round-robin by the ranks of a torchrun job")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the oracle sample")
    ap.add_argument("--vote", action="store_true", help="NEXT-2: measure GPU Alg. 1 voting instead of the solve")
    ap.add_argument("--no-self-check", action="store_true", help="N > 1: skip the slab-vs-one-context check")
    # solver parameters (SPEC.md:387-388 names lambda, alpha0, alpha1; R1, R7): the workload's by default
    ap.add_argument("--lambda", dest="lam", type=float, default=None, help="data weight lambda (R1)")
    ap.add_argument("--alpha0", type=float, default=None)
    ap.add_argument("--alpha1", type=float, default=None)
    ap.add_argument("--tau", type=float, default=None)
    ap.add_argument("--sigma", type=float, default=None)
    a = ap.parse_args()
    global ARGS
    ARGS = a
    return a


ARGS = None


def load_workload(name):
    """synth.workload(name) with the command line's solver parameters applied."""
    import dataclasses

    import synth
    wl = synth.workload(name)
    over = {k: getattr(ARGS, k) for k in ("lam", "alpha0", "alpha1", "tau", "sigma")
            if ARGS is not None and getattr(ARGS, k) is not None}
    return dataclasses.replace(wl, **over) if over else wl


# workloads whose inputs are voted on the GPU (bit-identical to the CPU generator,
# tests/test_gpu_vote.py) because a host vote of 10^9 voxels x 64 cameras is slow
GPU_VOTED = {"C3", "C4"}


def cams_of(wl):
    return [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
             "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]


def render_shared(wl, rank, world):
    """All depth maps of the workload; with several ranks each renders every world-th
    camera and the maps are exchanged (torch.distributed all_gather_object)."""
    import synth
    if world == 1:
        return synth.render_depths(wl)
    import copy

    import torch.distributed as dist
    mine = list(range(rank, len(wl.cams), world))
    # keep each camera's noise stream: render_depths numbers cameras 0.., so render one at a time
    out = {}
    for i in mine:
        one = copy.copy(wl)
        one.cams = [wl.cams[i]]
        d = synth.render_depths_indexed(one, i)
        out[i] = d
    gathered = [None] * world
    dist.all_gather_object(gathered, out)
    allmaps = {}
    for g in gathered:
        allmaps.update(g)
    return [allmaps[i] for i in range(len(wl.cams))]


def energy_roofline(tm, info, nvox, peak):
    """Algorithmic GB/s of the energy sweep (13 fp32 state fields + the stored counts per
    voxel, read once) from its per-launch CUDA-event time in the timed region."""
    if not tm.get("energy_launches"):
        return None
    ms = tm["energy_ms"] / tm["energy_launches"]
    bpv = 13 * 4 + info["count_slots"] * info["count_bytes"]
    gbs = bpv * nvox / (ms * 1e-3) / 1e9
    return {"kernel_ms": ms, "bytes_per_voxel": bpv, "achieved": gbs, "frac": gbs / peak}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(rows[0][1]),
                "power_w_max": max((num(r[2]) or 0) for r in rows), "samples": len(rows), "reasons": reasons}


def cpu_oracle_rate(workload: str, target_s: float, steps: int = 0, warmup: int = 0):
    """Time the fp64 oracle (as it stands) on this host on a bounded sample of
    the workload: the full grid (or, above 256^3 voxels, a 16-plane slab of it as
    its own grid) for k iterations, all host threads."""
    import oracle
    import synth
    wl = load_workload(workload)
    nx, ny, nz = wl.shape
    zs = nz if wl.nvox <= 256 ** 3 else 16
    h = synth.make_histograms(workload, 0, zs)
    shape = (nx, ny, zs)
    threads = oracle.max_threads()
    o = oracle.Oracle(shape, lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma,
                      centers=np.asarray(wl.centers)).load(h)
    nvox = nx * ny * zs
    what = f"{workload} full grid {wl.shape}" if zs == nz else f"{workload} planes 0..{zs} ({nx}x{ny}x{zs})"
    t0 = time.perf_counter()
    o.iterate(1, threads=threads)
    t1 = time.perf_counter() - t0
    if steps:  # reference arm: `warmup` untimed + `steps` timed single-iteration steps
        for _ in range(warmup):
            o.iterate(1, threads=threads)
        t0 = time.perf_counter()
        for _ in range(steps):
            o.iterate(1, threads=threads)
        el = time.perf_counter() - t0
        return nvox * steps / el, threads, f"{what}, {steps} timed iterations of 1", el
    k = int(max(1, min(1000, round(target_s / max(t1, 1e-6)))))
    t0 = time.perf_counter()
    o.iterate(k, threads=threads)
    el = time.perf_counter() - t0
    return nvox * k / el, threads, f"{what}, {k} iterations (after 1 warm-up)", el


def cpu_oracle_rate_1core(workload: str, target_s: float):
    """The same oracle on ONE host thread (1 core and all cores),
    over a bounded slab of the workload (at most 32 planes) as its own grid."""
    import oracle
    import synth
    wl = load_workload(workload)
    nx, ny, nz = wl.shape
    zs = min(nz, 32)
    h = synth.make_histograms(workload, 0, zs)
    o = oracle.Oracle((nx, ny, zs), lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma,
                      centers=np.asarray(wl.centers)).load(h)
    t0 = time.perf_counter()
    o.iterate(1, threads=1)
    t1 = time.perf_counter() - t0
    k = int(max(1, min(1000, round(target_s / max(t1, 1e-6)))))
    t0 = time.perf_counter()
    o.iterate(k, threads=1)
    el = time.perf_counter() - t0
    return nx * ny * zs * k / el, f"{workload} planes 0..{zs} ({nx}x{ny}x{zs}), {k} iterations, 1 thread"


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    wl = load_workload(a.workload)
    v, threads, sample, el = cpu_oracle_rate(a.workload, 0, steps=a.steps, warmup=a.warmup)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * el / a.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{wl.name}: {wl.description}", "shape": list(wl.shape), "iters_per_step": 1},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_vote(a, s, wl, rank, world, z0, z1, barrier_fn=None):
    """NEXT-2 measurement: GPU Alg. 1 (H2D of the depth maps, pyramids, votes,
    u16/u8 packing) per step; metric = voxel-camera votes per second, all ranks."""
    import torch
    import torch.distributed as dist
    cams, depths = cams_of(wl), render_shared(wl, rank, world)
    nx, ny, _ = wl.shape
    for _ in range(a.warmup):
        s.vote(cams, depths, voxel_radius=wl.voxel_radius)
    if barrier_fn:
        barrier_fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        s.vote(cams, depths, voxel_radius=wl.voxel_radius)
    torch.cuda.synchronize()
    el = torch.tensor([(time.perf_counter() - t0) / a.steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    votes = wl.nvox * len(cams)
    if rank == 0:
        print(json.dumps({
            "metric": "Alg. 1 voxel-camera lookups/sec (NEXT-2 GPU voting)", "value": votes / float(el[0]),
            "unit": "lookups/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": float(el[0]) * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{wl.name}: {wl.description}", "shape": list(wl.shape), "cameras": len(cams),
                       "step": "H2D depth maps + pyramids + Alg. 1 votes + count packing + state init"},
        }), flush=True)
    if barrier_fn:
        barrier_fn()
    s.close()
    return None


def run_out_of_core(a):
    """NEXT-3 measurement: the out-of-core solve (paper_2107_14790_b200.out_of_core)
    from host counts to host u, v; every leaf's H2D / prolongation / iterations / D2H
    inside the timed region.  Metric: voxel-iterations of all leaves of all levels per
    second (host to host, so it is its own end-to-end number)."""
    import torch

    import synth
    from paper_2107_14790_b200 import out_of_core
    from paper_2107_14790_b200.multilevel import level_shapes
    wl = load_workload(a.workload)
    iters = a.iters or 200
    levels = max(1, a.levels)
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
    if a.workload in GPU_VOTED:  # GPU Alg. 1 per 128-plane slab (bit-exact vs the CPU generator), narrowed to u8
        from paper_2107_14790_b200 import Solver
        nx, ny, nz = wl.shape
        cams, depths = cams_of(wl), render_shared(wl, 0, 1)
        counts = np.empty((nz, ny, nx, 8), np.uint8)
        for z0 in range(0, nz, 128):
            z1 = min(nz, z0 + 128)
            leaf = Solver.leaf(wl.shape, list(wl.centers), z0, z1, **kw).vote(cams, depths,
                                                                               voxel_radius=wl.voxel_radius)
            c = leaf.read_counts()
            assert c.max() <= 255
            counts[z0:z1] = c
            leaf.close()
    else:
        counts = synth.make_histograms(a.workload)
    vox_its = sum(int(np.prod(sh)) for sh in level_shapes(wl.shape, levels)) * iters
    # the leaf pool and the pinned host level buffers are allocated outside the timed region
    ooc = out_of_core.OutOfCore(wl.shape, list(wl.centers), levels=levels, iters=iters, leaf_voxels=a.out_of_core,
                                keep_pool=True, pinned=True, **kw)
    # the input: the finest counts in host memory, pinned, in the narrowest type that holds them
    narrow = np.uint8 if counts.max() <= 255 else (np.uint16 if counts.max() <= 65535 else np.uint32)
    counts = torch.from_numpy(counts.astype(narrow)).pin_memory().numpy()
    for _ in range(a.warmup):
        ooc.solve(counts)
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        ooc.solve(counts)
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / a.steps
    clk = clocks.stop()
    leaves = ooc.leaves  # finest first
    shapes = level_shapes(wl.shape, levels)
    # every level loads the fine counts of its leaves; every finer level uploads its parents' u, v
    h2d = int(levels * counts.nbytes + sum(4 * 4 * np.prod(sh) for sh in shapes[1:]))
    d2h = int(sum(4 * 4 * np.prod(sh) for sh in shapes))
    ooc.close()
    print(json.dumps({
        "metric": "TGV voxel-iterations/sec (NEXT-3 out-of-core leaves, host to host)", "value": vox_its / el,
        "unit": UNIT, "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": el * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{wl.name}: {wl.description}", "shape": list(wl.shape), "levels": levels,
                   "iters_per_level": iters, "leaf_voxels": a.out_of_core, "count_type": str(counts.dtype), "leaves_per_level_finest_first": leaves,
                   "step": "per level, per z-slab leaf: H2D fine counts + coarsen, H2D parent u/v + prolong "
                           "(borders frozen), iters fused iterations, D2H u, v; 2 pooled leaf contexts per size, "
                           "pinned host buffers"},
        "e2e": {"value": vox_its / el, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "clocks": clk,
    }), flush=True)


def slab_self_check(rank, world, local):
    """N > 1, before the timed region: a small grid (96 x 64 x 16N, C2-like random
    counts) solved in z-slabs across the N ranks (the bench's own halo mode) and, on
    every rank, in one context of its own; each rank compares its slab of u, v, p, q
    bitwise (any decomposition is bitwise the one-GPU iterate).  Returns
    (all ranks bitwise equal, halo mode, communicator size)."""
    import torch
    import torch.distributed as dist

    import synth
    from paper_2107_14790_b200 import Solver
    from paper_2107_14790_b200.tgv import slab
    shape = (96, 64, 16 * world)
    h = synth.random_histograms(shape, 77)
    c = [-0.875 + 0.25 * b for b in range(8)]
    z0, z1 = slab(shape[2], rank, world)
    d = Solver.distributed(shape, c, z0, z1, local).load(np.ascontiguousarray(h[z0:z1])).iterate(23)
    one = Solver(shape, c, device=local).load(h).iterate(23)
    ok = True
    for f in ("u", "v", "p", "q"):
        a_, b_ = d.get(f), one.get(f)
        b_ = b_[z0:z1] if f == "u" else b_[:, z0:z1]
        ok &= bool(np.array_equal(a_, b_))
    info = d.info()
    e1, e2 = d.energy(), one.energy()
    ok &= abs(e1["E"] - e2["E"]) <= 1e-12 * abs(e2["E"])
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.barrier()  # peer mode: no rank frees state a neighbour may still write
    d.close()
    one.close()
    return bool(flag.item()), ("peer" if info.get("peer_halo") else "nccl"), int(info.get("nranks", world))


def run_ours(a):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2107_14790_b200 import Solver
    from paper_2107_14790_b200.tgv import slab

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    check = None
    if world > 1 and not a.no_self_check:
        ok, mode, nr = slab_self_check(rank, world, local)
        check = {"slab_bitwise": ok, "halo_mode": mode, "comm_ranks": nr,
                 "grid": [96, 64, 16 * world], "iters": 23}
    wl = load_workload(a.workload)
    iters = a.iters or wl.iters
    nx, ny, nz = wl.shape
    z0, z1 = slab(nz, rank, world)
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
    if world > 1:
        s = Solver.distributed(wl.shape, list(wl.centers), z0, z1, local, **kw)
    else:
        s = Solver(wl.shape, list(wl.centers), device=local, **kw)
    s.set_schedule(a.schedule).set_model(a.model)
    if a.vote:
        return run_vote(a, s, wl, rank, world, z0, z1, barrier_fn=(dist.barrier if world > 1 else None))
    if a.workload in GPU_VOTED:  # NEXT-2 on the GPU: the same counts as synth.make_histograms
        s.vote(cams_of(wl), render_shared(wl, rank, world), voxel_radius=wl.voxel_radius)
        counts = s.read_counts() if (z1 - z0) * ny * nx * 32 <= (40 << 30) else None
    else:
        counts = synth.make_histograms(a.workload, z0, z1)
        s.load(counts)
    info = s.info()
    nvox_local = (z1 - z0) * ny * nx
    # NEXT-1: coarser levels (single GPU), allocated outside the timed region
    levels = [s]
    if a.levels > 1:
        assert world == 1, "--levels needs a single GPU"
        from paper_2107_14790_b200.multilevel import level_shapes
        for shp in level_shapes(wl.shape, a.levels)[1:]:
            levels.append(Solver(shp, list(wl.centers), device=local, **kw).set_schedule(a.schedule)
                          .set_model(a.model).restrict_from(levels[-1]))
    vox_its = sum(int(np.prod(lv.shape)) for lv in levels) * iters  # per step, all levels

    def barrier():
        if world > 1:
            dist.barrier()

    def solve():
        if len(levels) == 1:
            s.iterate(iters)
        else:  # restrict down from the resident fine histograms, solve coarse-to-fine
            for lev in range(1, len(levels)):
                levels[lev].restrict_from(levels[lev - 1])
            levels[-1].iterate(iters)
            for lev in range(len(levels) - 2, -1, -1):
                levels[lev].prolong_from(levels[lev + 1]).iterate(iters)

    def step():
        if len(levels) == 1:
            s.reset()
        solve()
        s.energy()

    for _ in range(a.warmup):
        step()
    # ---- timed region: device-resident inputs --------------------------------
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    for lv in levels:
        lv.set_timing(True)
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    barrier()
    ms = ev0.elapsed_time(ev1) / a.steps
    tm = s.timing()
    tms = [lv.timing() for lv in levels]
    for lv in levels:
        lv.set_timing(False)
    clk = clocks.stop()
    ms_t = torch.tensor([ms, wall * 1e3 / a.steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t[0])
    value = vox_its / (ms_max * 1e-3)

    # roofline of the dominant kernel: the kernel with the largest device time per step
    peak, peak_src = measured_peaks()
    kern = {}
    for name, bkey in (("fused", "bytes_fused"), ("dual", "bytes_dual"), ("primal", "bytes_primal")):
        if tm[f"{name}_launches"]:
            kern[name] = (tm[f"{name}_ms"] / tm[f"{name}_launches"], info[bkey], tm[f"{name}_ms"])
    dom = max(kern, key=lambda k: kern[k][2])
    kms, bpv, _ = kern[dom]
    achieved = bpv * nvox_local / (kms * 1e-3) / 1e9
    bytes_per_it = info["bytes_fused"] if a.schedule == "fused" else \
        info["bytes_dual"] + info["bytes_primal"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            key = dom if a.model == "tgv" else f"{a.model}_{dom}"
            traffic = json.load(open(tp)).get(a.workload, {}).get(key)
        except Exception:
            traffic = None
    step_kernel_ms = tm["primal_ms"] + tm["dual_ms"] + tm["fused_ms"] + tm["energy_ms"]
    # + init + 2 energy kernels (+ the u8 compaction only at load)
    launches_per_step = sum(t["dual_launches"] + t["primal_launches"] + t["fused_launches"] for t in tms) / a.steps \
        + 3 + 4 * (len(levels) - 1)  # + init, 2 energy kernels; per coarse level restrict + compact + init + prolong

    # ---- e2e: host buffers, H2D + D2H inside the timed region ------------------
    e2e = None
    if not a.no_e2e and counts is not None:
        # the host input in the narrowest unsigned type that holds it (u8 when every
        # count <= 255): tgv_load_histograms_coarsened with factor 1 is the narrow loader
        cmax = int(counts.max()) if counts.size else 0
        narrow = np.uint8 if cmax <= 255 else (np.uint16 if cmax <= 65535 else np.uint32)
        hc = torch.from_numpy(counts.astype(narrow)).pin_memory()
        hcn = hc.numpy()
        del counts  # the u32 read-back (34 GB at C4) is not needed any more
        hu = torch.empty((z1 - z0, ny, nx), dtype=torch.float32).pin_memory()
        hu2 = torch.empty((z1 - z0, ny, nx), dtype=torch.float32).pin_memory()
        from paper_2107_14790_b200 import tgv

        def timed(fn, k):
            barrier()
            torch.cuda.synchronize()
            t0_ = time.perf_counter()
            fn(k)
            torch.cuda.synchronize()
            el_ = torch.tensor([(time.perf_counter() - t0_) / k], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(el_, op=dist.ReduceOp.MAX)
            return float(el_[0])

        def pipelined(k):
            # every step uploads its counts and downloads its u; the upload of step j+1 and the
            # download of step j run on the library's copy streams beside step j+1's iterations
            tgv.tgv_stage_histograms(s.ctx, hcn)
            for j in range(k):
                tgv.tgv_load_staged(s.ctx)
                if j + 1 < k:
                    tgv.tgv_stage_histograms(s.ctx, hcn)
                solve()
                s.energy()
                tgv.tgv_read_u_async(s.ctx, hu if j % 2 == 0 else hu2)
            tgv.tgv_wait_io(s.ctx)

        def serial(k):
            for _ in range(k):
                tgv.tgv_load_histograms_coarsened(s.ctx, hcn, wl.shape, 1)
                solve()
                s.energy()
                tgv.tgv_read_u(s.ctx, hu)

        el = timed(pipelined, a.steps)
        d2h = int(hu.numel() * 4 + 6 * 8)
        e2e = {"value": vox_its / el, "unit": UNIT, "h2d_bytes_per_step": int(hcn.nbytes),
               "d2h_bytes_per_step": d2h, "count_type": str(hcn.dtype),
               "calls": "tgv_stage_histograms (next step's counts) + tgv_load_staged, tgv_iterate, tgv_energy, "
                        "tgv_read_u_async (this step's u): the copies on the library's copy streams overlap the "
                        "iterations; tgv_wait_io at the end"}
        k_ser = min(a.steps, 2)
        el = timed(serial, k_ser)
        e2e["serial"] = {"value": vox_its / el, "unit": UNIT, "steps": k_ser, "h2d_bytes_per_step": int(hcn.nbytes),
                         "d2h_bytes_per_step": d2h,
                         "calls": "tgv_load_histograms_coarsened (factor 1), tgv_iterate, tgv_energy, tgv_read_u"}
        del hc
        # the north-star loader: tgv_load_histograms with host uint32 counts (4x the bytes)
        k32 = min(a.steps, 2)
        h32 = torch.empty(tuple(hcn.shape), dtype=torch.int32).pin_memory()
        h32n = h32.numpy().view(np.uint32)
        h32n[...] = hcn
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k32):
            tgv.tgv_load_histograms(s.ctx, h32n)
            solve()
            s.energy()
            tgv.tgv_read_u(s.ctx, hu)
        torch.cuda.synchronize()
        el = torch.tensor([(time.perf_counter() - t0) / k32], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        e2e["u32_loader"] = {"value": vox_its / float(el[0]), "unit": UNIT, "steps": k32,
                             "h2d_bytes_per_step": int(h32n.nbytes), "d2h_bytes_per_step": int(hu.numel() * 4 + 6 * 8),
                             "calls": "tgv_load_histograms (uint32), tgv_iterate, tgv_energy, tgv_read_u"}
        del h32, h32n, hcn

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        v, threads, sample, _ = cpu_oracle_rate(a.workload, a.cpu_seconds)
        v1, sample1 = cpu_oracle_rate_1core(a.workload, a.cpu_seconds / 3)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
               "single_core": {"value": v1, "unit": UNIT, "cores": 1, "sample": sample1}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{wl.name}: {wl.description}", "shape": list(wl.shape), "iters_per_step": iters,
                       "step": ("reset + iters x (dual, primal+over-relax) + energy/gap" if a.levels == 1 else
                                f"coarse-to-fine: restrict to {a.levels} levels, iters per level, prolong, energy"),
                       "model": a.model, "schedule": a.schedule, "levels": a.levels,
                       "params": {"lambda": wl.lam, "alpha0": wl.alpha0, "alpha1": wl.alpha1, "tau": wl.tau,
                                  "sigma": wl.sigma},
                       "parallelism": (f"z-slab x{world}, halos " + ("written by the kernel into the neighbours "
                                       "(peer mode)" if info.get("peer_halo") else "by NCCL send/recv"))
                       if world > 1 else "single GPU",
                       "l2": f"no flush: resident state+histograms {info['device_bytes'] / 1e9:.2f} GB per GPU "
                             f">> 126 MB L2"},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_voxel": bpv, "kernel_ms": kms,
                         "schedule": a.schedule, "bytes_per_voxel_iteration": bytes_per_it,
                         "count_bytes": info["count_bytes"],
                         "schedule_gbs": bytes_per_it * vox_its / (ms_max * 1e-3) / 1e9 / world,
                         "kernel_share_of_step": step_kernel_ms / a.steps / ms,
                         # (a4) the energy / gap sweep once per step: 13 fp32 fields + the counts per voxel
                         "energy": energy_roofline(tm, info, nvox_local, peak)},
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": int(round(launches_per_step * a.steps)),
            **({"slab_bitwise": check["slab_bitwise"], "halo_mode": check["halo_mode"],
                "comm_ranks": check["comm_ranks"], "multi_gpu_check": check} if check else {}),
            "kernel_ms": {**{k: v[0] for k, v in kern.items()},
                          "energy": tm["energy_ms"] / max(1, tm["energy_launches"])},
            "wall_ms_per_step": float(ms_t[1]),
        }
        print(json.dumps(line), flush=True)
    barrier()  # peer halo mode: no rank frees its state while a neighbour's kernel may still write it
    s.close()
    if world > 1:
        dist.destroy_process_group()


def run_brick_parts(a):
    """NEXT-3 parts (R26, BASELINE configs[4] "streamed out-of-core across 8 B200"): the
    coarse brick levels are solved on every rank (redundantly, counted once), the finest
    level in --parts Morton parts with frozen shells, parts r, r + N, ... on rank r.
    Parts need no exchange, so there is no collective in the solve.  With more parts
    than ranks each rank streams its parts through its GPU (one part resident at a time,
    counts in pinned host memory, H2D + D2H of every part inside the timed region).
    value = solved voxel-iterations of all levels / the slowest rank's step time."""
    import torch
    import torch.distributed as dist

    import synth
    from paper_2107_14790_b200.brick_levels import BrickLevels, PartSolver
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = load_workload(a.workload)
    iters = a.iters or wl.iters
    levels = max(2, a.levels if a.levels > 1 else 3)
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma, centers=list(wl.centers))
    cams, depths = cams_of(wl), render_shared(wl, rank, world)
    bl = BrickLevels(wl.shape, cams, depths, levels=levels, edge=32, voxel_radius=wl.voxel_radius,
                     resident_finest=False, device=local, **kw)
    mine = list(range(rank, a.parts, world))
    ps = PartSolver(bl, a.parts, mine=mine, pinned=True, schedule=a.schedule)
    stream = len(ps.mine) > 1  # several parts per GPU: one resident at a time
    pool = None if stream else {}
    coarse_solved = sum(int((~bl.frozen[lev]).sum()) for lev in range(1, levels)) * 32 ** 3
    fine_solved_all = int((~bl.frozen[0]).sum()) * 32 ** 3
    vox_its = (coarse_solved + fine_solved_all) * iters

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(a.warmup):
        ps.solve(iters, pool)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        ps.solve(iters, pool)
    torch.cuda.synchronize()
    el = (time.perf_counter() - t0) / a.steps
    barrier()
    clk = clocks.stop()
    t = torch.tensor([el], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    el_max = float(t[0])
    pv = ps.part_voxels()
    h2d = sum(int(ps.sets[p][2].nbytes) for p in ps.mine)
    d2h = sum(int((~ps.sets[p][1]).sum()) * 32 ** 3 * 4 for p in ps.mine)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC + " (NEXT-3 brick parts, frozen shells)", "value": vox_its / el_max, "unit": UNIT,
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": el_max * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{wl.name}: {wl.description}", "levels": levels, "iters_per_level": iters,
                       "parts": a.parts, "parts_rank0": mine, "part_voxels_rank0": pv, "schedule": ps.schedule,
                       "bricks_solved_frozen_finest_first": bl.bricks(),
                       "step": "coarse levels (every rank), then per owned part: H2D counts (pinned u8), prolong "
                               "from level 1 (frozen shell), iters, D2H of its solved u",
                       "parallelism": f"{world} rank(s), parts round-robin, no collective in the solve",
                       "resident": "one part at a time" if stream else "each rank's part resident"},
            "e2e": {"value": vox_its / el_max, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "note": "the step itself is host to host (counts H2D, u D2H per part)"},
            "clocks": clk,
        }), flush=True)
    if pool:
        for s_ in pool.values():
            s_.close()
    bl.close()
    if world > 1:
        dist.destroy_process_group()


def run_bricks(a):
    """NEXT-3 block-sparse brick sets (BASELINE configs[4], workload C5): the brick
    levels are built once from the GPU votes (brick_levels.BrickLevels); a step is the
    coarse-to-fine solve (coarsest from its votes, each finer level prolongated with
    its frozen shell, iters per level) plus the finest level's energy / gap.
    value = voxel-iterations of the solved voxels per second (value_S: of the voxels
    whose duals are updated, S = solved + frozen face-adjacent, R24)."""
    import torch

    import synth
    from paper_2107_14790_b200.brick_levels import BrickLevels
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and int(os.environ.get("RANK", "0")) != 0:
        return  # single-GPU measurement: the other ranks have no work
    wl = load_workload(a.workload)
    iters = a.iters or wl.iters
    levels = max(2, a.levels if a.levels > 1 else 3)
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma, centers=list(wl.centers))
    cams, depths = cams_of(wl), render_shared(wl, 0, 1)
    t_build = time.perf_counter()
    bl = BrickLevels(wl.shape, cams, depths, levels=levels, edge=32, voxel_radius=wl.voxel_radius,
                     resident_finest=not a.mixed, **kw)
    t_build = time.perf_counter() - t_build
    for s_ in bl.solvers:
        if s_ is not None:
            s_.set_schedule(a.schedule)  # FUSED by default (32^3 bricks), SPLIT on request
    sols = bl.solvers
    if a.mixed:  # R27: the finest level as a 2:1 mixed-level set (SPLIT by default; an explicit --schedule applies)
        m = bl.build_mixed()
        if any(x == "--schedule" or x.startswith("--schedule=") for x in sys.argv):
            m.set_schedule(a.schedule)
        sols = [m] + bl.solvers[1:]
    vox = [int(s_.info()["nbricks"]) * 32 ** 3 for s_ in sols]
    infos = [s.info() for s in sols]
    solved = [i["solved_voxels"] for i in infos]
    svox = [i["s_voxels"] for i in infos]
    vox_its, vox_its_s = sum(solved) * iters, sum(svox) * iters

    solve = bl.solve_mixed if a.mixed else bl.solve

    def step():
        solve(iters).energy()

    for _ in range(a.warmup):
        step()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    for s in sols:
        s.set_timing(True)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        step()  # every library call synchronises its own stream before returning
    ev1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / a.steps
    ms = ev0.elapsed_time(ev1) / a.steps
    tms = [s.timing() for s in sols]
    for s in sols:
        s.set_timing(False)
    clk = clocks.stop()
    cb = sols[0].info()["count_bytes"]
    fused = infos[0]["schedule"] == 0
    # algorithmic bytes, per level by its own schedule: SPLIT: dual on S,
    # 17 reads + 9 writes; primal on the solved voxels, 13 reads + counts + 4 writes.
    # FUSED: the frozen-face dual on S minus the solved voxels (104 B) and the single
    # sweep over the solved voxels (17 reads + counts + 13 writes)
    dual_b = primal_b = 0
    for inf, sv, so in zip(infos, svox, solved):
        if inf["schedule"] == 0:
            dual_b += (sv - so) * 104 * iters
            primal_b += so * (120 + 8 * cb) * iters
        else:
            dual_b += sv * 104 * iters
            primal_b += so * (68 + 8 * cb) * iters
    dual_ms = sum(t["dual_ms"] for t in tms) / a.steps
    primal_ms = sum(t["primal_ms"] + t["fused_ms"] for t in tms) / a.steps
    mixed = None
    if a.mixed:  # the finest level's mixed kernels alone
        t0_ = tms[0]
        dms0, pms0 = t0_["dual_ms"] / a.steps, t0_["primal_ms"] / a.steps
        lv_ = bl.mixed[2]
        mixed = {"bricks_level0": int((lv_ == 0).sum()), "bricks_level1": int((lv_ == 1).sum()),
                 "solved_bricks": int((~bl.mixed[3]).sum()), "s_voxels": svox[0],
                 "dual_ms_per_step": dms0, "primal_ms_per_step": pms0,
                 "dual_gbs": svox[0] * 104 * iters / (dms0 * 1e-3) / 1e9,
                 "primal_gbs": solved[0] * (68 + 8 * cb) * iters / (pms0 * 1e-3) / 1e9}
    peak, peak_src = measured_peaks()
    if fused:
        dom, dbytes, dms = "fused", primal_b, primal_ms
    else:
        dom, dbytes, dms = ("dual", dual_b, dual_ms) if dual_ms >= primal_ms else ("primal", primal_b, primal_ms)
    achieved = dbytes / (dms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(a.workload, {}).get(f"brick_{dom}")
    launches = sum(t["dual_launches"] + t["primal_launches"] + t["fused_launches"] + t["energy_launches"]
                   for t in tms) / a.steps \
        + 2 * levels  # + per level the init / prolongation kernel; + the energy final kernel

    # e2e through the public API: H2D of the depth maps and Alg. 1 votes into every
    # level's bricks, the coarse-to-fine solve, energy, D2H of the finest u
    e2e = None
    if not a.no_e2e:
        hu = None
        # the step's host data in pinned memory (the contract's "from pinned host memory"):
        # the depth maps in, the finest level's u out
        pdepths = [torch.from_numpy(np.ascontiguousarray(d)).pin_memory().numpy() for d in depths]
        hbuf = torch.empty(int(sols[0].nvox), dtype=torch.float32).pin_memory().numpy()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            for lev, s in enumerate(sols):
                # a mixed set votes each brick at its own level (level 0 here)
                s.vote(cams, pdepths, voxel_size=float(1 << lev), voxel_radius=wl.voxel_radius * (1 << lev))
            f = solve(iters)
            f.energy()
            hu = f.read_u(hbuf)
        el = (time.perf_counter() - t0) / a.steps
        h2d = levels * sum(int(d.nbytes) for d in depths)
        e2e = {"value": vox_its / el, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(hu.nbytes) + 48,
               "calls": "tgv_bricks_vote_depth_maps per level, tgv_bricks_reset / prolong_from / iterate per level, "
                        "tgv_bricks_energy, tgv_bricks_read"}
    cpu = None
    if not a.no_cpu_baseline:
        cpu = cpu_brick_oracle_rate(bl, a.cpu_seconds, kw, solver=sols[0],
                                    sets=(bl.mixed[1], bl.mixed[3]) if a.mixed else None)
    bricks = bl.bricks()
    line = {
        "metric": METRIC + " (NEXT-3 block-sparse brick sets)", "value": vox_its / (ms * 1e-3), "unit": UNIT,
        "value_S": vox_its_s / (ms * 1e-3), "n_gpus": 1, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{wl.name}: {wl.description}", "extent": list(wl.shape), "edge": 32, "levels": levels,
                   "iters_per_level": iters,
                   "bricks_solved_frozen_finest_first": bricks, "bricks_total": int(sum(a_ + b_ for a_, b_ in bricks)),
                   "voxels_per_level_finest_first": vox, "solved_voxels_per_level": solved,
                   "s_voxels_per_level": svox, "build_s": t_build,
                   "step": "coarse-to-fine over the brick levels: reset coarsest, iters; per finer level prolong "
                           "(frozen shell from the parent), iters; energy/gap of the finest",
                   "parallelism": "single GPU",
                   "l2": "no flush: resident brick state >> 126 MB L2"},
        "roofline": {"bound": "hbm", "kernel": f"brick_{dom}", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_voxel": {"dual": 104, "primal": 68 + 8 * cb, "fused": 120 + 8 * cb}[dom],
                     "schedule": "fused" if fused else "split", "kernel_ms_per_step": dms,
                     "schedule_gbs": (dual_b + primal_b) / (ms * 1e-3) / 1e9, "count_bytes": cb,
                     "kernel_share_of_step": (dual_ms + primal_ms) / ms},
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": int(round(launches * a.steps)),
        "mixed_finest": mixed,
        "kernel_ms": {"dual" if not fused else "frozen_face_dual": dual_ms,
                      "primal" if not fused else "fused": primal_ms,
                      "energy": sum(t["energy_ms"] for t in tms) / a.steps},
        "wall_ms_per_step": wall * 1e3,
    }
    print(json.dumps(line), flush=True)
    bl.close()


def cpu_brick_oracle_rate(bl, target_s, kw, solver=None, sets=None):
    """The brick-set oracle (oracle/bricks.py, numpy fp64) as it stands, on a bounded
    sample: the first 8 solved bricks of the finest level with their counts."""
    import oracle.bricks as ob
    s = solver if solver is not None else bl.solvers[0]
    coords, frozen = sets if sets is not None else (bl.coords[0], bl.frozen[0])
    sel = np.nonzero(~np.asarray(frozen))[0][:8]
    counts = s.read_counts()[sel]
    o = ob.BrickOracle(bl.edge, np.asarray(coords)[sel], **kw).load(counts)
    t0 = time.perf_counter()
    o.iterate(1)
    t1 = time.perf_counter() - t0
    k = int(max(1, min(1000, round(target_s / max(t1, 1e-6)))))
    t0 = time.perf_counter()
    o.iterate(k)
    el = time.perf_counter() - t0
    nv = len(sel) * bl.edge ** 3
    return {"value": nv * k / el, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"C5 finest level, {len(sel)} solved 32^3 bricks as their own set, {k} iterations (numpy fp64)"}


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.out_of_core:
        run_out_of_core(a)
    elif a.workload == "C5" and a.parts:
        run_brick_parts(a)
    elif a.workload == "C5":
        run_bricks(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
