"""Write the full-count oracle goldens of the BASELINE sizes C3 and C4 (tests/golden/).

Calls only oracle/ (the fp64 CPU scheme) and synth/ (the seeded input generator):
no value here comes from the CUDA path.  The GPU tests
(tests/test_gpu_full_size.py) solve the same workloads at their stated counts on
the full grid and compare sampled 32^3 blocks, and (C3) the full-grid energy terms,
restricted gap (R14) and max|v|, against these files.

  C3  512^3, 1000 iterations (R10): 1000 > the grid, so the oracle solves the FULL
      grid; blocks of u, the full-grid energy / gap / max|v|.
  C4  1024^3, 200 iterations: after n iterations u(x) depends only on the input within
      L-inf distance 2n of x (each half-step reads +-1 neighbours), so each 32^3 block is
      solved on its own window with a margin of 2n + 4 (clipped at the grid faces, where
      the window face is the grid's own Neumann face).  u of the blocks only.

Each record carries the sha256 of the uint32 counts the oracle solved, so the GPU
test can check that its (GPU Alg. 1) counts are the same integers.

usage: python scripts/make_goldens.py [C3] [C4] [--out tests/golden] [--threads T]
(C3: 1.3e11 voxel-iterations, ~30 GB; C4: ~6e10, <= 30 GB per window; about 45 and 25 min on 16 host threads.)
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

B = 32


def blocks(wl):
    """32^3 blocks (x0, y0, z0): grid corners (boundary faces) and surface crossings
    (the same choice as tests/test_gpu_full_size.py)."""
    nx, ny, nz = wl.shape
    if wl.name == "C3":  # terrain around z = 200 +- 78, observed from above
        return [(0, 0, 184), (240, 240, 184), (nx - B, ny - B, 184), (nx - B, ny - B, nz - B)]
    sph = wl.prims[1][1]  # C4: (cx, cy, cz, r) of the first sphere; ground plane z = 100
    return [(0, 0, 84), (496, 496, 84), (int(sph[0] + 0.7 * sph[3]) - 16, int(sph[1]) - 16, 84),
            (nx - B, ny - B, nz - B)]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.uint32).tobytes()).hexdigest()


def kw_of(wl):
    return dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)


def c3(out, threads):
    wl = synth.workload("C3")
    nx, ny, nz = wl.shape
    t0 = time.time()
    h = synth.make_histograms("C3")
    print(f"C3 counts {h.shape} in {time.time() - t0:.0f} s", flush=True)
    o = oracle.Oracle(wl.shape, centers=np.asarray(wl.centers), **kw_of(wl)).load(h)
    rec = {"workload": "C3", "shape": list(wl.shape), "iters": wl.iters, "counts_sha256": sha(h),
           "params": kw_of(wl), "centers": list(map(float, wl.centers)), "blocks": []}
    del h
    t0 = time.time()
    done = 0
    for ck in (100, 250, 500, wl.iters):  # progress checkpoints
        o.iterate(ck - done, threads=threads)
        done = ck
        print(f"C3 {done}/{wl.iters} iterations, {time.time() - t0:.0f} s", flush=True)
    e = o.energy()
    rec["energy"] = {k: float(e[k]) for k in ("E", "alpha1", "alpha0", "data", "gap", "vmax")}
    arrs = {}
    u = o.get("u")
    for k, (x0, y0, z0) in enumerate(blocks(wl)):
        x0, y0 = min(max(x0, 0), nx - B), min(max(y0, 0), ny - B)
        arrs[f"u{k}"] = u[z0:z0 + B, y0:y0 + B, x0:x0 + B].copy()
        rec["blocks"].append([x0, y0, z0])
    write(out, "c3_full_count", rec, arrs)


def c4_blocks(wl):
    """C4's golden blocks: near the grid's x / y faces, so that the light-cone windows are
    clipped by the grid's own (Neumann) faces and stay affordable (an interior block's
    840 x 840 x 520 window needs ~65 GB of fp64 oracle state): the ground-plane corner, the
    flank of a sphere near the (+x, +y) corner (sphere surface and ground plane), and the
    top corner above the scene."""
    nx, ny, nz = wl.shape
    sph = min((p for kind, p in wl.prims if kind == 0), key=lambda p: (nx - p[0]) ** 2 + (ny - p[1]) ** 2)
    return [(0, 0, 84), (int(sph[0] + 0.7 * sph[3]) - 16, int(sph[1]) - 16, 84), (nx - B, ny - B, nz - B)]


def c4(out, threads):
    wl = synth.workload("C4")
    nx, ny, nz = wl.shape
    n = wl.iters
    M = 2 * n + 4
    rec = {"workload": "C4", "shape": list(wl.shape), "iters": n, "margin": M, "params": kw_of(wl),
           "centers": list(map(float, wl.centers)), "blocks": [], "windows": [], "window_counts_sha256": []}
    arrs = {}
    for k, (x0, y0, z0) in enumerate(c4_blocks(wl)):
        x0, y0 = min(max(x0, 0), nx - B), min(max(y0, 0), ny - B)
        wz0, wz1 = max(z0 - M, 0), min(z0 + B + M, nz)
        wy0, wy1 = max(y0 - M, 0), min(y0 + B + M, ny)
        wx0, wx1 = max(x0 - M, 0), min(x0 + B + M, nx)
        t0 = time.time()
        h = synth.make_histograms_box("C4", (wx0, wx1, wy0, wy1, wz0, wz1))
        o = oracle.Oracle((wx1 - wx0, wy1 - wy0, wz1 - wz0), centers=np.asarray(wl.centers), **kw_of(wl)).load(h)
        o.iterate(n, threads=threads)
        arrs[f"u{k}"] = o.u[z0 - wz0:z0 - wz0 + B, y0 - wy0:y0 - wy0 + B, x0 - wx0:x0 - wx0 + B].copy()
        rec["blocks"].append([x0, y0, z0])
        rec["windows"].append([wx0, wx1, wy0, wy1, wz0, wz1])
        rec["window_counts_sha256"].append(sha(h))
        print(f"C4 block {k} window {wx1 - wx0}x{wy1 - wy0}x{wz1 - wz0}: {time.time() - t0:.0f} s", flush=True)
        del o, h
    write(out, "c4_full_count", rec, arrs)


def write(out, name, rec, arrs):
    os.makedirs(out, exist_ok=True)
    rec["written_by"] = "scripts/make_goldens.py (oracle/ + synth/ only)"
    rec["oracle_threads_note"] = "the oracle is bitwise thread-count invariant (DESIGN.md §3)"
    np.savez_compressed(os.path.join(out, name + ".npz"), **arrs)
    with open(os.path.join(out, name + ".json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(f"wrote {out}/{name}.json/.npz", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="*", default=["C3", "C4"])
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    oracle.build()
    synth.build()
    th = a.threads or oracle.max_threads()
    print(f"oracle threads {th}, host cores {os.cpu_count()}", flush=True)
    for w in a.which:
        {"C3": c3, "C4": c4}[w](a.out, th)


if __name__ == "__main__":
    main()
