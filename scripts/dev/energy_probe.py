"""A/B the dense energy sweeps (register-streaming default, TGV_ENERGY_IMPL=tma / tma2) on C4 and
C2 after a few iterations, timing each with the library's per-launch CUDA events (dev tool).
Prints ms per energy launch, the implied algorithmic GB/s (60 B/voxel with u8 counts) and
the relative difference of E and the gap between the two."""
import os

import synth
from paper_2107_14790_b200 import Solver


def cams_of(wl):
    return [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
             "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]


for name in ("C4", "C2"):
    wl = synth.workload(name)
    kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
    s = Solver(wl.shape, list(wl.centers), **kw)
    s.vote(cams_of(wl), synth.render_depths(wl), voxel_radius=wl.voxel_radius)
    s.iterate(10)
    nvox = wl.shape[0] * wl.shape[1] * wl.shape[2]
    for rep in range(3):
        res = {}
        for impl in ("regs", "tma", "tma2", "default"):
            if impl == "default":
                os.environ.pop("TGV_ENERGY_IMPL", None)
            else:
                os.environ["TGV_ENERGY_IMPL"] = impl
            s.energy()
            s.set_timing(True)
            for _ in range(5):
                e = s.energy()
            t = s.timing()
            s.set_timing(False)
            ms = t["energy_ms"] / max(1, t["energy_launches"])
            res[impl] = (ms, e)
            print(f"{name} rep{rep} {impl}: {ms:.3f} ms per energy launch, {60 * nvox / ms / 1e6:.0f} GB/s algorithmic, "
                  f"E {e['E']:.12g} gap {e['gap']:.12g} vmax {e['vmax']:.9g}", flush=True)
        b, eb = res["regs"]
        for impl in ("tma", "tma2", "default"):
            a, ea = res[impl]
            print(f"{name} rep{rep} {impl} vs regs: rel dE {abs(ea['E'] - eb['E']) / abs(eb['E']):.2e} "
                  f"d gap {abs(ea['gap'] - eb['gap']) / abs(eb['E']):.2e} speedup {b / a:.3f}", flush=True)
    os.environ.pop("TGV_ENERGY_IMPL", None)
    s.close()
