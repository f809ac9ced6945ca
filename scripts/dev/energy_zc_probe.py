"""C2: the energy sweeps at several lock-step chunk sizes (TGV_ENERGY_ZC) -- whether the 2-CTA TMA sweep
beats the register sweep once the grid has whole rounds (dev tool)."""
import os

import synth
from paper_2107_14790_b200 import Solver

wl = synth.workload("C2")
kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
s = Solver(wl.shape, list(wl.centers), **kw)
cams = [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
         "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]
s.vote(cams, synth.render_depths(wl), voxel_radius=wl.voxel_radius)
s.iterate(10)
for rep in range(2):
    for impl, zc in (("regs", None), ("tma2", None), ("tma2", "128"), ("tma2", "64"), ("tma2", "32"), ("tma", "64")):
        os.environ["TGV_ENERGY_IMPL"] = impl
        if zc:
            os.environ["TGV_ENERGY_ZC"] = zc
        else:
            os.environ.pop("TGV_ENERGY_ZC", None)
        s.energy()
        s.set_timing(True)
        for _ in range(10):
            e = s.energy()
        t = s.timing()
        s.set_timing(False)
        print(f"C2 rep{rep} {impl} zc={zc}: {t['energy_ms'] / t['energy_launches']:.3f} ms  E {e['E']:.10g}", flush=True)
