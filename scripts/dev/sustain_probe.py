"""Sustained vs duty-cycled fused-sweep rate on a 1024 x 1024 x Z slab of C4 (dev tool):
is the in-bench launch slower than ncu's because of something that builds up over a
long back-to-back run (HBM temperature, power)?  Prints per-20-launch averages of a long
run, then the average of short bursts separated by idle gaps; nvidia-smi samples the
memory temperature / clocks / power alongside.  usage: sustain_probe.py Z [n_long]"""
import os
import subprocess
import sys
import time

import synth
from paper_2107_14790_b200 import Solver

Z = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
N = int(sys.argv[2]) if len(sys.argv) > 2 else 300
wl = synth.workload("C4")
cams = [{"origin": c.origin, "rot": c.rot, "fx": c.f, "fy": c.f, "cx": c.width / 2.0, "cy": c.height / 2.0,
         "width": c.width, "height": c.height, "vote_weight": c.vote_weight} for c in wl.cams]
depths = synth.render_depths(wl)
kw = dict(lam=wl.lam, alpha0=wl.alpha0, alpha1=wl.alpha1, tau=wl.tau, sigma=wl.sigma)
s = Solver((1024, 1024, Z), list(wl.centers), **kw)
s.vote(cams, depths, voxel_radius=wl.voxel_radius)
s.iterate(3)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,temperature.gpu,temperature.memory,clocks.sm,clocks.mem,"
                        "power.draw,clocks_event_reasons.active", "--format=csv,noheader", "-lms", "250"],
                       stdout=open(os.environ.get("SMI_OUT", "/tmp/smi_sustain.csv"), "w"))
time.sleep(0.5)


def timed(n):
    s.set_timing(True)
    s.iterate(n)
    t = s.timing()
    s.set_timing(False)
    return t["fused_ms"] / max(1, t["fused_launches"])


print(f"Z={Z} zc={s.info()['fused_zc']}", flush=True)
blk = [timed(20) for _ in range(N // 20)]
print("long run, ms per launch per block of 20:", " ".join(f"{x:.2f}" for x in blk), flush=True)
gaps = []
for r in range(8):
    time.sleep(2.0)
    gaps.append(timed(4))
print("bursts of 4 after 2 s idle:", " ".join(f"{x:.2f}" for x in gaps), flush=True)
blk2 = [timed(20) for _ in range(5)]
print("long again:", " ".join(f"{x:.2f}" for x in blk2), flush=True)
smi.terminate()
s.close()
