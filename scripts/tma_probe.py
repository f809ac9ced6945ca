"""Quick TMA fused-kernel probe: tiny grids vs the split schedule (bitwise) with a watchdog."""
import sys
import numpy as np
sys.path.insert(0, ".")
import synth
from paper_2107_14790_b200 import Solver

c = [-0.875 + 0.25 * b for b in range(8)]
for shape in [(24, 20, 17), (64, 28, 9), (33, 15, 5), (256, 256, 32)]:
    h = synth.random_histograms(shape, 1)
    a = Solver(shape, c).set_schedule("split").load(h).iterate(5)
    b = Solver(shape, c).set_schedule("fused").load(h).iterate(5)
    du = np.max(np.abs(a.read_u() - b.read_u()))
    dq = np.max(np.abs(a.get("q") - b.get("q")))
    print(shape, "max|du|", du, "max|dq|", dq, "tma", b.info()["fused_tma"], flush=True)
