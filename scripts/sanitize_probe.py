"""Small runs of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2107_14790_b200 import Group, Solver  # noqa: E402
from paper_2107_14790_b200.multilevel import coarse_to_fine  # noqa: E402

C8 = [-0.875 + 0.25 * b for b in range(8)]
shape = (70, 33, 21)
h = synth.random_histograms(shape, 1)
for sched in ("fused", "split"):
    s = Solver(shape, C8).set_schedule(sched).load(h).iterate(3)
    s.energy()
    s.close()
os.environ["TGV_FUSED_IMPL"] = "regs"
Solver(shape, C8).load(h).iterate(3).close()
os.environ.pop("TGV_FUSED_IMPL")
Solver(shape, C8).set_model("tvl1").load(h).iterate(3).close()  # TMA single sweep
Solver(shape, C8).set_schedule("split").set_model("tvl1").load(h).iterate(3).close()
os.environ["TGV_FUSED_IMPL"] = "regs"
Solver(shape, C8).set_model("tvl1").load(h).iterate(3).close()
os.environ.pop("TGV_FUSED_IMPL")
Group(shape, [0, 7, 21], C8).load(h).iterate(3).close()
coarse_to_fine(shape, h, C8, levels=2, iters=2).close()
cam = {"origin": (35.0, 16.0, -40.0), "rot": np.eye(3), "fx": 40.0, "fy": 40.0, "cx": 32.0, "cy": 32.0,
       "width": 64, "height": 64}
Solver(shape, C8).vote([cam], [np.full((64, 64), 50.0, np.float32)]).iterate(2).close()
# NEXT-3: leaves (border duals stored), device coarsening of narrow counts, slab prolongation
from paper_2107_14790_b200 import out_of_core  # noqa: E402
leaf = Solver.leaf(shape, C8, 5, 14).load_coarsened(h[5:14].astype(np.uint8), shape, 1)
cs = tuple((n + 1) // 2 for n in shape)
leaf.prolong_slab(np.zeros((6, cs[1], cs[0]), np.float32), np.zeros((3, 6, cs[1], cs[0]), np.float32), 2)
leaf.iterate(3).close()
out_of_core.solve(shape, h, C8, levels=2, iters=2, leaf_voxels=70 * 33 * 6)
# NEXT-3 brick sets: votes, refinement, dual (solved bricks + frozen faces), primal,
# prolongation, energy, count read-back
from paper_2107_14790_b200.bricks import BrickSolver  # noqa: E402
bc = np.array([(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 1), (2, 1, 1)], np.int32)
bf = np.array([0, 0, 1, 0, 1], bool)
coarse = BrickSolver(8, np.unique(bc // 2, axis=0)).vote([cam], [np.full((64, 64), 50.0, np.float32)])
coarse.refine_flags(1)
coarse.iterate(2)
fine = BrickSolver(8, bc, bf).vote([cam], [np.full((64, 64), 50.0, np.float32)]).prolong_from(coarse)
fine.iterate(3)
fine.energy()
fine.read_counts()
fine.close()
coarse.close()
# the fused brick sweep (32^3 bricks): frozen x-neighbours on both sides (x-face cells, cp.async rings),
# a frozen y-neighbour (face launch), a missing z-neighbour
fc = np.array([(0, 0, 0), (1, 0, 0), (2, 0, 0), (1, 1, 0)], np.int32)
ff = np.array([1, 0, 1, 1], bool)
hb = synth.random_histograms((32, 32, 4 * 32), 3).reshape(4, 32, 32, 32, 8)
fb = BrickSolver(32, fc, ff).load(hb)
fb.set_primal(np.full((4, 32, 32, 32), 0.25, np.float32), np.full((4, 3, 32, 32, 32), 0.01, np.float32))
fb.iterate(2)
fb.energy()
fb.close()
# 2:1 mixed-level set (R27): a level-1 brick with level-0 bricks on its +x face (one quadrant
# missing) and a same-level chain; frozen bricks of both levels; the uniform kernels on its
# regular bricks, the mixed kernels (dual on solved bricks and frozen faces, primal, energy),
# votes per level and prolongation into levels 0 / 1
ml = np.array([1, 0, 0, 0, 0, 1], np.uint8)
mc = np.array([(0, 0, 0), (2, 0, 0), (2, 1, 0), (2, 0, 1), (3, 0, 0), (0, 1, 0)], np.int32)
mf = np.array([0, 0, 1, 0, 0, 1], bool)
mco = BrickSolver(8, np.array([(0, 0, 0), (1, 0, 0), (0, 1, 0)], np.int32)).vote([cam], [np.full((64, 64), 50.0, np.float32)])
mco.iterate(2)
mx = BrickSolver(8, mc, mf, levels=ml).vote([cam], [np.full((64, 64), 50.0, np.float32)]).prolong_from(mco)
mx.iterate(3)
mx.energy()
mx.close()
mco.close()
print("sanitize probe done")
