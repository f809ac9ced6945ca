"""NEXT-1: coarse-to-fine TGV solve on a dense grid ("we have
implemented primal-dual iterations over a coarse-to-fine scheme ... 200 iterations
are enough for convergence on each level"; §4.5).

Orchestration only: every step (restriction of the histograms, the iterations,
the prolongation of u and v) runs in libtgv.so's kernels through the C ABI
(tgv_restrict_from, tgv_iterate, tgv_prolong_from).
"""
from __future__ import annotations

from .tgv import Solver


def level_shapes(shape, levels):
    shapes = [tuple(int(n) for n in shape)]
    for _ in range(levels - 1):
        shapes.append(tuple((n + 1) // 2 for n in shapes[-1]))
    return shapes


def coarse_to_fine(shape, counts, centers, levels=3, iters=200, schedule="fused", device=0, **params):
    """Load `counts` on the finest grid, restrict to `levels` levels, solve the
    coarsest from its initialisation, then `iters` iterations per level, each finer
    level restarted from the coarser solution.  Returns the finest Solver."""
    shapes = level_shapes(shape, levels)
    solvers = [Solver(shapes[0], centers, device=device, **params).set_schedule(schedule).load(counts)]
    for lev in range(1, levels):
        solvers.append(Solver(shapes[lev], centers, device=device, **params).set_schedule(schedule)
                       .restrict_from(solvers[-1]))
    solvers[-1].iterate(iters)
    for lev in range(levels - 2, -1, -1):
        solvers[lev].prolong_from(solvers[lev + 1]).iterate(iters)
        solvers[lev + 1].close()
    return solvers[0]
