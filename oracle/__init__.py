"""CPU oracle for the TGV hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package.  The product package
``paper_2107_14790_b200`` never imports it, and this package never imports the
product: the two share no code (see oracle/tgv_oracle.c header).

The arithmetic lives in ``tgv_oracle.c`` (plain fp64 loops, each function
citing the passage it follows).  This module only compiles it and marshals
numpy arrays.  Parity status of every function is listed in DESIGN.md §3;
the 3-D minimum value of the functional has no closed form and is pinned by an
independent cone-program optimiser on tiny grids (tests/test_oracle_socp_pin.py)
and by the restricted gap elsewhere.
"""
from __future__ import annotations

import ctypes
import functools
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tgv_oracle.c")
_LIB = os.path.join(_HERE, "libtgv_oracle.so")

# oracle field ids (its own numbering)
U, V0, UBAR, VBAR0, P0, Q0 = 0, 1, 4, 5, 8, 11
FIELDS = {"u": [U], "v": [V0, V0 + 1, V0 + 2], "ubar": [UBAR], "vbar": [VBAR0, VBAR0 + 1, VBAR0 + 2],
          "p": [P0, P0 + 1, P0 + 2], "q": [Q0 + m for m in range(6)]}


def build(force: bool = False) -> str:
    """gcc -O2 -ffp-contract=off (no FMA contraction, no fast-math) + OpenMP."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
                               "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


@functools.lru_cache(maxsize=1)
def _lib():
    lib = ctypes.CDLL(build())
    i64, dbl, vp = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
    lib.oracle_create.argtypes = [i64, i64, i64, i64, i64, ctypes.c_int, vp, dbl, dbl, dbl, dbl, dbl]
    lib.oracle_create.restype = vp
    lib.oracle_destroy.argtypes = [vp]
    lib.oracle_load.argtypes = [vp, vp]
    lib.oracle_dual.argtypes = [vp, ctypes.c_int]
    lib.oracle_primal.argtypes = [vp, ctypes.c_int]
    lib.oracle_iterate.argtypes = [vp, ctypes.c_int, ctypes.c_int]
    lib.oracle_dual_halo.argtypes = [vp]
    lib.oracle_set_tvl1.argtypes = [vp, ctypes.c_int]
    lib.oracle_energy.argtypes = [vp, dbl, vp]
    for fn in ("oracle_get", "oracle_set"):
        getattr(lib, fn).argtypes = [vp, ctypes.c_int, vp]
    for fn in ("oracle_get_plane", "oracle_set_plane"):
        getattr(lib, fn).argtypes = [vp, ctypes.c_int, i64, vp]
    lib.oracle_prox.argtypes = [dbl, dbl, ctypes.c_int, vp, vp]
    lib.oracle_prox.restype = dbl
    for fn in ("oracle_grad", "oracle_div", "oracle_symgrad", "oracle_div2"):
        getattr(lib, fn).argtypes = [i64, i64, i64, vp, vp]
    lib.oracle_max_threads.restype = ctypes.c_int
    lib.oracle_alg1_vote.argtypes = [vp, ctypes.c_int, ctypes.POINTER(vp), i64, i64, i64, i64, vp, dbl, dbl, vp]
    return lib


def max_threads() -> int:
    return int(_lib().oracle_max_threads())


def default_centers(nbins: int = 8) -> np.ndarray:
    """Midpoints of nbins equal bins over [-1, 1] (reading R3; Alg. 1)."""
    return np.array([-1.0 + (2.0 * b + 1.0) / nbins for b in range(nbins)], dtype=np.float64)


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------
# single-voxel prox and whole-grid operators (pinned in tests/test_oracle_*.py)
# ---------------------------------------------------------------------------
def prox(ut: float, t: float, h, c) -> float:
    """argmin_{u in [-1,1]} 1/2 (u-ut)^2 + t sum_b h_b |u - c_b|."""
    h, c = _c(h), _c(c)
    return float(_lib().oracle_prox(float(ut), float(t), len(h), h.ctypes.data, c.ctypes.data))


def _op(name, inp, ncomp_in, ncomp_out):
    inp = _c(inp)
    shape = inp.shape[-3:] if ncomp_in > 1 else inp.shape
    nz, ny, nx = shape
    out = np.empty((ncomp_out, nz, ny, nx) if ncomp_out > 1 else (nz, ny, nx), dtype=np.float64)
    rc = getattr(_lib(), name)(nx, ny, nz, inp.ctypes.data, out.ctypes.data)
    assert rc == 0
    return out


def grad(u):  # [nz,ny,nx] -> [3,nz,ny,nx]
    return _op("oracle_grad", u, 1, 3)


def div(p):  # [3,...] -> [...]
    return _op("oracle_div", p, 3, 1)


def symgrad(v):  # [3,...] -> [6,...] (xx, yy, zz, xy, xz, yz)
    return _op("oracle_symgrad", v, 3, 6)


def div2(q):  # [6,...] -> [3,...]
    return _op("oracle_div2", q, 6, 3)


# ---------------------------------------------------------------------------
# the iteration
# ---------------------------------------------------------------------------
class Oracle:
    """fp64 CPU state of the TGV primal-dual scheme on a grid (or a z-slab of it).

    shape = (nx, ny, nz) of the GLOBAL grid; the state owns planes [zb, ze).
    """

    def __init__(self, shape, lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25, centers=None, zb=0, ze=None,
                 model="tgv"):
        nx, ny, nz = shape
        ze = nz if ze is None else ze
        self.shape, self.zb, self.ze = (nx, ny, nz), zb, ze
        c = default_centers(8) if centers is None else _c(centers)
        self.centers = c
        self.nbins = len(c)
        self._ptr = _lib().oracle_create(nx, ny, nz, zb, ze, len(c), c.ctypes.data, lam, alpha0, alpha1, tau, sigma)
        if not self._ptr:
            raise ValueError("oracle_create: invalid arguments")
        self.model = model
        _lib().oracle_set_tvl1(self._ptr, 1 if model == "tvl1" else 0)

    def __del__(self):
        if getattr(self, "_ptr", None):
            _lib().oracle_destroy(self._ptr)
            self._ptr = None

    @property
    def local_shape(self):
        nx, ny, _ = self.shape
        return (self.ze - self.zb, ny, nx)

    def load(self, counts):
        counts = _c(counts, np.uint32)
        assert counts.shape == self.local_shape + (self.nbins,), counts.shape
        _lib().oracle_load(self._ptr, counts.ctypes.data)
        return self

    def dual(self, threads=1):
        _lib().oracle_dual(self._ptr, threads)

    def dual_halo(self):
        """Slab mode: recompute p on the bottom halo plane and q on the top one."""
        _lib().oracle_dual_halo(self._ptr)

    def primal(self, threads=1):
        _lib().oracle_primal(self._ptr, threads)

    def iterate(self, n, threads=1):
        _lib().oracle_iterate(self._ptr, int(n), int(threads))
        return self

    def get(self, name):
        ids = FIELDS[name]
        out = np.empty((len(ids),) + self.local_shape, dtype=np.float64)
        for k, f in enumerate(ids):
            _lib().oracle_get(self._ptr, f, out[k].ctypes.data)
        return out[0] if len(ids) == 1 else out

    def set(self, name, arr):
        ids = FIELDS[name]
        arr = _c(arr)
        arr = arr.reshape((len(ids),) + self.local_shape)
        for k, f in enumerate(ids):
            _lib().oracle_set(self._ptr, f, np.ascontiguousarray(arr[k]).ctypes.data)

    def get_plane(self, name, comp, z):
        nx, ny, _ = self.shape
        out = np.empty((ny, nx), dtype=np.float64)
        assert _lib().oracle_get_plane(self._ptr, FIELDS[name][comp], z, out.ctypes.data) == 0
        return out

    def set_plane(self, name, comp, z, plane):
        plane = _c(plane)
        assert _lib().oracle_set_plane(self._ptr, FIELDS[name][comp], z, plane.ctypes.data) == 0

    def energy(self, V=None):
        """TGV: V = 2 bounds v in the restricted dual (reading R14); TV-L1 has no v (V = 0)."""
        if V is None:
            V = 0.0 if self.model == "tvl1" else 2.0
        out = np.zeros(7, dtype=np.float64)
        _lib().oracle_energy(self._ptr, V, out.ctypes.data)
        return {"E": out[0], "alpha1": out[1], "alpha0": out[2], "data": out[3], "gap": out[4], "vmax": out[5],
                "dual": out[6]}

    @property
    def u(self):
        return self.get("u")


# ---------------------------------------------------------------------------
# NEXT-1 coarse-to-fine on the dense grid (
# SURVEY.md §8(f) NEXT-1; readings R18-R20)
# ---------------------------------------------------------------------------
def restrict_counts(counts):
    """Coarse voxel (X, Y, Z) = sum of the counts of its <= 8 children
    (2X+{0,1}, 2Y+{0,1}, 2Z+{0,1}) inside the fine grid.  [nz,ny,nx,nb] -> ceil halves."""
    counts = np.asarray(counts, dtype=np.uint64)
    nz, ny, nx, nb = counts.shape
    out = np.zeros(((nz + 1) // 2, (ny + 1) // 2, (nx + 1) // 2, nb), dtype=np.uint64)
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                part = counts[dz::2, dy::2, dx::2]
                out[:part.shape[0], :part.shape[1], :part.shape[2]] += part
    return out.astype(np.uint32)


def prolong_into(fine, coarse):
    """Restart the fine state from the coarse solution: u = parent u, v = parent v / 2
    (per-voxel slope on a grid of half the spacing), ubar = u, vbar = v, p = q = 0."""
    nz, ny, nx = fine.local_shape

    def up(a):
        return np.repeat(np.repeat(np.repeat(a, 2, axis=-3), 2, axis=-2), 2, axis=-1)[..., :nz, :ny, :nx]

    u = up(coarse.get("u"))
    v = up(coarse.get("v")) * 0.5
    fine.set("u", u)
    fine.set("ubar", u)
    fine.set("v", v)
    fine.set("vbar", v)
    fine.set("p", np.zeros((3, nz, ny, nx)))
    fine.set("q", np.zeros((6, nz, ny, nx)))
    return fine


def coarse_to_fine(shape, counts, levels, iters, threads=1, **kw):
    """Solve `levels` levels (coarsest = finest / 2^(levels-1)), `iters` iterations each,
    initialising each finer level from the coarser solution.  Returns the finest Oracle."""
    hs = [np.asarray(counts, dtype=np.uint32)]
    shapes = [tuple(shape)]
    for _ in range(levels - 1):
        hs.append(restrict_counts(hs[-1]))
        shapes.append(tuple((n + 1) // 2 for n in shapes[-1]))
    o = Oracle(shapes[-1], **kw).load(hs[-1]).iterate(iters, threads=threads)
    for lev in range(levels - 2, -1, -1):
        f = Oracle(shapes[lev], **kw).load(hs[lev])
        prolong_into(f, o)
        o = f.iterate(iters, threads=threads)
    return o


# ---------------------------------------------------------------------------
# NEXT-3 z-slab leaves with frozen borders (§4.5, Fig. 9;
# SURVEY.md §8(f) NEXT-3; R23)
# ---------------------------------------------------------------------------
def leaf_step(o, threads=1):
    """One iteration of a leaf: the scheme over the cubes of A (the
    owned planes) while the indicator of B (the halo planes) is frozen.  The duals on
    the edges between A and B (p on the plane below, q on the plane above) are the
    ones a slab recomputes for its halo (oracle_dual_halo), from the frozen values."""
    o.dual(threads)
    o.dual_halo()
    o.primal(threads)


def leaf_from_parent(shape, zb, ze, counts_slab, parent_u, parent_v, **kw):
    """Leaf [zb, ze) of a level: histograms `counts_slab`; u = parent u, v = parent v / 2,
    ubar = u, vbar = v, p = q = 0 on A (R19); on B (planes zb-1, ze inside the grid)
    the same parent values, frozen ("equal to indicator values of
    their parenting cubes, which were estimated on the previous level").
    parent_u [cnz, cny, cnx] / parent_v [3, ...]: the whole parent level."""
    nx, ny, nz = shape
    o = Oracle(shape, zb=zb, ze=ze, **kw).load(counts_slab)

    def up(a):
        return np.repeat(np.repeat(np.repeat(a, 2, axis=-3), 2, axis=-2), 2, axis=-1)[..., :nz, :ny, :nx]

    U_, V_ = up(np.asarray(parent_u, np.float64)), up(np.asarray(parent_v, np.float64)) * 0.5
    o.set("u", U_[zb:ze])
    o.set("ubar", U_[zb:ze])
    o.set("v", V_[:, zb:ze])
    o.set("vbar", V_[:, zb:ze])
    o.set("p", np.zeros((3, ze - zb, ny, nx)))
    o.set("q", np.zeros((6, ze - zb, ny, nx)))
    for z in (zb - 1, ze):
        if 0 <= z < nz:
            o.set_plane("u", 0, z, U_[z])
            o.set_plane("ubar", 0, z, U_[z])
            for d in range(3):
                o.set_plane("v", d, z, V_[d, z])
                o.set_plane("vbar", d, z, V_[d, z])
    return o


def out_of_core(shape, counts, levels, iters, leaf_voxels, threads=1, **kw):
    """Coarse-to-fine over z-slab leaves: level by level (coarsest first), leaves of
    max(1, leaf_voxels // (nx ny)) consecutive planes from z = 0 (a level of at most
    leaf_voxels voxels is one leaf), each solved for `iters`
    iterations with frozen borders from the parent level.  The coarsest level must be
    one leaf.  Returns (u, v) of the finest level, fp64."""
    hs = [np.asarray(counts, dtype=np.uint32)]
    shapes = [tuple(shape)]
    for _ in range(levels - 1):
        hs.append(restrict_counts(hs[-1]))
        shapes.append(tuple((n + 1) // 2 for n in shapes[-1]))
    prev = None
    for lev in range(levels - 1, -1, -1):
        nx, ny, nz = shapes[lev]
        planes = nz if nx * ny * nz <= leaf_voxels else max(1, leaf_voxels // (nx * ny))
        if prev is None and planes < nz:
            raise ValueError("the coarsest level must fit in one leaf")
        u = np.zeros((nz, ny, nx))
        v = np.zeros((3, nz, ny, nx))
        for zb in range(0, nz, planes):
            ze = min(zb + planes, nz)
            if prev is None:
                o = Oracle(shapes[lev], zb=zb, ze=ze, **kw).load(hs[lev][zb:ze])
            else:
                o = leaf_from_parent(shapes[lev], zb, ze, hs[lev][zb:ze], prev[0], prev[1], **kw)
            for _ in range(iters):
                leaf_step(o, threads)
            u[zb:ze] = o.u
            v[:, zb:ze] = o.get("v")
        prev = (u, v)
    return prev


# ---------------------------------------------------------------------------
# NEXT-2 histogram voting, Alg. 1
# ---------------------------------------------------------------------------
class OracleCamera(ctypes.Structure):
    _fields_ = [("origin", ctypes.c_double * 3), ("rot", ctypes.c_double * 9), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("vote_weight", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


def alg1_vote(cams, depths, nx, ny, z0, z1, origin=(0.0, 0.0, 0.0), voxel_size=1.0, r=0.5):
    """cams: sequence of dicts (origin, rot 3x3 world<-camera, fx, fy, cx, cy, width, height, vote_weight);
    depths: float32 [h, w] z-depth maps (NaN = none).  -> uint32 [z1-z0, ny, nx, 8]."""
    arr = (OracleCamera * len(cams))()
    for i, c in enumerate(cams):
        arr[i].origin[:] = [float(x) for x in c["origin"]]
        arr[i].rot[:] = [float(x) for x in np.asarray(c["rot"], dtype=np.float64).reshape(-1)]
        arr[i].fx, arr[i].fy, arr[i].cx, arr[i].cy = c["fx"], c["fy"], c["cx"], c["cy"]
        arr[i].width, arr[i].height, arr[i].vote_weight = c["width"], c["height"], c.get("vote_weight", 1)
    ds = [np.ascontiguousarray(d, dtype=np.float32) for d in depths]
    ptrs = (ctypes.c_void_p * len(ds))(*[d.ctypes.data for d in ds])
    out = np.empty((z1 - z0, ny, nx, 8), dtype=np.uint32)
    o = np.asarray(origin, dtype=np.float64)
    _lib().oracle_alg1_vote(arr, len(cams), ptrs, nx, ny, z0, z1, o.ctypes.data, float(voxel_size), float(r),
                            out.ctypes.data)
    return out
