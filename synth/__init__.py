"""Seeded synthetic inputs for the TGV hot path (the one module both the oracle
side and the CUDA side use).  It holds none of the method's arithmetic: it
renders analytic depth maps and votes them into 8-bin histograms with the
paper's Alg. 1, and defines the workload recipes of
SURVEY.md §8(d) / BASELINE.json ``configs`` (C1-C4).

The recipe (scene, cameras, noise, seed, iteration count, solver parameters)
is restated in DESIGN.md §"Input recipe".
"""
from __future__ import annotations

import ctypes
import functools
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tgv_synth.c")
_LIB = os.path.join(_HERE, "libtgv_synth.so")


def build(force: bool = False) -> str:
    """Compile the generator (gcc, OpenMP).  Returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Prim(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pad", ctypes.c_int32), ("a", ctypes.c_double * 24)]


class _Cam(ctypes.Structure):
    _fields_ = [
        ("origin", ctypes.c_double * 3),
        ("rot", ctypes.c_double * 9),
        ("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
        ("width", ctypes.c_int32), ("height", ctypes.c_int32),
        ("vote_weight", ctypes.c_int32), ("pad", ctypes.c_int32),
    ]


@functools.lru_cache(maxsize=1)
def _lib():
    lib = ctypes.CDLL(build())
    lib.synth_render.argtypes = [ctypes.POINTER(_Prim), ctypes.c_int, ctypes.POINTER(_Cam), ctypes.c_int64,
                                 ctypes.c_uint64, ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
    lib.synth_vote.argtypes = [ctypes.POINTER(_Cam), ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int64,
                               ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p]
    lib.synth_vote_box.argtypes = [ctypes.POINTER(_Cam), ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)] + \
        [ctypes.c_int64] * 6 + [ctypes.c_double, ctypes.c_void_p]
    lib.synth_alg1_bin.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double]
    lib.synth_alg1_bin.restype = ctypes.c_int
    return lib


# ---------------------------------------------------------------------------
# scene / camera description
# ---------------------------------------------------------------------------
@dataclass
class Camera:
    origin: tuple
    rot: np.ndarray  # 3x3 world<-camera, columns = camera x (right), y (down), z (forward)
    f: float
    width: int
    height: int
    vote_weight: int = 1


def look_at(origin, target, width, height, fov_deg, vote_weight=1) -> Camera:
    o = np.asarray(origin, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - o
    fwd /= np.linalg.norm(fwd)
    up = np.array([0.0, 0.0, 1.0])
    if abs(float(fwd @ up)) > 0.99:
        up = np.array([0.0, 1.0, 0.0])
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    rot = np.stack([right, down, fwd], axis=1)
    f = (width / 2.0) / math.tan(math.radians(fov_deg) / 2.0)
    return Camera(tuple(o), rot, f, width, height, vote_weight)


def sphere(c, r):
    return (0, [c[0], c[1], c[2], r])


def plane(z):
    return (1, [z])


def heightfield(base, waves, zmin, zmax):
    a = [0.0] * 24
    a[0] = base
    for o, (amp, kx, ky, ph) in enumerate(waves):
        a[1 + 4 * o: 5 + 4 * o] = [amp, kx, ky, ph]
    a[21], a[22] = zmin, zmax
    a[23] = sum(abs(amp) * math.hypot(kx, ky) for amp, kx, ky, _ in waves)  # Lipschitz bound of H
    return (2, a)


def box(lo, hi):
    """Axis-aligned box (a building of the C5 urban scene)."""
    return (3, [float(lo[0]), float(lo[1]), float(lo[2]), float(hi[0]), float(hi[1]), float(hi[2])])


def fibonacci_sphere(n):
    pts = []
    ga = math.pi * (3.0 - math.sqrt(5.0))
    for i in range(n):
        z = 1.0 - 2.0 * (i + 0.5) / n
        r = math.sqrt(max(0.0, 1.0 - z * z))
        pts.append((r * math.cos(ga * i), r * math.sin(ga * i), z))
    return pts


def hemisphere_dirs(n, el_min_deg=15.0, el_max_deg=85.0):
    ga = math.pi * (3.0 - math.sqrt(5.0))
    s0, s1 = math.sin(math.radians(el_min_deg)), math.sin(math.radians(el_max_deg))
    out = []
    for i in range(n):
        sz = s0 + (i + 0.5) / n * (s1 - s0)
        c = math.sqrt(1.0 - sz * sz)
        out.append((c * math.cos(ga * i), c * math.sin(ga * i), sz))
    return out


# ---------------------------------------------------------------------------
# workloads (BASELINE.json configs[0..3])
# ---------------------------------------------------------------------------
@dataclass
class Workload:
    name: str
    shape: tuple  # (nx, ny, nz)
    iters: int
    seed: int
    noise: float
    floaters: float
    description: str
    # solver parameters of every config (SURVEY.md §8(d) "Parameters for every config")
    lam: float = 0.5
    alpha1: float = 1.0
    alpha0: float = 2.0
    tau: float = 0.25
    sigma: float = 0.25
    centers: tuple = tuple(-0.875 + 0.25 * b for b in range(8))
    voxel_radius: float = 0.5
    prims: list = field(default_factory=list)
    cams: list = field(default_factory=list)

    @property
    def nvox(self) -> int:
        return self.shape[0] * self.shape[1] * self.shape[2]


def _c1() -> Workload:
    c = (15.5, 15.5, 15.5)
    cams = [look_at((c[0] + 40 * d[0], c[1] + 40 * d[1], c[2] + 40 * d[2]), c, 64, 64, 50.0) for d in fibonacci_sphere(16)]
    return Workload("C1", (32, 32, 32), 100, 1, 0.0, 0.0,
                    "32^3 grid, sphere R=10 from 16 depth maps 64x64, 8 bins, 100 iterations",
                    prims=[sphere(c, 10.0)], cams=cams)


def _c2() -> Workload:
    tgt = (128.0, 128.0, 128.0)
    cams = [look_at((tgt[0] + 320 * d[0], tgt[1] + 320 * d[1], tgt[2] + 320 * d[2]), tgt, 512, 512, 60.0)
            for d in hemisphere_dirs(32)]
    return Workload("C2", (256, 256, 256), 500, 2, 0.5, 0.02,
                    "256^3 brick, sphere R=60 + ground plane, 32 depth maps 512x512 with N(0,0.5) noise + 2% floaters, "
                    "8 bins, 500 iterations",
                    prims=[sphere((128.0, 128.0, 150.0), 60.0), plane(70.0)], cams=cams)


def _c3() -> Workload:
    rng = np.random.default_rng(3)
    waves = []
    for o in range(1, 6):
        th = rng.uniform(0, 2 * math.pi)
        k = 2 * math.pi * (2 ** o) / 512.0
        waves.append((80.0 / 2 ** o, k * math.cos(th), k * math.sin(th), rng.uniform(0, 2 * math.pi)))
    amp = sum(w[0] for w in waves)
    cams = []
    for i in range(10):
        for j in range(10):
            x, y = 25.6 + 51.2 * i, 25.6 + 51.2 * j
            cams.append(look_at((x, y, 1500.0), (x, y, 200.0), 1024, 1024, 20.0))
    for h in range(4):
        hd = (math.cos(h * math.pi / 2), math.sin(h * math.pi / 2))
        for i in range(5):
            for j in range(5):
                tx, ty = 51.2 + 102.4 * i, 51.2 + 102.4 * j
                d = 1300.0
                o = (tx - hd[0] * d / math.sqrt(2), ty - hd[1] * d / math.sqrt(2), 200.0 + d / math.sqrt(2))
                cams.append(look_at(o, (tx, ty, 200.0), 1024, 1024, 20.0))
    return Workload("C3", (512, 512, 512), 1000, 3, 1.0, 0.0,
                    "512^3 grid, terrain heightfield from 200 aerial depth maps 1024x1024 (100 nadir + 100 oblique), "
                    "N(0,1) noise, 8 bins, 1000 iterations",
                    prims=[heightfield(200.0, waves, 200.0 - amp - 1, 200.0 + amp + 1)], cams=cams)


def _c4() -> Workload:
    rng = np.random.default_rng(4)
    prims = [plane(100.0)]
    for _ in range(64):
        r = float(rng.uniform(20, 120))
        prims.append(sphere((float(rng.uniform(100, 924)), float(rng.uniform(100, 924)), 100.0 + 0.5 * r), r))
    tgt = (512.0, 512.0, 300.0)
    cams = [look_at((tgt[0] + 1300 * d[0], tgt[1] + 1300 * d[1], tgt[2] + 1300 * d[2]), tgt, 1024, 1024, 60.0)
            for d in hemisphere_dirs(64)]
    return Workload("C4", (1024, 1024, 1024), 200, 4, 0.5, 0.0,
                    "1024^3 grid, 64 spheres (R 20-120) on a ground plane, 64 depth maps 1024x1024, N(0,0.5) noise, "
                    "8 bins, 200 iterations",
                    prims=prims, cams=cams)


def _c5() -> Workload:
    """BASELINE configs[4]: a block-sparse brick set of an urban scene, 3 scale levels.
    The finest level spans 2048 x 2048 x 256 voxels (64 x 64 x 8 bricks of 32^3); which
    bricks exist is decided by the votes (R24), about 2 x 10^4 over the
    levels.  120 buildings (boxes, footprints 40-160, heights 30-200) on a ground plane
    at z = 40, seen by 36 nadir and 28 oblique aerial cameras, 1024 x 1024."""
    rng = np.random.default_rng(5)
    ground = 40.0
    prims = [plane(ground)]
    for _ in range(120):
        w, d = float(rng.uniform(40, 160)), float(rng.uniform(40, 160))
        x0, y0 = float(rng.uniform(64, 1984 - w)), float(rng.uniform(64, 1984 - d))
        prims.append(box((x0, y0, ground - 5.0), (x0 + w, y0 + d, ground + float(rng.uniform(30, 200)))))
    cams = []
    for i in range(6):
        for j in range(6):
            x, y = 170.0 + 341.0 * i, 170.0 + 341.0 * j
            cams.append(look_at((x, y, 2400.0), (x + 1e-3, y, ground), 1024, 1024, 45.0))
    for h in range(4):
        hd = (math.cos(h * math.pi / 2 + 0.3), math.sin(h * math.pi / 2 + 0.3))
        for i in range(7):
            tx, ty = 300.0 + 240.0 * i, 300.0 + 240.0 * ((i * 3 + h) % 7)
            dd = 1800.0
            o = (tx - hd[0] * dd / math.sqrt(2), ty - hd[1] * dd / math.sqrt(2), ground + dd / math.sqrt(2))
            cams.append(look_at(o, (tx, ty, ground), 1024, 1024, 40.0))
    return Workload("C5", (2048, 2048, 256), 200, 5, 0.5, 0.0,
                    "block-sparse brick set of an urban scene (120 buildings on a ground plane), finest level "
                    "2048x2048x256 in 32^3 bricks selected by the votes, 3 scale levels, 64 aerial depth maps "
                    "1024x1024, N(0,0.5) noise, 8 bins, 200 iterations per level",
                    prims=prims, cams=cams)


WORKLOADS = {"C1": _c1, "C2": _c2, "C3": _c3, "C4": _c4, "C5": _c5}


@functools.lru_cache(maxsize=8)
def workload(name: str) -> Workload:
    return WORKLOADS[name]()


def _cams_struct(cams):
    arr = (_Cam * len(cams))()
    for i, c in enumerate(cams):
        arr[i].origin[:] = list(c.origin)
        arr[i].rot[:] = list(np.asarray(c.rot, dtype=np.float64).reshape(-1))
        arr[i].fx = arr[i].fy = c.f
        arr[i].cx, arr[i].cy = c.width / 2.0, c.height / 2.0
        arr[i].width, arr[i].height, arr[i].vote_weight = c.width, c.height, c.vote_weight
    return arr


def render_depths(wl: Workload):
    lib = _lib()
    prims = (_Prim * len(wl.prims))()
    for i, (k, a) in enumerate(wl.prims):
        prims[i].kind = k
        prims[i].a[: len(a)] = list(a)
    cams = _cams_struct(wl.cams)
    depths = []
    for i in range(len(wl.cams)):
        d = np.empty((wl.cams[i].height, wl.cams[i].width), dtype=np.float32)
        lib.synth_render(prims, len(wl.prims), ctypes.byref(cams[i]), i, wl.seed, wl.noise, wl.floaters,
                         d.ctypes.data)
        depths.append(d)
    return depths


def render_depths_indexed(wl: Workload, cam_id: int):
    """Depth map of the single camera wl.cams[0], drawn with global camera index cam_id."""
    lib = _lib()
    prims = (_Prim * len(wl.prims))()
    for i, (k, a) in enumerate(wl.prims):
        prims[i].kind = k
        prims[i].a[: len(a)] = list(a)
    cams = _cams_struct(wl.cams)
    d = np.empty((wl.cams[0].height, wl.cams[0].width), dtype=np.float32)
    lib.synth_render(prims, len(wl.prims), ctypes.byref(cams[0]), cam_id, wl.seed, wl.noise, wl.floaters,
                     d.ctypes.data)
    return d


def vote(cams, depths, nx, ny, z0, z1, r):
    """Alg. 1 over global planes [z0, z1) of an nx*ny*? grid -> uint32 [z1-z0, ny, nx, 8]."""
    lib = _lib()
    cs = _cams_struct(cams)
    ptrs = (ctypes.c_void_p * len(depths))(*[d.ctypes.data for d in depths])
    out = np.empty((z1 - z0, ny, nx, 8), dtype=np.uint32)
    lib.synth_vote(cs, len(cams), ptrs, nx, ny, z0, z1, r, out.ctypes.data)
    return out


def vote_box(cams, depths, box, r):
    """Alg. 1 over the voxel box (x0, x1, y0, y1, z0, z1) -> uint32 [z1-z0, y1-y0, x1-x0, 8]
    (the full-plane vote cropped to the box)."""
    x0, x1, y0, y1, z0, z1 = (int(b) for b in box)
    lib = _lib()
    cs = _cams_struct(cams)
    ptrs = (ctypes.c_void_p * len(depths))(*[d.ctypes.data for d in depths])
    out = np.empty((z1 - z0, y1 - y0, x1 - x0, 8), dtype=np.uint32)
    lib.synth_vote_box(cs, len(cams), ptrs, x0, x1, y0, y1, z0, z1, r, out.ctypes.data)
    return out


def make_histograms_box(name: str, box) -> np.ndarray:
    """uint32 counts of the voxel box (x0, x1, y0, y1, z0, z1) of workload `name`."""
    wl = workload(name)
    return vote_box(wl.cams, _depths_cached(name), box, wl.voxel_radius)


def alg1_bin(depth: float, distance: float, r: float) -> int:
    return _lib().synth_alg1_bin(depth, distance, r)


@functools.lru_cache(maxsize=4)
def _depths_cached(name):
    return render_depths(workload(name))


def make_histograms(name: str, z0: int = 0, z1: int | None = None) -> np.ndarray:
    """uint32 counts [z1-z0, ny, nx, 8] for global planes [z0, z1) of workload `name`."""
    wl = workload(name)
    nx, ny, nz = wl.shape
    z1 = nz if z1 is None else z1
    return vote(wl.cams, _depths_cached(name), nx, ny, z0, z1, wl.voxel_radius)


def random_histograms(shape, seed: int, max_count: int = 12, p_empty: float = 0.2, p_free: float = 0.4):
    """Small seeded histograms with the workloads' value structure (SURVEY.md §8(d)
    'Value structure'): unobserved voxels (W = 0), free-space voxels with all
    votes in bin 7, and mixed near-surface voxels.  uint32 [nz, ny, nx, 8]."""
    nx, ny, nz = shape
    rng = np.random.default_rng(seed)
    h = rng.integers(0, max_count // 3 + 1, size=(nz, ny, nx, 8)).astype(np.uint32)
    kind = rng.uniform(size=(nz, ny, nx))
    h[kind < p_empty] = 0
    free = (kind >= p_empty) & (kind < p_empty + p_free)
    h[free] = 0
    h[free, 7] = rng.integers(1, max_count + 1, size=int(free.sum())).astype(np.uint32)
    return h
