"""Thin ctypes binding of include/tgv_bricks.h: block-sparse brick sets (NEXT-3,
DESIGN.md reading R24).  Argument marshalling only; every step runs in libtgv.so.

``BrickSolver`` keeps the context's lifetime and converts brick-major numpy arrays:
u [nbricks, E, E, E] (z, y, x inside a brick), v [nbricks, 3, E, E, E] (the ABI's
component-major v is transposed here), counts [nbricks, E, E, E, nbins].
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import tgv
from .tgv import _check, lib, tgv_params, tgv_timing

EXPORTS = ["tgv_bricks_create", "tgv_bricks_load", "tgv_bricks_set_primal", "tgv_bricks_iterate", "tgv_bricks_read",
           "tgv_bricks_energy", "tgv_bricks_set_timing", "tgv_bricks_get_timing", "tgv_bricks_info",
           "tgv_bricks_last_error", "tgv_bricks_destroy", "tgv_bricks_vote_depth_maps", "tgv_bricks_read_counts",
           "tgv_bricks_reset", "tgv_bricks_refine_flags", "tgv_bricks_prolong_from", "tgv_bricks_set_schedule",
           "tgv_bricks_create_mixed"]


class tgv_bricks_info_t(ctypes.Structure):
    _fields_ = [("device_bytes", ctypes.c_int64), ("count_bytes", ctypes.c_int32), ("edge", ctypes.c_int32),
                ("nbricks", ctypes.c_int64), ("nfrozen", ctypes.c_int64), ("solved_voxels", ctypes.c_int64),
                ("s_voxels", ctypes.c_int64), ("schedule", ctypes.c_int32), ("pad", ctypes.c_int32)]


class tgv_brickset(ctypes.Structure):
    _fields_ = [("edge", ctypes.c_int32), ("nbricks", ctypes.c_int64), ("coords", ctypes.c_void_p),
                ("frozen", ctypes.c_void_p)]


def _setup():
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    lib.tgv_bricks_create.argtypes = [ctypes.POINTER(tgv_brickset), ctypes.POINTER(tgv_params), ctypes.c_int,
                                      ctypes.POINTER(vp)]
    lib.tgv_bricks_create_mixed.argtypes = [ctypes.POINTER(tgv_brickset), vp, ctypes.POINTER(tgv_params), ctypes.c_int,
                                            ctypes.POINTER(vp)]
    lib.tgv_bricks_load.argtypes = [vp, vp, ctypes.c_int, i64]
    lib.tgv_bricks_set_primal.argtypes = [vp, vp, vp, i64]
    lib.tgv_bricks_iterate.argtypes = [vp, i32]
    lib.tgv_bricks_read.argtypes = [vp, ctypes.c_int, vp, i64]
    lib.tgv_bricks_energy.argtypes = [vp, vp]
    lib.tgv_bricks_set_timing.argtypes = [vp, ctypes.c_int]
    lib.tgv_bricks_get_timing.argtypes = [vp, ctypes.POINTER(tgv_timing)]
    lib.tgv_bricks_info.argtypes = [vp, ctypes.POINTER(tgv_bricks_info_t)]
    lib.tgv_bricks_vote_depth_maps.argtypes = [vp, ctypes.POINTER(tgv.tgv_camera), ctypes.c_int, ctypes.POINTER(vp),
                                               vp, ctypes.c_double, ctypes.c_double]
    lib.tgv_bricks_read_counts.argtypes = [vp, vp, i64]
    lib.tgv_bricks_reset.argtypes = [vp]
    lib.tgv_bricks_refine_flags.argtypes = [vp, i32, vp, i64]
    lib.tgv_bricks_prolong_from.argtypes = [vp, vp]
    lib.tgv_bricks_set_schedule.argtypes = [vp, ctypes.c_int]
    lib.tgv_bricks_last_error.argtypes = [vp]
    lib.tgv_bricks_last_error.restype = ctypes.c_char_p
    lib.tgv_bricks_destroy.argtypes = [vp]
    lib.tgv_bricks_destroy.restype = None
    for n in EXPORTS:
        if n not in ("tgv_bricks_last_error", "tgv_bricks_destroy"):
            getattr(lib, n).restype = ctypes.c_int


_setup()


def _bcheck(rc, ctx=None):
    if rc != tgv.TGV_OK:
        raise tgv.TgvError(rc, lib.tgv_bricks_last_error(ctx).decode(errors="replace"))


class BrickSolver:
    """One block-sparse level on one GPU (include/tgv_bricks.h)."""

    def __init__(self, edge, coords, frozen=None, centers=None, lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25,
                 device=0, levels=None):
        """levels: per-brick level of a 2:1 mixed-level set (tgv_bricks_create_mixed, R27),
        coordinates in each brick's own level units; None = a one-level set."""
        coords = np.ascontiguousarray(np.asarray(coords, dtype=np.int32).reshape(-1, 3))
        self.E, self.nbricks = int(edge), len(coords)
        self.nvox = self.nbricks * self.E ** 3
        fr = None if frozen is None else np.ascontiguousarray(np.asarray(frozen, dtype=np.uint8).reshape(-1))
        centers = [-0.875 + 0.25 * b for b in range(8)] if centers is None else [float(x) for x in centers]
        self.nbins = len(centers)
        cc = (ctypes.c_float * len(centers))(*centers)
        P = tgv_params(len(centers), ctypes.cast(cc, ctypes.POINTER(ctypes.c_float)), lam, alpha0, alpha1, tau, sigma)
        S = tgv_brickset(self.E, self.nbricks, coords.ctypes.data, None if fr is None else fr.ctypes.data)
        lv = None if levels is None else np.ascontiguousarray(np.asarray(levels, dtype=np.uint8).reshape(-1))
        self._keep = (coords, fr, lv)
        out = ctypes.c_void_p()
        if lv is None:
            _bcheck(lib.tgv_bricks_create(ctypes.byref(S), ctypes.byref(P), int(device), ctypes.byref(out)))
        else:
            if lv.size != self.nbricks:
                raise ValueError(f"levels has {lv.size} entries for {self.nbricks} bricks")
            _bcheck(lib.tgv_bricks_create_mixed(ctypes.byref(S), lv.ctypes.data, ctypes.byref(P), int(device),
                                                ctypes.byref(out)))
        self.ctx = out

    def close(self):
        if getattr(self, "ctx", None):
            lib.tgv_bricks_destroy(self.ctx)
            self.ctx = None

    __del__ = close

    def load(self, counts):
        a = np.ascontiguousarray(counts)
        if a.dtype not in (np.uint8, np.uint16, np.uint32):
            a = a.astype(np.uint32)
        _bcheck(lib.tgv_bricks_load(self.ctx, a.ctypes.data, a.dtype.itemsize, a.size), self.ctx)
        return self

    def vote(self, cams, depths, grid_origin=(0.0, 0.0, 0.0), voxel_size=1.0, voxel_radius=0.5):
        """cams / depths as tgv.tgv_vote_depth_maps (dicts; float32 [h, w], NaN = no depth)."""
        arr, ptrs, ds = tgv._camera_args(cams, depths)
        o = np.asarray(grid_origin, dtype=np.float64)
        _bcheck(lib.tgv_bricks_vote_depth_maps(self.ctx, arr, len(cams), ptrs, o.ctypes.data, float(voxel_size),
                                               float(voxel_radius)), self.ctx)
        return self

    def read_counts(self):
        out = np.empty((self.nbricks,) + (self.E,) * 3 + (self.nbins,), dtype=np.uint32)
        _bcheck(lib.tgv_bricks_read_counts(self.ctx, out.ctypes.data, out.size), self.ctx)
        return out

    def reset(self):
        _bcheck(lib.tgv_bricks_reset(self.ctx), self.ctx)
        return self

    def refine_flags(self, min_votes=2):
        out = np.empty((self.nbricks, 8), dtype=np.uint8)
        _bcheck(lib.tgv_bricks_refine_flags(self.ctx, int(min_votes), out.ctypes.data, out.size), self.ctx)
        return out

    def prolong_from(self, coarse: "BrickSolver"):
        _bcheck(lib.tgv_bricks_prolong_from(self.ctx, coarse.ctx), self.ctx)
        return self

    def set_primal(self, u, v=None):
        u = np.ascontiguousarray(u, dtype=np.float32).reshape(-1)
        vv = None
        if v is not None:  # [nbricks, 3, ...] -> component-major [3, nbricks, ...]
            vv = np.ascontiguousarray(np.moveaxis(np.asarray(v, np.float32).reshape(self.nbricks, 3, -1), 1, 0))
        _bcheck(lib.tgv_bricks_set_primal(self.ctx, u.ctypes.data, None if vv is None else vv.ctypes.data, u.size),
                self.ctx)
        return self

    def iterate(self, n):
        _bcheck(lib.tgv_bricks_iterate(self.ctx, int(n)), self.ctx)
        return self

    def read(self, field, out=None):
        """One field of every brick as [nbricks, E, E, E] float32.  out: a C-contiguous float32
        host buffer of nvox elements to fill instead of a new array (pinned: a fast D2H)."""
        if out is None:
            out = np.empty(self.nvox, dtype=np.float32)
        elif not (isinstance(out, np.ndarray) and out.dtype == np.float32 and out.flags.c_contiguous
                  and out.size == self.nvox):
            raise ValueError("out must be a C-contiguous float32 array of nvox elements")
        _bcheck(lib.tgv_bricks_read(self.ctx, int(field), out.ctypes.data, out.size), self.ctx)
        return out.reshape((self.nbricks,) + (self.E,) * 3)

    def get(self, name):
        ids = tgv.FIELDS[name]
        if len(ids) == 1:
            return self.read(ids[0])
        return np.stack([self.read(f) for f in ids], axis=1)

    def read_u(self, out=None):
        return self.read(tgv.FIELD_U, out)

    def energy(self):
        out = np.zeros(6, dtype=np.float64)
        _bcheck(lib.tgv_bricks_energy(self.ctx, out.ctypes.data), self.ctx)
        return {"E": out[0], "alpha1": out[1], "alpha0": out[2], "data": out[3], "gap": out[4], "vmax": out[5]}

    def set_schedule(self, schedule):
        """"fused" (default for 32^3 bricks) or "split" (or the tgv.SCHEDULE_* value)."""
        v = {"fused": tgv.SCHEDULE_FUSED, "split": tgv.SCHEDULE_SPLIT}.get(schedule, schedule)
        _bcheck(lib.tgv_bricks_set_schedule(self.ctx, int(v)), self.ctx)
        return self

    def set_timing(self, enable=True):
        _bcheck(lib.tgv_bricks_set_timing(self.ctx, 1 if enable else 0), self.ctx)

    def timing(self):
        t = tgv_timing()
        _bcheck(lib.tgv_bricks_get_timing(self.ctx, ctypes.byref(t)), self.ctx)
        return {k: getattr(t, k) for k, _ in tgv_timing._fields_}

    def info(self):
        t = tgv_bricks_info_t()
        _bcheck(lib.tgv_bricks_info(self.ctx, ctypes.byref(t)))
        return {k: getattr(t, k) for k, _ in tgv_bricks_info_t._fields_}
