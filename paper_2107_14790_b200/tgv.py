"""Thin ctypes binding of the C ABI in include/tgv.h (argument marshalling only).

Every step of the solver runs in libtgv.so's sm_100a kernels; this module
never computes.  The functions carry the ABI's names; ``Solver`` is a small
convenience wrapper (context lifetime, torch.distributed bootstrap of the NCCL
unique id, numpy/torch host buffers).  There is no fallback: if libtgv.so is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TGV_LIB") or os.path.join(_PKG, "lib", "libtgv.so")  # TGV_LIB: A/B builds (dev)

TGV_OK, TGV_EINVAL, TGV_ENOMEM, TGV_ECUDA, TGV_ENCCL, TGV_ESTATE, TGV_ERANGE = 0, -1, -2, -3, -4, -5, -6
SCHEDULE_FUSED, SCHEDULE_SPLIT = 0, 1
MODEL_TGV, MODEL_TVL1 = 0, 1
FIELD_U, FIELD_V, FIELD_UBAR, FIELD_VBAR, FIELD_P, FIELD_Q, NUM_FIELDS = 0, 1, 4, 5, 8, 11, 17
FIELDS = {"u": [0], "v": [1, 2, 3], "ubar": [4], "vbar": [5, 6, 7], "p": [8, 9, 10],
          "q": [11, 12, 13, 14, 15, 16]}

EXPORTS = ["tgv_get_unique_id", "tgv_create", "tgv_load_histograms", "tgv_reset", "tgv_iterate", "tgv_read_u",
           "tgv_read_field", "tgv_write_field", "tgv_energy", "tgv_set_schedule", "tgv_set_model", "tgv_set_timing", "tgv_get_timing", "tgv_info",
           "tgv_destroy", "tgv_status_string", "tgv_last_error", "tgv_create_group", "tgv_group_iterate",
           "tgv_group_energy", "tgv_restrict_from", "tgv_prolong_from", "tgv_vote_depth_maps", "tgv_read_counts",
           "tgv_create_leaf", "tgv_set_border", "tgv_load_histograms_coarsened", "tgv_prolong_slab",
           "tgv_leaf_rebind", "tgv_iterate_async", "tgv_sync", "tgv_peer_export", "tgv_peer_import",
           "tgv_stage_histograms", "tgv_load_staged", "tgv_read_u_async", "tgv_wait_io"]


class tgv_layout(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
                ("z_begin", ctypes.c_int64), ("z_end", ctypes.c_int64), ("brick", ctypes.c_int32 * 3)]


class tgv_params(ctypes.Structure):
    _fields_ = [("nbins", ctypes.c_int32), ("bin_centers", ctypes.POINTER(ctypes.c_float)),
                ("lambda_", ctypes.c_float), ("alpha0", ctypes.c_float), ("alpha1", ctypes.c_float),
                ("tau", ctypes.c_float), ("sigma", ctypes.c_float)]


class tgv_timing(ctypes.Structure):
    _fields_ = [("dual_ms", ctypes.c_double), ("primal_ms", ctypes.c_double), ("fused_ms", ctypes.c_double),
                ("energy_ms", ctypes.c_double), ("halo_ms", ctypes.c_double), ("dual_launches", ctypes.c_int64),
                ("primal_launches", ctypes.c_int64), ("fused_launches", ctypes.c_int64),
                ("energy_launches", ctypes.c_int64), ("halo_exchanges", ctypes.c_int64)]


class tgv_camera(ctypes.Structure):
    _fields_ = [("origin", ctypes.c_double * 3), ("rot", ctypes.c_double * 9), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("vote_weight", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


class tgv_info_t(ctypes.Structure):
    _fields_ = [("row_pitch", ctypes.c_int64), ("device_bytes", ctypes.c_int64), ("count_bytes", ctypes.c_int32),
                ("count_slots", ctypes.c_int32), ("schedule", ctypes.c_int32), ("model", ctypes.c_int32),
                ("fused_zc", ctypes.c_int32), ("fused_tma", ctypes.c_int32),
                ("bytes_dual", ctypes.c_int64), ("bytes_primal", ctypes.c_int64), ("bytes_fused", ctypes.c_int64),
                ("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("iteration", ctypes.c_int64),
                ("peer_halo", ctypes.c_int32), ("pad", ctypes.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtgv.so not built ({LIB_PATH}); run __graft_entry__.build() -- there is no fallback")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    lib.tgv_get_unique_id.argtypes = [ctypes.c_char_p]
    lib.tgv_create.argtypes = [ctypes.POINTER(tgv_layout), ctypes.POINTER(tgv_params), ctypes.c_int, ctypes.c_int,
                               ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(vp)]
    lib.tgv_load_histograms.argtypes = [vp, vp, i64]
    lib.tgv_reset.argtypes = [vp]
    lib.tgv_iterate.argtypes = [vp, i32]
    lib.tgv_iterate_async.argtypes = [vp, i32]
    lib.tgv_sync.argtypes = [vp]
    lib.tgv_read_u.argtypes = [vp, vp, i64]
    lib.tgv_stage_histograms.argtypes = [vp, vp, ctypes.c_int, i64]
    lib.tgv_load_staged.argtypes = [vp]
    lib.tgv_read_u_async.argtypes = [vp, vp, i64]
    lib.tgv_wait_io.argtypes = [vp]
    lib.tgv_read_field.argtypes = [vp, ctypes.c_int, vp, i64]
    lib.tgv_write_field.argtypes = [vp, ctypes.c_int, vp, i64]
    lib.tgv_energy.argtypes = [vp, vp]
    lib.tgv_set_schedule.argtypes = [vp, ctypes.c_int]
    lib.tgv_set_model.argtypes = [vp, ctypes.c_int]
    lib.tgv_set_timing.argtypes = [vp, ctypes.c_int]
    lib.tgv_get_timing.argtypes = [vp, ctypes.POINTER(tgv_timing)]
    lib.tgv_info.argtypes = [vp, ctypes.POINTER(tgv_info_t)]
    lib.tgv_create_group.argtypes = [ctypes.POINTER(tgv_layout), ctypes.POINTER(tgv_params), ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_int), ctypes.POINTER(vp)]
    lib.tgv_group_iterate.argtypes = [ctypes.POINTER(vp), ctypes.c_int, i32]
    lib.tgv_group_energy.argtypes = [ctypes.POINTER(vp), ctypes.c_int, vp]
    lib.tgv_vote_depth_maps.argtypes = [vp, ctypes.POINTER(tgv_camera), ctypes.c_int, ctypes.POINTER(vp), vp,
                                        ctypes.c_double, ctypes.c_double]
    lib.tgv_read_counts.argtypes = [vp, vp, i64]
    lib.tgv_restrict_from.argtypes = [vp, vp]
    lib.tgv_prolong_from.argtypes = [vp, vp]
    lib.tgv_create_leaf.argtypes = [ctypes.POINTER(tgv_layout), ctypes.POINTER(tgv_params), ctypes.c_int,
                                    ctypes.POINTER(vp)]
    lib.tgv_set_border.argtypes = [vp, ctypes.c_int, vp, vp, vp, vp]
    lib.tgv_load_histograms_coarsened.argtypes = [vp, vp, ctypes.c_int, i64, i64, i64, i64, ctypes.c_int]
    lib.tgv_prolong_slab.argtypes = [vp, vp, vp, i64, i64, i64, i64]
    lib.tgv_leaf_rebind.argtypes = [vp, i64, i64]
    lib.tgv_peer_export.argtypes = [vp, ctypes.c_char_p]
    lib.tgv_peer_import.argtypes = [vp, ctypes.c_int, ctypes.c_char_p]
    lib.tgv_destroy.argtypes = [vp]
    lib.tgv_destroy.restype = None
    lib.tgv_status_string.argtypes = [ctypes.c_int]
    lib.tgv_status_string.restype = ctypes.c_char_p
    lib.tgv_last_error.argtypes = [vp]
    lib.tgv_last_error.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("tgv_destroy", "tgv_status_string", "tgv_last_error"):
            getattr(lib, name).restype = ctypes.c_int
    return lib


lib = _load()


class TgvError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{lib.tgv_status_string(status).decode()} -- {detail}")
        self.status = status


def _check(rc: int, ctx=None):
    if rc != TGV_OK:
        raise TgvError(rc, lib.tgv_last_error(ctx).decode(errors="replace"))


def _host_ptr(a, dtype):
    """Pointer + element count of a C-contiguous host buffer (numpy or torch CPU tensor)."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(a, torch.Tensor):
        if a.device.type != "cpu" or not a.is_contiguous():
            raise ValueError("host buffer must be a contiguous CPU tensor")
        if a.dtype != {np.uint32: torch.uint32, np.float32: torch.float32}[dtype]:
            raise TypeError(f"host buffer dtype {a.dtype}, expected {np.dtype(dtype).name}")
        return a.data_ptr(), a.numel()
    if not isinstance(a, np.ndarray):
        raise TypeError(f"host buffer must be a numpy array or CPU tensor, got {type(a).__name__}")
    if a.dtype != dtype:
        raise TypeError(f"host buffer dtype {a.dtype}, expected {np.dtype(dtype).name}")
    if not a.flags.c_contiguous:
        raise ValueError("host buffer must be C-contiguous (no negative or gapped strides)")
    return a.ctypes.data, a.size


# ---- ABI-named functions -------------------------------------------------------
def tgv_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.tgv_get_unique_id(buf))
    return buf.raw


def tgv_create(shape, z_begin, z_end, centers, lam, alpha0, alpha1, tau, sigma, rank=0, nranks=1, uid=None,
               device=0):
    nx, ny, nz = shape
    L = tgv_layout(nx, ny, nz, z_begin, z_end, (ctypes.c_int32 * 3)(0, 0, 0))
    c = (ctypes.c_float * len(centers))(*[float(x) for x in centers])
    P = tgv_params(len(centers), ctypes.cast(c, ctypes.POINTER(ctypes.c_float)), lam, alpha0, alpha1, tau, sigma)
    out = ctypes.c_void_p()
    _check(lib.tgv_create(ctypes.byref(L), ctypes.byref(P), rank, nranks, uid, device, ctypes.byref(out)))
    return out


def tgv_load_histograms(ctx, counts):
    p, n = _host_ptr(counts, np.uint32)
    _check(lib.tgv_load_histograms(ctx, p, n), ctx)


def tgv_reset(ctx):
    _check(lib.tgv_reset(ctx), ctx)


def tgv_iterate(ctx, n: int):
    _check(lib.tgv_iterate(ctx, int(n)), ctx)


def tgv_iterate_async(ctx, n: int):
    _check(lib.tgv_iterate_async(ctx, int(n)), ctx)


def tgv_sync(ctx):
    _check(lib.tgv_sync(ctx), ctx)


def tgv_read_u(ctx, out):
    p, n = _host_ptr(out, np.float32)
    _check(lib.tgv_read_u(ctx, p, n), ctx)
    return out


def tgv_stage_histograms(ctx, counts):
    """counts: C-contiguous uint8 / uint16 / uint32 array (pinned for overlap); must stay alive
    and unchanged until the next tgv_load_staged."""
    a = counts
    if not isinstance(a, np.ndarray) or a.dtype not in (np.uint8, np.uint16, np.uint32):
        raise TypeError("counts must be a uint8 / uint16 / uint32 numpy array")
    if not a.flags.c_contiguous:
        raise ValueError("counts must be C-contiguous")
    _check(lib.tgv_stage_histograms(ctx, a.ctypes.data, a.dtype.itemsize, a.size), ctx)


def tgv_load_staged(ctx):
    _check(lib.tgv_load_staged(ctx), ctx)


def tgv_read_u_async(ctx, out):
    """out must stay alive until tgv_wait_io."""
    p, n = _host_ptr(out, np.float32)
    _check(lib.tgv_read_u_async(ctx, p, n), ctx)
    return out


def tgv_wait_io(ctx):
    _check(lib.tgv_wait_io(ctx), ctx)


def tgv_read_field(ctx, field: int, out):
    p, n = _host_ptr(out, np.float32)
    _check(lib.tgv_read_field(ctx, int(field), p, n), ctx)
    return out


def tgv_write_field(ctx, field: int, arr):
    p, n = _host_ptr(arr, np.float32)
    _check(lib.tgv_write_field(ctx, int(field), p, n), ctx)


def tgv_energy(ctx) -> np.ndarray:
    out = np.zeros(6, dtype=np.float64)
    _check(lib.tgv_energy(ctx, out.ctypes.data), ctx)
    return out


def tgv_set_schedule(ctx, schedule: int):
    _check(lib.tgv_set_schedule(ctx, int(schedule)), ctx)


def tgv_set_model(ctx, model: int):
    _check(lib.tgv_set_model(ctx, int(model)), ctx)


def tgv_set_timing(ctx, enable: bool):
    _check(lib.tgv_set_timing(ctx, 1 if enable else 0), ctx)


def tgv_get_timing(ctx) -> dict:
    t = tgv_timing()
    _check(lib.tgv_get_timing(ctx, ctypes.byref(t)), ctx)
    return {k: getattr(t, k) for k, _ in tgv_timing._fields_}


def tgv_info(ctx) -> dict:
    t = tgv_info_t()
    _check(lib.tgv_info(ctx, ctypes.byref(t)), ctx)
    return {k: getattr(t, k) for k, _ in tgv_info_t._fields_}


def tgv_destroy(ctx):
    lib.tgv_destroy(ctx)


def _camera_args(cams, depths):
    """ctypes camera table and depth-map pointers (the arrays are returned to keep them alive)."""
    arr = (tgv_camera * max(1, len(cams)))()
    for i, c in enumerate(cams):
        arr[i].origin[:] = [float(x) for x in c["origin"]]
        arr[i].rot[:] = [float(x) for x in np.asarray(c["rot"], dtype=np.float64).reshape(-1)]
        arr[i].fx, arr[i].fy, arr[i].cx, arr[i].cy = c["fx"], c["fy"], c["cx"], c["cy"]
        arr[i].width, arr[i].height, arr[i].vote_weight = c["width"], c["height"], c.get("vote_weight", 1)
    ds = [np.ascontiguousarray(d, dtype=np.float32) for d in depths]
    ptrs = (ctypes.c_void_p * max(1, len(ds)))(*[d.ctypes.data for d in ds])
    return arr, ptrs, ds


def tgv_vote_depth_maps(ctx, cams, depths, grid_origin=(0.0, 0.0, 0.0), voxel_size=1.0, voxel_radius=0.5):
    """cams: dicts (origin, rot 3x3 world<-camera, fx, fy, cx, cy, width, height, vote_weight);
    depths: float32 [h, w] host arrays (NaN = no depth)."""
    arr, ptrs, ds = _camera_args(cams, depths)
    o = np.asarray(grid_origin, dtype=np.float64)
    _check(lib.tgv_vote_depth_maps(ctx, arr, len(cams), ptrs, o.ctypes.data, float(voxel_size), float(voxel_radius)),
           ctx)


def tgv_read_counts(ctx, out):
    p, n = _host_ptr(out, np.uint32)
    _check(lib.tgv_read_counts(ctx, p, n), ctx)
    return out


def tgv_restrict_from(coarse, fine):
    _check(lib.tgv_restrict_from(coarse, fine), coarse)


def tgv_prolong_from(fine, coarse):
    _check(lib.tgv_prolong_from(fine, coarse), fine)


def tgv_create_leaf(shape, z_begin, z_end, centers, lam, alpha0, alpha1, tau, sigma, device=0):
    nx, ny, nz = shape
    L = tgv_layout(nx, ny, nz, z_begin, z_end, (ctypes.c_int32 * 3)(0, 0, 0))
    P, keep = _params(centers, lam, alpha0, alpha1, tau, sigma)
    out = ctypes.c_void_p()
    _check(lib.tgv_create_leaf(ctypes.byref(L), ctypes.byref(P), device, ctypes.byref(out)))
    return out


def tgv_set_border(ctx, side: int, u=None, v=None, p=None, q=None):
    ptr = [None if a is None else _host_ptr(a, np.float32)[0] for a in (u, v, p, q)]
    _check(lib.tgv_set_border(ctx, int(side), *ptr), ctx)


def tgv_peer_export(ctx) -> bytes:
    buf = ctypes.create_string_buffer(192)
    _check(lib.tgv_peer_export(ctx, buf), ctx)
    return buf.raw


def tgv_peer_import(ctx, side: int, rec: bytes):
    if len(rec) != 192:
        raise ValueError(f"peer record must be 192 bytes, got {len(rec)}")
    _check(lib.tgv_peer_import(ctx, int(side), rec), ctx)


def tgv_leaf_rebind(ctx, z_begin: int, z_end: int):
    _check(lib.tgv_leaf_rebind(ctx, int(z_begin), int(z_end)), ctx)


def tgv_load_histograms_coarsened(ctx, fine_counts, fine_shape, factor: int):
    """fine_counts: C-contiguous uint8 / uint16 / uint32 numpy array."""
    a = fine_counts
    if not isinstance(a, np.ndarray) or a.dtype not in (np.uint8, np.uint16, np.uint32):
        raise TypeError("fine_counts must be a uint8 / uint16 / uint32 numpy array")
    if not a.flags.c_contiguous:
        raise ValueError("fine_counts must be C-contiguous")
    nxf, nyf, nzf = fine_shape
    _check(lib.tgv_load_histograms_coarsened(ctx, a.ctypes.data, a.dtype.itemsize, a.size, nxf, nyf, nzf,
                                             int(factor)), ctx)


def tgv_prolong_slab(ctx, u_c, v_c, cz0: int):
    """u_c float32 [cnz, cny, cnx], v_c float32 [3, cnz, cny, cnx]: coarse planes [cz0, cz0 + cnz)."""
    pu, nu = _host_ptr(u_c, np.float32)
    pv, nv = _host_ptr(v_c, np.float32)
    cnz, cny, cnx = u_c.shape
    if nv != 3 * nu:
        raise ValueError(f"v_c must hold 3 x {nu} floats, got {nv}")
    _check(lib.tgv_prolong_slab(ctx, pu, pv, cnx, cny, int(cz0), cnz), ctx)


def _params(centers, lam, alpha0, alpha1, tau, sigma):
    c = (ctypes.c_float * len(centers))(*[float(x) for x in centers])
    return tgv_params(len(centers), ctypes.cast(c, ctypes.POINTER(ctypes.c_float)), lam, alpha0, alpha1, tau,
                      sigma), c


def tgv_create_group(shape, cuts, centers, lam, alpha0, alpha1, tau, sigma, devices):
    nx, ny, nz = shape
    n = len(cuts) - 1
    L = (tgv_layout * n)(*[tgv_layout(nx, ny, nz, cuts[r], cuts[r + 1], (ctypes.c_int32 * 3)(0, 0, 0))
                           for r in range(n)])
    P, keep = _params(centers, lam, alpha0, alpha1, tau, sigma)
    dev = (ctypes.c_int * n)(*devices)
    out = (ctypes.c_void_p * n)()
    _check(lib.tgv_create_group(L, ctypes.byref(P), n, dev, out))
    return [ctypes.c_void_p(out[r]) for r in range(n)]


def _ctx_array(ctxs):
    return (ctypes.c_void_p * len(ctxs))(*[c.value for c in ctxs])


def tgv_group_iterate(ctxs, n_iter: int):
    _check(lib.tgv_group_iterate(_ctx_array(ctxs), len(ctxs), int(n_iter)), ctxs[0])


def tgv_group_energy(ctxs) -> np.ndarray:
    out = np.zeros(6, dtype=np.float64)
    _check(lib.tgv_group_energy(_ctx_array(ctxs), len(ctxs), out.ctypes.data), ctxs[0])
    return out


# ---- multi-rank bootstrap -------------------------------------------------------------
def broadcast_unique_id(device=0):
    """Rank 0's NCCL unique id (tgv_get_unique_id) on every rank of the default
    torch.distributed group; None for a single rank."""
    import torch
    import torch.distributed as dist
    if dist.get_world_size() == 1:
        return None
    dev = f"cuda:{device}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if dist.get_rank() == 0:
        t.copy_(torch.frombuffer(bytearray(tgv_get_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tobytes())


def slab(nz: int, rank: int, world: int):
    """z-slab [z0, z1) of `rank`: contiguous, in rank order, sizes differing by at most one."""
    base, rem = divmod(nz, world)
    z0 = rank * base + min(rank, rem)
    return z0, z0 + base + (1 if rank < rem else 0)


# ---- convenience wrappers ---------------------------------------------------------
class Group:
    """z-slabs [cuts[r], cuts[r+1]) of one grid in this process (tgv_create_group)."""

    def __init__(self, shape, cuts, centers, lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25, devices=None):
        self.shape, self.cuts = tuple(shape), list(cuts)
        n = len(cuts) - 1
        self.ctxs = tgv_create_group(shape, cuts, centers, lam, alpha0, alpha1, tau, sigma,
                                     devices if devices is not None else [0] * n)

    def set_model(self, model):
        for c in self.ctxs:
            tgv_set_model(c, {"tgv": MODEL_TGV, "tvl1": MODEL_TVL1}.get(model, model))
        return self

    def set_schedule(self, schedule):
        for c in self.ctxs:
            tgv_set_schedule(c, {"fused": SCHEDULE_FUSED, "split": SCHEDULE_SPLIT}.get(schedule, schedule))
        return self

    def load(self, counts):
        """counts: the WHOLE grid's uint32 [nz, ny, nx, nbins]; each member loads its slab."""
        for r, c in enumerate(self.ctxs):
            tgv_load_histograms(c, np.ascontiguousarray(counts[self.cuts[r]:self.cuts[r + 1]]))
        return self

    def iterate(self, n: int):
        tgv_group_iterate(self.ctxs, n)
        return self

    def read_u(self):
        nx, ny, _ = self.shape
        parts = []
        for r, c in enumerate(self.ctxs):
            out = np.empty((self.cuts[r + 1] - self.cuts[r], ny, nx), np.float32)
            parts.append(tgv_read_u(c, out))
        return np.concatenate(parts, axis=0)

    def get(self, name):
        nx, ny, _ = self.shape
        ids = FIELDS[name]
        parts = []
        for r, c in enumerate(self.ctxs):
            out = np.empty((len(ids), self.cuts[r + 1] - self.cuts[r], ny, nx), np.float32)
            for k, f in enumerate(ids):
                tgv_read_field(c, f, out[k])
            parts.append(out)
        res = np.concatenate(parts, axis=1)
        return res[0] if len(ids) == 1 else res

    def energy(self) -> dict:
        e = tgv_group_energy(self.ctxs)
        return {"E": e[0], "alpha1": e[1], "alpha0": e[2], "data": e[3], "gap": e[4], "vmax": e[5]}

    def close(self):
        for c in getattr(self, "ctxs", []):
            tgv_destroy(c)
        self.ctxs = []

    def __del__(self):
        self.close()


class Solver:
    """One context on one GPU owning z-slab [z_begin, z_end) of an (nx, ny, nz) grid.

    With ``nranks > 1`` pass ``uid`` (from rank 0's ``tgv_get_unique_id``), or
    call ``Solver.distributed(...)`` which broadcasts it with torch.distributed.
    """

    def __init__(self, shape, centers, lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25, z_begin=0,
                 z_end=None, rank=0, nranks=1, uid=None, device=0):
        self.shape = tuple(int(s) for s in shape)
        self.z_begin = int(z_begin)
        self.z_end = self.shape[2] if z_end is None else int(z_end)
        self.nbins = len(centers)
        self.ctx = tgv_create(self.shape, self.z_begin, self.z_end, centers, lam, alpha0, alpha1, tau, sigma, rank,
                              nranks, uid, device)

    @classmethod
    def leaf(cls, shape, centers, z_begin, z_end, lam=0.5, alpha0=2.0, alpha1=1.0, tau=0.25, sigma=0.25, device=0):
        """NEXT-3: a leaf over z-slab [z_begin, z_end) whose border planes are frozen (tgv_create_leaf)."""
        self = cls.__new__(cls)
        self.shape = tuple(int(s) for s in shape)
        self.z_begin, self.z_end, self.nbins = int(z_begin), int(z_end), len(centers)
        self.ctx = tgv_create_leaf(self.shape, self.z_begin, self.z_end, centers, lam, alpha0, alpha1, tau, sigma,
                                   device)
        return self

    @classmethod
    def distributed(cls, shape, centers, z_begin, z_end, device, **kw):
        """One rank of a z-slab decomposition: the NCCL unique id is broadcast with torch.distributed."""
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        uid = broadcast_unique_id(device)
        return cls(shape, centers, z_begin=z_begin, z_end=z_end, rank=rank, nranks=world, uid=uid, device=device, **kw)

    @property
    def local_shape(self):
        nx, ny, _ = self.shape
        return (self.z_end - self.z_begin, ny, nx)

    def load(self, counts):
        tgv_load_histograms(self.ctx, counts)
        return self

    def reset(self):
        tgv_reset(self.ctx)

    def iterate(self, n: int):
        tgv_iterate(self.ctx, n)
        return self

    def iterate_async(self, n: int):
        """Enqueue n iterations and return (tgv_iterate_async); sync() or any read waits."""
        tgv_iterate_async(self.ctx, n)
        return self

    def sync(self):
        tgv_sync(self.ctx)
        return self

    def read_u(self, out=None):
        out = np.empty(self.local_shape, np.float32) if out is None else out
        return tgv_read_u(self.ctx, out)

    def get(self, name: str) -> np.ndarray:
        ids = FIELDS[name]
        out = np.empty((len(ids),) + self.local_shape, np.float32)
        for k, f in enumerate(ids):
            tgv_read_field(self.ctx, f, out[k])
        return out[0] if len(ids) == 1 else out

    def get_into(self, name: str, out):
        """Like get(), into caller-provided float32 arrays (out[k] C-contiguous per component)."""
        ids = FIELDS[name]
        if len(ids) == 1:
            tgv_read_field(self.ctx, ids[0], out)
        else:
            for k, f in enumerate(ids):
                tgv_read_field(self.ctx, f, out[k])
        return out

    def set(self, name: str, arr):
        ids = FIELDS[name]
        arr = np.ascontiguousarray(arr, dtype=np.float32).reshape((len(ids),) + self.local_shape)
        for k, f in enumerate(ids):
            tgv_write_field(self.ctx, f, np.ascontiguousarray(arr[k]))

    def energy(self) -> dict:
        e = tgv_energy(self.ctx)
        return {"E": e[0], "alpha1": e[1], "alpha0": e[2], "data": e[3], "gap": e[4], "vmax": e[5]}

    def set_schedule(self, schedule):
        """'fused' (default), 'split', or a TGV_SCHEDULE_* value."""
        tgv_set_schedule(self.ctx, {"fused": SCHEDULE_FUSED, "split": SCHEDULE_SPLIT}.get(schedule, schedule))
        return self

    def vote(self, cams, depths, grid_origin=(0.0, 0.0, 0.0), voxel_size=1.0, voxel_radius=0.5):
        """NEXT-2: histograms of this slab from depth maps by Alg. 1 on the GPU; state reset."""
        tgv_vote_depth_maps(self.ctx, cams, depths, grid_origin, voxel_size, voxel_radius)
        return self

    def read_counts(self):
        nz, ny, nx = self.local_shape
        return tgv_read_counts(self.ctx, np.empty((nz, ny, nx, self.nbins), np.uint32))

    def restrict_from(self, fine: "Solver"):
        """NEXT-1: this coarse solver's histograms = 2x2x2 sums of `fine`'s; state reset."""
        tgv_restrict_from(self.ctx, fine.ctx)
        return self

    def prolong_from(self, coarse: "Solver"):
        """NEXT-1: restart this solver from `coarse`'s solution (u, v / 2; duals zero)."""
        tgv_prolong_from(self.ctx, coarse.ctx)
        return self

    def set_border(self, side: int, u=None, v=None, p=None, q=None):
        """NEXT-3: frozen values of the plane below (side 0) / above (side 1) a leaf."""
        f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)
        tgv_set_border(self.ctx, side, f(u), f(v), f(p), f(q))
        return self

    def rebind(self, z_begin: int, z_end: int):
        """NEXT-3: move this leaf to slab [z_begin, z_end) (same plane count), keeping its memory."""
        tgv_leaf_rebind(self.ctx, z_begin, z_end)
        self.z_begin, self.z_end = int(z_begin), int(z_end)
        return self

    def load_coarsened(self, fine_counts, fine_shape, factor: int):
        """NEXT-1/3: histograms = sums of factor^3 fine voxels; fine_counts covers this slab's fine planes."""
        a = np.asarray(fine_counts)
        if a.dtype not in (np.uint8, np.uint16, np.uint32):
            a = a.astype(np.uint32)
        tgv_load_histograms_coarsened(self.ctx, np.ascontiguousarray(a), fine_shape, factor)
        return self

    def prolong_slab(self, u_c, v_c, cz0: int):
        """NEXT-1/3: restart from host coarse u / v planes [cz0, cz0 + len(u_c)) (borders of a leaf too)."""
        tgv_prolong_slab(self.ctx, np.ascontiguousarray(u_c, dtype=np.float32),
                         np.ascontiguousarray(v_c, dtype=np.float32), cz0)
        return self

    def set_model(self, model):
        """'tgv' (default) or 'tvl1' (NEXT-4, Eq. 1); a loaded solver restarts."""
        tgv_set_model(self.ctx, {"tgv": MODEL_TGV, "tvl1": MODEL_TVL1}.get(model, model))
        return self

    def set_timing(self, on: bool):
        tgv_set_timing(self.ctx, on)

    def timing(self) -> dict:
        return tgv_get_timing(self.ctx)

    def info(self) -> dict:
        return tgv_info(self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            tgv_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()
