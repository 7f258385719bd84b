"""ctypes binding of the C-ABI (include/ctproj_b200.h) -> libctproj_b200.so.

This is the only way the package reaches the projector arithmetic: there is
no CPU fallback.  If the shared library is missing or fails to load,
``NativeLibraryError`` is raised at first use.

``Plan`` owns one ``ctp_plan`` (validated geometry + per-view footprint
coefficients resident on one device) and launches the SF kernels on the
current torch stream with workspace from torch's caching allocator, so calls
are stream-ordered and never synchronise the host.
"""

from __future__ import annotations

import ctypes
import os
import threading
from collections import OrderedDict

import numpy as np

from .errors import (
    CudaRuntimeError,
    InvalidValueError,
    NativeLibraryError,
    SpecMismatchError,
    UnsupportedGeometryError,
)
from .geometry import Geometry, VolumeSpec, kernel_args

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CTPROJ_LIB") or os.path.join(_HERE, "csrc", "libctproj_b200.so")
ABI_VERSION = 2

CTP_OK = 0
_STATUS_ERRORS = {
    1: InvalidValueError,
    2: UnsupportedGeometryError,
    3: SpecMismatchError,
    4: CudaRuntimeError,
    5: CudaRuntimeError,
    6: CudaRuntimeError,
}
FLAG_ACCUMULATE = 1
FLAG_TIME_KERNEL = 2

#: every symbol include/ctproj_b200.h declares (checked by tests)
EXPORTED_SYMBOLS = (
    "ctp_abi_version",
    "ctp_status_string",
    "ctp_last_error",
    "ctp_plan_create",
    "ctp_plan_destroy",
    "ctp_plan_shape",
    "ctp_sf_workspace_bytes",
    "ctp_sf_forward",
    "ctp_sf_back",
    "ctp_sf_fbp_back",
    "ctp_plan_kernel_time_ms",
    "ctp_sf_forward_oneshot",
    "ctp_sf_back_oneshot",
    "ctp_siddon_forward",
    "ctp_siddon_back",
    "ctp_dist_unique_id",
    "ctp_dist_create",
    "ctp_dist_destroy",
    "ctp_dist_slab",
    "ctp_sf_back_sharded_workspace_bytes",
    "ctp_sf_back_sharded",
)


class CtpGeom(ctypes.Structure):
    """struct ctp_geom (include/ctproj_b200.h)."""

    _fields_ = [
        ("kind", ctypes.c_int32),
        ("num_views", ctypes.c_int32),
        ("num_rows", ctypes.c_int32),
        ("num_cols", ctypes.c_int32),
        ("num_x", ctypes.c_int32),
        ("num_y", ctypes.c_int32),
        ("num_z", ctypes.c_int32),
        ("reserved0", ctypes.c_int32),
        ("pixel_width", ctypes.c_double),
        ("pixel_height", ctypes.c_double),
        ("center_row", ctypes.c_double),
        ("center_col", ctypes.c_double),
        ("sdd", ctypes.c_double),
        ("x0", ctypes.c_double),
        ("y0", ctypes.c_double),
        ("z0", ctypes.c_double),
        ("voxel_width", ctypes.c_double),
        ("voxel_height", ctypes.c_double),
        ("poses", ctypes.POINTER(ctypes.c_double)),
    ]


_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libctproj_b200.so and declare its signatures (raises loudly)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{path} not found; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " or `make -C paper_2307_05801_b200/csrc` (there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
        missing = [s for s in EXPORTED_SYMBOLS if not hasattr(lib, s)]
        if missing:
            raise NativeLibraryError(f"{path} lacks symbols {missing}")
        vp, sz, i32, u32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32
        lib.ctp_abi_version.restype = i32
        lib.ctp_status_string.argtypes = [i32]
        lib.ctp_status_string.restype = ctypes.c_char_p
        lib.ctp_last_error.argtypes = [ctypes.c_char_p, sz]
        lib.ctp_last_error.restype = i32
        lib.ctp_plan_create.argtypes = [ctypes.POINTER(CtpGeom), i32, ctypes.POINTER(vp)]
        lib.ctp_plan_create.restype = i32
        lib.ctp_plan_destroy.argtypes = [vp]
        lib.ctp_plan_destroy.restype = i32
        lib.ctp_plan_shape.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        lib.ctp_plan_shape.restype = i32
        lib.ctp_sf_workspace_bytes.argtypes = [vp, i32, i32]
        lib.ctp_sf_workspace_bytes.restype = sz
        for name in ("ctp_sf_forward", "ctp_sf_back"):
            fn = getattr(lib, name)
            fn.argtypes = [vp, vp, vp, i32, vp, sz, u32, vp]
            fn.restype = i32
        lib.ctp_sf_fbp_back.argtypes = [vp, vp, vp, i32, ctypes.c_double, vp, sz, u32, vp]
        lib.ctp_sf_fbp_back.restype = i32
        lib.ctp_plan_kernel_time_ms.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_float)]
        lib.ctp_plan_kernel_time_ms.restype = i32
        for name in ("ctp_sf_forward_oneshot", "ctp_sf_back_oneshot"):
            fn = getattr(lib, name)
            fn.argtypes = [ctypes.POINTER(CtpGeom), vp, vp, i32, vp]
            fn.restype = i32
        for name in ("ctp_siddon_forward", "ctp_siddon_back"):
            fn = getattr(lib, name)
            fn.argtypes = [vp, ctypes.c_double, vp, vp, i32, u32, vp]
            fn.restype = i32
        lib.ctp_dist_unique_id.argtypes = [ctypes.c_char_p, sz]
        lib.ctp_dist_unique_id.restype = i32
        lib.ctp_dist_create.argtypes = [ctypes.c_char_p, sz, i32, i32, i32, ctypes.POINTER(vp)]
        lib.ctp_dist_create.restype = i32
        lib.ctp_dist_destroy.argtypes = [vp]
        lib.ctp_dist_destroy.restype = i32
        lib.ctp_dist_slab.argtypes = [vp, vp, i32, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        lib.ctp_dist_slab.restype = i32
        lib.ctp_sf_back_sharded_workspace_bytes.argtypes = [vp, vp, i32]
        lib.ctp_sf_back_sharded_workspace_bytes.restype = sz
        lib.ctp_sf_back_sharded.argtypes = [vp, vp, vp, vp, i32, vp, sz, vp]
        lib.ctp_sf_back_sharded.restype = i32
        if lib.ctp_abi_version() != ABI_VERSION:
            raise NativeLibraryError(
                f"ABI version mismatch: library {lib.ctp_abi_version()} != binding {ABI_VERSION}")
        _lib = lib
        return lib


def _raise_status(lib, status: int, what: str):
    buf = ctypes.create_string_buffer(1024)
    lib.ctp_last_error(buf, len(buf))
    msg = buf.value.decode(errors="replace") or lib.ctp_status_string(status).decode()
    raise _STATUS_ERRORS.get(status, CudaRuntimeError)(f"{what}: {msg}")


def make_geom(g: Geometry, spec: VolumeSpec):
    """(CtpGeom, keep-alive pose array) for a geometry / grid pair."""
    a = kernel_args(g, spec)
    poses = np.ascontiguousarray(a.pop("poses").reshape(-1), dtype=np.float64)
    geom = CtpGeom(reserved0=0, poses=poses.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), **a)
    return geom, poses


class Plan:
    """A ctp_plan bound to one CUDA device."""

    def __init__(self, g: Geometry, spec: VolumeSpec, device_index: int):
        import torch

        self.lib = load_library()
        self.geometry = g
        self.spec = spec
        self.device = torch.device("cuda", device_index)
        geom, keep = make_geom(g, spec)
        handle = ctypes.c_void_p()
        st = self.lib.ctp_plan_create(ctypes.byref(geom), int(device_index), ctypes.byref(handle))
        del keep
        if st != CTP_OK:
            _raise_status(self.lib, st, "ctp_plan_create")
        self._h = handle
        self.vol_shape = spec.shape
        self.sino_shape = g.shape

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self.lib.ctp_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def workspace_bytes(self, direction: int, batch: int) -> int:
        return int(self.lib.ctp_sf_workspace_bytes(self._h, int(direction), int(batch)))

    def kernel_time_ms(self, direction: int) -> float:
        """Device time of the last timed projector kernel launch (CUDA events)."""
        ms = ctypes.c_float()
        st = self.lib.ctp_plan_kernel_time_ms(self._h, int(direction), ctypes.byref(ms))
        if st != CTP_OK:
            _raise_status(self.lib, st, "ctp_plan_kernel_time_ms")
        return float(ms.value)

    def _check_io(self, direction: int, inp, out):
        in_shape = self.vol_shape if direction == 0 else self.sino_shape
        out_shape = self.sino_shape if direction == 0 else self.vol_shape
        _check_device_tensor(inp, (None,) + tuple(in_shape), self.device, "input")
        _check_device_tensor(out, (int(inp.shape[0]),) + tuple(out_shape), self.device, "output")

    def _run(self, direction: int, inp, out, accumulate: bool, time_kernel: bool = False):
        import torch

        self._check_io(direction, inp, out)
        batch = int(inp.shape[0])
        nbytes = self.workspace_bytes(direction, batch)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        fn = self.lib.ctp_sf_forward if direction == 0 else self.lib.ctp_sf_back
        flags = (FLAG_ACCUMULATE if accumulate else 0) | (FLAG_TIME_KERNEL if time_kernel else 0)
        st = fn(self._h, inp.data_ptr(), out.data_ptr(), batch, ws.data_ptr(), nbytes, flags, stream)
        if st != CTP_OK:
            _raise_status(self.lib, st, "ctp_sf_forward" if direction == 0 else "ctp_sf_back")
        return out

    def _run_siddon(self, direction: int, inp, out, accumulate: bool, time_kernel: bool = False):
        import torch

        # kernel_geom's parallel-beam ray back-off (_common.py:21-24), same expression
        back = float(self.spec.circumscribed_radius() + self.spec.voxelWidth)
        self._check_io(direction, inp, out)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        fn = self.lib.ctp_siddon_forward if direction == 0 else self.lib.ctp_siddon_back
        flags = (FLAG_ACCUMULATE if accumulate else 0) | (FLAG_TIME_KERNEL if time_kernel else 0)
        st = fn(self._h, back, inp.data_ptr(), out.data_ptr(), int(inp.shape[0]), flags, stream)
        if st != CTP_OK:
            _raise_status(self.lib, st, "ctp_siddon_forward" if direction == 0 else "ctp_siddon_back")
        return out

    def siddon_forward(self, x, out=None, accumulate: bool = False, time_kernel: bool = False):
        """Siddon y = A x on device tensors (same layouts as ``forward``)."""
        import torch

        if out is None:
            out = torch.empty((x.shape[0],) + self.sino_shape, dtype=torch.float32, device=self.device)
        return self._run_siddon(0, x, out, accumulate, time_kernel)

    def siddon_back(self, y, out=None, accumulate: bool = False, time_kernel: bool = False):
        """Siddon x = A^T y on device tensors (same layouts as ``back``)."""
        import torch

        if out is None:
            out = torch.empty((y.shape[0],) + self.vol_shape, dtype=torch.float32, device=self.device)
        return self._run_siddon(1, y, out, accumulate, time_kernel)

    def forward(self, x, out=None, accumulate: bool = False, time_kernel: bool = False):
        """y[B, nv, nr, nc] = A x[B, nz, ny, nx]; device tensors, f32, contiguous."""
        import torch

        if out is None:
            out = torch.empty((x.shape[0],) + self.sino_shape, dtype=torch.float32, device=self.device)
        return self._run(0, x, out, accumulate, time_kernel)

    def back(self, y, out=None, accumulate: bool = False, time_kernel: bool = False):
        """x[B, nz, ny, nx] = A^T y[B, nv, nr, nc]; device tensors, f32, contiguous."""
        import torch

        if out is None:
            out = torch.empty((y.shape[0],) + self.vol_shape, dtype=torch.float32, device=self.device)
        return self._run(1, y, out, accumulate, time_kernel)


    def fbp_back(self, y, scale: float, out=None, time_kernel: bool = False):
        """x = A^T (ramp(y) * scale): the FBP input stage (Ram-Lak row filter,
        recon.py:39-61) fused with the back projection's layout change, then
        the SF back projection (ctp_sf_fbp_back); device tensors."""
        import torch

        if out is None:
            out = torch.empty((y.shape[0],) + self.vol_shape, dtype=torch.float32, device=self.device)
        self._check_io(1, y, out)
        batch = int(y.shape[0])
        nbytes = self.workspace_bytes(1, batch)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        flags = FLAG_TIME_KERNEL if time_kernel else 0
        st = self.lib.ctp_sf_fbp_back(self._h, y.data_ptr(), out.data_ptr(), batch, float(scale), ws.data_ptr(),
                                      nbytes, flags, stream)
        if st != CTP_OK:
            _raise_status(self.lib, st, "ctp_sf_fbp_back")
        return out


class Dist:
    """A ctp_dist: NCCL communicator of the view-sharded back projection
    (include/ctproj_b200.h, multi-GPU section).  ``unique_id`` (128 bytes) is
    made by ``Dist.make_id()`` on rank 0 and shared out of band."""

    ID_BYTES = 128

    @staticmethod
    def make_id() -> bytes:
        lib = load_library()
        buf = ctypes.create_string_buffer(Dist.ID_BYTES)
        st = lib.ctp_dist_unique_id(buf, Dist.ID_BYTES)
        if st != CTP_OK:
            _raise_status(lib, st, "ctp_dist_unique_id")
        return buf.raw

    def __init__(self, unique_id: bytes, nranks: int, rank: int, device_index: int):
        self.lib = load_library()
        if len(unique_id) != self.ID_BYTES:
            raise InvalidValueError("unique_id must be 128 bytes")
        h = ctypes.c_void_p()
        st = self.lib.ctp_dist_create(unique_id, self.ID_BYTES, int(nranks), int(rank), int(device_index),
                                      ctypes.byref(h))
        if st != CTP_OK:
            _raise_status(self.lib, st, "ctp_dist_create")
        self._h = h
        self.nranks, self.rank, self.device_index = int(nranks), int(rank), int(device_index)

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self.lib.ctp_dist_destroy(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def slab(self, plan: "Plan", rank: int | None = None):
        """(first slice, slice count) of ``rank``'s z-slab (default: this rank)."""
        z0, n = ctypes.c_int(), ctypes.c_int()
        st = self.lib.ctp_dist_slab(plan._h, self._h, self.rank if rank is None else int(rank),
                                    ctypes.byref(z0), ctypes.byref(n))
        if st != CTP_OK:
            _raise_status(self.lib, st, "ctp_dist_slab")
        return z0.value, n.value

    def back_sharded(self, plan: "Plan", y, out=None):
        """This rank's z-slab [B, S, ny, nx] of sum_ranks A_shard^T y_shard:
        back projection of ``y`` ([B, nv_r, nr, nc], this rank's views, on the
        plan's device) fused with per-z-chunk NCCL reductions to the slab
        owners, overlapped with the remaining back projection."""
        import torch

        _check_device_tensor(y, (None,) + plan.sino_shape, plan.device, "y")
        B = int(y.shape[0])
        _, S = self.slab(plan)
        spec = plan.spec
        if out is None:
            out = torch.empty((B, S, spec.numY, spec.numX), dtype=torch.float32, device=plan.device)
        _check_device_tensor(out, (B, S, spec.numY, spec.numX), plan.device, "out")
        nbytes = int(self.lib.ctp_sf_back_sharded_workspace_bytes(plan._h, self._h, B))
        ws = torch.empty(nbytes, dtype=torch.uint8, device=plan.device)
        stream = torch.cuda.current_stream(plan.device).cuda_stream
        st = self.lib.ctp_sf_back_sharded(plan._h, self._h, y.data_ptr(), out.data_ptr(), B, ws.data_ptr(),
                                          nbytes, stream)
        if st != CTP_OK:
            _raise_status(self.lib, st, "ctp_sf_back_sharded")
        return out


def _check_device_tensor(t, shape, device, what):
    """f32, contiguous, on ``device``, matching ``shape`` (None = any extent):
    anything else would be read out of bounds by the kernels."""
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidValueError(f"{what} must be a CUDA tensor")
    if t.dtype != torch.float32:
        raise InvalidValueError(f"{what} must be float32, got {t.dtype}")
    if not t.is_contiguous():
        raise InvalidValueError(f"{what} must be contiguous")
    if t.device != device:
        raise InvalidValueError(f"{what} is on {t.device}, the plan on {device}")
    if len(t.shape) != len(shape) or any(s is not None and int(a) != int(s) for a, s in zip(t.shape, shape)):
        raise SpecMismatchError(f"{what} has shape {tuple(t.shape)}, expected "
                                f"{tuple('B' if s is None else s for s in shape)}")


_plans: "OrderedDict[tuple, Plan]" = OrderedDict()
_plans_lock = threading.Lock()
_PLAN_CACHE_SIZE = 64  # z-slab streaming builds one plan per slab


def get_plan(g: Geometry, spec: VolumeSpec, device_index: int) -> Plan:
    """Cached plan per (geometry, grid, device)."""
    key = (g, spec, int(device_index))
    with _plans_lock:
        p = _plans.get(key)
        if p is not None:
            _plans.move_to_end(key)
            return p
    p = Plan(g, spec, device_index)
    with _plans_lock:
        _plans[key] = p
        while len(_plans) > _PLAN_CACHE_SIZE:
            _plans.popitem(last=False)
    return p
