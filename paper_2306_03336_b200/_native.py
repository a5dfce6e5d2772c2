"""ctypes binding of the C ABI in include/dtb_b200.h (libdtb_b200.so).

The library is built in-tree by :func:`paper_2306_03336_b200.build.build_native`
(``__graft_entry__.build()``). There is no fallback: if the shared object is
missing or CUDA is unusable every solve raises, it never drops to a CPU path.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_uint, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DTB_LIB") or os.path.join(_HERE, "libdtb_b200.so")  # DTB_LIB: A/B builds

DTB_OK = 0
DTB_EINVAL = 1
DTB_ERANGE = 2
DTB_EINFEASIBLE = 3
DTB_ECUDA = 4
DTB_ECAPACITY = 5

FLAG_POISON = 1
FLAG_FORCE_STREAM = 2
FLAG_FORCE_NAIVE = 4
FLAG_FORCE_DEPTH = 8
FLAG_TRACE = 16
FLAG_FORCE_PIPE = 32
FLAG_FORCE_RESIDENT = 64
FLAG_SLAB_COPY = 128
FLAG_SLAB_FUSED = 256
FLAG_COUNT = 512


class DtbRect(ctypes.Structure):
    _fields_ = [("x0", c_int64), ("y0", c_int64), ("width", c_int64), ("height", c_int64)]


class DtbReport(ctypes.Structure):
    _fields_ = [
        ("global_load_cells", c_int64),
        ("global_store_cells", c_int64),
        ("halo_exchanged_cells", c_int64),
        ("redundant_compute_cells", c_int64),
        ("useful_compute_cells", c_int64),
        ("scratchpad_peak_bytes", c_int64),
        ("elem_bytes", c_int64),
    ]


class DtbPlanInfo(ctypes.Structure):
    _fields_ = [
        ("mode", c_int32),
        ("elem_bytes", c_int32),
        ("lane_elems", c_int32),
        ("warps", c_int32),
        ("halo", c_int32),
        ("tiles_x", c_int32),
        ("tiles_y", c_int32),
        ("ctas", c_int32),
        ("ctas_per_sm", c_int32),
        ("dyn", c_int32),
        ("smem_bytes", c_int64),
        ("tile_w", c_int64),
        ("tile_h", c_int64),
        ("load_w", c_int64),
        ("load_h", c_int64),
        ("computed_cells_per_step", c_int64),
        ("est_cells_per_clk", c_double),
    ]


class DtbHaloMirror(ctypes.Structure):
    _fields_ = [("peer", c_void_p * 2), ("r0", c_int64 * 2), ("r1", c_int64 * 2),
                ("p0", c_int64 * 2), ("sw0", c_int64), ("sw1", c_int64)]


IpcHandle = ctypes.c_uint8 * 64


# every symbol include/dtb_b200.h declares, with its ctypes signature
_SIGNATURES = {
    "dtb_j2d5pt_f64": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, POINTER(c_double),
                               c_int64, c_int64, POINTER(DtbRect), c_int, c_int, c_uint,
                               POINTER(DtbReport)]),
    "dtb_j2d5pt_f32": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, POINTER(c_float),
                               c_int64, c_int64, POINTER(DtbRect), c_int, c_int, c_uint,
                               POINTER(DtbReport)]),
    "dtb_j2d5pt_f64_dev": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                   POINTER(c_double), c_int64, c_int64, POINTER(DtbRect), c_uint,
                                   c_void_p, POINTER(DtbReport)]),
    "dtb_j2d5pt_f32_dev": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                   POINTER(c_float), c_int64, c_int64, POINTER(DtbRect), c_uint,
                                   c_void_p, POINTER(DtbReport)]),
    "dtb_plan": (c_int, [c_int64, c_int64, c_int32, c_int64, c_int64, c_uint,
                         POINTER(DtbPlanInfo)]),
    "dtb_last_launch_count": (c_int64, []),
    "dtb_last_min_required_bytes": (c_int64, []),
    "dtb_last_trace": (c_int64, [POINTER(c_int64), c_int64]),
    "dtb_device_info": (c_int, [POINTER(c_int32), POINTER(c_int64), POINTER(c_int64),
                                POINTER(c_int32), POINTER(c_int32)]),
    "dtb_fill_random_f64": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_uint64, c_double,
                                    c_void_p]),
    "dtb_fill_random_f32": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_uint64, c_double,
                                    c_void_p]),
    "dtb_fill_random_rows_f64": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_uint64, c_double,
                                         c_int64, c_int64, c_void_p]),
    "dtb_last_error": (c_char_p, []),
    "dtb_j2d5pt_f64_dev_mirror": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                          POINTER(c_double), c_int64, POINTER(DtbHaloMirror),
                                          c_void_p, POINTER(DtbReport)]),
    "dtb_j2d5pt_f32_dev_mirror": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                          POINTER(c_float), c_int64, POINTER(DtbHaloMirror),
                                          c_void_p, POINTER(DtbReport)]),
    "dtb_ipc_malloc": (c_int, [c_int64, POINTER(c_void_p), IpcHandle]),
    "dtb_ipc_free": (c_int, [c_void_p]),
    "dtb_ipc_open": (c_int, [IpcHandle, POINTER(c_void_p)]),
    "dtb_ipc_close": (c_int, [c_void_p]),
    "dtb_ipc_event_create": (c_int, [POINTER(c_void_p), IpcHandle]),
    "dtb_ipc_event_open": (c_int, [IpcHandle, POINTER(c_void_p)]),
    "dtb_event_destroy": (c_int, [c_void_p]),
    "dtb_event_record": (c_int, [c_void_p, c_void_p]),
    "dtb_stream_wait_event": (c_int, [c_void_p, c_void_p]),
    "dtb_debug_pipe_probe": (c_int, [POINTER(c_uint64)]),
}

_lib = None


class NativeLibraryError(RuntimeError):
    """libdtb_b200.so is missing or failed to load (no CPU fallback exists)."""


def lib():
    """Load (once) and return the native library; raise if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not built; run __graft_entry__.build() "
                "(the B200 path has no CPU fallback)")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().dtb_last_error()
    return msg.decode() if msg else ""
