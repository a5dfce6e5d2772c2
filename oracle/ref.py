"""TEST INFRASTRUCTURE ONLY — see oracle/__init__.py."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_ORACLE_PATH = os.path.join(HERE, "libj2d5pt_oracle.so")


def jacobi_numpy(data: np.ndarray, weights, steps: int, dtype=np.float64) -> np.ndarray:
    """Whole-interior double-buffered sweep (oracle.py:19-34); each step is
    kernel.py:137-139 evaluated with ilp=1: (((W*w + E*e) + S*s) + C*c) + N*n.
    ``data`` is the padded (ny+2, nx+2) buffer; returns a new padded buffer."""
    if steps < 0:
        raise ValueError("steps must be non-negative")
    dt = np.dtype(dtype)
    a = np.array(data, dtype=dt, copy=True)
    b = a.copy()
    w, e, s, c, n = (dt.type(v) for v in weights)
    for _ in range(steps):
        mid = a[1:-1]
        b[1:-1, 1:-1] = (mid[:, :-2] * w + mid[:, 2:] * e + a[:-2, 1:-1] * s
                         + mid[:, 1:-1] * c + a[2:, 1:-1] * n)
        a, b = b, a
    return a


def build_c_oracle() -> str:
    """Compile oracle/j2d5pt_oracle.c (gcc, -ffp-contract=off) if stale."""
    src = os.path.join(HERE, "j2d5pt_oracle.c")
    if (not os.path.exists(C_ORACLE_PATH)
            or os.path.getmtime(C_ORACLE_PATH) < os.path.getmtime(src)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return C_ORACLE_PATH


_clib = None


def load_c_oracle():
    global _clib
    if _clib is None:
        if not os.path.exists(C_ORACLE_PATH):
            build_c_oracle()
        lib = ctypes.CDLL(C_ORACLE_PATH)
        for name, ct in (("oracle_j2d5pt_f64", ctypes.c_double), ("oracle_j2d5pt_f32", ctypes.c_float)):
            fn = getattr(lib, name)
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                           ctypes.c_int64, ctypes.POINTER(ct), ctypes.c_int64, ctypes.c_int]
        lib.oracle_random_interior.restype = None
        lib.oracle_random_interior.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                               ctypes.c_uint64]
        _clib = lib
    return _clib


def jacobi_c(data: np.ndarray, weights, steps: int, dtype=np.float64,
             threads: int | None = None) -> np.ndarray:
    """C restatement of the same sweep; bitwise equal to jacobi_numpy."""
    dt = np.dtype(dtype)
    src = np.ascontiguousarray(data, dtype=dt)
    out = np.empty_like(src)
    ny, nx = src.shape[0] - 2, src.shape[1] - 2
    lib = load_c_oracle()
    if dt == np.float64:
        w = (ctypes.c_double * 5)(*[float(v) for v in weights])
        fn = lib.oracle_j2d5pt_f64
    elif dt == np.float32:
        w = (ctypes.c_float * 5)(*[float(np.float32(v)) for v in weights])
        fn = lib.oracle_j2d5pt_f32
    else:
        raise ValueError(f"unsupported dtype {dt}")
    t = threads if threads is not None else (os.cpu_count() or 1)
    rc = fn(src.ctypes.data, out.ctypes.data, nx, ny, nx + 2, w, steps, t)
    if rc != 0:
        raise RuntimeError(f"oracle_j2d5pt failed rc={rc}")
    return out


def random_interior_c(nx: int, ny: int, seed: int) -> np.ndarray:
    out = np.empty((ny, nx), dtype=np.float64)
    load_c_oracle().oracle_random_interior(out.ctypes.data, nx, ny, seed & (2 ** 64 - 1))
    return out
