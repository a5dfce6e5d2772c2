"""Seeded synthetic inputs (the reference's portable generator, prng.py:45-67).

``random_interior(nx, ny, seed)`` yields the same bits as the reference's
counter-mode splitmix64 fill; ``fill_random_device`` produces them directly
in HBM through the native kernel (dtb_fill_random_*), so 32768^2 inputs need
no host fill or H2D copy.
"""

from __future__ import annotations

import ctypes

import numpy as np

__all__ = ["splitmix64", "random_doubles", "random_interior", "Xoshiro256StarStar",
           "fill_random_device"]

_GOLDEN = np.uint64(0x9E3779B97F4B7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, n: int) -> np.ndarray:
    if n < 0:
        raise ValueError("n must be non-negative")
    z = np.uint64(seed & (2 ** 64 - 1)) + np.arange(1, n + 1, dtype=np.uint64) * _GOLDEN
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def random_doubles(seed: int, n: int) -> np.ndarray:
    return (splitmix64(seed, n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def random_interior(nx: int, ny: int, seed: int) -> np.ndarray:
    return random_doubles(seed, nx * ny).reshape(ny, nx)


class Xoshiro256StarStar:
    """Sequential xoshiro256** stream whose four state words are the first four
    splitmix64 outputs of ``seed`` (prng.py:74-111); the reference's tests and
    acceptance batch draw their configurations from it."""

    _M = (1 << 64) - 1

    def __init__(self, seed: int):
        self._s = [int(v) for v in splitmix64(seed, 4)]

    @classmethod
    def _rotl(cls, x: int, k: int) -> int:
        return ((x << k) | (x >> (64 - k))) & cls._M

    def next_u64(self) -> int:
        a, b, c, d = self._s
        out = (self._rotl((b * 5) & self._M, 7) * 9) & self._M
        t = (b << 17) & self._M
        c ^= a
        d ^= b
        b ^= c
        a ^= d
        self._s = [a, b, c ^ t, self._rotl(d, 45)]
        return out

    def random(self) -> float:
        """Uniform double in [0, 1)."""
        return (self.next_u64() >> 11) * (2.0 ** -53)

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.random()

    def randint(self, lo: int, hi: int) -> int:
        """Uniform integer in [lo, hi] (inclusive)."""
        if hi < lo:
            raise ValueError("empty range")
        return lo + self.next_u64() % (hi - lo + 1)

    def choice(self, seq):
        return seq[self.randint(0, len(seq) - 1)]


def _check_fill_buffer(buf, nx: int, ny: int, rows: int, dtypes):
    import torch
    if not isinstance(buf, torch.Tensor) or not buf.is_cuda:
        raise TypeError("expected a CUDA tensor")
    if buf.dtype not in dtypes:
        raise ValueError(f"buffer dtype must be one of {[str(d) for d in dtypes]}, got {buf.dtype}")
    if buf.dim() != 2 or buf.stride(1) != 1 or buf.shape[0] < rows or buf.shape[1] < nx + 2:
        raise ValueError(f"expected a row-major ({rows}, >= {nx + 2}) buffer, got "
                         f"{tuple(buf.shape)} with strides {buf.stride()}")


def fill_random_device(buf, nx: int, ny: int, seed: int, ghost: float = 0.0, stream=None):
    """Fill a padded (ny+2, pitch) CUDA tensor like grid_new(nx, ny, random_interior(...), ghost)."""
    import torch
    from . import _native
    _check_fill_buffer(buf, nx, ny, ny + 2, (torch.float64, torch.float32))
    with torch.cuda.device(buf.device):
        if stream is None:
            stream = torch.cuda.current_stream(buf.device).cuda_stream
        fn = _native.lib().dtb_fill_random_f64 if buf.dtype == torch.float64 else \
            _native.lib().dtb_fill_random_f32
        rc = fn(buf.data_ptr(), nx, ny, buf.stride(0), seed & (2 ** 64 - 1), float(ghost),
                ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(_native.last_error())


def fill_random_rows_device(buf, nx: int, ny: int, seed: int, row0: int, ghost: float = 0.0,
                            stream=None):
    """Rows [row0, row0 + buf.shape[0]) of the padded fp64 random grid into ``buf``."""
    import torch
    from . import _native
    _check_fill_buffer(buf, nx, ny, 0, (torch.float64,))
    with torch.cuda.device(buf.device):
        if stream is None:
            stream = torch.cuda.current_stream(buf.device).cuda_stream
        rc = _native.lib().dtb_fill_random_rows_f64(buf.data_ptr(), nx, ny, buf.stride(0),
                                                     seed & (2 ** 64 - 1), float(ghost), row0,
                                                     buf.shape[0], ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(_native.last_error())
