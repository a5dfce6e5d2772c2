"""The reference's one-step micro-kernel entry (`dtb.kernel`, kernel.py:44-144)
on the B200.

`j2d5pt_update(win_in, win_out, weights, cols, cfg)` applies one weighted
5-point update over `cols` of two windows, with the reference's contract:
same coordinate frame for both windows, reads `cols` dilated by one cell,
writes `cols` exactly, IndexError for a region outside a window or a stencil
reach not backed by the input buffer, ValueError when input and output alias
over the update region, zero-area `cols` a no-op (kernel.py:82-127).

The update itself runs on the GPU: the input patch (cols dilated by one) is a
padded grid whose ring is the frozen boundary, so one B200 solve step of it
(`dtb_j2d5pt_f64`, include/dtb_b200.h) is exactly the W,E,S,C,N update of
kernel.py:137-144; its interior is written into `win_out`. `cfg.ilp` cannot
change bits (test_kernel.py:69-75) and is only validated.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .engine import KernelConfig, _solve_host
from .grid import Rect, StencilWeights

__all__ = ["KernelConfig", "Window", "j2d5pt_update"]


@dataclass
class Window:
    """A width x height view into a 2D float64 buffer: window (x, y) is
    ``buf[y0 + y, x0 + x]`` (kernel.py:44-80)."""

    buf: np.ndarray
    x0: int
    y0: int
    width: int
    height: int

    def __post_init__(self):
        if self.buf.ndim != 2 or self.buf.dtype != np.float64:
            raise ValueError("window buffer must be a 2D float64 array")
        if self.width < 0 or self.height < 0:
            raise ValueError("window dims must be non-negative")

    @property
    def stride(self) -> int:
        """Row pitch of the backing buffer, in cells."""
        return self.buf.shape[1]

    @property
    def base(self) -> int:
        """Flat offset of window cell (0, 0) in the backing buffer."""
        return self.y0 * self.stride + self.x0

    @classmethod
    def over_interior(cls, grid_data: np.ndarray) -> "Window":
        """Window whose (0, 0) is interior cell (0, 0) of a padded grid buffer."""
        rows, cols = grid_data.shape
        return cls(grid_data, 1, 1, cols - 2, rows - 2)


def _check_region(win: Window, cols: Rect, reach: int, what: str) -> None:
    if cols.x0 < 0 or cols.y0 < 0 or cols.x1 > win.width or cols.y1 > win.height:
        raise IndexError(f"update region {cols} outside {what} window {win.width}x{win.height}")
    rows_buf, cols_buf = win.buf.shape
    if (win.x0 + cols.x0 - reach < 0 or win.x0 + cols.x1 + reach > cols_buf
            or win.y0 + cols.y0 - reach < 0 or win.y0 + cols.y1 + reach > rows_buf):
        raise IndexError(f"{what} window too small for stencil reach at {cols}")


def j2d5pt_update(win_in: Window, win_out: Window, weights: StencilWeights, cols: Rect,
                  cfg: KernelConfig = KernelConfig()) -> None:
    """One W,E,S,C,N update of ``cols`` from ``win_in`` into ``win_out`` on the
    GPU (kernel.py:94-144); bitwise equal to the reference for any ``cfg``."""
    if cfg is not None and cfg.ilp < 1:
        raise ValueError(f"ilp must be at least 1, got {cfg.ilp}")
    if cols.is_empty:
        return
    _check_region(win_in, cols, 1, "input")
    _check_region(win_out, cols, 0, "output")
    bi, bo = win_in.buf, win_out.buf
    ix, iy = win_in.x0 + cols.x0, win_in.y0 + cols.y0
    ox, oy = win_out.x0 + cols.x0, win_out.y0 + cols.y0
    cw, ch = cols.width, cols.height
    patch_in = bi[iy - 1:iy + ch + 1, ix - 1:ix + cw + 1]
    target = bo[oy:oy + ch, ox:ox + cw]
    if bi is bo:
        if not (ox + cw <= ix - 1 or ix + cw + 1 <= ox or oy + ch <= iy - 1 or iy + ch + 1 <= oy):
            raise ValueError("input and output windows alias over the update region")
    elif np.shares_memory(patch_in, target):
        raise ValueError("input and output windows alias over the update region")
    out, _ = _solve_host(np.ascontiguousarray(patch_in), cw, ch, weights, 1, 1, None, 1, 0,
                         np.float64)
    target[...] = out[1:-1, 1:-1]
