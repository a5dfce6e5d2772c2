"""TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.

CPU restatements of the reference's two CPU code paths *with the reference's
own structure*, so that bench.py can time them on the GPU box (where
/root/reference does not exist) as the BASELINE.md §4 CPU legs:

* :func:`jacobi_rowwise` — jacobi_reference (oracle.py:19-34): per step, one
  j2d5pt_update over the whole interior at ilp=1, i.e. a Python loop over
  rows, each staging its three source rows (kernel.py:131-144). This is the
  per-row numpy dispatch that dominates the reference's wall time.
* :func:`run_dtb_port` — the reference's deep-temporal-blocking engine
  (engine.py:232-302): tiles of the reference plan processed one after the
  other; inside a tile every logical worker owns a column slice with
  double-buffered front/back arrays; each time block runs load -> T x
  (halo exchange, trapezoid update) -> store, every phase dispatched over a
  thread pool whose join is the modelled grid barrier (engine.py:91-111).

Both are bitwise equal to jacobi_c / jacobi_numpy (tests/test_oracle_pins.py);
the product path never imports them.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np


def update_rows(src: np.ndarray, dst: np.ndarray, y0: int, x0: int, h: int, w: int,
                weights) -> None:
    """dst[y0:y0+h, x0:x0+w] = one step of src (kernel.py:131-144, ilp=1):
    row by row, ((((W*w + E*e) + S*s) + C*c) + N*n) on a staged 3-row copy."""
    ww, we, ws, wc, wn = weights
    for r in range(y0, y0 + h):
        stage = src[r - 1:r + 2, x0:x0 + w].copy()
        dst[r, x0:x0 + w] = (src[r, x0 - 1:x0 - 1 + w] * ww + src[r, x0 + 1:x0 + 1 + w] * we
                             + stage[0] * ws + stage[1] * wc + stage[2] * wn)


def jacobi_rowwise(data: np.ndarray, weights, steps: int) -> np.ndarray:
    """jacobi_reference's structure (oracle.py:19-34) on a padded fp64 buffer."""
    a = np.array(data, dtype=np.float64, copy=True)
    b = a.copy()
    ny, nx = a.shape[0] - 2, a.shape[1] - 2
    wts = tuple(float(v) for v in weights)
    for _ in range(steps):
        update_rows(a, b, 1, 1, ny, nx, wts)
        a, b = b, a
    return a


class _Workers:
    """A tile's logical workers: column slices of its load region, each with
    front/back buffers (rows x (owned width + 2 halo columns))."""

    def __init__(self, tile, device, nx: int, ny: int):
        from paper_2306_03336_b200.planner import partition_subtiles
        load = tile.load_region
        self.tile = tile
        self.row0, self.lh = load.y0, load.height
        self.cols = [s.cols for s in partition_subtiles(tile, device)]
        self.front = [np.empty((self.lh, c.width + 2)) if c.width else None for c in self.cols]
        self.back = [np.empty((self.lh, c.width + 2)) if c.width else None for c in self.cols]
        self.n = len(self.cols)

    def load(self, i: int, g: np.ndarray) -> None:  # engine.py:152-162
        c = self.cols[i]
        if not c.width:
            return
        f = self.front[i]
        f[:, 1:c.width + 1] = g[self.row0 + 1:self.row0 + 1 + self.lh, c.x0 + 1:c.x0 + 1 + c.width]
        self.back[i][:] = f

    def exchange(self, i: int) -> None:  # engine.py:53-71: neighbours' edge columns
        c = self.cols[i]
        if not c.width:
            return
        if i > 0 and self.cols[i - 1].width:
            self.front[i][:, 0] = self.front[i - 1][:, self.cols[i - 1].width]
        if i + 1 < self.n and self.cols[i + 1].width:
            self.front[i][:, c.width + 1] = self.front[i + 1][:, 1]

    def compute(self, i: int, active, weights) -> None:  # engine.py:167-185
        c = self.cols[i]
        if not c.width:
            return
        sub = active.intersect(c)
        if not sub.is_empty:
            update_rows(self.front[i], self.back[i], sub.y0 - self.row0, sub.x0 - c.x0 + 1,
                        sub.height, sub.width, weights)
        self.front[i], self.back[i] = self.back[i], self.front[i]

    def store(self, i: int, g: np.ndarray) -> None:  # engine.py:187-200
        c, it = self.cols[i], self.tile.interior
        x0, x1 = max(it.x0, c.x0), min(it.x0 + it.width, c.x0 + c.width)
        if not c.width or x1 <= x0:
            return
        g[it.y0 + 1:it.y0 + it.height + 1, x0 + 1:x1 + 1] = \
            self.front[i][it.y0 - self.row0:it.y0 + it.height - self.row0,
                          x0 - c.x0 + 1:x1 - c.x0 + 1]


def run_dtb_port(data: np.ndarray, weights, total_steps: int, plan, threads: int = 1
                 ) -> np.ndarray:
    """The reference engine's schedule (engine.py:232-302) for a reference
    TilingPlan on a padded fp64 buffer; every phase goes over a thread pool
    (one thread: a plain loop), as _PhasePool does (engine.py:91-111)."""
    from paper_2306_03336_b200.grid import Rect
    from paper_2306_03336_b200.planner import tile_active_region
    if total_steps < 1 or total_steps % plan.t_depth:
        raise ValueError("total_steps must be a positive multiple of t_depth")
    valid = Rect(0, 0, plan.nx, plan.ny)
    wts = tuple(float(v) for v in weights)
    states = [_Workers(t, plan.device, plan.nx, plan.ny) for t in plan.tiles]
    bufs = [np.array(data, dtype=np.float64, copy=True), np.array(data, dtype=np.float64)]
    pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None

    def each(fn, n):
        if pool is None:
            for i in range(n):
                fn(i)
        else:
            list(pool.map(fn, range(n)))

    src = 0
    try:
        for _ in range(total_steps // plan.t_depth):
            g_in, g_out = bufs[src], bufs[1 - src]
            for ws in states:
                each(lambda i: ws.load(i, g_in), ws.n)
                for step in range(1, plan.t_depth + 1):
                    each(ws.exchange, ws.n)
                    active = tile_active_region(ws.tile, step, valid)
                    each(lambda i: ws.compute(i, active, wts), ws.n)
                each(lambda i: ws.store(i, g_out), ws.n)
            src = 1 - src
    finally:
        if pool is not None:
            pool.shutdown(wait=True)
    return bufs[src]
