"""Tile planning: the reference-compatible capacity plan and the B200 plan.

Two planners live here:

* :func:`plan_device_tiles` — the reference's capacity planner contract
  (planner.py:188-243): a :class:`TilingPlan` of row-major tiles whose
  T-dilated load regions fit a :class:`DeviceModel`'s per-worker scratchpad
  under the reference's double-buffer footprint (planner.py:151-169). Callers
  of ``run_dtb`` build and pass these; the B200 engine honours their
  ``t_depth`` / dims / capacity contract and reports their traffic model.
* :func:`plan_b200` — what actually runs: the native planner
  (csrc/dtb_plan.cpp) choosing a resident (whole grid in 148 SMs' smem) or
  streaming (h fused steps per HBM pass) schedule with a single-buffered,
  in-place tile footprint ``load_h * 32K * elem`` per CTA.
"""

from __future__ import annotations

import configparser
import ctypes
import os
from dataclasses import dataclass

from .grid import Rect

__all__ = ["DEFAULT_ELEM_BYTES", "DeviceModel", "DeviceTile", "SubTile", "TilingPlan",
           "InfeasiblePlanError", "scratchpad_footprint", "plan_device_tiles",
           "partition_widths", "partition_subtiles", "tile_active_region", "B200Plan",
           "plan_b200", "b200_device_model", "load_presets"]

DEFAULT_ELEM_BYTES = 8


class InfeasiblePlanError(Exception):
    """No tile fits the capacity model (planner.py:51-56)."""

    def __init__(self, message: str, min_required_bytes: int):
        super().__init__(message)
        self.min_required_bytes = min_required_bytes


@dataclass(frozen=True)
class DeviceModel:
    """(name, workers, scratchpad bytes per worker) (planner.py:59-75)."""

    name: str
    workers: int
    scratchpad_bytes_per_worker: int

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError(f"workers must be at least 1, got {self.workers}")
        if self.scratchpad_bytes_per_worker < 1:
            raise ValueError("scratchpad_bytes_per_worker must be positive")

    @property
    def total_bytes(self) -> int:
        return self.workers * self.scratchpad_bytes_per_worker


@dataclass(frozen=True)
class DeviceTile:
    interior: Rect
    halo: int
    load_region: Rect

    def to_dict(self) -> dict:
        return {"interior": self.interior.to_dict(), "halo": self.halo,
                "load_region": self.load_region.to_dict()}


@dataclass(frozen=True)
class SubTile:
    """One worker's column slice of a tile's load region (planner.py:91-112)."""

    owner: int
    cols: Rect
    stage_left: Rect | None
    stage_right: Rect | None

    def to_dict(self) -> dict:
        return {"owner": self.owner, "cols": self.cols.to_dict(),
                "stage_left": self.stage_left.to_dict() if self.stage_left else None,
                "stage_right": self.stage_right.to_dict() if self.stage_right else None}


@dataclass(frozen=True)
class TilingPlan:
    nx: int
    ny: int
    t_depth: int
    elem_bytes: int
    device: DeviceModel
    tiles: tuple
    footprint_bytes: int

    def to_dict(self) -> dict:
        return {"domain": {"nx": self.nx, "ny": self.ny}, "t_depth": self.t_depth,
                "elem_bytes": self.elem_bytes,
                "device": {"name": self.device.name, "workers": self.device.workers,
                           "scratchpad_bytes_per_worker":
                               self.device.scratchpad_bytes_per_worker},
                "footprint_bytes": self.footprint_bytes,
                "tiles": [dict(t.to_dict(), subtiles=[s.to_dict() for s in
                                                      partition_subtiles(t, self.device)])
                          for t in self.tiles]}


def scratchpad_footprint(tile_load_dims, t_depth: int, elem_bytes: int, workers: int) -> int:
    """Reference per-worker footprint 2*(ceil(w/workers)+2)*h*elem (planner.py:151-169)."""
    width, height = tile_load_dims
    if width < 0 or height < 0:
        raise ValueError(f"negative load dims {tile_load_dims}")
    if t_depth < 0 or elem_bytes < 0:
        raise ValueError("negative t_depth or elem_bytes")
    if workers < 1:
        raise ValueError(f"workers must be at least 1, got {workers}")
    return 2 * ((width + workers - 1) // workers + 2) * height * elem_bytes


def plan_device_tiles(domain, device: DeviceModel, t_depth: int,
                      elem_bytes: int = DEFAULT_ELEM_BYTES) -> TilingPlan:
    """Largest tile whose load region fits ``device`` (planner.py:188-243):
    full width if a 1-row band fits, else the widest 1-row tile; then the
    tallest height at that width; tiles emitted row-major, edges clipped."""
    nx, ny = domain
    if nx < 1 or ny < 1:
        raise ValueError(f"domain dims must be at least 1x1, got {nx}x{ny}")
    if t_depth < 1:
        raise ValueError(f"t_depth must be at least 1, got {t_depth}")
    if elem_bytes < 1:
        raise ValueError(f"elem_bytes must be at least 1, got {elem_bytes}")
    cap, h = device.scratchpad_bytes_per_worker, t_depth

    def need(tw: int, th: int) -> int:
        dims = (min(tw + 2 * h, nx + 2), min(th + 2 * h, ny + 2))
        return scratchpad_footprint(dims, h, elem_bytes, device.workers)

    if need(1, 1) > cap:
        raise InfeasiblePlanError(
            f"device {device.name!r} scratchpad {cap} B/worker cannot hold a 1x1 tile "
            f"interior at t_depth={t_depth}: needs at least {need(1, 1)} B/worker",
            need(1, 1))

    def largest(pred, hi: int) -> int:  # pred(1) holds; monotone
        lo = 1
        while lo < hi:
            mid = (lo + hi + 1) // 2
            lo, hi = (mid, hi) if pred(mid) else (lo, mid - 1)
        return lo

    tw = nx if need(nx, 1) <= cap else largest(lambda t: need(t, 1) <= cap, nx)
    th = largest(lambda t: need(tw, t) <= cap, ny)
    ghosted = Rect(-1, -1, nx + 2, ny + 2)
    tiles = []
    for y in range(0, ny, th):
        for x in range(0, nx, tw):
            it = Rect(x, y, min(tw, nx - x), min(th, ny - y))
            tiles.append(DeviceTile(it, h, it.dilate(h).intersect(ghosted)))
    fp = max(scratchpad_footprint((t.load_region.width, t.load_region.height), h,
                                  elem_bytes, device.workers) for t in tiles)
    return TilingPlan(nx, ny, t_depth, elem_bytes, device, tuple(tiles), fp)


def partition_widths(load_width: int, workers: int) -> list[int]:
    """Per-worker column widths, differing by <= 1, wider first (planner.py:246-269)."""
    base, rem = divmod(load_width, workers)
    return [base + (1 if i < rem else 0) for i in range(workers)]


def partition_subtiles(tile, device) -> list[SubTile]:
    load = tile.load_region
    out, x = [], load.x0
    for i, w in enumerate(partition_widths(load.width, device.workers)):
        left = Rect(x - 1, load.y0, 1, load.height) if w and x > load.x0 else None
        right = Rect(x + w, load.y0, 1, load.height) if w and x + w < load.x0 + load.width else None
        out.append(SubTile(i, Rect(x, load.y0, w, load.height), left, right))
        x += w
    return out


def tile_active_region(tile, step: int, valid) -> Rect:
    """Trapezoid of cells computable at superstep ``step`` (planner.py:272-286)."""
    if step < 1 or step > tile.halo:
        raise ValueError(f"step {step} outside 1..{tile.halo}")
    core = Rect(tile.interior.x0, tile.interior.y0, tile.interior.width,
                tile.interior.height).intersect(valid)
    if core.is_empty:
        return core
    return core.dilate(tile.halo - step).intersect(valid)


# --- the plan that actually runs on the B200 ---------------------------------

MODES = {0: "resident", 1: "streaming", 2: "naive", 3: "pipe"}


@dataclass(frozen=True)
class B200Plan:
    """Native plan summary (dtb_plan_info, include/dtb_b200.h)."""

    mode: str
    elem_bytes: int
    lane_elems: int
    warps: int
    halo: int
    tiles_x: int
    tiles_y: int
    ctas: int
    ctas_per_sm: int
    dyn: bool
    smem_bytes: int
    tile_w: int
    tile_h: int
    load_w: int
    load_h: int
    computed_cells_per_step: int
    est_cells_per_clk: float


def plan_b200(nx: int, ny: int, elem_bytes: int = 8, total_steps: int = 1, t_depth: int = 1,
              flags: int = 0) -> B200Plan:
    """Ask the native planner for the schedule it would run (no GPU needed:
    without one it plans for a 148-SM, 227 KB/CTA B200)."""
    from . import _native
    info = _native.DtbPlanInfo()
    rc = _native.lib().dtb_plan(nx, ny, elem_bytes, total_steps, t_depth, flags,
                                ctypes.byref(info))
    if rc != _native.DTB_OK:
        msg = _native.last_error()
        if rc == _native.DTB_EINFEASIBLE:
            raise InfeasiblePlanError(msg, int(_native.lib().dtb_last_min_required_bytes()))
        raise ValueError(msg)
    return B200Plan(MODES[info.mode], info.elem_bytes, info.lane_elems, info.warps, info.halo,
                    info.tiles_x, info.tiles_y, info.ctas, info.ctas_per_sm, bool(info.dyn),
                    info.smem_bytes, info.tile_w, info.tile_h, info.load_w, info.load_h,
                    info.computed_cells_per_step, info.est_cells_per_clk)


def b200_device_model(sms: int | None = None, smem: int | None = None) -> DeviceModel:
    """A reference-style DeviceModel for this device (148 x 232448)."""
    if sms is None or smem is None:
        from . import _native
        s, m, l2, ma, mi = (ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(),
                            ctypes.c_int32(), ctypes.c_int32())
        if _native.lib().dtb_device_info(ctypes.byref(s), ctypes.byref(m), ctypes.byref(l2),
                                         ctypes.byref(ma), ctypes.byref(mi)) == 0:
            sms, smem = sms or s.value, smem or m.value
        else:
            sms, smem = sms or 148, smem or 232448
    return DeviceModel("b200", sms, smem)


# --- device presets (planner.py:291-313 of the reference) -------------------
PRESETS_PATH = os.path.join(os.path.dirname(__file__), "presets.ini")


def load_presets(path=None) -> dict:
    """Device capacity presets from an INI file (sections with ``workers`` and
    ``scratchpad_bytes_per_worker``); the shipped file includes ``b200``."""
    parser = configparser.ConfigParser()
    with open(PRESETS_PATH if path is None else path) as fh:
        parser.read_file(fh)
    return {name: DeviceModel(name, parser[name].getint("workers"),
                              parser[name].getint("scratchpad_bytes_per_worker"))
            for name in parser.sections()}
