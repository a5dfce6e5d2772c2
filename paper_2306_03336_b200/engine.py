"""The drop-in solver entry points (mirrors dtb.engine.run_dtb, engine.py:305-326,
and dtb.oracle.jacobi_reference, oracle.py:19-34), executed on the B200.

Every call crosses into libdtb_b200.so once (ctypes releases the GIL), which
copies the padded grid to the device, runs the resident or streaming sm_100a
kernel chosen by the native planner, and copies the result back. Results are
bitwise identical to the reference's jacobi_reference for any plan, worker
count, ILP or thread count — the contract of SPEC.md:312-314 — because every
cell update is the same FMA-free W,E,S,C,N expression. There is no CPU path:
a missing library or CUDA failure raises :class:`EngineError`.
"""

from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass

import numpy as np

from . import _native
from .grid import Grid2D, Rect, as_weights_tuple
from .metrics import TrafficReport, model_dtb_traffic
from .planner import InfeasiblePlanError, partition_widths, tile_active_region

__all__ = ["EngineError", "KernelConfig", "run_dtb", "run_dtb_b200", "run_dtb_trace", "j2d5pt",
           "j2d5pt_trace", "jacobi", "j2d5pt_device", "last_launch_count", "TileTrace",
           "TileBlockTrace"]


class EngineError(RuntimeError):
    """Runtime contract violation inside the engine (engine.py:49-50), incl. CUDA errors."""


@dataclass(frozen=True)
class KernelConfig:
    """Accepted for API parity (kernel.py:33-41); cannot change results."""

    ilp: int = 1

    def __post_init__(self):
        if self.ilp < 1:
            raise ValueError(f"ilp must be at least 1, got {self.ilp}")


_DTYPES = {np.dtype(np.float64): ("f64", ctypes.c_double, 8),
           np.dtype(np.float32): ("f32", ctypes.c_float, 4)}


def _raise(rc: int):
    msg = _native.last_error()
    if rc == _native.DTB_EINVAL:
        raise ValueError(msg)
    if rc == _native.DTB_ERANGE:
        raise IndexError(msg)
    if rc == _native.DTB_EINFEASIBLE:
        raise InfeasiblePlanError(msg, int(_native.lib().dtb_last_min_required_bytes()))
    raise EngineError(msg)


def _rect(valid) -> _native.DtbRect | None:
    if valid is None:
        return None
    return _native.DtbRect(int(valid.x0), int(valid.y0), int(valid.width), int(valid.height))


def _check_plan(grid, total_steps: int, plan, valid, elem_bytes: int):
    """The reference's argument contract (engine.py:236-251) and capacity
    guard (engine.py:141-145) for a caller-supplied TilingPlan."""
    if (grid.nx, grid.ny) != (plan.nx, plan.ny):
        raise ValueError(f"plan is for {plan.nx}x{plan.ny}, grid is {grid.nx}x{grid.ny}")
    if total_steps < 1 or total_steps % plan.t_depth:
        raise ValueError(f"total_steps {total_steps} is not a positive multiple of "
                         f"t_depth {plan.t_depth}")
    if plan.elem_bytes != elem_bytes:
        raise ValueError(f"plan.elem_bytes {plan.elem_bytes} does not match the "
                         f"{elem_bytes}-byte compute dtype")
    cap = plan.device.scratchpad_bytes_per_worker
    for tile in plan.tiles:
        lh = tile.load_region.height
        for w in partition_widths(tile.load_region.width, plan.device.workers):
            used = 2 * (w + 2) * lh * 8 if w else 0
            if used > cap:
                raise EngineError(f"worker buffer {used} B exceeds scratchpad capacity "
                                  f"{cap} B for tile {tile.interior}")


def _check_valid(nx: int, ny: int, valid):
    if valid is None:
        return
    if (valid.width == 0 or valid.height == 0 or valid.x0 < 0 or valid.y0 < 0
            or valid.x0 + valid.width > nx or valid.y0 + valid.height > ny):
        raise ValueError(f"valid region {valid} not within domain Rect(0, 0, {nx}, {ny})")


def _solve_host(data: np.ndarray, nx: int, ny: int, weights, steps: int, t_depth: int,
                valid, ilp: int, flags: int, dtype, n_gpus: int = 1
                ) -> tuple[np.ndarray, _native.DtbReport]:
    dt = np.dtype(dtype)
    if dt not in _DTYPES:
        raise ValueError(f"dtype must be float64 or float32, got {dt}")
    tag, ctype, _ = _DTYPES[dt]
    src = np.ascontiguousarray(data, dtype=dt)
    out = np.empty_like(src)
    w = (ctype * 5)(*[dt.type(v) for v in as_weights_tuple(weights)])
    rep = _native.DtbReport()
    vr = _rect(valid)
    fn = getattr(_native.lib(), f"dtb_j2d5pt_{tag}")
    rc = fn(src.ctypes.data, out.ctypes.data, nx, ny, nx + 2, w, steps, t_depth,
            ctypes.byref(vr) if vr is not None else None, ilp, n_gpus, flags, ctypes.byref(rep))
    if rc != _native.DTB_OK:
        _raise(rc)
    return out, rep


def _report(rep: _native.DtbReport, counted: bool = False) -> TrafficReport:
    return TrafficReport(rep.global_load_cells, rep.global_store_cells, rep.halo_exchanged_cells,
                         rep.redundant_compute_cells, rep.useful_compute_cells,
                         rep.scratchpad_peak_bytes, rep.elem_bytes,
                         source="b200 counted" if counted else "b200 model")


def run_dtb(grid, weights, total_steps: int, plan=None, cfg: KernelConfig = KernelConfig(), *,
            valid=None, threads: int | None = None, poison: bool = False,
            dtype=np.float64) -> tuple[Grid2D, TrafficReport]:
    """Advance ``grid`` by ``total_steps`` Jacobi steps on the B200 (engine.py:305-326).

    ``plan`` is a reference-style TilingPlan (its t_depth, dims and capacity
    contract are enforced and its traffic model is reported) or None (the
    native B200 planner alone decides; the report is the B200 schedule's).
    ``threads`` is accepted for API parity and ignored; ``poison`` runs the
    kernels' NaN-poison debug mode. ``dtype=np.float32`` rounds the grid and
    weights to fp32 once, computes in fp32 and widens the result exactly.
    The input grid is never modified; a new Grid2D is returned.
    """
    del threads
    elem = np.dtype(dtype).itemsize
    if plan is not None:
        _check_plan(grid, total_steps, plan, valid, elem)
        t_depth = plan.t_depth
    else:
        if total_steps < 1:
            raise ValueError(f"total_steps {total_steps} is not a positive multiple of t_depth 1")
        t_depth = 1
    _check_valid(grid.nx, grid.ny, valid)
    ilp = cfg.ilp if cfg is not None else 1
    flags = _native.FLAG_POISON if poison else 0
    out, rep = _solve_host(grid.data, grid.nx, grid.ny, weights, total_steps, t_depth, valid,
                           ilp, flags, dtype)
    result = Grid2D(grid.nx, grid.ny, out.astype(np.float64, copy=False))
    if plan is not None:
        # the reference plan's counters (the reconciliation contract), labelled;
        # the traffic of the B200 schedule that actually ran rides along
        model = model_dtb_traffic(plan, total_steps, valid)
        return result, dataclasses.replace(model, source="reference-plan model",
                                           b200=_report(rep))
    return result, _report(rep)


def run_dtb_b200(grid, weights, total_steps: int, *, valid=None, poison: bool = False,
                 dtype=np.float64, flags: int = 0, depth: int | None = None, n_gpus: int = 1,
                 count: bool = False) -> tuple[Grid2D, TrafficReport]:
    """Like run_dtb without a reference plan, returning the B200 schedule's own
    traffic (dtb_report). ``flags`` takes _native.FLAG_FORCE_* for tests;
    ``depth`` pins the temporal halo depth; ``n_gpus`` > 1 splits the grid
    into y-slabs over the visible GPUs inside the library (one process);
    ``count`` reports the traffic the kernels counted instead of the model."""
    _check_valid(grid.nx, grid.ny, valid)
    if depth is not None:
        flags |= _native.FLAG_FORCE_DEPTH
    if count:
        flags |= _native.FLAG_COUNT
    out, rep = _solve_host(grid.data, grid.nx, grid.ny, weights, total_steps,
                           depth if depth is not None else 1, valid, 1,
                           flags | (_native.FLAG_POISON if poison else 0), dtype, n_gpus)
    return (Grid2D(grid.nx, grid.ny, out.astype(np.float64, copy=False)),
            _report(rep, counted=count))


@dataclass
class TileBlockTrace:
    """One time block at the probed tile (engine.py:215-222): the load-region
    image after the load, one image per superstep, the stored interior."""

    load: np.ndarray
    steps: list
    store: np.ndarray


@dataclass
class TileTrace:
    """engine.py:225-229."""

    tile_index: int
    load_region: Rect
    blocks: list


def _superstep_image(base: np.ndarray, load: Rect, states: list, s: int, tile, valid: Rect,
                     poison: bool) -> np.ndarray:
    """The probed tile's assembled front buffer after superstep ``s`` of the
    reference's double-buffered schedule (engine.py:178-194): state ``s`` on
    the active trapezoid; outside it the buffer still holds the state its
    parity last received (s-2, s-4, ..., down to the loaded block start), or
    NaN on the valid cells in poison mode. ``states[t]`` is the padded grid
    after t steps of the block, computed on the B200."""
    img = base.copy()
    if poison:
        pv = load.intersect(valid)
        img[pv.y0 - load.y0:pv.y1 - load.y0, pv.x0 - load.x0:pv.x1 - load.x0] = np.nan
        ts = (s,)
    else:
        ts = range(2 if s % 2 == 0 else 1, s + 1, 2)
    for t in ts:
        a = tile_active_region(tile, t, valid)
        if a.is_empty:
            continue
        img[a.y0 - load.y0:a.y1 - load.y0, a.x0 - load.x0:a.x1 - load.x0] = \
            states[t][a.y0 + 1:a.y1 + 1, a.x0 + 1:a.x1 + 1]
    return img


def run_dtb_trace(grid, weights, total_steps: int, plan, cfg: KernelConfig = KernelConfig(), *,
                  probe: int, valid=None, threads: int | None = None,
                  poison: bool = False) -> tuple[Grid2D, TrafficReport, TileTrace]:
    """Like :func:`run_dtb` but record the probed tile's buffers
    (engine.py:329-345): per time block the load-region image after the load,
    one image per superstep and the stored interior slice.

    The states come from the B200: the solve advances one step per call so
    every intermediate grid exists, and the images are assembled from them
    with the reference schedule's buffer semantics (state s on the active
    trapezoid, the parity's older states on the rim). Debug path: one launch
    and one host round trip per step. Raises IndexError for a bad probe.
    """
    del threads
    _check_plan(grid, total_steps, plan, valid, 8)
    _check_valid(grid.nx, grid.ny, valid)
    if not 0 <= probe < len(plan.tiles):
        raise IndexError(f"probe tile {probe} out of range (plan has {len(plan.tiles)} tiles)")
    vrect = valid if valid is not None else Rect(0, 0, grid.nx, grid.ny)
    tile = plan.tiles[probe]
    load, it = tile.load_region, tile.interior
    ilp = cfg.ilp if cfg is not None else 1
    flags = _native.FLAG_POISON if poison else 0
    cur = np.array(grid.data, dtype=np.float64, copy=True)
    blocks = []
    for _ in range(total_steps // plan.t_depth):
        states = [cur]
        for _s in range(plan.t_depth):
            nxt, _rep = _solve_host(states[-1], grid.nx, grid.ny, weights, 1, 1, valid, ilp,
                                    flags, np.float64)
            states.append(nxt)
        base = cur[load.y0 + 1:load.y1 + 1, load.x0 + 1:load.x1 + 1].copy()
        steps = [_superstep_image(base, load, states, s, tile, vrect, poison)
                 for s in range(1, plan.t_depth + 1)]
        cur = states[-1]
        blocks.append(TileBlockTrace(base, steps,
                                     cur[it.y0 + 1:it.y1 + 1, it.x0 + 1:it.x1 + 1].copy()))
    model = model_dtb_traffic(plan, total_steps, valid)
    return (Grid2D(grid.nx, grid.ny, cur), dataclasses.replace(model, source="reference-plan model"),
            TileTrace(probe, load, blocks))


def j2d5pt_trace(grid, weights, steps: int, stride: int = 1, *, dtype=np.float64) -> list:
    """The B200 twin of jacobi_reference_trace (oracle.py:37-59): copies of the
    state at t = 0, stride, 2*stride, ... plus always the final step, each one
    B200 solve of ``stride`` steps from the previous snapshot (a solve of a+b
    steps equals a solve of a then b, bitwise)."""
    if steps < 0:
        raise ValueError(f"steps must be non-negative, got {steps}")
    if stride < 1:
        raise ValueError(f"stride must be at least 1, got {stride}")
    cur = np.array(grid.data, dtype=np.float64, copy=True)
    out = [Grid2D(grid.nx, grid.ny, cur.copy())]
    t = 0
    while t < steps:
        n = min(stride - t % stride, steps - t)
        nxt, _ = _solve_host(cur, grid.nx, grid.ny, weights, n, 1, None, 1, 0, dtype)
        cur = nxt.astype(np.float64, copy=False)
        t += n
        out.append(Grid2D(grid.nx, grid.ny, cur.copy()))
    return out


def j2d5pt(grid, weights, steps: int, *, dtype=np.float64) -> Grid2D:
    """``steps`` whole-interior updates; the B200 twin of jacobi_reference
    (oracle.py:19-34): input untouched, ghost ring carried, steps=0 copies."""
    if steps < 0:
        raise ValueError(f"steps must be non-negative, got {steps}")
    if steps == 0:
        return Grid2D(grid.nx, grid.ny, np.array(grid.data, dtype=np.float64, copy=True))
    out, _ = _solve_host(grid.data, grid.nx, grid.ny, weights, steps, 1, None, 1, 0, dtype)
    return Grid2D(grid.nx, grid.ny, out.astype(np.float64, copy=False))


jacobi = j2d5pt


def j2d5pt_device(src, dst, nx: int, ny: int, weights, steps: int, *, valid=None,
                  flags: int = 0, depth: int | None = None, stream=None) -> TrafficReport:
    """Device-resident solve on torch CUDA tensors (or raw pointers): ``src``
    and ``dst`` are padded (ny+2, pitch) float64/float32 buffers on the
    current device; runs on ``stream`` (default: torch's current stream)."""
    import torch
    if not isinstance(src, torch.Tensor) or not isinstance(dst, torch.Tensor):
        raise TypeError("j2d5pt_device expects torch CUDA tensors")
    if src.dtype not in (torch.float64, torch.float32):
        raise ValueError(f"src/dst dtype must be float64 or float32, got {src.dtype}")
    if src.dtype != dst.dtype or src.shape != dst.shape or not src.is_cuda:
        raise ValueError("src/dst must be CUDA tensors of equal dtype and shape")
    if dst.device != src.device:
        raise ValueError(f"src is on {src.device}, dst on {dst.device}")
    if src.dim() != 2 or src.shape[0] != ny + 2 or src.shape[1] < nx + 2:
        raise ValueError(f"expected ({ny + 2}, >= {nx + 2}) buffers, got {tuple(src.shape)}")
    if src.stride(1) != 1 or dst.stride() != src.stride():
        raise ValueError("buffers must be row-major with equal strides")
    pitch = src.stride(0)
    tag, ctype = ("f64", ctypes.c_double) if src.dtype == torch.float64 else ("f32", ctypes.c_float)
    pin, pout = src.data_ptr(), dst.data_ptr()
    w = (ctype * 5)(*as_weights_tuple(weights))
    if depth is not None:
        flags |= _native.FLAG_FORCE_DEPTH
    rep = _native.DtbReport()
    vr = _rect(valid)
    fn = getattr(_native.lib(), f"dtb_j2d5pt_{tag}_dev")
    # the library plans, allocates scratch and launches on the current device
    with torch.cuda.device(src.device):
        if stream is None:
            stream = torch.cuda.current_stream(src.device).cuda_stream
        rc = fn(pin, pout, nx, ny, pitch, w, steps, depth if depth is not None else 1,
                ctypes.byref(vr) if vr is not None else None, flags, ctypes.c_void_p(stream),
                ctypes.byref(rep))
    if rc != _native.DTB_OK:
        _raise(rc)
    return _report(rep)


def last_launch_count() -> int:
    """Kernel launches issued by the most recent solve on this thread."""
    return int(_native.lib().dtb_last_launch_count())
