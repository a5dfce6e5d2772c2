"""Traffic accounting (mirrors dtb.metrics' TrafficReport and models, metrics.py:39-126).

``run_dtb`` returns a :class:`TrafficReport`. When the caller passes a
reference-style :class:`~.planner.TilingPlan`, the report is that plan's
model — exactly the counters the reference engine reconciles to
(``report == model_dtb_traffic(plan, steps, valid)``, test_engine.py:41-50),
labelled ``source="reference-plan model"``; the B200 never runs that
serial-tile schedule, so the traffic of what did run rides along as
``report.b200``. ``run_dtb_b200`` returns the B200 schedule's report
directly: ``source="b200 model"`` (the analytic model of the schedule,
dtb_host.cu fill_report) or, with ``count=True``, ``source="b200 counted"``
(the kernels' device counters at their copy and compute sites; the tests
require both to agree exactly).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .grid import Rect
from .planner import DEFAULT_ELEM_BYTES, tile_active_region

__all__ = ["TrafficReport", "model_naive_traffic", "model_dtb_traffic", "RUN_CSV_COLUMNS",
           "run_csv_header", "run_csv_row", "format_bytes", "presets_csv",
           "sota_footprint_table", "sota_footprint_csv"]


@dataclass(frozen=True)
class TrafficReport:
    global_load_cells: int
    global_store_cells: int
    halo_exchanged_cells: int
    redundant_compute_cells: int
    useful_compute_cells: int
    scratchpad_peak_bytes: int
    elem_bytes: int = DEFAULT_ELEM_BYTES
    # provenance; not part of the reference's counters (not compared)
    source: str = field(default="model", compare=False)
    b200: "TrafficReport | None" = field(default=None, compare=False, repr=False)

    @property
    def global_load_bytes(self) -> int:
        return self.global_load_cells * self.elem_bytes

    @property
    def global_store_bytes(self) -> int:
        return self.global_store_cells * self.elem_bytes

    @property
    def halo_exchanged_bytes(self) -> int:
        return self.halo_exchanged_cells * self.elem_bytes

    @property
    def traffic_cells(self) -> int:
        return self.global_load_cells + self.global_store_cells


def model_naive_traffic(domain, steps: int, elem_bytes: int = DEFAULT_ELEM_BYTES) -> TrafficReport:
    """One load + one store per cell per step (metrics.py:69-86)."""
    nx, ny = domain
    if nx < 0 or ny < 0:
        raise ValueError(f"negative domain dims {domain}")
    if steps < 0:
        raise ValueError(f"negative steps {steps}")
    n = nx * ny * steps
    return TrafficReport(n, n, 0, 0, n, 0, elem_bytes)


def model_dtb_traffic(plan, total_steps: int, valid=None) -> TrafficReport:
    """Counters of the reference schedule for ``plan`` (metrics.py:89-126):
    per time block, every tile loads its load region's domain cells and
    stores its interior; 2*(active workers-1) halo columns of the domain rows
    per superstep; compute = the trapezoid areas."""
    if total_steps < 1 or total_steps % plan.t_depth:
        raise ValueError(f"total_steps {total_steps} is not a positive multiple of "
                         f"t_depth {plan.t_depth}")
    domain = Rect(0, 0, plan.nx, plan.ny)
    if valid is None:
        valid = domain
    elif not domain.contains(valid) or valid.width == 0 or valid.height == 0:
        raise ValueError(f"valid region {valid} not within domain {domain}")
    blocks = total_steps // plan.t_depth
    loads = stores = halo = compute = 0
    for tile in plan.tiles:
        lr = tile.load_region
        covered = domain.intersect(lr)
        loads += covered.area
        stores += tile.interior.width * tile.interior.height
        active = min(plan.device.workers, lr.width)
        halo += 2 * max(active - 1, 0) * covered.height * plan.t_depth
        compute += sum(tile_active_region(tile, s, valid).area
                       for s in range(1, plan.t_depth + 1))
    useful = valid.width * valid.height * total_steps
    return TrafficReport(loads * blocks, stores * blocks, halo * blocks,
                         compute * blocks - useful, useful, plan.footprint_bytes,
                         plan.elem_bytes)


# --- CSV rows of the harness (metrics.py:133-205 of the reference) ----------
# One stable schema for `run` and `sweep` rows; absent values stay empty.
RUN_CSV_COLUMNS = (
    "status", "nx", "ny", "valid_x0", "valid_y0", "valid_nx", "valid_ny",
    "t_depth", "total_steps", "device", "workers",
    "scratchpad_bytes_per_worker", "threads", "ilp", "seed",
    "weight_w", "weight_e", "weight_s", "weight_c", "weight_n",
    "tiles", "tile_w", "tile_h", "footprint_bytes", "elem_bytes",
    "global_load_cells", "global_store_cells", "halo_exchanged_cells",
    "redundant_compute_cells", "useful_compute_cells", "scratchpad_peak_bytes",
    "bit_equal", "max_abs_diff", "wall_time_s", "host_model_gflops",
)

# published scratchpad footprints the paper compares against
SOTA_FOOTPRINTS = (("StencilGen", "4.32 MB"), ("AN5D", "0.864 MB"))


def run_csv_header() -> str:
    return ",".join(RUN_CSV_COLUMNS)


def run_csv_row(record: dict) -> str:
    unknown = set(record) - set(RUN_CSV_COLUMNS)
    if unknown:
        raise ValueError(f"unknown CSV fields: {sorted(unknown)}")

    def cell(v) -> str:
        if v is None:
            return ""
        if isinstance(v, bool):
            return "true" if v else "false"
        return str(v)

    return ",".join(cell(record.get(c)) for c in RUN_CSV_COLUMNS)


def format_bytes(n: int) -> str:
    """KB below 1 MiB, MB with two decimals above (1 KB = 1024 B)."""
    if n < 0:
        raise ValueError(f"negative byte count {n}")
    kb = n / 1024.0
    return f"{kb:g} KB" if kb < 1024.0 else f"{kb / 1024.0:.2f} MB"


def sota_footprint_table(device=None) -> list:
    rows = list(SOTA_FOOTPRINTS)
    if device is not None:
        rows.append((f"dtb-{device.name}", format_bytes(device.total_bytes)))
    return rows


def sota_footprint_csv(device=None) -> str:
    return "\n".join(["name,scratchpad"]
                     + [f"{n},{v}" for n, v in sota_footprint_table(device)]) + "\n"


def presets_csv(presets: dict) -> str:
    lines = ["name,workers,scratchpad_bytes_per_worker,total_bytes,total"]
    for name, dev in presets.items():
        lines.append(f"{name},{dev.workers},{dev.scratchpad_bytes_per_worker},"
                     f"{dev.total_bytes},{format_bytes(dev.total_bytes)}")
    return "\n".join(lines) + "\n"
