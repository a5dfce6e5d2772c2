"""CPU-side tests: the C ABI loads and exports what include/dtb_b200.h declares,
the native planner (callable without a GPU), the reference-compatible planner
and traffic model against the reference's recorded reports, and the argument
contract of run_dtb (validated before any CUDA call)."""

import os
import re

import numpy as np
import pytest

from paper_2306_03336_b200 import (DeviceModel, EngineError, Rect, StencilWeights, grid_new,
                                   model_dtb_traffic, plan_b200, plan_device_tiles, run_dtb)
from paper_2306_03336_b200 import _native
from paper_2306_03336_b200.prng import random_interior

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "dtb_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(dtb_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native._SIGNATURES)


def test_struct_layouts_match_header():
    import ctypes
    assert ctypes.sizeof(_native.DtbReport) == 7 * 8
    assert ctypes.sizeof(_native.DtbRect) == 4 * 8
    assert ctypes.sizeof(_native.DtbPlanInfo) == 10 * 4 + 6 * 8 + 8


def test_native_planner_resident_for_c2():
    p = plan_b200(1900, 1900, 8, 10000, 1)
    assert p.mode == "resident"
    assert p.ctas <= 148
    assert p.smem_bytes <= 232448
    assert p.tiles_x * p.tiles_y == p.ctas
    assert p.load_w <= 32 * p.lane_elems


def test_native_planner_resident_for_c3a_fp32():
    p = plan_b200(2700, 2700, 4, 10000, 1)
    assert p.mode == "resident" and p.elem_bytes == 4


def test_native_planner_streams_large_domains():
    for nx, elem in ((16384, 8), (8192, 4), (32768, 8)):
        p = plan_b200(nx, nx, elem, 1000, 1)
        assert p.mode in ("pipe", "streaming"), (nx, elem)
        assert p.halo >= 2


def test_native_planner_small_grids_and_flags():
    p = plan_b200(3, 3, 8, 2, 1)
    assert p.tiles_x == 1 and p.tiles_y == 1 and p.dyn
    p = plan_b200(256, 256, 8, 100, 1, _native.FLAG_FORCE_STREAM)
    assert p.mode == "streaming"
    p = plan_b200(256, 256, 8, 100, 1, _native.FLAG_FORCE_NAIVE)
    assert p.mode == "naive"
    p = plan_b200(1900, 1900, 8, 100, 6, _native.FLAG_FORCE_DEPTH)
    assert p.halo == 6


def test_native_planner_covers_domain_exactly():
    # computed cells = sum of inner load areas >= domain; redundancy bounded
    for nx, ny, elem in ((1900, 1900, 8), (256, 256, 8), (2700, 2700, 4), (1000, 37, 8)):
        p = plan_b200(nx, ny, elem, 100, 1)
        assert p.computed_cells_per_step >= nx * ny
        assert p.computed_cells_per_step < 4 * nx * ny + 64 * 64


def test_reference_planner_matches_recorded_plans(golden):
    meta, _ = golden
    for run in meta["runs"]:
        plan = plan_device_tiles((run["nx"], run["ny"]), DeviceModel("d", run["workers"], run["cap"]),
                                 run["t_depth"])
        assert len(plan.tiles) == run["tiles"]
        assert plan.footprint_bytes == run["footprint"]


def test_traffic_model_matches_reference_engine_counters(golden):
    meta, _ = golden
    for run in meta["runs"]:
        plan = plan_device_tiles((run["nx"], run["ny"]), DeviceModel("d", run["workers"], run["cap"]),
                                 run["t_depth"])
        v = Rect(*run["valid"]) if run["valid"] else None
        rep = model_dtb_traffic(plan, run["steps"], v)
        assert [rep.global_load_cells, rep.global_store_cells, rep.halo_exchanged_cells,
                rep.redundant_compute_cells, rep.useful_compute_cells,
                rep.scratchpad_peak_bytes, rep.elem_bytes] == run["report"]


def _fixed_band_plan(t):
    from paper_2306_03336_b200 import DeviceTile, TilingPlan, scratchpad_footprint
    device = DeviceModel("fixed", 8, 131072)
    clip = Rect(-1, -1, 514, 514)
    tiles = tuple(DeviceTile(Rect(0, ty, 512, 64), t, Rect(0, ty, 512, 64).dilate(t).intersect(clip))
                  for ty in range(0, 512, 64))
    fp = max(scratchpad_footprint((x.load_region.width, x.load_region.height), t, 8, 8)
             for x in tiles)
    return TilingPlan(512, 512, t, 8, device, tiles, fp)


def test_traffic_reduction_acceptance_5():
    # test_acceptance.py:210-240 — the published modelled traffic numbers
    from paper_2306_03336_b200 import model_naive_traffic
    assert model_naive_traffic((512, 512), 8).traffic_cells == 4_194_304
    got = {t: model_dtb_traffic(_fixed_band_plan(t), 8).traffic_cells for t in (2, 4, 8)}
    assert got == {2: 2_154_496, 4: 1_105_920, 8: 581_632}


W = StencilWeights.diffusive(0.2)


def g8():
    return grid_new(8, 8, random_interior(8, 8, 0))


def test_run_dtb_rejects_bad_arguments_like_the_reference():
    # test_engine.py:138-154 — all raised before touching the device
    g = g8()
    plan = plan_device_tiles((8, 8), DeviceModel("d", 2, 4096), 4)
    with pytest.raises(ValueError):
        run_dtb(g, W, 6, plan)
    with pytest.raises(ValueError):
        run_dtb(g, W, 0, plan)
    with pytest.raises(ValueError):
        run_dtb(grid_new(4, 4, 0.0), W, 4, plan)
    with pytest.raises(ValueError):
        run_dtb(g, W, 4, plan, valid=Rect(4, 4, 8, 8))
    with pytest.raises(ValueError):
        run_dtb(g, W, 4, plan, valid=Rect(2, 2, 0, 0))
    f32_plan = plan_device_tiles((8, 8), DeviceModel("d", 2, 4096), 4, elem_bytes=4)
    with pytest.raises(ValueError):
        run_dtb(g, W, 4, f32_plan)


def test_run_dtb_capacity_guard():
    # test_engine.py:157-162
    import dataclasses
    g = grid_new(16, 16, random_interior(16, 16, 1))
    plan = plan_device_tiles((16, 16), DeviceModel("big", 1, 1 << 20), 2)
    lying = dataclasses.replace(plan, device=DeviceModel("small", 1, 64))
    with pytest.raises(EngineError):
        run_dtb(g, W, 2, lying)


def test_native_validation_errors_without_gpu():
    # the ABI validates arguments before any CUDA call and maps them to codes
    import ctypes
    lib = _native.lib()
    buf = np.zeros((6, 6))
    out = np.zeros_like(buf)
    w = (ctypes.c_double * 5)(0.2, 0.2, 0.2, 0.2, float("nan"))
    rc = lib.dtb_j2d5pt_f64(buf.ctypes.data, out.ctypes.data, 4, 4, 6, w, 2, 1, None, 1, 1, 0, None)
    assert rc == _native.DTB_EINVAL and "non-finite" in _native.last_error()
    w = (ctypes.c_double * 5)(0.2, 0.2, 0.2, 0.2, 0.2)
    rc = lib.dtb_j2d5pt_f64(buf.ctypes.data, out.ctypes.data, 4, 4, 6, w, 3, 2, None, 1, 1, 0, None)
    assert rc == _native.DTB_EINVAL and "multiple" in _native.last_error()
    r = _native.DtbRect(1, 1, 9, 9)
    rc = lib.dtb_j2d5pt_f64(buf.ctypes.data, out.ctypes.data, 4, 4, 6, w, 2, 1, ctypes.byref(r), 1, 1, 0, None)
    assert rc == _native.DTB_EINVAL and "valid region" in _native.last_error()
    rc = lib.dtb_j2d5pt_f64(buf.ctypes.data, out.ctypes.data, 4, 4, 5, w, 2, 1, None, 1, 1, 0, None)
    assert rc == _native.DTB_EINVAL and "pitch" in _native.last_error()
    rc = lib.dtb_j2d5pt_f64(buf.ctypes.data, out.ctypes.data, 4, 4, 6, w, 2, 1, None, 1, 0, 0, None)
    assert rc == _native.DTB_EINVAL and "n_gpus" in _native.last_error()
    r = _native.DtbRect(1, 1, 4, 2)
    rc = lib.dtb_j2d5pt_f64(buf.ctypes.data, out.ctypes.data, 4, 4, 6, w, 2, 1, ctypes.byref(r), 1, 2, 0, None)
    assert rc == _native.DTB_EINVAL and "valid region" in _native.last_error()


def test_weights_validation():
    with pytest.raises(ValueError):
        StencilWeights(0.2, 0.2, float("inf"), 0.2, 0.2)


def test_infeasible_plan_carries_min_required_bytes():
    """InfeasiblePlanError(msg, min_required_bytes) (planner.py:51-56,222-228):
    the B200 planner reports the smallest per-CTA shared memory a plan of the
    requested kind would need, through dtb_last_min_required_bytes."""
    from paper_2306_03336_b200 import InfeasiblePlanError
    # 16384^2 fp64 cannot be smem-resident on one B200 (2.1 GB vs 34 MB)
    with pytest.raises(InfeasiblePlanError) as ei:
        plan_b200(16384, 16384, 8, 100, 1, _native.FLAG_FORCE_RESIDENT)
    need = ei.value.min_required_bytes
    assert need > 232448, need
    assert str(need) in str(ei.value)
    # a forced depth whose halo rows alone overflow a CTA's shared memory
    with pytest.raises(InfeasiblePlanError) as ei:
        plan_b200(4096, 4096, 8, 400, 200, _native.FLAG_FORCE_STREAM | _native.FLAG_FORCE_DEPTH)
    assert ei.value.min_required_bytes == (1 + 2 * 200) * 1024
    # success clears it
    plan_b200(256, 256, 8, 100, 1)
    assert _native.lib().dtb_last_min_required_bytes() == 0


def test_device_entry_rejects_other_dtypes_before_any_cuda_call():
    """a 2-byte or integer buffer must raise, not run the f32 path
    with a pitch read in the wrong element size (checked before the device)."""
    import torch
    from paper_2306_03336_b200 import j2d5pt_device
    w = StencilWeights.diffusive(0.2)
    for dt in (torch.float16, torch.bfloat16, torch.int32, torch.int64):
        a = torch.zeros((10, 12), dtype=dt)
        with pytest.raises(ValueError, match="dtype"):
            j2d5pt_device(a, a.clone(), 8, 8, w, 2)
    with pytest.raises(TypeError):
        j2d5pt_device(np.zeros((10, 10)), np.zeros((10, 10)), 8, 8, w, 2)
