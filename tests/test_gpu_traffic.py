"""Counted traffic == modelled traffic (the reference's reconciliation
contract, engine.py:260-301 vs metrics.py:89-126, applied to the B200).

With count=True the kernels add what they actually move and compute —
cells loaded from global memory, stored back, exchanged between CTAs or
slabs, and every cell update performed — into device counters at their copy
and compute sites (DTB_FLAG_COUNT). Without it the library reports the
analytic model of the same schedule (dtb_host.cu fill_report). The two must
agree exactly, for every execution mode, and the grids must stay bitwise
equal to the oracle.
"""

import numpy as np
import pytest

from oracle import jacobi_c
from paper_2306_03336_b200 import (DeviceModel, KernelConfig, Rect, StencilWeights, grid_new,
                                   plan_device_tiles, run_dtb, run_dtb_b200)
from paper_2306_03336_b200 import _native
from paper_2306_03336_b200.prng import random_interior

pytestmark = pytest.mark.gpu

W02 = StencilWeights.diffusive(0.2)
MIXED = StencilWeights(0.11, -0.2, 0.37, 0.5, -0.07)
F = _native


def fields(r):
    return (r.global_load_cells, r.global_store_cells, r.halo_exchanged_cells,
            r.redundant_compute_cells, r.useful_compute_cells, r.scratchpad_peak_bytes,
            r.elem_bytes)


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


CASES = [
    # (nx, ny, steps, flags, depth, poison, dtype)
    (1900, 1900, 24, 0, None, False, np.float64),        # C2 geometry, resident h=4
    (700, 500, 13, 0, None, False, np.float64),          # resident, odd step tail
    (700, 500, 12, 0, 3, False, np.float64),             # resident, odd depth (one-step sweeps)
    (700, 500, 12, 0, 6, False, np.float64),
    (700, 520, 10, 0, 2, True, np.float64),              # resident poison mode
    (2700, 900, 16, 0, None, False, np.float32),         # fp32 resident
    (1500, 1400, 20, F.FLAG_FORCE_PIPE, None, False, np.float64),   # pipelined streaming
    (1500, 1400, 19, F.FLAG_FORCE_PIPE, None, False, np.float32),
    (900, 700, 18, F.FLAG_FORCE_STREAM, None, False, np.float64),   # tile-sweep streaming
    (900, 700, 9, F.FLAG_FORCE_STREAM, 3, True, np.float64),
    (129, 77, 7, 0, None, False, np.float64),            # one tile, dyn lane width
    (3, 7, 5, 0, None, False, np.float64),
]


@pytest.mark.parametrize("nx,ny,steps,flags,depth,poison,dt", CASES)
def test_counted_traffic_equals_model(nx, ny, steps, flags, depth, poison, dt):
    g = grid_new(nx, ny, random_interior(nx, ny, nx + ny), ghost=0.25)
    w = MIXED if nx % 2 else W02
    out_m, model = run_dtb_b200(g, w, steps, flags=flags, depth=depth, poison=poison, dtype=dt)
    out_c, counted = run_dtb_b200(g, w, steps, flags=flags, depth=depth, poison=poison, dtype=dt,
                                  count=True)
    assert counted.source == "b200 counted" and model.source == "b200 model"
    assert fields(counted) == fields(model), (fields(counted), fields(model))
    assert counted.useful_compute_cells == nx * ny * steps
    assert counted.redundant_compute_cells >= 0
    assert counted.global_load_cells >= nx * ny and counted.global_store_cells >= nx * ny
    want = jacobi_c(g.data, w.astuple(), steps, dt)
    assert np.array_equal(out_c.data.astype(dt).view(np.uint64 if dt == np.float64 else np.uint32),
                          want.view(np.uint64 if dt == np.float64 else np.uint32))


@pytest.mark.parametrize("n_gpus,flags", [(2, F.FLAG_SLAB_COPY), (3, F.FLAG_SLAB_FUSED),
                                          (4, F.FLAG_SLAB_FUSED)])
def test_counted_traffic_slabs(n_gpus, flags):
    nx, ny, steps = 1100, 900, 40
    g = grid_new(nx, ny, random_interior(nx, ny, 3))
    _, model = run_dtb_b200(g, W02, steps, n_gpus=n_gpus, flags=flags)
    out, counted = run_dtb_b200(g, W02, steps, n_gpus=n_gpus, flags=flags, count=True)
    assert fields(counted) == fields(model)
    if flags == F.FLAG_SLAB_FUSED:  # the slabs run the pipe: no intra-slab CTA exchange
        # every non-final epoch moves depth rows across each of the n-1 seams, both ways
        epochs = -(-steps // 16)
        assert counted.halo_exchanged_cells == (epochs - 1) * 2 * (n_gpus - 1) * 16 * nx
    assert np.array_equal(bits(out.data), bits(jacobi_c(g.data, W02.astuple(), steps)))


def test_counted_traffic_valid_window():
    g = grid_new(300, 260, random_interior(300, 260, 9))
    v = Rect(17, 9, 250, 231)
    _, model = run_dtb_b200(g, W02, 12, valid=v)
    _, counted = run_dtb_b200(g, W02, 12, valid=v, count=True)
    assert fields(counted) == fields(model)
    assert counted.useful_compute_cells == v.area * 12


def test_reference_plan_report_is_labelled_and_carries_the_b200_one():
    g = grid_new(64, 64, random_interior(64, 64, 2))
    plan = plan_device_tiles((64, 64), DeviceModel("d", 2, 8192), 4)
    _, rep = run_dtb(g, W02, 8, plan, KernelConfig(4))
    assert rep.source == "reference-plan model"
    assert rep.b200 is not None and rep.b200.source == "b200 model"
    assert rep.b200.useful_compute_cells == rep.useful_compute_cells == 64 * 64 * 8
