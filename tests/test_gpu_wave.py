"""The host-buffer pass wavefront (dtb_host.cu solve_host_wave, dtb_pipe.cuh
launch_pipe_wave): input row blocks stream in while the first passes run as
diagonals over them, the middle passes run plainly, the last passes run as a
wavefront whose final row blocks stream out.

DTB_WAVE_ROWS / DTB_WAVE_PASSES force it onto small grids with small row
blocks and every phase split: all passes in one wavefront, wavefront + plain
+ wavefront, a partial last pass. Tolerance: none — bit patterns against the
pinned C oracle; counted traffic == the phase-wise model.
"""

import numpy as np
import pytest

from oracle import jacobi_c
from paper_2306_03336_b200 import StencilWeights, grid_new, run_dtb_b200
from paper_2306_03336_b200 import _native
from paper_2306_03336_b200.prng import random_interior

pytestmark = pytest.mark.gpu

W02 = StencilWeights.diffusive(0.2)
MIXED = StencilWeights(0.11, -0.2, 0.37, 0.5, -0.07)


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def fields(r):
    return (r.global_load_cells, r.global_store_cells, r.halo_exchanged_cells,
            r.redundant_compute_cells, r.useful_compute_cells)


# (nx, ny, steps, rows per block, wavefront passes, weights, dtype)
CASES = [
    (300, 200, 24, 16, 1, W02, np.float64),      # A: pass 1, B: pass 2, C: pass 3
    (300, 200, 40, 16, 2, MIXED, np.float64),    # 2 + 1 + 2 passes
    (300, 200, 37, 24, 2, W02, np.float64),      # partial last pass in the C phase
    (300, 200, 21, 20, 9, MIXED, np.float64),    # all passes in one wavefront
    (513, 333, 64, 17, 3, W02, np.float64),      # odd sizes, many blocks
    (1000, 97, 30, 8, 2, W02, np.float64),       # 8-row blocks (the minimum)
    (700, 260, 48, 32, 2, MIXED, np.float32),    # fp32
    (640, 300, 1000, 40, 4, W02, np.float64),    # long solve, 117 plain passes between
]


@pytest.mark.parametrize("nx,ny,steps,rows,m,w,dt", CASES)
def test_wavefront_bitwise_and_counted(monkeypatch, nx, ny, steps, rows, m, w, dt):
    monkeypatch.setenv("DTB_WAVE_ROWS", str(rows))
    monkeypatch.setenv("DTB_WAVE_PASSES", str(m))
    g = grid_new(nx, ny, random_interior(nx, ny, nx + steps), ghost=0.25)
    want = jacobi_c(g.data, w.astuple(), steps, dt)
    out, model = run_dtb_b200(g, w, steps, dtype=dt, flags=_native.FLAG_FORCE_PIPE)
    got = out.data.astype(dt)
    assert np.array_equal(bits(got), bits(want))
    out2, counted = run_dtb_b200(g, w, steps, dtype=dt, flags=_native.FLAG_FORCE_PIPE, count=True)
    assert np.array_equal(bits(out2.data.astype(dt)), bits(want))
    assert fields(counted) == fields(model)
    assert model.useful_compute_cells == nx * ny * steps


def test_wavefront_off_matches(monkeypatch):
    """DTB_WAVE_ROWS=0 is the plain H2D + passes + D2H path: same bits, and
    the report is that of a different schedule."""
    nx, ny, steps = 400, 300, 40
    g = grid_new(nx, ny, random_interior(nx, ny, 5))
    monkeypatch.setenv("DTB_WAVE_ROWS", "24")
    monkeypatch.setenv("DTB_WAVE_PASSES", "2")
    a, ra = run_dtb_b200(g, W02, steps, flags=_native.FLAG_FORCE_PIPE)
    monkeypatch.setenv("DTB_WAVE_ROWS", "0")
    b, rb = run_dtb_b200(g, W02, steps, flags=_native.FLAG_FORCE_PIPE)
    assert np.array_equal(bits(a.data), bits(b.data))
    assert ra.useful_compute_cells == rb.useful_compute_cells
    assert fields(ra) != fields(rb)
