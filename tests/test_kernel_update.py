"""The one-step entry `j2d5pt_update` / `Window` (paper_2306_03336_b200/kernel.py),
mirroring the reference's tests/test_kernel.py: argument errors on the host
(no GPU), bitwise updates on the GPU against the numpy restatement."""

import numpy as np
import pytest

from oracle import jacobi_numpy
from paper_2306_03336_b200 import (Grid2D, KernelConfig, Rect, StencilWeights, Window,
                                   Xoshiro256StarStar, grid_new, j2d5pt_update, splitmix64)
from paper_2306_03336_b200.prng import random_interior

ALL_02 = StencilWeights(0.2, 0.2, 0.2, 0.2, 0.2)


def fresh(nx, ny, seed, ghost=0.0):
    return grid_new(nx, ny, random_interior(nx, ny, seed), ghost=ghost)


def update_grid(g, w, cols=None, cfg=KernelConfig()):
    out = Grid2D(g.nx, g.ny, g.data.copy())
    cols = cols if cols is not None else Rect(0, 0, g.nx, g.ny)
    j2d5pt_update(Window.over_interior(g.data), Window.over_interior(out.data), w, cols, cfg)
    return out


# --- host: argument contract (no GPU call is reached) --------------------------

def test_window_geometry_and_validation():
    buf = np.zeros((5, 7))
    w = Window(buf, 2, 1, 3, 2)
    assert w.stride == 7 and w.base == 9
    iw = Window.over_interior(buf)
    assert (iw.x0, iw.y0, iw.width, iw.height) == (1, 1, 5, 3)
    with pytest.raises(ValueError):
        Window(np.zeros((3, 3), dtype=np.float32), 0, 0, 1, 1)
    with pytest.raises(ValueError):
        Window(buf, 0, 0, -1, 2)
    with pytest.raises(ValueError):
        KernelConfig(0)


def test_empty_cols_is_noop():
    g = fresh(5, 5, 3)
    before = g.data.copy()
    out = np.full_like(g.data, 7.0)
    j2d5pt_update(Window.over_interior(g.data), Window.over_interior(out), ALL_02,
                  Rect(1, 1, 0, 3), KernelConfig(3))
    assert np.array_equal(out, np.full_like(out, 7.0)) and np.array_equal(g.data, before)


def test_rejects_aliasing_and_out_of_range():
    buf = np.zeros((8, 8))
    win = Window.over_interior(buf)
    with pytest.raises(ValueError):
        j2d5pt_update(win, win, ALL_02, Rect(0, 0, 6, 6))
    a = np.zeros((8, 10))
    with pytest.raises(ValueError):  # views sharing memory
        j2d5pt_update(Window(a, 1, 1, 8, 6), Window(a[1:, :], 1, 1, 8, 4), ALL_02, Rect(0, 0, 8, 4))
    wi, wo = Window(np.zeros((7, 8)), 1, 1, 6, 4), Window(np.zeros((7, 8)), 1, 1, 6, 4)
    with pytest.raises(IndexError):
        j2d5pt_update(wi, wo, ALL_02, Rect(0, 0, 6, 5))
    with pytest.raises(IndexError):
        j2d5pt_update(wi, wo, ALL_02, Rect(-1, 0, 2, 2))
    with pytest.raises(IndexError):  # stencil reach not backed by the input buffer
        j2d5pt_update(Window(np.zeros((6, 6)), 0, 0, 6, 6), Window(np.zeros((6, 6)), 0, 0, 6, 6),
                      ALL_02, Rect(0, 0, 6, 6))


def test_xoshiro_stream():
    # frozen vector of the reference (test_prng.py:27-28, 74-76)
    r = Xoshiro256StarStar(42)
    assert [r.next_u64() for _ in range(4)] == [8753603600186813506, 8273390160575518493,
                                                6071410674495273587, 7033778288727411263]
    assert Xoshiro256StarStar(123)._s == [int(v) for v in splitmix64(123, 4)]
    r = Xoshiro256StarStar(5)
    vals = [r.random() for _ in range(500)]
    assert all(0.0 <= v < 1.0 for v in vals)
    assert all(3 <= Xoshiro256StarStar(i).randint(3, 9) <= 9 for i in range(50))
    assert Xoshiro256StarStar(8).choice("abc") in "abc"
    assert all(2.5 <= Xoshiro256StarStar(i).uniform(2.5, 3.25) < 3.25 for i in range(50))
    with pytest.raises(ValueError):
        r.randint(5, 4)


# --- GPU: the update itself -----------------------------------------------------

@pytest.mark.gpu
def test_spike_and_accumulation_order():
    g = grid_new(3, 3, lambda x, y: 1.0 if (x, y) == (1, 1) else 0.0)
    out = update_grid(g, ALL_02)
    assert np.array_equal(out.interior, [[0.0, 0.2, 0.0], [0.2, 0.2, 0.2], [0.0, 0.2, 0.0]])
    g = grid_new(1, 1, 1.0, ghost=1.0)
    out = update_grid(g, StencilWeights(0.1, 0.3, 0.7, 1e-3, 0.2))
    assert out.interior[0, 0] == 1.0 * 0.1 + 1.0 * 0.3 + 1.0 * 0.7 + 1.0 * 1e-3 + 1.0 * 0.2


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny,ilp", [(37, 41, 1), (37, 41, 5), (1, 9, 2), (130, 3, 4)])
def test_matches_restatement_bitwise(nx, ny, ilp):
    w = StencilWeights(0.11, -0.2, 0.37, 0.5, -0.07)
    g = fresh(nx, ny, nx * ny, ghost=0.375)
    out = update_grid(g, w, cfg=KernelConfig(ilp))
    assert np.array_equal(out.data.view(np.uint64), jacobi_numpy(g.data, w.astuple(), 1).view(np.uint64))


@pytest.mark.gpu
def test_partial_cols_and_disjoint_regions_of_one_buffer():
    g = fresh(9, 8, 4)
    out = update_grid(g, ALL_02, cols=Rect(2, 3, 4, 2))
    full = jacobi_numpy(g.data, ALL_02.astuple(), 1)
    mask = np.zeros_like(g.data, dtype=bool)
    mask[1 + 3:1 + 5, 1 + 2:1 + 6] = True
    assert np.array_equal(out.data[mask], full[mask])
    assert np.array_equal(out.data[~mask], g.data[~mask])
    buf = np.arange(80, dtype=np.float64).reshape(10, 8) / 7.0
    want = buf.copy()
    src = buf[0:5, 0:8].copy()
    want[5:7, 1:7] = jacobi_numpy(src, ALL_02.astuple(), 1)[1:3, 1:7]
    j2d5pt_update(Window(buf, 1, 1, 6, 3), Window(buf, 1, 5, 6, 2), ALL_02, Rect(0, 0, 6, 2))
    assert np.array_equal(buf, want)


@pytest.mark.gpu
def test_power_of_two_scaling_and_locality():
    g = fresh(11, 13, 8)
    w = StencilWeights(0.3, 0.1, -0.25, 0.6, 0.25)
    out = update_grid(g, w)
    scaled = Grid2D(g.nx, g.ny, g.data * 2.0 ** 12)
    assert np.array_equal(update_grid(scaled, w).interior, out.interior * 2.0 ** 12)
    g = fresh(10, 9, 11)
    h = Grid2D(g.nx, g.ny, g.data.copy())
    h.interior[4, 6] += 0.5
    diff = update_grid(g, ALL_02).interior != update_grid(h, ALL_02).interior
    changed = {(int(x), int(y)) for y, x in zip(*np.nonzero(diff))}
    assert 1 <= len(changed) and changed <= {(6, 4), (5, 4), (7, 4), (6, 3), (6, 5)}
