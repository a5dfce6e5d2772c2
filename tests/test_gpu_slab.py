"""Multi-GPU slab decomposition on one B200: every virtual rank's local solve
runs the real sm_100a kernel; the halo exchange is an in-process copy. Must
be bitwise equal to the single-domain oracle (and so to jacobi_reference)."""

import numpy as np
import pytest

from oracle import jacobi_c
from paper_2306_03336_b200 import StencilWeights, j2d5pt_device
from paper_2306_03336_b200.grid import grid_new
from paper_2306_03336_b200.prng import fill_random_rows_device, random_interior
from paper_2306_03336_b200.slab import SlabGeometry, VirtualSlabs

pytestmark = pytest.mark.gpu

W = StencilWeights(0.11, -0.2, 0.37, 0.5, -0.07)


def gpu_local_solve(src, dst, nx, ny, steps):
    j2d5pt_device(src, dst, nx, ny, W, steps)


@pytest.mark.parametrize("nx,ny,world,depth,steps", [
    (300, 257, 2, 4, 13), (300, 257, 4, 6, 20), (1000, 600, 3, 16, 40), (129, 64, 8, 3, 7)])
def test_virtual_slabs_on_gpu_bitwise(nx, ny, world, depth, steps):
    import torch
    g = grid_new(nx, ny, random_interior(nx, ny, 3), ghost=0.25)
    v = VirtualSlabs(nx, ny, world, depth, gpu_local_solve)
    v.load(torch.from_numpy(g.data).cuda())
    v.run(steps)
    torch.cuda.synchronize()
    out = v.gather(torch.from_numpy(g.data).cuda().clone()).cpu().numpy()
    want = jacobi_c(g.data, W.astuple(), steps)
    assert np.array_equal(out.view(np.uint64), want.view(np.uint64))


def test_slab_row_fill_matches_host_fill():
    import torch
    nx, ny, world = 333, 200, 3
    g = grid_new(nx, ny, random_interior(nx, ny, 1))
    for rank in range(world):
        geo = SlabGeometry(nx, ny, world, rank, 5)
        buf = torch.empty((geo.local_ny + 2, nx + 2 + 7), dtype=torch.float64, device="cuda")
        fill_random_rows_device(buf, nx, ny, 1, geo.global_row0)
        r0 = geo.global_row0
        got = buf[:, :nx + 2].cpu().numpy()
        assert np.array_equal(got.view(np.uint64), g.data[r0:r0 + geo.local_ny + 2].view(np.uint64))


@pytest.mark.parametrize("n_gpus,nx,ny,steps,dt", [
    (2, 300, 257, 40, np.float64), (3, 1900, 1900, 36, np.float64), (4, 513, 64, 17, np.float32),
    (5, 128, 5, 9, np.float64)])
def test_host_entry_n_gpus_slabs_bitwise(n_gpus, nx, ny, steps, dt):
    """n_gpus > 1 through the C ABI (native y-slabs, 16-row halo copies): on a
    one-GPU box the slabs share the device in order; bitwise equal to one GPU
    and to the oracle."""
    from oracle import jacobi_c
    from paper_2306_03336_b200 import Grid2D, StencilWeights, grid_new, run_dtb_b200
    from paper_2306_03336_b200.prng import random_interior
    g = grid_new(nx, ny, random_interior(nx, ny, n_gpus), ghost=0.375)
    w = StencilWeights(0.11, -0.2, 0.37, 0.5, -0.07)
    one, _ = run_dtb_b200(g, w, steps, dtype=dt)
    multi, rep = run_dtb_b200(g, w, steps, dtype=dt, n_gpus=n_gpus)
    assert np.array_equal(multi.data.view(np.uint64), one.data.view(np.uint64))
    want = jacobi_c(g.data, w.astuple(), steps, dt)
    assert np.array_equal(multi.data.astype(dt), want)
    assert rep.useful_compute_cells == nx * ny * steps and rep.halo_exchanged_cells > 0


@pytest.mark.parametrize("n_gpus,nx,ny,steps,dt", [
    (2, 1000, 700, 40, np.float64), (3, 777, 1201, 33, np.float32), (4, 2048, 512, 48, np.float64)])
def test_host_entry_fused_slab_halos_bitwise(n_gpus, nx, ny, steps, dt):
    """Fused exchange: each slab's pipelined kernel stores the neighbours' halo
    rows into their next input in-kernel (HaloMirror), its own stores limited
    to its owned rows; bitwise equal to the copy exchange, one GPU and the oracle."""
    from oracle import jacobi_c
    from paper_2306_03336_b200 import StencilWeights, _native, grid_new, run_dtb_b200
    from paper_2306_03336_b200.prng import random_interior
    g = grid_new(nx, ny, random_interior(nx, ny, 7 * n_gpus), ghost=-1.5)
    w = StencilWeights(0.11, -0.2, 0.37, 0.5, -0.07)
    fused, rep = run_dtb_b200(g, w, steps, dtype=dt, n_gpus=n_gpus, flags=_native.FLAG_SLAB_FUSED)
    copy, _ = run_dtb_b200(g, w, steps, dtype=dt, n_gpus=n_gpus, flags=_native.FLAG_SLAB_COPY)
    assert np.array_equal(fused.data.view(np.uint64), copy.data.view(np.uint64))
    assert np.array_equal(fused.data.astype(dt), jacobi_c(g.data, w.astuple(), steps, dt))
    assert rep.halo_exchanged_cells == 2 * (n_gpus - 1) * 16 * nx * ((steps - 1) // 16)


def test_host_entry_n_gpus_with_valid_region():
    """A pruned (valid=) solve split over slabs equals the one-GPU pruned solve
    and the oracle on the extracted region (engine.py:26-30)."""
    from oracle import jacobi_c
    from paper_2306_03336_b200 import Rect, StencilWeights, grid_extract, grid_new, run_dtb_b200
    from paper_2306_03336_b200.prng import random_interior
    g = grid_new(300, 260, random_interior(300, 260, 3), ghost=0.125)
    w = StencilWeights(0.11, -0.2, 0.37, 0.5, -0.07)
    v = Rect(17, 9, 250, 231)
    one, _ = run_dtb_b200(g, w, 40, valid=v)
    for n in (2, 3):
        multi, rep = run_dtb_b200(g, w, 40, valid=v, n_gpus=n)
        assert np.array_equal(multi.data.view(np.uint64), one.data.view(np.uint64))
        assert rep.useful_compute_cells == 250 * 231 * 40
    sub = grid_extract(g, v)
    want = jacobi_c(sub.data, w.astuple(), 40)
    assert np.array_equal(one.data[v.y0:v.y0 + v.height + 2, v.x0:v.x0 + v.width + 2], want)


@pytest.mark.parametrize("flags_name", ["FLAG_SLAB_FUSED", "FLAG_SLAB_COPY"])
def test_host_entry_slabs_across_real_devices(flags_name):
    """Slabs on distinct GPUs: the fused mode's in-kernel stores go to a peer
    device over NVLink (peer access enabled and checked by the library, copy
    mode otherwise). Skipped on boxes with one GPU."""
    import torch
    from paper_2306_03336_b200 import _native, run_dtb_b200
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs two or more GPUs")
    nx, ny, steps = 1100, 900, 40
    g = grid_new(nx, ny, random_interior(nx, ny, 5))
    out, _ = run_dtb_b200(g, W, steps, n_gpus=min(n, 4), flags=getattr(_native, flags_name))
    want = jacobi_c(g.data, W.astuple(), steps)
    assert np.array_equal(out.data.view(np.uint64), want.view(np.uint64))
