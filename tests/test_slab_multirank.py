"""Multi-rank slab decomposition on CPU: world_size 2..4 over gloo (real
processes, torch.distributed point-to-point), with the pinned CPU oracle as
the per-rank local solver (test infrastructure) — checks that decomposition +
depth-T halo exchange is bitwise identical to a single-domain solve."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import jacobi_c
from paper_2306_03336_b200.grid import grid_new
from paper_2306_03336_b200.prng import random_interior
from paper_2306_03336_b200.slab import SlabGeometry, SlabSolver, VirtualSlabs, slab_rows

W = (0.11, -0.2, 0.37, 0.5, -0.07)


def oracle_local_solve(src, dst, nx, ny, steps):
    dst.copy_(torch.from_numpy(jacobi_c(src.numpy(), W, steps, threads=1)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, nx, ny, depth, steps, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = grid_new(nx, ny, random_interior(nx, ny, 5), ghost=0.25)
        solver = SlabSolver(SlabGeometry(nx, ny, world, rank, depth), oracle_local_solve, dist)
        solver.load(torch.from_numpy(g.data.copy()))
        solver.run(steps)
        y0, y1 = solver.geo.rows
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), solver.owned_view().numpy())
        np.save(os.path.join(out_dir, f"rows{rank}.npy"), np.array([y0, y1]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,depth,steps", [(2, 3, 10), (3, 4, 9), (4, 2, 7)])
def test_gloo_slabs_bitwise_equal_single_domain(tmp_path, world, depth, steps):
    nx, ny = 37, 29
    mp.spawn(_worker, args=(world, free_port(), nx, ny, depth, steps, str(tmp_path)),
             nprocs=world, join=True)
    g = grid_new(nx, ny, random_interior(nx, ny, 5), ghost=0.25)
    want = jacobi_c(g.data, W, steps)
    got = g.data.copy()
    for r in range(world):
        y0, y1 = np.load(tmp_path / f"rows{r}.npy")
        got[y0 + 1:y1 + 1] = np.load(tmp_path / f"rank{r}.npy")
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("world,depth", [(1, 4), (2, 1), (2, 5), (5, 3), (8, 2)])
def test_virtual_slabs_bitwise(world, depth):
    nx, ny, steps = 23, 41, 11
    g = grid_new(nx, ny, random_interior(nx, ny, 9), ghost=-0.5)
    v = VirtualSlabs(nx, ny, world, depth, oracle_local_solve).load(torch.from_numpy(g.data))
    v.run(steps)
    out = v.gather(torch.from_numpy(g.data.copy())).numpy()
    want = jacobi_c(g.data, W, steps)
    assert np.array_equal(out.view(np.uint64), want.view(np.uint64))


def test_slab_rows_partition():
    for ny in (8, 29, 1000):
        for world in (1, 2, 3, 8):
            rows = [slab_rows(ny, world, r) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == ny
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            sizes = [b - a for a, b in rows]
            assert max(sizes) - min(sizes) <= 1


def test_slab_geometry_rejects_thin_slabs():
    with pytest.raises(ValueError):
        SlabGeometry(10, 8, 4, 0, 3).validate()
