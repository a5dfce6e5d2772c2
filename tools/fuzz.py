"""Randomised edge-case sweep of every entry point against the C oracle
(GPU box): random shapes, odd-column valid windows, mixed-sign weights, both
dtypes, forced modes and depths, n_gpus slabs (fused and copy exchange),
device views with odd pitch/offset. Usage: python tools/fuzz.py CASES SEED"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import jacobi_c
from paper_2306_03336_b200 import (Rect, StencilWeights, _native, grid_extract, grid_new,
                                   j2d5pt_device, run_dtb_b200)
from paper_2306_03336_b200.prng import random_interior

n_cases, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
F = _native
MODES = [0, F.FLAG_FORCE_STREAM, F.FLAG_FORCE_PIPE, F.FLAG_FORCE_RESIDENT, F.FLAG_FORCE_NAIVE]
bad = skipped = 0
for c in range(n_cases):
    maxn = int(os.environ.get("FUZZ_MAXN", "900"))
    nx, ny = int(rng.integers(1, maxn)), int(rng.integers(1, maxn))
    steps = int(rng.integers(1, 50))
    dt = np.float32 if rng.random() < 0.35 else np.float64
    g = grid_new(nx, ny, random_interior(nx, ny, c + seed), ghost=float(rng.choice([0.0, 0.375, -2.0])))
    w = StencilWeights(*(float(x) for x in rng.uniform(-0.7, 0.7, 5)))
    if rng.random() < 0.35:  # isotropic (w = e = s = n): the shared-product kernels
        a = float(rng.uniform(-0.7, 0.7))
        w = StencilWeights(a, a, a, float(rng.uniform(-0.7, 0.7)), a)
    valid = None
    if rng.random() < 0.4 and nx > 2 and ny > 2:
        x0, y0 = int(rng.integers(0, nx - 1)), int(rng.integers(0, ny - 1))
        valid = Rect(x0, y0, int(rng.integers(1, nx - x0 + 1)), int(rng.integers(1, ny - y0 + 1)))
    flags = int(rng.choice(MODES))
    depth = int(rng.integers(1, 9)) if rng.random() < 0.2 else None
    if depth and steps % depth:
        depth = None
    n_gpus = int(rng.choice([1, 1, 2, 3, 4]))
    if n_gpus > 1:
        flags = int(rng.choice([0, F.FLAG_SLAB_COPY, F.FLAG_SLAB_FUSED]))
        depth = None
    src = g if valid is None else grid_extract(g, valid)
    want = jacobi_c(src.data, w.astuple(), steps, dt)
    try:
        out, _ = run_dtb_b200(g, w, steps, valid=valid, dtype=dt, flags=flags, depth=depth,
                              n_gpus=n_gpus)
    except Exception as e:
        msg = str(e)
        if not any(k in msg for k in ("fit", "feasible", "resident", "rows cannot", "pipelined")):
            print("ERROR", c, nx, ny, steps, dt.__name__, valid, flags, depth, n_gpus, msg[:200])
            bad += 1
        skipped += 1
        continue
    got = out.data if valid is None else out.data[valid.y0:valid.y0 + valid.height + 2,
                                                  valid.x0:valid.x0 + valid.width + 2]
    ok = np.array_equal(got.astype(dt).view(np.uint64 if dt == np.float64 else np.uint32),
                        want.view(np.uint64 if dt == np.float64 else np.uint32))
    if valid is not None:  # cells outside the window are carried unchanged
        mask = np.ones_like(g.data, dtype=bool)
        mask[valid.y0 + 1:valid.y0 + valid.height + 1, valid.x0 + 1:valid.x0 + valid.width + 1] = False
        ok = ok and np.array_equal(out.data[mask].astype(dt), g.data[mask].astype(dt))
    if not ok:
        print("MISMATCH", c, nx, ny, steps, dt.__name__, valid, flags, depth, n_gpus)
        bad += 1
# device views: odd pitch / offset origin
for c in range(20):
    nx, ny = int(rng.integers(1, 400)), int(rng.integers(1, 300))
    off, extra = int(rng.integers(0, 5)), int(rng.integers(0, 9))
    dt = torch.float64 if c % 2 else torch.float32
    g = grid_new(nx, ny, random_interior(nx, ny, c), ghost=0.25)
    base = torch.zeros((ny + 2, off + nx + 2 + extra), dtype=dt, device="cuda")
    base[:, off:off + nx + 2] = torch.from_numpy(g.data).to(dt).cuda()
    dst_base = torch.zeros_like(base)
    steps = int(rng.integers(1, 30))
    w = StencilWeights(*(float(x) for x in rng.uniform(-0.7, 0.7, 5)))
    if rng.random() < 0.35:  # isotropic (w = e = s = n): the shared-product kernels
        a = float(rng.uniform(-0.7, 0.7))
        w = StencilWeights(a, a, a, float(rng.uniform(-0.7, 0.7)), a)
    j2d5pt_device(base[:, off:], dst_base[:, off:], nx, ny, w, steps)
    npdt = np.float64 if dt == torch.float64 else np.float32
    want = jacobi_c(g.data, w.astuple(), steps, npdt)
    got = dst_base[:, off:off + nx + 2].cpu().numpy()
    if not np.array_equal(got, want):
        print("VIEW MISMATCH", c, nx, ny, off, extra, dt)
        bad += 1
print(f"fuzz: {n_cases} cases ({skipped} infeasible for the forced mode) + 20 views, {bad} bad")
sys.exit(1 if bad else 0)
