"""TMEM-capped resident tiles (dtb_caps.cuh): bitwise parity against the C
oracle on capped plans, counted == modelled traffic, then C2 timing of the
capped depths against the default plan. Run with DTB_CAPS=1 on a B200."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import jacobi_c
from paper_2306_03336_b200 import StencilWeights, grid_new, j2d5pt_device, plan_b200, run_dtb_b200
from paper_2306_03336_b200 import _native
from paper_2306_03336_b200.prng import fill_random_device, random_interior

W02 = StencilWeights.diffusive(0.2)
MIXED = StencilWeights(0.11, -0.2, 0.37, 0.5, -0.07)


def fields(r):
    return (r.global_load_cells, r.global_store_cells, r.halo_exchanged_cells,
            r.redundant_compute_cells, r.useful_compute_cells)


def parity(nx, ny, steps, depth, dt, w):
    elem = 8 if dt == np.float64 else 4
    p = plan_b200(nx, ny, elem, steps, depth, _native.FLAG_FORCE_DEPTH)
    g = grid_new(nx, ny, random_interior(nx, ny, nx * 7 + ny), ghost=0.25)
    out, rep = run_dtb_b200(g, w, steps, depth=depth, dtype=dt)
    out_c, cnt = run_dtb_b200(g, w, steps, depth=depth, dtype=dt, count=True)
    want = jacobi_c(g.data, w.astuple(), steps, dt)
    u = np.uint64 if dt == np.float64 else np.uint32
    ok = np.array_equal(out.data.astype(dt).view(u), want.view(u))
    ok_c = np.array_equal(out_c.data.astype(dt).view(u), want.view(u))
    bad = int(np.sum(out.data.astype(dt).view(u) != want.view(u)))
    print(json.dumps({"case": [nx, ny, steps, depth, elem], "mode": p.mode, "h": p.halo,
                      "tiles": [p.tiles_x, p.tiles_y], "load_h": p.load_h,
                      "tmem_rows": p.tmem_rows, "bitwise": ok, "bitwise_counted": ok_c,
                      "mismatches": bad, "counted_eq_model": fields(cnt) == fields(rep)}),
          flush=True)
    return ok and ok_c and fields(cnt) == fields(rep)


def timeit(nx, ny, steps, depth, reps=3):
    a = torch.empty((ny + 2, (nx + 2 + 31) // 32 * 32), dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    fill_random_device(a, nx, ny, 1)
    j2d5pt_device(a, b, nx, ny, W02, steps, depth=depth)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e30
    for _ in range(reps):
        s.record()
        j2d5pt_device(a, b, nx, ny, W02, steps, depth=depth)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    p = plan_b200(nx, ny, 8, steps, depth or 1, _native.FLAG_FORCE_DEPTH if depth else 0)
    print(json.dumps({"c2": [nx, ny, steps], "depth": depth, "mode": p.mode, "h": p.halo,
                      "tiles": [p.tiles_x, p.tiles_y], "tmem_rows": p.tmem_rows,
                      "ms": round(best, 3), "gcells": round(nx * ny * steps / best / 1e6, 1)}),
          flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    good = True
    if what in ("all", "parity"):
        for case in [(1900, 1900, 24, 8, np.float64, W02), (1900, 1900, 23, 8, np.float64, MIXED),
                     (1900, 1900, 40, 6, np.float64, W02), (1900, 1900, 30, 10, np.float64, MIXED),
                     (1500, 1700, 33, 8, np.float64, W02), (2700, 2700, 24, 8, np.float32, W02),
                     (2700, 2300, 17, 6, np.float32, MIXED)]:
            good &= parity(*case)
        print("PARITY", "OK" if good else "FAIL", flush=True)
    if what in ("all", "time") and good:
        timeit(1900, 1900, 10000, None)
        for d in (6, 8, 10):
            timeit(1900, 1900, 10000, d)
        timeit(1900, 1900, 10000, None)
