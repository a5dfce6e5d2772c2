"""Ad-hoc timing sweep of the B200 solver over plans/depths (CUDA events)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_03336_b200 import StencilWeights, j2d5pt_device, plan_b200
from paper_2306_03336_b200 import _native
from paper_2306_03336_b200.prng import fill_random_device

def timeit(nx, ny, steps, dtype, flags=0, depth=None, reps=3):
    tdt = torch.float64 if dtype == "f64" else torch.float32
    a = torch.empty((ny + 2, (nx + 2 + 31) // 32 * 32), dtype=tdt, device="cuda"); b = torch.empty_like(a)
    fill_random_device(a, nx, ny, 1)
    w = StencilWeights.diffusive(0.2)
    j2d5pt_device(a, b, nx, ny, w, steps, flags=flags, depth=depth)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e30
    for _ in range(reps):
        s.record(); j2d5pt_device(a, b, nx, ny, w, steps, flags=flags, depth=depth); e.record()
        torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
    return best

if __name__ == "__main__":
    ap = argparse.ArgumentParser(); ap.add_argument("cases", nargs="*")
    args = ap.parse_args()
    for c in args.cases:
        nx, ny, steps, dtype, flags, depth = c.split(":")
        nx, ny, steps, flags = int(nx), int(ny), int(steps), int(flags)
        depth = int(depth) if depth != "-" else None
        p = plan_b200(nx, ny, 8 if dtype == "f64" else 4, steps, depth or 1,
                      flags | (_native.FLAG_FORCE_DEPTH if depth else 0))
        ms = timeit(nx, ny, steps, dtype, flags, depth)
        extra = {}
        if os.environ.get("DTB_TRACE") and p.mode == "streaming":
            import ctypes
            tdt = torch.float64 if dtype == "f64" else torch.float32
            a = torch.empty((ny + 2, (nx + 2 + 31) // 32 * 32), dtype=tdt, device="cuda"); b = torch.empty_like(a)
            fill_random_device(a, nx, ny, 1)
            j2d5pt_device(a, b, nx, ny, StencilWeights.diffusive(0.2), steps,
                          flags=flags | _native.FLAG_TRACE, depth=depth)
            torch.cuda.synchronize()
            buf = (ctypes.c_int64 * (8 * 2048))()
            n = min(2048, _native.lib().dtb_last_trace(buf, 8 * 2048))
            v = [list(buf[8 * i:8 * i + 8]) for i in range(n)]
            tot = [sum(x[k] for x in v) / max(n, 1) for k in range(8)]
            cyc = tot[0] + tot[1] + tot[2]
            extra = {"stream_frac": {"compute": round(tot[0] / cyc, 3), "store": round(tot[1] / cyc, 3),
                                     "load_wait": round(tot[2] / cyc, 3)},
                     "tiles_per_cta": round(tot[4], 1), "cycles_per_tile": round(cyc / max(tot[4], 1))}
        if os.environ.get("DTB_TRACE") and p.mode == "resident":
            import ctypes
            tdt = torch.float64 if dtype == "f64" else torch.float32
            a = torch.empty((ny + 2, (nx + 2 + 31) // 32 * 32), dtype=tdt, device="cuda"); b = torch.empty_like(a)
            fill_random_device(a, nx, ny, 1)
            j2d5pt_device(a, b, nx, ny, StencilWeights.diffusive(0.2), steps,
                          flags=flags | _native.FLAG_TRACE, depth=depth)
            torch.cuda.synchronize()
            buf = (ctypes.c_int64 * (8 * 2048))()
            n = min(2048, _native.lib().dtb_last_trace(buf, 8 * 2048))
            v = [list(buf[8 * i:8 * i + 8]) for i in range(n)]
            tot = [sum(x[k] for x in v) / n for k in range(8)]
            cyc = sum(tot[:4])
            extra = {"trace_frac": {k: round(tot[i] / cyc, 3) for i, k in
                                    enumerate(["compute", "publish", "wait", "refresh"])},
                     "publish_split": {"stores": round(tot[5] / cyc, 3), "barrier": round(tot[6] / cyc, 3)},
                     "cycles_per_epoch": round(cyc / max(tot[4], 1)),
                     "compute_cycles_per_step_max": round(max(x[0] for x in v) / steps),
                     "compute_cycles_per_step_min": round(min(x[0] for x in v) / steps)}
        print(json.dumps({**extra, "case": c, "ms": round(ms, 3), "us_per_step": round(1e3 * ms / steps, 3),
                          "gcells": round(nx * ny * steps / ms / 1e6, 1), "mode": p.mode,
                          "h": p.halo, "K": p.lane_elems, "tiles": [p.tiles_x, p.tiles_y],
                          "load": [p.load_w, p.load_h]}), flush=True)
