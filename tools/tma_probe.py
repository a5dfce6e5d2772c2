"""Debug aid: which pipe configurations fail with the TMA feed."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import numpy as np
    from oracle import jacobi_c
    from paper_2306_03336_b200 import StencilWeights, grid_new, run_dtb_b200, _native
    from paper_2306_03336_b200.prng import random_interior
    nx, ny, steps, dt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    npdt = np.float64 if dt == "f64" else np.float32
    g = grid_new(nx, ny, random_interior(nx, ny, 1))
    w = StencilWeights.diffusive(0.2)
    try:
        out, _ = run_dtb_b200(g, w, steps, flags=_native.FLAG_FORCE_PIPE, dtype=npdt)
        want = jacobi_c(g.data, w.astuple(), steps, npdt)
        ok = np.array_equal(out.data.astype(npdt), want)
        print(nx, ny, steps, dt, "ok" if ok else "MISMATCH", flush=True)
    except Exception as e:
        print(nx, ny, steps, dt, "ERROR", str(e)[:200], flush=True)
    sys.exit(0)
for case in ["1 1 8 f64", "64 48 8 f64", "64 48 1 f64", "300 257 8 f64", "300 257 17 f64",
             "1000 37 8 f64", "600 2000 16 f64", "2000 2000 8 f64", "300 257 8 f32", "2000 2000 8 f32"]:
    r = subprocess.run([sys.executable, __file__, *case.split()], capture_output=True, text=True,
                       timeout=120, env={**os.environ, "CUDA_LAUNCH_BLOCKING": "1"})
    print(r.stdout.strip() or (case, r.stderr[-300:]), flush=True)
