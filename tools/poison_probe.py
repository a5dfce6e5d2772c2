"""Where does the resident poison mode disagree with the oracle? (debug aid)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import jacobi_c
from paper_2306_03336_b200 import StencilWeights, grid_new, run_dtb_b200, plan_b200, _native
from paper_2306_03336_b200.prng import random_interior
w = StencilWeights.diffusive(0.2)
for nx, ny, steps, depth in [(700, 520, 10, 2), (700, 520, 8, 4), (700, 520, 4, 2), (700, 520, 2, 2), (300, 260, 4, 2)]:
    g = grid_new(nx, ny, random_interior(nx, ny, 3), ghost=0.25)
    want = jacobi_c(g.data, w.astuple(), steps)
    p = plan_b200(nx, ny, 8, steps, depth, _native.FLAG_FORCE_DEPTH)
    for poison in (False, True):
        out, _ = run_dtb_b200(g, w, steps, depth=depth, poison=poison)
        bad = np.argwhere(out.data.view(np.uint64) != want.view(np.uint64))
        nan = np.isnan(out.data).sum()
        print(nx, ny, steps, depth, p.mode, p.tiles_x, p.tiles_y, "poison" if poison else "plain",
              "mismatch", len(bad), "nan", nan, bad[:5].tolist())
