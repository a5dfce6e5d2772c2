"""Small solves of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2306_03336_b200 import StencilWeights, grid_new, run_dtb_b200, _native
from paper_2306_03336_b200.prng import random_interior

w = StencilWeights(0.11, -0.2, 0.37, 0.5, -0.07)
for nx, ny, steps, flags, dt in [(300, 260, 12, 0, np.float64), (300, 260, 12, 0, np.float32),
                                 (700, 300, 16, _native.FLAG_FORCE_PIPE, np.float64),
                                 (700, 300, 16, _native.FLAG_FORCE_STREAM, np.float64),
                                 (64, 64, 8, _native.FLAG_POISON, np.float64)]:
    g = grid_new(nx, ny, random_interior(nx, ny, 3))
    out, _ = run_dtb_b200(g, w, steps, flags=flags, dtype=dt)
    print(nx, ny, steps, flags, dt.__name__, float(out.data.sum()))
