"""C1 fixed cost per solve: device time of 256^2 fp64 solves of 2/100/1000
steps, back to back, after a torch L2-flush fill, and after one of the
library's own kernels (a 256 MB seeded fill)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_03336_b200.engine import j2d5pt_device
from paper_2306_03336_b200.prng import fill_random_device
from paper_2306_03336_b200.grid import StencilWeights
w = StencilWeights.diffusive(0.2)
nx = ny = 256
a = torch.empty((ny + 2, 272), dtype=torch.float64, device="cuda"); b = torch.empty_like(a)
fill_random_device(a, nx, ny, 1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
big = torch.empty((4098, 8192), dtype=torch.float64, device="cuda")
def timed(steps, between):
    ts = []
    for _ in range(12):
        between()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); j2d5pt_device(a, b, nx, ny, w, steps); e.record()
        torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return round(ts[len(ts) // 2], 1)
cases = {"none": lambda: None, "torch_fill": lambda: flush.fill_(1),
         "own_fill": lambda: fill_random_device(big, 8190, 4096, 3)}
for steps in (2, 100, 1000):
    print(steps, {k: timed(steps, f) for k, f in cases.items()}, "us")
