import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, json
from paper_2306_03336_b200.engine import j2d5pt_device
from paper_2306_03336_b200.prng import fill_random_device
from paper_2306_03336_b200.planner import plan_b200
from paper_2306_03336_b200.grid import StencilWeights
w = StencilWeights.diffusive(0.2)
nx = ny = 256
a = torch.empty((ny + 2, 272), dtype=torch.float64, device="cuda"); b = torch.empty_like(a)
fill_random_device(a, nx, ny, 1)
for steps, depth in [(100, None), (10, None), (2, None), (100, 20), (100, 50), (100, 25)]:
    try:
        p = plan_b200(nx, ny, 8, steps, depth or 1, (8 if depth else 0))
    except Exception as e:
        print(steps, depth, 'plan fail', e); continue
    for _ in range(3): j2d5pt_device(a, b, nx, ny, w, steps, depth=depth)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        s.record(); j2d5pt_device(a, b, nx, ny, w, steps, depth=depth); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    t0 = time.perf_counter()
    for _ in range(10): j2d5pt_device(a, b, nx, ny, w, steps, depth=depth)
    torch.cuda.synchronize(); wall = (time.perf_counter() - t0) / 10
    print(steps, depth, p.mode, p.halo, p.ctas, p.load_w, p.load_h, 'gpu ms', round(min(ts), 4), 'wall ms', round(wall * 1e3, 4))

# host cost of one call (no sync) and the device time of back-to-back solves
for steps in (2, 100):
    torch.cuda.synchronize()
    hs = []
    for _ in range(20):
        t0 = time.perf_counter(); j2d5pt_device(a, b, nx, ny, w, steps); hs.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2_000_000)  # let the host queue run ahead of the device
    s.record()
    for _ in range(20): j2d5pt_device(a, b, nx, ny, w, steps)
    e.record(); torch.cuda.synchronize()
    print('steps', steps, 'host us/call', round(sorted(hs)[10] * 1e6, 1),
          'device us/solve back-to-back', round(s.elapsed_time(e) * 1e3 / 20, 1))
