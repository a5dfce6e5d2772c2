import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2306_03336_b200.engine import j2d5pt_device
from paper_2306_03336_b200.prng import fill_random_device
from paper_2306_03336_b200.grid import StencilWeights
w = StencilWeights.diffusive(0.2)
nx = ny = 256
for pitch in (272, 288):
    a = torch.empty((ny + 2, pitch), dtype=torch.float64, device="cuda"); b = torch.empty_like(a)
    fill_random_device(a, nx, ny, 1)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    for _ in range(3): j2d5pt_device(a, b, nx, ny, w, 100)
    torch.cuda.synchronize()
    for mode in ("bench", "bench_sleep", "sync_each"):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        if mode == "bench_sleep": torch.cuda._sleep(10_000_000)
        for i in range(10):
            flush.fill_(i)
            ev[i][0].record(); j2d5pt_device(a, b, nx, ny, w, 100); ev[i][1].record()
            if mode == "sync_each": torch.cuda.synchronize()
        torch.cuda.synchronize()
        ms = [s.elapsed_time(e) * 1e3 for s, e in ev]
        print(pitch, mode, [round(x) for x in ms])
