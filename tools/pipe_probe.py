"""Per-stage wait fractions of the pipe kernel (build with -DDTB_PIPE_PROBE=1)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_03336_b200 import StencilWeights, j2d5pt_device, _native
from paper_2306_03336_b200.prng import fill_random_device
nx, ny, steps, dt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
tdt = torch.float64 if dt == "f64" else torch.float32
a = torch.empty((ny + 2, (nx + 2 + 31) // 32 * 32), dtype=tdt, device="cuda"); b = torch.empty_like(a)
fill_random_device(a, nx, ny, 1)
lib = _native.lib()
probe = lib.dtb_debug_pipe_probe if dt == "f64" else lib.dtb_debug_pipe_probe_f32
probe.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
buf = (ctypes.c_uint64 * 24)()
j2d5pt_device(a, b, nx, ny, StencilWeights.diffusive(0.2), steps); torch.cuda.synchronize()
probe(buf)
j2d5pt_device(a, b, nx, ny, StencilWeights.diffusive(0.2), steps); torch.cuda.synchronize()
assert probe(buf) == 0
for s in range(4):
    wi, wo, tot = buf[3 * s], buf[3 * s + 1], buf[3 * s + 2]
    print(f"stage {s}: wait_in {wi / tot:.3f}  wait_out {wo / tot:.3f}  busy {1 - (wi + wo) / tot:.3f}")
