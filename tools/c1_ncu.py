import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_03336_b200.engine import j2d5pt_device
from paper_2306_03336_b200.prng import fill_random_device
from paper_2306_03336_b200.grid import StencilWeights
w = StencilWeights.diffusive(0.2)
a = torch.empty((258, 272), dtype=torch.float64, device="cuda"); b = torch.empty_like(a)
fill_random_device(a, 256, 256, 1)
for steps in (100, 100, 2, 2):
    j2d5pt_device(a, b, 256, 256, w, steps)
torch.cuda.synchronize()
