"""Lab: one small exact-chain launch (128 rollouts x 64 tokens, H 5120) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2505_07291_b200.exact import build_commitments_device
R, T, H = 128, 64, 5120
x = torch.randn(R * T, H, device="cuda").to(torch.bfloat16)
offs = np.arange(R + 1) * T
build_commitments_device(x, offs, 32)
torch.cuda.synchronize()
