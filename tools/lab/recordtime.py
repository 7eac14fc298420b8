"""tl_record_checks at configuration-2 size (256 records x 8192 probabilities), lab timing."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2505_07291_b200 import api  # noqa: E402

R, T = 256, 8192
probs = torch.rand(R * T, dtype=torch.float64, device="cuda")
offs = np.arange(R + 1, dtype=np.int64) * T
th = api.RecordThresholds(max_len=16384)
args = (probs, offs, [64] * R, [1] * R, th)
api.record_checks(*args)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    api.record_checks(*args)
b.record()
torch.cuda.synchronize()
print(f"record_checks 256 x 8192: {a.elapsed_time(b) / 20 * 1e3:.1f} us per call (incl. host->device of small arrays)")
