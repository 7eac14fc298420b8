"""tl_commit alone on configuration 2's selection (lab): python tools/lab/committime.py [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2505_07291_b200 import api, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
R, T, H = 256, 8192, 5120
h = synth.synth_device(R * T, H, 1000, "normal")
plan = api.engine().plan(np.arange(R + 1, dtype=np.int64) * T, H)
plan.select(h)
del h
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
plan.commit()
ev[0].record()
for i in range(reps):
    plan.commit()
    ev[i + 1].record()
torch.cuda.synchronize()
t = np.array([ev[i].elapsed_time(ev[i + 1]) for i in range(reps)])
print(f"{os.environ.get('TOPLOC_B200_LIB', 'default')}: commit mean {t.mean():.4f} ms  min {t.min():.4f}  max {t.max():.4f}")
