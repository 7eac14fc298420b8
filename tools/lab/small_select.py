"""Eager select + commit + verify launches on one small batch (lab: a target for ncu).

    ncu --set full --import-source on -k regex:ring_stream -s 6 -c 2 -o prof python tools/lab/small_select.py 1 2048 1024
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch  # noqa: E402
from paper_2505_07291_b200 import api  # noqa: E402
from paper_2505_07291_b200.synth import synth_device  # noqa: E402

R, T, H = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (1, 2048, 1024)
offs = np.arange(R + 1, dtype=np.int64) * T
prv = synth_device(R * T, H, 1000).view(torch.int16)
val = synth_device(R * T, H, 1000, jitter_thr=3277, jitter_seed=1001).view(torch.int16)
plan = api.engine().plan(offs, H)
for _ in range(6):
    plan.select(prv)
    plan.commit()
    plan.verify(val)
torch.cuda.synchronize()
print("ok", int(plan.rollout_accept.sum()))
