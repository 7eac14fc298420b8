"""Per-kernel event times for select / commit / verify in isolation and in the bench's
step order (lab): python tools/lab/seqtime.py [normal|massive]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2505_07291_b200 import api, synth  # noqa: E402

dist = sys.argv[1] if len(sys.argv) > 1 else "normal"
R, T, H = 256, 8192, 5120
prv = synth.synth_device(R * T, H, 1000, dist)
val = synth.synth_device(R * T, H, 1000, dist, jitter_thr=3277, jitter_seed=1001)
offs = np.arange(R + 1, dtype=np.int64) * T
plan = api.engine().plan(offs, H)


def timed(fn, n=5):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    for i in range(n):
        fn()
        ev[i + 1].record()
    torch.cuda.synchronize()
    return [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(n)]


print(dist, "select(prv)", timed(lambda: plan.select(prv)))
print(dist, "select(val)", timed(lambda: plan.select(val)))
plan.select(prv)
plan.commit()
print(dist, "verify(val)", timed(lambda: plan.verify(val)))
print(dist, "verify(prv)", timed(lambda: plan.verify(prv)))
s = torch.cuda.current_stream()
for it in range(4):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record(); plan.select(prv); e[1].record(); plan.commit(); e[2].record(); plan.verify(val); e[3].record()
    torch.cuda.synchronize()
    print(dist, "step", [round(e[i].elapsed_time(e[i + 1]), 3) for i in range(3)])
