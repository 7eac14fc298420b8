"""Lab: where do the partitioned pipeline's extra ~0.1 ms per step go?  Times the main
(streaming) partition alone, with and without the cross-partition event waits.
    python tools/lab/partgap.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2505_07291_b200 import api, synth  # noqa: E402

R, T, H = 256, 8192, 5120
prv = synth.synth_device(R * T, H, 1000, "normal")
val = synth.synth_device(R * T, H, 1000, "normal", jitter_thr=3277, jitter_seed=1001)
offs = np.arange(R + 1, dtype=np.int64) * T
eng = api.engine()
pp = api.PartitionedPipeline(eng, offs, H, commit_sms=24)
n = 30


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def main_only(wait):
    cur = torch.cuda.current_stream()
    m, s = pp.main, pp.side
    m.wait_stream(cur)
    s.wait_stream(cur)
    for k in range(n):
        pl = pp.plans[k % 2]
        pl.select(prv, m, 0)
        if wait:
            e = torch.cuda.Event()
            e.record(m)
            s.wait_event(e)
            pl.commit(s, co_resident=False)
            e2 = torch.cuda.Event()
            e2.record(s)
            m.wait_event(e2)
        pl.verify(val, None, api.Thresholds(), m, 0)
    cur.wait_stream(m)
    cur.wait_stream(s)


print(f"partitioned pipeline.run : {timed(lambda: pp.run([prv] * n, [val] * n)):.3f} ms/step")
print(f"main partition, no commit: {timed(lambda: main_only(False)):.3f} ms/step")
print(f"main + commit serialised : {timed(lambda: main_only(True)):.3f} ms/step")
pipe = api.Pipeline(eng, offs, H)
print(f"co-resident pipeline.run : {timed(lambda: pipe.run([prv] * n, [val] * n)):.3f} ms/step")
print(f"partitioned pipeline.run : {timed(lambda: pp.run([prv] * n, [val] * n)):.3f} ms/step")
pp.close()
