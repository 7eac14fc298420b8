"""Lab: select and verify on two streams of the streaming partition (verify lagging two
batches behind), the commitment on its own partition -- does letting one kernel fill the
other's tail beat api.PartitionedPipeline?  python tools/lab/pipe_dual.py [steps]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2505_07291_b200 import _ffi, api, synth  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
R, T, H = 256, 8192, 5120
prv = synth.synth_device(R * T, H, 1000, "normal")
val = synth.synth_device(R * T, H, 1000, "normal", jitter_thr=3277, jitter_seed=1001)
offs = np.arange(R + 1, dtype=np.int64) * T
eng = api.engine()
lib = eng.lib


def partition():
    sm, sc = ctypes.c_void_p(), ctypes.c_void_p()
    nm, nc = ctypes.c_int32(), ctypes.c_int32()
    _ffi.check(lib.tl_partition_create(24, ctypes.byref(sm), ctypes.byref(sc), ctypes.byref(nm), ctypes.byref(nc)),
               "partition")
    return (torch.cuda.ExternalStream(sm.value), torch.cuda.ExternalStream(sc.value))


(a_str, side), (b_str, _side2) = partition(), partition()
plans = [api.Plan(eng, offs, H) for _ in range(3)]
for p in plans:
    p.ws_v = torch.empty_like(p.ws)
th = api.Thresholds().to_c()


def verify(pl, h, st):
    _ffi.check(lib.tl_verify_ex(h.data_ptr(), pl.offs_dev.data_ptr(), pl.n_roll, pl.n_rows, pl.H, eng.chunk, eng.topk,
                                pl.n_chunks, pl.proofs.data_ptr(), ctypes.byref(th), pl.stats.data_ptr(),
                                pl.chunk_accept.data_ptr(), pl.rollout_accept.data_ptr(), pl.ws_v.data_ptr(),
                                pl.ws_v.numel(), 0, st.cuda_stream), "verify")


def run_dual(n):
    cur = torch.cuda.current_stream()
    for s in (a_str, b_str, side):
        s.wait_stream(cur)
    com, ver = [None] * n, [None] * n
    outs = []
    for k in range(n + 2):
        if k < n:
            pl = plans[k % 3]
            pl.select(prv, a_str, 0)
            e = torch.cuda.Event()
            e.record(a_str)
            side.wait_event(e)
            if k >= 3:
                side.wait_event(ver[k - 3])  # proofs of this plan read
            pl.commit(side, co_resident=False)
            com[k] = torch.cuda.Event()
            com[k].record(side)
        if k >= 2:
            j = k - 2
            b_str.wait_event(com[j])
            verify(plans[j % 3], val, b_str)
            with torch.cuda.stream(b_str):
                outs.append(plans[j % 3].rollout_accept.clone())
            ver[j] = torch.cuda.Event()
            ver[j].record(b_str)
    for s in (a_str, b_str, side):
        cur.wait_stream(s)
    return outs


def timed(fn, n):
    fn(3)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = fn(n)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n, r


pp = api.PartitionedPipeline(eng, offs, H, commit_sms=24)
for rep in range(2):
    ms1, r1 = timed(lambda n: pp.run([prv] * n, [val] * n), steps)
    ms2, r2 = timed(run_dual, steps)
    ok = all(torch.equal(x, r1[0]) for x in r2)
    print(f"PartitionedPipeline {ms1:.3f} ms/step ({R * T / ms1 / 1e3:.1f} M tok/s)   dual-stream {ms2:.3f} ms/step "
          f"({R * T / ms2 / 1e3:.1f} M tok/s)  verdicts equal {ok}", flush=True)
