"""Lab: three-stream pipeline (select / commit / verify each on its own stream) vs api.Pipeline.
    python tools/lab/pipe2.py [steps]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2505_07291_b200 import _ffi, api, synth  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
R, T, H = 256, 8192, 5120
prv = synth.synth_device(R * T, H, 1000, "normal")
val = synth.synth_device(R * T, H, 1000, "normal", jitter_thr=3277, jitter_seed=1001)
offs = np.arange(R + 1, dtype=np.int64) * T
eng = api.engine()


class Pipe3:
    def __init__(self, ctas=16, side_prio=0):
        self.plans = [api.Plan(eng, offs, H), api.Plan(eng, offs, H)]
        for p in self.plans:  # verify gets its own workspace (prefix, chunk counter, speculation)
            p.ws_v = torch.empty_like(p.ws)
        self.ctas = ctas
        self.side = torch.cuda.Stream(priority=side_prio)
        self.vs = torch.cuda.Stream()

    def verify(self, pl, h, stream):
        th = api.Thresholds().to_c()
        _ffi.check(eng.lib.tl_verify_ex(h.data_ptr(), pl.offs_dev.data_ptr(), pl.n_roll, pl.n_rows, pl.H, eng.chunk,
                                        eng.topk, pl.n_chunks, pl.proofs.data_ptr(), ctypes.byref(th),
                                        pl.stats.data_ptr(), pl.chunk_accept.data_ptr(), pl.rollout_accept.data_ptr(),
                                        pl.ws_v.data_ptr(), pl.ws_v.numel(), self.ctas, stream.cuda_stream),
                   "tl_verify")

    def run(self, n):
        main = torch.cuda.current_stream()
        com = [None] * n
        ver = [None] * n
        outs = []
        for k in range(n + 1):
            if k < n:
                pl = self.plans[k % 2]
                if k >= 2:
                    main.wait_event(com[k - 2])  # idx/bits of this plan consumed
                pl.select(prv, main, self.ctas)
                e = torch.cuda.Event()
                e.record(main)
                self.side.wait_event(e)
                if k >= 2:
                    self.side.wait_event(ver[k - 2])  # proofs of this plan consumed
                pl.commit(self.side, co_resident=True)
                com[k] = torch.cuda.Event()
                com[k].record(self.side)
            if k >= 1:
                pl = self.plans[(k - 1) % 2]
                self.vs.wait_event(com[k - 1])
                self.verify(pl, val, self.vs)
                with torch.cuda.stream(self.vs):
                    outs.append(pl.rollout_accept.clone())
                ver[k - 1] = torch.cuda.Event()
                ver[k - 1].record(self.vs)
        main.wait_stream(self.vs)
        main.wait_stream(self.side)
        return outs


def timeit(fn, n):
    fn(3)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    r = fn(n)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    return ms, r


p2 = api.Pipeline(eng, offs, H)
p2h = api.Pipeline(eng, offs, H)
p2h.side = torch.cuda.Stream(priority=-1)
p3 = Pipe3(16, -1)
ref = None
for rep in range(2):
    for name, fn in (("api.Pipeline prio 0", lambda n: p2.run([prv] * n, [val] * n)),
                     ("api.Pipeline prio -1", lambda n: p2h.run([prv] * n, [val] * n)),
                     ("3-stream prio -1", p3.run)):
        ms, r = timeit(fn, steps)
        ref = r[0] if ref is None else ref
        ok = all(torch.equal(a, ref) for a in r)
        print(f"{name}: {ms:.3f} ms/step  {R * T / ms / 1e3:.1f} M tok/s  verdicts equal {ok}", flush=True)
