"""CTA 0's timeline inside the ring kernels for small batches (lab; -DTL_RING_STATS=1).

    python -c "from paper_2505_07291_b200 import _build; _build.build(out=_build.OUT_DIR + '/libtoploc_ringstats.so', defines=['TL_RING_STATS=1'])"
    python tools/lab/ring_timeline.py [--shapes 1x2048x1024,1x32x5120]

REPS launches of select (then verify) captured in one CUDA graph and replayed; per launch
the globaltimer stamps of g_ring_tl (entry, roles start, first stages issued, first stage
landed, chunk end, cooperative finish barriers, done) relative to entry, medians over the
launches, and the gap from one launch's done to the next one's entry."""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2505_07291_b200 import _build  # noqa: E402

os.environ.setdefault("TOPLOC_B200_LIB", os.path.join(_build.OUT_DIR, "libtoploc_ringstats.so"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="1x32x1024,1x2048x1024,1x32x5120,1x2048x5120")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--pattern", default="normal", choices=["normal", "ascending_narrow", "ascending_wide", "zeros"])
    args = ap.parse_args()
    import torch
    from paper_2505_07291_b200 import _ffi, api
    from paper_2505_07291_b200.synth import synth_device
    lib = _ffi.load()
    lib.tl_ring_lab_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
    eng = api.engine()
    names = ["entry", "roles", "issued", "landed", "chunk_end", "coop_bar1", "coop_bar2", "done"]
    out = {}
    for spec in args.shapes.split(","):
        R, T, H = map(int, spec.split("x"))
        offs = np.arange(R + 1, dtype=np.int64) * T
        prv = synth_device(R * T, H, 1000).view(torch.int16)
        val = synth_device(R * T, H, 1000, jitter_thr=3277, jitter_seed=1001).view(torch.int16)
        if args.pattern != "normal":  # tools/bench_adversarial.py's cost patterns, every chunk alike
            n = 32 * H
            i = torch.arange(n, device="cuda", dtype=torch.int64)
            pat = {"ascending_narrow": 0x3F80 + (i * 127) // n, "ascending_wide": (i * 0x7F7F) // n,
                   "zeros": i * 0}[args.pattern].to(torch.int16)
            prv = pat.view(32, H).repeat(R * T // 32, 1).contiguous()
            val = prv
        plan = eng.plan(offs, H)
        for _ in range(3):
            plan.select(prv)
            plan.commit()
            plan.verify(val)
        torch.cuda.synchronize()
        row = {}
        for what, fn in (("select", lambda: plan.select(prv)), ("verify", lambda: plan.verify(val))):
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                fn()
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                for _ in range(args.reps):
                    fn()
            tl = np.zeros((64, 32), dtype=np.uint64)
            lib.tl_ring_lab_timeline(tl.ctypes.data, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            lib.tl_ring_lab_timeline(tl.ctypes.data, 1)
            tl = tl[:args.reps].astype(np.int64)
            rel = tl - tl[:, :1]
            rel[tl == 0] = -1
            med = {names[k]: float(np.median(rel[1:, k])) / 1e3 for k in range(8)}
            med["stages_landed_scanned"] = [[float(np.median(rel[1:, 8 + 2 * q])) / 1e3, float(np.median(rel[1:, 9 + 2 * q])) / 1e3]
                                            for q in range(12) if np.all(tl[:, 8 + 2 * q] > 0)]
            gaps = (tl[1:, 0] - tl[:-1, 7]) / 1e3 if np.all(tl[:, 7] > 0) else None
            row[what] = {"us_from_entry": med,
                         "gap_done_to_next_entry_us": float(np.median(gaps)) if gaps is not None else None,
                         "entry_to_entry_us": float(np.median(np.diff(tl[:, 0]))) / 1e3,
                         "event_us_per_launch": e0.elapsed_time(e1) * 1e3 / args.reps}
        out[spec] = row
    print(json.dumps(out))


if __name__ == "__main__":
    main()
