"""Lab: ring-kernel counters (TL_RING_STATS build) for the speculation-defeating patterns of
tools/bench_adversarial.py at a small-batch shape.

    TOPLOC_B200_LIB=build_lab/lib_stats.so python tools/lab/pattern_stats.py [--hidden 1024 --tokens 2048]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rollouts", type=int, default=1)
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--hidden", type=int, default=1024)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2505_07291_b200 import api
    from paper_2505_07291_b200.synth import synth_device
    R, T, H, C = args.rollouts, args.tokens, args.hidden, 32
    n_rows, n = R * T, C * H
    offs = np.arange(R + 1, dtype=np.int64) * T
    eng = api.engine()
    dev = eng.device
    i = torch.arange(n, device=dev, dtype=torch.int64)
    base = synth_device(n_rows, H, seed=1, device=dev).view(torch.int16)

    def tile(chunk):
        t = chunk.to(torch.int16).view(C, H).repeat(-(-n_rows // C), 1)[:n_rows].contiguous()
        return t

    pats = {"normal": base, "zeros": torch.zeros_like(base), "all_equal": torch.full_like(base, 0x3F80),
            "ascending_narrow_span": tile(0x3F80 + (i * 127) // n)}
    lab = eng.lib.tl_ring_lab_stats
    buf = (ctypes.c_ulonglong * 8)()
    out = {}
    for name, h in pats.items():
        plan = eng.plan(offs, H)
        for _ in range(3):
            plan.select(h)
        torch.cuda.synchronize()
        lab(buf, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.select(h)
        e1.record()
        torch.cuda.synchronize()
        lab(buf, 1)
        k = max(1, buf[0])
        out[name] = {"select_us": e0.elapsed_time(e1) * 1e3, "chunks": buf[0], "candidates": buf[1] / k,
                     "rescans": buf[2] / k, "compacted": buf[3] / k, "finish_us": buf[4] / k / 1.9e3}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
