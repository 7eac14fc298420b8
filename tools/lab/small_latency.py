"""Per-stage latency of the small-batch path (lab probe, not product).

Each stage (select, commit, verify) of one Plan is captured alone in a CUDA graph of
REPS back-to-back launches and replayed; the per-launch time is the replay time / REPS.
A graph of REPS trivial torch kernels gives the launch floor.  Shapes: 1 to 64 chunks
at hidden 1024 (configuration 1 is 64 chunks) and 5120.

    python tools/lab/small_latency.py [--reps 50 --iters 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--shapes", default="1x32x1024,1x256x1024,1x2048x1024,1x32x5120,1x2048x5120")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2505_07291_b200 import api
    from paper_2505_07291_b200.synth import synth_device

    eng = api.engine()

    def graph_us(fn):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(args.reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(args.iters):
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / args.reps)
        return round(best, 2)

    x = torch.zeros(1, device="cuda")
    out = {"reps": args.reps, "floor_us": graph_us(lambda: x.add_(1))}
    for spec in args.shapes.split(","):
        R, T, H = map(int, spec.split("x"))
        offs = np.arange(R + 1, dtype=np.int64) * T
        prv = synth_device(R * T, H, 1000).view(torch.int16)
        val = synth_device(R * T, H, 1000, jitter_thr=3277, jitter_seed=1001).view(torch.int16)
        row = {}
        for mode, ctas in (("auto", 0), ("warp", -1)):
            plan = eng.plan(offs, H)
            plan.select(prv, ctas_per_sm=ctas)
            plan.commit()
            plan.verify(val, ctas_per_sm=ctas)
            torch.cuda.synchronize()
            row[mode] = {"select": graph_us(lambda: plan.select(prv, ctas_per_sm=ctas)),
                         "commit": graph_us(lambda: plan.commit()),
                         "verify": graph_us(lambda: plan.verify(val, ctas_per_sm=ctas))}
        row["n_chunks"] = int(plan.n_chunks)
        out[spec] = row
    print(json.dumps(out))


if __name__ == "__main__":
    main()
