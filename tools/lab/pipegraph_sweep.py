"""Small-batch pipelined schedule (api.DualStreamPipeline captured as api.PipelineGraph):
step time by buffer sets and streams per stage (lab).

    python tools/lab/pipegraph_sweep.py [--rollouts 1 --tokens 2048 --hidden 1024 --steps 200]
"""
import argparse
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
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--sets", default="3,6,9,12")
    ap.add_argument("--streams", default="1,2,3,4")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2505_07291_b200 import api
    from paper_2505_07291_b200.synth import synth_device
    R, T, H = args.rollouts, args.tokens, args.hidden
    offs = np.arange(R + 1, dtype=np.int64) * T
    eng = api.engine()
    prv = synth_device(R * T, H, 1000).view(torch.int16)
    val = synth_device(R * T, H, 1000, jitter_thr=3277, jitter_seed=1001).view(torch.int16)
    out = {"shape": [R, T, H], "steps": args.steps, "ms_per_step": {}}
    for nb in map(int, args.sets.split(",")):
        for ns in map(int, args.streams.split(",")):
            pipe = api.DualStreamPipeline(eng, offs, H, buffer_sets=nb, streams_per_stage=ns)
            g = api.PipelineGraph(pipe, [prv] * args.steps, [val] * args.steps)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()  # the first launch of the instantiated graph (uploads it)
            e1.record()
            torch.cuda.synchronize()
            out.setdefault("first_replay_ms_per_step", {})[f"sets{nb}_streams{ns}"] = round(
                e0.elapsed_time(e1) / args.steps, 5)
            best = 1e9
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) / args.steps)
            ok = all(bool(o.all()) for o in g.out)
            out["ms_per_step"][f"sets{nb}_streams{ns}"] = round(best, 5) if ok else f"{best:.5f} (verdicts wrong)"
            del g, pipe
    print(json.dumps(out))


if __name__ == "__main__":
    main()
