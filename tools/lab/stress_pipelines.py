"""Lab: randomized stress of the pipelined schedules -- for random batch shapes, K batches of
different data go through api.Pipeline (co-resident), api.PartitionedPipeline (green
contexts), api.DualStreamPipeline and its CUDA-graph capture (api.PipelineGraph); every
batch's rollout verdicts and the last batch's proofs must equal the serial Plan calls.
One JSON line.

    python tools/lab/stress_pipelines.py --seconds 300
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2505_07291_b200 import api
    from paper_2505_07291_b200.synth import synth_device
    eng = api.engine()
    rng = np.random.default_rng(args.seed)
    t_end = time.time() + args.seconds
    cases, bad = 0, []
    while time.time() < t_end:
        seed = int(rng.integers(1 << 30))
        r = np.random.default_rng(seed)
        H = int(r.choice([1024, 1030, 2048, 5120]))
        R = int(r.integers(1, 24))
        T = r.integers(1, int(r.choice([64, 800, 4000])), size=R)
        offs = np.concatenate([[0], np.cumsum(T)]).astype(np.int64)
        n_rows = int(offs[-1])
        if n_rows * H > 1.2e9:
            continue
        K = int(r.integers(2, 6))
        prv = [synth_device(n_rows, H, seed + k) for k in range(K)]
        val = [synth_device(n_rows, H, seed + k, jitter_thr=3277 if k % 2 else 0, jitter_seed=seed + 99)
               if k % 3 else synth_device(n_rows, H, seed + 1000 + k) for k in range(K)]
        ref = eng.plan(offs, H)
        want, want_proof = [], None
        for k in range(K):
            ref.select(prv[k])
            ref.commit()
            want.append(ref.verify(val[k]).clone())
            want_proof = ref.proofs.clone()
        torch.cuda.synchronize()
        kind = str(r.choice(["pipeline", "partition", "dual", "graph"]))
        try:
            if kind == "pipeline":
                pipe = api.Pipeline(eng, offs, H)
                got = pipe.run(prv, val)
            elif kind == "partition":
                pipe = api.PartitionedPipeline(eng, offs, H)
                got = pipe.run(prv, val)
            else:
                pipe = api.DualStreamPipeline(eng, offs, H)
                if kind == "dual":
                    got = pipe.run(prv, val)
                else:
                    got = api.PipelineGraph(pipe, prv, val).replay()
            torch.cuda.synchronize()
            ok = all(torch.equal(g.cpu(), w.cpu()) for g, w in zip(got, want))
            last = pipe.plans[(K - 1) % len(pipe.plans)].proofs
            ok = ok and torch.equal(last, want_proof)
            if hasattr(pipe, "close"):
                pipe.close()
        except Exception as e:  # noqa: BLE001 -- reported, not raised, so the sweep goes on
            ok = False
            kind += f" raised {type(e).__name__}: {e}"
        if not ok:
            bad.append({"seed": seed, "kind": kind, "H": H, "R": R, "K": K})
        cases += 1
    print(json.dumps({"cases": cases, "mismatches": bad[:20], "n_mismatches": len(bad)}))


if __name__ == "__main__":
    main()
