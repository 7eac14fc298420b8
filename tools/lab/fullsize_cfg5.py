"""Lab: parity of the WHOLE configs[4] batch (1024 rollouts x 4096 tokens, hidden 8192:
2 x 68.7 GB in HBM) against the CPU oracle on sampled chunks -- the first and last chunk of
every 4th rollout plus 256 random ones: indices, values, proof bytes, verify statistics,
chunk verdicts; every rollout verdict against its chunks.  (tests/test_gpu_fullsize.py runs
a 256-rollout slice so the suite stays within one test's memory.)  One JSON line.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np
    import torch

    from fullsize_util import boundary_chunks, check_prove, check_verify, chunk_rows
    from oracle import toploc_oracle as TO
    from paper_2505_07291_b200 import api
    from paper_2505_07291_b200.synth import synth_device
    R, T, H = 1024, 4096, 8192
    offs = np.arange(R + 1, dtype=np.int64) * T
    eng = api.engine()
    plan = eng.plan(offs, H)
    prv = synth_device(R * T, H, 1000)
    plan.select(prv)
    plan.commit()
    val = synth_device(R * T, H, 1000, jitter_thr=3277, jitter_seed=1001)
    plan.verify(val)
    torch.cuda.synchronize()
    t0 = time.time()
    table = chunk_rows(offs)
    rng = np.random.default_rng(5)
    js = sorted(set(boundary_chunks(offs, every=4)) | set(rng.choice(plan.n_chunks, 256, replace=False).tolist()))
    proofs, bad_p = check_prove(prv, table, js, plan.idx, plan.bits, plan.proofs)
    st = plan.stats.cpu().numpy().view(api.STATS_DTYPE).reshape(-1)
    cacc = plan.chunk_accept.cpu().numpy()
    racc = plan.rollout_accept.cpu().numpy()
    bad_v, _ = check_verify(val, table, js, proofs, st, cacc, TO.Thresholds())
    cpr = T // 32
    roll_ok = all(bool(racc[r]) == bool(cacc[r * cpr:(r + 1) * cpr].all()) for r in range(R))
    print(json.dumps({"workload": "configs[4] whole: 1024 x 4096 tokens, hidden 8192", "n_chunks": plan.n_chunks,
                      "chunks_checked": len(js), "prove_mismatches": bad_p[:8], "verify_mismatches": bad_v[:8],
                      "rollout_verdicts_consistent": roll_ok, "rollouts_accepted": int(racc.sum()),
                      "oracle_seconds": round(time.time() - t0, 1)}))


if __name__ == "__main__":
    main()
