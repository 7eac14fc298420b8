"""Full-size parity at BASELINE.json's named configurations (``-m gpu``, ``slow``).

The whole batch runs on the GPU; the oracle then checks sampled chunks bit for bit:
the first and last chunk of every rollout, random chunks, and -- for the adversarial
validator variants of configs[3] -- every rejected chunk (a random 1024 of them when a
variant rejects more).  Compared per chunk: top-k indices and value bits, proof bytes,
exponent mismatches, match counts, mantissa sums, means and medians, chunk verdicts;
per rollout: the verdict equals the AND of its chunks' verdicts.  This is the verdict
contract of swarm/validator/checks.py:209-213 with the TOPLOC check in place of the
digest compare.

The configs[3] verdict matrix (with ``oracle_agree`` per variant) is written to
``gpurun_out/r02_adversarial_matrix.json`` when that directory exists."""

import dataclasses
import json
import os

import numpy as np
import pytest
import torch

from fullsize_util import boundary_chunks, check_prove, check_verify, chunk_rows
from paper_2505_07291_b200 import api
from paper_2505_07291_b200.synth import synth_device

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_RANDOM = 256
MAX_REJECTED = 1024


def run_batch(R, T, H, seed=1000, dist="normal"):
    offs = np.arange(R + 1, dtype=np.int64) * T
    eng = api.engine()
    plan = eng.plan(offs, H)
    prv = synth_device(R * T, H, seed, dist)
    plan.select(prv)
    plan.commit()
    torch.cuda.synchronize()
    return offs, plan, prv


def sample(plan, offs, extra=()):
    rng = np.random.default_rng(plan.n_chunks)
    js = set(boundary_chunks(offs))
    js.update(rng.choice(plan.n_chunks, size=min(N_RANDOM, plan.n_chunks), replace=False).tolist())
    js.update(extra)
    return sorted(js)


def verify_and_check(plan, offs, prv, val, proofs_by_chunk, js_base, table, proofs=None, th=api.Thresholds()):
    """Verify the whole batch on the GPU, then check js_base plus the rejected chunks (whose
    proofs are first checked against the oracle's prove of the prover states)."""
    from oracle import toploc_oracle as TO
    plan.verify(val.view(torch.int16), proofs)
    torch.cuda.synchronize()
    st = plan.stats.cpu().numpy().view(api.STATS_DTYPE).reshape(-1)
    cacc = plan.chunk_accept.cpu().numpy()
    racc = plan.rollout_accept.cpu().numpy()
    rejected = np.nonzero(cacc == 0)[0]
    rng = np.random.default_rng(len(rejected))
    rej = rejected if rejected.size <= MAX_REJECTED else np.sort(rng.choice(rejected, MAX_REJECTED, replace=False))
    js = sorted(set(js_base) | set(rej.tolist()))
    missing = [j for j in js if j not in proofs_by_chunk]
    if missing:
        extra, bad_prove = check_prove(prv, table, missing, plan.idx, plan.bits,
                                       plan.proofs if proofs is None else proofs)
        assert not bad_prove, f"prove mismatches at chunks {bad_prove[:16]}"
        proofs_by_chunk.update(extra)
    bad, oacc = check_verify(val, table, js, proofs_by_chunk, st, cacc,
                             TO.Thresholds(th.max_exp_mismatch, th.max_mant_mean, th.max_mant_median))
    co = np.concatenate([[0], np.cumsum(-(-np.diff(offs) // 32))])
    roll_ok = all(bool(racc[r]) == bool(np.all(cacc[co[r]:co[r + 1]])) for r in range(len(offs) - 1))
    return {"chunks_checked": len(js), "rejected_chunks": int(rejected.size), "rejected_checked": int(rej.size),
            "mismatches": bad[:16], "rollout_verdicts_consistent": roll_ok,
            "rollouts_accepted": int(racc.sum()), "rollouts": int(racc.size),
            "chunks_accepted_frac": float(cacc.mean())}


def full_check(R, T, H, jitter=3277):
    offs, plan, prv = run_batch(R, T, H)
    table = chunk_rows(offs)
    js = sample(plan, offs)
    proofs_by_chunk, bad = check_prove(prv, table, js, plan.idx, plan.bits, plan.proofs)
    assert not bad, f"prove mismatches at chunks {bad[:16]}"
    val = synth_device(R * T, H, 1000, jitter_thr=jitter, jitter_seed=1001)
    res = verify_and_check(plan, offs, prv, val, proofs_by_chunk, js, table)
    assert not res["mismatches"], res
    assert res["rollout_verdicts_consistent"]
    return res, plan


def test_configs1_full_shape_sampled_against_oracle():
    """configs[1]: 256 rollouts x 8192 tokens, hidden 5120 (65536 chunks, 2 x 21.5 GB)."""
    res, plan = full_check(256, 8192, 5120)
    assert plan.n_chunks == 65536 and res["chunks_checked"] >= 512
    del plan
    torch.cuda.empty_cache()


def test_configs2_long_rollouts_sampled_against_oracle():
    """configs[2]: 64 rollouts x 32768 tokens, hidden 5120 (1024 chunks per rollout)."""
    res, plan = full_check(64, 32768, 5120)
    assert plan.n_chunks == 65536 and res["chunks_checked"] >= 380
    del plan
    torch.cuda.empty_cache()


def test_configs4_llama70b_shape_slice_sampled_against_oracle():
    """configs[4]: hidden 8192 x 4096-token rollouts, a 256-rollout slice of the 1024
    (2 x 17.2 GB; the whole configuration is the bench's, 2 x 68.7 GB)."""
    res, plan = full_check(256, 4096, 8192)
    assert plan.n_chunks == 32768 and res["chunks_checked"] >= 512
    del plan
    torch.cuda.empty_cache()


def test_configs3_adversarial_matrix_at_configs1_shape():
    """configs[3] at the configs[1] shape: one honest prover batch proven once, each
    validator variant verified against those proofs on the GPU; the oracle re-checks
    every rejected chunk (up to 1024), the rollout boundaries and random chunks."""
    R, T, H, C = 256, 8192, 5120, 32
    offs, plan, prv = run_batch(R, T, H, seed=1)
    table = chunk_rows(offs)
    js = sample(plan, offs)
    proofs_by_chunk, bad = check_prove(prv, table, js, plan.idx, plan.bits, plan.proofs)
    assert not bad, f"prove mismatches at chunks {bad[:16]}"
    proofs = plan.proofs.clone()
    dev = prv.device
    n_rows = R * T

    def tampered_rows():
        t = prv.clone()
        t[torch.arange(R, device=dev) * T + T // 2] = synth_device(R, H, seed=77, device=dev)
        return t

    def tampered_chunk():
        t = prv.clone()
        rows = (torch.arange(R, device=dev) * T + 2 * C)[:, None] + torch.arange(C, device=dev)[None, :]
        t[rows.reshape(-1)] = synth_device(rows.numel(), H, seed=78, device=dev)
        return t

    def scaled_row():
        t = prv.clone()
        r = torch.arange(R, device=dev) * T + 5
        t[r] = (t[r].float() * 1.5).to(torch.bfloat16)
        return t

    def swapped_chunks():
        t = prv.clone()
        a = (torch.arange(R, device=dev) * T)[:, None] + torch.arange(C, device=dev)[None, :]
        b = a + C
        ta, tb = t[a.reshape(-1)].clone(), t[b.reshape(-1)].clone()
        t[a.reshape(-1)], t[b.reshape(-1)] = tb, ta
        return t

    variants = {
        "identical": lambda: prv,
        "jitter_5pct_1ulp": lambda: synth_device(n_rows, H, seed=1, jitter_thr=3277, jitter_seed=5, device=dev),
        "fp8_e4m3": lambda: prv.to(torch.float8_e4m3fn).to(torch.bfloat16),
        "fp8_e5m2": lambda: prv.to(torch.float8_e5m2).to(torch.bfloat16),
        "tampered_row_per_rollout": tampered_rows,
        "scaled_row_per_rollout": scaled_row,
        "tampered_chunk_per_rollout": tampered_chunk,
        "swapped_chunks_per_rollout": swapped_chunks,
        "zero_chunk_per_rollout": lambda: _zero_first_chunk(prv, R, T, C),
        "other_seed": lambda: synth_device(n_rows, H, seed=2, device=dev),
    }
    matrix = {}
    for name, make in variants.items():
        val = make()
        res = verify_and_check(plan, offs, prv, val, dict(proofs_by_chunk), js, table, proofs=proofs)
        res["oracle_agree"] = not res["mismatches"] and res["rollout_verdicts_consistent"]
        matrix[name] = res
        del val
        torch.cuda.empty_cache()
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "r02_adversarial_matrix.json"), "w") as f:
            json.dump({"workload": f"configs[3] at the configs[1] shape: {R} rollouts x {T} tokens, hidden {H}",
                       "thresholds": dataclasses.asdict(api.Thresholds()),
                       "prove_chunks_checked": len(js), "variants": matrix}, f, indent=1)
    assert all(v["oracle_agree"] for v in matrix.values()), {k: v["mismatches"] for k, v in matrix.items()}
    assert matrix["identical"]["rollouts_accepted"] == R and matrix["other_seed"]["rollouts_accepted"] == 0


def _zero_first_chunk(prv, R, T, C):
    t = prv.clone()
    rows = (torch.arange(R, device=prv.device) * T)[:, None] + torch.arange(C, device=prv.device)[None, :]
    t[rows.reshape(-1)] = 0
    return t


def test_configs4_whole_batch_sampled_against_oracle():
    """configs[4] whole: 1024 rollouts x 4096 tokens, hidden 8192 -- 2 x 68.7 GB in HBM
    (skipped when the device has less than 150 GB free)."""
    torch.cuda.empty_cache()
    if torch.cuda.mem_get_info()[0] < 150e9:
        pytest.skip("needs 150 GB of free device memory")
    res, plan = full_check(1024, 4096, 8192)
    assert plan.n_chunks == 131072 and res["chunks_checked"] >= 512
    del plan
    torch.cuda.empty_cache()
