"""Generate the committed golden fixtures (run HERE, where /root/reference exists).

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

* exact_golden.json   -- digests produced by the REFERENCE's own
  ``swarm.worker.rollout.build_commitments`` (rollout.py:51-68) on seeded inputs
  that any machine can regenerate (numpy default_rng / the synthetic generator),
  plus edge-value KATs.  This pins the exact-mode oracle and the GPU exact path.
* forge_golden.npz    -- hidden states and digests from the reference's own
  adversarial corpus (``swarm.validator.adversaries.Forge``, tests/test_validator.py
  fixture): honest records, the validator's prefill of them, and the
  ``wrong-model`` (stale checkpoint) records.  Used to check that the GPU exact
  path reproduces the reference's digests and verdicts, and to run the TOPLOC
  verifier on real reference activations.
* toploc_golden.json  -- outputs of the TOPLOC oracle (self-generated; parity vs
  upstream toploc is unpinned) on small seeded synthetic cases.

Nothing on the GPU box reads /root/reference; it only reads these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from swarm.worker.rollout import build_commitments as ref_build_commitments  # noqa: E402

from oracle import toploc_oracle as TO  # noqa: E402
from oracle.synth_cpu import synth_bits  # noqa: E402

EDGE_VALUES = [1e303, -1e303, float("nan"), float("inf"), float("-inf"), -0.0, 0.0, 5e-324,
               0.5e-6, 1.5e-6, 2.5e-6, -2.5e-6, 1.7976931348623157e308, 0.1234565,
               4503599627370497.0, 1e-7, -1e-7, 0.1234561, 0.1234561 + 2e-8, 123456.7654325]


def bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def exact_cases():
    cases = []
    # KATs mirrored from the reference tests (tests/test_rollout.py:48-78)
    cases.append({"name": "ones_2x2", "kind": "array", "data": np.ones((2, 2)).tolist(), "k": 32})
    cases.append({"name": "empty_0x4", "kind": "array", "data": np.zeros((0, 4)).tolist(),
                  "shape": [0, 4], "k": 32})
    cases.append({"name": "arange65x3", "kind": "array",
                  "data": (np.arange(65 * 3).reshape(65, 3) * 0.1234567).tolist(), "k": 32})
    cases.append({"name": "edge_values", "kind": "array",
                  "data": np.array(EDGE_VALUES).reshape(4, 5).tolist(), "k": 3})
    for (seed, T, H, k) in [(0, 5, 8, 32), (0, 65, 8, 32), (1, 70, 8, 32), (2, 33, 17, 32),
                            (3, 100, 64, 7), (4, 64, 64, 1), (5, 31, 5, 100), (6, 200, 130, 32)]:
        cases.append({"name": f"rng{seed}_{T}x{H}_k{k}", "kind": "rng_normal",
                      "seed": seed, "T": T, "H": H, "k": k})
    # configuration 1 shape: 2048 x 1024 bf16 from the synthetic generator, upcast to f64
    cases.append({"name": "cfg1_synth_2048x1024", "kind": "synth", "seed": 0, "row0": 0,
                  "T": 2048, "H": 1024, "dist": 0, "k": 32})
    cases.append({"name": "synth_massive_96x512", "kind": "synth", "seed": 3, "row0": 64,
                  "T": 96, "H": 512, "dist": 1, "k": 32})
    out = []
    for c in cases:
        if c["kind"] == "array":
            arr = np.array(c["data"], dtype=np.float64).reshape(c.get("shape", np.array(c["data"]).shape))
            c["data_hex"] = arr.astype("<f8").tobytes().hex()
            c["shape"] = list(arr.shape)
            del c["data"]
        elif c["kind"] == "rng_normal":
            arr = np.random.default_rng(c["seed"]).normal(size=(c["T"], c["H"]))
        else:
            arr = bits_to_f64(synth_bits(c["row0"], c["T"], c["H"], c["seed"], c["dist"]))
        c["digests"] = [d.hex() for d in ref_build_commitments(arr, c["k"])]
        c["input_sha256"] = hashlib.sha256(np.ascontiguousarray(arr, dtype="<f8").tobytes()).hexdigest()
        out.append(c)
    return out


def forge_fixture(path: str):
    """Run the reference's own Forge corpus (tests/test_validator.py:1-45 setup)."""
    from swarm.config import TOY_MODEL
    from swarm.keys import SigningKey
    from swarm.policy import init_params, sequence_logprobs
    from swarm.tasks import generate_dataset, task_for_step
    from swarm.validator.adversaries import Forge
    from swarm.validator.checks import validate_file
    from swarm.validator import CheckContext
    from swarm.worker.files import parse_rollout_file

    mcfg = TOY_MODEL
    dataset = generate_dataset(seed=10, n=64)
    key = SigningKey.from_seed(7, 0)
    params = init_params(mcfg, seed=2, scale=1.0)
    stale = params.copy()
    rng = np.random.default_rng(3)
    for a in stale.arrays():
        a += rng.normal(0, 1e-3, a.shape)
    other = init_params(mcfg, seed=77, scale=1.0)
    forge = Forge(params=params, stale_params=stale, other_params=other, mcfg=mcfg,
                  dataset=dataset, key=key, checkpoint_version=5)
    ctx = CheckContext(mcfg=mcfg, dataset=dataset, alpha=0.01, budgets=(8, 16, 24, 32),
                       group_size=4, p_low=0.005, load_checkpoint=lambda v: {5: params, 2: stale}.get(v))
    by_id = {t.task_id: t for t in dataset}
    arrays, meta = {}, []
    n = 0
    for kind in ("honest", "wrong-model"):
        for step in range(1, 6):
            blob = forge.honest(step, 0) if kind == "honest" else forge.generate(kind, step, 0)
            verdict = validate_file(blob, ctx)
            f = parse_rollout_file(blob)
            for ri, rec in enumerate(f.records):
                task = task_for_step(by_id[rec.task_id], f.step, ctx.budgets)
                # the validator's prefill under the CLAIMED checkpoint (checks.py:200)
                _, h_val = sequence_logprobs(params, mcfg, list(task.prompt_tokens), rec.output_tokens)
                # the prover's hidden states (stale params for wrong-model, Forge.wrong_model)
                _, h_prv = sequence_logprobs(params if kind == "honest" else stale, mcfg,
                                             list(task.prompt_tokens), rec.output_tokens)
                assert [d.hex() for d in ref_build_commitments(h_prv, f.commit_interval)] == rec.commitments
                arrays[f"val_{n}"] = h_val
                arrays[f"prv_{n}"] = h_prv
                meta.append({"i": n, "kind": kind, "step": step, "record": ri,
                             "commitments": rec.commitments,
                             "ref_val_digests": [d.hex() for d in ref_build_commitments(h_val, f.commit_interval)],
                             "file_verdict": verdict.result, "failed_check": verdict.failed_check})
                n += 1
    np.savez_compressed(path, **arrays)
    return meta


def toploc_cases():
    cases = []
    spec = [
        # (name, row_offsets, H, seed, dist, K, C)
        ("cfg1_2048x1024", [0, 2048], 1024, 0, 0, 128, 32),
        ("ragged_h640", [0, 45, 45, 110, 141], 640, 1, 0, 128, 32),
        ("massive_h2048", [0, 96], 2048, 2, 1, 128, 32),
        ("zeros_h256", [0, 40], 256, 0, 2, 128, 32),
        ("ones_h256", [0, 33], 256, 0, 3, 128, 32),
        ("tiny_h3", [0, 5, 37], 3, 4, 0, 128, 32),
        ("h5120_collide", [0, 32 * 40], 5120, 5, 0, 128, 32),
    ]
    for name, offs, H, seed, dist, K, C in spec:
        bits = synth_bits(0, offs[-1], H, seed, dist)
        tab, chunks = TO._chunks_of(bits, offs, C)
        idxs, vals, proofs = TO.prove_chunks(chunks, K)
        jit = synth_bits(0, offs[-1], H, seed, dist, jitter_thr=3277, jitter_seed=seed + 100)
        per = [[] for _ in range(len(offs) - 1)]
        for (r, _, _), pr in zip(tab, proofs):
            per[r].append(pr)
        stats, verdict = TO.verify_proofs(jit, offs, per, C, K)
        other = synth_bits(0, offs[-1], H, seed + 1, 0)
        wstats, wverdict = TO.verify_proofs(other, offs, per, C, K)
        cases.append({
            "name": name, "row_offsets": offs, "H": H, "seed": seed, "dist": dist, "K": K, "C": C,
            "jitter_thr": 3277, "jitter_seed": seed + 100,
            "n_chunks": len(tab),
            "moduli": [int.from_bytes(p[:2], "big") for p in proofs],
            "proofs_sha256": hashlib.sha256(b"".join(proofs)).hexdigest(),
            "first_proof": proofs[0].hex(),
            "idx_sha256": hashlib.sha256(b"".join(np.asarray(i, "<i4").tobytes() for i in idxs)).hexdigest(),
            "first_idx": [int(v) for v in idxs[0]],
            "jitter_stats": [[s.exp_mismatch, s.n_match, s.mant_sum, s.mant_median, s.accept] for s in stats],
            "jitter_verdict": verdict,
            "wrong_stats": [[s.exp_mismatch, s.n_match, s.mant_sum, s.mant_median, s.accept] for s in wstats],
            "wrong_verdict": wverdict,
        })
    return cases


if __name__ == "__main__":
    with open(os.path.join(HERE, "exact_golden.json"), "w") as f:
        json.dump(exact_cases(), f, indent=1)
    meta = forge_fixture(os.path.join(HERE, "forge_golden.npz"))
    with open(os.path.join(HERE, "forge_golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    with open(os.path.join(HERE, "toploc_golden.json"), "w") as f:
        json.dump(toploc_cases(), f, indent=1)
    print("wrote golden fixtures")
