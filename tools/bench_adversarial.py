"""Configuration 4 (adversarial validation) at scale, and input-dependent cost.

Two tables, one JSON line:

* ``verdicts``: a prover tensor (synthetic N(0,1) bf16) is proven once; validator
  tensors derived from it -- identical, 5 % of elements +-1 ulp, fp8 e4m3 / e5m2
  round trips, one tampered row (1 of 32 in a chunk) or one whole tampered chunk per
  rollout, another seed -- are verified against
  those proofs.  Reports the accept rate per variant and the verify time.
* ``patterns``: the streaming top-k is threshold-speculative, so its cost depends
  on the data.  For inputs built to defeat it (every value equal, magnitudes
  ascending through each chunk so every element beats the running threshold, a
  magnitude span wider than the 32-bit ranking keys, 128 spikes in zeros, heavy
  ties after an fp8 round trip) it times select, commit and verify of the same
  tensor (an honest validator: every chunk must accept).

    python tools/bench_adversarial.py [--rollouts 256 --tokens 8192 --hidden 5120]   # configs[1] shape
    python tools/bench_adversarial.py --rollouts 1 --tokens 2048 --hidden 1024        # configs[0] shape
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rollouts", type=int, default=256)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=5120)
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2505_07291_b200 import api
    from paper_2505_07291_b200.synth import synth_device

    R, T, H, C = args.rollouts, args.tokens, args.hidden, api.CHUNK
    n_rows = R * T
    offs = np.arange(R + 1, dtype=np.int64) * T
    eng = api.engine()
    plan = eng.plan(offs, H)
    dev = eng.device
    tokens = float(n_rows)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.iters

    def as_bits(t):
        return t.view(torch.int16)

    def tile_chunk(chunk_bits):
        """(C*H,) int16 pattern for one chunk -> (n_rows, H) tensor, every chunk the same."""
        reps = -(-n_rows // C)
        return chunk_bits.view(C, H).repeat(reps, 1)[:n_rows].contiguous()

    # ------------------------------------------------------------- verdict matrix
    prover = synth_device(n_rows, H, seed=1, device=dev)
    plan.select(prover)
    plan.commit()
    proofs = plan.proofs.clone()
    def tampered_rows():
        t = prover.clone()
        t[torch.arange(R, device=dev) * T + min(T - 1, T // 2)] = synth_device(R, H, seed=77, device=dev)
        return t

    def tampered_chunk():
        t = prover.clone()
        c0 = min(2 * C, max(0, T - C))
        rows = (torch.arange(R, device=dev) * T + c0)[:, None] + torch.arange(min(C, T), device=dev)[None, :]
        t[rows.reshape(-1)] = synth_device(rows.numel(), H, seed=78, device=dev)
        return t

    variants = {  # built one at a time, so configuration 2's full shape fits
        "identical": lambda: prover,
        "jitter_5pct_1ulp": lambda: synth_device(n_rows, H, seed=1, jitter_thr=3277, jitter_seed=5, device=dev),
        "fp8_e4m3": lambda: prover.to(torch.float8_e4m3fn).to(torch.bfloat16),
        "fp8_e5m2": lambda: prover.to(torch.float8_e5m2).to(torch.bfloat16),
        "tampered_row_per_rollout": tampered_rows,
        "tampered_chunk_per_rollout": tampered_chunk,
        "other_seed": lambda: synth_device(n_rows, H, seed=2, device=dev),
    }
    verdicts = {}
    for name, make in variants.items():
        v = make()
        vb = as_bits(v)
        ms = timed(lambda: plan.verify(vb, proofs))
        verdicts[name] = {
            "rollouts_accepted": int(plan.rollout_accept.sum().item()),
            "chunks_accepted_frac": float(plan.chunk_accept.float().mean().item()),
            "verify_ms": ms, "verify_tokens_per_s": tokens / ms * 1e3,
        }
        del v, vb

    # ------------------------------------------------------------- cost by pattern
    n = C * H
    i = torch.arange(n, device=dev, dtype=torch.int64)
    rng = torch.Generator(device=dev)
    rng.manual_seed(3)
    spikes = torch.zeros(n, dtype=torch.int64, device=dev)
    spikes[torch.randperm(n, device=dev, generator=rng)[:128]] = 0x4300  # 128.0
    patterns = {
        "normal": lambda: as_bits(prover),
        "massive_channels": lambda: as_bits(synth_device(n_rows, H, seed=1, dist="massive", device=dev)),
        "zeros": lambda: torch.zeros((n_rows, H), dtype=torch.int16, device=dev),
        "all_equal": lambda: torch.full((n_rows, H), 0x3F80, dtype=torch.int16, device=dev),
        "fp8_e4m3_ties": lambda: as_bits(prover.to(torch.float8_e4m3fn).to(torch.bfloat16)),
        "ascending_narrow_span": lambda: tile_chunk((0x3F80 + (i * 127) // n).to(torch.int16)),
        "ascending_wide_span": lambda: tile_chunk(((i * 0x7F7F) // n).to(torch.int16)),
        "ascending_alternating_sign": lambda: tile_chunk((((i * 0x7F7F) // n) | ((i & 1) << 15)).to(torch.int16)),
        "descending_wide_span": lambda: tile_chunk((((n - 1 - i) * 0x7F7F) // n).to(torch.int16)),
        "spikes_in_zeros": lambda: tile_chunk(spikes.to(torch.int16)),
    }
    by_pattern = {}
    for name, make in patterns.items():
        h = make()
        sel = timed(lambda: plan.select(h))
        com = timed(lambda: plan.commit())
        ver = timed(lambda: plan.verify(h))
        torch.cuda.synchronize()
        by_pattern[name] = {
            "select_ms": sel, "commit_ms": com, "verify_ms": ver,
            "prove_verify_tokens_per_s": tokens / (sel + com + ver) * 1e3,
            "honest_chunks_accepted_frac": float(plan.chunk_accept.float().mean().item()),
        }
        del h
    base = by_pattern["normal"]["select_ms"] + by_pattern["normal"]["commit_ms"] + by_pattern["normal"]["verify_ms"]
    for v in by_pattern.values():
        v["slowdown_vs_normal"] = (v["select_ms"] + v["commit_ms"] + v["verify_ms"]) / base
    print(json.dumps({
        "workload": f"{R} rollouts x {T} tokens, hidden {H}, bf16 (synthetic)",
        "timing": "serial calls, CUDA events, mean over iters", "iters": args.iters, "verdicts": verdicts, "patterns": by_pattern,
    }))


if __name__ == "__main__":
    main()
