"""Verdict-threshold calibration on transformer activations.

A random-init Llama-shaped model at hidden 5120 (no checkpoints are reachable here, so the
weights are the architecture's default initialisation) generates rollouts with the
generation-time capture hook (capture.py); the captured last-layer rows are proven on the
GPU.  Validators then recompute the rows with one teacher-forced prefill under honest and
dishonest conditions, and every chunk's verify statistics (exponent mismatches, mantissa
mean and median) are collected:

  honest:   prefill at the prover's batch size (prefill vs decode kernels differ), each
            sequence prefilled alone (other GEMM shapes), the math SDPA backend, the
            fp32-accumulating model (bf16 weights upcast; a different precision path)
  forgery:  fp8-e4m3 weights (per-tensor scale), weights perturbed by 1 % of their std,
            another seed's model, one decoder layer fewer

Prints one JSON line: per scenario the distribution of each statistic (percentiles), the
rollout/chunk acceptance at the current defaults, and the thresholds the data supports.

    python tools/calibrate_thresholds.py [--batch 16 --new-tokens 512 --layers 8]
"""
import argparse
import dataclasses
import copy
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--prompt", type=int, default=64)
    ap.add_argument("--new-tokens", type=int, default=512)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--hidden", type=int, default=5120)
    args = ap.parse_args()
    import numpy as np
    import torch
    from torch.nn.attention import SDPBackend, sdpa_kernel
    from transformers import LlamaConfig, LlamaForCausalLM

    from paper_2505_07291_b200 import api
    from paper_2505_07291_b200.capture import ProofCapture, prefill_rows

    H, B, T = args.hidden, args.batch, args.new_tokens

    def make(seed, layers=args.layers):
        torch.manual_seed(seed)
        cfg = LlamaConfig(vocab_size=32000, hidden_size=H, intermediate_size=int(2.7 * H) // 256 * 256,
                          num_hidden_layers=layers, num_attention_heads=H // 128, num_key_value_heads=8,
                          max_position_embeddings=4096)
        return LlamaForCausalLM(cfg).to(device="cuda", dtype=torch.bfloat16).eval()

    model = make(0)
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    prompt = torch.randint(0, 32000, (B, args.prompt), device="cuda", generator=g)
    cap = ProofCapture(H, max_tokens=T, batch=B)
    cap.attach(model.model.norm)
    torch.manual_seed(2)
    with torch.no_grad():
        out = model.generate(prompt, max_new_tokens=T, do_sample=True, temperature=1.0, top_k=0, top_p=1.0,
                             eos_token_id=None, pad_token_id=0)
    cap.detach()
    output = out[:, prompt.shape[1]:]
    eng = api.engine()
    proofs = cap.prove()
    offs = np.arange(B + 1, dtype=np.int64) * T
    # thresholds that accept everything, so the statistics come back for every chunk
    th_all = api.Thresholds(max_exp_mismatch=1 << 30, max_mant_mean=1e300, max_mant_median=1e300)

    def stats_of(rows):
        vb = eng.verify(rows, offs, proofs, th_all)
        return vb.stats_host()

    @torch.no_grad()
    def rows_of(m, per_sequence=False, math_sdpa=False, fp32=False):
        mm = m
        if fp32:
            mm = copy.deepcopy(m).float()
        ctx = sdpa_kernel([SDPBackend.MATH]) if math_sdpa else torch.nn.attention.sdpa_kernel(
            [SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION, SDPBackend.CUDNN_ATTENTION,
             SDPBackend.MATH])
        with ctx:
            if per_sequence:
                r = torch.cat([prefill_rows(mm, mm.model.norm, prompt[b:b + 1], output[b:b + 1]) for b in range(B)])
            else:
                r = prefill_rows(mm, mm.model.norm, prompt, output)
        if fp32:
            del mm
            torch.cuda.empty_cache()
        return r.to(torch.bfloat16).contiguous()

    def fp8_weights(m):
        q = copy.deepcopy(m)
        with torch.no_grad():
            for mod in q.modules():
                if isinstance(mod, torch.nn.Linear):
                    w = mod.weight.float()
                    s = w.abs().amax().clamp_min(1e-12) / 448.0
                    mod.weight.copy_(((w / s).to(torch.float8_e4m3fn).float() * s).to(mod.weight.dtype))
        return q

    def perturbed(m, rel):
        q = copy.deepcopy(m)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(7)
        with torch.no_grad():
            for p in q.parameters():
                if p.dim() >= 2:
                    p.add_((torch.randn(p.shape, device=p.device, generator=gen) * p.float().std() * rel).to(p.dtype))
        return q

    scenarios = {}
    scenarios["honest_prefill_same_batch"] = stats_of(rows_of(model))
    scenarios["honest_prefill_per_sequence"] = stats_of(rows_of(model, per_sequence=True))
    scenarios["honest_math_sdpa"] = stats_of(rows_of(model, math_sdpa=True))
    scenarios["honest_fp32_model"] = stats_of(rows_of(model, fp32=True))
    m8 = fp8_weights(model)
    scenarios["forgery_fp8_e4m3_weights"] = stats_of(rows_of(m8))
    del m8
    mp = perturbed(model, 0.01)
    scenarios["forgery_weights_perturbed_1pct"] = stats_of(rows_of(mp))
    del mp
    torch.cuda.empty_cache()
    other = make(99)
    scenarios["forgery_other_seed_model"] = stats_of(rows_of(other))
    del other
    torch.cuda.empty_cache()
    fewer = copy.deepcopy(model)
    fewer.model.layers = fewer.model.layers[:-1]
    fewer.config.num_hidden_layers -= 1
    scenarios["forgery_one_layer_fewer"] = stats_of(rows_of(fewer))
    del fewer

    # the benchmarks' validator model on synthetic N(0,1) states: 5 % of elements +-1 ulp
    from paper_2505_07291_b200.synth import synth_device
    sp = synth_device(B * T, H, 1000)
    sv = synth_device(B * T, H, 1000, jitter_thr=3277, jitter_seed=1001)
    sproofs = eng.prove(sp, offs)
    scenarios["honest_synthetic_jitter_5pct_1ulp"] = eng.verify(sv, offs, sproofs, th_all).stats_host()
    scenarios["forgery_synthetic_fp8_e4m3_roundtrip"] = eng.verify(
        sp.to(torch.float8_e4m3fn).to(torch.bfloat16), offs, sproofs, th_all).stats_host()

    def dist(x):
        x = np.asarray(x, dtype=np.float64)
        x = x[np.isfinite(x)] if x.size else x
        if x.size == 0:
            return None
        q = np.percentile(x, [0, 0.1, 1, 10, 50, 90, 99, 99.9, 100])
        return dict(zip(["min", "p0.1", "p1", "p10", "p50", "p90", "p99", "p99.9", "max"], [float(v) for v in q]))

    def accept(st, th):
        ok = (st["exp_mismatch"] <= th.max_exp_mismatch) & (st["mant_mean"] <= th.max_mant_mean) & \
             (st["mant_median"] <= th.max_mant_median)
        per_roll = ok.reshape(B, -1).all(axis=1)
        return {"chunks": float(ok.mean()), "rollouts": f"{int(per_roll.sum())}/{B}"}

    honest = {k: v for k, v in scenarios.items() if k.startswith("honest") and "synthetic" not in k}
    forged = {k: v for k, v in scenarios.items() if k.startswith("forgery")}
    # supported thresholds: the honest maxima with head-room (x1.5 + 2), checked against the forgeries
    hmax = {f: max(float(np.max(v[f])) for v in honest.values()) for f in ("exp_mismatch", "mant_mean", "mant_median")}
    proposal = api.Thresholds(max_exp_mismatch=int(np.ceil(hmax["exp_mismatch"] * 1.5 + 2)),
                              max_mant_mean=float(np.ceil(hmax["mant_mean"] * 1.5 + 2)),
                              max_mant_median=float(np.ceil(hmax["mant_median"] * 1.5 + 2)))
    out = {"model": f"random-init Llama, hidden {H}, {args.layers} layers, vocab 32000, bf16",
           "rollouts": B, "tokens_per_rollout": T, "chunks_per_scenario": int(B * T // 32),
           "defaults": dataclasses.asdict(api.Thresholds()),
           "paper": dataclasses.asdict(api.Thresholds.paper()),
           "honest_maxima": hmax,
           "supported_thresholds": {"max_exp_mismatch": proposal.max_exp_mismatch,
                                    "max_mant_mean": proposal.max_mant_mean,
                                    "max_mant_median": proposal.max_mant_median,
                                    "rule": "honest maximum x 1.5 + 2, rounded up"},
           "scenarios": {}}
    for k, st in scenarios.items():
        out["scenarios"][k] = {
            "exp_mismatch": dist(st["exp_mismatch"]), "mant_mean": dist(st["mant_mean"]),
            "mant_median": dist(st["mant_median"]),
            "accept_at_defaults": accept(st, api.Thresholds()), "accept_at_supported": accept(st, proposal),
            "accept_at_paper": accept(st, api.Thresholds.paper())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
