"""Generation-time proving overhead: a random-init Llama-shaped model at
hidden 5120 generates a batch greedily with and without the ProofCapture hook; the
captured rows are proven on the GPU and verified against a teacher-forced prefill.

    python tools/bench_capture.py [--batch 16 --new-tokens 256 --layers 2]

Prints one JSON line (generation time with / without capture, prove time, verdicts)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--prompt", type=int, default=64)
    ap.add_argument("--new-tokens", type=int, default=256)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--hidden", type=int, default=5120)
    args = ap.parse_args()
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    from paper_2505_07291_b200 import api
    from paper_2505_07291_b200.capture import ProofCapture, prefill_rows, verify_rows

    torch.manual_seed(0)
    H = args.hidden
    cfg = LlamaConfig(vocab_size=32000, hidden_size=H, intermediate_size=int(2.7 * H) // 256 * 256,
                      num_hidden_layers=args.layers, num_attention_heads=H // 128, num_key_value_heads=8,
                      max_position_embeddings=4096)
    model = LlamaForCausalLM(cfg).to(device="cuda", dtype=torch.bfloat16).eval()
    B, T = args.batch, args.new_tokens
    prompt = torch.randint(0, 32000, (B, args.prompt), device="cuda")

    def generate(cap):
        if cap is not None:
            cap.reset()
            cap.attach(model.model.norm)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = model.generate(prompt, max_new_tokens=T, do_sample=False, eos_token_id=None, pad_token_id=0)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if cap is not None:
            cap.detach()
        return out[:, prompt.shape[1]:], dt

    cap = ProofCapture(H, max_tokens=T, batch=B)
    generate(None)  # warm-up
    _, t_plain = generate(None)
    output, t_cap = generate(cap)
    _, t_plain2 = generate(None)
    eng = api.engine()
    pb = cap.prove()  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        pb = cap.prove()
    torch.cuda.synchronize()
    t_prove = (time.perf_counter() - t0) / 10
    honest = prefill_rows(model, model.model.norm, prompt, output)
    vb = verify_rows(honest, B, pb, eng=eng)
    base = min(t_plain, t_plain2)
    print(json.dumps({
        "model": f"random-init Llama, hidden {H}, {args.layers} layers, vocab 32000 (bf16)",
        "batch": B, "new_tokens": T, "generation_s": base, "generation_with_capture_s": t_cap,
        "capture_overhead_frac": (t_cap - base) / base, "prove_ms": t_prove * 1e3,
        "prove_frac_of_generation": t_prove / base, "proofs": int(pb.proofs.shape[0]),
        "verify_accept_prefill": [bool(v) for v in vb.rollout_accept.cpu().tolist()],
    }))


if __name__ == "__main__":
    main()
