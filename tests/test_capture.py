"""Generation-time capture of the committed hidden rows.

CPU: the hook stores, per sequence, the last prompt position of the prefill and one row
per decode step -- the rows ``policy/model.py:143-150`` commits (row t sees
prompt + output[:t]) -- and the validator's teacher-forced ``prefill_rows`` yields the
same rows.  GPU: proofs built from the capture buffer verify against the validator's
prefill, and a different model is rejected."""

import pytest
import torch

from paper_2505_07291_b200.capture import ProofCapture, prefill_rows


def tiny_llama(seed: int, H: int = 256, device="cpu"):
    from transformers import LlamaConfig, LlamaForCausalLM
    torch.manual_seed(seed)
    cfg = LlamaConfig(vocab_size=512, hidden_size=H, intermediate_size=2 * H, num_hidden_layers=2,
                      num_attention_heads=4, num_key_value_heads=4, max_position_embeddings=512)
    return LlamaForCausalLM(cfg).to(device=device, dtype=torch.float32).eval()


def generate_with_capture(model, prompt, T, cap):
    cap.reset()
    cap.attach(model.model.norm)
    try:
        out = model.generate(prompt, max_new_tokens=T, do_sample=False, eos_token_id=None, pad_token_id=0)
    finally:
        cap.detach()
    return out[:, prompt.shape[1]:]


def test_capture_rows_match_teacher_forced_prefill():
    model = tiny_llama(0, H=64)
    prompt = torch.randint(0, 512, (2, 7), generator=torch.Generator().manual_seed(1))
    T = 12
    cap = ProofCapture(64, max_tokens=16, batch=2, device="cpu")
    output = generate_with_capture(model, prompt, T, cap)
    assert cap.pos == T and output.shape == (2, T)
    rows, offs = cap.rows()
    assert rows.shape == (2 * T, 64) and list(offs) == [0, T, 2 * T]
    ref = prefill_rows(model, model.model.norm, prompt, output)
    # decode (KV cache) and teacher-forced prefill agree to float32 rounding; bf16 rows
    # differ in at most a few ulps -- exactly the nondeterminism TOPLOC tolerates
    diff = (rows.float() - ref.float()).abs().max().item()
    assert diff <= 0.02 * ref.float().abs().max().item()


def test_capture_bounds_and_shape_checks():
    cap = ProofCapture(8, max_tokens=2, batch=1, device="cpu")
    cap.hook(None, (), torch.zeros(1, 5, 8))
    cap.hook(None, (), torch.zeros(1, 1, 8))
    with pytest.raises(ValueError):
        cap.hook(None, (), torch.zeros(1, 1, 8))   # more rows than max_tokens
    cap.reset()
    with pytest.raises(ValueError):
        cap.hook(None, (), torch.zeros(2, 1, 8))   # wrong batch
    cap.lengths = [1]
    rows, offs = cap.rows()
    assert list(offs) == [0, 0] and rows.shape == (0, 8)


@pytest.mark.gpu
def test_capture_proves_and_verifies_on_gpu():
    from paper_2505_07291_b200 import api
    from paper_2505_07291_b200.capture import verify_rows
    H, T, B = 256, 96, 2
    model = tiny_llama(0, H=H, device="cuda").to(torch.bfloat16)
    prompt = torch.randint(0, 512, (B, 9), generator=torch.Generator().manual_seed(2)).cuda()
    cap = ProofCapture(H, max_tokens=T, batch=B)
    output = generate_with_capture(model, prompt, T, cap)
    pb = cap.prove()
    assert pb.proofs.shape == (B * T // 32, 258)
    # proofs from the capture buffer equal proofs of the same rows proven separately
    rows, offs = cap.rows()
    assert torch.equal(pb.proofs, api.engine().prove(rows, offs).proofs)
    honest = prefill_rows(model, model.model.norm, prompt, output)
    vb = verify_rows(honest, B, pb)
    assert bool(vb.rollout_accept.all())
    other = tiny_llama(1, H=H, device="cuda").to(torch.bfloat16)
    forged = prefill_rows(other, other.model.norm, prompt, output)
    assert not bool(verify_rows(forged, B, pb).rollout_accept.any())
