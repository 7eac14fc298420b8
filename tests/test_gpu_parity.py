"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact bar: top-k indices, value bits, moduli, proof bytes, per-chunk
exponent-mismatch / match counts / mantissa sums and medians, accept/reject
verdicts.  The mantissa mean is compared exactly too (it is an exact integer sum
divided once in float64 on both sides; the north-star tolerance of 1e-6 relative
is asserted as the weaker bound).
"""

import hashlib
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import toploc_oracle as TO
from oracle.synth_cpu import synth_bits
from paper_2505_07291_b200 import api
from paper_2505_07291_b200.synth import synth_device

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MEAN_RTOL = 1e-6


def bits_np(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def gpu_prove(bits: np.ndarray, offs, K=128, C=32):
    eng = api.engine(chunk=C, topk=K)
    pb = eng.prove(torch.from_numpy(bits.view(np.int16)).cuda(), offs, return_indices=True)
    torch.cuda.synchronize()
    return pb


def check_prove_against_oracle(bits: np.ndarray, offs, K=128, C=32):
    pb = gpu_prove(bits, offs, K, C)
    tab, chunks = TO._chunks_of(bits, offs, C)
    idxs, vals, proofs = TO.prove_chunks(chunks, K)
    gi = pb.indices.cpu().numpy()
    gv = pb.values.cpu().numpy().view(np.uint16)
    gp = pb.proofs.cpu().numpy()
    assert gp.shape == (len(tab), 2 + 2 * K)
    for j in range(len(tab)):
        kk = len(idxs[j])
        assert np.array_equal(gi[j, :kk], idxs[j]), f"chunk {j} indices"
        assert np.all(gi[j, kk:] == -1)
        assert np.array_equal(gv[j, :kk], vals[j]), f"chunk {j} values"
        assert gp[j].tobytes() == proofs[j], f"chunk {j} proof (p={int.from_bytes(proofs[j][:2], 'big')})"
    return pb, proofs


def stats_tuple(s):
    return (int(s["exp_mismatch"]), int(s["n_match"]), int(s["mant_sum"]), float(s["mant_median"]),
            bool(s["flags"] & 1))


def check_verify_against_oracle(vbits: np.ndarray, offs, proofs_flat, th=api.Thresholds(), K=128, C=32):
    eng = api.engine(chunk=C, topk=K)
    vb = eng.verify(torch.from_numpy(vbits.view(np.int16)).cuda(), offs, proofs_flat, th)
    torch.cuda.synchronize()
    st = vb.stats_host()
    per = []
    tab = TO.chunk_table(offs, C)
    it = iter(proofs_flat)
    per = [[] for _ in range(len(offs) - 1)]
    for (r, _, _), pr in zip(tab, it):
        per[r].append(pr)
    ost, over = TO.verify_proofs(vbits, offs, per, C, K, TO.Thresholds(th.max_exp_mismatch, th.max_mant_mean,
                                                                         th.max_mant_median))
    assert len(st) == len(ost)
    for j, (g, o) in enumerate(zip(st, ost)):
        assert stats_tuple(g) == (o.exp_mismatch, o.n_match, o.mant_sum, o.mant_median, o.accept), f"chunk {j}"
        if math.isinf(o.mant_mean):
            assert math.isinf(g["mant_mean"])
        else:
            assert g["mant_mean"] == o.mant_mean
            assert abs(g["mant_mean"] - o.mant_mean) <= MEAN_RTOL * max(1.0, abs(o.mant_mean))
    assert [bool(v) for v in vb.rollout_accept.cpu().tolist()] == over
    assert [bool(v) for v in vb.chunk_accept.cpu().tolist()] == [s.accept for s in ost]
    return vb, ost, over


# ----------------------------------------------------------------------------- synth
@pytest.mark.parametrize("H,dist,jit", [(1024, 0, 0), (5120, 1, 3277), (1030, 1, 0), (7, 0, 100),
                                         (256, 2, 3277), (256, 3, 0)])
def test_synth_device_matches_cpu_twin(H, dist, jit):
    g = synth_device(70, H, seed=5, dist=dist, row0=33, jitter_thr=jit, jitter_seed=8)
    torch.cuda.synchronize()
    c = synth_bits(33, 70, H, 5, dist, jitter_thr=jit, jitter_seed=8)
    assert np.array_equal(bits_np(g), c)


# ----------------------------------------------------------------------------- prove
def golden_cases():
    with open(os.path.join(GOLDEN, "toploc_golden.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c["name"])
def test_prove_and_verify_golden(case):
    offs, H = case["row_offsets"], case["H"]
    bits = synth_bits(0, offs[-1], H, case["seed"], case["dist"])
    pb = gpu_prove(bits, offs, case["K"], case["C"])
    gp = pb.proofs.cpu().numpy()
    assert hashlib.sha256(gp.tobytes()).hexdigest() == case["proofs_sha256"]
    assert gp[0].tobytes().hex() == case["first_proof"]
    assert list(pb.indices[0, :len(case["first_idx"])].cpu().numpy()) == case["first_idx"]
    jit = synth_bits(0, offs[-1], H, case["seed"], case["dist"], jitter_thr=case["jitter_thr"],
                     jitter_seed=case["jitter_seed"])
    eng = api.engine(chunk=case["C"], topk=case["K"])
    vb = eng.verify(torch.from_numpy(jit.view(np.int16)).cuda(), offs, pb)
    st = vb.stats_host()
    assert [list(stats_tuple(s)) for s in st] == case["jitter_stats"]
    assert [bool(v) for v in vb.rollout_accept.cpu().tolist()] == case["jitter_verdict"]
    other = synth_bits(0, offs[-1], H, case["seed"] + 1, 0)
    vb = eng.verify(torch.from_numpy(other.view(np.int16)).cuda(), offs, pb)
    assert [list(stats_tuple(s)) for s in vb.stats_host()] == case["wrong_stats"]
    assert [bool(v) for v in vb.rollout_accept.cpu().tolist()] == case["wrong_verdict"]


@pytest.mark.parametrize("H,offs", [
    (1024, [0, 2048]),                     # configuration 1
    (5120, [0, 96, 96 + 45]),              # ragged, H of the north star
    (8192, [0, 64]),                       # configuration 5 hidden
    (3, [0, 1, 33, 34]),                   # chunks smaller than K
    (17, [0, 100]),                        # odd H: unaligned chunk starts
    (2047, [0, 64]),                       # idx just above 65497
])
def test_prove_matches_oracle_shapes(H, offs):
    bits = synth_bits(0, offs[-1], H, seed=H, dist=0)
    check_prove_against_oracle(bits, offs)


def test_prove_many_chunks_mixed_distributions():
    """More chunks than resident CTAs so every CTA carries its threshold speculation
    across normal, massive-activation, all-zero and all-equal chunks (speculation
    failures, overflow re-processing and tie resolution across tiles)."""
    H, C = 1024, 32
    n_chunks = 2400
    parts = []
    for j in range(n_chunks):
        d = [0, 1, 2, 3, 0, 1][j % 6] if j % 7 else 2
        parts.append(synth_bits(j * C, C, H, seed=j % 5, dist=d))
    bits = np.concatenate(parts)
    bits[5 * C + 3, 100] = 0x7FC0      # NaN
    bits[11 * C, 7] = 0xFF80           # -inf
    bits[13 * C + 31, H - 1] = 0x0001  # denormal
    offs = list(range(0, n_chunks * C + 1, C * 48))
    check_prove_against_oracle(bits, offs)


def test_speculation_state_is_only_a_hint():
    """The per-warp threshold speculation persists in the workspace between launches
    (csrc/toploc_b200.cu, spec_load/spec_store: 16-byte slots at offset 0).  Whatever
    the slots hold -- garbage, thresholds far too high (every chunk re-scanned),
    zero, or plausible values -- select and verify stay bit-exact."""
    H, C, K = 1024, 32, 128
    n_chunks = 600
    bits = np.concatenate([synth_bits(j * C, C, H, seed=j % 3, dist=[0, 1, 3][j % 3]) for j in range(n_chunks)])
    offs = list(range(0, n_chunks * C + 1, C * 40))
    _, chunks = TO._chunks_of(bits, offs, C)
    idxs, vals, proofs = TO.prove_chunks(chunks, K)
    h = torch.from_numpy(bits.view(np.int16)).cuda()
    plan = api.engine().plan(offs, H)
    slots = plan.ws[:8192 * 16].view(torch.int32).view(-1, 4)
    magic = 0x53504543
    g = torch.Generator(device="cpu").manual_seed(7)
    fills = {
        "garbage": torch.randint(-2**31, 2**31 - 1, tuple(slots.shape), generator=g, dtype=torch.int32),
        "too_high": torch.tensor([0x7FFF, 0x7FFF, 1, magic], dtype=torch.int32),
        "zero": torch.tensor([0, 0, 1, magic], dtype=torch.int32),
        "plausible": torch.tensor([0x4050, 0x4070, 40, magic], dtype=torch.int32),
    }
    for name, fill in fills.items():
        slots[:] = fill.cuda()
        plan.select(h)
        gi = plan.idx.cpu().numpy()
        gv = plan.bits.cpu().numpy().view(np.uint16)
        for j in range(n_chunks):
            assert np.array_equal(gi[j], idxs[j]) and np.array_equal(gv[j], vals[j]), f"{name}: chunk {j}"
        plan.commit()
        assert all(plan.proofs[j].cpu().numpy().tobytes() == proofs[j] for j in range(n_chunks)), name
        slots[:] = fill.cuda()
        plan.verify(h)
        assert bool(plan.chunk_accept.all()), name
        st = plan.stats.cpu().numpy().view(np.uint32).reshape(n_chunks, 8)
        assert np.all(st[:, 0] == 0) and np.all(st[:, 1] == K), name


@pytest.mark.parametrize("n", [60, 700])
def test_prove_collisions_use_fallback_primes(n):
    """60 chunks: the small-batch commitment (commit_coop_kernel); 700 (> 4 per SM): the
    table-based one-warp commitment."""
    H = 5120
    bits = synth_bits(0, 32 * n, H, seed=5, dist=0)
    _, proofs = check_prove_against_oracle(bits, [0, 32 * n])
    assert any(int.from_bytes(p[:2], "big") != 65497 for p in proofs)


# ----------------------------------------------------------------------------- verify
def flat_proofs(pb):
    return [bytes(b) for b in pb.proofs.cpu().numpy()]


@pytest.mark.parametrize("H", [1024, 5120])
def test_verify_variants_match_oracle(H):
    offs = [0, 64, 96, 160]
    bits = synth_bits(0, offs[-1], H, seed=21, dist=1)
    pb = gpu_prove(bits, offs)
    pf = flat_proofs(pb)
    t = torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)
    variants = {
        "identical": bits,
        "jitter": synth_bits(0, offs[-1], H, 21, 1, jitter_thr=3277, jitter_seed=4),
        "fp8": bits_np(t.to(torch.float8_e4m3fn).to(torch.bfloat16)),
        "scaled_row": bits.copy(),
        "tampered_row": bits.copy(),
        "swapped_chunks": bits.copy(),
        "zeros_chunk": bits.copy(),
        "other_model": synth_bits(0, offs[-1], H, 99, 1),
    }
    v = variants
    v["scaled_row"][40] = bits_np((t[40].float() * 1.5).to(torch.bfloat16).view(1, -1))[0]
    v["tampered_row"][70] = synth_bits(1000, 1, H, 3, 0)[0]
    v["swapped_chunks"][0:32], v["swapped_chunks"][32:64] = bits[32:64].copy(), bits[0:32].copy()
    v["zeros_chunk"][96:128] = 0
    for th in (api.Thresholds(), api.Thresholds(8, 2.0, 1.0), api.Thresholds(0, 0.0, 0.0)):
        for name, vb in v.items():
            check_verify_against_oracle(vb, offs, pf, th)


def _adversarial_chunk(name: str, H: int, C: int = 32) -> np.ndarray:
    """One chunk's (C, H) bits built to defeat threshold speculation (tools/bench_adversarial.py)."""
    n = C * H
    i = np.arange(n, dtype=np.int64)
    rng = np.random.default_rng(5)
    if name == "ascending_narrow_span":
        b = 0x3F80 + (i * 127) // n
    elif name == "ascending_wide_span":
        b = (i * 0x7F7F) // n
    elif name == "ascending_alternating_sign":
        b = ((i * 0x7F7F) // n) | ((i & 1) << 15)
    elif name == "descending_wide_span":
        b = ((n - 1 - i) * 0x7F7F) // n
    elif name == "spikes_in_zeros":
        b = np.zeros(n, dtype=np.int64)
        b[rng.choice(n, 128, replace=False)] = 0x4300
    elif name == "three_values":
        b = rng.choice(np.array([0x3F80, 0xBF80, 0x4000]), n)
    elif name == "fp8_e4m3_ties":
        t = torch.from_numpy(synth_bits(0, C, H, seed=4).view(np.int16)).view(torch.bfloat16)
        return bits_np(t.float().to(torch.float8_e4m3fn).to(torch.bfloat16))
    else:
        raise ValueError(name)
    return b.astype(np.uint16).reshape(C, H)


@pytest.mark.parametrize("name", ["ascending_narrow_span", "ascending_wide_span", "ascending_alternating_sign",
                                  "descending_wide_span", "spikes_in_zeros", "three_values", "fp8_e4m3_ties"])
@pytest.mark.parametrize("H", [1024, 5120])
def test_adversarial_orderings_match_oracle(name, H):
    """Inputs that defeat the threshold speculation (every element beats the running
    threshold, key spans beyond the 32-bit ranking keys, heavy ties) prove and verify
    bit-exactly; whole chunks and a ragged tail, after a normal chunk so the carried
    speculation is wrong for them."""
    pat = _adversarial_chunk(name, H)
    bits = np.concatenate([synth_bits(0, 32, H, seed=3), pat, pat, pat[:17]])
    offs = [0, 64, 96, 113]
    _, proofs = check_prove_against_oracle(bits, offs)
    check_verify_against_oracle(bits, offs, proofs)
    e5m2 = bits_np(torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).float()
                   .to(torch.float8_e5m2).to(torch.bfloat16))
    check_verify_against_oracle(e5m2, offs, proofs)


def test_verify_identical_accepts_and_wrong_rejects():
    offs = [0, 128, 256]
    bits = synth_bits(0, 256, 1024, seed=1, dist=0)
    pb = gpu_prove(bits, offs)
    eng = api.engine()
    vb = eng.verify(torch.from_numpy(bits.view(np.int16)).cuda(), offs, pb)
    assert vb.rollout_accept.cpu().tolist() == [1, 1]
    st = vb.stats_host()
    assert np.all(st["exp_mismatch"] == 0) and np.all(st["mant_sum"] == 0)
    other = synth_bits(0, 256, 1024, seed=2, dist=0)
    vb = eng.verify(torch.from_numpy(other.view(np.int16)).cuda(), offs, pb)
    assert vb.rollout_accept.cpu().tolist() == [0, 0]


def test_verify_malformed_proofs():
    offs = [0, 96]
    H = 640
    bits = synth_bits(0, 96, H, seed=3, dist=0)
    pf = flat_proofs(gpu_prove(bits, offs))
    bad = list(pf)
    bad[0] = b"\x00\x00" + pf[0][2:]                       # p = 0
    bad[1] = b"\x00\x01" + pf[1][2:]                       # p = 1
    bad[2] = pf[2][:2] + b"\xff\xff" * 128                  # coefficients >= p
    check_verify_against_oracle(bits, offs, bad)
    bad2 = list(pf)
    bad2[0] = b"\xff\xff" + pf[0][2:]                      # p = 65535 (composite)
    check_verify_against_oracle(bits, offs, bad2)


@pytest.mark.parametrize("p", [2, 3, 97, 127, 128, 32769, 32770, 65499, 65521])
def test_forged_modulus_proofs_are_bad_proofs(p):
    """A proof is only as strong as its modulus.  With p <= 128 every claimed and observed
    value is below 128, so all exponent fields are 0 and p = 2 with zero coefficients
    would pass for any activations.  Every modulus that is not one of the
    prover's primes in [32771, 65497] is a bad proof: rejected, stats at +inf."""
    offs = [0, 64, 96]
    bits = synth_bits(0, 96, 640, seed=11, dist=0)
    forged = [p.to_bytes(2, "big") + b"\x00" * 256] * 3
    vb, ost, over = check_verify_against_oracle(bits, offs, forged)
    assert over == [False, False]
    assert all((s["flags"] & 2) and math.isinf(s["mant_mean"]) for s in vb.stats_host())


def test_rollout_verdict_fails_closed_on_short_chunk_count():
    """A C-ABI caller that passes too small an n_chunks gets the uncovered chunks
    rejected (they were never verified), not accepted from stale bytes."""
    import ctypes
    from paper_2505_07291_b200 import _ffi
    lib = _ffi.load()
    H, offs = 256, np.array([0, 64, 128], dtype=np.int64)
    bits = synth_bits(0, 128, H, seed=5, dist=0)
    h = torch.from_numpy(bits.view(np.int16)).cuda()
    pf = gpu_prove(bits, offs).proofs
    od = torch.from_numpy(offs).cuda()
    need = int(lib.tl_workspace_bytes(2, 4, 128))
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    cacc = torch.ones(4, dtype=torch.uint8, device="cuda")       # stale "accept" bytes
    racc = torch.zeros(2, dtype=torch.uint8, device="cuda")
    th = api.Thresholds().to_c()
    for n_chunks, want in ((4, [1, 1]), (2, [1, 0]), (0, [0, 0])):
        cacc.fill_(1)
        rc = lib.tl_verify(h.data_ptr(), od.data_ptr(), 2, 128, H, 32, 128, n_chunks, pf.data_ptr(), ctypes.byref(th),
                           None, cacc.data_ptr(), racc.data_ptr(), ws.data_ptr(), ws.numel(), None)
        assert rc == 0
        torch.cuda.synchronize()
        assert racc.cpu().tolist() == want, n_chunks


def test_api_argument_errors():
    eng = api.engine()
    x = torch.zeros((64, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        eng.prove(x, [0, 65])
    with pytest.raises(ValueError):
        eng.verify(x, [0, 64], [b"\x00" * 257, b"\x00" * 258])
    with pytest.raises(ValueError):
        api.ToplocEngine(topk=129)
    with pytest.raises(ValueError):
        api.ToplocEngine(chunk=0)


def test_toploc_on_reference_forge_corpus():
    """TOPLOC prove / verify on the reference's own activations (tests/golden/forge_*,
    produced by swarm's Forge): honest records verify, GPU stats and verdicts equal
    the oracle's for every record, at default and exact thresholds."""
    from paper_2505_07291_b200.swarm_adapter import to_bf16_bits
    with open(os.path.join(GOLDEN, "forge_golden.json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, "forge_golden.npz"))
    eng = api.engine()
    for th in (api.Thresholds(), api.Thresholds(0, 0.0, 0.0))[:]:
        for m in meta:
            prv = to_bf16_bits(arrays[f"prv_{m['i']}"])
            val = to_bf16_bits(arrays[f"val_{m['i']}"])
            offs = [0, prv.shape[0]]
            pb = gpu_prove(prv, offs)
            assert pb.to_bytes() == TO.build_proofs(prv, offs)
            vb, ost, over = check_verify_against_oracle(val, offs, flat_proofs(pb), th)
            if m["kind"] == "honest":
                assert over == [True]


@pytest.mark.parametrize("kind", ["pipeline", "partition"])
def test_pipeline_matches_serial(kind):
    """The two-stream pipelined schedules -- commit(k) overlapping verify(k-1), either
    co-resident (16 one-warp CTAs + the half-table commitment per SM) or on separate SM
    partitions (green contexts) -- give exactly the serial results."""
    H, offs = 2048, [0, 160, 256, 320]
    n = 5
    prv = [synth_bits(400 * k, 320, H, seed=k, dist=k % 2) for k in range(n)]
    val = [synth_bits(400 * k, 320, H, seed=k, dist=k % 2, jitter_thr=3277 * (k % 3), jitter_seed=9)
           for k in range(n)]
    val[3] = synth_bits(0, 320, H, seed=77)   # a wrong model in batch 3
    dp = [torch.from_numpy(b.view(np.int16)).cuda() for b in prv]
    dv = [torch.from_numpy(b.view(np.int16)).cuda() for b in val]
    eng = api.engine()
    pipe = api.Pipeline(eng, offs, H) if kind == "pipeline" else api.PartitionedPipeline(eng, offs, H, commit_sms=16)
    outs = pipe.run(dp, dv)
    torch.cuda.synchronize()
    if kind == "partition":
        assert pipe.sms[1] >= 16 and pipe.sms[0] + pipe.sms[1] <= torch.cuda.get_device_properties(0).multi_processor_count
        assert eng.lib.tl_stream_sms(pipe.main.cuda_stream) == pipe.sms[0]
    for k in range(n):
        pb = eng.prove(dp[k], offs)
        vb = eng.verify(dv[k], offs, pb)
        assert outs[k].cpu().tolist() == vb.rollout_accept.cpu().tolist(), k
        assert pb.to_bytes() == TO.build_proofs(prv[k], offs)
    assert torch.equal(pipe.plans[(n - 1) % len(pipe.plans)].proofs, eng.prove(dp[n - 1], offs).proofs)
    assert outs[3].cpu().tolist() == [0, 0, 0]


def test_scheduler_verify_sharded_single_rank():
    from paper_2505_07291_b200 import scheduler
    H, offs = 1024, [0, 100, 100, 164, 300]
    prv = synth_bits(0, 300, H, seed=8)
    val = prv.copy()
    val[120:122] = synth_bits(1000, 2, H, seed=9)          # tamper rollout 2
    eng = api.engine()
    acc = scheduler.verify_sharded(eng, torch.from_numpy(prv.view(np.int16)).cuda(),
                                   torch.from_numpy(val.view(np.int16)).cuda(), offs,
                                   thresholds=api.Thresholds(0, 0.0, 0.0))
    _, want = TO.verify_proofs(val, offs, TO.build_proofs(prv, offs), th=TO.Thresholds(0, 0.0, 0.0))
    assert [bool(v) for v in acc.cpu().tolist()] == want == [True, True, False, True]


@pytest.mark.parametrize("K,C,H,offs", [(64, 32, 640, [0, 70]), (1, 32, 256, [0, 40]), (128, 16, 512, [0, 50, 77]),
                                        (17, 1, 96, [0, 9]), (128, 64, 2048, [0, 130]), (100, 8, 16384, [0, 20])])
def test_prove_verify_other_chunk_and_topk(K, C, H, offs):
    bits = synth_bits(0, offs[-1], H, seed=K + C, dist=1)
    check_prove_against_oracle(bits, offs, K=K, C=C)
    pf = [bytes(b) for b in gpu_prove(bits, offs, K, C).proofs.cpu().numpy()]
    jit = synth_bits(0, offs[-1], H, K + C, 1, jitter_thr=6000, jitter_seed=3)
    for th in (api.Thresholds(), api.Thresholds(0, 0.0, 0.0)):
        check_verify_against_oracle(jit, offs, pf, th, K=K, C=C)


# ----------------------------------------------------------------------------- record checks
def test_record_checks_match_oracle():
    """tl_record_checks (termination, sampling, commitment in the reference's order,
    checks.py:204-213) against oracle/checks_oracle.py, boundaries included."""
    from oracle import checks_oracle as CO
    rng = np.random.default_rng(11)
    probs, prompt, eos = [], [], []
    for i in range(500):
        T = int(rng.integers(0, 80)) if i else 0
        p = rng.choice([0.005, 0.0049999999, 0.1, 0.10000001, 0.5, 1e-4, 0.9], size=T) if i % 3 == 0 \
            else rng.random(T) ** 3
        probs.append(p)
        prompt.append(int(rng.integers(1, 40)))
        eos.append(int(rng.integers(0, 2)))
    probs += [np.array([0.001] * 4 + [0.5] * 12), np.array([0.001] * 5 + [0.5] * 11), np.array([0.5] * 15 + [0.1])]
    prompt += [1, 1, 1]
    eos += [1, 1, 1]
    R = len(probs)
    acc = rng.integers(0, 2, size=R)
    chk = rng.integers(0, 2, size=R)
    offs = np.concatenate([[0], np.cumsum([len(p) for p in probs])])
    th = api.RecordThresholds(max_len=64)
    verdict, frac, p_last = api.record_checks(np.concatenate(probs), offs, prompt, eos, th, acc, chk)
    want = CO.record_verdicts(probs, prompt, eos, 64, commit_accept=acc, commit_checked=chk)
    v, f, pl = verdict.cpu().numpy(), frac.cpu().numpy(), p_last.cpu().numpy()
    assert [int(x) for x in v] == [w[0] for w in want]
    assert np.array_equal(f, np.array([w[1] for w in want]))   # exact count / T, like np.mean
    for r in range(R):
        assert (np.isnan(pl[r]) and len(probs[r]) == 0) or pl[r] == probs[r][-1]


def test_step_graph_matches_eager():
    """A Plan's prove + verify captured as one CUDA graph replays to the eager results."""
    H, offs = 1024, [0, 70, 128, 2048]
    bits = synth_bits(0, offs[-1], H, seed=4, dist=1)
    jit = synth_bits(0, offs[-1], H, seed=4, dist=1, jitter_thr=3277, jitter_seed=5)
    prv = torch.from_numpy(bits.view(np.int16)).cuda()
    val = torch.from_numpy(jit.view(np.int16)).cuda()
    plan = api.engine().plan(offs, H)
    plan.select(prv)
    plan.commit()
    plan.verify(val)
    torch.cuda.synchronize()
    want_p, want_s, want_a = plan.proofs.clone(), plan.stats.clone(), plan.rollout_accept.clone()
    g = api.StepGraph(plan, prv, val)
    assert g.uploaded  # cuGraphUpload at construction: the first replay does not upload
    for _ in range(3):
        plan.proofs.zero_()
        plan.stats.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(plan.proofs, want_p) and torch.equal(plan.stats, want_s)
        assert torch.equal(plan.rollout_accept, want_a)
    _, _, proofs = TO.prove_chunks(TO._chunks_of(bits, offs, 32)[1], 128)
    assert all(plan.proofs[j].cpu().numpy().tobytes() == proofs[j] for j in range(len(proofs)))


@pytest.mark.parametrize("case", range(24))
def test_fuzz_prove_verify_small_shapes(case):
    """Seeded random shapes against the oracle: odd H (unaligned chunk starts), ragged and
    empty rollouts, chunks smaller than K, K and C away from the defaults, all value
    distributions and a jittered validator."""
    rng = np.random.default_rng(1000 + case)
    H = int(rng.choice([1, 3, 7, 17, 64, 129, 640, 1031]))
    C = int(rng.choice([1, 4, 32, 32, 32, 33]))
    K = int(rng.choice([1, 5, 64, 128, 128]))
    if C * H >= (1 << 24) - 1:
        C = 4
    lens = rng.integers(0, 3 * C + 2, size=int(rng.integers(1, 6)))
    offs = [0] + np.cumsum(lens).tolist()
    if offs[-1] == 0:
        offs[-1] = 1
    dist = int(rng.integers(0, 4))
    bits = synth_bits(0, offs[-1], H, seed=case, dist=dist)
    check_prove_against_oracle(bits, offs, K=K, C=C)
    pf = [bytes(b) for b in gpu_prove(bits, offs, K, C).proofs.cpu().numpy()]
    jit = synth_bits(0, offs[-1], H, seed=case, dist=dist, jitter_thr=int(rng.integers(0, 20000)),
                     jitter_seed=case + 7)
    check_verify_against_oracle(jit, offs, pf, K=K, C=C)


def test_many_ragged_rollouts_sampled_against_oracle():
    """8,000 ragged rollouts (1..100 tokens) at an unaligned H: ~16k
    chunks through the chunk prefix, the device-side rollout lookup and dynamic chunk
    claiming.  Every chunk's proof and stats come from the GPU; 300 sampled chunks are
    re-derived by the oracle."""
    rng = np.random.default_rng(5)
    H, R = 333, 8000
    lens = rng.integers(1, 101, size=R)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    bits = synth_bits(0, int(offs[-1]), H, seed=9, dist=1)
    jit = synth_bits(0, int(offs[-1]), H, seed=9, dist=1, jitter_thr=3277, jitter_seed=4)
    eng = api.engine()
    pb = eng.prove(torch.from_numpy(bits.view(np.int16)).cuda(), offs)
    vb = eng.verify(torch.from_numpy(jit.view(np.int16)).cuda(), offs, pb)
    torch.cuda.synchronize()
    tab = TO.chunk_table(offs, 32)
    assert pb.proofs.shape[0] == len(tab)
    proofs = pb.proofs.cpu().numpy()
    st = vb.stats_host()
    for j in sorted(rng.choice(len(tab), size=300, replace=False).tolist()):
        _, s, n = tab[j]
        _, _, want = TO.prove_chunks([bits[s:s + n].reshape(-1)], 128)
        assert proofs[j].tobytes() == want[0], f"chunk {j}"
        o = TO.verify_chunk(jit[s:s + n].reshape(-1), want[0])
        assert stats_tuple(st[j]) == (o.exp_mismatch, o.n_match, o.mant_sum, o.mant_median, o.accept), f"chunk {j}"
    # rollout verdict = AND of its chunks
    acc = vb.chunk_accept.cpu().numpy()
    co = pb.chunk_offsets
    want_r = [bool(acc[co[r]:co[r + 1]].all()) for r in range(R)]
    assert [bool(v) for v in vb.rollout_accept.cpu().tolist()] == want_r


def test_wide_chunks_rank_with_64_bit_keys():
    """Chunks of 32 x 20000 = 640,000 elements: indices past 2^19 - 1 cannot use the
    32-bit chunk-end ranking, so the kernels take the 64-bit path (plus a partial chunk)."""
    H, offs = 20000, [0, 32, 77]
    bits = synth_bits(0, offs[-1], H, seed=3, dist=1)
    check_prove_against_oracle(bits, offs)
    pf = [bytes(b) for b in gpu_prove(bits, offs).proofs.cpu().numpy()]
    jit = synth_bits(0, offs[-1], H, seed=3, dist=1, jitter_thr=3277, jitter_seed=8)
    check_verify_against_oracle(jit, offs, pf)


def test_engine_calls_on_two_streams_do_not_share_the_workspace_concurrently():
    """The engine's workspace carries the running launch's chunk counter and prefix;
    calls issued on different streams are ordered on it, so both stay exact."""
    H, offs = 2048, [0, 300, 640]
    a = synth_bits(0, 640, H, seed=21, dist=0)
    b = synth_bits(0, 640, H, seed=22, dist=1)
    ta, tb = (torch.from_numpy(x.view(np.int16)).cuda() for x in (a, b))
    eng = api.engine()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s1):
            pa = eng.prove(ta, offs)
        with torch.cuda.stream(s2):
            pb = eng.prove(tb, offs)
        torch.cuda.synchronize()
        assert pa.to_bytes() == TO.build_proofs(a, offs)
        assert pb.to_bytes() == TO.build_proofs(b, offs)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_partitioned_pipeline_short_runs(n):
    """Fill and drain of the dual-stream partitioned schedule (verify two batches behind
    select, three buffer sets) for runs shorter than, equal to and just past the lag."""
    H, offs = 1024, [0, 96, 200]
    prv = [synth_bits(300 * k, 200, H, seed=30 + k, dist=k % 2) for k in range(n)]
    val = [synth_bits(300 * k, 200, H, seed=30 + k, dist=k % 2, jitter_thr=3277, jitter_seed=k) for k in range(n)]
    dp = [torch.from_numpy(b.view(np.int16)).cuda() for b in prv]
    dv = [torch.from_numpy(b.view(np.int16)).cuda() for b in val]
    eng = api.engine()
    pipe = api.PartitionedPipeline(eng, offs, H, commit_sms=16)
    outs = pipe.run(dp, dv)
    torch.cuda.synchronize()
    assert len(outs) == n
    for k in range(n):
        vb = eng.verify(dv[k], offs, eng.prove(dp[k], offs))
        assert outs[k].cpu().tolist() == vb.rollout_accept.cpu().tolist(), k
    pipe.close()


def test_cross_process_determinism():
    """Proof bytes, per-chunk statistics and verdicts are a pure function of the input:
    a fresh process (fresh speculation state, other grid timing) reproduces them bit for
    bit (the reference's cross-process check, tests/test_policy.py:124-139)."""
    import subprocess
    import sys
    code = r'''
import hashlib, numpy as np, torch
from paper_2505_07291_b200 import api
from paper_2505_07291_b200.synth import synth_device
offs = np.array([0, 300, 300, 1024, 2048], dtype=np.int64)
eng = api.engine()
h = synth_device(2048, 5120, seed=4, dist="massive")
v = synth_device(2048, 5120, seed=4, dist="massive", jitter_thr=3277, jitter_seed=9)
pb = eng.prove(h, offs)
vb = eng.verify(v, offs, pb)
torch.cuda.synchronize()
d = hashlib.sha256()
for t in (pb.proofs, vb.stats, vb.chunk_accept, vb.rollout_accept):
    d.update(t.cpu().numpy().tobytes())
print(d.hexdigest())
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = [subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
            for _ in range(2)]
    for r in runs:
        assert r.returncode == 0, r.stderr[-2000:]
    digests = [r.stdout.strip().splitlines()[-1] for r in runs]
    local = {}
    exec(code.replace("print(d.hexdigest())", "local['d'] = d.hexdigest()"), {"local": local})
    assert digests[0] == digests[1] == local["d"]


@pytest.mark.parametrize("H,C,K,offs", [
    (2048, 32, 128, [0, 32, 65, 97]),        # 4 parts per chunk, a 1-row chunk
    (8192, 32, 128, [0, 33, 64]),            # 5 parts per chunk
    (16, 8192, 128, [0, 8197]),              # 5 parts; the 5-row tail chunk has parts < K and empty parts
    (5120, 32, 5, [0, 40, 41]),              # 5 parts, K = 5
    (1024, 32, 128, [0, 64, 100]),           # configuration 1's shape: 2 parts
])
def test_split_chunks_match_oracle(H, C, K, offs):
    """Small batches split each chunk over several warps (csrc select_split: up to 5 parts
    of >= 16K elements, the last part merges the partial top-k lists).  Bit-exact against
    the oracle for prove and verify, including parts smaller than K and empty parts."""
    bits = synth_bits(0, offs[-1], H, seed=H + C + K, dist=1)
    _, proofs = check_prove_against_oracle(bits, offs, K=K, C=C)
    jit = synth_bits(0, offs[-1], H, seed=H + C + K, dist=1, jitter_thr=3277, jitter_seed=2)
    check_verify_against_oracle(jit, offs, proofs, K=K, C=C)
    check_verify_against_oracle(bits, offs, proofs, K=K, C=C)


@pytest.mark.parametrize("case", range(16))
def test_fuzz_split_chunks(case):
    """Seeded random small batches of wide chunks, so the kernels split chunks over
    several warps (odd H, C and K away from the defaults, ragged rollouts, all value
    distributions, a jittered validator) -- against the oracle."""
    rng = np.random.default_rng(5000 + case)
    H = int(rng.choice([2048, 3001, 4096, 5120, 8192]))
    C = int(rng.choice([16, 32, 32]))
    K = int(rng.choice([1, 64, 128, 128]))
    lens = rng.integers(1, 2 * C + 9, size=int(rng.integers(1, 4)))
    offs = [0] + np.cumsum(lens).tolist()
    dist = int(rng.integers(0, 4))
    bits = synth_bits(0, offs[-1], H, seed=case, dist=dist)
    _, proofs = check_prove_against_oracle(bits, offs, K=K, C=C)
    jit = synth_bits(0, offs[-1], H, seed=case, dist=dist, jitter_thr=int(rng.integers(0, 20000)),
                     jitter_seed=case + 3)
    check_verify_against_oracle(jit, offs, proofs, K=K, C=C)


def test_pipeline_graph_matches_serial():
    """api.DualStreamPipeline captured as one CUDA graph (api.PipelineGraph): each batch's
    verdicts equal the serial Plan calls, batches with different verdicts included, and
    the graph replays with refreshed inputs."""
    H, offs = 2048, [0, 40, 96, 130]
    eng = api.engine()
    plan = eng.plan(offs, H)
    n = 5
    prv = [torch.from_numpy(synth_bits(0, offs[-1], H, seed=10 + k, dist=k % 2).view(np.int16)).cuda()
           for k in range(n)]
    val = [p.clone() for p in prv]
    val[1][40:72] = torch.from_numpy(synth_bits(0, 32, H, seed=99).view(np.int16)).cuda()  # a chunk of rollout 1
    val[3] = torch.from_numpy(synth_bits(0, offs[-1], H, seed=77).view(np.int16)).cuda()   # another model
    want = []
    for k in range(n):
        plan.select(prv[k])
        plan.commit()
        want.append(plan.verify(val[k]).clone())
    pipe = api.DualStreamPipeline(eng, offs, H)
    assert len(pipe.plans) == 12 and len(pipe.vstreams) == 4  # 3 chunks: the small-batch shape
    pg = api.PipelineGraph(pipe, prv, val)
    assert pg.uploaded
    for _ in range(2):
        got = pg.replay()
        torch.cuda.synchronize()
        assert [g.tolist() for g in got] == [w.tolist() for w in want]
    assert want[1].tolist() == [1, 0, 1] and want[3].tolist() == [0, 0, 0]
    # inputs refreshed in place are picked up by the next replay
    val[0].copy_(val[3])
    got = pg.replay()
    torch.cuda.synchronize()
    assert got[0].tolist() == [0, 0, 0]
    pipe.close()


def test_first_commits_on_two_streams_without_prepare_build_correct_tables():
    """The inverse tables are built by the first tl_commit when tl_prepare was not called.
    Two first calls racing on two streams of a fresh process must both produce the oracle's
    proofs (the ready flag rises only when every table piece was written).  640 chunks per
    call: more than 4 per SM, so the table-based commitment (not commit_coop_kernel) runs."""
    import subprocess
    import sys
    code = r'''
import ctypes, numpy as np, torch
from oracle import toploc_oracle as TO
from oracle.synth_cpu import synth_bits
from paper_2505_07291_b200 import _ffi
L = _ffi.load()                       # no ToplocEngine: tl_prepare is never called
H, T = 256, 32 * 640
offs = np.array([0, T], dtype=np.int64)
assert T // 32 > 4 * int(L.tl_stream_sms(None))
outs = []
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
bits = [synth_bits(0, T, H, seed=s, dist=1) for s in (1, 2)]
for s, b in zip(streams, bits):
    h = torch.from_numpy(b.view(np.int16)).cuda()
    od = torch.from_numpy(offs).cuda()
    n = T // 32
    ws = torch.empty(int(L.tl_workspace_bytes(1, n, 128)), dtype=torch.uint8, device="cuda")
    pr = torch.empty((n, 258), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    outs.append((h, od, ws, pr, s, b))
for h, od, ws, pr, s, b in outs:      # both launched back to back, no sync between them
    rc = L.tl_prove(h.data_ptr(), od.data_ptr(), 1, T, H, 32, 128, T // 32, pr.data_ptr(), None, None,
                    ws.data_ptr(), ws.numel(), s.cuda_stream)
    assert rc == 0
torch.cuda.synchronize()
for h, od, ws, pr, s, b in outs:
    want = TO.build_proofs(b, offs)[0]
    got = [bytes(r) for r in pr.cpu().numpy()]
    assert got == want
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("H,lens,dist", [(5120, [700, 1, 33, 0, 64], 0), (3, [40, 7, 1], 1), (64, [1000, 1], 0),
                                          (1024, [2048], 2), (8192, [300, 20], 3), (256, [129] * 9, 1)])
def test_small_batch_commitment_kernels_agree(H, lens, dist):
    """A small batch's commitment (commit_coop_kernel: Lagrange form over a subproduct tree)
    and the co-resident one-warp kernel (Newton form, inverse tables) give the same proof
    bytes for every chunk -- fallback primes (H 5120, 8192), chunks of fewer than K
    elements (kk < 128: H 3, the one-row chunks), all-equal and tie-heavy values."""
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    bits = synth_bits(0, int(offs[-1]), H, seed=17, dist=dist)
    eng = api.engine()
    plan = eng.plan(offs, H)
    assert plan.n_chunks <= 4 * int(eng.lib.tl_stream_sms(None))
    plan.select(torch.from_numpy(bits.view(np.int16)).cuda())
    plan.commit()
    torch.cuda.synchronize()
    coop = plan.proofs.clone()
    plan.commit(co_resident=True)
    torch.cuda.synchronize()
    assert torch.equal(coop, plan.proofs)
    got = [bytes(b) for b in coop.cpu().numpy()]
    assert got == [p for r in TO.build_proofs(bits, offs) for p in r]
