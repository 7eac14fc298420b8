"""The TMA-ring streaming kernels (large batches, H % 8 == 0) against the one-warp-per-chunk
kernels over WHOLE batches (two independent GPU implementations: every index, value,
proof byte, statistic and verdict must agree) and against the CPU oracle on sampled
chunks (rollout boundaries plus random ones).

Shapes cover 2 to 16 ring stages per chunk, chunks smaller than one stage, ragged
rollouts with partial last chunks, ties across the four consumer warps (all-equal and
all-zero chunks, fp8 round trips), orderings built against the threshold speculation,
speculation slots pre-filled with garbage (forcing the global-memory re-scan), and
validator variants."""

import numpy as np
import pytest
import torch

from fullsize_util import boundary_chunks, check_prove, check_verify, chunk_rows
from paper_2505_07291_b200 import _ffi, api
from paper_2505_07291_b200.synth import synth_device

pytestmark = pytest.mark.gpu
N_RANDOM = 48


RING = -2   # ctas_per_sm that selects the ring kernels for select and verify


def ring_grid(h, H, n_chunks, ctas=RING, verify=1):
    return int(_ffi.load().tl_ring_grid(h.data_ptr(), H, n_chunks, ctas, verify,
                                        torch.cuda.current_stream().cuda_stream))


KEYS = ("idx", "bits", "proofs", "stats", "chunk_accept", "rollout_accept")


def both_ways(h_prv, h_val, offs, H, th=api.Thresholds()):
    """Prove + verify with the ring kernels (ctas_per_sm = -2) and with the one-warp
    kernels (-1); returns the two plans' host outputs.  Each plan runs twice: the first
    launches start from an untrained speculation state (every element a candidate), the
    second from the trained one -- for a batch of one chunk per ring CTA the second takes
    the cooperative finish (ring_coop_finish), the first its general path."""
    eng = api.engine()
    outs = []
    for ctas in (RING, -1):
        plan = eng.plan(offs, H)
        runs = []
        for _ in range(2):
            plan.select(h_prv, ctas_per_sm=ctas)
            plan.commit()
            plan.verify(h_val, thresholds=th, ctas_per_sm=ctas)
            torch.cuda.synchronize()
            runs.append({k: getattr(plan, k).cpu().numpy() for k in KEYS})
        for k in KEYS:
            assert np.array_equal(runs[0][k], runs[1][k]), f"second launch differs in {k} (ctas {ctas})"
        outs.append(runs[1])
        outs[-1]["plan"] = plan
    return outs


def check_case(prv, val, offs, H, th=api.Thresholds(), n_random=N_RANDOM):
    offs = np.asarray(offs, dtype=np.int64)
    n_chunks = int(np.sum(-(-np.diff(offs) // 32)))
    assert ring_grid(prv, H, n_chunks) > 0, "the case must take the ring path"
    ring, warp = both_ways(prv.view(torch.int16), val.view(torch.int16), offs, H, th)
    for k in KEYS:
        assert np.array_equal(ring[k], warp[k]), f"ring vs one-warp kernels differ in {k}"
    plan = ring["plan"]
    table = chunk_rows(offs)
    rng = np.random.default_rng(n_chunks)
    js = sorted(set(boundary_chunks(offs, every=max(1, (len(offs) - 1) // 16))) |
                set(rng.choice(n_chunks, size=min(n_random, n_chunks), replace=False).tolist()))
    rej = np.nonzero(ring["chunk_accept"] == 0)[0]
    js = sorted(set(js) | set(rej[:64].tolist()))
    proofs_by_chunk, bad = check_prove(prv, table, js, plan.idx, plan.bits, plan.proofs)
    assert not bad, f"prove mismatches vs oracle at chunks {bad[:16]}"
    from oracle import toploc_oracle as TO
    st = ring["stats"].view(api.STATS_DTYPE).reshape(-1)
    badv, _ = check_verify(val, table, js, proofs_by_chunk, st, ring["chunk_accept"],
                           TO.Thresholds(th.max_exp_mismatch, th.max_mant_mean, th.max_mant_median))
    assert not badv, f"verify mismatches vs oracle at chunks {badv[:16]}"
    return ring


@pytest.mark.parametrize("R,T,H", [(1, 2048, 1024),       # configuration 1: auto picks the ring
                                   (1, 8192, 5120), (3, 700, 5120), (2, 33, 8192),
                                   (40, 1024, 5120),      # 10 stages per chunk
                                   (64, 1024, 1024),      # 2 stages
                                   (48, 1024, 8192),      # 16 stages
                                   (10, 8192, 128)])      # a chunk is a quarter of one stage
def test_ring_matches_warp_kernels_and_oracle(R, T, H):
    offs = np.arange(R + 1, dtype=np.int64) * T
    prv = synth_device(R * T, H, seed=21)
    val = synth_device(R * T, H, seed=21, jitter_thr=3277, jitter_seed=22)
    check_case(prv, val, offs, H)


def test_ring_ragged_rollouts_with_partial_chunks():
    rng = np.random.default_rng(4)
    T = rng.integers(1, 900, size=160)
    T[::7] = 0
    offs = np.concatenate([[0], np.cumsum(T)]).astype(np.int64)
    H = 2048
    prv = synth_device(int(offs[-1]), H, seed=31, dist="massive")
    val = synth_device(int(offs[-1]), H, seed=31, dist="massive", jitter_thr=3277, jitter_seed=32)
    check_case(prv, val, offs, H)


@pytest.mark.parametrize("R", [40, 2])
@pytest.mark.parametrize("dist", ["zeros", "ones"])
def test_ring_ties_across_consumer_warps(dist, R):
    """All-equal chunks: the top-128 are the 128 lowest flat indices, all in the first
    consumer warp's first tile; the other warps hold only losing ties.  R = 2: one chunk
    per ring CTA (cooperative finish, or its fallback when the ties overflow it)."""
    T, H = 1024, 1024
    offs = np.arange(R + 1, dtype=np.int64) * T
    prv = synth_device(R * T, H, seed=1, dist=dist)
    ring = check_case(prv, prv, offs, H)
    idx = ring["idx"]
    assert np.all(idx == np.arange(128)[None, :])


@pytest.mark.parametrize("R", [40, 3])
@pytest.mark.parametrize("kind", ["fp8_ties", "ascending", "descending", "spikes", "alternating"])
def test_ring_adversarial_orderings(kind, R):
    T, H = 1024, 1024
    C, n = 32, 32 * 1024
    offs = np.arange(R + 1, dtype=np.int64) * T
    dev = torch.device("cuda")
    base = synth_device(R * T, H, seed=5)
    i = torch.arange(n, device=dev, dtype=torch.int64)
    if kind == "fp8_ties":
        prv = base.to(torch.float8_e4m3fn).to(torch.bfloat16)
    else:
        if kind == "ascending":
            pat = 0x3F80 + (i * 127) // n
        elif kind == "descending":
            pat = ((n - 1 - i) * 0x7F7F) // n
        elif kind == "alternating":
            pat = ((i * 0x7F7F) // n) | ((i & 1) << 15)
        else:
            g = torch.Generator(device=dev)
            g.manual_seed(3)
            pat = torch.zeros(n, dtype=torch.int64, device=dev)
            pat[torch.randperm(n, device=dev, generator=g)[:128]] = 0x4300
        chunk = pat.to(torch.int16).view(C, H)
        prv = chunk.repeat(R * T // C, 1).contiguous().view(torch.bfloat16)
        # every other chunk normal, so the speculation carries across the patterns
        prv.view(R * T // C, C, H)[::2] = base.view(R * T // C, C, H)[::2]
    val = prv.to(torch.float8_e5m2).to(torch.bfloat16)
    check_case(prv, prv, offs, H)
    check_case(prv, val, offs, H)


@pytest.mark.parametrize("R", [40, 2])
@pytest.mark.parametrize("fill", ["garbage", "too_high", "zero"])
def test_ring_speculation_state_is_only_a_hint(fill, R):
    """Workspace speculation slots pre-filled so that the first chunks start far too high
    (the ring re-scans them from global memory) or at zero (every element is a candidate,
    the consumer warps compact): results stay bit-exact.  R = 2 (64 chunks, one per ring
    CTA): the cooperative finish hands both cases to the finisher's general path."""
    T, H = 1024, 5120
    offs = np.arange(R + 1, dtype=np.int64) * T
    prv = synth_device(R * T, H, seed=8)
    val = synth_device(R * T, H, seed=8, jitter_thr=3277, jitter_seed=9)
    eng = api.engine()
    plan = eng.plan(offs, H)
    spec = plan.ws[:8192 * 16].view(torch.int32).view(8192, 4)
    if fill == "garbage":
        spec.copy_(torch.randint(-2**31, 2**31 - 1, (8192, 4), dtype=torch.int32, device="cuda"))
    elif fill == "too_high":
        spec[:, 0] = 0x7F00
        spec[:, 1] = 0x7F00
        spec[:, 2] = 1
        spec[:, 3] = 0x53504543
    else:
        spec[:, 0] = 0
        spec[:, 1] = 0
        spec[:, 2] = 1
        spec[:, 3] = 0x53504543
    plan.select(prv.view(torch.int16), ctas_per_sm=RING)
    plan.commit()
    plan.verify(val.view(torch.int16), ctas_per_sm=RING)
    torch.cuda.synchronize()
    ref = eng.plan(offs, H)
    ref.select(prv.view(torch.int16), ctas_per_sm=-1)
    ref.commit()
    ref.verify(val.view(torch.int16), ctas_per_sm=-1)
    torch.cuda.synchronize()
    for k in KEYS:
        assert torch.equal(getattr(plan, k), getattr(ref, k)), k


def test_ring_is_selected_only_where_it_applies():
    h = torch.empty((64, 1024), dtype=torch.bfloat16, device="cuda")
    sms = int(_ffi.load().tl_stream_sms(None))
    g = ring_grid(h, 1024, 8 * sms)
    assert g > 0 and g % sms == 0
    assert ring_grid(h, 1024, 8 * sms, verify=0) == g
    assert ring_grid(h, 1024, 8 * sms, ctas=0, verify=0) == 0   # auto: large batches keep the one-warp kernels
    assert ring_grid(h, 1024, 8 * sms, ctas=0, verify=1) == 0
    assert ring_grid(h, 1024, 64, ctas=0, verify=1) == 64       # auto: a batch of one chunk per ring CTA
    assert ring_grid(h, 1024, g, ctas=0) == g and ring_grid(h, 1024, g + 1, ctas=0) == 0
    assert ring_grid(h, 1024, 8 * sms, ctas=16) == 0            # co-resident pipeline shape
    assert ring_grid(h, 1024, 64, ctas=-1) == 0
    assert ring_grid(h, 1030, 64, ctas=0) == 0                  # chunks not 16-byte aligned
    hv = h.view(-1)[1:1 + 63 * 1024].view(63, 1024)             # unaligned base pointer
    assert ring_grid(hv, 1024, 64, ctas=0) == 0


def test_ring_small_batch_over_many_tiny_rollouts():
    """A small batch (one chunk per ring CTA) over more rollouts than a CTA builds its own
    chunk prefix for (> 256): the chunk_prefix_kernel path with no chunk claims, with empty
    rollouts in between and partial chunks."""
    rng = np.random.default_rng(12)
    T = rng.integers(1, 33, size=300)
    T[::5] = 0
    offs = np.concatenate([[0], np.cumsum(T)]).astype(np.int64)
    n_chunks = int(np.sum(-(-T // 32)))
    H = 1024
    prv = synth_device(int(offs[-1]), H, seed=41)
    assert 256 < len(T) and 0 < n_chunks <= ring_grid(prv, H, n_chunks, ctas=0, verify=0)
    val = synth_device(int(offs[-1]), H, seed=41, jitter_thr=3277, jitter_seed=42)
    check_case(prv, val, offs, H)


def test_ring_cooperative_verify_forged_and_short_chunks():
    """One chunk per ring CTA (cooperative finish once the speculation is trained) with
    chunks shorter than K (one row of hidden 64: kk = 64) and forged proofs: moduli 2, 97
    and 32769 (bad proofs) and the right coefficients under another prover prime. Ring and
    one-warp verify agree in every statistic and verdict, over two launches each."""
    H = 64
    offs = np.array([0, 993, 993 + 65], dtype=np.int64)
    prv = synth_device(int(offs[-1]), H, seed=51)
    val = synth_device(int(offs[-1]), H, seed=51, jitter_thr=3277, jitter_seed=52)
    eng = api.engine()
    ref = eng.plan(offs, H)
    ref.select(prv.view(torch.int16), ctas_per_sm=-1)
    ref.commit()
    torch.cuda.synchronize()
    n = ref.n_chunks
    assert ring_grid(prv, H, n, ctas=0) >= n
    forged = ref.proofs.clone().view(n, -1)
    for c, p in ((0, 2), (1, 97), (2, 32769), (3, 65479)):
        forged[c, 0], forged[c, 1] = p >> 8, p & 0xFF
    forged[0, 2:] = 0
    outs = {}
    for ctas in (RING, -1):
        plan = eng.plan(offs, H)
        plan.select(prv.view(torch.int16), ctas_per_sm=ctas)   # trains the speculation
        runs = []
        for _ in range(2):
            plan.verify(val.view(torch.int16), forged.view(-1), ctas_per_sm=ctas)
            torch.cuda.synchronize()
            runs.append({k: getattr(plan, k).cpu().numpy() for k in ("stats", "chunk_accept", "rollout_accept")})
        for k in runs[0]:
            assert np.array_equal(runs[0][k], runs[1][k]), k
        outs[ctas] = runs[1]
    for k in outs[RING]:
        assert np.array_equal(outs[RING][k], outs[-1][k]), f"ring vs one-warp verify differ in {k}"
    st = outs[RING]["stats"].view(api.STATS_DTYPE).reshape(-1)
    assert all(st["flags"][c] & 2 for c in (0, 1, 2)) and not st["flags"][3] & 2
    from oracle import toploc_oracle as TO
    assert 65479 in TO.PRIME_SET
    fp = forged.cpu().numpy()
    th = api.Thresholds()
    bad, _ = check_verify(val, chunk_rows(offs), list(range(n)), {j: bytes(fp[j]) for j in range(n)}, st,
                          outs[RING]["chunk_accept"], TO.Thresholds(th.max_exp_mismatch, th.max_mant_mean,
                                                                    th.max_mant_median))
    assert not bad, bad[:8]


@pytest.mark.parametrize("H", [8, 16, 40])
def test_ring_tiny_rows_and_short_chunks(H):
    """Rows of 8-40 elements: every chunk holds fewer than K = 128 elements at H 8 (kk = the
    chunk's element count), ragged rollouts leave one-row chunks; small batches (one chunk
    per ring CTA), so the cooperative finish ranks and evaluates kk < 128 points."""
    rng = np.random.default_rng(H)
    T = rng.integers(1, 70, size=9)
    offs = np.concatenate([[0], np.cumsum(T)]).astype(np.int64)
    prv = synth_device(int(offs[-1]), H, seed=61)
    val = synth_device(int(offs[-1]), H, seed=61, jitter_thr=3277, jitter_seed=62)
    check_case(prv, val, offs, H)
