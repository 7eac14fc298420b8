"""GPU exact mode against digests produced by the reference itself.

``paper_2505_07291_b200.api.build_commitments`` must be byte-identical to the
reference's ``build_commitments`` (pkg/src/swarm/worker/rollout.py:51-68) on the
inputs of tests/golden/exact_golden.json and on the reference's own adversarial
corpus (forge_golden.*)."""

import json
import os

import numpy as np
import pytest
import torch

from paper_2505_07291_b200 import api
from paper_2505_07291_b200.exact import round6_device

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

from test_oracle_exact import load_cases, regen_input  # noqa: E402


@pytest.mark.parametrize("case", load_cases(), ids=lambda c: c["name"])
def test_gpu_exact_matches_reference(case):
    arr = regen_input(case)
    assert [d.hex() for d in api.build_commitments(arr, case["k"])] == case["digests"]


def test_gpu_round6_bitwise_equals_numpy():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.normal(size=100000) * 10.0 ** rng.integers(-12, 12, size=100000),
                        np.array([1e303, -1e303, np.nan, -np.nan, np.inf, -0.0, 5e-324, 2.5e-6, -3.5e-6])])
    with np.errstate(over="ignore", invalid="ignore"):
        want = np.round(x, 6)
    got = round6_device(x).cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_gpu_round6_every_float32():
    """The branch-free division in round6_value (csrc, FMA-corrected reciprocal) against
    a correctly rounded division, for every float32 bit pattern (which includes every
    bfloat16 and float16 value).  The reference side is rint(x * 1e6) / 1e6 in float64
    on the GPU (IEEE division), itself checked against numpy on a sample."""
    sample = np.random.default_rng(7).integers(0, 1 << 32, size=1 << 16, dtype=np.uint64).astype(np.uint32)
    xs = sample.view(np.float32).astype(np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        ref_np = np.round(xs, 6)
    tx = torch.from_numpy(xs).cuda()
    # a tensor divisor: torch turns division by a Python scalar into a reciprocal multiply
    ref_t = (torch.round(tx * 1e6) / torch.full_like(tx, 1e6)).cpu().numpy()
    fin = np.isfinite(xs)
    assert np.array_equal(ref_np[fin].view(np.uint64), ref_t[fin].view(np.uint64))
    step = 1 << 28
    for start in range(0, 1 << 32, step):
        v = torch.arange(start, start + step, dtype=torch.int64, device="cuda")
        x = torch.where(v >= (1 << 31), v - (1 << 32), v).to(torch.int32).view(torch.float32)
        got = round6_device(x)
        xd = x.double()
        want = torch.round(xd * 1e6) / torch.full_like(xd, 1e6)
        nan = torch.isnan(x)
        same = (got.view(torch.int64) == want.view(torch.int64)) | nan
        assert bool(same.all()), f"slice {start:#x}: first mismatch at {int((~same).nonzero()[0]) + start:#x}"
        assert bool(torch.isnan(got[nan]).all())
        del v, x, xd, got, want, nan, same


def test_gpu_round6_random_float64_bit_patterns():
    """Random float64 bit patterns over the whole exponent range, and values a few ulps
    from multiples of 1e-6 (the hardest quotients), against numpy."""
    rng = np.random.default_rng(11)
    bits = rng.integers(0, 1 << 63, size=1 << 22, dtype=np.int64).astype(np.uint64)
    bits |= rng.integers(0, 2, size=bits.size, dtype=np.uint64) << np.uint64(63)
    x = bits.view(np.float64)
    near = (rng.integers(-10**12, 10**12, size=1 << 20) / 1e6).astype(np.float64)
    near = np.nextafter(near, np.where(rng.integers(0, 2, size=near.size) == 1, np.inf, -np.inf))
    x = np.concatenate([x, near, near * 0.5 + 0.5e-6])
    with np.errstate(over="ignore", invalid="ignore"):
        want = np.round(x, 6)
    got = round6_device(x).cpu().numpy()
    ok = (got.view(np.uint64) == want.view(np.uint64)) | np.isnan(x)
    assert ok.all(), x[~ok][:5]


def test_gpu_round6_from_bf16_f32_f16():
    rng = np.random.default_rng(1)
    x = torch.from_numpy(rng.normal(size=(64, 33)).astype(np.float32))
    for dt in (torch.float32, torch.bfloat16, torch.float16):
        t = x.to(dt)
        with np.errstate(over="ignore", invalid="ignore"):
            want = np.round(t.to(torch.float64).numpy(), 6)
        got = round6_device(t.cuda()).cpu().numpy()
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), dt


def test_gpu_exact_on_reference_forge_corpus():
    with open(os.path.join(GOLDEN, "forge_golden.json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, "forge_golden.npz"))
    for m in meta:
        prv, val = arrays[f"prv_{m['i']}"], arrays[f"val_{m['i']}"]
        assert [d.hex() for d in api.build_commitments(prv)] == m["commitments"]
        got_val = [d.hex() for d in api.build_commitments(torch.from_numpy(val).cuda())]
        assert got_val == m["ref_val_digests"]
        # the validator's verdict (checks.py:209-213): equal digest lists
        assert (got_val == m["commitments"]) == (m["kind"] == "honest")


def test_gpu_exact_errors():
    with pytest.raises(ValueError, match="interval"):
        api.build_commitments(np.ones((2, 2)), k=0)


def test_gpu_exact_batch_matches_reference_per_rollout():
    rng = np.random.default_rng(4)
    lens = [70, 0, 33, 129, 5]
    offs = np.concatenate([[0], np.cumsum(lens)])
    h = rng.normal(size=(int(offs[-1]), 24))
    from paper_2505_07291_b200.exact import build_commitments_batch
    from oracle import exact_oracle as EO
    got = build_commitments_batch(torch.from_numpy(h).cuda(), offs, 32, group_rows=100)
    want = [EO.build_commitments(h[offs[r]:offs[r + 1]], 32) for r in range(len(lens))]
    assert got == want
    hb = torch.from_numpy(h.astype(np.float32)).to(torch.bfloat16)
    got = build_commitments_batch(hb, offs, 7, group_rows=64)
    want = [EO.build_commitments(hb.to(torch.float64).numpy()[offs[r]:offs[r + 1]], 7) for r in range(len(lens))]
    assert got == want


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.bfloat16, torch.float16])
def test_device_sha_chains_equal_host_chains(dtype):
    """tl_exact_chains (SHA-256 chains on the GPU, one thread per rollout) against the
    host chains over the same rounded values: ragged rollouts, T = 0, T < k, T % k != 0,
    odd H, NaN / inf / -0.0 and huge values."""
    from paper_2505_07291_b200.exact import build_commitments_batch, build_commitments_device
    rng = np.random.default_rng(3)
    H = 37
    lens = [0, 1, 31, 32, 33, 64, 95, 200, 0, 7]
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    x = rng.normal(size=(int(offs[-1]), H)) * 10.0 ** rng.integers(-8, 8, size=(int(offs[-1]), H))
    x[3, :4] = [np.nan, -np.inf, -0.0, 1e300]
    t = torch.from_numpy(x).to(dtype)
    for k in (32, 5):
        got = build_commitments_device(t, offs, k)
        want = build_commitments_batch(t, offs, k, sha="host")
        assert got == want, (dtype, k)
        assert all(len(g) == max(1, -(-n // k)) for g, n in zip(got, lens))


def test_device_sha_matches_reference_goldens():
    from paper_2505_07291_b200.exact import build_commitments_device
    for case in load_cases():
        arr = regen_input(case)
        a2 = np.asarray(arr, dtype=np.float64)
        if a2.ndim != 2:
            continue
        got = build_commitments_device(a2, [0, a2.shape[0]], case["k"])[0]
        assert [d.hex() for d in got] == case["digests"], case["name"]


def test_device_sha_empty_rows_and_empty_batches():
    """H = 0 (rows without values) and all-empty rollouts: digests over the chained
    prefix only, exactly as the reference's hashlib chain."""
    from paper_2505_07291_b200.exact import build_commitments_batch, build_commitments_device
    for shape, offs in (((40, 0), [0, 33, 33, 40]), ((0, 5), [0, 0, 0])):
        x = np.zeros(shape)
        assert build_commitments_device(x, offs, 32) == build_commitments_batch(x, offs, 32, sha="host")


def test_batch_auto_switches_to_device_chains_at_threshold(monkeypatch):
    """sha="auto" hashes on the GPU from DEVICE_SHA_MIN_ROLLOUTS rollouts and on the host
    below; both give the reference's digests."""
    from paper_2505_07291_b200 import exact
    from oracle import exact_oracle as EO
    rng = np.random.default_rng(9)
    R = exact.DEVICE_SHA_MIN_ROLLOUTS
    lens = rng.integers(0, 70, size=R)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    h = torch.from_numpy(rng.normal(size=(int(offs[-1]), 12)).astype(np.float32)).to(torch.bfloat16)
    used = []
    real = exact.build_commitments_device
    monkeypatch.setattr(exact, "build_commitments_device", lambda *a, **k: used.append(1) or real(*a, **k))
    big = exact.build_commitments_batch(h.cuda(), offs, 32)
    assert used, "auto did not take the GPU chains at the threshold"
    n_small = R // 2
    small = exact.build_commitments_batch(h[:offs[n_small]].cuda(), offs[:n_small + 1], 32)
    assert len(used) == 1, "auto took the GPU chains below the threshold"
    h64 = h.to(torch.float64).numpy()
    for r in list(range(8)) + [R - 1]:
        assert big[r] == EO.build_commitments(h64[offs[r]:offs[r + 1]], 32)
    assert small == big[:n_small]
