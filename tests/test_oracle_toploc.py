"""TOPLOC oracle: pinned by independent restatements and committed golden vectors.

Upstream ``toploc`` is absent (parity vs upstream unpinned), so
the oracle is cross-checked here against (a) a full stable sort for top-k, (b)
Lagrange interpolation over Python ints for the polynomial, (c) the defining
property P(x_i) = y_i, and (d) tests/golden/toploc_golden.json (regression).
"""

import hashlib
import json
import math
import os
import random

import numpy as np
import pytest

from oracle import toploc_oracle as TO
from oracle.synth_cpu import synth_bits
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def ref_topk(bits, K):
    """Independent: full sort by (|bits| desc, index asc)."""
    order = sorted(range(len(bits)), key=lambda i: (-(int(bits[i]) & 0x7FFF), i))
    return order[:min(K, len(bits))]


@pytest.mark.parametrize("seed", range(6))
def test_select_matches_full_sort(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    # few distinct magnitudes -> many ties at the threshold
    bits = rng.integers(0, 64, size=n).astype(np.uint16) | (rng.integers(0, 2, size=n).astype(np.uint16) << 15)
    idx, vals = TO.select_topk(bits, 128)
    assert list(idx) == ref_topk(bits, 128)
    assert np.array_equal(vals, bits[idx])


def test_select_batch_matches_single():
    rng = np.random.default_rng(7)
    B = rng.integers(0, 1 << 16, size=(9, 4096)).astype(np.uint16)
    I, V = TO.select_topk_batch(B, 128)
    for j in range(9):
        i1, v1 = TO.select_topk(B[j], 128)
        assert np.array_equal(I[j], i1) and np.array_equal(V[j], v1)


def test_select_ties_take_lowest_indices_and_nan_first():
    bits = np.full(1000, 0x3F80, dtype=np.uint16)
    idx, _ = TO.select_topk(bits, 128)
    assert list(idx) == list(range(128))
    bits[500] = 0x7FC0   # NaN ranks above everything (by bit pattern)
    bits[700] = 0xFF80   # -inf
    idx, _ = TO.select_topk(bits, 128)
    assert list(idx[:2]) == [500, 700]


@pytest.mark.parametrize("n,seed", [(1, 0), (2, 1), (5, 2), (17, 3), (40, 4)])
def test_newton_equals_lagrange_and_interpolates(n, seed):
    rnd = random.Random(seed)
    p = TO.PRIMES_DESC[seed]
    x = rnd.sample(range(p), n)
    y = [rnd.randrange(1 << 16) for _ in range(n)]
    cn = TO.interpolate_newton(x, y, p)
    cl = TO.interpolate_lagrange(x, y, p)
    assert cn == cl
    assert list(TO.eval_poly(cn, p, x)) == [v % p for v in y]
    cb = TO.interpolate_batch(np.array([x]), np.array([[v % p for v in y]]), np.array([p]))[0]
    assert list(cb) == cn


def test_modulus_prime_and_injective():
    import sympy
    assert all(sympy.isprime(p) for p in TO.PRIMES_DESC[:50])
    assert TO.PRIMES_DESC[0] == 65497 and TO.PRIMES_DESC[-1] == 32771
    assert TO.find_modulus([0, 1, 2]) == 65497
    assert TO.find_modulus([0, 65497]) == 65479          # collision at 65497
    assert TO.find_modulus([0, 65497, 65479 * 2]) == 65449
    P = TO.find_modulus_batch(np.array([[0, 65497, 5], [1, 2, 3]]))
    assert list(P) == [65479, 65497]


def test_proof_format():
    pr = TO.proof_bytes(65497, [1, 2, 0xABCD], K=128)
    assert len(pr) == 258 and pr[:2] == bytes([0xFF, 0xD9]) and pr[2:8] == bytes([0, 1, 0, 2, 0xAB, 0xCD])
    assert pr[8:] == b"\x00" * 250
    p, c = TO.parse_proof(pr)
    assert p == 65497 and list(c[:3]) == [1, 2, 0xABCD]
    with pytest.raises(ValueError):
        TO.parse_proof(pr[:-1])


def test_prove_verify_roundtrip_and_rejections():
    bits = synth_bits(0, 70, 96, seed=11)
    offs = [0, 70]
    proofs = TO.build_proofs(bits, offs)
    assert [len(p) for p in proofs] == [3] and all(len(x) == 258 for x in proofs[0])
    stats, verdict = TO.verify_proofs(bits, offs, proofs)
    assert verdict == [True] and all(s.exp_mismatch == 0 and s.mant_sum == 0 for s in stats)
    other = synth_bits(0, 70, 96, seed=12)
    stats, verdict = TO.verify_proofs(other, offs, proofs)
    assert verdict == [False]
    bad = [[b"\x00\x01" + proofs[0][0][2:]] + proofs[0][1:]]   # p = 1 -> invalid proof
    stats, verdict = TO.verify_proofs(bits, offs, bad)
    assert verdict == [False] and stats[0].n_match == 0 and math.isinf(stats[0].mant_mean)


@pytest.mark.parametrize("p", [2, 3, 97, 128, 32769, 65521])
def test_forged_small_or_composite_modulus_is_a_bad_proof(p):
    """p = 2 with zero coefficients makes every claimed and observed value < 2, so all
    exponents agree and the mantissa diffs are <= 1: without the modulus check it passes
    for any activations.  Only the prover's primes are accepted."""
    bits = synth_bits(0, 64, 96, seed=13)
    forged = [[p.to_bytes(2, "big") + bytes(256)] * 2]
    stats, verdict = TO.verify_proofs(bits, [0, 64], forged)
    assert verdict == [False]
    assert all(s.exp_mismatch == 128 and s.n_match == 0 and math.isinf(s.mant_median) for s in stats)


def test_median_is_statistics_median():
    claimed = np.array([0x3F80, 0x3F81, 0x3F84, 0x3F88], dtype=np.int64)
    observed = np.array([0x3F80, 0x3F80, 0x3F80, 0x3F80], dtype=np.int64)
    st = TO.chunk_stats(claimed, observed, TO.Thresholds())
    assert (st.exp_mismatch, st.n_match, st.mant_sum) == (0, 4, 13)
    assert st.mant_mean == 13 / 4 and st.mant_median == 2.5


def load_golden():
    with open(os.path.join(GOLDEN, "toploc_golden.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", load_golden(), ids=lambda c: c["name"])
def test_oracle_regression_golden(case):
    offs, H, K, C = case["row_offsets"], case["H"], case["K"], case["C"]
    bits = synth_bits(0, offs[-1], H, case["seed"], case["dist"])
    tab, chunks = TO._chunks_of(bits, offs, C)
    idxs, _, proofs = TO.prove_chunks(chunks, K)
    assert len(proofs) == case["n_chunks"]
    assert [int.from_bytes(p[:2], "big") for p in proofs] == case["moduli"]
    assert hashlib.sha256(b"".join(proofs)).hexdigest() == case["proofs_sha256"]
    assert proofs[0].hex() == case["first_proof"]
    assert [int(v) for v in idxs[0]] == case["first_idx"]
    per = [[] for _ in range(len(offs) - 1)]
    for (r, _, _), pr in zip(tab, proofs):
        per[r].append(pr)
    jit = synth_bits(0, offs[-1], H, case["seed"], case["dist"], jitter_thr=case["jitter_thr"],
                     jitter_seed=case["jitter_seed"])
    stats, verdict = TO.verify_proofs(jit, offs, per, C, K)
    assert [[s.exp_mismatch, s.n_match, s.mant_sum, s.mant_median, s.accept] for s in stats] == case["jitter_stats"]
    assert verdict == case["jitter_verdict"]


def test_collision_case_exercises_fallback_prime():
    case = next(c for c in load_golden() if c["name"] == "h5120_collide")
    assert any(p != 65497 for p in case["moduli"])


def test_synth_cpu_is_deterministic_and_row_addressable():
    a = synth_bits(0, 40, 1030, seed=3, dist=1)
    b = synth_bits(17, 10, 1030, seed=3, dist=1)
    assert np.array_equal(a[17:27], b)
    j = synth_bits(0, 40, 1030, seed=3, dist=1, jitter_thr=3277, jitter_seed=9)
    frac = np.mean(a != j)
    assert 0.03 < frac < 0.07
