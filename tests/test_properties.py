"""Property tests (hypothesis, as the reference's own suite uses for GRPO,
tests/test_grpo.py:46-49,117-149) for the host-side pieces and the oracle the GPU
kernels are checked against."""

import numpy as np
from hypothesis import given, settings, strategies as st

from oracle import toploc_oracle as TO
from paper_2505_07291_b200 import codec, scheduler


@settings(max_examples=60, deadline=None)
@given(st.lists(st.integers(0, 40), min_size=1, max_size=12), st.integers(0, 2**31 - 1))
def test_codec_round_trip(chunks_per_rollout, seed):
    n = sum(chunks_per_rollout)
    rng = np.random.default_rng(seed)
    arr = rng.integers(0, 256, size=(n, codec.PROOF_BYTES), dtype=np.uint8)
    p = rng.choice(TO.PRIMES_DESC + [0], size=n)          # a prover modulus (0: unprovable chunk)
    arr[:, 0], arr[:, 1] = p >> 8, p & 0xFF
    co = np.concatenate([[0], np.cumsum(chunks_per_rollout)])
    hexed = codec.encode(arr, chunk_offsets=co)
    assert [len(h) for h in hexed] == chunks_per_rollout
    back, co2 = codec.decode(hexed, n_tokens=[32 * c for c in chunks_per_rollout])
    assert np.array_equal(back, arr) and np.array_equal(co2, co)


@settings(max_examples=80, deadline=None)
@given(st.lists(st.integers(0, 5000), min_size=0, max_size=60), st.integers(1, 9))
def test_shards_tile_contiguously_and_balance(lengths, world):
    ranges = scheduler.shard_by_tokens(lengths, world)
    assert len(ranges) == world
    assert ranges[0][0] == 0 and ranges[-1][1] == len(lengths)
    for (a, b), (c, _) in zip(ranges, ranges[1:]):
        assert a <= b == c
    total = sum(lengths)
    if total and lengths:
        # each rank's token count stays within one rollout of its share
        worst = max(lengths)
        for lo, hi in ranges:
            assert sum(lengths[lo:hi]) <= total / world + worst + 1e-9


@settings(max_examples=40, deadline=None)
@given(st.integers(2, 48), st.integers(0, 2**31 - 1))
def test_newton_interpolation_matches_lagrange_and_passes_through_points(n, seed):
    rng = np.random.default_rng(seed)
    p = 65497
    x = rng.choice(p, size=n, replace=False)
    y = rng.integers(0, 1 << 16, size=n)
    c_newton = TO.interpolate_newton(x, y, p)
    assert c_newton == TO.interpolate_lagrange(x, y, p)
    vals = TO.eval_poly(c_newton + [0] * (128 - n), p, x)
    assert [int(v) for v in vals] == [int(v) % p for v in y]


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 600), st.integers(1, 140), st.integers(0, 2**31 - 1), st.booleans())
def test_topk_equals_a_stable_full_sort(n, K, seed, ties):
    rng = np.random.default_rng(seed)
    bits = (rng.integers(0, 4, size=n) * 0x1111 if ties else rng.integers(0, 1 << 16, size=n)).astype(np.uint16)
    idx, vals = TO.select_topk(bits, K)
    order = sorted(range(n), key=lambda i: (-(int(bits[i]) & 0x7FFF), i))[:min(K, n)]
    assert idx.tolist() == order and vals.tolist() == [int(bits[i]) for i in order]
