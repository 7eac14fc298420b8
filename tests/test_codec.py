"""TOPLOC proofs on the rollout-file wire format: hex encoding, count and
interval rules (worker/files.py:37,184-186; validator/checks.py:211), and -- where the
reference package is importable -- a round trip through the reference's own signed
file writer and parser."""


import numpy as np
import pytest

from paper_2505_07291_b200 import codec


def random_proofs(n, seed=0):
    rng = np.random.default_rng(seed)
    arr = rng.integers(0, 256, size=(n, codec.PROOF_BYTES), dtype=np.uint8)
    p = rng.choice([65497, 65479, 32771, 0], size=n)       # prover moduli (0: unprovable chunk)
    arr[:, 0], arr[:, 1] = p >> 8, p & 0xFF
    return arr


def test_encode_matches_bytes_hex_and_round_trips():
    arr = random_proofs(11)
    co = [0, 3, 3, 11]
    hexed = codec.encode(arr, chunk_offsets=co)
    assert [len(h) for h in hexed] == [3, 0, 8]
    flat = [s for h in hexed for s in h]
    assert flat == [arr[j].tobytes().hex() for j in range(11)]
    back, co2 = codec.decode(hexed, n_tokens=[70, 0, 256])
    assert np.array_equal(back, arr) and list(co2) == co


def test_encode_from_row_offsets_uses_the_32_token_rule():
    arr = random_proofs(5)
    hexed = codec.encode(arr, row_offsets=[0, 33, 33, 129])  # 2 + 0 + 3 chunks
    assert [len(h) for h in hexed] == [2, 0, 3]
    assert codec.expected_count(33) == 2 and codec.expected_count(0) == 0 and codec.expected_count(32) == 1


@pytest.mark.parametrize("bad,msg", [
    ([["ab" * 258, "cd" * 258]], "commitments"),      # count: T=32 needs 1
    ([["ab" * 257]], "516-char"),                      # short item
    ([["zz" * 258]], "not hex"),
    ([[b"\x00" * 258]], "516-char"),                   # bytes, not a hex string
])
def test_decode_rejects_malformed_lists(bad, msg):
    with pytest.raises(codec.ProofFormatError, match=msg):
        codec.decode(bad, n_tokens=[32])


@pytest.mark.parametrize("p", [1, 2, 97, 128, 32769, 32770, 65498, 65521, 65535])
def test_decode_rejects_non_prover_moduli(p):
    """Only 0 (unprovable chunk) or a prime in [32771, 65497] is a proof modulus; p = 2 with
    zero coefficients would match any activations."""
    good = (65497).to_bytes(2, "big").hex() + "00" * 256
    forged = p.to_bytes(2, "big").hex() + "00" * 256
    with pytest.raises(codec.ProofFormatError, match=f"item 1: modulus {p} "):
        codec.decode([[good], [good, forged]], n_tokens=[32, 64])


def test_interval_is_enforced():
    codec.check_interval(32)
    with pytest.raises(codec.ProofFormatError):
        codec.check_interval(16)
    with pytest.raises(codec.ProofFormatError):
        codec.decode([[]], n_tokens=[0], interval=64)
    with pytest.raises(ValueError):
        codec.expected_count(10, 0)


def test_modulus_field():
    p = (65497).to_bytes(2, "big") + bytes(256)
    assert codec.modulus(p) == 65497 and codec.modulus(p.hex()) == 65497


def test_round_trip_through_reference_file_format():
    from refpath import add_ref_to_path
    add_ref_to_path()
    files = pytest.importorskip("swarm.worker.files")
    from swarm.keys import SigningKey
    key = SigningKey.from_seed(7, 0)
    arr = random_proofs(2 * 3 + 2 * 1, seed=3)
    T = [70, 65, 20, 1]                           # 3, 3, 1, 1 chunks
    hexed = codec.encode(arr, row_offsets=np.concatenate([[0], np.cumsum(T)]))
    recs = [files.RolloutRecord(node_address=key.address, step=4, submission_index=0, task_id=9, group_index=g,
                                member_index=m, checkpoint_version=1, output_tokens=[1] * T[2 * g + m],
                                chosen_probs=[0.5] * T[2 * g + m], commitments=hexed[2 * g + m],
                                eos_prob_at_end=None, r_task=0, r_total=0.0, advantage=0.0)
            for g in range(2) for m in range(2)]
    f = files.RolloutFile(node_address=key.address, step=4, submission_index=0, checkpoint_version=1, group_size=2,
                          num_groups=2, commit_interval=codec.TOPLOC_INTERVAL, records=recs)
    parsed = files.parse_rollout_file(files.build_rollout_file(f, key))  # the reference's count check passes
    codec.check_interval(parsed.commit_interval)
    back, co = codec.decode([r.commitments for r in parsed.records], n_tokens=[len(r.output_tokens)
                                                                            for r in parsed.records])
    assert np.array_equal(back, arr) and list(co) == [0, 3, 6, 7, 8]
