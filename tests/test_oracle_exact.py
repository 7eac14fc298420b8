"""Exact-mode oracle pinned against digests produced by the reference itself.

Golden digests come from ``swarm.worker.rollout.build_commitments``
(reference ``pkg/src/swarm/worker/rollout.py:51-68``) via tests/golden/make_golden.py.
The KATs mirror the reference's own tests (``pkg/tests/test_rollout.py:48-78``).
"""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import exact_oracle as EO
from oracle.synth_cpu import synth_bits
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_cases():
    with open(os.path.join(GOLDEN, "exact_golden.json")) as f:
        return json.load(f)


def regen_input(c):
    if c["kind"] == "array":
        return np.frombuffer(bytes.fromhex(c["data_hex"]), dtype="<f8").reshape(c["shape"])
    if c["kind"] == "rng_normal":
        return np.random.default_rng(c["seed"]).normal(size=(c["T"], c["H"]))
    bits = synth_bits(c["row0"], c["T"], c["H"], c["seed"], c["dist"])
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("case", load_cases(), ids=lambda c: c["name"])
def test_oracle_matches_reference_digests(case):
    arr = regen_input(case)
    assert hashlib.sha256(np.ascontiguousarray(arr, dtype="<f8").tobytes()).hexdigest() == case["input_sha256"]
    with np.errstate(over="ignore", invalid="ignore"):
        got = [d.hex() for d in EO.build_commitments(arr, case["k"])]
    assert got == case["digests"]


class TestReferenceKATs:
    """Same assertions as reference tests/test_rollout.py:48-78."""

    def test_short_sequence_single_digest(self):
        assert len(EO.build_commitments(np.random.default_rng(0).normal(size=(5, 8)), k=32)) == 1

    def test_length_65_gives_three_digests(self):
        assert len(EO.build_commitments(np.random.default_rng(0).normal(size=(65, 8)), k=32)) == 3

    def test_perturbation_changes_first_affected_digest(self):
        hidden = np.random.default_rng(1).normal(size=(70, 8))
        base = EO.build_commitments(hidden, k=32)
        mutated = hidden.copy()
        mutated[40, 3] += 1e-3
        changed = EO.build_commitments(mutated, k=32)
        assert changed[0] == base[0] and changed[1] != base[1] and changed[2] != base[2]

    def test_sub_rounding_perturbation_is_invisible(self):
        hidden = np.full((4, 3), 0.1234561)
        assert EO.build_commitments(hidden) == EO.build_commitments(hidden + 2e-8)

    def test_chaining_from_zero_digest(self):
        block = np.round(np.ones((2, 2)), 6).astype("<f8").tobytes()
        assert EO.build_commitments(np.ones((2, 2)), k=32) == [hashlib.sha256(b"\x00" * 32 + block).digest()]

    def test_empty_gives_hash_of_zero_digest(self):
        assert EO.build_commitments(np.zeros((0, 4))) == [hashlib.sha256(b"\x00" * 32).digest()]

    def test_interval_must_be_positive(self):
        with pytest.raises(ValueError, match="interval"):
            EO.build_commitments(np.ones((2, 2)), k=0)


def test_forge_fixture_digests_are_reference_digests():
    """The reference's own adversarial corpus: honest prover digests reproduce, the
    wrong-model (stale checkpoint) digests differ from the validator's recompute."""
    with open(os.path.join(GOLDEN, "forge_golden.json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, "forge_golden.npz"))
    kinds = {"honest": 0, "wrong-model": 0}
    for m in meta:
        prv, val = arrays[f"prv_{m['i']}"], arrays[f"val_{m['i']}"]
        assert [d.hex() for d in EO.build_commitments(prv)] == m["commitments"]
        assert [d.hex() for d in EO.build_commitments(val)] == m["ref_val_digests"]
        assert EO.verify_commitments(val, m["commitments"]) == (m["kind"] == "honest")
        kinds[m["kind"]] += 1
        assert m["file_verdict"] == ("accept" if m["kind"] == "honest" else "reject")
    assert kinds["honest"] > 0 and kinds["wrong-model"] > 0
