"""TOPLOC proofs on the rollout-file wire format.

The reference carries one commitment per ``commit_interval`` output tokens as a hex
string in ``RolloutRecord.commitments`` (``worker/files.py:37``), checks the count
``ceil(T / commit_interval)`` (``files.py:184-186``) and trusts the header's interval
(``validator/checks.py:211``).  A 258-byte TOPLOC proof is 516 hex characters in the
same field with the same count, so the file schema does not change; TOPLOC mode
additionally requires ``commit_interval == 32`` because proofs are defined over
32-token chunks.

``encode`` turns a proof batch into per-rollout hex lists; ``decode`` validates and
packs per-rollout hex lists back into the (n_chunks, 258) uint8 layout ``tl_verify``
reads; a modulus field that is neither 0 (unprovable chunk) nor a prime in
[32771, 65497] is a format error, since such a "proof" (p = 2, say) would match
any activations.  Errors raise ``ProofFormatError`` (a ``ValueError``, like the reference's
``RolloutSchemaError``) naming the rollout and item.
"""

from __future__ import annotations

import numpy as np

TOPLOC_INTERVAL = 32
PROOF_BYTES = 258
PROOF_HEX = 2 * PROOF_BYTES


class ProofFormatError(ValueError):
    """A commitment list that cannot be a TOPLOC proof list."""


def expected_count(n_tokens: int, interval: int = TOPLOC_INTERVAL) -> int:
    """Commitments per record: ceil(T / interval) (``files.py:184-186``)."""
    if interval < 1:
        raise ValueError("interval must be >= 1")
    return -(-int(n_tokens) // int(interval))


def check_interval(commit_interval: int) -> None:
    if int(commit_interval) != TOPLOC_INTERVAL:
        raise ProofFormatError(f"commit_interval {commit_interval} != {TOPLOC_INTERVAL} (TOPLOC chunks)")


def _as_array(proofs) -> np.ndarray:
    if hasattr(proofs, "proofs"):  # api.ProofBatch
        proofs = proofs.proofs
    if hasattr(proofs, "detach"):  # torch tensor (device or host)
        proofs = proofs.detach().cpu().numpy()
    arr = np.ascontiguousarray(np.asarray(proofs, dtype=np.uint8))
    if arr.ndim != 2 or arr.shape[1] != PROOF_BYTES:
        raise ProofFormatError(f"proofs must be (n, {PROOF_BYTES}) bytes, got {arr.shape}")
    return arr


def encode(proofs, row_offsets=None, chunk_offsets=None) -> list[list[str]]:
    """(n_chunks, 258) proofs -> per-rollout lists of 516-char lowercase hex strings.

    ``chunk_offsets`` (or ``row_offsets``, converted with the 32-token rule) gives each
    rollout's proof range; without either, one rollout holds every proof."""
    if chunk_offsets is None and hasattr(proofs, "chunk_offsets"):
        chunk_offsets = proofs.chunk_offsets
    arr = _as_array(proofs)
    if chunk_offsets is None:
        if row_offsets is None:
            chunk_offsets = [0, arr.shape[0]]
        else:
            lens = np.diff(np.asarray(row_offsets, dtype=np.int64))
            chunk_offsets = np.concatenate([[0], np.cumsum(-(-lens // TOPLOC_INTERVAL))])
    co = np.asarray(chunk_offsets, dtype=np.int64)
    if co[0] != 0 or co[-1] != arr.shape[0] or np.any(np.diff(co) < 0):
        raise ProofFormatError("chunk offsets do not tile the proofs")
    text = arr.tobytes().hex()  # one C-level hex pass, then string slices
    rows = [text[i:i + PROOF_HEX] for i in range(0, len(text), PROOF_HEX)]
    return [rows[int(co[r]):int(co[r + 1])] for r in range(len(co) - 1)]


def decode(commitments, n_tokens=None, interval: int = TOPLOC_INTERVAL) -> tuple[np.ndarray, np.ndarray]:
    """Per-rollout hex lists -> ((n_chunks, 258) uint8, chunk offsets).

    Checks each item is 516 hex characters and, when ``n_tokens`` (one per rollout)
    is given, that every list has ``ceil(T / interval)`` items."""
    check_interval(interval)
    counts, texts = [], []
    for r, items in enumerate(commitments):
        items = list(items)
        if n_tokens is not None:
            want = expected_count(n_tokens[r], interval)
            if len(items) != want:
                raise ProofFormatError(f"rollout {r}: {len(items)} commitments, expected {want}")
        for i, s in enumerate(items):
            if not isinstance(s, str) or len(s) != PROOF_HEX:
                raise ProofFormatError(f"rollout {r} item {i}: not a {PROOF_HEX}-char proof")
        texts.extend(items)
        counts.append(len(items))
    try:  # one C-level parse of the concatenation
        blob = bytes.fromhex("".join(texts))
    except ValueError:
        bad = next(i for i, s in enumerate(texts) if not _is_hex(s))
        r = int(np.searchsorted(np.cumsum(counts), bad, side="right"))
        raise ProofFormatError(f"rollout {r} item {bad - int(np.sum(counts[:r]))}: not hex") from None
    arr = np.frombuffer(blob, dtype=np.uint8).reshape(-1, PROOF_BYTES).copy()
    p = arr[:, 0].astype(np.int64) << 8 | arr[:, 1]
    bad = np.nonzero((p != 0) & ~_PROVER_MODULUS[p])[0]
    if bad.size:
        q = int(bad[0])
        r = int(np.searchsorted(np.cumsum(counts), q, side="right"))
        raise ProofFormatError(f"rollout {r} item {q - int(np.sum(counts[:r]))}: modulus {int(p[q])} is not a "
                               f"prime in [{P_MIN}, {P_MAX}]")
    return arr, np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)


P_MIN, P_MAX = 32771, 65497


def _prover_moduli() -> np.ndarray:
    """Mask over u16 values: True for the moduli a prover emits (primes in [P_MIN, P_MAX])."""
    sieve = np.ones(1 << 16, dtype=bool)
    sieve[:2] = False
    for i in range(2, 256):
        if sieve[i]:
            sieve[i * i::i] = False
    sieve[:P_MIN] = False
    sieve[P_MAX + 1:] = False
    return sieve


_PROVER_MODULUS = _prover_moduli()


def _is_hex(s: str) -> bool:
    try:
        bytes.fromhex(s)
        return True
    except ValueError:
        return False


def modulus(proof_hex_or_bytes) -> int:
    """The proof's modulus field (big-endian u16): a prime in [32771, 65497], or 0 for an
    unprovable chunk (``decode`` rejects anything else; ``tl_verify`` marks it a bad proof)."""
    b = bytes.fromhex(proof_hex_or_bytes) if isinstance(proof_hex_or_bytes, str) else bytes(proof_hex_or_bytes)
    return int.from_bytes(b[:2], "big")


__all__ = ["ProofFormatError", "TOPLOC_INTERVAL", "PROOF_BYTES", "PROOF_HEX", "expected_count", "check_interval",
           "encode", "decode", "modulus"]
