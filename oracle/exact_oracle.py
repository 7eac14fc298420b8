"""Exact-mode commitment oracle -- TEST INFRASTRUCTURE ONLY (never shipped).

Restates the reference's ``build_commitments`` (``swarm/worker/rollout.py:51-68``)
and ``ZERO_DIGEST`` / ``sha256`` (``swarm/wire.py:18,25-26``):

    d_{-1} = 0^32,  d_j = SHA-256(d_{j-1} || LE-f64(round(h[jk:(j+1)k], 6)))

``max(1, ceil(T/k))`` digests; ``T == 0`` yields ``[SHA-256(0^32)]``.  Parity is
PINNED: ``tests/golden/exact_golden.json`` holds digests produced by the reference
itself (``tests/golden/make_golden.py``) and ``tests/test_oracle_exact.py`` checks
this restatement against them.
"""

from __future__ import annotations

import hashlib

import numpy as np

ZERO_DIGEST = b"\x00" * 32


def round6(hidden) -> np.ndarray:
    """``np.round(x, 6)`` -- numpy computes rint(x * 1e6) / 1e6 (rollout.py:65)."""
    return np.round(np.asarray(hidden, dtype=np.float64), 6)


def build_commitments(hidden, k: int = 32) -> list[bytes]:
    if k < 1:
        raise ValueError("interval must be >= 1")          # rollout.py:59-60
    hidden = np.asarray(hidden, dtype=np.float64)
    out, prev = [], ZERO_DIGEST
    for start in range(0, max(len(hidden), 1), k):         # rollout.py:64
        block = round6(hidden[start:start + k])
        prev = hashlib.sha256(prev + np.ascontiguousarray(block, dtype="<f8").tobytes()).digest()
        out.append(prev)
    return out


def verify_commitments(hidden, commitments_hex, k: int = 32) -> bool:
    """The digest-list compare of ``swarm/validator/checks.py:209-213``."""
    return [d.hex() for d in build_commitments(hidden, k)] == list(commitments_hex)
