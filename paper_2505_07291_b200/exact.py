"""Exact-mode commitments: the reference's own scheme, byte for byte.

``build_commitments(hidden, k)`` reproduces ``swarm/worker/rollout.py:51-68``:

    d_{-1} = 0^32 (wire.py:18),  d_j = SHA-256(d_{j-1} || LE-f64(round(h[jk:(j+1)k], 6)))

The data-parallel half -- ``round(x, 6)`` == ``rint(x * 1e6) / 1e6`` in float64
for every element -- runs on the GPU (``tl_round6``).  The SHA-256 chain is
inherently serial per rollout (each block hashes the previous digest), so it runs
on the host over the rounded bytes (hashlib, SHA-NI); SURVEY.md section 7.3-6
explains why a thread-per-chain GPU SHA cannot beat it.  This is the designed
split, not a fallback: without the CUDA library the call raises.
"""

from __future__ import annotations

import hashlib

import numpy as np
import torch

from . import _ffi

ZERO_DIGEST = b"\x00" * 32
_DTYPE_CODE = {torch.float64: 0, torch.float32: 1, torch.bfloat16: 2, torch.float16: 3}


def round6_device(hidden, device=None) -> torch.Tensor:
    """GPU ``np.round(x, 6)`` in float64; returns a device float64 tensor."""
    if not torch.cuda.is_available():
        raise RuntimeError("exact mode needs a CUDA device (no CPU fallback)")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if isinstance(hidden, torch.Tensor):
        t = hidden
        if t.dtype not in _DTYPE_CODE:
            t = t.to(torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(hidden, dtype=np.float64)))
    t = t.to(dev, non_blocking=True).contiguous()
    out = torch.empty(t.shape, dtype=torch.float64, device=dev)
    lib = _ffi.load()
    rc = lib.tl_round6(t.data_ptr(), _DTYPE_CODE[t.dtype], t.numel(), out.data_ptr(),
                       torch.cuda.current_stream(dev).cuda_stream)
    _ffi.check(rc, "tl_round6")
    return out


def chain_digests(rounded: np.ndarray, k: int) -> list[bytes]:
    """Host SHA-256 chain over k-row blocks of an already-rounded float64 array."""
    rows = rounded.shape[0] if rounded.ndim else 1
    data = np.ascontiguousarray(rounded, dtype="<f8")
    row_bytes = data[:1].nbytes if rows else 0
    buf = memoryview(data.reshape(-1).view(np.uint8)) if data.size else memoryview(b"")
    out, prev = [], ZERO_DIGEST
    for start in range(0, max(rows, 1), k):
        stop = min(start + k, rows)
        prev = hashlib.sha256(prev + bytes(buf[start * row_bytes:stop * row_bytes])).digest()
        out.append(prev)
    return out


def build_commitments(hidden, k: int = 32) -> list[bytes]:
    """Drop-in for ``swarm.worker.rollout.build_commitments`` (same bytes, same errors)."""
    if k < 1:
        raise ValueError("interval must be >= 1")          # rollout.py:59-60
    if isinstance(hidden, torch.Tensor):
        shape = tuple(hidden.shape)
    else:
        hidden = np.asarray(hidden, dtype=np.float64)      # rollout.py:61
        shape = hidden.shape
    if len(shape) == 0:
        raise ValueError("hidden must have at least one dimension")
    rounded = round6_device(hidden).cpu().numpy().reshape(shape)
    return chain_digests(rounded, k)
