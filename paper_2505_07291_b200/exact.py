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
import threading

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
        a = np.ascontiguousarray(np.asarray(hidden, dtype=np.float64))
        t = torch.from_numpy(a if a.flags.writeable else a.copy())  # torch wants a writable buffer
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
        h = hashlib.sha256(prev)
        h.update(buf[start * row_bytes:stop * row_bytes])   # zero-copy; hashlib drops the GIL
        prev = h.digest()
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


_STAGING: dict = {}
_STAGING_LOCK = threading.Lock()  # one build_commitments_batch at a time uses the staging


def release_staging() -> None:
    """Free the cached device and pinned host staging of ``build_commitments_batch``
    (2 x group_rows x H float64 each, 2.7 GB per buffer at the defaults and H = 5120)."""
    _STAGING.clear()


def _staging(dev, elems: int):
    """Double-buffered device + pinned host float64 staging, reused across calls
    (pinning gigabytes per call would dominate); ``release_staging`` frees it."""
    key = dev.index
    cur = _STAGING.get(key)
    if cur is None or cur[0][0].numel() < elems:
        cur = ([torch.empty(elems, dtype=torch.float64, device=dev) for _ in range(2)],
               [torch.empty(elems, dtype=torch.float64).pin_memory() for _ in range(2)])
        _STAGING[key] = cur
    return cur


def build_commitments_device(hidden, row_offsets, k: int = 32) -> list[list[bytes]]:
    """Exact-mode commitments with the whole SHA-256 chains on the GPU
    (``tl_exact_chains``, one thread per rollout).  Byte-identical to
    ``build_commitments`` per rollout.  Each chain is latency-bound (~38 MB/s per
    rollout), so the kernel time is flat in the rollout count: it passes host SHA-NI
    on all cores at ~700 rollouts (``DEVICE_SHA_MIN_ROLLOUTS``)."""
    if k < 1:
        raise ValueError("interval must be >= 1")
    if not torch.cuda.is_available():
        raise RuntimeError("exact mode needs a CUDA device (no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device())
    if isinstance(hidden, torch.Tensor):
        t = hidden
    else:
        a = np.ascontiguousarray(hidden)
        t = torch.from_numpy(a if a.flags.writeable else a.copy())
    if t.dim() != 2:
        raise ValueError("hidden must be (rows, H)")
    if t.dtype not in _DTYPE_CODE:
        t = t.to(torch.float64)
    t = t.to(dev).contiguous()
    offs = np.asarray(row_offsets, dtype=np.int64)
    n_rows, H = t.shape
    if offs[0] != 0 or offs[-1] != n_rows or np.any(np.diff(offs) < 0):
        raise ValueError("row_offsets must start at 0, be non-decreasing and end at n_rows")
    R = len(offs) - 1
    nd = np.maximum(1, -(-np.diff(offs) // k))
    doff = np.concatenate([[0], np.cumsum(nd)]).astype(np.int64)
    out = torch.empty((max(int(doff[-1]), 1), 32), dtype=torch.uint8, device=dev)
    # keep the device copies referenced until the kernel is enqueued (a temporary's
    # memory would be handed to the next allocation before the launch)
    offs_dev = torch.from_numpy(offs).to(dev)
    doff_dev = torch.from_numpy(doff[:-1].copy()).to(dev)
    if t.numel() == 0:  # every rollout empty: the kernel reads no element, but wants a pointer
        t = torch.zeros(1, dtype=t.dtype, device=dev)
    rc = _ffi.load().tl_exact_chains(t.data_ptr(), _DTYPE_CODE[t.dtype], offs_dev.data_ptr(), R, H, k,
                                     doff_dev.data_ptr(), out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    _ffi.check(rc, "tl_exact_chains")
    host = out.cpu().numpy()
    return [[host[j].tobytes() for j in range(doff[r], doff[r + 1])] for r in range(R)]


# Rollouts from which the GPU chains beat host SHA-NI on all cores
# (tools/bench_exact.py --device-sweep, H=5120, 2048 tokens: 512 -> 0.47 M vs 0.62 M
# tokens/s, 1024 -> 0.93 M vs 0.62 M, 4096 -> 3.46 M vs 0.64 M).
DEVICE_SHA_MIN_ROLLOUTS = 768


def build_commitments_batch(hidden, row_offsets, k: int = 32, threads: int | None = None,
                            group_rows: int = 65536, sha: str = "auto") -> list[list[bytes]]:
    """Exact-mode commitments for many rollouts at once (the validator's batch form).

    ``hidden`` is a (sum T, H) tensor (device or host; bf16 / f16 / f32 / f64) and
    ``row_offsets`` delimits rollouts.  Row groups are rounded on the GPU
    (``tl_round6``), copied to pinned host buffers on a side stream (double
    buffered) and hashed by a thread pool -- hashlib releases the GIL, so the
    serial-per-rollout SHA-256 chains of different rollouts run on all host cores
    while the next group is rounded and copied.  Byte-identical to
    ``build_commitments`` per rollout (rollout.py:51-68)."""
    if sha not in ("auto", "host", "device"):
        raise ValueError("sha must be 'auto', 'host' or 'device'")
    if sha == "device" or (sha == "auto" and len(row_offsets) - 1 >= DEVICE_SHA_MIN_ROLLOUTS):
        return build_commitments_device(hidden, row_offsets, k)
    if k < 1:
        raise ValueError("interval must be >= 1")
    if not torch.cuda.is_available():
        raise RuntimeError("exact mode needs a CUDA device (no CPU fallback)")
    t = hidden if isinstance(hidden, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(hidden))
    if t.dim() != 2:
        raise ValueError("hidden must be (rows, H)")
    if t.dtype not in _DTYPE_CODE:
        t = t.to(torch.float64)
    offs = np.asarray(row_offsets, dtype=np.int64)
    n_rows, H = t.shape
    if offs[0] != 0 or offs[-1] != n_rows or np.any(np.diff(offs) < 0):
        raise ValueError("row_offsets must start at 0, be non-decreasing and end at n_rows")
    dev = torch.device("cuda", torch.cuda.current_device())
    R = len(offs) - 1
    # groups of whole rollouts, ~group_rows rows each
    groups, start = [], 0
    while start < R:
        end = start + 1
        while end < R and offs[end + 1] - offs[start] <= group_rows:
            end += 1
        groups.append((start, end))
        start = end
    max_rows = max((int(offs[e] - offs[b]) for b, e in groups), default=0)
    with _STAGING_LOCK:
        return _batch_locked(t, offs, k, threads, groups, max_rows, H, R, dev)


def _batch_locked(t, offs, k, threads, groups, max_rows, H, R, dev):
    import concurrent.futures as cf
    import os

    lib = _ffi.load()
    side = torch.cuda.Stream(dev)
    dbuf, hbuf = _staging(dev, max(max_rows, 1) * H)
    dbuf = [d[:max(max_rows, 1) * H].view(max(max_rows, 1), H) for d in dbuf]
    hbuf = [h[:max(max_rows, 1) * H].view(max(max_rows, 1), H) for h in hbuf]
    done = [torch.cuda.Event() for _ in range(2)]
    out: list = [None] * R
    pool = cf.ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 1)
    pending: list = [[], []]

    def hash_rollout(r, view):
        out[r] = chain_digests(view, k)

    try:
        for gi, (b, e) in enumerate(groups):
            slot = gi & 1
            for f in pending[slot]:      # host buffer free again?
                f.result()
            pending[slot] = []
            r0, r1 = int(offs[b]), int(offs[e])
            src = t[r0:r1].to(dev, non_blocking=True).contiguous()
            rows = r1 - r0
            if rows:
                rc = lib.tl_round6(src.data_ptr(), _DTYPE_CODE[src.dtype], src.numel(), dbuf[slot].data_ptr(),
                                   torch.cuda.current_stream(dev).cuda_stream)
                _ffi.check(rc, "tl_round6")
            ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                side.wait_event(ready)
                if rows:
                    hbuf[slot][:rows].copy_(dbuf[slot][:rows], non_blocking=True)
                done[slot].record(side)
            done[slot].synchronize()
            host = hbuf[slot].numpy()
            for r in range(b, e):
                a0, a1 = int(offs[r] - r0), int(offs[r + 1] - r0)
                pending[slot].append(pool.submit(hash_rollout, r, host[a0:a1]))
        for slot in (0, 1):
            for f in pending[slot]:
                f.result()
    finally:
        pool.shutdown(wait=True)
    return out
