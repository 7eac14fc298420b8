"""On-device synthetic hidden states (bench / test input, not the proof path).

A stateless counter-based generator so that any chunk can be regenerated bit for
bit on the CPU (``oracle/synth_cpu.py``) without copying tens of GB off the GPU
(SURVEY.md section 7.3-7).  The mixer is the reference's SplitMix64 finalizer
(``swarm/prng.py:18-23``).

Element (row, c) of a (rows, H) tensor:

    g = c >> 2, lane = c & 3, ctr = row * ceil(H/4) + g
    z = mix64(ctr + seed_mix(seed));  u = (z >> 16*lane) & 0xFFFF
    bits = NORMAL[u]                          # bf16 of Phi^-1((u + 0.5) / 65536)

``dist``: 0 normal, 1 normal with six "massive activation" channels scaled by
200 (f32 multiply, bf16 round-to-nearest-even), 2 all zeros, 3 all ones.
``jitter_thr`` > 0 perturbs ``jitter_thr / 65536`` of the elements by +-1 in the
magnitude bits (the GPU-nondeterminism model for the validator's recompute):
``h = (mix64(ctr + jitter_mix(jseed)) >> 16*lane) & 0xFFFF``; if ``h < jitter_thr``
the magnitude goes up (``h`` odd, below 0x7F7F) or down (``h`` even, above 0).
"""

from __future__ import annotations

import ctypes
import functools
import statistics

import numpy as np

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
SEED_SALT = 0x5851F42D4C957F2D
JITTER_SALT = 0xD1B54A32D192ED03
N_MASSIVE = 6
MASSIVE_SCALE = 200.0

DIST_NORMAL, DIST_MASSIVE, DIST_ZEROS, DIST_ONES = 0, 1, 2, 3
DISTS = {"normal": DIST_NORMAL, "massive": DIST_MASSIVE, "zeros": DIST_ZEROS, "ones": DIST_ONES}


def mix64(z: int) -> int:
    """SplitMix64 finalizer, identical to ``swarm/prng.py:18-23``."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def seed_mix(seed: int) -> int:
    return mix64((seed & MASK64) ^ SEED_SALT)


def jitter_mix(seed: int) -> int:
    return mix64((seed & MASK64) ^ JITTER_SALT)


def massive_channels(seed: int, H: int) -> list[int]:
    sm = seed_mix(seed)
    return [mix64((sm + 0x1000 + m) & MASK64) % H for m in range(N_MASSIVE)]


def f32_to_bf16_bits(f: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bits (NaN kept quiet)."""
    u = np.asarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF
    r = np.where(nan, ((u >> 16) | 0x40) & 0xFFFF, r)
    return r.astype(np.uint16)


@functools.lru_cache(maxsize=1)
def normal_table() -> np.ndarray:
    """65536 bf16 bit patterns: NORMAL[u] = bf16(Phi^-1((u + 0.5) / 65536))."""
    nd = statistics.NormalDist()
    vals = np.array([nd.inv_cdf((u + 0.5) / 65536.0) for u in range(65536)], dtype=np.float64)
    return f32_to_bf16_bits(vals.astype(np.float32))


_TABLES: dict = {}


def synth_device(n_rows: int, H: int, seed: int, dist=DIST_NORMAL, *, row0: int = 0,
                 jitter_thr: int = 0, jitter_seed: int = 0, device=None, out=None):
    """Generate rows [row0, row0+n_rows) of the synthetic tensor on the GPU (bf16)."""
    import torch

    from . import _ffi

    if isinstance(dist, str):
        dist = DISTS[dist]
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    tab = _TABLES.get(dev.index)
    if tab is None:
        tab = _TABLES[dev.index] = torch.from_numpy(normal_table().view(np.int16)).to(dev)
    if out is None:
        out = torch.empty((n_rows, H), dtype=torch.bfloat16, device=dev)
    mv = (ctypes.c_int32 * N_MASSIVE)(*massive_channels(seed, H))
    rc = _ffi.load().tl_synth_bf16(out.data_ptr(), row0, n_rows, H, seed_mix(seed), int(dist), tab.data_ptr(),
                                   ctypes.cast(mv, ctypes.c_void_p), int(jitter_thr), jitter_mix(jitter_seed),
                                   torch.cuda.current_stream(dev).cuda_stream)
    _ffi.check(rc, "tl_synth_bf16")
    return out
