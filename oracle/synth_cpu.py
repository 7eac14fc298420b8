"""CPU twin of the on-device synthetic generator -- TEST INFRASTRUCTURE ONLY.

Regenerates any row range of the bf16 hidden states produced by
``tl_synth_bf16`` (see ``paper_2505_07291_b200/synth.py`` for the definition),
bit for bit, so parity checks at full benchmark sizes can sample chunks without
copying the whole tensor back to the host.
"""

from __future__ import annotations

import numpy as np

from paper_2505_07291_b200.synth import (
    DIST_MASSIVE, DIST_NORMAL, DIST_ONES, DIST_ZEROS, MASSIVE_SCALE,
    f32_to_bf16_bits, jitter_mix, massive_channels, normal_table, seed_mix,
)

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _lanes(row0: int, n_rows: int, H: int, salt: int) -> np.ndarray:
    G = (H + 3) // 4
    rows = np.arange(row0, row0 + n_rows, dtype=np.uint64)[:, None]
    c = np.arange(H, dtype=np.uint64)[None, :]
    ctr = rows * np.uint64(G) + (c >> np.uint64(2))
    z = mix64_np(ctr + np.uint64(salt))
    return ((z >> ((c & np.uint64(3)) * np.uint64(16))) & np.uint64(0xFFFF)).astype(np.int64)


def synth_bits(row0: int, n_rows: int, H: int, seed: int, dist: int = DIST_NORMAL,
               jitter_thr: int = 0, jitter_seed: int = 0) -> np.ndarray:
    """Rows [row0, row0+n_rows) of the synthetic (rows, H) tensor as uint16 bits."""
    if dist == DIST_ZEROS:
        out = np.zeros((n_rows, H), dtype=np.uint16)
    elif dist == DIST_ONES:
        out = np.full((n_rows, H), 0x3F80, dtype=np.uint16)
    else:
        out = normal_table()[_lanes(row0, n_rows, H, seed_mix(seed))]
        if dist == DIST_MASSIVE:
            for ch in sorted(set(massive_channels(seed, H))):
                f = (out[:, ch].astype(np.uint32) << 16).view(np.float32)
                out[:, ch] = f32_to_bf16_bits(f * np.float32(MASSIVE_SCALE))
        elif dist != DIST_NORMAL:
            raise ValueError(f"unknown dist {dist}")
    if jitter_thr > 0:
        h = _lanes(row0, n_rows, H, jitter_mix(jitter_seed))
        hit = h < jitter_thr
        up = (h & 1) == 1
        mag = out.astype(np.int64) & 0x7FFF
        sign = out.astype(np.int64) & 0x8000
        new = np.where(up & (mag < 0x7F7F), mag + 1, np.where(~up & (mag > 0), mag - 1, mag))
        out = np.where(hit, sign | new, out.astype(np.int64)).astype(np.uint16)
    return out
