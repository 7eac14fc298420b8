"""Full-size parity helpers (tests only): compare the GPU's select / commit / verify outputs
on sampled chunks of a large device-resident batch with the CPU oracle.

The sampled chunks' bytes are copied back from the device, so the oracle sees exactly
the prover and validator states the kernels saw (whatever generated them: the
counter-based synthesiser, an fp8 round trip, a tampered row)."""

from __future__ import annotations

import math

import numpy as np
import torch

from oracle import toploc_oracle as TO

CHUNK, TOPK = 32, 128


def chunk_rows(offs: np.ndarray, C: int = CHUNK):
    """(first row, rows) of every chunk, in chunk order."""
    out = []
    for r in range(len(offs) - 1):
        T = int(offs[r + 1] - offs[r])
        for s in range(0, T, C):
            out.append((int(offs[r]) + s, min(C, T - s)))
    return out


def fetch_chunks(h: torch.Tensor, table, js) -> list[np.ndarray]:
    """Flattened uint16 bits of chunks js of the (rows, H) device tensor h."""
    H = h.shape[1]
    rows = [(table[j][0], table[j][1]) for j in js]
    idx = torch.tensor([r0 + i for r0, n in rows for i in range(n)], dtype=torch.int64, device=h.device)
    flat = h.view(torch.int16).index_select(0, idx).cpu().numpy().view(np.uint16)
    out, o = [], 0
    for _, n in rows:
        out.append(flat[o:o + n].reshape(-1).copy())
        o += n
    assert o * 1 == flat.shape[0] and all(a.size == n * H for a, (_, n) in zip(out, rows))
    return out


def boundary_chunks(offs: np.ndarray, C: int = CHUNK, every: int = 1) -> list[int]:
    """First and last chunk of every `every`-th rollout."""
    co = np.concatenate([[0], np.cumsum(-(-np.diff(offs) // C))])
    js = set()
    for r in range(0, len(offs) - 1, every):
        if co[r + 1] > co[r]:
            js.update((int(co[r]), int(co[r + 1] - 1)))
    return sorted(js)


def check_prove(prv: torch.Tensor, table, js, idx: torch.Tensor, bits: torch.Tensor, proofs: torch.Tensor):
    """Oracle prove of chunks js; returns (oracle proofs by chunk, list of mismatching chunks)."""
    chunks = fetch_chunks(prv, table, js)
    oi, ov, op = TO.prove_chunks(chunks, TOPK)
    sel = torch.tensor(js, dtype=torch.int64, device=idx.device)
    gi = idx.index_select(0, sel).cpu().numpy()
    gb = bits.index_select(0, sel).cpu().numpy().view(np.uint16)
    gp = proofs.index_select(0, sel).cpu().numpy()
    bad = []
    for t, j in enumerate(js):
        kk = len(oi[t])
        if not (np.array_equal(gi[t, :kk], oi[t]) and np.all(gi[t, kk:] == -1) and np.array_equal(gb[t, :kk], ov[t])
                and gp[t].tobytes() == op[t]):
            bad.append(j)
    return dict(zip(js, op)), bad


def check_verify(val: torch.Tensor, table, js, proofs_by_chunk, stats_host: np.ndarray, chunk_accept: np.ndarray,
                 th=TO.Thresholds()):
    """Oracle verify of chunks js against the given proofs; returns (mismatching chunks,
    oracle accept per chunk).  Compared: exp_mismatch, n_match, mant_sum, median,
    mean (exactly; 1e-6 relative is the north-star bound), chunk verdict."""
    chunks = fetch_chunks(val, table, js)
    bad, acc = [], {}
    for t, j in enumerate(js):
        o = TO.verify_chunk(chunks[t], proofs_by_chunk[j], TOPK, th)
        g = stats_host[j]
        same = (int(g["exp_mismatch"]), int(g["n_match"]), int(g["mant_sum"]), float(g["mant_median"]),
                bool(g["flags"] & 1), bool(chunk_accept[j])) == (o.exp_mismatch, o.n_match, o.mant_sum,
                                                                o.mant_median, o.accept, o.accept)
        gm = float(g["mant_mean"])
        same = same and ((math.isinf(gm) and math.isinf(o.mant_mean)) or
                         (gm == o.mant_mean and abs(gm - o.mant_mean) <= 1e-6 * max(1.0, abs(o.mant_mean))))
        if not same:
            bad.append(j)
        acc[j] = o.accept
    return bad, acc
