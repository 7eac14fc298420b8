"""TOPLOC prove/verify CPU oracle -- TEST INFRASTRUCTURE ONLY (never shipped).

Restates, in numpy + Python ints, the algorithm the CUDA path implements, so the
GPU results can be checked bit for bit.  Only ``tests/``, ``__graft_entry__.smoke``
and ``bench.py`` (cpu_baseline leg / ``--impl reference`` arm) may import it.

Provenance and pinning
----------------------
* Chunking follows the reference's commitment chunking: output rows only, blocks
  of ``C`` rows, final partial block included, ``ceil(T/C)`` items per rollout
  (``swarm/worker/rollout.py:51-68``; count contract ``swarm/worker/files.py:184-186``).
* The proof replaces the reference's per-chunk SHA-256 digest
  (``rollout.py:66``) and is carried in the same ``RolloutRecord.commitments``
  slot (``files.py:37``); verification replaces the digest-list compare of
  ``swarm/validator/checks.py:209-213``.
* The TOPLOC arithmetic itself (top-k, GF(p) polynomial, 258-byte proof,
  exponent / mantissa statistics) lives in the third-party ``toploc`` package
  (PrimeIntellect-ai/toploc, TOPLOC paper arXiv:2501.16007), which is NOT a
  dependency of the reference (``pkg/pyproject.toml:10-19``), not vendored and
  not installed here.  PARITY AGAINST UPSTREAM ``toploc`` IS UNPINNED.  The
  choices below are pinned by this oracle
  and cross-checked by independent restatements in ``tests/test_oracle_toploc.py``
  (stable full sort for top-k, Lagrange-over-Python-ints for the polynomial).

Pinned semantics (DESIGN.md section 3 repeats them)
----------------------------------------------------
1. Top-k: chunk flattened row-major (flat index ``i = r*H + c``); order key is the
   15-bit magnitude pattern ``bits & 0x7FFF`` descending, then flat index
   ascending.  ``kk = min(K, rows*H)`` entries.  NaN sorts above Inf (by bits).
2. Modulus: the largest prime ``p`` in ``[32771, 65497]`` for which the residues
   ``idx mod p`` are pairwise distinct; ``p = 0`` if none (unprovable chunk).
3. Points ``x_i = idx_i mod p``, ``y_i = bits_i mod p``; coefficients
   ``c_0..c_{kk-1}`` of the unique polynomial of degree < kk over GF(p) with
   ``P(x_i) = y_i``; ``c_k = 0`` for ``k >= kk``.
4. Proof bytes: ``p`` as u16 big-endian, then ``c_0 .. c_{K-1}`` as u16 big-endian
   (2 + 2K = 258 bytes for K = 128).
5. Verify: re-select top-kk on the validator chunk; ``claimed = P(idx mod p)``
   (Horner mod p, coefficients reduced mod p), ``observed = bits mod p``;
   exponent ``(v >> 7) & 0xFF``, mantissa ``v & 0x7F``; ``exp_mismatch`` counts
   exponent differences; mantissa |diff| over exponent-equal points gives
   ``mean = sum / n`` (f64) and ``median`` = ``statistics.median`` (average of
   the two middle values).  No exponent-equal point, or a proof modulus that is not
   a prime in ``[32771, 65497]`` (a bad proof): mean = median = +inf.
6. Chunk accepted iff ``exp_mismatch <= max_exp_mismatch and mean <=
   max_mant_mean and median <= max_mant_median``; a rollout is accepted iff all
   its chunks are.
"""

from __future__ import annotations

import math
import statistics
from dataclasses import dataclass

import numpy as np

P_MAX = 65497          # 0xFFD9, prime
P_MIN = 32771          # smallest prime above 2**15
SORT_IDX_BITS = 24     # flat index must stay below 2**24 inside a chunk


def _primes_desc(lo: int = P_MIN, hi: int = P_MAX) -> list[int]:
    sieve = bytearray([1]) * (hi + 1)
    sieve[0:2] = b"\x00\x00"
    for i in range(2, int(hi ** 0.5) + 1):
        if sieve[i]:
            sieve[i * i::i] = bytearray(len(sieve[i * i::i]))
    return [p for p in range(hi, lo - 1, -1) if sieve[p]]


PRIMES_DESC = _primes_desc()
PRIME_SET = frozenset(PRIMES_DESC)


@dataclass(frozen=True)
class Thresholds:
    """Verdict thresholds (explicit parameters; defaults documented in DESIGN.md)."""

    max_exp_mismatch: int = 29      # measured defaults, as api.Thresholds (profiles/r02_calibration.json)
    max_mant_mean: float = 7.0
    max_mant_median: float = 5.0


@dataclass
class ChunkStats:
    exp_mismatch: int
    n_match: int
    mant_sum: int
    mant_mean: float
    mant_median: float
    accept: bool


# --------------------------------------------------------------------------- chunking
def chunk_table(row_offsets, C: int = 32):
    """[(rollout, first_row, n_rows)] in rollout order (rollout.py:64 blocking)."""
    out = []
    offs = [int(v) for v in row_offsets]
    for r in range(len(offs) - 1):
        T = offs[r + 1] - offs[r]
        for s in range(0, T, C):
            out.append((r, offs[r] + s, min(C, T - s)))
    return out


# --------------------------------------------------------------------------- top-k
def sort_keys(bits: np.ndarray) -> np.ndarray:
    """Composite int64 key: (bits & 0x7FFF) << 24 | (2^24 - 1 - idx); unique per chunk."""
    bits = np.asarray(bits, dtype=np.uint16)
    n = bits.shape[-1]
    assert n <= (1 << SORT_IDX_BITS)
    idx = np.arange(n, dtype=np.int64)
    return ((bits.astype(np.int64) & 0x7FFF) << SORT_IDX_BITS) | ((1 << SORT_IDX_BITS) - 1 - idx)


def select_topk(bits: np.ndarray, K: int = 128):
    """Top-kk of one flattened chunk -> (idx int64[kk], bits uint16[kk]) in rank order."""
    bits = np.asarray(bits, dtype=np.uint16).reshape(-1)
    kk = min(K, bits.size)
    s = sort_keys(bits)
    part = np.argpartition(-s, kk - 1)[:kk] if kk < bits.size else np.arange(bits.size)
    order = part[np.argsort(-s[part], kind="stable")]
    return order.astype(np.int64), bits[order]


def select_topk_batch(bits2d: np.ndarray, K: int = 128):
    """Vectorised select over equal-size chunks: bits2d (m, n) -> idx (m, kk), bits (m, kk)."""
    bits2d = np.asarray(bits2d, dtype=np.uint16)
    m, n = bits2d.shape
    kk = min(K, n)
    s = sort_keys(bits2d)
    if kk < n:
        part = np.argpartition(-s, kk - 1, axis=1)[:, :kk]
    else:
        part = np.broadcast_to(np.arange(n), (m, n)).copy()
    ps = np.take_along_axis(s, part, axis=1)
    order = np.take_along_axis(part, np.argsort(-ps, axis=1, kind="stable"), axis=1)
    return order.astype(np.int64), np.take_along_axis(bits2d, order, axis=1)


# --------------------------------------------------------------------------- modulus
def find_modulus(idx) -> int:
    idx = np.asarray(idx, dtype=np.int64)
    for p in PRIMES_DESC:
        if np.unique(idx % p).size == idx.size:
            return p
    return 0


def find_modulus_batch(idx2d: np.ndarray) -> np.ndarray:
    idx2d = np.asarray(idx2d, dtype=np.int64)
    m = idx2d.shape[0]
    P = np.zeros(m, dtype=np.int64)
    todo = np.arange(m)
    for p in PRIMES_DESC:
        if todo.size == 0:
            break
        r = np.sort(idx2d[todo] % p, axis=1)
        ok = np.all(np.diff(r, axis=1) != 0, axis=1) if r.shape[1] > 1 else np.ones(todo.size, bool)
        P[todo[ok]] = p
        todo = todo[~ok]
    return P


# --------------------------------------------------------------------------- GF(p) interpolation
_INV_CACHE: dict[int, np.ndarray] = {}


def _inv_table(p: int) -> np.ndarray:
    t = _INV_CACHE.get(p)
    if t is None:
        a = np.arange(p, dtype=np.int64)
        r = np.ones(p, dtype=np.int64)
        e = p - 2
        b = a.copy()
        while e:
            if e & 1:
                r = r * b % p
            b = b * b % p
            e >>= 1
        r[0] = 0
        t = _INV_CACHE[p] = r
    return t


def interpolate_newton(x, y, p: int) -> list[int]:
    """Newton divided differences then Newton->monomial, Python ints (scalar)."""
    x = [int(v) for v in x]
    c = [int(v) % p for v in y]
    n = len(x)
    for j in range(1, n):
        for i in range(n - 1, j - 1, -1):
            c[i] = (c[i] - c[i - 1]) * pow((x[i] - x[i - j]) % p, p - 2, p) % p
    poly = [0] * n
    poly[0] = c[n - 1]
    for i in range(n - 2, -1, -1):
        new = [0] * n
        for k in range(n):
            new[k] = ((poly[k - 1] if k else 0) - x[i] * poly[k]) % p
        new[0] = (new[0] + c[i]) % p
        poly = new
    return poly


def interpolate_lagrange(x, y, p: int) -> list[int]:
    """Independent restatement: sum_i y_i * prod_{j!=i} (X - x_j)/(x_i - x_j)."""
    x = [int(v) for v in x]
    n = len(x)
    out = [0] * n
    for i in range(n):
        num = [1]
        den = 1
        for j in range(n):
            if j == i:
                continue
            num = [((num[k - 1] if k else 0) - x[j] * (num[k] if k < len(num) else 0)) % p
                   for k in range(len(num) + 1)]
            den = den * (x[i] - x[j]) % p
        w = int(y[i]) % p * pow(den, p - 2, p) % p
        for k in range(n):
            out[k] = (out[k] + w * num[k]) % p
    return out


def interpolate_batch(X: np.ndarray, Y: np.ndarray, P: np.ndarray) -> np.ndarray:
    """Vectorised Newton over rows; X, Y (m, n) already reduced mod P (m,), P prime."""
    X = np.asarray(X, dtype=np.int64)
    c = np.asarray(Y, dtype=np.int64).copy()
    P = np.asarray(P, dtype=np.int64)
    m, n = X.shape
    out = np.zeros((m, n), dtype=np.int64)
    for p in np.unique(P):
        rows = np.nonzero(P == p)[0]
        p = int(p)
        inv = _inv_table(p)
        x = X[rows]
        cc = c[rows] % p
        for j in range(1, n):
            num = (cc[:, j:] - cc[:, j - 1:-1]) % p
            den = (x[:, j:] - x[:, :-j]) % p
            cc[:, j:] = num * inv[den] % p
        poly = np.zeros((rows.size, n), dtype=np.int64)
        poly[:, 0] = cc[:, n - 1]
        for i in range(n - 2, -1, -1):
            shifted = np.zeros_like(poly)
            shifted[:, 1:] = poly[:, :-1]
            poly = (shifted - x[:, i:i + 1] * poly) % p
            poly[:, 0] = (poly[:, 0] + cc[:, i]) % p
        out[rows] = poly
    return out


def proof_bytes(p: int, coeffs, K: int = 128) -> bytes:
    c = [int(v) for v in coeffs] + [0] * (K - len(coeffs))
    return int(p).to_bytes(2, "big") + b"".join(int(v).to_bytes(2, "big") for v in c)


def parse_proof(proof: bytes, K: int = 128):
    if len(proof) != 2 + 2 * K:
        raise ValueError(f"proof must be {2 + 2 * K} bytes, got {len(proof)}")
    a = np.frombuffer(proof, dtype=">u2").astype(np.int64)
    return int(a[0]), a[1:]


def eval_poly(coeffs, p: int, x) -> np.ndarray:
    x = np.asarray(x, dtype=np.int64) % p
    r = np.zeros_like(x)
    for c in np.asarray(coeffs, dtype=np.int64)[::-1]:
        r = (r * x + int(c)) % p
    return r


# --------------------------------------------------------------------------- prove
def prove_chunks(bits2d_list, K: int = 128, batch: int = 256):
    """List of flattened chunks (uint16) -> (idx list, bits list, proofs list)."""
    idxs, vals, proofs = [], [], []
    by_size: dict[int, list[int]] = {}
    for j, b in enumerate(bits2d_list):
        by_size.setdefault(int(np.asarray(b).size), []).append(j)
    res: dict[int, tuple] = {}
    groups = [(n, js[i:i + batch]) for n, js in by_size.items() for i in range(0, len(js), batch)]
    for n, js in groups:
        B = np.stack([np.asarray(bits2d_list[j], dtype=np.uint16).reshape(-1) for j in js])
        I, V = select_topk_batch(B, K)
        P = find_modulus_batch(I)
        Pc = np.where(P == 0, 1, P)[:, None]
        coeffs = np.zeros((len(js), I.shape[1]), dtype=np.int64)
        ok = P != 0
        if ok.any():
            coeffs[ok] = interpolate_batch(I[ok] % Pc[ok], V[ok].astype(np.int64) % Pc[ok], P[ok])
        for t, j in enumerate(js):
            res[j] = (I[t], V[t], proof_bytes(int(P[t]), coeffs[t] if P[t] else [], K))
    for j in range(len(bits2d_list)):
        idxs.append(res[j][0])
        vals.append(res[j][1])
        proofs.append(res[j][2])
    return idxs, vals, proofs


def _chunks_of(hidden_bits: np.ndarray, row_offsets, C: int):
    H = hidden_bits.shape[1]
    tab = chunk_table(row_offsets, C)
    return tab, [hidden_bits[s:s + n].reshape(-1) for (_, s, n) in tab]


def build_proofs(hidden_bits: np.ndarray, row_offsets, C: int = 32, K: int = 128):
    """hidden_bits (rows, H) uint16 -> list (per rollout) of list of 258-byte proofs."""
    hidden_bits = np.asarray(hidden_bits, dtype=np.uint16)
    tab, chunks = _chunks_of(hidden_bits, row_offsets, C)
    _, _, proofs = prove_chunks(chunks, K)
    out = [[] for _ in range(len(row_offsets) - 1)]
    for (r, _, _), pr in zip(tab, proofs):
        out[r].append(pr)
    return out


# --------------------------------------------------------------------------- verify
def chunk_stats(claimed: np.ndarray, observed: np.ndarray, th: Thresholds) -> ChunkStats:
    ce, oe = (claimed >> 7) & 0xFF, (observed >> 7) & 0xFF
    eq = ce == oe
    mism = int(np.count_nonzero(~eq))
    diffs = [int(v) for v in np.abs((claimed[eq] & 0x7F) - (observed[eq] & 0x7F))]
    if diffs:
        s = sum(diffs)
        mean = s / len(diffs)
        median = float(statistics.median(diffs))
    else:
        s, mean, median = 0, math.inf, math.inf
    acc = (mism <= th.max_exp_mismatch and mean <= th.max_mant_mean
           and median <= th.max_mant_median)
    return ChunkStats(mism, len(diffs), s, mean, median, bool(acc))


def verify_chunk(bits_chunk, proof: bytes, K: int = 128, th: Thresholds = Thresholds()) -> ChunkStats:
    idx, vals = select_topk(bits_chunk, K)
    p, coeffs = parse_proof(proof, K)
    if p not in PRIME_SET:  # only a prover modulus is a proof (p = 2 would match any exponent)
        return ChunkStats(len(idx), 0, 0, math.inf, math.inf, False)
    claimed = eval_poly(coeffs % p, p, idx)
    observed = vals.astype(np.int64) % p
    return chunk_stats(claimed, observed, th)


def verify_proofs(hidden_bits: np.ndarray, row_offsets, proofs, C: int = 32, K: int = 128,
                  th: Thresholds = Thresholds()):
    """-> (list of ChunkStats in chunk order, list of per-rollout accept bools)."""
    hidden_bits = np.asarray(hidden_bits, dtype=np.uint16)
    tab, chunks = _chunks_of(hidden_bits, row_offsets, C)
    flat = [p for per in proofs for p in per]
    if len(flat) != len(tab):
        raise ValueError(f"expected {len(tab)} proofs, got {len(flat)}")
    stats = [verify_chunk(ch, pr, K, th) for ch, pr in zip(chunks, flat)]
    verdict = [True] * (len(row_offsets) - 1)
    for (r, _, _), st in zip(tab, stats):
        verdict[r] = verdict[r] and st.accept
    return stats, verdict
