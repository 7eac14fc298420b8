"""Python host API of the TOPLOC prove / verify path (CUDA through the C ABI).

Reference-facing names (the reference binds its path by name, see
``include/toploc_b200.h``):

* ``build_commitments(hidden, k=32)``  -- exact mode, byte-identical to
  ``swarm/worker/rollout.py:51-68`` (GPU ``round(x, 6)`` + serialisation, host
  SHA-256 chain, see ``exact.py``).
* ``build_proofs(hidden, row_offsets, chunk=32, topk=128)`` -- TOPLOC prove: one
  258-byte proof per 32-row chunk, ``ceil(T/32)`` per rollout, the same count the
  rollout-file schema requires for ``commitments`` (``swarm/worker/files.py:184-186``).
* ``verify_proofs(hidden, row_offsets, proofs, ...)`` -- TOPLOC verify, the
  replacement of the digest compare at ``swarm/validator/checks.py:209-213``.

``ToplocEngine`` is the device-resident form (inputs and outputs stay in HBM;
this is what the benchmark times).  There is no CPU fallback: without a CUDA
device or the in-tree library every call raises.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _ffi

CHUNK = 32
TOPK = 128

STATS_DTYPE = np.dtype([("exp_mismatch", "<u4"), ("n_match", "<u4"), ("mant_sum", "<u4"),
                        ("flags", "<u4"), ("mant_mean", "<f8"), ("mant_median", "<f8")])
assert STATS_DTYPE.itemsize == ctypes.sizeof(_ffi.ChunkStats) == 32


@dataclass(frozen=True)
class Thresholds:
    """Chunk accepted iff exp_mismatch <= max_exp_mismatch, mean <= max_mant_mean and
    median <= max_mant_median.

    Defaults are measured (tools/calibrate_thresholds.py, profiles/r02_calibration.json):
    on a hidden-5120 Llama-shaped bf16 model, honest recomputations (prefill vs decode
    kernels, other batch shapes, the math attention backend, an fp32 model) reach at most
    18 exponent mismatches, mean 2.84 and median 2 per chunk over 3072 chunks each; the
    defaults are those maxima x 1.5 + 2, rounded up.  They reject every rollout of
    fp8-e4m3 weights, weights perturbed by 1 % of their std, another model and one layer
    fewer (as do the paper's values recalled in ``paper()``, which pass 88 % of the 1 %
    perturbation's chunks and 43 of 48 rollouts of fp8-rounded activations, against 5)."""

    max_exp_mismatch: int = 29
    max_mant_mean: float = 7.0
    max_mant_median: float = 5.0

    @classmethod
    def paper(cls) -> "Thresholds":
        """The thresholds as recalled from the TOPLOC paper (>= 90 of 128 exponents agree,
        mean <= 10, median <= 8); not checkable here (upstream toploc is absent)."""
        return cls(38, 10.0, 8.0)

    def to_c(self) -> _ffi.Thresholds:
        return _ffi.Thresholds(int(self.max_exp_mismatch), 0, float(self.max_mant_mean),
                               float(self.max_mant_median))


@dataclass(frozen=True)
class RecordThresholds:
    """The prefill-sharing record checks' parameters: ``ModelConfig.max_len`` and
    ``CheckContext`` (swarm/validator/checks.py:62-65) with the reference's defaults."""

    max_len: int
    min_sampling_len: int = 16
    eos_prob_floor: float = 0.1
    p_low: float = 0.005
    theta: float = 0.25

    def to_c(self) -> _ffi.RecordThresholds:
        return _ffi.RecordThresholds(int(self.max_len), int(self.min_sampling_len), float(self.eos_prob_floor),
                                     float(self.p_low), float(self.theta))


# verdict codes of record_checks / tl_record_checks (the reference's failed_check names)
RECORD_VERDICTS = ("accept", "termination", "sampling", "commitment")


@dataclass
class VerificationResult:
    """Per-chunk result (field names follow upstream toploc's VerificationResult)."""

    exp_mismatches: int
    n_match: int
    mant_err_sum: int
    mant_err_mean: float
    mant_err_median: float
    accept: bool
    bad_proof: bool = False


def _require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("TOPLOC B200 path needs a CUDA device (no CPU fallback)")


def _stream_handle(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def as_bf16_bits(hidden, device) -> torch.Tensor:
    """Accept a bf16 tensor (any device), a uint16 bit array, or a float array/tensor
    (cast to bf16 RNE) and return a contiguous int16 view on ``device``."""
    if isinstance(hidden, np.ndarray):
        if hidden.dtype == np.uint16:
            t = torch.from_numpy(hidden.view(np.int16))
        else:
            t = torch.from_numpy(np.ascontiguousarray(hidden, dtype=np.float32)).to(torch.bfloat16).view(torch.int16)
    elif isinstance(hidden, torch.Tensor):
        if hidden.dtype == torch.bfloat16:
            t = hidden.view(torch.int16)
        elif hidden.dtype in (torch.int16, torch.uint16):
            t = hidden.view(torch.int16)
        else:
            t = hidden.to(torch.bfloat16).view(torch.int16)
    else:
        raise TypeError(f"unsupported hidden type {type(hidden)}")
    if t.dim() != 2:
        raise ValueError(f"hidden must be 2-D (rows, H), got shape {tuple(t.shape)}")
    return t.to(device, non_blocking=True).contiguous()


def normalize_offsets(row_offsets, n_rows: int) -> np.ndarray:
    if row_offsets is None:
        row_offsets = [0, n_rows]
    offs = np.asarray(row_offsets.cpu() if isinstance(row_offsets, torch.Tensor) else row_offsets,
                      dtype=np.int64).reshape(-1)
    if offs.size < 1 or offs[0] != 0 or offs[-1] != n_rows or np.any(np.diff(offs) < 0):
        raise ValueError("row_offsets must start at 0, be non-decreasing and end at n_rows")
    return offs


def count_chunks(offs: np.ndarray, chunk: int) -> int:
    T = np.diff(offs)
    return int(np.sum((T + chunk - 1) // chunk))


@dataclass
class ProofBatch:
    proofs: torch.Tensor               # uint8 [n_chunks, 2 + 2K] on device
    row_offsets: np.ndarray            # host int64 [R + 1]
    chunk_offsets: np.ndarray          # host int64 [R + 1]: rollout r owns chunks [co[r], co[r+1])
    indices: torch.Tensor | None = None  # int32 [n_chunks, K]
    values: torch.Tensor | None = None   # uint16 bits as int16 [n_chunks, K]

    def to_bytes(self) -> list[list[bytes]]:
        host = self.proofs.cpu().numpy()
        return [[host[j].tobytes() for j in range(self.chunk_offsets[r], self.chunk_offsets[r + 1])]
                for r in range(len(self.chunk_offsets) - 1)]


@dataclass
class VerifyBatch:
    stats: torch.Tensor                # uint8 [n_chunks, 32] (tl_chunk_stats)
    chunk_accept: torch.Tensor         # uint8 [n_chunks]
    rollout_accept: torch.Tensor       # uint8 [R]
    chunk_offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int64))

    def stats_host(self) -> np.ndarray:
        return self.stats.cpu().numpy().view(STATS_DTYPE).reshape(-1)

    def results(self) -> list[list[VerificationResult]]:
        st = self.stats_host()
        out = []
        for r in range(len(self.chunk_offsets) - 1):
            out.append([VerificationResult(int(s["exp_mismatch"]), int(s["n_match"]), int(s["mant_sum"]),
                                           float(s["mant_mean"]), float(s["mant_median"]),
                                           bool(s["flags"] & _ffi.TL_STAT_ACCEPT),
                                           bool(s["flags"] & _ffi.TL_STAT_BADPROOF))
                        for s in st[self.chunk_offsets[r]:self.chunk_offsets[r + 1]]])
        return out


class ToplocEngine:
    """Device-resident prove / verify on one CUDA device (one host thread per engine)."""

    def __init__(self, device=None, chunk: int = CHUNK, topk: int = TOPK):
        _require_cuda()
        dev = torch.device(device) if device is not None else torch.device("cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.chunk, self.topk = int(chunk), int(topk)
        if self.chunk < 1:
            raise ValueError("interval must be >= 1")
        if not 1 <= self.topk <= _ffi.TL_MAX_K:
            raise ValueError(f"topk must be in [1, {_ffi.TL_MAX_K}]")
        self.lib = _ffi.load()
        with torch.cuda.device(self.device):  # the inverse tables, once per device (tl_prepare)
            _ffi.check(self.lib.tl_prepare(), "tl_prepare")
        self._ws = torch.empty(0, dtype=torch.uint8, device=self.device)
        self._ws_done: torch.cuda.Event | None = None  # the last call's use of _ws
        self.proof_bytes = 2 + 2 * self.topk

    # ----------------------------------------------------------------- plumbing
    def _workspace(self, n_roll: int, n_chunks: int) -> torch.Tensor:
        """The engine's scratch.  Calls on different streams are ordered on it: the
        workspace holds the chunk counter and prefix of the running launch, so two calls
        must never share it concurrently (include/toploc_b200.h)."""
        cur = torch.cuda.current_stream(self.device)
        if self._ws_done is not None:
            cur.wait_event(self._ws_done)
        need = int(self.lib.tl_workspace_bytes(n_roll, n_chunks, self.topk))
        if self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def _workspace_used(self) -> None:
        cur = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(cur)
        self._ws_done = ev
        # if a later call grows the workspace, the allocator must not hand this block out
        # again before the work queued here on another stream has finished
        self._ws.record_stream(cur)

    def _offsets(self, offs: np.ndarray):
        co = np.zeros(len(offs), dtype=np.int64)
        T = np.diff(offs)
        co[1:] = np.cumsum((T + self.chunk - 1) // self.chunk)
        dev = torch.from_numpy(offs).to(self.device, non_blocking=True)
        return co, dev

    def plan(self, row_offsets, H: int) -> "Plan":
        return Plan(self, row_offsets, H)

    # ----------------------------------------------------------------- prove
    def prove(self, hidden, row_offsets=None, *, return_indices: bool = False,
              out: torch.Tensor | None = None) -> ProofBatch:
        h = as_bf16_bits(hidden, self.device)
        n_rows, H = h.shape
        offs = normalize_offsets(row_offsets, n_rows)
        co, offs_dev = self._offsets(offs)
        n_chunks = int(co[-1])
        proofs = out if out is not None else torch.empty((n_chunks, self.proof_bytes), dtype=torch.uint8,
                                                         device=self.device)
        if proofs.shape != (n_chunks, self.proof_bytes) or proofs.dtype != torch.uint8:
            raise ValueError("out must be uint8 [n_chunks, 2 + 2K]")
        idx = vals = None
        if return_indices:
            idx = torch.empty((n_chunks, self.topk), dtype=torch.int32, device=self.device)
            vals = torch.empty((n_chunks, self.topk), dtype=torch.int16, device=self.device)
        ws = self._workspace(len(offs) - 1, n_chunks)
        rc = self.lib.tl_prove(h.data_ptr(), offs_dev.data_ptr(), len(offs) - 1, n_rows, H, self.chunk,
                               self.topk, n_chunks, proofs.data_ptr(), _ptr(idx), _ptr(vals),
                               ws.data_ptr(), ws.numel(), _stream_handle(self.device))
        _ffi.check(rc, "tl_prove")
        self._workspace_used()
        return ProofBatch(proofs, offs, co, idx, vals)

    # ----------------------------------------------------------------- verify
    def verify(self, hidden, row_offsets, proofs, thresholds: Thresholds = Thresholds()) -> VerifyBatch:
        h = as_bf16_bits(hidden, self.device)
        n_rows, H = h.shape
        offs = normalize_offsets(row_offsets, n_rows)
        co, offs_dev = self._offsets(offs)
        n_chunks = int(co[-1])
        pr = self._proof_tensor(proofs, n_chunks)
        stats = torch.empty((n_chunks, 32), dtype=torch.uint8, device=self.device)
        cacc = torch.empty(n_chunks, dtype=torch.uint8, device=self.device)
        racc = torch.empty(len(offs) - 1, dtype=torch.uint8, device=self.device)
        ws = self._workspace(len(offs) - 1, n_chunks)
        th = thresholds.to_c()
        rc = self.lib.tl_verify(h.data_ptr(), offs_dev.data_ptr(), len(offs) - 1, n_rows, H, self.chunk,
                                self.topk, n_chunks, pr.data_ptr(), ctypes.byref(th), stats.data_ptr(),
                                cacc.data_ptr(), racc.data_ptr(), ws.data_ptr(), ws.numel(),
                                _stream_handle(self.device))
        _ffi.check(rc, "tl_verify")
        self._workspace_used()
        return VerifyBatch(stats, cacc, racc, co)

    def _proof_tensor(self, proofs, n_chunks: int) -> torch.Tensor:
        if isinstance(proofs, ProofBatch):
            proofs = proofs.proofs
        if isinstance(proofs, np.ndarray):  # (n_chunks, 2 + 2K) uint8, e.g. codec.decode's output
            proofs = torch.from_numpy(np.ascontiguousarray(proofs, dtype=np.uint8))
        if isinstance(proofs, torch.Tensor):
            t = proofs.to(self.device).contiguous()
        else:  # list (per rollout) of list of bytes / hex str, or flat list
            flat = []
            for item in proofs:
                if isinstance(item, (bytes, bytearray, str)):
                    flat.append(item)
                else:
                    flat.extend(item)
            blobs = [bytes.fromhex(p) if isinstance(p, str) else bytes(p) for p in flat]
            if any(len(b) != self.proof_bytes for b in blobs):
                raise ValueError(f"every proof must be {self.proof_bytes} bytes")
            arr = np.frombuffer(b"".join(blobs), dtype=np.uint8).reshape(-1, self.proof_bytes) \
                if blobs else np.zeros((0, self.proof_bytes), np.uint8)
            t = torch.from_numpy(arr.copy()).to(self.device)
        if t.dtype != torch.uint8 or t.shape != (n_chunks, self.proof_bytes):
            raise ValueError(f"expected {n_chunks} proofs of {self.proof_bytes} bytes, got {tuple(t.shape)}")
        return t


class Plan:
    """Pre-allocated device buffers for a fixed batch shape (rollout lengths, H).

    Reusing a plan keeps the hot loop free of allocation and host->device offset
    copies: ``select`` / ``commit`` / ``prove`` / ``verify`` are one C-ABI call each
    (the benchmark and the scheduler use this form)."""

    def __init__(self, eng: ToplocEngine, row_offsets, H: int):
        self.eng = eng
        self.offs = normalize_offsets(row_offsets, int(np.asarray(row_offsets)[-1]))
        self.co, self.offs_dev = eng._offsets(self.offs)
        self.H = int(H)
        self.n_roll = len(self.offs) - 1
        self.n_rows = int(self.offs[-1])
        self.n_chunks = int(self.co[-1])
        dev, K = eng.device, eng.topk
        need = int(eng.lib.tl_workspace_bytes(self.n_roll, self.n_chunks, K))
        self.ws = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
        self.idx = torch.empty((self.n_chunks, K), dtype=torch.int32, device=dev)
        self.bits = torch.empty((self.n_chunks, K), dtype=torch.int16, device=dev)
        self.proofs = torch.empty((self.n_chunks, eng.proof_bytes), dtype=torch.uint8, device=dev)
        self.stats = torch.empty((self.n_chunks, 32), dtype=torch.uint8, device=dev)
        self.chunk_accept = torch.empty(self.n_chunks, dtype=torch.uint8, device=dev)
        self.rollout_accept = torch.empty(self.n_roll, dtype=torch.uint8, device=dev)

    def _check_hidden(self, h: torch.Tensor) -> torch.Tensor:
        if h.device != self.eng.device or h.shape != (self.n_rows, self.H) or not h.is_contiguous():
            raise ValueError(f"hidden must be a contiguous ({self.n_rows}, {self.H}) tensor on {self.eng.device}")
        return h

    def _stream(self, stream) -> int:
        return (stream if stream is not None else torch.cuda.current_stream(self.eng.device)).cuda_stream

    def select(self, h: torch.Tensor, stream=None, ctas_per_sm: int = 0) -> None:
        h = self._check_hidden(h)
        e = self.eng
        _ffi.check(e.lib.tl_select_ex(h.data_ptr(), self.offs_dev.data_ptr(), self.n_roll, self.n_rows, self.H,
                                      e.chunk, e.topk, self.n_chunks, self.idx.data_ptr(), self.bits.data_ptr(),
                                      self.ws.data_ptr(), self.ws.numel(), ctas_per_sm, self._stream(stream)),
                   "tl_select")

    def commit(self, stream=None, co_resident: bool = False) -> None:
        e = self.eng
        _ffi.check(e.lib.tl_commit_ex(self.idx.data_ptr(), self.bits.data_ptr(), self.n_chunks, e.topk,
                                      self.proofs.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                                      1 if co_resident else 0, self._stream(stream)), "tl_commit")

    def prove(self, h: torch.Tensor) -> torch.Tensor:
        self.select(h)
        self.commit()
        return self.proofs

    def verify(self, h: torch.Tensor, proofs: torch.Tensor | None = None,
               thresholds: Thresholds = Thresholds(), stream=None, ctas_per_sm: int = 0,
               workspace: torch.Tensor | None = None, rollout_out: torch.Tensor | None = None) -> torch.Tensor:
        """tl_verify; ``workspace`` (same size as ``ws``) lets a verify run concurrently
        with this plan's select on another stream; ``rollout_out`` (uint8, one per rollout)
        receives the rollout verdicts instead of ``rollout_accept`` (the pipelines give every
        batch its own, so no copy is needed to keep them)."""
        h = self._check_hidden(h)
        e = self.eng
        pr = self.proofs if proofs is None else proofs
        ws = self.ws if workspace is None else workspace
        ra = self.rollout_accept
        if rollout_out is not None:
            if rollout_out.dtype != torch.uint8 or rollout_out.numel() != self.n_roll or \
                    rollout_out.device != self.eng.device or not rollout_out.is_contiguous():
                raise ValueError(f"rollout_out must be a contiguous uint8 tensor of {self.n_roll} on {self.eng.device}")
            ra = rollout_out
        th = thresholds.to_c()
        _ffi.check(e.lib.tl_verify_ex(h.data_ptr(), self.offs_dev.data_ptr(), self.n_roll, self.n_rows, self.H,
                                      e.chunk, e.topk, self.n_chunks, pr.data_ptr(), ctypes.byref(th),
                                      self.stats.data_ptr(), self.chunk_accept.data_ptr(),
                                      ra.data_ptr(), ws.data_ptr(), ws.numel(),
                                      ctas_per_sm, self._stream(stream)), "tl_verify")
        return ra


def _upload_graph(graph: "torch.cuda.CUDAGraph", device) -> bool:
    """Upload an instantiated graph to the device without running it (cuGraphUpload), so its
    first replay does not pay the upload (~1 ms for a graph of 200 pipelined batches).
    Returns False when the driver bindings are unavailable (the first replay uploads it)."""
    try:
        from cuda.bindings import driver
        ex = graph.raw_cuda_graph_exec()
        st = torch.cuda.current_stream(device).cuda_stream
        err, = driver.cuGraphUpload(driver.CUgraphExec(ex), driver.CUstream(st))
        torch.cuda.synchronize(device)
        return err == driver.CUresult.CUDA_SUCCESS
    except Exception:
        return False


class StepGraph:
    """One prove + verify step of a ``Plan`` captured as a CUDA graph (select, commit,
    verify and their small kernels: 7 launches replayed as one).  The captured tensors
    are the ones given at capture time; refill them in place between replays.  Launch
    overhead matters for small batches (configuration 1 is launch-bound); results are
    identical to the eager calls."""

    def __init__(self, plan: "Plan", prover: torch.Tensor, validator: torch.Tensor,
                 thresholds: Thresholds = Thresholds()):
        self.plan = plan
        dev = plan.eng.device
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # warm the kernels' attributes outside the capture
            plan.select(prover)
            plan.commit()
            plan.verify(validator, None, thresholds)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            plan.select(prover)
            plan.commit()
            plan.verify(validator, None, thresholds)
        self.uploaded = _upload_graph(self.graph, dev)

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        return self.plan.rollout_accept


class PipelineGraph:
    """``len(provers)`` batches of a ``Pipeline`` captured as one CUDA graph.

    For small batches every kernel is latency-bound and uses a fraction of the GPU, so
    the pipeline's overlap (select(k+1) beside verify(k-1), commit(k) on the side stream)
    runs the three stages of different batches concurrently, and the graph removes the
    per-launch host cost.  ``replay()`` proves and verifies every captured batch and
    returns their rollout-accept vectors; results are identical to the serial calls."""

    def __init__(self, pipe: "Pipeline", provers, validators, thresholds: Thresholds = Thresholds()):
        self.pipe = pipe
        dev = pipe.eng.device
        cur = torch.cuda.current_stream(dev)
        warm = torch.cuda.Stream(dev)
        warm.wait_stream(cur)
        with torch.cuda.stream(warm):  # kernel attributes and allocations outside the capture
            pipe.run(provers[:2], validators[:2], thresholds)
        cur.wait_stream(warm)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.out = pipe.run(provers, validators, thresholds)
        self.uploaded = _upload_graph(self.graph, dev)

    def replay(self) -> list[torch.Tensor]:
        self.graph.replay()
        return self.out


class Pipeline:
    """Prove + verify a stream of equally-shaped batches with the commitment of batch
    k overlapping the verification of batch k-1.

    Main stream: select(k), verify(k-1), select(k+1), verify(k), ...  Side stream:
    commit(k) after select(k).  Two buffer sets alternate.  select/verify run 16
    one-warp CTAs per SM (16 x 32 x 96 registers) and the commitment its co-resident
    form (8 warps, <= 64 registers, 64 KiB half inverse table), which together fill
    the SM's 64 Ki registers exactly: the issue-bound commitment runs in the slots the
    HBM-bound streaming kernels leave idle.  Results are identical to the serial
    ``Plan`` calls."""

    def __init__(self, eng: "ToplocEngine", row_offsets, H: int, ctas_per_sm: int = 16):
        self.plans = [Plan(eng, row_offsets, H), Plan(eng, row_offsets, H)]
        self.eng = eng
        self.ctas = ctas_per_sm
        self.co_resident = True
        self.edge_on_main = False  # commit the first and last batch on the main stream
        self.main = None  # None: the caller's current stream
        self.side = torch.cuda.Stream(eng.device)

    def run(self, provers, validators, thresholds: Thresholds = Thresholds(), on_verify=None,
            on_select=None, on_commit=None) -> list[torch.Tensor]:
        """provers / validators: sequences of (rows, H) device tensors.  Returns the
        rollout-accept vectors (device uint8) per batch.  ``on_select(k, what, stream)`` /
        ``on_commit`` / ``on_verify`` are called around the launches (for event timing)."""
        caller = torch.cuda.current_stream(self.eng.device)
        main = self.main if self.main is not None else caller
        if main is not caller:
            main.wait_stream(caller)
        self.side.wait_stream(caller)
        n = len(provers)
        out = []
        outs = [torch.empty(self.plans[0].n_roll, dtype=torch.uint8, device=self.eng.device) for _ in range(n)]
        sel_done = [None] * n
        com_done = [None] * n
        for k in range(n + 1):
            if k < n:
                pl = self.plans[k % 2]
                if on_select:
                    on_select(k, "start", main)
                pl.select(provers[k], main, self.ctas)
                if on_select:
                    on_select(k, "end", main)
                sel_done[k] = torch.cuda.Event()
                sel_done[k].record(main)
                edge = self.edge_on_main and (k == 0 or k == n - 1)
                if not edge:
                    self.side.wait_event(sel_done[k])
                    self._commit(pl, k, self.side, self.co_resident, on_commit, com_done)
                elif k == 0:  # pipeline fill: nothing to overlap yet, commit on the main SMs
                    self._commit(pl, k, main, False, on_commit, com_done)
            if k >= 1:
                pl = self.plans[(k - 1) % 2]
                main.wait_event(com_done[k - 1])
                if on_verify:
                    on_verify(k - 1, "start", main)
                out.append(pl.verify(validators[k - 1], None, thresholds, main, self.ctas, rollout_out=outs[k - 1]))
                if on_verify:
                    on_verify(k - 1, "end", main)
                if self.edge_on_main and k == n - 1:  # pipeline drain: the last commit on the main SMs
                    self._commit(self.plans[k % 2], k, main, False, on_commit, com_done)
        if main is not caller:
            caller.wait_stream(main)
        caller.wait_stream(self.side)
        return out

    @staticmethod
    def _commit(pl: "Plan", k: int, stream, co_resident: bool, on_commit, com_done) -> None:
        if on_commit:
            on_commit(k, "start", stream)
        pl.commit(stream, co_resident=co_resident)
        if on_commit:
            on_commit(k, "end", stream)
        com_done[k] = torch.cuda.Event()
        com_done[k].record(stream)


class PartitionedPipeline(Pipeline):
    """Prove + verify a stream of batches on two disjoint SM partitions of the GPU (driver
    green contexts, ``tl_partition_create``).

    - The 32-warp commitment (128 KiB shared-memory inverse table) runs on
      ``commit_sms`` SMs; it never competes with the streams for an SM.
    - select and verify run at full occupancy on the other SMs, on two streams:
      select(k) on one, verify(k-2) on the other, with commit(k-1) on the partition.
      Persistent kernels on one stream leave their tail idle; the other stream's next
      kernel fills it.  HBM reads saturate on ~124 of the 148 SMs (tools/lab/greenctx.cu).
    - Three buffer sets rotate; each verify has its own workspace.
    Results are identical to the serial calls."""

    def __init__(self, eng: "ToplocEngine", row_offsets, H: int, commit_sms: int = 24):
        super().__init__(eng, row_offsets, H, ctas_per_sm=0)
        self.plans.append(Plan(eng, row_offsets, H))
        self.ws_verify = [torch.empty_like(p.ws) for p in self.plans]
        streams = (ctypes.c_void_p * 3)()
        sms = (ctypes.c_int32 * 2)()
        with torch.cuda.device(eng.device):
            _ffi.check(eng.lib.tl_partition_create(int(commit_sms), streams, sms), "tl_partition_create")
        self._handles = streams
        self.main = torch.cuda.ExternalStream(streams[0], device=eng.device)   # select
        self.vstream = torch.cuda.ExternalStream(streams[1], device=eng.device)  # verify
        self.side = torch.cuda.ExternalStream(streams[2], device=eng.device)   # commit
        self.co_resident = False
        self.sms = (sms[0], sms[1])  # (streaming, commitment)

    def run(self, provers, validators, thresholds: Thresholds = Thresholds(), on_verify=None,
            on_select=None, on_commit=None) -> list[torch.Tensor]:
        caller = torch.cuda.current_stream(self.eng.device)
        sels = getattr(self, "sstreams", None) or [self.main]
        sides = getattr(self, "cstreams", None) or [self.side]
        vers = getattr(self, "vstreams", None) or [self.vstream]
        for st in (*sels, *sides, *vers):
            st.wait_stream(caller)
        n = len(provers)
        nb = len(self.plans)  # rotating buffer sets
        out = []
        outs = [torch.empty(self.plans[0].n_roll, dtype=torch.uint8, device=self.eng.device) for _ in range(n)]
        com_done = [None] * n
        ver_done = [None] * n
        for k in range(n + 2):
            if k < n:
                pl = self.plans[k % nb]
                sel, side = sels[k % len(sels)], sides[k % len(sides)]
                if k >= nb:
                    sel.wait_event(com_done[k - nb])  # this plan's idx / bits consumed
                if on_select:
                    on_select(k, "start", sel)
                pl.select(provers[k], sel, self.ctas)
                if on_select:
                    on_select(k, "end", sel)
                done = torch.cuda.Event()
                done.record(sel)
                side.wait_event(done)
                if k >= nb:
                    side.wait_event(ver_done[k - nb])  # this plan's proofs read
                self._commit(pl, k, side, self.co_resident, on_commit, com_done)
            if k >= 2:
                j = k - 2
                pl = self.plans[j % nb]
                ver = vers[j % len(vers)]
                ver.wait_event(com_done[j])
                if on_verify:
                    on_verify(j, "start", ver)
                out.append(pl.verify(validators[j], None, thresholds, ver, self.ctas, workspace=self.ws_verify[j % nb],
                                     rollout_out=outs[j]))
                if on_verify:
                    on_verify(j, "end", ver)
                ver_done[j] = torch.cuda.Event()
                ver_done[j].record(ver)
        for st in (*sels, *sides, *vers):
            caller.wait_stream(st)
        return out

    def close(self) -> None:
        if getattr(self, "_handles", None) is not None:
            _ffi.check(self.eng.lib.tl_partition_destroy(self._handles), "tl_partition_destroy")
            self._handles = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DualStreamPipeline(PartitionedPipeline):
    """The partitioned pipeline's schedule (select(k) and verify(k-2) on two streams,
    commit(k-1) on a third, rotating buffer sets) on ordinary streams of the whole
    GPU, with the co-resident commitment.  For small batches, whose kernels each use a
    fraction of the GPU, the three stages of different batches run concurrently; unlike
    green-context streams these can be captured in one CUDA graph (``PipelineGraph``)."""

    def __init__(self, eng: "ToplocEngine", row_offsets, H: int, ctas_per_sm: int = 0,
                 buffer_sets: int | None = None, streams_per_stage: int | None = None):
        Pipeline.__init__(self, eng, row_offsets, H, ctas_per_sm=ctas_per_sm)
        # more buffer sets and streams put more batches in flight: worth it while a batch's
        # kernels leave most SMs idle (configuration 1, 64 chunks, per step: 3 sets x 1 stream
        # 14.3 us, 6 x 2 8.3 us, 12 x 4 6.5 us; tools/lab/pipegraph_sweep.py), not once they
        # fill the GPU (256 chunks at H 5120: 3 x 2 41.9 us, 6 x 2 42.6, 3 x 3 46.4)
        small = self.plans[0].n_chunks <= int(eng.lib.tl_stream_sms(None))
        if buffer_sets is None:
            buffer_sets = 12 if small else 3
        if streams_per_stage is None:
            streams_per_stage = 4 if small else 2
        while len(self.plans) < max(3, buffer_sets):
            self.plans.append(Plan(eng, row_offsets, H))
        self.ws_verify = [torch.empty_like(p.ws) for p in self.plans]
        self._handles = None
        self.main = torch.cuda.Stream(eng.device)     # select
        self.vstream = torch.cuda.Stream(eng.device)  # verify
        self.side = torch.cuda.Stream(eng.device)     # commit
        # a small batch's kernels each use a fraction of the SMs: every stage alternates
        # between two streams, so the same stage of consecutive batches can run at once
        # (their plans, workspaces and verdict buffers are distinct: ``buffer_sets`` sets
        # rotate, and the waits in run() order every reuse)
        more = max(0, streams_per_stage - 1)
        self.sstreams = [self.main] + [torch.cuda.Stream(eng.device) for _ in range(more)]
        self.cstreams = [self.side] + [torch.cuda.Stream(eng.device) for _ in range(more)]
        self.vstreams = [self.vstream] + [torch.cuda.Stream(eng.device) for _ in range(more)]
        # a batch of at most one chunk per SM sub-partition leaves most SMs free: its
        # commitment runs the small-batch kernel (commit_coop_kernel, one launch, one CTA
        # per chunk) instead of the co-resident form
        n_chunks = self.plans[0].n_chunks
        self.co_resident = n_chunks > 4 * int(eng.lib.tl_stream_sms(None))
        self.sms = None


_ENGINES: dict[tuple, ToplocEngine] = {}


def engine(device=None, chunk: int = CHUNK, topk: int = TOPK) -> ToplocEngine:
    _require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (dev.index, chunk, topk)
    if key not in _ENGINES:
        _ENGINES[key] = ToplocEngine(dev, chunk, topk)
    return _ENGINES[key]


def build_proofs(hidden, row_offsets=None, chunk: int = CHUNK, topk: int = TOPK, device=None) -> list[list[bytes]]:
    """TOPLOC prove -> per rollout, ``ceil(T/chunk)`` proofs of ``2 + 2*topk`` bytes."""
    eng = engine(device, chunk, topk)
    return eng.prove(hidden, row_offsets).to_bytes()


def verify_proofs(hidden, row_offsets, proofs, chunk: int = CHUNK, topk: int = TOPK,
                  thresholds: Thresholds = Thresholds(), device=None):
    """TOPLOC verify -> (per-rollout lists of VerificationResult, per-rollout accept)."""
    eng = engine(device, chunk, topk)
    vb = eng.verify(hidden, row_offsets, proofs, thresholds)
    return vb.results(), [bool(v) for v in vb.rollout_accept.cpu().tolist()]


def record_checks(probs, row_offsets, prompt_len, ends_with_eos, thresholds: RecordThresholds,
                  commit_accept=None, commit_checked=None, device=None):
    """tl_record_checks: the validator's per-record termination and sampling checks on
    the prefill's chosen-token probabilities, then the commitment verdict, in the
    reference's order (checks.py:204-213).  ``probs``: float64 per output token,
    rollouts concatenated by ``row_offsets``; ``commit_accept`` e.g. a VerifyBatch's
    ``rollout_accept``.  Returns device tensors (verdict int32 codes indexing
    RECORD_VERDICTS, fraction of probs below p_low, last-token prob)."""
    _require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    p = torch.as_tensor(probs, dtype=torch.float64).reshape(-1).to(dev).contiguous()
    offs = normalize_offsets(row_offsets, p.numel())
    R = len(offs) - 1
    offs_dev = torch.from_numpy(offs).to(dev)

    def vec(x, dtype):
        t = None if x is None else torch.as_tensor(x).reshape(-1).to(dev, dtype).contiguous()
        if t is not None and t.numel() != R:
            raise ValueError(f"per-record arrays need {R} entries, got {t.numel()}")
        return t

    pl, eos = vec(prompt_len, torch.int32), vec(ends_with_eos, torch.uint8)
    ca, cc = vec(commit_accept, torch.uint8), vec(commit_checked, torch.uint8)
    verdict = torch.empty(R, dtype=torch.int32, device=dev)
    frac = torch.empty(R, dtype=torch.float64, device=dev)
    p_last = torch.empty(R, dtype=torch.float64, device=dev)
    th = thresholds.to_c()
    rc = _ffi.load().tl_record_checks(p.data_ptr(), offs_dev.data_ptr(), R, _ptr(pl), _ptr(eos), ctypes.byref(th),
                                      _ptr(ca), _ptr(cc), verdict.data_ptr(), frac.data_ptr(), p_last.data_ptr(),
                                      _stream_handle(dev))
    _ffi.check(rc, "tl_record_checks")
    return verdict, frac, p_last


def build_commitments(hidden, k: int = CHUNK) -> list[bytes]:
    """Exact-mode drop-in for ``swarm.worker.rollout.build_commitments`` (rollout.py:51-68)."""
    from .exact import build_commitments as _bc
    return _bc(hidden, k)
