"""On-GPU capture of last-layer hidden states during generation, proven on the device.

SURVEY.md §8(f)-4: the step before the path.  The paper's workers prove
asynchronously on the CPU after generation; the reference commits
``hidden`` from a separate teacher-forced pass (``rollout.py:105-112``,
``policy/model.py:160-173``).  Here a forward hook on the model's final norm copies
each step's committed rows into a preallocated bf16 device buffer -- no host round
trip, no synchronisation inside the hook -- and ``prove()`` runs ``tl_prove`` on the
buffer directly.

Row t of a sequence is the activation whose context is ``prompt + output[:t]`` (the
state that predicts output token t), as in ``policy/model.py:143-150``: the last
prompt position of the prefill, then one row per decode step.  With
``generate(max_new_tokens=T)`` that is exactly T rows (prefill + T-1 decode steps).

The validator side is ``prefill_rows``: one teacher-forced forward over
``prompt + output[:-1]`` through the same hook point, returning the same T rows, which
``ToplocEngine.verify`` checks against the proofs.
"""

from __future__ import annotations

import numpy as np
import torch

from .api import CHUNK, ProofBatch, Thresholds, ToplocEngine, VerifyBatch, engine as get_engine


class ProofCapture:
    """Collects the committed hidden rows of ``batch`` sequences (up to ``max_tokens``
    generated tokens each) from a forward hook and proves them on the GPU.

    ``attach(module)`` registers the hook (for Hugging Face causal LMs, the final norm:
    ``model.model.norm``); a forward with sequence length S > 1 is a prefill and
    contributes its last position, S == 1 is a decode step.  ``reset()`` starts a new
    batch; ``lengths`` can be lowered per sequence when a sequence stops early."""

    def __init__(self, hidden_size: int, max_tokens: int, batch: int, device="cuda",
                 eng: ToplocEngine | None = None):
        self.eng = eng  # resolved on first prove(); the capture itself is plain tensor code
        self.device = torch.device(device) if eng is None else eng.device
        self.H = int(hidden_size)
        self.max_tokens = int(max_tokens)
        self.batch = int(batch)
        self.buf = torch.empty((self.batch, self.max_tokens, self.H), dtype=torch.bfloat16, device=self.device)
        self.pos = 0
        self.lengths = None
        self._handle = None

    # ------------------------------------------------------------------ capture
    def reset(self) -> None:
        self.pos = 0
        self.lengths = None

    def hook(self, module, args, output) -> None:
        h = output[0] if isinstance(output, tuple) else output
        if h.dim() != 3 or h.shape[0] != self.batch or h.shape[-1] != self.H:
            raise ValueError(f"expected hidden states (batch={self.batch}, S, H={self.H}), got {tuple(h.shape)}")
        if self.pos >= self.max_tokens:
            raise ValueError(f"more than max_tokens={self.max_tokens} committed rows")
        # prefill: the last prompt position predicts output token 0; decode: the new position
        self.buf[:, self.pos].copy_(h[:, -1], non_blocking=True)
        self.pos += 1

    def attach(self, module: torch.nn.Module):
        self.detach()
        self._handle = module.register_forward_hook(self.hook)
        return self._handle

    def detach(self) -> None:
        if self._handle is not None:
            self._handle.remove()
            self._handle = None

    # ------------------------------------------------------------------ prove
    def rows(self) -> tuple[torch.Tensor, np.ndarray]:
        """Packed (sum T_b, H) bf16 rows of the batch and their row offsets."""
        lens = np.full(self.batch, self.pos, dtype=np.int64) if self.lengths is None else \
            np.minimum(np.asarray(self.lengths, dtype=np.int64), self.pos)
        offs = np.concatenate([[0], np.cumsum(lens)])
        if np.all(lens == self.pos):
            packed = self.buf[:, :self.pos].reshape(self.batch * self.pos, self.H)
        else:
            packed = torch.cat([self.buf[b, :int(lens[b])] for b in range(self.batch)])
        return packed.contiguous(), offs

    def prove(self) -> ProofBatch:
        """tl_prove over every captured sequence: ceil(T_b / 32) 258-byte proofs each."""
        packed, offs = self.rows()
        if self.eng is None:
            self.eng = get_engine(self.device)
        return self.eng.prove(packed, offs)


@torch.no_grad()
def prefill_rows(model, norm: torch.nn.Module, prompt_ids: torch.Tensor, output_ids: torch.Tensor) -> torch.Tensor:
    """Validator side: the T committed rows of each sequence from one teacher-forced
    forward over ``prompt + output[:-1]`` (B, P) + (B, T) -> (B*T, H) bf16, captured at
    the same hook point as ``ProofCapture``."""
    P, T = prompt_ids.shape[1], output_ids.shape[1]
    seq = torch.cat([prompt_ids, output_ids[:, :-1]], dim=1)
    got = []
    handle = norm.register_forward_hook(lambda m, a, o: got.append(o[0] if isinstance(o, tuple) else o))
    try:
        model(input_ids=seq, use_cache=False)
    finally:
        handle.remove()
    h = got[-1]
    return h[:, P - 1:P - 1 + T].reshape(-1, h.shape[-1]).to(torch.bfloat16).contiguous()


def verify_rows(rows: torch.Tensor, batch: int, proofs, thresholds: Thresholds = Thresholds(),
                eng: ToplocEngine | None = None) -> VerifyBatch:
    """``ToplocEngine.verify`` over ``batch`` equal-length sequences packed in ``rows``."""
    eng = eng if eng is not None else get_engine(rows.device)
    T = rows.shape[0] // batch
    offs = np.arange(batch + 1, dtype=np.int64) * T
    return eng.verify(rows, offs, proofs, thresholds)


__all__ = ["ProofCapture", "prefill_rows", "verify_rows", "CHUNK"]
