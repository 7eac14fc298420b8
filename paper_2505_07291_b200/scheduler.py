"""Batch scheduler: shard rollouts over the GPUs of one box, gather verdicts.

North-star subsystem (d).  The reference leases one rollout file to one validator
process at a time (``swarm/orchestrator/storage.py:67-83``, consumed by
``swarm/node.py:304-339``); verification itself is embarrassingly parallel per
rollout, and within a rollout per 32-token chunk.  Here each rank (one process per
GPU, ``torchrun``) owns a contiguous range of rollouts balanced by token count,
proves / verifies its range from its own HBM with no data-path collective, and the
only communication is one gather of the per-rollout accept bytes (NCCL over
NVLink on GPUs; gloo in the CPU tests).  Chunks never span ranks, so results do
not depend on the GPU count.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


def shard_by_tokens(lengths, world: int) -> list[tuple[int, int]]:
    """Contiguous rollout ranges [(lo, hi)] per rank with near-equal token counts.

    Rank r takes the rollouts whose token prefix midpoint falls in the r-th
    1/world of the total (deterministic; every rollout assigned exactly once)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    lengths = np.asarray(lengths, dtype=np.int64)
    if np.any(lengths < 0):
        raise ValueError("lengths must be non-negative")
    n = lengths.size
    total = int(lengths.sum())
    if n == 0:
        return [(0, 0)] * world
    mid = np.cumsum(lengths) - lengths / 2.0
    owner = np.minimum((mid * world / max(total, 1)).astype(np.int64), world - 1) if total else \
        np.minimum(np.arange(n) * world // n, world - 1)
    owner = np.maximum.accumulate(owner)      # keep ranges contiguous and ordered
    bounds = []
    for r in range(world):
        idx = np.nonzero(owner == r)[0]
        if idx.size:
            bounds.append((int(idx[0]), int(idx[-1]) + 1))
        else:
            prev = bounds[-1][1] if bounds else 0
            bounds.append((prev, prev))
    # close gaps so that ranges tile [0, n)
    fixed, start = [], 0
    for lo, hi in bounds:
        hi = max(hi, start)
        fixed.append((start, hi))
        start = hi
    fixed[-1] = (fixed[-1][0], n)
    return fixed


def shard_lpt(lengths, world: int) -> list[np.ndarray]:
    """Longest-processing-time assignment for ragged batches: rollouts in decreasing token
    count, each to the currently least-loaded rank (ties to the lower rank).  Returns each
    rank's rollout indices in increasing order.  Not contiguous, but within 4/3 of the
    optimal makespan, against one whole rollout of slack for ``shard_by_tokens``."""
    if world < 1:
        raise ValueError("world must be >= 1")
    lengths = np.asarray(lengths, dtype=np.int64)
    if np.any(lengths < 0):
        raise ValueError("lengths must be non-negative")
    load = np.zeros(world, dtype=np.int64)
    owner = np.empty(lengths.size, dtype=np.int64)
    for i in np.argsort(-lengths, kind="stable"):
        r = int(np.argmin(load))
        owner[i] = r
        load[r] += lengths[i]
    return [np.nonzero(owner == r)[0] for r in range(world)]


def gather_verdicts_lpt(local: torch.Tensor, shards: list[np.ndarray], group=None) -> torch.Tensor:
    """``gather_verdicts`` for an LPT sharding: scatter every rank's verdicts back to the
    global rollout order."""
    counts = [len(s) for s in shards]
    flat = gather_verdicts(local, counts, group)
    order = torch.from_numpy(np.concatenate(shards) if shards else np.zeros(0, np.int64)).to(flat.device)
    out = torch.empty_like(flat)
    out[order] = flat
    return out


def gather_verdicts(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """All-gather per-rank uint8 verdict vectors (lengths `counts`) into rollout order.

    Works on NCCL (device tensors, one ``all_gather_into_tensor``) and gloo (CPU)."""
    world = dist.get_world_size(group)
    if len(counts) != world:
        raise ValueError("counts must have one entry per rank")
    m = max(max(counts), 1)
    pad = torch.zeros(m, dtype=torch.uint8, device=local.device)
    pad[:local.numel()] = local.reshape(-1).to(torch.uint8)
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * m, dtype=torch.uint8, device=local.device)
        dist.all_gather_into_tensor(out, pad, group=group)
        parts = list(out.view(world, m))
    else:
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)])


@dataclass
class ShardPlan:
    rank: int
    world: int
    ranges: list[tuple[int, int]]

    @property
    def lo(self) -> int:
        return self.ranges[self.rank][0]

    @property
    def hi(self) -> int:
        return self.ranges[self.rank][1]

    def counts(self) -> list[int]:
        return [hi - lo for lo, hi in self.ranges]

    def local_offsets(self, row_offsets) -> np.ndarray:
        """Row offsets of this rank's rollouts, rebased to start at 0."""
        offs = np.asarray(row_offsets, dtype=np.int64)
        return offs[self.lo:self.hi + 1] - offs[self.lo]


def plan(lengths, rank: int | None = None, world: int | None = None) -> ShardPlan:
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    return ShardPlan(rank, world, shard_by_tokens(lengths, world))


def verify_sharded(engine, prover_hidden_local, validator_hidden_local, row_offsets, thresholds=None,
                   group=None):
    """Prove and verify this rank's shard, then gather every rank's verdicts.

    ``*_hidden_local`` hold only this rank's rollouts (rows of
    ``plan(...).local_offsets(row_offsets)``); returns the full uint8 verdict
    vector in global rollout order on every rank."""
    from .api import Thresholds
    lengths = np.diff(np.asarray(row_offsets, dtype=np.int64))
    sp = plan(lengths)
    offs = sp.local_offsets(row_offsets)
    pb = engine.prove(prover_hidden_local, offs)
    vb = engine.verify(validator_hidden_local, offs, pb, thresholds or Thresholds())
    if sp.world == 1:
        return vb.rollout_accept
    return gather_verdicts(vb.rollout_accept, sp.counts(), group)
