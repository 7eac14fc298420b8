"""Host-side scheduler logic: token-balanced rollout sharding and the verdict
gather, including a world_size-2 gloo run (the N>1 path without GPUs)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_07291_b200.scheduler import gather_verdicts, gather_verdicts_lpt, plan, shard_by_tokens, shard_lpt


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_shards_tile_and_balance(world, seed):
    rng = np.random.default_rng(seed)
    lengths = rng.integers(0, 40000, size=int(rng.integers(1, 300)))
    ranges = shard_by_tokens(lengths, world)
    assert len(ranges) == world
    assert ranges[0][0] == 0 and ranges[-1][1] == len(lengths)
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    loads = [int(lengths[lo:hi].sum()) for lo, hi in ranges]
    assert sum(loads) == int(lengths.sum())
    assert max(loads) <= lengths.sum() / world + lengths.max() + 1


def test_shards_degenerate():
    assert shard_by_tokens([], 3) == [(0, 0)] * 3
    assert shard_by_tokens([5], 4)[-1][1] == 1
    assert shard_by_tokens([0, 0, 0, 0], 2)[-1][1] == 4
    eq = shard_by_tokens([8192] * 256, 4)
    assert [hi - lo for lo, hi in eq] == [64] * 4          # equal rollouts: equal shards
    with pytest.raises(ValueError):
        shard_by_tokens([1, 2], 0)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_lpt_partitions_and_balances_ragged_batches(world):
    rng = np.random.default_rng(world)
    lengths = np.concatenate([rng.integers(1, 500, size=60), [40000, 39000, 20000]])  # a few very long
    shards = shard_lpt(lengths, world)
    allidx = np.sort(np.concatenate(shards))
    assert np.array_equal(allidx, np.arange(lengths.size))           # a partition
    loads = [int(lengths[s].sum()) for s in shards]
    # LPT bound: makespan <= 4/3 OPT, OPT >= max(mean load, longest job)
    opt_lb = max(lengths.sum() / world, lengths.max())
    assert max(loads) <= 4 / 3 * opt_lb + 1
    contiguous = [int(lengths[lo:hi].sum()) for lo, hi in shard_by_tokens(lengths, world)]
    assert max(loads) <= max(contiguous)


def test_plan_local_offsets():
    offs = np.array([0, 10, 30, 30, 60, 100])
    sp = plan(np.diff(offs), rank=1, world=2)
    lo, hi = sp.ranges[1]
    assert list(sp.local_offsets(offs)) == list(offs[lo:hi + 1] - offs[lo])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker_lpt(rank, world, port, lengths, truth, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shards = shard_lpt(lengths, world)
        local = torch.tensor([truth[i] for i in shards[rank]], dtype=torch.uint8)
        q.put((rank, gather_verdicts_lpt(local, shards).tolist()))
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, lengths, truth, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sp = plan(lengths)
        local = torch.tensor(truth[sp.lo:sp.hi], dtype=torch.uint8)
        full = gather_verdicts(local, sp.counts())
        q.put((rank, full.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_gather_matches_single_process(world):
    rng = np.random.default_rng(5)
    lengths = rng.integers(1, 9000, size=37)
    truth = (rng.random(37) < 0.7).astype(np.uint8).tolist()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lengths, truth, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, full in out:
        assert full == truth


def test_gloo_lpt_gather_restores_rollout_order():
    rng = np.random.default_rng(9)
    lengths = rng.integers(1, 9000, size=29)
    truth = (rng.random(29) < 0.6).astype(np.uint8).tolist()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_lpt, args=(r, 2, port, lengths, truth, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for _, full in out:
        assert full == truth
