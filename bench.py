#!/usr/bin/env python
"""TOPLOC prove+verify throughput (BASELINE.json metric) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--config cfg2] [--impl b200|reference]

One step = prove (tl_select + tl_commit) + verify (tl_verify) of every rollout of
this rank's batch, inputs resident in HBM (configs[1] = 256 rollouts x 8192
tokens, hidden 5120, per GPU; weak scaling over ranks).  Rank 0 prints one JSON
line.  ``--impl reference`` times the CPU TOPLOC restatement (oracle port) on the
host cores instead (the reference has no TOPLOC code of its own).
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TOPLOC tokens/sec (prove+verify) at hidden 5120; % of HBM roofline"
CONFIGS = {
    "cfg1": dict(R=1, T=2048, H=1024, name="configs[0]: 1 rollout x 2048 tokens, hidden 1024"),
    "cfg2": dict(R=256, T=8192, H=5120, name="configs[1]: QwQ-32B shape, 256 rollouts x 8192 tokens, hidden 5120"),
    "cfg3": dict(R=64, T=32768, H=5120, name="configs[2]: 64 rollouts x 32768 tokens, hidden 5120"),
    "cfg5": dict(R=1024, T=4096, H=8192, name="configs[4]: Llama-3-70B shape, 1024 rollouts x 4096 tokens, hidden 8192"),
}
CHUNK, TOPK = 32, 128
PROOF_BYTES = 2 + 2 * TOPK
JITTER_THR = 3277          # 5 % of elements +-1 ulp in the validator's recompute
# --schedule auto: the partitioned pipeline from this many chunks per GPU; below it the
# pipelined schedule captured as one CUDA graph (small batches: every kernel is
# latency-bound and the stages of different batches overlap).  Measured ms per step at
# H 5120 (pipegraph / partition, after the graph upload and the wider small-batch
# schedule): 1024 chunks 0.116 / 0.157, 2048 0.206 / 0.240, 4096 0.396 / 0.402,
# 8192 0.790 / 0.748; configuration 1 (64 chunks, H 1024) 0.009 / 0.115.
AUTO_PIPELINE_MIN_CHUNKS = 8192
LAUNCHES_PER_STEP = 7      # select: prefix+select; commit: inv_table+commit; verify: prefix+verify+verdict


def launches_per_step(eng, hidden, plan, co_resident: bool) -> int:
    """Kernels one prove+verify step launches: 7 for large batches; a batch the ring grid
    covers (<= 256 rollouts) needs no chunk_prefix_kernel (select 1, verify 2), and a small
    commitment (<= 4 chunks per SM) is one commit_coop_kernel launch (DESIGN 5.1b, 5.2)."""
    import torch
    st = torch.cuda.current_stream(hidden.device).cuda_stream
    g = int(eng.lib.tl_ring_grid(hidden.data_ptr(), plan.H, plan.n_chunks, 0, 0, st))
    own_prefix = 0 < plan.n_chunks <= g and plan.n_roll <= 256
    small_commit = not co_resident and plan.n_chunks <= 4 * int(eng.lib.tl_stream_sms(st))
    return (1 if own_prefix else 2) + (1 if small_commit else 2) + (2 if own_prefix else 3)


def select_kernel_name(eng, hidden, plan) -> str:
    """The kernel tl_select launches for this batch (the roofline's dominant kernel)."""
    import torch
    st = torch.cuda.current_stream(hidden.device).cuda_stream
    if int(eng.lib.tl_ring_grid(hidden.data_ptr(), plan.H, plan.n_chunks, 0, 0, st)) > 0:
        return "ring_stream_kernel<0> (tl_select, TMA ring: one chunk per CTA)"
    return "prove_select_kernel (tl_select)"


def algorithmic_bytes_per_token(H: int) -> float:
    """prove reads 2H + writes 258/32; verify reads 2H + 258/32."""
    return 4 * H + 2 * PROOF_BYTES / CHUNK


def select_bytes_per_token(H: int) -> float:
    """tl_select alone: reads 2H per token, writes K x (4 + 2) bytes per 32-token chunk."""
    return 2 * H + TOPK * 6 / CHUNK


NOMINAL_GBS = 8000.0  # B200 nominal HBM3e bandwidth


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self._t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baseline (oracle port)
def _cpu_pool_worker(kind, T, H, seed, cmd_q, res_q):
    """One host core: holds one rollout's prover and validator states (generated once,
    outside any timed region) and, per step command, proves and verifies it.

    kind "toploc": the TOPLOC restatement (oracle/toploc_oracle.py prove + verify).
    kind "exact": the reference's own exact-mode algorithm (oracle/exact_oracle.py restates
    rollout.py:51-68): commitments from the prover's states, then the validator's recompute
    and digest-list compare (checks.py:209-213)."""
    os.environ["OMP_NUM_THREADS"] = "1"
    import numpy as np
    from oracle import exact_oracle as EO
    from oracle import toploc_oracle as TO
    from oracle.synth_cpu import synth_bits
    prv = np.concatenate([synth_bits(r, min(512, T - r), H, seed) for r in range(0, T, 512)])
    if kind == "toploc":
        val = np.concatenate([synth_bits(r, min(512, T - r), H, seed, jitter_thr=JITTER_THR, jitter_seed=seed + 1)
                              for r in range(0, T, 512)])
        for p in TO.PRIMES_DESC[:8]:   # the port's inverse tables: built once, before any timing
            TO._inv_table(p)
    else:
        hidden = (prv.astype(np.uint32) << 16).view(np.float32)
    offs = [0, T]
    res_q.put(("ready", None))
    while cmd_q.get() is not None:
        t0 = time.perf_counter()
        if kind == "toploc":
            _, chunks = TO._chunks_of(prv, offs, CHUNK)
            _, _, proofs = TO.prove_chunks(chunks, TOPK, batch=16)
            _, verdict = TO.verify_proofs(val, offs, [proofs], CHUNK, TOPK)
            ok = bool(verdict[0])
        else:
            claimed = EO.build_commitments(hidden, CHUNK)
            ok = EO.build_commitments(hidden, CHUNK) == claimed
        res_q.put(("done", (time.perf_counter() - t0, T, ok)))


class CpuPool:
    """`workers` host processes (one per core), each holding one T-token rollout of the
    workload; a step = every worker proves and verifies its rollout once, wall-timed from
    the go signal to the last result.  Data generation and the port's table set-up happen
    once, at start, outside every timed step."""

    def __init__(self, kind: str, T: int, H: int, workers: int, seed0: int = 7):
        ctx = mp.get_context("spawn")
        self.T, self.workers = T, workers
        self.res_q = ctx.Queue()
        self.cmd_qs = [ctx.Queue() for _ in range(workers)]
        self.procs = [ctx.Process(target=_cpu_pool_worker, args=(kind, T, H, seed0 + w, self.cmd_qs[w], self.res_q),
                                  daemon=True) for w in range(workers)]
        for p in self.procs:
            p.start()
        for _ in self.procs:  # a worker that dies raises queue.Empty here instead of hanging the bench
            assert self.res_q.get(timeout=900)[0] == "ready"

    def step(self):
        t0 = time.perf_counter()
        for q in self.cmd_qs:
            q.put(1)
        done = [self.res_q.get(timeout=1800)[1] for _ in self.procs]
        return time.perf_counter() - t0, sum(d[1] for d in done), all(d[2] for d in done)

    def run(self, steps: int, warmup: int = 0):
        """-> (tokens/s over the timed steps, mean wall per step, all accepted)."""
        for _ in range(warmup):
            self.step()
        res = [self.step() for _ in range(steps)]
        self.step_ms = [round(r[0] * 1e3, 1) for r in res]
        wall = sum(r[0] for r in res)
        return sum(r[1] for r in res) / wall, wall / len(res), all(r[2] for r in res)

    def close(self):
        for q in self.cmd_qs:
            q.put(None)
        for p in self.procs:
            p.join(timeout=30)


def cpu_workers(T: int = 8192, H: int = 5120) -> int:
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:  # each worker holds its rollout twice plus the port's intermediates
        import psutil
        per_worker = 4 * T * H * 2 + (1 << 30)
        n = min(n, max(1, int(psutil.virtual_memory().available * 0.6 // per_worker)))
    except Exception:
        pass
    return max(1, min(n, 64))


def cpu_rollout_tokens(cfg) -> int:
    """Tokens per CPU worker: a whole rollout, or an 8192-token slice of a longer one."""
    return min(cfg["T"], 8192)


def config_block(args, cfg, R, R_total, world):
    """The workload description both arms print (the reference arm's step is a bounded
    sample of it, described in its cpu_baseline.sample)."""
    return {"workload": cfg["name"], "config": args.config, "rollouts_per_gpu": R, "rollouts_total": R_total,
            "tokens_per_rollout": cfg["T"], "hidden": cfg["H"], "chunk": CHUNK, "topk": TOPK, "dist": args.dist,
            "validator": "same states with 5% of elements +-1 ulp (GPU nondeterminism model)",
            "l2": (f"inputs {2 * R * cfg['T'] * cfg['H'] * 2 / 1e9:.1f} GB per GPU >> 126 MB L2; no flush needed"
                   if 2 * R * cfg["T"] * cfg["H"] * 2 > 4 * 126e6 else
                   f"inputs {2 * R * cfg['T'] * cfg['H'] * 2 / 1e6:.1f} MB fit in the 126 MB L2 (latency-bound "
                   f"configuration, not a roofline one); not flushed"),
            "parallelism": f"rollout-sharded x{world}"}


def cpu_baseline_block(cfg, steps: int, warmup: int, exact_steps: int = 1):
    """The oracle port timed on this host's cores (one process per core, whole rollouts),
    plus the reference's own exact-mode path on the same cores for scale."""
    T, H = cpu_rollout_tokens(cfg), cfg["H"]
    workers = cpu_workers(T, H)
    pool = CpuPool("toploc", T, H, workers)
    try:
        tps, per_step, ok = pool.run(steps, warmup)
    finally:
        pool.close()
    what = "whole" if T == cfg["T"] else f"{T}-token slices of"
    out = {"value": tps, "unit": "tokens/s", "cores": workers, "kind": "port", "per_core": tps / workers,
           "ms_per_step": per_step * 1e3, "steps": steps, "all_accepted": ok, "step_ms": pool.step_ms,
           "sample": f"per step {workers} processes (one per host core) each prove+verify {what} {cfg['T']}-token "
                     f"rollout(s) x H={H} with oracle/toploc_oracle.py; data and the port's inverse tables built "
                     f"before timing"}
    epool = CpuPool("exact", T, H, workers)
    try:
        etps, ewall, eok = epool.run(exact_steps, 1)
    finally:
        epool.close()
    out["reference_exact_mode"] = {
        "value": etps, "unit": "tokens/s", "cores": workers, "per_core": etps / workers, "digests_match": eok,
        "sample": f"per step {workers} processes each run build_commitments + recompute-and-compare on {what} "
                  f"{cfg['T']}-token rollout(s) x H={H} (oracle/exact_oracle.py, the reference's rollout.py:51-68 "
                  f"and checks.py:209-213)"}
    return out


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, cfg, rank, world):
    """The reference's CPU path for this workload on the box's host cores (rank 0 only;
    the reference has no TOPLOC code, so this is the oracle port, kind "port")."""
    if rank != 0:
        return
    cpu = cpu_baseline_block(cfg, args.steps, args.warmup)
    n_gpus = max(world, args.gpus)
    line = {
        "impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": "tokens/s", "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cpu["ms_per_step"], "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": config_block(args, cfg, cfg["R"], cfg["R"] * n_gpus, n_gpus),
        "cpu_baseline": cpu,
        "e2e": {"value": cpu["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "all_accepted": cpu["all_accepted"],
    }
    print(json.dumps(line), flush=True)


def e2e_rollouts(args, R, T, H, dev) -> int:
    """Rollouts per GPU in the e2e leg: --e2e-rollouts, or (0, the default) the whole batch
    when its pinned host copies (prover + validator) fit in 40 % of the host's available
    memory shared by this node's ranks and its device copies in 80 % of the free HBM; else
    as many as fit, at least 16."""
    if args.e2e_rollouts > 0:
        return min(R, args.e2e_rollouts)
    import torch
    per = 2 * T * H * 2
    local = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    try:
        import psutil
        host = psutil.virtual_memory().available * 0.4 / local
    except Exception:
        host = 16 * per
    dev_free = torch.cuda.mem_get_info(dev)[0] * 0.8
    return int(max(min(R, 16), min(R, host // per, dev_free // per)))


# ----------------------------------------------------------------------------- host placement
_AFFINITY0 = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None


def pin_to_gpu_numa_node(dev) -> dict | None:
    """Restrict this rank to the host cores of its GPU's NUMA node (sysfs local_cpulist), so
    pinned host buffers allocated afterwards are first-touched on that node and the e2e
    copies do not cross the socket interconnect.  Returns what was done, or None."""
    import torch
    try:
        pr = torch.cuda.get_device_properties(dev)
        bus = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        base = f"/sys/bus/pci/devices/{bus}"
        with open(f"{base}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        node = -1
        if os.path.exists(f"{base}/numa_node"):
            with open(f"{base}/numa_node") as f:
                node = int(f.read().strip())
        cpus &= _AFFINITY0 or cpus
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        return {"pci": bus, "numa_node": node, "cpus": len(cpus)}
    except Exception:
        return None


def restore_affinity() -> None:
    if _AFFINITY0 is not None:
        try:
            os.sched_setaffinity(0, _AFFINITY0)
        except OSError:
            pass


# ----------------------------------------------------------------------------- parity spot check
def spot_check(plan, T, H, seed, d, row0, n_random):
    """Full-size parity on sampled chunks, outside the timed region: the first and last
    chunk of the first, a middle and the last rollout plus `n_random` random chunks.
    Each is re-derived on the CPU from the counter-based generator (prover and validator
    states) and compared with the oracle: indices and value bits (select), proof bytes
    (commit), exponent mismatches, match counts, mantissa sums, means, medians and chunk
    verdicts (verify), and each sampled rollout's verdict against its chunks."""
    import numpy as np
    from oracle import toploc_oracle as TO
    from oracle.synth_cpu import synth_bits
    cpr = -(-T // CHUNK)
    R = plan.n_roll
    rng = np.random.default_rng(0)
    js = set(rng.choice(plan.n_chunks, size=min(n_random, plan.n_chunks), replace=False).tolist())
    for r in sorted({0, R // 2, R - 1}):
        js.update((r * cpr, r * cpr + cpr - 1))
    js = sorted(js)
    got_p = plan.proofs.cpu().numpy()
    got_i = plan.idx.cpu().numpy()
    got_b = plan.bits.cpu().numpy().view(np.uint16)
    st = plan.stats.cpu().numpy().view(_stats_dtype()).reshape(-1)
    cacc = plan.chunk_accept.cpu().numpy()
    racc = plan.rollout_accept.cpu().numpy()
    prv, val = [], []
    for j in js:
        r, c = divmod(j, cpr)
        r0 = row0 + r * T + c * CHUNK
        rows = min(CHUNK, T - c * CHUNK)
        prv.append(synth_bits(r0, rows, H, seed, d).reshape(-1))
        val.append(synth_bits(r0, rows, H, seed, d, jitter_thr=JITTER_THR, jitter_seed=seed + 1).reshape(-1))
    idxs, vals, proofs = TO.prove_chunks(prv, TOPK)
    bad = {"select": [], "proof": [], "stats": [], "chunk_verdict": []}
    for t, j in enumerate(js):
        kk = len(idxs[t])
        if not (np.array_equal(got_i[j, :kk], idxs[t]) and np.array_equal(got_b[j, :kk], vals[t])):
            bad["select"].append(j)
        if got_p[j].tobytes() != proofs[t]:
            bad["proof"].append(j)
        o = TO.verify_chunk(val[t], proofs[t], TOPK)
        g = st[j]
        if (int(g["exp_mismatch"]), int(g["n_match"]), int(g["mant_sum"]), float(g["mant_median"])) != \
                (o.exp_mismatch, o.n_match, o.mant_sum, o.mant_median) or not (
                float(g["mant_mean"]) == o.mant_mean):
            bad["stats"].append(j)
        if bool(cacc[j]) != o.accept or bool(g["flags"] & 1) != o.accept:
            bad["chunk_verdict"].append(j)
    roll_ok = all(bool(racc[r]) == bool(np.all(cacc[r * cpr:(r + 1) * cpr])) for r in sorted({0, R // 2, R - 1}))
    return {"chunks_checked": len(js), "boundary_rollouts": sorted({0, R // 2, R - 1}),
            "proofs_bit_exact": not bad["proof"], "select_bit_exact": not bad["select"],
            "verify_stats_exact": not bad["stats"], "chunk_verdicts_match": not bad["chunk_verdict"],
            "rollout_verdicts_consistent": roll_ok, "mismatches": {k: v[:8] for k, v in bad.items() if v},
            "chunks_rejected": int(sum(1 for j in js if not cacc[j]))}


def _stats_dtype():
    from paper_2505_07291_b200.api import STATS_DTYPE
    return STATS_DTYPE


# ----------------------------------------------------------------------------- B200 arm
def run_b200(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2505_07291_b200 import api
    from paper_2505_07291_b200.synth import DISTS, synth_device

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    R, T, H = cfg["R"], cfg["T"], cfg["H"]
    R_total = R
    d = DISTS[args.dist]
    shard = None
    if args.scaling == "strong":
        # the configuration's rollouts are one job sharded over the ranks by token count
        # (scheduler.shard_by_tokens); every rank generates its slice of the same tensor
        from paper_2505_07291_b200 import scheduler
        shard = scheduler.plan(np.full(R_total, T, dtype=np.int64), rank, world)
        R, row0, seed = shard.hi - shard.lo, shard.lo * T, 1000
        if R < 1:
            raise SystemExit(f"rank {rank}: no rollouts to shard ({R_total} rollouts over {world} ranks)")
    else:
        row0, seed = 0, 1000 + rank
    n_rows = R * T
    prv = synth_device(n_rows, H, seed, d, row0=row0, device=dev)
    val = synth_device(n_rows, H, seed, d, row0=row0, jitter_thr=JITTER_THR, jitter_seed=seed + 1, device=dev)
    offs = np.arange(R + 1, dtype=np.int64) * T
    eng = api.engine(dev)
    plan = eng.plan(offs, H)
    stream = torch.cuda.current_stream(dev)

    def step():
        plan.select(prv)
        plan.commit()
        plan.verify(val)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # serial per-phase times (informational: kernels run back to back, 4 CTAs/SM)
    ser = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(5)]
    for e in ser:
        e[0].record(stream)
        plan.select(prv)
        e[1].record(stream)
        plan.commit()
        e[2].record(stream)
        plan.verify(val)
        e[3].record(stream)
    torch.cuda.synchronize(dev)
    serial_ms = {k: sum(e[i].elapsed_time(e[i + 1]) for e in ser) / len(ser)
                 for i, k in enumerate(("select", "commit", "verify"))}

    # parity at full size on sampled chunks (outside the timed region): every rollout's
    # first and last chunk of a few rollouts plus random ones, proofs AND verify statistics
    # and verdicts against the oracle, re-derived on the CPU from the counter-based generator
    spot = None
    if args.spot_check and rank == 0:
        spot = spot_check(plan, T, H, seed, d, row0, args.spot_chunks)

    if args.schedule == "auto":
        # small batches are latency-bound: one CUDA graph per step beats the pipelines
        args.schedule = "partition" if plan.n_chunks >= AUTO_PIPELINE_MIN_CHUNKS else "pipegraph"
    args.pipeline_on = args.schedule in ("pipeline", "partition")
    pipe = None
    if args.schedule == "partition":
        try:
            pipe = api.PartitionedPipeline(eng, offs, H, commit_sms=args.commit_sms)
        except (RuntimeError, ValueError) as e:  # no green contexts: the co-resident pipeline instead
            print(f"bench: SM partition unavailable ({e}); using --schedule pipeline", file=sys.stderr)
            args.schedule = "pipeline"
    if pipe is None:
        pipe = api.Pipeline(eng, offs, H, ctas_per_sm=args.ctas) if args.pipeline_on else None
    graph = api.StepGraph(plan, prv, val) if args.schedule == "graph" else None
    pgraph = None
    if args.schedule == "pipegraph":
        pgraph_pipe = api.DualStreamPipeline(eng, offs, H, ctas_per_sm=args.pg_ctas)
        for _ in range(args.warmup):
            pgraph_pipe.run([prv], [val])
        pgraph = api.PipelineGraph(pgraph_pipe, [prv] * args.steps, [val] * args.steps)
    if graph is not None:
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize(dev)
    if pipe is not None:
        pipe.run([prv] * args.warmup, [val] * args.warmup)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sel_ev, ver_ev, com_ev = {}, {}, {}
    side_ms = None
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if pipe is not None:
        def mark(store):
            def f(k, what, st):
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(st)
                store.setdefault(k, {})[what] = ev
            return f
        t_start.record(stream)
        outs = pipe.run([prv] * args.steps, [val] * args.steps, on_select=mark(sel_ev), on_verify=mark(ver_ev),
                        on_commit=mark(com_ev))
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        sel_ms = sum(v["start"].elapsed_time(v["end"]) for v in sel_ev.values()) / args.steps
        ver_ms = sum(v["start"].elapsed_time(v["end"]) for v in ver_ev.values()) / args.steps
        com_ms = serial_ms["commit"]
        # the commitments as they ran beside the streams (side stream / partition; the first
        # and last of a partitioned run ran on the streaming SMs)
        side = [v["start"].elapsed_time(v["end"]) for k, v in sorted(com_ev.items())[1:-1]]
        side_ms = sum(side) / len(side) if side else None
        accepted = int(outs[-1].sum().item())
        assert all(int(o.sum().item()) == accepted for o in outs)
        spot_pipe = bool(torch.equal(pipe.plans[(args.steps - 1) % len(pipe.plans)].proofs, plan.proofs))
        if spot is not None:
            spot["pipeline_proofs_equal_serial"] = spot_pipe
    elif args.schedule == "graph":
        t_start.record(stream)
        for k in range(args.steps):
            graph.replay()
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        sel_ms, com_ms, ver_ms = serial_ms["select"], serial_ms["commit"], serial_ms["verify"]
        accepted = int(plan.rollout_accept.sum().item())
    elif args.schedule == "pipegraph":
        t_start.record(stream)
        outs = pgraph.replay()  # all K batches, pipelined, one graph launch
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        sel_ms, com_ms, ver_ms = serial_ms["select"], serial_ms["commit"], serial_ms["verify"]
        accepted = int(outs[-1].sum().item())
        assert all(int(o.sum().item()) == accepted for o in outs)
        spot_pipe = bool(torch.equal(pgraph_pipe.plans[(args.steps - 1) % len(pgraph_pipe.plans)].proofs, plan.proofs))
        if spot is not None:
            spot["pipeline_proofs_equal_serial"] = spot_pipe
    else:
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
        t_start.record(stream)
        for k in range(args.steps):
            e = evs[k]
            e[0].record(stream)
            plan.select(prv)
            e[1].record(stream)
            plan.commit()
            e[2].record(stream)
            plan.verify(val)
            e[3].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize(dev)
        sel_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
        com_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
        ver_ms = sum(e[2].elapsed_time(e[3]) for e in evs) / args.steps
        accepted = int(plan.rollout_accept.sum().item())
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)

    # max over ranks (device-timed)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    gather_ms = None
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)

        def gather():
            if shard is not None:
                from paper_2505_07291_b200 import scheduler
                return scheduler.gather_verdicts(plan.rollout_accept, shard.counts())
            out = torch.empty(world * R, dtype=torch.uint8, device=dev)
            dist.all_gather_into_tensor(out, plan.rollout_accept)
            return out

        gather()  # first call sets up the collective's buffers; time the second
        dist.barrier()
        torch.cuda.synchronize(dev)
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        gather()
        g1.record(stream)
        torch.cuda.synchronize(dev)
        gather_ms = g0.elapsed_time(g1)
    max_ms = float(t.item())
    tokens = (R_total if shard is not None else world * R) * T * args.steps
    value = tokens / (max_ms / 1e3)
    ms_per_step = max_ms / args.steps

    # e2e through the public API with host buffers (bounded sample of rollouts)
    e2e = None
    if args.e2e:
        Re = e2e_rollouts(args, R, T, H, dev)
        rows = Re * T
        numa = pin_to_gpu_numa_node(dev)   # pinned buffers first-touched on the GPU's NUMA node
        hp = torch.empty((rows, H), dtype=torch.bfloat16, pin_memory=True)
        hv = torch.empty((rows, H), dtype=torch.bfloat16, pin_memory=True)
        hp.copy_(prv[:rows])
        hv.copy_(val[:rows])
        torch.cuda.synchronize(dev)
        offs_e = offs[:Re + 1]
        times = []
        h2d = d2h = 0
        for it in range(1 + args.e2e_steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            pb = eng.prove(hp, offs_e)                      # H2D inside the call
            proofs_host = pb.proofs.cpu()                   # prover ships proofs
            vb = eng.verify(hv, offs_e, proofs_host)        # validator: H2D hidden + proofs
            verdict_host = vb.rollout_accept.cpu()
            b.record(stream)
            torch.cuda.synchronize(dev)
            if it >= 1:
                times.append(a.elapsed_time(b))
            h2d = 2 * rows * H * 2 + proofs_host.numel() + (len(offs_e)) * 8 * 2
            d2h = proofs_host.numel() + verdict_host.numel()
        del hp, hv  # the pinned copies (whole batch: 43 GB) before the CPU legs
        te = torch.tensor([sum(times) / len(times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": world * rows / (float(te.item()) / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "rollouts_per_gpu": Re, "of_rollouts_per_gpu": R,
               "h2d_gbs_per_gpu": h2d / (float(te.item()) / 1e3) / 1e9, "host_numa": numa,
               "note": "public API (ToplocEngine.prove/verify) from pinned host tensors; proofs and verdicts read "
                       "back; bound by the host link (h2d_gbs_per_gpu against ~55 GB/s for PCIe 5 x16)"}

    peak, peak_src = measured_peak()
    sel_bytes = n_rows * select_bytes_per_token(H)
    # the kernel's own launch time: in the partitioned schedule select and verify overlap on
    # two streams, so their spans there are not launch durations; use the serial pass
    kern_ms = serial_ms["select"] if args.schedule == "partition" else sel_ms
    achieved = sel_bytes / (kern_ms / 1e3) / 1e9
    ver_bytes = n_rows * (2 * H + PROOF_BYTES / CHUNK) + plan.n_chunks * 33 + R
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_select_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            if pj.get("config") == args.config:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:
            pass

    # the reference's own (exact-mode) algorithm on this GPU, for scale: whole SHA-256
    # chains over round(h, 6) (tl_exact_chains), checked against the host chains
    exact = None
    if args.exact and rank == 0 and world == 1:
        from paper_2505_07291_b200.exact import build_commitments_batch
        Rx, Tx = 4096, 256
        hx = torch.empty((Rx * Tx, H), dtype=torch.bfloat16, device=dev)
        synth_device(Rx * Tx, H, seed=11, device=dev, out=hx)
        ox = np.arange(Rx + 1, dtype=np.int64) * Tx
        build_commitments_batch(hx[:Tx], ox[:2], 32, sha="device")  # warm-up
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        dg = build_commitments_batch(hx, ox, 32, sha="device")
        tx = time.perf_counter() - t0
        ok = all(dg[r] == build_commitments_batch(hx[r * Tx:(r + 1) * Tx], ox[:2], 32, sha="host")[0]
                 for r in (0, Rx - 1))
        exact = {"value": Rx * Tx / tx, "unit": "tokens/s", "rollouts": Rx, "tokens_per_rollout": Tx,
                 "digests_match_host": ok,
                 "note": "the reference's exact-mode commitments (rollout.py:51-68) as whole SHA-256 chains on "
                         "the GPU, one lane per rollout, wall time including the digest read-back; compare "
                         "cpu_baseline.reference_exact_mode"}
        del hx

    cpu = None
    if args.cpu_baseline and rank == 0:   # after the timed region; the other ranks wait at the final barrier
        restore_affinity()
        cpu = cpu_baseline_block(cfg, steps=10, warmup=2)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "u16", "data": "synthetic",
            "config": config_block(args, cfg, R, R_total if shard is not None else world * R, world),
            "roofline": {"bound": "hbm", "kernel": select_kernel_name(eng, prv, plan), "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": sel_bytes, "avg_launch_ms": kern_ms, "peak_source": peak_src,
                         "launch_timing": ("serial pass (in the timed schedule the kernel overlaps verify)"
                                           if args.schedule == "partition" else "timed schedule")},
            "step_roofline": {"bytes_per_token": algorithmic_bytes_per_token(H),
                              "achieved_gbs": value / world * algorithmic_bytes_per_token(H) / 1e9,
                              "frac": value / world * algorithmic_bytes_per_token(H) / 1e9 / peak,
                              # report both denominators; the primary is the measured peak
                              "frac_of_nominal_8tbs": value / world * algorithmic_bytes_per_token(H) / 1e9 / NOMINAL_GBS},
            "phases_ms": {"select": sel_ms, "commit": com_ms, "verify": ver_ms,
                          "note": ("select and verify spans overlap (two streams); see serial for launch times"
                                   if args.schedule == "partition" else None),
                          "commit_beside_streams": side_ms if pipe is not None else None,
                          "verify_gbs": ver_bytes / ((serial_ms["verify"] if args.schedule == "partition" else ver_ms)
                                                     / 1e3) / 1e9, "verdict_gather": gather_ms,
                          "serial": serial_ms,
                          "schedule": (f"partitioned: commit on {pipe.sms[1]} SMs; select and verify (lagging two "
                                       f"batches) on two streams over the other {pipe.sms[0]} SMs (green contexts)"
                                       if args.schedule == "partition" else
                                       f"pipelined: commit(k) on a side stream overlaps verify(k-1); "
                                       f"select/verify {args.ctas} CTAs/SM" if args.pipeline_on else
                                       "graph: serial step replayed as one CUDA graph" if args.schedule == "graph"
                                       else f"pipegraph: select, commit and verify of different batches, each stage "
                                            f"alternating between {len(pgraph_pipe.sstreams)} streams, "
                                            f"{len(pgraph_pipe.plans)} rotating buffer sets, all {args.steps} batches "
                                            f"captured as one CUDA graph, uploaded before the timed region: "
                                            f"{pgraph.uploaded}"
                                       if args.schedule == "pipegraph"
                                       else "serial")},
            "cpu_baseline": cpu,
            "exact_mode": exact,
            "e2e": e2e,
            "gpu_launches": launches_per_step(eng, prv, plan, args.schedule == "pipeline") * args.steps,
            "comm": ({"backend": "nccl", "nranks": world, "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                      "data_path_collectives": 0, "collective": "one all_gather of the per-rollout verdict bytes"}
                     if world > 1 else None),
            "clocks": clk,
            "rollouts_accepted": f"{accepted}/{R}",
            "parity_spot_check": spot,
        }
        print(json.dumps(line), flush=True)


def self_launch(n: int) -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # keep stdout to the one JSON line
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--dist", default="normal", choices=["normal", "massive"])
    ap.add_argument("--rollouts", type=int, default=0, help="override the configuration's rollout count (sweeps)")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--e2e-rollouts", type=int, default=0,
                    help="rollouts per GPU through the public API from host memory (0: the whole batch when "
                         "host and device memory allow, e2e_rollouts())")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-exact", dest="exact", action="store_false",
                    help="skip the exact-mode (reference algorithm) GPU measurement")
    ap.add_argument("--cpu-tokens", type=int, default=8192)
    ap.add_argument("--no-spot-check", dest="spot_check", action="store_false")
    ap.add_argument("--spot-chunks", type=int, default=64, help="random chunks in the full-size parity check")
    ap.add_argument("--schedule", default="auto",
                    choices=["auto", "partition", "pipeline", "serial", "graph", "pipegraph"],
                    help="auto (default): partition from 8192 chunks per GPU (AUTO_PIPELINE_MIN_CHUNKS), pipegraph below; "
                         "partition: the pipeline on two SM partitions (green contexts), commit on "
                         "--commit-sms SMs, select/verify on the rest; "
                         "pipeline: commit(k) on a side stream, co-resident with verify(k-1) and select(k+1); "
                         "serial: tl_select, tl_commit, tl_verify back to back; graph: the serial step "
                         "captured as one CUDA graph (api.StepGraph) and replayed; pipegraph: select, commit "
                         "and verify of different batches on three streams (api.DualStreamPipeline), all K "
                         "batches captured as one CUDA graph (api.PipelineGraph)")
    ap.add_argument("--commit-sms", type=int, default=24, help="SMs of the commitment partition (--schedule partition)")
    ap.add_argument("--pipeline", dest="schedule", action="store_const", const="pipeline")
    ap.add_argument("--partition", dest="schedule", action="store_const", const="partition")
    ap.add_argument("--serial", dest="schedule", action="store_const", const="serial")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak (default): every rank runs the configuration; strong: the configuration's "
                         "rollouts are sharded over the ranks by token count (scheduler.plan)")
    ap.add_argument("--pg-ctas", type=int, default=0,
                    help="select/verify CTAs per SM in the pipegraph schedule (0: full occupancy)")
    ap.add_argument("--ctas", type=int, default=16,
                    help="select/verify one-warp CTAs per SM in pipeline mode (leaves room for the commit CTA)")
    args = ap.parse_args()
    args.pipeline_on = args.schedule in ("pipeline", "partition")
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")

    if args.impl == "b200" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` without a launcher: re-execute under torch.distributed.run,
        # one NCCL rank per GPU (NCCL's init lines, with the communicator's nranks, go to stderr)
        sys.exit(self_launch(args.gpus))

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "b200" and world != args.gpus and rank == 0:
        print(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}; running {world} ranks", file=sys.stderr)
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    cfg = dict(CONFIGS[args.config])
    if args.rollouts:
        cfg["R"] = args.rollouts
        cfg["name"] = f"{cfg['name']} (rollouts overridden: {args.rollouts})"
    if args.impl == "reference":     # rank 0 alone times the CPU path; other ranks exit 0
        run_reference(args, cfg, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        if rank == 0:  # the communicator the verdict gather uses (NCCL's own INIT lines need NCCL_DEBUG=INFO)
            print(f"bench: NCCL communicator up: nranks {world} (NCCL {'.'.join(map(str, torch.cuda.nccl.version()))}, "
                  f"one process per GPU)", file=sys.stderr, flush=True)
    try:
        run_b200(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
