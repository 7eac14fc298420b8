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
# three-stream pipeline captured as one CUDA graph (small batches: every kernel is
# latency-bound and the stages of different batches overlap).  Measured ms per step,
# pipegraph / graph / partition: configuration 1 (64 chunks, H 1024) 0.047 / 0.066 / 0.115;
# H 5120 at 256 chunks 0.078 / 0.113 / 0.118, 1024 chunks 0.146 / 0.208 / 0.161, 2048 chunks
# 0.268 / - / 0.257, 4096 chunks 0.431 / 0.554 / 0.432.
AUTO_PIPELINE_MIN_CHUNKS = 2048
LAUNCHES_PER_STEP = 7      # select: prefix+select; commit: inv_table+commit; verify: prefix+verify+verdict


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
def _cpu_worker(args):
    """One worker = one rollout slice: oracle prove + verify (TOPLOC restatement)."""
    (T, H, seed, start_evt, q) = args
    os.environ["OMP_NUM_THREADS"] = "1"
    import numpy as np
    from oracle import toploc_oracle as TO
    from oracle.synth_cpu import synth_bits
    prv = np.concatenate([synth_bits(r, min(512, T - r), H, seed) for r in range(0, T, 512)])
    val = np.concatenate([synth_bits(r, min(512, T - r), H, seed, jitter_thr=JITTER_THR, jitter_seed=seed + 1)
                          for r in range(0, T, 512)])
    offs = [0, T]
    q.put(("ready", None))
    start_evt.wait()
    t0 = time.perf_counter()
    tab, chunks = TO._chunks_of(prv, offs, CHUNK)
    _, _, proofs = TO.prove_chunks(chunks, TOPK, batch=16)
    stats, verdict = TO.verify_proofs(val, offs, [proofs], CHUNK, TOPK)
    dt = time.perf_counter() - t0
    q.put(("done", (dt, T, bool(verdict[0]))))


def _cpu_exact_worker(args):
    """One worker = one rollout slice through the reference's own exact-mode algorithm
    (oracle/exact_oracle.py restates rollout.py:51-68): commitments from the prover's
    states, then the validator's recompute and digest-list compare (checks.py:209-213)."""
    (T, H, seed, start_evt, q) = args
    os.environ["OMP_NUM_THREADS"] = "1"
    import numpy as np
    from oracle import exact_oracle as EO
    from oracle.synth_cpu import synth_bits
    bits = np.concatenate([synth_bits(r, min(512, T - r), H, seed) for r in range(0, T, 512)])
    hidden = (bits.astype(np.uint32) << 16).view(np.float32)
    q.put(("ready", None))
    start_evt.wait()
    t0 = time.perf_counter()
    claimed = EO.build_commitments(hidden, CHUNK)
    ok = EO.build_commitments(hidden, CHUNK) == claimed
    dt = time.perf_counter() - t0
    q.put(("done", (dt, T, ok)))


def cpu_sample(T: int, H: int, workers: int, steps: int = 1, warmup: int = 0, worker=None):
    """Run `warmup + steps` rounds of `workers` parallel oracle prove+verify slices."""
    ctx = mp.get_context("spawn")
    results = []
    for it in range(warmup + steps):
        q = ctx.Queue()
        evt = ctx.Event()
        procs = [ctx.Process(target=worker or _cpu_worker, args=((T, H, 7 + it * 1000 + w, evt, q),))
                 for w in range(workers)]
        for p in procs:
            p.start()
        for _ in procs:  # a worker that dies raises queue.Empty here instead of hanging the bench
            assert q.get(timeout=600)[0] == "ready"
        t0 = time.perf_counter()
        evt.set()
        done = [q.get(timeout=1800)[1] for _ in procs]
        wall = time.perf_counter() - t0
        for p in procs:
            p.join()
        if it >= warmup:
            results.append((wall, sum(d[1] for d in done), all(d[2] for d in done)))
    wall = sum(r[0] for r in results)
    toks = sum(r[1] for r in results)
    return toks / wall, wall / len(results), all(r[2] for r in results)


def cpu_workers() -> int:
    n = os.cpu_count() or 1
    try:
        import psutil
        mem_gb = psutil.virtual_memory().available / 2 ** 30
        n = min(n, max(1, int(mem_gb // 2)))
    except Exception:
        pass
    return max(1, min(n, 64))


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    workers = cpu_workers()
    T_slice = 1024
    tps, per_step, ok = cpu_sample(T_slice, cfg["H"], workers, steps=args.steps, warmup=args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": tps, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
        "config": {"workload": cfg["name"], "hidden": cfg["H"], "chunk": CHUNK, "topk": TOPK,
                   "sample": f"{workers} parallel slices of {T_slice} tokens x H={cfg['H']} per step"},
        "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": workers, "kind": "port",
                         "sample": f"{workers} x {T_slice}-token slices (hidden {cfg['H']}) per step, "
                                   "oracle/toploc_oracle.py prove+verify, one process per core"},
        "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "all_accepted": ok,
    }
    # the reference's own exact-mode path (rollout.py:51-68 + checks.py:209-213) on the same cores
    etps, ewall, eok = cpu_sample(T_slice, cfg["H"], workers, steps=1, warmup=0, worker=_cpu_exact_worker)
    line["cpu_baseline"]["reference_exact_mode"] = {
        "value": etps, "unit": "tokens/s", "cores": workers, "digests_match": eok,
        "sample": f"{workers} x {T_slice}-token slices: build_commitments + recompute-and-compare "
                  "(oracle/exact_oracle.py)"}
    print(json.dumps(line), flush=True)


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

    # spot-check bit-exactness at full size on sampled chunks (outside the timed region)
    spot = None
    if args.spot_check and rank == 0:
        from oracle import toploc_oracle as TO
        from oracle.synth_cpu import synth_bits
        rng = np.random.default_rng(0)
        js = sorted(rng.choice(plan.n_chunks, size=min(3, plan.n_chunks), replace=False).tolist())
        got = plan.proofs.cpu().numpy()
        okp = []
        for j in js:
            r0 = (j // (T // CHUNK)) * T + (j % (T // CHUNK)) * CHUNK
            rows = min(CHUNK, T - (j % (T // CHUNK)) * CHUNK)
            bits = synth_bits(r0, rows, H, seed, d)
            _, _, pr = TO.prove_chunks([bits.reshape(-1)], TOPK)
            okp.append(pr[0] == got[j].tobytes())
        spot = {"chunks": js, "proofs_bit_exact": all(okp)}

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
        spot_pipe = bool(torch.equal(pgraph_pipe.plans[(args.steps - 1) % 3].proofs, plan.proofs))
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
        Re = min(R, args.e2e_rollouts)
        rows = Re * T
        hp = torch.empty((rows, H), dtype=torch.bfloat16).pin_memory()
        hv = torch.empty((rows, H), dtype=torch.bfloat16).pin_memory()
        hp.copy_(prv[:rows].cpu())
        hv.copy_(val[:rows].cpu())
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
        te = torch.tensor([sum(times) / len(times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": world * rows / (float(te.item()) / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "rollouts_per_gpu": Re,
               "h2d_gbs_per_gpu": h2d / (float(te.item()) / 1e3) / 1e9,
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
    if args.cpu_baseline and rank == 0 and world == 1:
        workers = cpu_workers()
        tps, wall, ok = cpu_sample(args.cpu_tokens, H, workers, steps=1, warmup=0)
        cpu = {"value": tps, "unit": "tokens/s", "cores": workers, "kind": "port",
               "sample": f"{workers} parallel {args.cpu_tokens}-token slices x H={H} "
                         f"(oracle/toploc_oracle.py prove+verify, one process per core), wall {wall:.1f}s"}
        # the reference's own (exact-mode) path on the same cores, for scale
        etps, ewall, eok = cpu_sample(4096, H, workers, steps=1, warmup=0, worker=_cpu_exact_worker)
        cpu["reference_exact_mode"] = {
            "value": etps, "unit": "tokens/s", "cores": workers, "per_core": etps / workers, "digests_match": eok,
            "sample": f"{workers} parallel 4096-token slices x H={H}: build_commitments + recompute-and-compare "
                      f"(oracle/exact_oracle.py, the reference's rollout.py:51-68), wall {ewall:.1f}s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "u16", "data": "synthetic",
            "config": {"workload": cfg["name"], "config": args.config, "rollouts_per_gpu": R,
                       "rollouts_total": R_total if shard is not None else world * R, "tokens_per_rollout": T,
                       "hidden": H, "chunk": CHUNK, "topk": TOPK, "dist": args.dist,
                       "validator": "same states with 5% of elements +-1 ulp (GPU nondeterminism model)",
                       "l2": f"inputs {2 * n_rows * H * 2 / 1e9:.1f} GB per GPU >> 126 MB L2; no flush needed",
                       "parallelism": f"rollout-sharded x{world}"},
            "roofline": {"bound": "hbm", "kernel": "prove_select_kernel (tl_select)", "achieved": achieved,
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
                                       else f"pipegraph: select, commit and verify of different batches on three "
                                            f"streams, all {args.steps} batches captured as one CUDA graph"
                                       if args.schedule == "pipegraph"
                                       else "serial")},
            "cpu_baseline": cpu,
            "exact_mode": exact,
            "e2e": e2e,
            "gpu_launches": LAUNCHES_PER_STEP * args.steps,
            "clocks": clk,
            "rollouts_accepted": f"{accepted}/{R}",
            "parity_spot_check": spot,
        }
        print(json.dumps(line), flush=True)


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
    ap.add_argument("--e2e-rollouts", type=int, default=16)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-exact", dest="exact", action="store_false",
                    help="skip the exact-mode (reference algorithm) GPU measurement")
    ap.add_argument("--cpu-tokens", type=int, default=8192)
    ap.add_argument("--no-spot-check", dest="spot_check", action="store_false")
    ap.add_argument("--schedule", default="auto",
                    choices=["auto", "partition", "pipeline", "serial", "graph", "pipegraph"],
                    help="auto (default): partition from 2048 chunks per GPU (AUTO_PIPELINE_MIN_CHUNKS), pipegraph below; "
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

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
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
    try:
        run_b200(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
