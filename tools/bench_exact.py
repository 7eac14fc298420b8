"""Exact-mode (reference parity shim) throughput: GPU round6 + pipelined host SHA-256
(exact.build_commitments_batch) vs the reference's algorithm on all host cores
(oracle/exact_oracle.py == swarm/worker/rollout.py:51-68, one process per core).

    python tools/bench_exact.py [--rollouts 32 --tokens 8192 --hidden 5120]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _cpu_worker(args):
    T, H, seed, q, evt = args
    import numpy as np
    from oracle import exact_oracle as EO
    from oracle.synth_cpu import synth_bits
    bits = np.concatenate([synth_bits(r, min(512, T - r), H, seed) for r in range(0, T, 512)])
    h = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    q.put("ready")
    evt.wait()
    t0 = time.perf_counter()
    d = EO.build_commitments(h, 32)
    q.put((time.perf_counter() - t0, len(d)))


def device_sweep(H: int, T: int, rollouts) -> dict:
    """Whole chains on the GPU (tl_exact_chains) vs the host-SHA path, by batch size."""
    import numpy as np
    import torch
    from paper_2505_07291_b200.exact import build_commitments_batch, build_commitments_device
    from paper_2505_07291_b200.synth import synth_device
    res = {}
    for R in rollouts:
        x = synth_device(R * T, H, seed=5)
        offs = np.arange(R + 1, dtype=np.int64) * T
        build_commitments_device(x[:T], offs[:2], 32)  # warm-up
        nw = min(R, max(1, 65536 // T))  # one full row group: allocates and pins the host staging
        build_commitments_batch(x[:nw * T], offs[:nw + 1], 32, sha="host")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev = build_commitments_device(x, offs, 32)
        t_dev = time.perf_counter() - t0
        t0 = time.perf_counter()
        host = build_commitments_batch(x, offs, 32, sha="host")
        t_host = time.perf_counter() - t0
        res[R] = {"device_s": t_dev, "host_s": t_host, "device_tokens_per_s": R * T / t_dev,
                  "host_tokens_per_s": R * T / t_host, "equal": dev == host}
        del x
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rollouts", type=int, default=32)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=5120)
    ap.add_argument("--cpu-workers", type=int, default=0)
    ap.add_argument("--device-sweep", default="", help="comma-separated rollout counts: GPU chains vs host SHA")
    args = ap.parse_args()
    if args.device_sweep:
        print(json.dumps({"mode": "exact, GPU SHA chains vs host SHA", "hidden": args.hidden,
                          "tokens_per_rollout": args.tokens,
                          "by_rollouts": device_sweep(args.hidden, args.tokens,
                                                      [int(v) for v in args.device_sweep.split(",")])}))
        return
    import numpy as np
    import torch
    from paper_2505_07291_b200.exact import build_commitments_batch
    from paper_2505_07291_b200.synth import synth_device
    R, T, H = args.rollouts, args.tokens, args.hidden
    x = synth_device(R * T, H, seed=3)
    offs = np.arange(R + 1, dtype=np.int64) * T
    build_commitments_batch(x, offs, 32, group_rows=65536)      # warm-up (allocates the staging)
    torch.cuda.synchronize()
    sweep = {}
    for gr in (4096, 8192, 16384, 65536):
        t0 = time.perf_counter()
        dig = build_commitments_batch(x, offs, 32, group_rows=gr)
        sweep[gr] = time.perf_counter() - t0
    gpu_s = min(sweep.values())
    # check two rollouts against the reference algorithm
    from oracle import exact_oracle as EO
    ok = all(dig[r] == EO.build_commitments(x[r * T:(r + 1) * T].to(torch.float64).cpu().numpy(), 32)
             for r in (0, R - 1))
    workers = args.cpu_workers or min(os.cpu_count() or 1, 16)
    ctx = mp.get_context("spawn")
    q, evt = ctx.Queue(), ctx.Event()
    ps = [ctx.Process(target=_cpu_worker, args=((T, H, 3 + w, q, evt),)) for w in range(workers)]
    for p in ps:
        p.start()
    for _ in ps:
        q.get()
    t1 = time.perf_counter()
    evt.set()
    res = [q.get() for _ in ps]
    cpu_wall = time.perf_counter() - t1
    for p in ps:
        p.join()
    print(json.dumps({
        "mode": "exact (reference parity shim)", "rollouts": R, "tokens_per_rollout": T, "hidden": H,
        "gpu_tokens_per_s": R * T / gpu_s, "gpu_wall_s": gpu_s, "group_rows_sweep_s": sweep, "bit_exact_vs_reference_algorithm": ok,
        "host_threads": os.cpu_count(),
        "cpu_reference_tokens_per_s": workers * T / cpu_wall, "cpu_workers": workers,
        "cpu_per_core_tokens_per_s": T / (sum(r[0] for r in res) / len(res)),
        "note": "GPU: round(x,6) on device, D2H f64 (8 B/elem) + SHA-256 chains on host threads; "
                "bounded by host SHA-NI and PCIe D2H"}))


if __name__ == "__main__":
    main()
