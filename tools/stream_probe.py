"""Time (or profile under ncu) the streaming kernels on one batch shape: the TMA-ring
kernels (ctas_per_sm 0) against the one-warp-per-chunk kernels (ctas_per_sm -1).

    python tools/stream_probe.py [--rollouts 64 --tokens 8192 --hidden 5120 --iters 5 --modes ring,warp]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rollouts", type=int, default=64)
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=5120)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--modes", default="ring,warp")
    ap.add_argument("--dist", default="normal")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2505_07291_b200 import api
    from paper_2505_07291_b200.synth import synth_device
    R, T, H = args.rollouts, args.tokens, args.hidden
    offs = np.arange(R + 1, dtype=np.int64) * T
    eng = api.engine()
    prv = synth_device(R * T, H, 1000, args.dist).view(torch.int16)
    val = synth_device(R * T, H, 1000, args.dist, jitter_thr=3277, jitter_seed=1001).view(torch.int16)
    out = {"shape": [R, T, H]}

    def entry_us(vt):  # per CTA: kernel entry -> first ring stage landed / first chunk handed to the finisher
        n = max(1, vt[7])
        return {"first_stage": round(vt[6] / n / 1.9e3, 3), "first_ready": round(vt[5] / n / 1.9e3, 3)}
    plans = {}
    for mode in args.modes.split(","):
        ctas = {"ring": -2, "auto": 0, "warp": -1}[mode]
        plan = plans[mode] = eng.plan(offs, H)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        for it in range(args.iters + 1):
            ev[0].record()
            plan.select(prv, ctas_per_sm=ctas)
            ev[1].record()
            plan.commit()
            plan.verify(val, ctas_per_sm=ctas)
            ev[2].record()
            torch.cuda.synchronize()
            if it == 1:
                sel, ver = [], []
            if it >= 1:
                sel.append(ev[0].elapsed_time(ev[1]))
                ver.append(ev[1].elapsed_time(ev[2]))
        lab = getattr(eng.lib, "tl_ring_lab_stats", None) if os.environ.get("TOPLOC_B200_LIB") else None
        if lab is not None and mode == "ring":  # lab build with TL_RING_STATS: per-chunk tail counters
            import ctypes
            buf = (ctypes.c_ulonglong * 8)()
            lab(buf, 1)
            tr = (ctypes.c_uint * 4096)()
            eng.lib.tl_ring_lab_trace(tr)
            plan.select(prv, ctas_per_sm=ctas)
            torch.cuda.synchronize()
            lab(buf, 1)
            eng.lib.tl_ring_lab_trace(tr)
            out["trace_select_cta0"] = [[tr[4 * i] & 0x7FFFFFFF, tr[4 * i] >> 31, tr[4 * i + 1], tr[4 * i + 2],
                                         tr[4 * i + 3]] for i in range(60)]
            n = max(1, buf[0])
            out["ring_stats_select"] = {"chunks": buf[0], "candidates_per_chunk": buf[1] / n,
                                        "rescans_per_chunk": buf[2] / n, "compacting_warps_per_chunk": buf[3] / n,
                                        "tail_us_per_chunk": buf[4] / n / 1.9e3}
            vt = (ctypes.c_ulonglong * 8)()
            eng.lib.tl_ring_lab_vt(vt)
            out["select_entry_us"] = entry_us(vt)
            plan.verify(val, ctas_per_sm=ctas)
            torch.cuda.synchronize()
            lab(buf, 1)
            eng.lib.tl_ring_lab_vt(vt)
            out["verify_tail_phase_us"] = [round(vt[i] / max(1, buf[0]) / 1.9e3, 3) for i in range(5)]
            out["verify_entry_us"] = entry_us(vt)
            n = max(1, buf[0])
            out["ring_stats_verify"] = {"chunks": buf[0], "candidates_per_chunk": buf[1] / n,
                                        "rescans_per_chunk": buf[2] / n, "compacting_warps_per_chunk": buf[3] / n,
                                        "tail_us_per_chunk": buf[4] / n / 1.9e3,
                                        "merge_us": buf[5] / n / 1.9e3, "spec_us": buf[6] / n / 1.9e3,
                                        "verify_tail_us": buf[7] / n / 1.9e3}
        gb = R * T * H * 2 / 1e9
        out[mode] = {"select_ms": min(sel), "select_gbs": gb / min(sel) * 1e3,
                     "commit_verify_ms": min(ver)}
    if "ring" in plans and "warp" in plans:
        a, b = plans["ring"], plans["warp"]
        out["identical"] = all(torch.equal(getattr(a, k), getattr(b, k)) for k in
                               ("idx", "bits", "proofs", "stats", "chunk_accept"))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
