"""Summarise ncu captures into profiles/ (tracked):

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep gpurun_out/launches.csv profiles/rNN [bench.json]

Writes <prefix>_ncu_summary.md (per-kernel metrics from the --set full capture and the
launch list of the same bench command) and profiles/ncu_prove_traffic.json /
ncu_select_traffic.json (DRAM bytes per tl_prove / tl_select launch, read by bench.py
for roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

rep, launches, prefix = sys.argv[1], sys.argv[2], sys.argv[3]
bench = json.load(open(sys.argv[4])) if len(sys.argv) > 4 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__shared_mem_per_block_static", "static smem/block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]
out = [f"# ncu summary ({os.path.basename(rep)})", "",
       "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
       "(cold, serialised replays: compare shares, not absolute times).", ""]
traffic = {}  # per streaming kernel
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    short = name.split("(")[0].split("::")[-1]
    out.append(f"## {short}")
    out.append("")
    out.append("| metric | value | unit |")
    out.append("|---|---|---|")
    for key, label in WANT:
        if key in hdr:
            i = hdr.index(key)
            out.append(f"| {label} (`{key}`) | {r[i]} | {units[i]} |")

    def val(key):
        i = hdr.index(key)
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
                 "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}.get(units[i], 1.0)
        return float(r[i].replace(",", "")) * scale

    try:
        gbs = (val("dram__bytes_read.sum") + val("dram__bytes_write.sum")) / val("gpu__time_duration.sum") / 1e9
        out.append(f"| achieved DRAM bandwidth (read + write) / duration | {gbs:.0f} | GB/s |")
        out.append(f"| ... of the measured 6,445 GB/s copy peak / the nominal 8,000 GB/s | "
                   f"{gbs / 6445.3:.3f} / {gbs / 8000:.3f} | |")
    except (ValueError, ZeroDivisionError):
        pass
    st = {}
    for i, n in enumerate(hdr):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                st[n.split("stalled_")[1]] = float(r[i])
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
    out.append("")
    out.append("Warp stall samples: " + ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in top))
    out.append("")
    if short.split("<")[0] in ("prove_kernel", "prove_select_kernel"):
        def gbytes(key):
            i = hdr.index(key)
            v = float(r[i])
            return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(units[i], 1.0)
        traffic[short.split("<")[0]] = {"kernel": short, "dram_bytes_per_launch": gbytes("dram__bytes_read.sum") + gbytes("dram__bytes_write.sum"),
                   "config": "cfg2", "source": os.path.basename(rep)}
# launch list
lrows = list(csv.reader(open(launches)))
hi = next(i for i, r in enumerate(lrows) if "Kernel Name" in r)
h = lrows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
per = {}
for r in lrows[hi + 1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    k = r[ki].split("(")[0].split("::")[-1]
    per.setdefault(k, []).append(float(r[vi].replace(",", "")) * (1e-6 if r[ui] == "ns" else 1e-3 if r[ui] == "us" else 1.0))
out.append("## Launch list (same bench command, `--metrics gpu__time_duration.sum --clock-control none`)")
out.append("")
out.append("| kernel | launches | mean ms | share of the step's main kernels |")
out.append("|---|---|---|---|")
STEP = ("prove_kernel", "prove_select_kernel", "commit_kernel", "verify_kernel")
step = sum(sum(v) / len(v) for k, v in per.items() if k.split("<")[0] in STEP)
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
    m = sum(v) / len(v)
    share = f"{m / step * 100:.1f}%" if k.split("<")[0] in STEP and step else ""
    out.append(f"| {k} | {len(v)} | {m:.4f} | {share} |")
if any(k.startswith("commit_kernel") for k in per):
    out.append("")
    out.append("Under ncu the commitment kernel runs on the whole GPU (the profiler's replay does not keep the "
               "bench's green-context partition), so its time is the standalone one; in the partitioned schedule "
               "it runs on 24 SMs beside the streaming kernels.")
if bench:
    out.append("")
    ph = bench.get("phases_ms", {})
    keys = [k for k in ("prove", "select", "commit", "verify") if isinstance(ph.get(k), (int, float))]
    live = sum(ph[k] for k in keys)
    out.append("Live (CUDA events, bench.py) shares: " + ", ".join(f"{k} {ph[k] / live * 100:.1f}%" for k in keys))
open(prefix + "_ncu_summary.md", "w").write("\n".join(out) + "\n")
for name, fn in (("prove_kernel", "ncu_prove_traffic.json"), ("prove_select_kernel", "ncu_select_traffic.json")):
    if name in traffic:
        json.dump(traffic[name], open(os.path.join(os.path.dirname(prefix), fn), "w"), indent=1)
print("\n".join(out))
