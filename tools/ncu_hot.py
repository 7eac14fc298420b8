"""Summarise an ncu report's SASS source page: hottest instruction windows.

    python tools/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX [window] [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
W = int(sys.argv[3]) if len(sys.argv) > 3 else 25
TOP = int(sys.argv[4]) if len(sys.argv) > 4 else 6
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si, ie, ws = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
L = []
for k, r in enumerate(rows[2:]):
    if r and r[0].startswith("Kernel Name"):
        break
    try:
        L.append((k, int(r[ie] or 0), int(r[ws] or 0), r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(x[1] for x in L) or 1
tws = sum(x[2] for x in L) or 1
print(f"instructions {tot}  stall samples {tws}  sass lines {len(L)}")
blocks = [(sum(x[1] for x in L[b:b + W]), sum(x[2] for x in L[b:b + W]), b) for b in range(0, len(L), W)]
for i_, s_, b in sorted(blocks, reverse=True)[:TOP]:
    print(f"== block {b}: inst {i_ / tot * 100:.1f}%  stall {s_ / tws * 100:.1f}%")
    for x in L[b:b + W]:
        if x[1]:
            print(f"   {x[0]:5d} {x[1]:>11d} {x[2]:>6d}  {x[3][:90]}")
