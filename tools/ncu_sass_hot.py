"""Summarise the SASS source page of every kernel in an ncu report: opcode mix by
instructions executed and stall samples, and the hottest instruction windows.

    python tools/ncu_sass_hot.py REPORT.ncu-rep [window] [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 24
TOP = int(sys.argv[3]) if len(sys.argv) > 3 else 5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kernels, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        kernels.append(cur)
    elif r and r[0] == "Address":
        cur[1] = r
    elif cur and cur[1] and r:
        cur[2].append(r)
for name, h, body in kernels:
    si, ie, ws = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    L = []
    for k, r in enumerate(body):
        try:
            L.append((k, int(r[ie] or 0), int(r[ws] or 0), r[si].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(x[1] for x in L) or 1
    tws = sum(x[2] for x in L) or 1
    print(f"##### {name[:90]}\ninstructions {tot}  stall samples {tws}")
    op, st = Counter(), Counter()
    for _, i, w, s in L:
        t = s.split()
        o = (t[1] if t and t[0].startswith("@") and len(t) > 1 else t[0] if t else "?").split(".")[0]
        op[o] += i
        st[o] += w
    for o, i in op.most_common(16):
        print(f"  {o:14s} {i / tot * 100:5.1f}% inst  {st[o] / tws * 100:5.1f}% stall")
    blocks = [(sum(x[1] for x in L[b:b + W]), sum(x[2] for x in L[b:b + W]), b) for b in range(0, len(L), W)]
    for i_, s_, b in sorted(blocks, reverse=True)[:TOP]:
        print(f"  == block {b}: inst {i_ / tot * 100:.1f}%  stall {s_ / tws * 100:.1f}%")
        for x in L[b:b + W]:
            if x[1]:
                print(f"     {x[0]:5d} {x[1]:>10d} {x[2]:>6d}  {x[3][:84]}")
