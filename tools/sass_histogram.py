"""Static SASS opcode histogram of the library's kernels (cuobjdump -sass), with the
instructions that show the Blackwell paths: UBLKCP (cp.async.bulk), UBLKPF (bulk L2
prefetch), UTMALDG (tensor-map TMA), SYNCS (mbarrier), HMNMX2 (bf16x2 |max|).

    python tools/sass_histogram.py [lib.so] > profiles/r02_sass_histogram.txt
"""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2505_07291_b200/_lib/libtoploc_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kernels, cur = {}, None
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        kernels[cur] = Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if cur and m:
        kernels[cur][m.group(2)] += 1
KEY = ("UBLKCP", "UBLKPF", "UTMALDG", "SYNCS", "HMNMX2", "LDG", "LDS", "SHFL", "IMAD", "VIMNMX")
print(f"# SASS opcode histogram of {lib} (static counts per kernel)\n")
for name in sorted(kernels, key=lambda n: -sum(kernels[n].values())):
    c = kernels[name]
    pretty = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
    print(f"## {pretty[:110]}\n   total {sum(c.values())}; " +
          ", ".join(f"{k} {c[k]}" for k in KEY if c[k]))
    print("   top: " + ", ".join(f"{k} {v}" for k, v in c.most_common(14)) + "\n")
