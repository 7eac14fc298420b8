"""Per-phase clock64 breakdown of prove_select_kernel (lab).

    TOPLOC_B200_LIB=paper_2505_07291_b200/_lib/libtoploc_prof.so python tools/lab/phaseprof.py

The library must be built with -DTL_PHASE_PROF=1 (tools/lab/phaseprof.py --build)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2505_07291_b200 import _build  # noqa: E402

LIB = os.path.join(_build.OUT_DIR, "libtoploc_prof.so")
if "--build" in sys.argv:
    extra = [a for a in sys.argv[2:]]
    _build.build(out=LIB, defines=["TL_PHASE_PROF=1"] + extra)
    sys.exit(0)
os.environ.setdefault("TOPLOC_B200_LIB", LIB)
import torch  # noqa: E402
from paper_2505_07291_b200 import _ffi, api, synth  # noqa: E402

lib = _ffi.load()
lib.tl_phase_prof.restype = ctypes.c_int
lib.tl_phase_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
n_roll, T, H = 256, 8192, 5120
dist = sys.argv[1] if len(sys.argv) > 1 else "normal"
kern = sys.argv[2] if len(sys.argv) > 2 else "select"
h = synth.synth_device(n_roll * T, H, 1234, dist)
offs = np.arange(n_roll + 1, dtype=np.int64) * T
plan = api.engine().plan(offs, H)
buf = np.zeros(16, dtype=np.uint64)
run = {"select": plan.select, "prove": plan.prove, "verify": lambda x: plan.verify(x)}[kern]
if kern == "verify":
    plan.prove(h)
for _ in range(2):
    run(h)
torch.cuda.synchronize()
lib.tl_phase_prof(buf.ctypes.data, 1)
reps = 5
for _ in range(reps):
    run(h)
torch.cuda.synchronize()
lib.tl_phase_prof(buf.ctypes.data, 1)
ghz = 1.95
names = ["geo", "pass", "re-scan", "sort+spec", "output/verify tail"]
c = buf[:8].astype(np.float64)
chunks = c[5]
print(f"{kern} dist {dist}: chunks {chunks:.0f}, mean candidates {c[6] / chunks:.1f}, re-scanned {c[7] / chunks:.4f}")
print("per chunk per warp, microseconds at %.2f GHz: " % ghz +
      "  ".join(f"{names[i]} {c[i] / chunks / (ghz * 1e3):.2f}" for i in range(5)) +
      f"  | total {(c[:5].sum() + buf[8]) / chunks / (ghz * 1e3):.2f}  theta=0 passes {buf[8] / chunks / (ghz * 1e3):.2f}")

lib.tl_phase_prof_warps.restype = ctypes.c_int
lib.tl_phase_prof_warps.argtypes = [ctypes.c_void_p]
run(h)
torch.cuda.synchronize()
wt = np.zeros((8192, 2), dtype=np.uint64)
lib.tl_phase_prof_warps(wt.ctypes.data)
used = wt[:, 1] > 0
st, en = wt[used, 0].astype(np.float64), wt[used, 1].astype(np.float64)
t0 = st.min()
q = np.percentile(en - t0, [0, 1, 10, 50, 90, 99, 100]) / 1e3
print(f"warps {used.sum()}: start spread {(st.max() - t0) / 1e3:.1f} us; end (us from first start) "
      "p0/1/10/50/90/99/100: " + " ".join(f"{v:.0f}" for v in q))
