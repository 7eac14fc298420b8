"""Per-phase clock64 breakdown of commit_kernel for small batches (lab).

    python tools/lab/commitprof.py --build      # here: libtoploc_cprof.so with -DTL_COMMIT_PROF=1
    python tools/lab/commitprof.py [reps]       # on the GPU

Global warp 0's cycles per phase, averaged over its chunks: table staging, idx/bits load,
modulus search, divided differences, Newton -> monomial conversion, serialisation."""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2505_07291_b200 import _build  # noqa: E402

LIB = os.path.join(_build.OUT_DIR, "libtoploc_cprof.so")
if "--build" in sys.argv:
    _build.build(out=LIB, defines=["TL_COMMIT_PROF=1"] + sys.argv[2:])
    sys.exit(0)
os.environ.setdefault("TOPLOC_B200_LIB", LIB)
import torch  # noqa: E402
from paper_2505_07291_b200 import _ffi, api, synth  # noqa: E402

lib = _ffi.load()
lib.tl_commit_prof.restype = ctypes.c_int
lib.tl_commit_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
names = ["staging", "load", "modulus", "ndd", "conversion", "serialise"]
coop_names = ["load", "modulus", "leaves", "weights", "trees", "serialise"]  # commit_coop_kernel
out = {"lib": os.environ["TOPLOC_B200_LIB"]}
for R, T, H in ((1, 32, 1024), (1, 2048, 1024), (1, 2048, 5120), (256, 8192, 5120)):
    h = synth.synth_device(R * T, H, 1000)
    plan = api.engine().plan(np.arange(R + 1, dtype=np.int64) * T, H)
    plan.select(h)
    plan.commit()
    torch.cuda.synchronize()
    buf = np.zeros(8, dtype=np.uint64)
    lib.tl_commit_prof(buf.ctypes.data, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.commit()
    e1.record()
    torch.cuda.synchronize()
    lib.tl_commit_prof(buf.ctypes.data, 1)
    n = max(int(buf[7]), 1)
    small = R * T // 32 <= 4 * int(lib.tl_stream_sms(None))
    row = {k: round(float(buf[i]) / n) for i, k in enumerate(coop_names if small else names)}
    if not small:
        row["staging"] = round(float(buf[0]) / reps)
    row["chunks_of_warp0"] = n
    row["launch_us"] = round(e0.elapsed_time(e1) * 1e3 / reps, 2)
    out[f"{R}x{T}x{H}"] = row
    del h, plan
    torch.cuda.empty_cache()
print(json.dumps(out))
