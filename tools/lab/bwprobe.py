"""Read-bandwidth ceiling on this B200 (lab): python tools/lab/bwprobe.py"""
import ctypes, json, os
import torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbwprobe.so"))
lib.probe.restype = ctypes.c_float
lib.probe.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
nbytes = 21_474_836_480
x = torch.empty(nbytes // 2, dtype=torch.int16, device="cuda")
x.random_()
res = []
for variant, name in [(0, "U4.na"), (1, "U8.na"), (2, "U4.ldg"), (3, "U16.na"), (4, "U2.na")]:
    for bps, thr in [(4, 256), (8, 256), (2, 512), (16, 128), (1, 1024)]:
        ms = lib.probe(x.data_ptr(), nbytes, variant, bps, thr, 5)
        res.append((name, bps, thr, ms, nbytes / ms / 1e6))
        print(f"{name:7s} blocks/SM {bps:2d} x {thr:4d}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s", flush=True)
best = max(res, key=lambda r: r[4])
print(json.dumps({"best_read_gbs": best[4], "config": best[:3]}))
