"""Chunked-stream read probe (lab): python tools/lab/chunkprobe.py  (see chunkprobe.cu)"""
import ctypes, os
import torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libchunkprobe.so"))
lib.probe_grid.restype = ctypes.c_float
lib.probe_grid.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_int] * 4
lib.probe_chunked.restype = ctypes.c_float
lib.probe_chunked.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_int] * 7
CHUNK = 32 * 5120 * 2
nbytes = 65536 * CHUNK  # configuration 2's tensor: 21.47 GB
x = torch.empty(nbytes // 2, dtype=torch.int16, device="cuda")
x.random_()
lib.probe_warp.restype = ctypes.c_float
lib.probe_warp.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_int] * 6
for U, bps, thr, tail in [(4, 8, 96, 0), (4, 8, 96, 8000), (4, 8, 96, 16000), (4, 6, 128, 8000), (8, 6, 128, 8000),
                          (4, 8, 128, 8000), (4, 16, 64, 8000)]:
    ms = lib.probe_warp(x.data_ptr(), nbytes, CHUNK, U, bps, thr, tail, 5)
    print(f"warp    U{U} {bps:2d} x {thr:4d} tail {tail:5d} ns: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s", flush=True)
for U, bps, thr in [(4, 8, 96), (4, 4, 256), (8, 4, 256)]:
    ms = lib.probe_grid(x.data_ptr(), nbytes, U, bps, thr, 5)
    print(f"grid    U{U} {bps:2d} x {thr:4d}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s", flush=True)
for U, bps, thr, tail, order in [(4, 8, 96, 0, 0), (4, 8, 96, 8000, 0)]:
    ms = lib.probe_chunked(x.data_ptr(), nbytes, CHUNK, U, bps, thr, tail, order, 5)
    print(f"chunked U{U} {bps:2d} x {thr:4d} tail {tail:5d} ns order {order}: {ms:.3f} ms  "
          f"{nbytes / ms / 1e6:.0f} GB/s", flush=True)
