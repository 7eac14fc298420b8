"""TMA-ring / cp.async-ring streaming ceilings (lab): python tools/lab/streamprobe.py"""
import ctypes, os
import torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstreamprobe.so"))
lib.probe_tma.restype = ctypes.c_float
lib.probe_tma.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_int] * 5
lib.probe_cpasync.restype = ctypes.c_float
lib.probe_cpasync.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_int] * 3
nbytes = 21_474_836_480
x = torch.empty(nbytes // 2, dtype=torch.int16, device="cuda")
x.random_()
for SB, S, W, C in [(16384, 12, 8, 1), (16384, 6, 8, 2), (8192, 12, 8, 2), (4096, 24, 8, 2), (2048, 24, 4, 4),
                    (32768, 6, 8, 1), (8192, 24, 8, 1), (4096, 12, 4, 4), (16384, 4, 4, 3), (65536, 3, 8, 1)]:
    ms = lib.probe_tma(x.data_ptr(), nbytes, SB, S, W, C, 5)
    print(f"tma  stage {SB:6d} x {S:2d}  consumers {W}  ctas/SM {C}: {ms:.3f} ms  {nbytes / ms / 1e6 if ms > 0 else 0:.0f} GB/s", flush=True)
for T, C in [(256, 4), (512, 2), (256, 6), (128, 8), (1024, 1)]:
    ms = lib.probe_cpasync(x.data_ptr(), nbytes, T, C, 5)
    print(f"cpasync threads {T:4d} ctas/SM {C}: {ms:.3f} ms  {nbytes / ms / 1e6 if ms > 0 else 0:.0f} GB/s", flush=True)
