"""tl_record_checks at configuration-2 size (256 records x 8192 probabilities), lab timing
of the kernel alone (inputs already on the device)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2505_07291_b200 import _ffi, api  # noqa: E402

R, T = 256, 8192
lib = _ffi.load()
probs = torch.rand(R * T, dtype=torch.float64, device="cuda")
offs = torch.from_numpy(np.arange(R + 1, dtype=np.int64) * T).cuda()
pl = torch.full((R,), 64, dtype=torch.int32, device="cuda")
eos = torch.ones(R, dtype=torch.uint8, device="cuda")
out = torch.empty(R, dtype=torch.int32, device="cuda")
frac = torch.empty(R, dtype=torch.float64, device="cuda")
plast = torch.empty(R, dtype=torch.float64, device="cuda")
th = api.RecordThresholds(max_len=16384).to_c()
s = torch.cuda.current_stream().cuda_stream


def call():
    _ffi.check(lib.tl_record_checks(probs.data_ptr(), offs.data_ptr(), R, pl.data_ptr(), eos.data_ptr(),
                                    ctypes.byref(th), None, None, out.data_ptr(), frac.data_ptr(), plast.data_ptr(), s),
               "tl_record_checks")


call()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    call()
b.record()
torch.cuda.synchronize()
us = a.elapsed_time(b) / 50 * 1e3
print(f"tl_record_checks 256 x 8192 (16.8 MB of float64): {us:.1f} us per call, {R * T * 8 / us / 1e3:.0f} GB/s")
