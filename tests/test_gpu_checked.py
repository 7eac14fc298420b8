"""The GPU fuzz and parity suites once more against the bounds-checked library
(-DTL_CHECKED=1: device asserts on flat indices, workspace offsets, split-part and ring-stage
bounds; paper_2505_07291_b200/_build.py:build_checked).  compute-sanitizer is closed on the
GPU pool, so this is its substitute: a violated bound traps, the launch fails and the
suite fails.  Runs in a subprocess because a process loads one library."""

import os
import subprocess
import sys

import pytest

from paper_2505_07291_b200 import _build

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["tests/test_gpu_parity.py", "tests/test_gpu_ring.py"]
SELECT = ("fuzz or split or ragged or many or malformed or forged or fails_closed or speculation or orderings or "
          "ties or golden or shapes or variants or matches_warp or wide or other_chunk or commitment or cooperative")


def test_fuzz_and_parity_suites_pass_under_the_checked_build():
    lib = _build.build_checked()
    env = dict(os.environ, TOPLOC_B200_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                        "-k", SELECT, *SUITES], cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    import re
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) >= 40, r.stdout[-2000:]   # the selection covers the fuzz / parity cases
    assert "TL_CHECK failed" not in r.stdout + r.stderr
    print(f"checked build: {m.group(0)}")


def test_checked_library_traps_on_a_bound_violation():
    """The asserts are live: a chunk count larger than the rows hold (the caller's n_chunks is
    trusted only up to the device-side prefix, so force a bad prefix through row offsets
    past the tensor) traps instead of reading past the hidden states."""
    lib = _build.build_checked()
    code = r'''
import ctypes, numpy as np, torch, sys
from paper_2505_07291_b200 import _ffi
L = _ffi.load()
H, rows = 1024, 64
h = torch.zeros((rows, H), dtype=torch.int16, device="cuda")
offs = torch.tensor([0, 64, 4096], dtype=torch.int64, device="cuda")   # rollout 1 claims rows past the tensor
n_chunks = 2 + (4096 - 64) // 32
ws = torch.empty(int(L.tl_workspace_bytes(2, n_chunks, 128)), dtype=torch.uint8, device="cuda")
idx = torch.empty((n_chunks, 128), dtype=torch.int32, device="cuda")
bits = torch.empty((n_chunks, 128), dtype=torch.int16, device="cuda")
rc = L.tl_select_ex(h.data_ptr(), offs.data_ptr(), 2, rows, H, 32, 128, n_chunks, idx.data_ptr(), bits.data_ptr(),
                    ws.data_ptr(), ws.numel(), -1, None)
try:
    torch.cuda.synchronize()
except Exception as e:
    print("trapped:", type(e).__name__)
    sys.exit(0)
print("no trap", rc)
sys.exit(1)
'''
    env = dict(os.environ, TOPLOC_B200_LIB=lib)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "TL_CHECK failed" in r.stdout + r.stderr
