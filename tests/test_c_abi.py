"""The C ABI from plain C (examples/c_abi_demo.c): built with gcc against
include/toploc_b200.h and the in-tree library, run on the GPU, and checked against the
same inputs through the Python layer."""

import os
import shutil
import subprocess

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def fnv1a(b: bytes) -> int:
    h = 1469598103934665603
    for x in b:
        h = ((h ^ x) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def test_c_program_matches_python(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    from paper_2505_07291_b200 import _build, _ffi, api
    lib_dir = os.path.dirname(_build.LIB)
    exe = str(tmp_path / "c_abi_demo")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", lib_dir, "-ltoploc_b200",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    H = 1024
    out = subprocess.run([exe, str(H)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    fields = out.stdout.split()
    n_chunks, got_hash = int(fields[1]), int(fields[3], 16)
    verdicts = [int(v) for v in fields[5:8]]

    # the same inputs through the Python layer
    lib = _ffi.load()
    offs = [0, 70, 128, 300]
    table = torch.tensor([(0x3000 + (i >> 4)) for i in range(65536)], dtype=torch.int32).to(torch.int16).cuda()
    prv = torch.empty((300, H), dtype=torch.int16, device="cuda")
    val = torch.empty((300, H), dtype=torch.int16, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _ffi.check(lib.tl_synth_bf16(prv.data_ptr(), 0, 300, H, 0x1234567, 0, table.data_ptr(), None, 0, 0, s), "synth")
    _ffi.check(lib.tl_synth_bf16(val.data_ptr(), 0, 300, H, 0x1234567, 0, table.data_ptr(), None, 3277, 0x99, s),
               "synth")
    eng = api.engine()
    pb = eng.prove(prv, offs)
    vb = eng.verify(val, offs, pb)
    proofs = pb.proofs.cpu().numpy()
    assert proofs.shape[0] == n_chunks
    assert fnv1a(proofs.tobytes()) == got_hash
    assert vb.rollout_accept.cpu().tolist() == verdicts
