"""The C-ABI library loads on a GPU-less host and exports exactly the header's symbols.

No compute calls here (there is no GPU); only host-side helpers and argument
validation, which return before touching the device."""

import ctypes
import os
import re

import pytest

from paper_2505_07291_b200 import _build, _ffi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "toploc_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(tl_[a-z0-9_]+)\s*\(", src))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _ffi.load()


def test_header_and_binding_agree():
    assert header_functions() == set(_ffi.SYMBOLS)


def test_library_exports_every_symbol(lib):
    for name in header_functions():
        assert getattr(lib, name) is not None


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_helpers(lib):
    assert lib.tl_version() == 1
    assert lib.tl_strerror(0) == b"ok"
    offs = (ctypes.c_int64 * 5)(0, 45, 45, 110, 141)
    assert lib.tl_count_chunks(ctypes.cast(offs, ctypes.c_void_p), 4, 32) == 2 + 0 + 3 + 1
    assert lib.tl_workspace_bytes(4, 6, 128) >= 8 * 65536 * 2 + 6 * 128 * 6


def test_argument_validation_before_device(lib):
    # K > 128, C*H too large, negative sizes: rejected without any CUDA call
    assert lib.tl_prove(None, None, 1, 32, 5120, 32, 129, 1, None, None, None, None, 0, None) == _ffi.TL_EUNSUPPORTED
    assert lib.tl_prove(None, None, 1, 32, 1 << 20, 32, 128, 1, None, None, None, None, 0, None) == _ffi.TL_EUNSUPPORTED
    assert lib.tl_prove(None, None, -1, 32, 64, 32, 128, 1, None, None, None, None, 0, None) == _ffi.TL_EINVAL
    th = _ffi.Thresholds(38, 0, 10.0, 8.0)
    assert lib.tl_verify(None, None, 1, 32, 64, 0, 128, 1, None, ctypes.byref(th), None, None, None, None, 0,
                         None) == _ffi.TL_EINVAL
    assert lib.tl_round6(None, 7, 10, None, None) == _ffi.TL_EINVAL
    assert lib.tl_synth_bf16(None, 0, 4, 0, 0, 0, None, None, 0, 0, None) == _ffi.TL_EINVAL


def test_workspace_and_pointer_checks_before_device(lib):
    """Undersized or misaligned workspaces and missing buffers are rejected on the host.
    The pointers are never dereferenced: every call returns before its first CUDA call."""
    fake = 1 << 20                                    # 256-aligned, never touched
    offs = (ctypes.c_int64 * 3)(0, 64, 128)
    ro = ctypes.cast(offs, ctypes.c_void_p).value
    need = int(lib.tl_workspace_bytes(2, 4, 128))
    th = _ffi.Thresholds(38, 0, 10.0, 8.0)
    E = _ffi.TL_EWORKSPACE
    for ws, nbytes in ((fake, need - 1), (fake + 16, need), (fake, 0)):
        assert lib.tl_select(fake, ro, 2, 128, 256, 32, 128, 4, fake, fake, ws, nbytes, None) == E
        assert lib.tl_prove(fake, ro, 2, 128, 256, 32, 128, 4, fake, None, None, ws, nbytes, None) == E
        assert lib.tl_verify(fake, ro, 2, 128, 256, 32, 128, 4, fake, ctypes.byref(th), None, None, None,
                             ws, nbytes, None) == E
    assert lib.tl_commit(fake, fake, 4, 128, fake, fake + 8, need, None) == E
    # a missing buffer is EINVAL, whatever the workspace
    assert lib.tl_select(fake, ro, 2, 128, 256, 32, 128, 4, None, fake, fake, need, None) == _ffi.TL_EINVAL
    assert lib.tl_prove(fake, ro, 2, 128, 256, 32, 128, 4, None, None, None, fake, need, None) == _ffi.TL_EINVAL
    assert lib.tl_verify(fake, ro, 2, 128, 256, 32, 128, 4, None, ctypes.byref(th), None, None, None,
                         fake, need, None) == _ffi.TL_EINVAL
    assert lib.tl_commit(None, fake, 4, 128, fake, fake, need, None) == _ffi.TL_EINVAL
    # empty batches are no-ops that never look at the buffers
    assert lib.tl_prove(None, None, 0, 0, 256, 32, 128, 0, None, None, None, None, 0, None) == _ffi.TL_OK
    assert lib.tl_commit(None, None, 0, 128, None, None, 0, None) == _ffi.TL_OK


def test_errors_map_to_python_exceptions(lib):
    with pytest.raises(ValueError):
        _ffi.check(_ffi.TL_EINVAL, "x")
    with pytest.raises(_ffi.ToplocError):
        _ffi.check(_ffi.TL_ECUDA, "x")


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2505_07291_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), f
