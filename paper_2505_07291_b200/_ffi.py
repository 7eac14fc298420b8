"""ctypes binding of ``include/toploc_b200.h`` (the C ABI of the CUDA path).

There is no fallback: if the in-tree shared library is missing or fails to load,
every entry point raises.  ``SYMBOLS`` lists exactly the functions the header
declares; ``tests/test_abi.py`` checks the two stay in sync.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import _build

c_i32, c_i64, c_u64, c_sz, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_void_p

TL_OK, TL_EINVAL, TL_EUNSUPPORTED, TL_EWORKSPACE, TL_ECUDA = 0, -1, -2, -3, -4
TL_MAX_K = 128
TL_STAT_ACCEPT, TL_STAT_BADPROOF = 1, 2


class Thresholds(ctypes.Structure):
    _fields_ = [("max_exp_mismatch", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("max_mant_mean", ctypes.c_double), ("max_mant_median", ctypes.c_double)]


class ChunkStats(ctypes.Structure):
    _fields_ = [("exp_mismatch", ctypes.c_uint32), ("n_match", ctypes.c_uint32),
                ("mant_sum", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("mant_mean", ctypes.c_double), ("mant_median", ctypes.c_double)]


class RecordThresholds(ctypes.Structure):
    _fields_ = [("max_len", ctypes.c_int32), ("min_sampling_len", ctypes.c_int32),
                ("eos_prob_floor", ctypes.c_double), ("p_low", ctypes.c_double), ("theta", ctypes.c_double)]


# name -> (restype, argtypes); must match include/toploc_b200.h
SYMBOLS = {
    "tl_strerror": (ctypes.c_char_p, [c_i32]),
    "tl_version": (c_i32, []),
    "tl_count_chunks": (c_i64, [c_vp, c_i32, c_i32]),
    "tl_workspace_bytes": (c_sz, [c_i32, c_i64, c_i32]),
    "tl_prove": (c_i32, [c_vp, c_vp, c_i32, c_i64, c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp,
                         c_vp, c_sz, c_vp]),
    "tl_select": (c_i32, [c_vp, c_vp, c_i32, c_i64, c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "tl_commit": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_sz, c_vp]),
    "tl_select_ex": (c_i32, [c_vp, c_vp, c_i32, c_i64, c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_sz, c_i32,
                             c_vp]),
    "tl_commit_ex": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_sz, c_i32, c_vp]),
    "tl_verify_ex": (c_i32, [c_vp, c_vp, c_i32, c_i64, c_i32, c_i32, c_i32, c_i64, c_vp,
                             ctypes.POINTER(Thresholds), c_vp, c_vp, c_vp, c_vp, c_sz, c_i32, c_vp]),
    "tl_verify": (c_i32, [c_vp, c_vp, c_i32, c_i64, c_i32, c_i32, c_i32, c_i64, c_vp,
                          ctypes.POINTER(Thresholds), c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "tl_round6": (c_i32, [c_vp, c_i32, c_i64, c_vp, c_vp]),
    "tl_exact_chains": (c_i32, [c_vp, c_i32, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "tl_partition_create": (c_i32, [c_i32, c_vp, c_vp]),
    "tl_partition_destroy": (c_i32, [c_vp]),
    "tl_stream_sms": (c_i32, [c_vp]),
    "tl_prepare": (c_i32, []),
    "tl_ring_grid": (c_i32, [c_vp, c_i32, c_i64, c_i32, c_i32, c_vp]),
    "tl_record_checks": (c_i32, [c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "tl_synth_bf16": (c_i32, [c_vp, c_i64, c_i64, c_i32, c_u64, c_i32, c_vp, c_vp, c_i32, c_u64, c_vp]),
}

_lock = threading.Lock()
_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load the in-tree library (building it first if absent and nvcc exists)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("TOPLOC_B200_LIB", _build.LIB)  # experiments: alternative builds
        if not os.path.exists(path):
            if not build_if_missing:
                raise RuntimeError(f"CUDA extension missing: {path} (run __graft_entry__.build())")
            _build.build()
        lib = ctypes.CDLL(path)
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class ToplocError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    if rc != TL_OK:
        msg = load().tl_strerror(rc).decode()
        if rc in (TL_EINVAL, TL_EUNSUPPORTED):
            raise ValueError(f"{what}: {msg} ({rc})")
        raise ToplocError(f"{what}: {msg} ({rc})")
