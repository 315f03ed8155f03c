"""ctypes loader for libsbmds.so (include/sbmds.h). Fails loudly: there is no fallback path."""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libsbmds.so")
_lock = threading.Lock()
_lib = None

SBMDS_OK, SBMDS_EINVAL, SBMDS_ENOMEM, SBMDS_ECUDA, SBMDS_ENOCONV, SBMDS_EBREAKDOWN = range(6)
SBMDS_BORROW_D = 1 << 0
SBMDS_VALIDATE = 1 << 1
SBMDS_REORDER_ROWS = 1 << 2
STATUS_NAMES = {0: "SBMDS_OK", 1: "SBMDS_EINVAL", 2: "SBMDS_ENOMEM", 3: "SBMDS_ECUDA",
                4: "SBMDS_ENOCONV", 5: "SBMDS_EBREAKDOWN"}

# Every symbol include/sbmds.h declares (checked by tests/test_abi.py on CPU).
EXPORTS = ("sbmds_create", "sbmds_apply", "sbmds_eigs", "sbmds_destroy", "sbmds_last_error",
           "sbmds_set_option", "sbmds_get_stat", "sbmds_launch_count", "sbmds_abi_version",
           "sbmds_plan_selfcheck", "sbmds_plan_selfcheck_rect", "sbmds_sparse_split_rows", "sbmds_create_shard", "sbmds_shard_stage", "sbmds_shard_exchange_bytes",
           "sbmds_shard_attach_nccl", "sbmds_nccl_unique_id", "sbmds_shard_plan_selfcheck", "sbmds_shard_tiles", "sbmds_bmds", "sbmds_sbha_p", "sbmds_sbha_build")
NCCL_UNIQUE_ID_BYTES = 128


class SbmdsInfo(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("n_applies", ctypes.c_int32),
                ("n_negative", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("max_residual", ctypes.c_double), ("orth_error", ctypes.c_double),
                ("gpu_ms", ctypes.c_double)]


class SbhaInfo(ctypes.Structure):
    _fields_ = [("nnz", ctypes.c_int64), ("p", ctypes.c_int32), ("bandwidth", ctypes.c_int32),
                ("window", ctypes.c_int32), ("seconds", ctypes.c_double)]


class SbmdsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib() -> ctypes.CDLL:
    """Load libsbmds.so; raise if it has not been built (no CPU or Python fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"libsbmds.so not found at {LIB_PATH}; run __graft_entry__.build() "
                    "(nvcc, sm_100a). There is no fallback implementation.")
            L = ctypes.CDLL(LIB_PATH)
            p, i32, i64, u32, u64, d = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                        ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double)
            L.sbmds_create.argtypes = [i64, i64, i64, p, p, p, p, u32, p, ctypes.POINTER(p)]
            L.sbmds_create.restype = ctypes.c_int
            L.sbmds_apply.argtypes = [p, i32, p, p, p]
            L.sbmds_apply.restype = ctypes.c_int
            L.sbmds_eigs.argtypes = [p, i32, i32, i32, d, u64, p, p, p, p,
                                     ctypes.POINTER(SbmdsInfo), p]
            L.sbmds_eigs.restype = ctypes.c_int
            L.sbmds_destroy.argtypes = [p]
            L.sbmds_destroy.restype = None
            L.sbmds_last_error.argtypes = []
            L.sbmds_last_error.restype = ctypes.c_char_p
            L.sbmds_set_option.argtypes = [p, ctypes.c_char_p, i64]
            L.sbmds_set_option.restype = ctypes.c_int
            L.sbmds_get_stat.argtypes = [p, ctypes.c_char_p, ctypes.POINTER(i64)]
            L.sbmds_get_stat.restype = ctypes.c_int
            L.sbmds_launch_count.argtypes = []
            L.sbmds_launch_count.restype = i64
            L.sbmds_abi_version.argtypes = []
            L.sbmds_abi_version.restype = i32
            L.sbmds_plan_selfcheck.argtypes = [i64, i32, i32, i32, i32]
            L.sbmds_plan_selfcheck.restype = i64
            L.sbmds_plan_selfcheck_rect.argtypes = [i64, i32, i32, i32, i32, i32, i32, i32]
            L.sbmds_plan_selfcheck_rect.restype = i64
            L.sbmds_sparse_split_rows.argtypes = [i64, i64, p, p, i32, p, i64]
            L.sbmds_sparse_split_rows.restype = i64
            L.sbmds_create_shard.argtypes = [i64, i64, i64, i64, i64, p, p, p, p, i32, i32, u32, p,
                                             ctypes.POINTER(p)]
            L.sbmds_create_shard.restype = ctypes.c_int
            L.sbmds_shard_stage.argtypes = [p, i32, i32, p, p, p, p, p]
            L.sbmds_shard_stage.restype = ctypes.c_int
            L.sbmds_shard_exchange_bytes.argtypes = [i64, i32, i32]
            L.sbmds_shard_exchange_bytes.restype = i64
            L.sbmds_shard_attach_nccl.argtypes = [p, p]
            L.sbmds_shard_attach_nccl.restype = ctypes.c_int
            L.sbmds_nccl_unique_id.argtypes = [p]
            L.sbmds_nccl_unique_id.restype = ctypes.c_int
            L.sbmds_shard_plan_selfcheck.argtypes = [i64, i32, i32, i32, i32, i32, i32]
            L.sbmds_shard_plan_selfcheck.restype = i64
            L.sbmds_shard_tiles.argtypes = [i64, i32, i32, i32, p, i64]
            L.sbmds_shard_tiles.restype = i64
            L.sbmds_bmds.argtypes = [p, i32, i32, i32, d, u64, p, p, p, ctypes.POINTER(SbmdsInfo), p]
            L.sbmds_bmds.restype = ctypes.c_int
            L.sbmds_sbha_p.argtypes = [i64, i64, d]
            L.sbmds_sbha_p.restype = i64
            L.sbmds_sbha_build.argtypes = [i64, p, i64, p, i64, p, d, p, p, p, ctypes.POINTER(SbhaInfo), p]
            L.sbmds_sbha_build.restype = ctypes.c_int
            _lib = L
    return _lib


def check(status: int):
    if status != SBMDS_OK:
        raise SbmdsError(status, lib().sbmds_last_error().decode(errors="replace"))
