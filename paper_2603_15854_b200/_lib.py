"""ctypes loader for libflashsample.so (the C ABI in include/flashsample.h).

Argument marshalling only.  The library is loaded from this package directory; if it is
missing the import fails loudly -- there is no CPU or PyTorch fallback for any step.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FS_LIB_PATH") or os.path.join(HERE, "libflashsample.so")   # override: A/B experiments

# Every symbol include/flashsample.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "fs_version", "fs_status_str", "fs_last_error", "fs_ctx_create", "fs_ctx_destroy",
    "fs_ctx_set_option", "fs_ctx_query", "fs_sample", "fs_sample_ex", "fs_sample_grouped", "fs_sample_logits",
    "fs_sample_logits_ex", "fs_sample_shard",
    "fs_combine_summaries", "fs_merge_summaries", "fs_random_bits", "fs_gumbel_from_bits",
    "fs_comm_window_create", "fs_comm_window_open", "fs_sample_tp_push", "fs_comm_window_destroy",
    "fs_copy_async", "fs_sample_staged", "fs_read_probe", "fs_comm_unique_id", "fs_comm_init", "fs_sample_tp", "fs_comm_destroy",
]

FS_OK, FS_ERR_INVALID, FS_ERR_UNSUPPORTED, FS_ERR_CUDA, FS_ERR_OOM, FS_ERR_NCCL = range(6)


class SampleArgs(ctypes.Structure):
    """fs_sample_args (include/flashsample.h)."""
    _fields_ = [("bias", ctypes.c_void_p), ("temperature", ctypes.c_void_p), ("mask", ctypes.c_void_p),
                ("seed", ctypes.c_uint64), ("step", ctypes.c_uint64), ("seeds", ctypes.c_void_p),
                ("steps", ctypes.c_void_p), ("group_size", ctypes.c_int), ("idx_out", ctypes.c_void_p),
                ("score_out", ctypes.c_void_p), ("logZ_out", ctypes.c_void_p), ("logprob_out", ctypes.c_void_p),
                ("groups_out", ctypes.c_void_p), ("top_k", ctypes.c_int), ("top_p", ctypes.c_float)]
FS_BF16, FS_F32 = 0, 1


class IpcHandle(ctypes.Structure):
    """fs_ipc_handle: 64 opaque bytes (a cudaIpcMemHandle_t)."""
    _fields_ = [("bytes", ctypes.c_ubyte * 64)]


class FlashSampleError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: status {status}: {msg}")
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -m paper_2603_15854_b200.build` "
            "(or __graft_entry__.build()); there is no fallback implementation")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u32, u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
    L.fs_version.restype = ctypes.c_char_p
    L.fs_status_str.restype = ctypes.c_char_p
    L.fs_status_str.argtypes = [i32]
    L.fs_last_error.restype = ctypes.c_char_p
    L.fs_ctx_create.argtypes = [i32, ctypes.POINTER(vp)]
    L.fs_ctx_destroy.argtypes = [vp]
    L.fs_ctx_destroy.restype = None
    L.fs_ctx_set_option.argtypes = [vp, ctypes.c_char_p, i64]
    L.fs_ctx_query.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_double)]
    L.fs_sample.argtypes = [vp, i32, vp, vp, vp, vp, vp, u64, u64, i32, i32, i32, vp, vp, vp]
    L.fs_sample_grouped.argtypes = [vp, i32, vp, vp, vp, vp, vp, u64, u64, i32, i32, i32, i32,
                                    vp, vp, vp, vp, vp, vp]
    L.fs_sample_logits.argtypes = [vp, i32, vp, i64, vp, vp, vp, u64, u64, i32, i32, vp, vp, vp, vp, vp]
    L.fs_sample_ex.argtypes = [vp, i32, vp, vp, i32, i32, i32, ctypes.POINTER(SampleArgs), vp]
    L.fs_sample_logits_ex.argtypes = [vp, i32, vp, i64, i32, i32, ctypes.POINTER(SampleArgs), vp]
    L.fs_sample_shard.argtypes = [vp, i32, vp, vp, vp, vp, vp, u64, u64, i32, i32, i32, i64, i64, vp, vp]
    L.fs_combine_summaries.argtypes = [vp, i32, i32, vp, vp, vp, vp]
    L.fs_merge_summaries.argtypes = [vp, vp, vp, i32, vp]
    L.fs_random_bits.argtypes = [u64, u64, u32, vp, vp, vp, i64, vp]
    L.fs_gumbel_from_bits.argtypes = [vp, vp, i64, vp]
    L.fs_read_probe.argtypes = [vp, ctypes.c_size_t, vp, i32, vp]
    L.fs_copy_async.argtypes = [vp, vp, vp, ctypes.c_size_t, vp]
    L.fs_sample_staged.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, u64, u64, i32, i32, i32, vp, vp, vp]
    L.fs_comm_window_create.argtypes = [vp, i32, i32, i32, ctypes.POINTER(IpcHandle)]
    L.fs_comm_window_open.argtypes = [vp, ctypes.POINTER(IpcHandle)]
    L.fs_comm_window_destroy.argtypes = [vp]
    L.fs_sample_tp_push.argtypes = [vp, i32, vp, vp, vp, vp, vp, u64, u64, i32, i32, i32, i64, i64, vp, vp, vp, vp]
    L.fs_comm_unique_id.argtypes = [vp]
    L.fs_comm_init.argtypes = [vp, vp, i32, i32]
    L.fs_comm_destroy.argtypes = [vp]
    L.fs_sample_tp.argtypes = [vp, i32, vp, vp, vp, vp, vp, u64, u64, i32, i32, i32, i64, i64, vp, vp, vp, vp, vp]
    for name in EXPORTS:
        if name not in ("fs_version", "fs_status_str", "fs_last_error", "fs_ctx_destroy"):
            getattr(L, name).restype = i32
    _lib = L
    return L


def check(status: int, where: str) -> None:
    if status != FS_OK:
        msg = lib().fs_last_error().decode(errors="replace")
        raise FlashSampleError(status, where, msg)
