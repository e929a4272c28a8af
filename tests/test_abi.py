"""CPU checks of the boundary: the C-ABI library builds/loads and exports every symbol that
include/flashsample.h declares; host-side validation rejects bad arguments without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flashsample.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fs_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_expected_entry_points():
    names = _declared()
    for n in ("fs_sample", "fs_sample_grouped", "fs_sample_shard", "fs_combine_summaries",
              "fs_merge_summaries", "fs_ctx_create"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2603_15854_b200 import _lib
    L = _lib.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert sorted(_lib.EXPORTS) == _declared()


def test_binding_has_no_cpu_fallback():
    # the binding never imports the oracle and routes every call through the C ABI
    pkg = os.path.join(ROOT, "paper_2603_15854_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            s = open(os.path.join(pkg, f)).read()
            assert "oracle" not in s.replace("no CPU", ""), f


def test_host_validation_without_gpu():
    from paper_2603_15854_b200 import _lib
    L = _lib.lib()
    assert L.fs_status_str(1) == b"FS_ERR_INVALID"
    # NULL ctx -> invalid, before any CUDA call
    st = L.fs_sample(None, 0, None, None, None, None, None, 0, 0, 1, 1, 1, None, None, None)
    assert st == _lib.FS_ERR_INVALID
    assert b"ctx" in L.fs_last_error()
    st = L.fs_combine_summaries(None, 1, 1, None, None, None, None)
    assert st == _lib.FS_ERR_INVALID


def test_version_string():
    import paper_2603_15854_b200 as fs
    assert "sm_100a" in fs.version()


def test_tp_entry_points_host_side():
    """§8(b) TP boundary without a GPU: NCCL is resolved at run time (a fresh unique id comes back),
    NULL arguments are rejected, and fs_sample_tp refuses a context without a communicator."""
    from paper_2603_15854_b200 import _lib
    L = _lib.lib()
    assert L.fs_status_str(_lib.FS_ERR_NCCL) == b"FS_ERR_NCCL"
    assert L.fs_comm_init(None, None, 1, 0) == _lib.FS_ERR_INVALID
    assert L.fs_comm_unique_id(None) == _lib.FS_ERR_INVALID
    a, b = ctypes.create_string_buffer(128), ctypes.create_string_buffer(128)
    assert L.fs_comm_unique_id(a) == _lib.FS_OK, L.fs_last_error()
    assert L.fs_comm_unique_id(b) == _lib.FS_OK
    assert a.raw != b"\0" * 128 and a.raw != b.raw
    st = L.fs_sample_tp(None, 0, None, None, None, None, None, 0, 0, 1, 1, 1, 0, 1, None, None, None, None, None)
    assert st == _lib.FS_ERR_INVALID
