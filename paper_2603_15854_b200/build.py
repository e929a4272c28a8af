"""Build libflashsample.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2603_15854_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libflashsample.so")
SOURCES = ["fs_api.cu", "fs_fused_tc.cu", "fs_fused_tc2.cu", "fs_fused_simt.cu", "fs_reduce.cu", "fs_logits.cu", "fs_topk.cu",
           "fs_probe.cu"]
HEADERS = ["fs_device.cuh", "fs_sm100.cuh", "fs_epilogue.cuh", "fs_kernels.h", "fs_peer.cuh", "fs_nccl.h",
           "fs_topk_epi.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_flags() -> list:
    """nccl.h of the pip NCCL torch loads (types only) and that library's path as the run-time
    default (csrc/fs_nccl.h resolves NCCL with dlopen; nothing is linked)."""
    try:
        import nvidia.nccl
        d = list(nvidia.nccl.__path__)[0]
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            flags = ["-I", os.path.join(d, "include")]
            lib = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(lib):
                flags.append(f'-DFS_NCCL_DEFAULT_PATH="{lib}"')
            return flags
    except Exception:
        pass
    return ["-I", "/usr/include"]


FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), *_nccl_flags()]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "flashsample.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    hdr_t = max(os.path.getmtime(d) for d in [os.path.join(CSRC, f) for f in HEADERS] +
                [os.path.join(ROOT, "include", "flashsample.h"), os.path.abspath(__file__)])
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(obj)
        if (not force and os.path.exists(obj) and
                os.path.getmtime(obj) > max(hdr_t, os.path.getmtime(os.path.join(CSRC, src)))):
            continue                                   # object newer than its source and every header
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        log = open(obj + ".log", "w")
        procs.append((subprocess.Popen(cmd, stdout=log, stderr=subprocess.STDOUT), cmd, obj + ".log"))
    for p, cmd, logf in procs:
        if p.wait() != 0:
            sys.stderr.write(open(logf).read())
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        if verbose:
            sys.stdout.write(open(logf).read())
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
