"""ctypes loader of oracle/csrc/flat_counts.c (TEST INFRASTRUCTURE ONLY).

The C file restates the oracle's flat sampler for one row (Philox4x32-10, App. C Gumbel map,
argmax with the smallest-id tie rule) so that the 1e6-draw chi-square pins of the north star
(reading R16) finish in seconds.  It is built with gcc by build() (and on first use),
pinned in tests/test_oracle_flat_c.py, and never used by the product path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "flat_counts.c")
LIB = os.path.join(HERE, "csrc", "liboracle_flat.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", SRC, "-o", tmp, "-lm"])
        os.replace(tmp, LIB)
    return LIB


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        p = ctypes.c_void_p
        L.oracle_philox.argtypes = [p, p, p]
        L.oracle_gumbel64.argtypes = [ctypes.c_uint32]
        L.oracle_gumbel64.restype = ctypes.c_double
        L.oracle_gumbel64_array.argtypes = [p, p, ctypes.c_int64]
        L.oracle_flat_sample.argtypes = [p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32]
        L.oracle_flat_sample.restype = ctypes.c_int64
        L.oracle_flat_counts.argtypes = [p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                         ctypes.c_uint32, p]
        _lib = L
    return _lib


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().oracle_philox(c.ctypes.data, k.ctypes.data, o.ctypes.data)
    return o


def gumbel64(r) -> np.ndarray:
    r = np.ascontiguousarray(r, np.uint32)
    g = np.empty(r.shape, np.float64)
    lib().oracle_gumbel64_array(r.ctypes.data, g.ctypes.data, r.size)
    return g


def flat_sample(lt_row, seed: int, step: int, b: int) -> int:
    lt = np.ascontiguousarray(lt_row, np.float64)
    return int(lib().oracle_flat_sample(lt.ctypes.data, lt.size, seed & (2**64 - 1), step & (2**64 - 1), b))


def flat_counts(lt_row, seed: int, step0: int, n: int, b: int = 0) -> np.ndarray:
    """Counts over v of the flat sample of row b at steps step0 .. step0+n-1 (undefined draws
    are dropped; they are impossible unless every l~ is -inf)."""
    lt = np.ascontiguousarray(lt_row, np.float64)
    counts = np.zeros(lt.size + 1, np.int64)
    lib().oracle_flat_counts(lt.ctypes.data, lt.size, seed & (2**64 - 1), step0 & (2**64 - 1), int(n), int(b),
                             counts.ctypes.data)
    return counts[:-1]
