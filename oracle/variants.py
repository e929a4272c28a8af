"""In-distribution sampling algorithms of the paper (test infrastructure only).

These are exact *in distribution* (Theorem P:103-110, Lemmas, Theorem
P:351-359) but not pathwise equal to the flat argmax, because they draw fresh outer
randomness.  The GPU build realises the grouped / online / TP variants by reusing the
group maxima (reading R8), which is pathwise equal to the flat
definition in sampler.py; the forms below are validated by chi-square only.

Each function works on one row of transformed logits l~ (fp64, -inf allowed) with
global ids v = 0..V-1 and draws its randomness from rng.random_bits with the tags
of DESIGN.md reading R1.
"""
from __future__ import annotations

import math
import numpy as np

from . import rng
from .sampler import logsumexp


def alg1_materialized(lt, seed, step, b) -> int:
    """Alg. 1: m = max, Z = sum exp(l~-m), p = exp(l~-m)/Z, c = prefix sum,
    u ~ U(0,1), return min{i : c_i >= u}."""
    lt = np.asarray(lt, np.float64)
    m = lt.max()                                    # line 3
    if not np.isfinite(m):
        return -1
    Z = np.sum(np.exp(lt - m))                      # line 4
    p = np.exp(lt - m) / Z                          # line 5
    c = np.cumsum(p)                                # line 6
    u = float(rng.uniform_open(rng.random_bits(seed, step, b, 0, rng.TAG_ALG1)))   # line 7
    hits = np.nonzero(c >= u)[0]                    # line 8
    if hits.size == 0:                              # rounding: c_V may be 1 - eps < u
        return int(np.nonzero(p > 0)[0][-1])
    return int(hits[0])


def alg_a1_streaming(lt, seed, step, b) -> int:
    """Alg. A.1: one pass keeping (m, i*); replace only on s > m."""
    m, istar = -math.inf, -1
    g = rng.gumbel_at(seed, step, b, np.arange(len(lt)))
    for i, li in enumerate(lt):                     # line 4
        s = li + g[i]                               # lines 5-6
        if s > m:                                   # line 7
            m, istar = s, i                         # line 8
    return istar


def _within_group(lt, g_tok, a, b_):
    """z_k = argmax_{j in G_k} (y_{k,j} + g_{k,j}) with the per-token Gumbels."""
    blk = lt[a:b_] + g_tok[a:b_]
    j = int(np.argmax(blk))
    return a + j, float(blk[j])


def alg_a2_parallel_fresh(lt, group_size, seed, step, b):
    """Alg. A.2: per group local sample z_k and L_k; outer
    k* = argmax_k (L_k + g_bar_k) with FRESH outer Gumbels (tag 1); z = global id."""
    lt = np.asarray(lt, np.float64)
    V = len(lt)
    g_tok = rng.gumbel_at(seed, step, b, np.arange(V))
    K = (V + group_size - 1) // group_size
    best, z = -math.inf, -1
    for k in range(K):
        a, e = k * group_size, min(V, (k + 1) * group_size)
        Lk = float(logsumexp(lt[a:e]))              # line 6
        if Lk == -math.inf:                         # zero-mass group: skipped
            continue
        zk, _ = _within_group(lt, g_tok, a, e)      # line 5
        gbar = float(rng.gumbel64(rng.random_bits(seed, step, b, k, rng.TAG_OUTER)))
        if Lk + gbar > best:                        # line 8
            best, z = Lk + gbar, zk                 # line 9 (global id directly)
    return z, float(logsumexp(np.array([logsumexp(lt)])))


def alg_a3_online_bernoulli(lt, group_size, seed, step, b):
    """Alg. A.3: stream groups keeping (l, z); replace z by z_k with
    probability exp(L_k - l_new) using a fresh uniform (tag 2)."""
    lt = np.asarray(lt, np.float64)
    V = len(lt)
    g_tok = rng.gumbel_at(seed, step, b, np.arange(V))
    K = (V + group_size - 1) // group_size
    ell, z = -math.inf, -1
    for k in range(K):
        a, e = k * group_size, min(V, (k + 1) * group_size)
        Lk = float(logsumexp(lt[a:e]))              # line 11
        if Lk == -math.inf:
            continue
        if ell == -math.inf:                        # first nonzero-mass group (lines 2-5)
            ell, z = Lk, _within_group(lt, g_tok, a, e)[0]
            continue
        l_new = float(logsumexp(np.array([ell, Lk])))     # line 12
        p_replace = math.exp(Lk - l_new)                  # line 13
        u = float(rng.uniform_open(rng.random_bits(seed, step, b, k, rng.TAG_MERGE)))  # line 14
        if u < p_replace:                                 # line 15
            z = _within_group(lt, g_tok, a, e)[0]         # lines 16-17
        ell = l_new                                       # line 19
    return z, ell


def alg_a4_distributed_fresh(lt, n, seed, step, b):
    """Alg. A.4: shards [kV/n, (k+1)V/n) as groups, fresh outer Gumbels."""
    lt = np.asarray(lt, np.float64)
    V = len(lt)
    g_tok = rng.gumbel_at(seed, step, b, np.arange(V))
    best, z, Ls = -math.inf, -1, []
    for k in range(n):
        a, e = k * V // n, (k + 1) * V // n
        Lk = float(logsumexp(lt[a:e]))              # line 3 (local log-mass)
        Ls.append(Lk)
        if Lk == -math.inf:
            continue
        zk, _ = _within_group(lt, g_tok, a, e)      # line 3 (local sample)
        gbar = float(rng.gumbel64(rng.random_bits(seed, step, b, k, rng.TAG_OUTER)))
        if Lk + gbar > best:                        # line 5
            best, z = Lk + gbar, zk                 # line 6
    return z, float(logsumexp(np.array(Ls)))
