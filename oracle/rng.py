"""Random-number layout and the exact-math Gumbel map (test infrastructure only).

Counter layout -- DESIGN.md reading R1 (the paper fixes only "counter-based RNG (e.g.
Philox)" indexed by the logical output position (b, i)):

    key = (seed mod 2^32, seed >> 32)
    ctr = (v, b >> 2, step mod 2^32, ((step >> 32) mod 2^24) | (tag << 24))
    r   = Philox4x32-10(ctr, key)[b mod 4]

  v    global 0-based vocabulary id (never a tile-, CTA- or shard-local id)
  b    0-based batch row
  tag  0 per-token Gumbel (Alg. 2 line "Draw u_{b,i}")
       1 outer group Gumbel  (Alg. A.2 P:779 / A.4 P:831; ctr word 0 = group / rank k)
       2 merge Bernoulli     (Alg. A.3;  ctr word 0 = group k)
       3 Alg. 1 uniform      (P:71;            ctr word 0 = 0)

Uniform map, App. C:  u = (r + 1) / (2^32 + 1) in (0, 1).
Gumbel,      App. C P:853 / Alg. 2:  g = -log(-log u)  ("exact-math mode").

gumbel64 evaluates g in fp64 without cancellation (reading R2): with
E = -log u,
    r <  2^31:  E = -log((r+1)/(2^32+1))
    r >= 2^31:  E = -log1p(-(2^32 - r)/(2^32+1))      (u = 1 - w, w small)
    g = -log(E)
Both branches equal -log(-log u) in exact arithmetic; the second avoids forming
1 - w.  Pinned against a 50-digit Decimal evaluation (tests/test_oracle_rng.py).
"""
from __future__ import annotations

import numpy as np

from .philox import philox4x32

TAG_TOKEN = 0
TAG_OUTER = 1
TAG_MERGE = 2
TAG_ALG1 = 3

TWO32 = 4294967296.0
DEN = TWO32 + 1.0        # 2^32 + 1 (exact in fp64)


def key_words(seed: int):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32


def counter_words(step, tag: int):
    """(c2, c3) for a scalar or array `step` (uint64 semantics)."""
    step = np.asarray(step).astype(np.uint64)
    c2 = step & np.uint64(0xFFFFFFFF)
    c3 = ((step >> np.uint64(32)) & np.uint64(0x00FFFFFF)) | np.uint64((int(tag) & 0xFF) << 24)
    return c2, c3


def random_bits(seed: int, step: int, b, v, tag: int = TAG_TOKEN) -> np.ndarray:
    """32-bit draw r for logical position (b, v) at `step`; b, v and step broadcast."""
    b = np.asarray(b, dtype=np.uint64)
    v = np.asarray(v, dtype=np.uint64)
    c2, c3 = counter_words(step, tag)
    b, v, c2, c3 = np.broadcast_arrays(b, v, c2, c3)
    k0, k1 = key_words(seed)
    out = philox4x32(v, b >> np.uint64(2), c2, c3, k0, k1)
    lane = (b & np.uint64(3)).astype(np.int64)
    stacked = np.stack(out, axis=0)
    return np.take_along_axis(stacked, lane[None], axis=0)[0]


# Per-request layout (reading R18): batch-position-invariant noise.
#   key = (seed_b mod 2^32, seed_b >> 32)
#   ctr = (v >> 2, 0x80000000, step_b mod 2^32, ((step_b >> 32) mod 2^24) | (tag << 24))
#   r   = Philox4x32-10(ctr, key)[v mod 4]
# Word 1 = 0x80000000 never equals b >> 2 of the shared layout for B < 2^33, so the two layouts
# draw from disjoint counters.
PER_REQUEST_WORD1 = 0x80000000


def random_bits_per_request(seeds, steps, v, tag: int = TAG_TOKEN) -> np.ndarray:
    """r for (request seed_b, step_b, vocabulary id v); seeds/steps/v broadcast (uint64)."""
    seeds = np.asarray(seeds).astype(np.uint64)
    v = np.asarray(v, dtype=np.uint64)
    c2, c3 = counter_words(steps, tag)
    seeds, v, c2, c3 = np.broadcast_arrays(seeds, v, c2, c3)
    k0 = seeds & np.uint64(0xFFFFFFFF)
    k1 = seeds >> np.uint64(32)
    o = philox4x32(v >> np.uint64(2), np.full(v.shape, PER_REQUEST_WORD1, np.uint64), c2, c3, k0, k1)
    lane = (v & np.uint64(3)).astype(np.int64)
    return np.take_along_axis(np.stack(o, axis=0), lane[None], axis=0)[0]


def uniform_open(r) -> np.ndarray:
    """u = (r+1)/(2^32+1) in fp64 (App. C)."""
    return (np.asarray(r, dtype=np.float64) + 1.0) / DEN


def gumbel64(r) -> np.ndarray:
    """g = -log(-log u), u = (r+1)/(2^32+1), evaluated in fp64 without cancellation."""
    r = np.asarray(r, dtype=np.float64)
    lower = r < 2147483648.0
    E = np.empty_like(r)
    E[lower] = -np.log((r[lower] + 1.0) / DEN)
    w = (TWO32 - r[~lower]) / DEN
    E[~lower] = -np.log1p(-w)
    return -np.log(E)


def gumbel_at(seed: int, step: int, b, v) -> np.ndarray:
    """Per-token Gumbel g_{b,v} (Alg. 2) for global vocabulary ids v."""
    return gumbel64(random_bits(seed, step, b, v, TAG_TOKEN))
