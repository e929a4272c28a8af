"""Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as 1, 2, 3").

PAPER.md P:195-197 (§3.2 "RNG determinism"): "RNG streams are indexed by the logical
output position (b,i) using a counter-based RNG (e.g. Philox), so each random number
is a deterministic function of a key and a counter."  The paper names Philox but not
the variant; reading R1 fixes Philox4x32 with 10 rounds.  Pinned by the
Random123 known-answer vectors (tests/test_oracle_rng.py).

Vectorised over numpy uint64 arrays holding 32-bit words.  Test infrastructure only.
"""
from __future__ import annotations

import numpy as np

M0 = 0xD2511F53          # multiplier applied to counter word 0
M1 = 0xCD9E8D57          # multiplier applied to counter word 2
W0 = 0x9E3779B9          # Weyl key increment, key word 0 (golden ratio)
W1 = 0xBB67AE85          # Weyl key increment, key word 1 (sqrt(3)-1)
MASK32 = np.uint64(0xFFFFFFFF)
ROUNDS = 10


def philox4x32(c0, c1, c2, c3, k0, k1, rounds: int = ROUNDS):
    """Return the four 32-bit output words for counters (c0..c3) under key (k0, k1).
    Counters and keys may be scalars or arrays (broadcast).

    One round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2 (64-bit products);
    new counter = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); the key is bumped by
    (W0, W1) between rounds.
    """
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & MASK32 for c in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & MASK32
    k1 = np.asarray(k1, dtype=np.uint64) & MASK32
    m0 = np.uint64(M0)
    m1 = np.uint64(M1)
    s32 = np.uint64(32)
    for r in range(rounds):
        if r:
            k0 = (k0 + np.uint64(W0)) & MASK32
            k1 = (k1 + np.uint64(W1)) & MASK32
        p0 = m0 * c0                 # < 2^64: exact in uint64
        p1 = m1 * c2
        hi0, lo0 = p0 >> s32, p0 & MASK32
        hi1, lo1 = p1 >> s32, p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    return c0, c1, c2, c3
