"""The mathematical claim behind the epilogue's exact Gumbel pruning (csrc/fs_epilogue.cuh
`gumbel_upper`): for the Gumbel map of App. C,
    g(r) = -ln(-ln u),  u = (r + 1) / (2^32 + 1),
and k = the number of leading one bits of the 32-bit word r,
    g(r) < (k + 1) ln 2 + 2^-32
(-ln u >= 1 - u, and 1 - u = (2^32 - r)/(2^32 + 1) > 2^-(k+1) * 2^32/(2^32 + 1)).
Checked here on the oracle's fp64 G64 (pinned to 50-digit Decimal values in test_oracle_rng.py)
at the worst case of every k -- g is increasing in r, so the largest r with exactly k leading ones
maximises g over that class -- and on 2^20 random words, with the 1e-3 margin the kernel adds
left over.  It also shows the bound is tight (within ln 2 of g at the class maximum), which is
what makes the pruning effective."""
import math

import numpy as np

from oracle import rng

LN2 = math.log(2.0)


def _leading_ones(r):
    r = np.asarray(r, dtype=np.uint64)
    k = np.zeros(r.shape, dtype=np.int64)
    for bit in range(31, -1, -1):
        done = ((r >> np.uint64(bit)) & np.uint64(1)) == 0
        k = np.where((k == 31 - bit) & ~done, k + 1, k)
    return k


def test_leading_ones_counter():
    assert list(_leading_ones([0, 0x80000000, 0xC0000000, 0xFFFFFFFE, 0xFFFFFFFF, 0x7FFFFFFF])) == [0, 1, 2, 31, 32, 0]


def test_bound_at_every_class_maximum():
    for k in range(33):
        r = 2**32 - 1 if k == 32 else (2**32 - 2**(32 - k)) + (2**(31 - k) - 1)
        assert _leading_ones([r])[0] == k
        g = float(rng.gumbel64(np.array([r], dtype=np.uint64))[0])
        bound = (k + 1) * LN2
        assert g < bound + 2.0**-32, (k, g, bound)
        assert bound - g < LN2 + 0.5, (k, g, bound)      # tight: within ln 2 (+ the E ~ w slack at small k)


def test_bound_on_random_words_with_margin():
    r = np.random.default_rng(20260317).integers(0, 2**32, size=1 << 20, dtype=np.uint64)
    g = rng.gumbel64(r)
    ub = (_leading_ones(r) + 1) * LN2
    assert np.all(g < ub)
    # the kernel compares l~ + ub + 1e-3 (+ 1e-6 |l~|) with a recorded fp32 score; G32 is within
    # 2.2e-6 of G64 (tests/test_gpu_rng.py), so the margin covers every rounding in that comparison
    assert np.min(ub - g) > -1e-3 + 2.2e-6
