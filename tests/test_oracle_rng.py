"""Pins of oracle.philox / oracle.rng against things other than the oracle itself.

* Philox4x32-10: the three Random123 known-answer vectors (kat_vectors file of the
  Random123 distribution, Salmon et al. SC'11), tests/golden/philox_kat.txt.
* Gumbel map (App. C): a 50-digit Decimal evaluation of
  -ln(-ln((r+1)/(2^32+1))), closed-form special values, monotonicity in r and
  finiteness over both 2^20-wide tails, and the Gumbel(0,1) moments (mean = Euler
  gamma, variance = pi^2/6).
"""
import math
import os
from decimal import Decimal, getcontext

import numpy as np
import pytest

from oracle import philox, rng

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    rows = []
    with open(os.path.join(GOLDEN, "philox_kat.txt")) as f:
        for line in f:
            line = line.split("#")[0].split()
            if line:
                rows.append([int(x, 16) for x in line])
    return rows


def test_philox_known_answer_vectors():
    kat = _kat()
    assert len(kat) == 3
    for c0, c1, c2, c3, k0, k1, o0, o1, o2, o3 in kat:
        out = philox.philox4x32(c0, c1, c2, c3, k0, k1)
        assert [int(x) for x in out] == [o0, o1, o2, o3]


def _g_decimal(r: int) -> Decimal:
    getcontext().prec = 50
    u = (Decimal(r) + 1) / (Decimal(2) ** 32 + 1)
    return -((-(u.ln())).ln())


def test_gumbel64_matches_50_digit_decimal():
    rs = [0, 1, 2, 3, 1000, 2**20, 2**31 - 2, 2**31 - 1, 2**31, 2**31 + 1, 3 * 2**30,
          2**32 - 2**20, 2**32 - 3, 2**32 - 2, 2**32 - 1]
    rs += [int(x) for x in np.random.default_rng(7).integers(0, 2**32, 300)]
    got = rng.gumbel64(np.array(rs, dtype=np.uint64))
    for r, g in zip(rs, got):
        ref = float(_g_decimal(r))
        assert abs(g - ref) <= 2e-14 * max(1.0, abs(ref)), (r, g, ref)


def test_gumbel_special_values():
    # r = 0: u = 1/(2^32+1) -> g = -ln(ln(2^32+1));  r = 2^32-1: u = 2^32/(2^32+1)
    g = rng.gumbel64(np.array([0, 2**32 - 1], dtype=np.uint64))
    assert g[0] == pytest.approx(-math.log(math.log(2.0**32 + 1)), abs=1e-12)
    assert g[0] == pytest.approx(-3.0992229822, abs=1e-9)
    assert g[1] == pytest.approx(22.1807097780, abs=1e-9)
    # continuous identities: u=e^-1 -> 0, u=e^-e -> -1, u=e^(-1/e) -> 1.
    # Take the r whose u is nearest; |dg/du| = 1/(u E) bounds the discretisation error.
    for target_u, target_g in [(math.exp(-1), 0.0), (math.exp(-math.e), -1.0),
                               (math.exp(-1 / math.e), 1.0)]:
        r = round(target_u * (2.0**32 + 1) - 1)
        u = (r + 1) / (2.0**32 + 1)
        slope = 1.0 / (u * -math.log(u))
        assert abs(rng.gumbel64(np.array([r], np.uint64))[0] - target_g) <= slope * 2.4e-10 + 1e-12


def test_gumbel_tails_finite_and_monotone():
    lo = np.arange(0, 2**20, dtype=np.uint64)
    hi = np.arange(2**32 - 2**20, 2**32, dtype=np.uint64)
    mid = np.arange(2**31 - 2**16, 2**31 + 2**16, dtype=np.uint64)
    for r in (lo, mid, hi):
        g = rng.gumbel64(r)
        assert np.all(np.isfinite(g))
        assert np.all(np.diff(g) > 0)          # g is strictly increasing in u
    assert rng.gumbel64(hi)[-1] < 22.19 and rng.gumbel64(lo)[0] > -3.11


def test_gumbel_moments_1e6():
    v = np.arange(1_000_000, dtype=np.uint64)
    g = rng.gumbel_at(seed=12345, step=0, b=0, v=v)
    assert abs(g.mean() - 0.5772156649) < 0.01
    assert abs(g.var() - math.pi**2 / 6) < 0.02


def test_counter_layout_is_the_documented_one():
    seed, step = 0x0123456789ABCDEF, (5 << 32) | 77
    for b in range(9):
        for v in (0, 1, 31, 128255, 262207):
            r = int(rng.random_bits(seed, step, b, v))
            out = philox.philox4x32(v, b >> 2, step & 0xFFFFFFFF, (step >> 32) & 0xFFFFFF,
                                    seed & 0xFFFFFFFF, seed >> 32)
            assert r == int(out[b & 3])
    # tags separate streams; steps give different noise
    a = rng.random_bits(1, 0, 0, np.arange(1000), rng.TAG_TOKEN)
    assert not np.any(a == rng.random_bits(1, 0, 0, np.arange(1000), rng.TAG_OUTER))
    assert not np.all(a == rng.random_bits(1, 1, 0, np.arange(1000)))


def test_uniform_bits_chi_square():
    r = rng.random_bits(99, 3, np.arange(64)[:, None], np.arange(8192)[None, :])
    counts = np.bincount((r >> np.uint64(24)).ravel().astype(np.int64), minlength=256)
    from oracle.stats import chi_square
    _, p = chi_square(counts, np.full(256, 1 / 256))
    assert p > 1e-4
