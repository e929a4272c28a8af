"""Pins of oracle/csrc/flat_counts.c (the C restatement of the oracle's flat sampler) and the
north-star 1e6-draw chi-square pins of the flat definition.

The C helper exists only so that 1e6 draws finish in seconds; it is pinned here against things
other than itself:
  * Philox4x32-10: the Random123 known-answer vectors (tests/golden/philox_kat.txt);
  * the Gumbel map: the numpy oracle's gumbel64, which test_oracle_rng.py pins to a 50-digit
    Decimal evaluation of App. C;
  * the sampled index: draw-by-draw equality with oracle.sampler.flat_sample (numpy) on the tiny
    config and on masked rows.
Then the exactness-in-distribution pins (Gumbel-Max theorem; §5.7 P:648-650 with the
north star's 1e6 draws at p > 0.001, reading R16, one retry with a fresh seed): the SPEC
fixtures V in {2, 8, 128} and every row of BASELINE.json's tiny config (B=4, D=64, V=1000, fp32).
"""
import os

import numpy as np
import pytest
import torch

import synth
from oracle import cflat, rng, sampler, stats

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
N_DRAWS = 1_000_000


def _kat():
    rows = []
    with open(os.path.join(GOLDEN, "philox_kat.txt")) as f:
        for line in f:
            line = line.split("#")[0].split()
            if line:
                rows.append([int(x, 16) for x in line])
    return rows


def test_c_philox_known_answer_vectors():
    for c0, c1, c2, c3, k0, k1, o0, o1, o2, o3 in _kat():
        assert cflat.philox([c0, c1, c2, c3], [k0, k1]).tolist() == [o0, o1, o2, o3]


def test_c_gumbel_matches_pinned_numpy_gumbel64():
    r = np.concatenate([np.array([0, 1, 2, 2**31 - 1, 2**31, 2**31 + 1, 2**32 - 2, 2**32 - 1], np.uint64),
                        np.random.default_rng(3).integers(0, 2**32, 200_000, dtype=np.uint64)])
    want = rng.gumbel64(r)
    got = cflat.gumbel64(r.astype(np.uint32))
    assert np.max(np.abs(got - want)) <= 1e-13


def _tiny():
    wl = synth.make_workload("tiny", 4)
    h, W = synth.as_numpy_exact(wl.h), synth.as_numpy_exact(wl.W)
    return wl, h, W


def test_c_flat_sample_equals_numpy_oracle_draw_by_draw():
    wl, h, W = _tiny()
    for step in range(0, 400, 7):
        sc = sampler.scores(h, W, seed=wl.seed, step=step)
        flat = sampler.flat_sample(sc, want_near=False)
        for b in range(4):
            assert cflat.flat_sample(sc.ltilde[b], wl.seed, step, b) == flat.idx[b], (step, b)
    # masked rows (mask bit 0 -> -inf) and a fully masked row (-> -1)
    allowed = np.random.default_rng(5).random((4, 1000)) < 0.3
    allowed[3, :] = False
    words = synth.as_numpy_exact(synth.pack_allowed_bits(torch.from_numpy(allowed)))
    for step in (0, 1, 99):
        sc = sampler.scores(h, W, seed=11, step=step, mask=words)
        flat = sampler.flat_sample(sc, want_near=False)
        for b in range(4):
            assert cflat.flat_sample(sc.ltilde[b], 11, step, b) == flat.idx[b], (step, b)


def _chi_square_1e6(lt, b=0, seeds=(20260101, 20260202), banned=None):
    for seed in seeds:                      # one retry with a fresh seed
        counts = cflat.flat_counts(lt, seed, 0, N_DRAWS, b)
        assert counts.sum() == N_DRAWS
        if banned is not None:
            assert counts[banned].sum() == 0          # banned tokens never appear (hard fail)
        _, p = stats.chi_square(counts, stats.softmax_probs(lt))
        if p > 1e-3:
            break
    return p


FIXTURES = {
    "uniform": lambda V: np.zeros(V),
    "ramp": lambda V: np.linspace(0, 3, V),
    "one_dominant": lambda V: np.where(np.arange(V) == V // 2, 4.0, 0.0),
    "half_masked": lambda V: np.where(np.arange(V) % 2 == 0, np.linspace(-1, 1, V), -np.inf),
}


@pytest.mark.parametrize("V", [2, 8, 128])
@pytest.mark.parametrize("pattern", list(FIXTURES))
def test_flat_chi_square_1e6(V, pattern):
    lt = FIXTURES[pattern](V).astype(np.float64)
    banned = np.nonzero(~np.isfinite(lt))[0] if pattern == "half_masked" else None
    assert _chi_square_1e6(lt, banned=banned) > 1e-3


def test_tiny_config_chi_square_1e6_every_row():
    """BASELINE.json configs[0]: B=4, D=64, V=1000 fp32; 1e6 draws (decode steps 0..1e6-1) per row."""
    wl, h, W = _tiny()
    sc = sampler.scores(h, W, seed=wl.seed, step=0)
    for b in range(4):
        assert _chi_square_1e6(sc.ltilde[b], b=b) > 1e-3, b


def test_chi_square_1e6_detects_a_wrong_distribution():
    """Negative control at the same scale: draws of l~ tested against softmax(0.97 l~) must fail."""
    lt = np.linspace(0, 3, 128)
    counts = cflat.flat_counts(lt, 5, 0, N_DRAWS, 0)
    _, p = stats.chi_square(counts, stats.softmax_probs(0.97 * lt))
    assert p < 1e-6
