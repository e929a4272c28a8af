"""Pins of oracle.variants (in-distribution algorithms) and of the grouped-summary laws.

* chi-square vs softmax(l~) (Theorem P:103-110; Lemmas; Theorem P:351-359)
  for Alg. 1, A.1, A.2 (fresh outer Gumbel), A.3 (Bernoulli merge), A.4 (fresh outer);
* SPEC S:297 worked example: l~ = [ln1, ln2, ln3, ln4], g = 2 -> probabilities
  [0.1, 0.2, 0.3, 0.4] (group masses ln3, ln7 -> 0.3 / 0.7);
* max-stability (Lemma P:254-270): M_k ~ Gumbel(L_k, 1): mean L_k + gamma, variance pi^2/6.
"""
import math

import numpy as np
import pytest

from oracle import sampler, stats, variants

LT8 = np.array([0.5, -1.0, 2.0, -np.inf, 0.0, 1.5, -0.5, 1.0])     # one banned token


def _freq(fn, n, V, **kw):
    counts = np.zeros(V, np.int64)
    for t in range(n):
        z = fn(step=t, **kw)
        z = z[0] if isinstance(z, tuple) else z
        counts[z] += 1
    return counts


@pytest.mark.parametrize("name", ["alg1", "a1", "a2", "a3", "a4"])
def test_variant_chi_square(name):
    n = 6000
    fns = {
        "alg1": lambda step: variants.alg1_materialized(LT8, 31, step, 0),
        "a1": lambda step: variants.alg_a1_streaming(LT8, 31, step, 0),
        "a2": lambda step: variants.alg_a2_parallel_fresh(LT8, 3, 31, step, 0),
        "a3": lambda step: variants.alg_a3_online_bernoulli(LT8, 3, 31, step, 0),
        "a4": lambda step: variants.alg_a4_distributed_fresh(LT8, 4, 31, step, 0),
    }
    counts = _freq(fns[name], n, 8)
    assert counts[3] == 0
    _, p = stats.chi_square(counts, stats.softmax_probs(LT8))
    assert p > 1e-3, (name, counts)


def test_variant_log_normalizer():
    ref = sampler.logsumexp(LT8)
    assert variants.alg_a3_online_bernoulli(LT8, 3, 1, 0, 0)[1] == pytest.approx(ref, abs=1e-12)
    assert variants.alg_a4_distributed_fresh(LT8, 4, 1, 0, 0)[1] == pytest.approx(ref, abs=1e-12)


def test_spec_group_example_probabilities():
    lt = np.log(np.array([1.0, 2.0, 3.0, 4.0]))
    np.testing.assert_allclose(stats.softmax_probs(lt), [0.1, 0.2, 0.3, 0.4], rtol=1e-12)
    h = np.tile(lt.astype(np.float32), (1, 1))
    sc = sampler.scores(h, np.eye(4, dtype=np.float32), seed=0, step=0)
    gr = sampler.group_summaries(sc, 2)
    L = gr.L[0]
    np.testing.assert_allclose(np.exp(L) / np.exp(L).sum(), [0.3, 0.7], rtol=1e-6)
    counts = _freq(lambda step: variants.alg_a3_online_bernoulli(lt, 2, 77, step, 0), 8000, 4)
    _, p = stats.chi_square(counts, [0.1, 0.2, 0.3, 0.4])
    assert p > 1e-3


def test_max_stability_moments():
    # Lemma P:254-270: M_k = max_{G_k} (l~ + g) ~ Gumbel(L_k, 1)
    rs = np.random.default_rng(0)
    lt = rs.standard_normal(64).astype(np.float32)
    n = 20000
    h = np.tile(lt, (n, 1))
    sc = sampler.scores(h, np.eye(64, dtype=np.float32), seed=4242, step=3)
    gr = sampler.group_summaries(sc, 16)
    for k in range(4):
        Mk = gr.M[:, k]
        Lk = gr.L[0, k]
        assert abs(Mk.mean() - (Lk + stats.EULER_GAMMA)) < 4 * math.sqrt(stats.GUMBEL_VAR / n)
        assert abs(Mk.var() - stats.GUMBEL_VAR) < 0.08
    # independence across groups (Lemma item 2): near-zero correlation
    c = np.corrcoef(gr.M[:, 0], gr.M[:, 1])[0, 1]
    assert abs(c) < 0.03
