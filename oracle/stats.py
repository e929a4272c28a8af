"""Statistical checks (test infrastructure only).

PAPER.md §5.7: kernel correctness is a chi-squared goodness-of-fit test of
sampled frequencies against the reference distribution ("no statistically significant
difference").  The paper gives 5,000 samples and no alpha; the north star fixes 1e6
draws at p > 0.001 (reading R16).  Bins with expected count < 5 are merged
(standard Pearson practice).
"""
from __future__ import annotations

import math
import numpy as np
from scipy import stats as _st

EULER_GAMMA = 0.57721566490153286061
GUMBEL_VAR = math.pi ** 2 / 6.0


def softmax_probs(lt) -> np.ndarray:
    """p(i) = exp(l~_i) / sum_j exp(l~_j)."""
    lt = np.asarray(lt, np.float64)
    m = lt.max()
    e = np.exp(lt - m)
    return e / e.sum()


def chi_square(counts, probs, min_expected: float = 5.0):
    """Pearson statistic and p-value of observed `counts` against `probs`.
    Categories with p = 0 must have zero counts (returns p-value 0 otherwise)."""
    counts = np.asarray(counts, np.float64)
    probs = np.asarray(probs, np.float64)
    n = counts.sum()
    if np.any(counts[probs == 0] > 0):
        return math.inf, 0.0
    keep = probs > 0
    counts, probs = counts[keep], probs[keep]
    exp = probs * n
    order = np.argsort(exp)
    # merge the smallest-expectation bins until every merged bin has >= min_expected
    obs_b, exp_b = [], []
    acc_o = acc_e = 0.0
    for i in order:
        acc_o += counts[i]
        acc_e += exp[i]
        if acc_e >= min_expected:
            obs_b.append(acc_o); exp_b.append(acc_e)
            acc_o = acc_e = 0.0
    if acc_e > 0:
        if exp_b:
            obs_b[-1] += acc_o; exp_b[-1] += acc_e
        else:
            obs_b.append(acc_o); exp_b.append(acc_e)
    obs_b, exp_b = np.array(obs_b), np.array(exp_b)
    stat = float(np.sum((obs_b - exp_b) ** 2 / exp_b))
    dof = max(1, len(obs_b) - 1)
    return stat, float(_st.chi2.sf(stat, dof))
