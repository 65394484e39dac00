"""Statistical helpers for the pins (test-only; no method arithmetic here).

Pearson chi-square with small-cell merging (SPEC S:476-484 idea): cells with
expected count < 5 are merged with their neighbours.  All tests use fixed
seeds, so every p-value below is deterministic; thresholds are 1e-3 (the
north star's "p > 1e-3").
"""
from __future__ import annotations

from fractions import Fraction
from math import comb

import numpy as np
from scipy import stats

ALPHA = 1e-3


def chisq_pvalue(observed, expected_prob, min_expected=5.0):
    obs = np.asarray(observed, dtype=np.float64)
    p = np.asarray(expected_prob, dtype=np.float64)
    total = obs.sum()
    exp = p * total
    # merge adjacent cells until each has expected >= min_expected
    mo, me = [], []
    co = ce = 0.0
    for o, e in zip(obs, exp):
        co += o
        ce += e
        if ce >= min_expected:
            mo.append(co)
            me.append(ce)
            co = ce = 0.0
    if ce > 0 or co > 0:
        if me:
            mo[-1] += co
            me[-1] += ce
        else:
            mo.append(co)
            me.append(ce)
    mo, me = np.array(mo), np.array(me)
    if len(mo) < 2:
        return 1.0
    chi2 = float(((mo - me) ** 2 / me).sum())
    return float(stats.chi2.sf(chi2, len(mo) - 1))


def hyper_pmf_exact(k, L, R):
    """Exact Hypergeom(k draws, L successes, R total) PMF as Fractions."""
    den = comb(R, k)
    lo, hi = max(0, k + L - R), min(k, L)
    return {x: Fraction(comb(L, x) * comb(R - L, k - x), den) for x in range(lo, hi + 1)}


def hyper_pmf_float(k, L, R):
    lo, hi = max(0, k + L - R), min(k, L)
    xs = np.arange(lo, hi + 1)
    return xs, stats.hypergeom.pmf(xs, R, L, k)


def binom_pmf(k, p):
    xs = np.arange(0, k + 1)
    return xs, stats.binom.pmf(xs, k, p)


def counts_over(values, support):
    values = np.asarray(values, dtype=np.int64)
    lo = int(support[0])
    idx = values - lo
    assert idx.min() >= 0 and idx.max() < len(support), "value outside support"
    return np.bincount(idx, minlength=len(support))
