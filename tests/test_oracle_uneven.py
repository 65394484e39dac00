"""Pins of the oracle's NEXT-2 uneven-universe count assignment (P:421-468,
Section 4.3): binomial-tree hypergeometric splits of n over PEs holding L_i
elements.  The joint law of the counts must be the multivariate
hypergeometric distribution  P(c) = prod_i C(L_i, c_i) / C(sum L, n)  -- a
uniform n-subset of the union, counted per PE -- checked exactly on small
cases; plus the paper's Fig. 3 instance (13 PEs, 229 elements, 50 samples;
its numbers are lost, the structure is checked) and the degenerate cases.
-m "not gpu"."""
from __future__ import annotations

import itertools
from fractions import Fraction
from math import comb

import numpy as np
import pytest

import oracle as O
from tests.stats_util import ALPHA, chisq_pvalue


def _mvh_support(L, n):
    ranges = [range(0, l + 1) for l in L]
    for c in itertools.product(*ranges):
        if sum(c) == n:
            yield c


@pytest.mark.parametrize("L,n", [([3, 1, 4, 2, 5], 6), ([2, 2, 2], 3), ([5, 0, 3, 4], 5),
                                 ([1, 1, 1, 1, 1, 1, 1], 3), ([6, 2, 1, 3, 2, 2], 7)])
def test_counts_are_multivariate_hypergeometric(L, n):
    tot = sum(L)
    support = list(_mvh_support(L, n))
    prob = [Fraction(np.prod([comb(l, c) for l, c in zip(L, cs)], dtype=object), comb(tot, n))
            for cs in support]
    assert sum(prob) == 1
    index = {cs: i for i, cs in enumerate(support)}
    obs = np.zeros(len(support))
    trials = 40000
    for s in range(trials):
        c = tuple(int(v) for v in O.uneven_counts(L, n, 1000003 * s + 7))
        obs[index[c]] += 1
    assert chisq_pvalue(obs, [float(p) for p in prob]) > ALPHA


def test_fig3_instance_structure():
    # Fig. 3: 13 PEs, 229 elements in total, 50 samples (the values are lost)
    L = [17, 3, 40, 0, 25, 9, 11, 30, 14, 22, 8, 31, 19]
    assert sum(L) == 229
    for seed in range(50):
        c = O.uneven_counts(L, 50, seed)
        assert c.sum() == 50
        assert np.all(c <= np.asarray(L, dtype=np.uint64))
        assert c[3] == 0                                    # an empty PE gets nothing
        assert np.array_equal(c, O.uneven_counts(L, 50, seed))   # deterministic


def test_degenerate_cases():
    L = [4, 0, 7, 1]
    assert np.array_equal(O.uneven_counts(L, 0, 3), [0, 0, 0, 0])
    assert np.array_equal(O.uneven_counts(L, 12, 3), L)      # everything
    assert np.array_equal(O.uneven_counts([9], 5, 3), [5])   # one PE
    with pytest.raises(Exception):
        O.uneven_counts(L, 13, 3)


def test_marginals_large():
    # each PE's marginal count is Hypergeom(n, L_i, sum L): mean n L_i / sum L
    L = [2 ** 30, 3 * 2 ** 28, 12345, 2 ** 31, 0, 77 * 2 ** 20]
    tot, n = sum(L), 2 ** 24
    cs = np.array([O.uneven_counts(L, n, s) for s in range(300)], dtype=np.float64)
    for i, l in enumerate(L):
        mean = n * l / tot
        var = n * (l / tot) * (1 - l / tot) * (tot - n) / (tot - 1)
        if var == 0:
            assert np.all(cs[:, i] == mean)
            continue
        z = (cs[:, i].mean() - mean) / np.sqrt(var / len(cs))
        assert abs(z) < 4.5, (i, z)


def test_local_seeds_distinct():
    seeds = {O.uneven_seed(1, i) for i in range(1000)}
    assert len(seeds) == 1000
