"""NEXT-4 pins: the oracle's Algorithm B + repair.

The method's plain definition is the distribution: a uniformly random
n-subset of 1..N, sorted.  Pinned by exact subset frequencies (chi-square over
all C(N, n) subsets, including the restart path with slack 0), the
inclusion probability n/N of every element, the special cases that reduce to
the already-pinned Bernoulli / WOR oracles (n' = n: no repair; rho' = 1: the
output is the complement of the removed positions), and the restart rate of a
zero-slack run (P(n' < n) close to 1/2).  -m "not gpu"."""
from __future__ import annotations

import itertools
import math

import numpy as np
import pytest

import oracle as O


def _chi2_crit(dof):
    # Wilson-Hilferty upper quantile at z = 4.5 (p ~ 3e-6)
    z = 4.5
    return dof * (1 - 2 / (9 * dof) + z * math.sqrt(2 / (9 * dof))) ** 3


@pytest.mark.parametrize("N,n,slack", [(6, 3, 0.0), (6, 2, 4.0), (7, 4, 1.0)])
def test_subsets_uniform(N, n, slack):
    subsets = {c: i for i, c in enumerate(itertools.combinations(range(1, N + 1), n))}
    reps = 200 * len(subsets)
    hist = np.zeros(len(subsets))
    for s in range(reps):
        v, a = O.algb(N, n, s, slack=slack)
        assert a >= 1
        hist[subsets[tuple(int(x) for x in v)]] += 1
    e = reps / len(subsets)
    chi2 = float(((hist - e) ** 2 / e).sum())
    assert chi2 < _chi2_crit(len(subsets) - 1), chi2


def test_inclusion_probability():
    N, n, reps = 40, 10, 4000
    hits = np.zeros(N + 1)
    for s in range(reps):
        v, _ = O.algb(N, n, 10_000 + s, slack=2.0)
        hits[v.astype(np.int64)] += 1
    p = n / N
    z = (hits[1:] / reps - p) / math.sqrt(p * (1 - p) / reps)
    assert np.abs(z).max() < 4.5


@pytest.mark.parametrize("N,n", [(1, 1), (10, 0), (10, 10), (1000, 1), (2 ** 30, 2 ** 20), (2 ** 48, 5000)])
def test_sorted_distinct_in_range(N, n):
    v, a = O.algb(N, n, 7)
    assert v.size == n and (n == 0 or (int(v[0]) >= 1 and int(v[-1]) <= N))
    assert np.all(np.diff(v.astype(np.int64)) > 0)
    if n == N:
        assert np.array_equal(v, np.arange(1, N + 1, dtype=np.uint64))


def test_no_repair_equals_bernoulli():
    # slack 0: rho' = n/N; whenever the first pass has exactly n elements the
    # output is that Bernoulli sample, untouched
    N, n, found = 200, 20, 0
    for s in range(400):
        b = O.bernoulli(N, n / N, s)
        if b.size == n:
            v, a = O.algb(N, n, s, slack=0.0)
            assert a == 1 and np.array_equal(v, b)
            found += 1
    assert found > 10


def test_rho_one_is_complement_of_removed_positions():
    # rho' = 1: S = 1..N, the removed positions are rs_sample_wor(N, N - n)
    N, n = 100, 95
    for s in range(20):
        v, a = O.algb(N, n, s, slack=4.0)
        assert a == 1
        rem = O.sample_wor(N, N - n, s)
        exp = np.setdiff1d(np.arange(1, N + 1, dtype=np.uint64), rem)
        assert np.array_equal(v, exp)


def test_repair_removes_wor_positions():
    # composition check against the pinned pieces: S = Bernoulli(rho'),
    # removed = positions rs_sample_wor(n', n' - n) (attempt 0)
    N, n, slack = 10 ** 6, 1000, 4.0
    rho = min(1.0, (n + slack * math.sqrt(n)) / N)
    for s in range(5):
        S = O.bernoulli(N, rho, s)
        if S.size < n:
            continue
        pos = O.sample_wor(S.size, S.size - n, s)
        keep = np.ones(S.size, dtype=bool)
        keep[pos.astype(np.int64) - 1] = False
        v, a = O.algb(N, n, s, slack=slack)
        assert a == 1 and np.array_equal(v, S[keep])


def test_restart_rate_zero_slack():
    # slack 0: P(n' < n) = P(Bin(N, n/N) < n) ~ 1/2 - O(1/sqrt(n)); attempts
    # are geometric, mean ~2
    N, n, reps = 1000, 100, 600
    att = np.array([O.algb(N, n, s, slack=0.0)[1] for s in range(reps)])
    frac_restart = float((att > 1).mean())
    assert 0.38 < frac_restart < 0.56
    assert 1.6 < att.mean() < 2.4


def test_arguments():
    with pytest.raises(ValueError):
        O.algb(10, 11, 1)
    with pytest.raises(ValueError):
        O.algb(10, 5, 1, slack=-1.0)
    with pytest.raises(ValueError):
        O.algb(10, 5, 1, slack=float("nan"))
