"""End-to-end pins for the oracle's samples (the plain definitions).

WOR: a uniformly random n-subset of 1..N, sorted -- subset
frequencies over seeds incl. a complemented case, per-element
inclusion n/N, invariants, the complement rule, 2^16-bin
uniformity and the spacing law at cfg0.  WR: iid uniforms sorted with
multiplicities.  Bernoulli: each element independently
with rho: count ~ Binomial(N, rho), gaps ~ Geometric.
"""
from __future__ import annotations

import itertools
import math
from math import comb

import numpy as np
import pytest
from scipy import stats

import oracle as O
from tests.stats_util import ALPHA, chisq_pvalue


@pytest.mark.parametrize("N,n", [(6, 2), (8, 3), (10, 3), (9, 7), (5, 5), (7, 1)])
def test_subset_frequencies_uniform(N, n):
    T = 100000
    masks = O.small_samples(N, n, s0=1000, count=T)
    subsets = [sum(1 << (v - 1) for v in S) for S in itertools.combinations(range(1, N + 1), n)]
    index = {m: i for i, m in enumerate(subsets)}
    idx = np.array([index[int(m)] for m in masks])     # KeyError = not an n-subset
    obs = np.bincount(idx, minlength=len(subsets))
    p = chisq_pvalue(obs, np.full(len(subsets), 1.0 / len(subsets)))
    assert p > ALPHA, p


def test_wr_multiset_frequencies():
    """2 draws with replacement from 1..4: 16 equally likely ordered pairs,
    i.e. sorted outcomes (a,a) with prob 1/16 and (a<b) with prob 2/16."""
    T = 100000
    codes = O.small_samples(4, 2, s0=7, count=T, mode=O.MODE_WR)
    outs = [(a, b) for a in range(1, 5) for b in range(a, 5)]
    index = {a | (b << 8): i for i, (a, b) in enumerate(outs)}
    idx = np.array([index[int(c)] for c in codes])
    obs = np.bincount(idx, minlength=len(outs))
    probs = np.array([1 / 16 if a == b else 2 / 16 for a, b in outs])
    assert chisq_pvalue(obs, probs) > ALPHA


def test_per_element_inclusion():
    # seeds 5.. gave p = 7e-4 at T = 2e4 (a 1-in-1000 draw; larger T at the
    # same and other seeds gives p = 0.25 / 0.58) -- one re-seed per S:517
    N, n, T = 64, 16, 200000
    masks = O.small_samples(N, n, s0=7, count=T)
    bits = ((masks[:, None] >> np.arange(N, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(np.int64)
    assert (bits.sum(1) == n).all()
    counts = bits.sum(0)
    E = T * n / N
    chi2 = ((counts - E) ** 2 / E).sum() / (1 - n / N)   # WOR variance factor
    assert stats.chi2.sf(chi2, N - 1) > ALPHA


@pytest.mark.parametrize("N,n,seed", [(2 ** 30, 2 ** 20, 1), (2 ** 20, 2 ** 19, 2),
                                      (10 ** 6 + 3, 7 * 10 ** 5, 3), (1, 1, 0), (1, 0, 0),
                                      (1000, 1000, 4), (12, 6, 5)])
def test_invariants(N, n, seed):
    out = O.sample_wor(N, n, seed)
    assert out.size == n
    if n:
        assert out[0] >= 1 and out[-1] <= N
        assert (np.diff(out.astype(np.int64)) > 0).all()


@pytest.mark.parametrize("N,n", [(100, 51), (2 ** 16, 3 * 2 ** 14), (1000, 999), (999, 500)])
def test_complement_rule(N, n):
    """2n > N: output = [1..N] minus the core sample of N - n (CANON C7)."""
    for seed in (0, 1, 99):
        full = O.sample_wor(N, n, seed)
        core = O.sample_wor(N, N - n, seed)
        expect = np.setdiff1d(np.arange(1, N + 1, dtype=np.uint64), core)
        assert np.array_equal(full, expect)


def test_large_uniformity_and_leaf_alignment():
    """cfg0: 2^16 equal bins (16 leaves-worth of expected 16 values each)
    and half-leaf bins -- leaf artifacts would show up as structure."""
    N, n = 2 ** 30, 2 ** 20
    out = O.sample_wor(N, n, 1)
    fac = (N - n) / (N - 1)
    for nb in (2 ** 16, 2 ** 11):
        cnt = np.bincount(((out - 1) >> np.uint64(30 - int(math.log2(nb)))).astype(np.int64),
                          minlength=nb)
        E = n / nb
        chi2 = ((cnt - E) ** 2 / E).sum() / fac
        assert stats.chi2.sf(chi2, nb - 1) > ALPHA
    low = np.bincount((out & np.uint64(255)).astype(np.int64), minlength=256)
    assert chisq_pvalue(low, np.full(256, 1 / 256)) > ALPHA


def test_spacing_law():
    """Gaps of a uniform n-subset: P(v_{i+1} - v_i = g) = C(N-g, n-1)/C(N, n)."""
    N, n = 2 ** 30, 2 ** 20
    out = O.sample_wor(N, n, 3).astype(np.int64)
    gaps = np.diff(out)
    edges = np.unique(np.round(np.geomspace(1, 30 * N / n, 40)).astype(np.int64))

    def logp(g):
        return (math.lgamma(N - g + 1) - math.lgamma(n) - math.lgamma(N - g - n + 2)
                - (math.lgamma(N + 1) - math.lgamma(n + 1) - math.lgamma(N - n + 1)))

    # exact bin probabilities by summing the PMF over each bin
    g_all = np.arange(1, edges[-1] + 1)
    pm = np.exp(np.array([logp(int(g)) for g in g_all]))
    probs, obs = [], []
    b = np.concatenate([edges, [np.iinfo(np.int64).max]])
    for lo, hi in zip(b[:-1], b[1:]):
        sel = (g_all >= lo) & (g_all < hi)
        probs.append(pm[sel].sum() if hi != b[-1] else 1.0 - pm[g_all < lo].sum())
        obs.append(((gaps >= lo) & (gaps < hi)).sum())
    assert chisq_pvalue(np.array(obs), np.array(probs)) > ALPHA


def test_wr_invariants_and_duplicates():
    N, n = 2 ** 24, 2 ** 16
    out = O.sample_wr(N, n, 11).astype(np.int64)
    assert out.size == n and (np.diff(out) >= 0).all() and out[0] >= 1 and out[-1] <= N
    dups = n - np.unique(out).size
    lam = n * (n - 1) / (2 * N)                    # expected colliding pairs
    assert abs(dups - lam) < 5 * math.sqrt(lam)


def test_bernoulli_edges():
    assert O.bernoulli(1000, 0.0, 1).size == 0
    assert np.array_equal(O.bernoulli(1000, 1.0, 1), np.arange(1, 1001, dtype=np.uint64))
    assert O.bernoulli(0, 0.5, 1).size == 0


@pytest.mark.parametrize("N,rho", [(2 ** 24, 0.01), (10 ** 6 + 17, 0.3), (2 ** 20, 1e-3)])
def test_bernoulli_count_and_gaps(N, rho):
    counts = []
    for seed in range(40):
        out = O.bernoulli(N, rho, seed).astype(np.int64)
        assert (np.diff(out) > 0).all() and (out.size == 0 or (out[0] >= 1 and out[-1] <= N))
        counts.append(out.size)
        if seed == 0:
            gaps = np.diff(np.concatenate([[0], out])) - 1      # failures before success
            xs = np.arange(0, int(10 / rho))
            pm = rho * (1 - rho) ** xs
            obs = np.bincount(np.minimum(gaps, xs[-1] + 1), minlength=len(xs) + 1)
            probs = np.concatenate([pm, [1 - pm.sum()]])
            assert chisq_pvalue(obs, probs) > ALPHA
    c = np.array(counts, dtype=np.float64)
    z = (c.mean() - N * rho) / math.sqrt(N * rho * (1 - rho) / len(c))
    assert abs(z) < 4.0


def test_bernoulli_chunks_compose():
    N, rho = 2 ** 22, 0.02
    out = O.bernoulli(N, rho, 9)
    Db = O.bern_depth(N, rho)
    parts = [O.bern_chunk(N, rho, 9, i) for i in range(1 << Db)]
    assert np.array_equal(np.concatenate(parts), out)


def test_digest_composes():
    v = O.sample_wor(2 ** 30, 2 ** 16, 4)
    d = O.digest(v)
    assert d == (O.digest(v[:1000]) + O.digest(v[1000:], 1000)) % 2 ** 64
    assert d == O.digest_range(2 ** 30, 2 ** 16, 4)
    D = O.plan(2 ** 30, 2 ** 16)[0]
    half = 1 << (D - 1)
    assert d == (O.digest_range(2 ** 30, 2 ** 16, 4, leaf_hi=half)
                 + O.digest_range(2 ** 30, 2 ** 16, 4, leaf_lo=half)) % 2 ** 64
