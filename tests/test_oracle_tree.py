"""Pins for the oracle's split tree (CANON C4, C7) and Algorithm P replay.

* Exact rational enumeration on tiny N: composing the EXACT hypergeometric
  PMFs at every internal node -- with the node parameters (lo, R, L) the
  oracle itself uses -- and uniform leaves gives P(S) = 1/C(N,n) for every
  subset S (the claim of P:218-222 applied recursively, Fig. 1).  A wrong
  boundary, a swapped child or an L that is not the left child's size fails.
* Conservation: leaf counts sum to m and agree with the output; path replay
  (Fig. 2, <= log p deviates per PE) reproduces every leaf's count and
  offset; shard info agrees with the full sample.
"""
from __future__ import annotations

import itertools
from fractions import Fraction
from math import comb

import numpy as np
import pytest

import oracle as O
from tests.stats_util import hyper_pmf_exact


def _subset_prob(N, S, D):
    """P(S) under the fixed-depth tree with exact PMFs (Fractions)."""
    S = sorted(S)

    def cnt(lo, R):
        return sum(1 for v in S if lo < v <= lo + R)   # values are offset+1

    prob = Fraction(1)
    for d in range(D):
        for i in range(1 << d):
            lo, R, L = O.node(N, d, i)
            k = cnt(lo, R)
            llo, lR, _ = O.node(N, d + 1, 2 * i)
            rlo, rR, _ = O.node(N, d + 1, 2 * i + 1)
            # children partition the parent and L is the left child's size
            assert llo == lo and lR == L and rlo == lo + L and lR + rR == R
            x = cnt(llo, lR)
            if R == 0:
                continue
            pmf = hyper_pmf_exact(k, L, R)
            prob *= pmf.get(x, Fraction(0))
    for i in range(1 << D):
        lo, R, _ = O.node(N, D, i)
        prob /= comb(R, cnt(lo, R))
    return prob


@pytest.mark.parametrize("N,n", [(6, 2), (7, 3), (8, 3), (10, 3), (5, 2), (9, 4), (3, 1)])
@pytest.mark.parametrize("extra_depth", [0, 1])
def test_tree_composition_is_uniform(N, n, extra_depth):
    D, comp, m = O.plan(N, n)
    assert not comp and m == n
    D += extra_depth
    target = Fraction(1, comb(N, n))
    total = Fraction(0)
    for S in itertools.combinations(range(1, N + 1), n):
        p = _subset_prob(N, S, D)
        assert p == target, (S, p, target)
        total += p
    assert total == 1


def test_node_boundaries_match_fig1_for_power_of_two():
    """b(d,i) = floor(i N / 2^d) splits every node at floor(R/2) when N is a
    power of two -- Fig. 1's split position."""
    for N in (1, 2, 4, 64, 1 << 20):
        for d in range(0, 6):
            for i in range(1 << d):
                lo, R, L = O.node(N, d, i)
                assert L == R // 2


def test_depth_rule():
    assert O.depth(0) == 3 and O.depth(1024) == 3 and O.depth(8 * 1024) == 3
    assert O.depth(2 ** 20) == 10 and O.depth(2 ** 30) == 20 and O.depth(2 ** 32) == 22
    assert O.depth(2 ** 20 + 1) == 11
    D, comp, m = O.plan(2 ** 32, 3 * 2 ** 30)
    assert comp and m == 2 ** 30 and D == 20
    # "n > N/2" read as 2n > N: n = N/2 is not complemented (CANON C7)
    assert O.plan(100, 50)[1] is False and O.plan(100, 51)[1] is True


@pytest.mark.parametrize("N,n,seed", [(2 ** 30, 2 ** 20, 1), (10 ** 9 + 7, 123457, 3),
                                      (2 ** 40, 50000, 9), (5000, 2400, 4)])
def test_conservation_and_path_replay(N, n, seed):
    D, comp, m = O.plan(N, n)
    cnt = O.tree_counts(N, m, seed, D)
    assert int(cnt.sum()) == m
    out = O.sample_wor(N, n, seed)
    if not comp:
        lo = np.array([O.node(N, D, i)[0] for i in range(1 << D)], dtype=np.uint64)
        per_leaf = np.bincount(np.searchsorted(lo, out - 1, side="right") - 1, minlength=1 << D)
        assert np.array_equal(per_leaf.astype(np.uint64), cnt)
    offs = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.uint64)
    rng = np.random.default_rng(seed)
    for i in list(rng.integers(0, 1 << D, 40)) + [0, (1 << D) - 1]:
        k, off = O.path(N, m, seed, D, int(i))
        assert k == cnt[i] and off == offs[i]


@pytest.mark.parametrize("mode", [O.MODE_WOR, O.MODE_WR])
@pytest.mark.parametrize("N,n", [(2 ** 30, 2 ** 20), (2 ** 16, 3 * 2 ** 14), (1000, 999)])
def test_shard_info_partitions_the_sample(N, n, mode):
    if mode == O.MODE_WR:
        out = O.sample_wr(N, n, 7)
    else:
        out = O.sample_wor(N, n, 7)
    for world in (1, 2, 4, 8):
        total = 0
        for rank in range(world):
            c, off = O.shard_info(N, n, 7, world, rank, mode)
            lo = (rank * N) // world
            hi = ((rank + 1) * N) // world
            seg = out[off: off + c]
            assert off == total
            assert c == 0 or (seg.min() > lo and seg.max() <= hi)
            total += c
        assert total == n


def test_leaf_replay_equals_full_output():
    for (N, n, mode) in [(2 ** 30, 2 ** 20, 0), (2 ** 16, 3 * 2 ** 14, 0), (2 ** 24, 2 ** 18, 1)]:
        out = O.sample_wr(N, n, 5) if mode else O.sample_wor(N, n, 5)
        D = O.plan(N, n, mode)[0]
        for i in sorted({0, 1, min(17, (1 << D) - 2), (1 << D) - 1}):
            vals, off = O.leaf(N, n, 5, i, mode)
            assert np.array_equal(out[off: off + len(vals)], vals)
