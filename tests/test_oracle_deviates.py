"""Distributional pins for the oracle's deviates (CANON C5, C8, C9).

HGD: exact-PMF chi-square over >= 10 parameter sets covering both the HYP
(k' < 16) and HRUA regimes, symmetry law, and z-tests of
mean kL/R and variance kL(R-L)(R-k)/(R^2(R-1)) at the headline sizes
(R = 2^48).  BIN: exact PMF over BINV and BTRS regimes.  GEO: mean
(1-rho)/rho and tail P(G >= g) = (1-rho)^g.  Seeds are fixed, so
every p-value is deterministic.
"""
from __future__ import annotations

import math

import numpy as np
import pytest
from scipy import stats

import oracle as O
from tests.stats_util import ALPHA, binom_pmf, chisq_pvalue, counts_over, hyper_pmf_exact

HGD_CASES = [
    # (k, L, R): HYP regime (k' < 16) ...
    (5, 5, 10), (3, 7, 20), (15, 30, 31), (12, 100, 1000), (9, 2, 50),
    # ... HRUA regime (k' >= 16), incl. reductions k > R/2, L > R/2
    (20, 20, 50), (100, 500, 1000), (37, 10, 60), (300, 450, 1000),
    (700, 400, 1000), (16, 32, 64), (60, 95, 100), (1024, 1 << 12, 1 << 13),
]


@pytest.mark.parametrize("k,L,R", HGD_CASES)
def test_hgd_exact_pmf(k, L, R):
    pmf = hyper_pmf_exact(k, L, R)
    xs = sorted(pmf)
    draws = O.hgd_batch(k, L, R, seed=12345, id0=1, count=60000)
    assert draws.min() >= xs[0] and draws.max() <= xs[-1]
    obs = counts_over(draws, xs)
    p = chisq_pvalue(obs, [float(pmf[x]) for x in xs])
    assert p > ALPHA, p


@pytest.mark.parametrize("k,L,R", [(20, 20, 50), (300, 450, 1000), (12, 100, 1000)])
def test_hgd_symmetry(k, L, R):
    """Hypergeom(k, L, R) is distributed as k - Hypergeom(k, R-L, R)."""
    a = O.hgd_batch(k, L, R, 99, 1, 40000).astype(np.int64)
    b = k - O.hgd_batch(k, R - L, R, 77, 1, 40000).astype(np.int64)
    lo, hi = min(a.min(), b.min()), max(a.max(), b.max())
    ca = np.bincount(a - lo, minlength=hi - lo + 1)
    cb = np.bincount(b - lo, minlength=hi - lo + 1)
    keep = (ca + cb) >= 10
    table = np.vstack([ca[keep], cb[keep]])
    p = stats.chi2_contingency(table)[1]
    assert p > ALPHA, p


@pytest.mark.parametrize("k,L,R", [
    (2 ** 32, 2 ** 47, 2 ** 48),     # headline root
    (2 ** 30, 2 ** 39, 2 ** 40),     # cfg1 root
    (1000, 2 ** 26, 2 ** 27),        # headline leaf-level split
    (2 ** 33, 2 ** 47, 2 ** 48),     # weak-scaling p=8 root
])
def test_hgd_large_moments_and_binned(k, L, R):
    n = 40000
    x = O.hgd_batch(k, L, R, seed=2024, id0=1, count=n).astype(np.float64)
    mean = k * L / R
    var = k * L * (R - L) * (R - k) / (R * R * (R - 1))
    z_mean = (x.mean() - mean) / math.sqrt(var / n)
    assert abs(z_mean) < 4.0, z_mean
    # sample variance z-test (kurtosis ~ 3 for the near-normal regime)
    z_var = (x.var(ddof=1) - var) / (var * math.sqrt(2.0 / (n - 1)))
    assert abs(z_var) < 4.0, z_var
    # binned chi-square over integer-edged bins at +-4 sigma: exact PMF sums
    # (scipy) for k <= 1e5, else the continuity-corrected normal CDF (its
    # error is O(1/k) ~ 1e-9 here)
    sd = math.sqrt(var)
    edges = np.unique(np.floor(mean + sd * np.linspace(-4, 4, 33)).astype(np.int64))
    if k <= 100000:
        cdf = stats.hypergeom.cdf(edges - 1, R, L, k)
    else:
        cdf = stats.norm.cdf((edges - 0.5 - mean) / sd)
    probs = np.diff(np.concatenate([[0.0], cdf, [1.0]]))
    idx = np.searchsorted(edges, x.astype(np.int64), side="right")
    obs = np.bincount(idx, minlength=len(edges) + 1)
    p = chisq_pvalue(obs, probs)
    assert p > ALPHA, p


def test_hgd_deterministic_and_keyed():
    a = O.hgd_batch(1000, 2 ** 26, 2 ** 27, 5, 1, 100)
    b = O.hgd_batch(1000, 2 ** 26, 2 ** 27, 5, 1, 100)
    c = O.hgd_batch(1000, 2 ** 26, 2 ** 27, 6, 1, 100)
    assert np.array_equal(a, b) and not np.array_equal(a, c)


BIN_CASES = [
    (10, 1, 2), (30, 1, 3), (7, 2, 9), (25, 1, 4), (40, 7, 20),      # BINV (k p' < 10)
    (1000, 3, 10), (200, 1, 2), (64, 17, 40), (500, 9, 10), (45, 1, 2),  # BTRS
]


@pytest.mark.parametrize("k,L,R", BIN_CASES)
def test_bin_exact_pmf(k, L, R):
    p = L / R
    xs, pmf = binom_pmf(k, p)
    draws = O.bin_batch(k, L, R, seed=4321, id0=1, count=60000)
    obs = counts_over(draws, xs)
    pv = chisq_pvalue(obs, pmf)
    assert pv > ALPHA, pv


@pytest.mark.parametrize("k,L,R", [(2 ** 32, 2 ** 35, 2 ** 36), (2 ** 20, 1, 2),
                                   (2 ** 32, 2 ** 35, 2 ** 36 + 1)])
def test_bin_large_moments(k, L, R):
    n = 40000
    x = O.bin_batch(k, L, R, 77, 1, n).astype(np.float64)
    p = L / R
    mean, var = k * p, k * p * (1 - p)
    assert abs((x.mean() - mean) / math.sqrt(var / n)) < 4.0
    assert abs((x.var(ddof=1) - var) / (var * math.sqrt(2.0 / (n - 1)))) < 4.0


@pytest.mark.parametrize("rho", [0.5, 0.01, 1e-4, 0.9])
def test_geo_mean_and_tail(rho):
    """G = floor(log U / log1p(-rho)): E G = (1-rho)/rho, P(G>=g) = (1-rho)^g."""
    n = 200000
    rng = np.random.default_rng(1)
    words = rng.integers(0, 2 ** 32, size=(n, 2), dtype=np.uint64)
    lr = O.log1p(-rho)
    G = np.array([O.geo(O.u52(int(a), int(b)), lr) for a, b in words])
    mean = (1 - rho) / rho
    sd = math.sqrt(1 - rho) / rho
    assert abs((G.mean() - mean) / (sd / math.sqrt(n))) < 4.0
    for g in (1, 2, 5, int(1 / rho)):
        emp = (G >= g).mean()
        th = (1 - rho) ** g
        assert abs(emp - th) < 5 * math.sqrt(th * (1 - th) / n) + 1e-12
