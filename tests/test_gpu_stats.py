"""Statistical checks of the DEVICE output at full size (BASELINE's
"chi-square uniformity tests on the GPU output must pass at p > 1e-3"),
complementing the bit-exact parity tests: low-order bits of WOR values
(in-leaf positions, which the split does not fix), WR multiplicities, and
Bernoulli gaps (geometric).  -m gpu."""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch
from scipy import stats

import paper_1610_05141_b200 as rs
from paper_1610_05141_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _chi2_uniform(counts: torch.Tensor) -> float:
    c = counts.double()
    E = float(c.sum()) / c.numel()
    chi2 = float(((c - E) ** 2 / E).sum())
    return stats.chi2.sf(chi2, c.numel() - 1)


def test_wor_low_bits_uniform():
    # values mod 2^16 over n = 2^30 of N = 2^40: each leaf spans 2^20 values,
    # so these bins test the in-leaf draws (Lemire, buckets, dedup)
    c = W.CFG1
    out = rs.sample_wor(c["N"], c["n"], 7).view(torch.int64)
    assert _chi2_uniform(torch.bincount(out & 0xFFFF, minlength=2 ** 16)) > 1e-3
    # positions inside the leaf: (v - 1) mod r with r = N / 2^20 = 2^20, 1024 bins
    assert _chi2_uniform(torch.bincount(((out - 1) & (2 ** 20 - 1)) >> 10, minlength=1024)) > 1e-3
    del out
    torch.cuda.empty_cache()


def test_wr_multiplicities():
    # WR n = 2^32 of N = 2^36: equal neighbours = n - #distinct; #distinct is
    # the occupancy count of n balls in N bins: mean N (1 - e^-a), variance
    # N e^-a (1 - (1 + a) e^-a), a = n / N (Poisson limit, N -> inf)
    c = W.CFG4
    N, n = c["N"], c["n"]
    out = rs.sample_wr(N, n, 3).view(torch.int64)
    assert bool((out[1:] >= out[:-1]).all())
    eq = int((out[1:] == out[:-1]).sum())
    a = n / N
    mean = n + N * math.expm1(-a)                         # n - N (1 - e^-a)
    var = N * math.exp(-a) * (1 - (1 + a) * math.exp(-a))
    z = (eq - mean) / math.sqrt(var)
    assert abs(z) < 6, (eq, mean, z)
    # low bits over the first 2^30 values (torch.bincount is slow beyond 2^31)
    assert _chi2_uniform(torch.bincount(out[: 2 ** 30] & 0xFFFF, minlength=2 ** 16)) > 1e-3
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("N,rho", [(2 ** 32, 0.01), (2 ** 40, 2 ** -16)])
def test_bernoulli_gaps_geometric(N, rho):
    out = rs.bernoulli(N, rho, 5).view(torch.int64)
    n = out.numel()
    mu, sd = N * rho, math.sqrt(N * rho * (1 - rho))
    assert abs(n - mu) < 6 * sd
    G = (out[1:] - out[:-1] - 1).double()                 # ~ Geometric(rho) on {0, 1, ...}
    # ~64 bins of about equal probability: bin i = [e_(i-1), e_i), P(G < e) = 1 - (1 - rho)^e
    q = np.arange(1, 64) / 64.0
    e = np.unique(np.floor(np.log1p(-q) / math.log1p(-rho)))
    e = e[e > 0]
    idx = torch.bucketize(G, torch.tensor(e, dtype=torch.float64, device=out.device), right=True)
    counts = torch.bincount(idx, minlength=e.size + 1).double().cpu().numpy()
    cdf = np.concatenate([[0.0], -np.expm1(e * math.log1p(-rho)), [1.0]])
    p = np.diff(cdf)
    m = n - 1
    chi2 = float(((counts - p * m) ** 2 / (p * m)).sum())
    assert stats.chi2.sf(chi2, e.size) > 1e-3, chi2
