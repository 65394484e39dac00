"""Pins for the oracle's primitives (CANON C0-C3, C5 log-ratio): -m "not gpu".

Each test checks the oracle against something other than itself: published
known-answer vectors, exhaustive enumeration, or mpmath at 50 digits.
"""
from __future__ import annotations

import math
import os
import random
import struct

import mpmath as mp
import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _ulp(x: float) -> float:
    return math.ulp(x)


# ---- C1 Philox ---------------------------------------------------------------

def test_philox_kat():
    """Random123 kat_vectors for philox4x32-10 (tests/golden, cited there)."""
    n = 0
    for line in open(os.path.join(GOLD, "philox4x32_10_kat.txt")):
        if not line.strip() or line.startswith("#"):
            continue
        w = [int(t, 16) for t in line.split()]
        assert O.philox(w[0:4], w[4:6]) == tuple(w[6:10])
        n += 1
    assert n == 3


# ---- C3 uniform maps ---------------------------------------------------------

def test_u52_range_and_symmetry():
    """u52 lies in (0,1), hits both extreme cells, and u52(a,b)+u52(~a,~b)==1
    exactly (the (M+0.5)/2^52 grid is symmetric about 1/2)."""
    rng = random.Random(7)
    for _ in range(20000):
        a, b = rng.getrandbits(32), rng.getrandbits(32)
        u = O.u52(a, b)
        assert 0.0 < u < 1.0
        assert u + O.u52(a ^ 0xFFFFFFFF, b ^ 0xFFFFFFFF) == 1.0
    assert O.u52(0, 0) == 2.0 ** -53
    assert O.u52(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 2.0 ** -53


@pytest.mark.slow
@pytest.mark.parametrize("r", [3, 1000003, (1 << 26) + 3])
def test_lemire_exhaustive(r):
    """All 2^32 words: every value of [0,r) has exactly floor(2^32/r)
    accepted preimages (no modulo bias), and exactly
    2^32 - (2^32 mod r) words are accepted."""
    hist, acc = O.lemire32_hist(r)
    q = (1 << 32) // r
    assert acc == q * r == (1 << 32) - ((1 << 32) % r)
    assert int(hist.min()) == q and int(hist.max()) == q


def test_lemire_power_of_two_is_shift():
    """For r = 2^s the map is value = word >> (32 - s), never rejecting."""
    rng = random.Random(3)
    for s in (1, 10, 20, 26, 31, 32):
        for _ in range(200):
            w = rng.getrandbits(32)
            import ctypes
            v = ctypes.c_uint64()
            ok = O.lib().rso_lemire32(w, 1 << s, ctypes.byref(v))
            assert ok == 1 and v.value == w >> (32 - s)


def _ceil_div(a, b):
    return -(-a // b)


@pytest.mark.parametrize("r", [(1 << 38) + 1, 3 * (1 << 37) + 12345, (1 << 40) - 3,
                               (1 << 44) + 777, (1 << 62) + 5, (1 << 63) - 25])
def test_lemire64_preimages(r):
    """CANON C3, r > 2^32 branch (rso_lemire64, used by rso_draw): value v's
    preimage words are exactly w in [ceil(v 2^64 / r), ceil((v+1) 2^64 / r))
    (floor(w r / 2^64) = v, exact integer arithmetic here), and of those exactly
    floor(2^64 / r) must be accepted -- the same count for every v, i.e. no
    modulo bias.  A reversed accept test or a wrong threshold changes
    the count for some v.  The words just outside the interval must not
    produce v."""
    q = (1 << 64) // r
    rng = random.Random(r)
    vs = {0, 1, r - 1, r // 2} | {rng.randrange(r) for _ in range(3)}
    for v in sorted(vs):
        lo = _ceil_div(v << 64, r)
        hi = min(_ceil_div((v + 1) << 64, r), 1 << 64)
        acc, other, rej = O.lemire64_scan(r, v, lo, hi)
        assert other == 0 and acc == q and acc + rej == hi - lo, (r, v, acc, other, rej)
        if lo > 0:
            assert O.lemire64_scan(r, v, lo - 1, lo)[0] == 0
        if hi < (1 << 64):
            assert O.lemire64_scan(r, v, hi, hi + 1)[0] == 0


def test_draw_in_range_and_64bit_path():
    for r in (1, 2, 7, 1 << 26, (1 << 32) - 1, 1 << 32, (1 << 32) + 1, 3 << 40, (1 << 62) + 5):
        for j in range(64):
            assert O.draw(11, 2, 1234, r, j) < r


# ---- C0 logarithms -------------------------------------------------------------

mp.mp.dps = 50


def _log_inputs():
    rng = random.Random(11)
    xs = [1.0, 2.0, 0.5, math.e, 1 + 2 ** -52, 1 - 2 ** -53, 2 ** -1074, 2 ** -1022,
          5e-324, 1.7976931348623157e308, 0.7071067811865476, 1.4142135623730951]
    for _ in range(30000):
        e = rng.uniform(-300, 300)
        xs.append(rng.random() * 10 ** e + 1e-300)
    for _ in range(20000):
        xs.append(1.0 + rng.uniform(-0.3, 0.3))
    for _ in range(5000):   # u52 grid values, the HRUA / GEO inputs
        xs.append(O.u52(rng.getrandbits(32), rng.getrandbits(32)))
    return xs


def test_log_within_one_ulp():
    worst = 0.0
    for x in _log_inputs():
        got = O.log(x)
        ref = mp.log(mp.mpf(x))
        err = abs(mp.mpf(got) - ref) / _ulp(float(ref)) if ref != 0 else abs(got)
        worst = max(worst, float(err))
    assert worst <= 1.0, worst
    assert O.log(0.0) == -math.inf
    assert math.isnan(O.log(-1.0))


def test_log1p_accuracy():
    rng = random.Random(5)
    xs = [-0.5, -0.01, -1e-10, 1e-300, -0.999999, 0.25, 3.0, 1e10, -2 ** -60]
    xs += [-(10 ** rng.uniform(-17, -0.0001)) for _ in range(10000)]
    xs += [10 ** rng.uniform(-17, 5) for _ in range(5000)]
    worst = 0.0
    for x in xs:
        got = O.log1p(x)
        ref = mp.log1p(mp.mpf(x))
        worst = max(worst, float(abs(mp.mpf(got) - ref) / _ulp(float(ref))))
    assert worst <= 4.0, worst


# ---- C5 Loader pieces ------------------------------------------------------------

def test_stirlerr_vs_mpmath():
    """stirlerr(n) = log n! - log(sqrt(2 pi n) (n/e)^n).  Table region exact
    to 1/2 ulp; series region (n > 15, Loader's 5-term asymptotic series)
    to 2e-16 absolute -- what T's absolute accuracy needs."""
    for n in list(range(1, 200)) + [500, 501, 10 ** 4, 2 ** 26, 2 ** 40, 2 ** 52]:
        ref = mp.loggamma(n + 1) - (n + mp.mpf(0.5)) * mp.log(n) + n - mp.log(2 * mp.pi) / 2
        got = O.stirlerr(n)
        tol = 0.5 * _ulp(float(ref)) if n <= 15 else 2e-16 + 4e-16 * abs(float(ref))
        assert abs(mp.mpf(got) - ref) <= tol, (n, got, ref)


def test_bd0_vs_mpmath():
    """bd0(x, np) = x log(x/np) + np - x, relative accuracy in both branches."""
    rng = random.Random(2)
    cases = [(10.0, 10.5), (1e6, 1e6 + 3), (2.0 ** 31, 2.0 ** 31 - 12345.5), (5.0, 50.0),
             (1000.0, 1040.0), (1.0, 0.3)]
    for _ in range(2000):
        npv = 10 ** rng.uniform(0, 15)
        x = float(max(1, round(npv * (1 + rng.uniform(-0.3, 0.3)))))
        cases.append((x, npv))
    for x, npv in cases:
        ref = mp.mpf(x) * mp.log(mp.mpf(x) / npv) + npv - x
        got = O.bd0(x, npv)
        assert abs(mp.mpf(got) - ref) <= 1e-13 * abs(ref) + 1e-300, (x, npv, got, ref)


def _lf(v):
    return mp.loggamma(mp.mpf(v) + 1)


def _T_exact(kp, g, R, K, M):
    def lpmf(x):
        return -(_lf(x) + _lf(g - x) + _lf(kp - x) + _lf(R - g - kp + x))
    return lpmf(K) - lpmf(M)


@pytest.mark.parametrize("kp,g,R", [
    (2 ** 32, 2 ** 47, 2 ** 48),        # headline root split
    (2 ** 30, 2 ** 39, 2 ** 40),        # cfg1 root split
    (1024, 2 ** 26, 2 ** 27),           # leaf-level split at the headline
    (3 * 2 ** 29, 2 ** 31, 2 ** 32),    # complement core root (cfg3a)
    (40, 1000, 5000),                   # small, skewed
])
def test_hgd_logratio_stable(kp, g, R):
    """T = log f(K) - log f(M) against mpmath loggamma at 50 digits on a grid
    of K = M +- {0.3 .. 12} sigma: abs err <= 1e-12.  The textbook
    sum-of-log-factorials is noise at R = 2^48 (lfact ~ 9e15, ulp 2)."""
    M = ((kp + 1) * (g + 1)) // (R + 2)
    p = g / R
    sd = math.sqrt(kp * p * (1 - p) * (R - kp) / (R - 1))
    for z in (-12, -5, -2, -1, -0.3, 0, 0.3, 1, 2, 5, 12):
        K = int(M + z * sd)
        K = min(max(K, 0), min(kp, g))
        got = O.hgd_logratio(kp, g, R, K, M)
        ref = _T_exact(kp, g, R, K, M)
        assert abs(mp.mpf(got) - ref) <= 1e-12 * max(1.0, abs(float(ref))), (K, M, got, ref)


def test_naive_logratio_is_noise_at_2_48():
    """Documents why CANON uses Loader's form: the lgamma-difference formula
    in doubles is off by O(1) at the headline root split."""
    kp, g, R = 2 ** 32, 2 ** 47, 2 ** 48
    M = ((kp + 1) * (g + 1)) // (R + 2)
    K = M + 40000
    naive = (math.lgamma(M + 1) + math.lgamma(g - M + 1) + math.lgamma(kp - M + 1)
             + math.lgamma(R - g - kp + M + 1)) - (math.lgamma(K + 1) + math.lgamma(g - K + 1)
             + math.lgamma(kp - K + 1) + math.lgamma(R - g - kp + K + 1))
    ref = float(_T_exact(kp, g, R, K, M))
    assert abs(naive - ref) > 1e-3
    assert abs(O.hgd_logratio(kp, g, R, K, M) - ref) < 1e-12


def test_spec_examples():
    """Degenerate supports and the log(36/70) example (tests/golden/spec_examples.txt)."""
    for line in open(os.path.join(GOLD, "spec_examples.txt")):
        if not line.strip() or line.startswith("#"):
            continue
        t = line.split()
        if t[0] == "hgd":
            k, L, R, x = map(int, t[1:])
            for s in range(20):
                assert O.hgd(k, L, R, s, 1) == x
        elif t[0] == "bin":
            k, L, R, x = map(int, t[1:])
            for s in range(20):
                assert O.binom(k, L, R, s, 1) == x
        elif t[0] == "logpmf":
            x, k, L, R = map(int, t[1:5])
            num, den = map(int, t[5].split("/"))
            # log f(x) - log f(mode) + log f(mode) == log pmf; pin the ratio
            M = ((k + 1) * (L + 1)) // (R + 2)
            from math import comb
            ref = math.log(num / den) - math.log(comb(L, M) * comb(R - L, k - M) / comb(R, k))
            assert abs(O.hgd_logratio(k, L, R, x, M) - ref) < 1e-14
