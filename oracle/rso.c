/*
 * oracle/rso.c -- the CPU ORACLE for the divide-and-conquer sampler of
 * Sanders, Lamm, Huebschle-Schneider, Schrade, Dachsbacher,
 * "Efficient Random Sampling -- Parallel, Vectorized, Cache-Efficient, and
 * Online" (arXiv 1610.05141).  P:n below = /root/reference/PAPER.md line n.
 *
 * THIS IS TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * (paper_1610_05141_b200/, librs.so) never includes, links or calls it, and
 * it shares no code, header, table or constant generator with the CUDA path.
 *
 * It is deliberately plain and slow: every function follows the paper's
 * algorithm in the paper's order, under the canonical readings ("CANON v1",
 * DESIGN.md section 3) wherever the paper is silent.  Build:
 *   gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread
 * (no FMA contraction, no fast-math; x86-64 SSE2 doubles, round-to-nearest).
 *
 * Pins (tests/test_oracle_*.py, all `-m "not gpu"`):
 *   philox          -- Random123 known-answer vectors.
 *   rso_draw        -- exhaustive 2^32-word enumeration: every value of
 *                      [0,r) has exactly floor(2^32/r) accepted preimages.
 *   rso_log/log1p   -- <= 1 ulp (log) / <= 4 ulp (log1p) vs mpmath.
 *   stirlerr/bd0    -- vs mpmath closed forms.
 *   rso_hgd         -- degenerate cases, exact-PMF chi-square (HYP and HRUA
 *                      regimes), mean/variance z-tests at R = 2^48, and the
 *                      log-ratio T vs mpmath loggamma (abs err <= 1e-12).
 *   rso_bin, geo    -- exact-PMF chi-square, closed-form mean / tail.
 *   tree            -- exact rational enumeration on tiny N composing exact
 *                      hypergeometric PMFs over the oracle's own node
 *                      parameters: P(S) = 1/C(N,n) for every subset S.
 *   end to end      -- subset-frequency chi-square over seeds, invariants
 *                      (n distinct sorted values in 1..N), complement rule.
 * The exact sample VALUES for a seed are fixed only by CANON (the paper prints
 * no RNG and no sample): "parity unpinned by the paper" for the values
 * themselves; the distribution is what the pins above fix.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <float.h>
#include <pthread.h>

typedef unsigned __int128 u128;
typedef uint64_t u64;
typedef uint32_t u32;

/* ------------------------------------------------------------------------- */
/* CANON C1: Philox4x32-10 (Salmon et al., SC'11).  Replaces the paper's     */
/* SpookyHash + Mersenne twister by one counter-based */
/* generator so that "the t-th random deviate is h((j,k,t))" is  */
/* literally a hash of (node id, purpose, t).                                */
/* ------------------------------------------------------------------------- */
void rso_philox(const u32 ctr[4], const u32 key[2], u32 out[4])
{
    u32 c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    u32 k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) {              /* bump the key before rounds 2..10 */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        u64 p0 = (u64)0xD2511F53u * (u64)c0;
        u64 p1 = (u64)0xCD9E8D57u * (u64)c2;
        u32 hi0 = (u32)(p0 >> 32), lo0 = (u32)p0;
        u32 hi1 = (u32)(p1 >> 32), lo1 = (u32)p1;
        u32 n0 = hi1 ^ c1 ^ k0;
        u32 n1 = lo1;
        u32 n2 = hi0 ^ c3 ^ k1;
        u32 n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* CANON C2: counter = (index, purpose<<24 | attempt, id_lo, id_hi),
 * key = (seed_lo, seed_hi).  Node id = 2^d + i (heap numbering, root 1). */
enum { PUR_HGD = 1, PUR_WOR = 2, PUR_BIN = 3, PUR_WR = 4, PUR_GEO = 5 };

static void block(u64 seed, u32 purpose, u32 attempt, u64 id, u32 index, u32 w[4])
{
    u32 ctr[4] = { index, (purpose << 24) | attempt, (u32)id, (u32)(id >> 32) };
    u32 key[2] = { (u32)seed, (u32)(seed >> 32) };
    rso_philox(ctr, key, w);
}

/* CANON C3: u52(a,b) = ((a<<32|b) >> 12) + 0.5) * 2^-52, in (0,1), never 0. */
double rso_u52(u32 a, u32 b)
{
    u64 x = ((u64)a << 32) | (u64)b;
    double m = (double)(x >> 12);          /* exact: < 2^52 */
    return (m + 0.5) * 0x1p-52;            /* exact */
}

/* The s-th uniform of a sequential stream: pair (s mod 2) of block s/2. */
static double stream_u52(u64 seed, u32 purpose, u64 id, u64 s)
{
    u32 w[4];
    block(seed, purpose, 0, id, (u32)(s >> 1), w);
    return (s & 1) ? rso_u52(w[2], w[3]) : rso_u52(w[0], w[1]);
}

/* CANON C3: the j-th bounded draw from [0, r) of a leaf stream (Lemire's
 * multiply-shift with rejection; "uniform deviates X from 1..N").
 * r <= 2^32: attempt 0 = word j%4 of block j/4; attempt a>=1 = word 0 of
 * block index j, attempt field a.  r > 2^32: 64-bit words (pair j%2 of block
 * j/2; retry = words 0,1 of block j, attempt a), 128-bit product. */
/* Lemire's map of one 32-bit word to [0, r), r <= 2^32: accept iff the
 * low half of word*r is >= 2^32 mod r; value = high half. */
int rso_lemire32(u32 word, u64 r, u64 *value)
{
    u64 thresh = 0x100000000ull % r;
    u64 prod = (u64)word * r;
    *value = prod >> 32;
    return (prod & 0xffffffffull) >= thresh;
}

/* Lemire's map of one 64-bit word to [0, r), 2^32 < r < 2^64: accept iff the
 * low half of the 128-bit product word*r is >= 2^64 mod r; value = high half
 * (the r > 2^32 branch of CANON C3; pinned by preimage counting:
 * tests/test_oracle_primitives.py::test_lemire64_preimages). */
int rso_lemire64(u64 word, u64 r, u64 *value)
{
    u64 thresh = (u64)(((u128)1 << 64) % r); /* 2^64 mod r */
    u128 prod = (u128)word * r;
    *value = (u64)(prod >> 64);
    return (u64)prod >= thresh;
}

u64 rso_draw(u64 seed, u32 purpose, u64 id, u64 r, u64 j)
{
    u32 w[4];
    if (r <= 0x100000000ull) {
        for (u32 a = 0;; a++) {
            u32 word;
            u64 v;
            if (a == 0) { block(seed, purpose, 0, id, (u32)(j >> 2), w); word = w[j & 3]; }
            else        { block(seed, purpose, a, id, (u32)j, w);        word = w[0]; }
            if (rso_lemire32(word, r, &v)) return v;
        }
    } else {
        for (u32 a = 0;; a++) {
            u64 word, v;
            if (a == 0) {
                block(seed, purpose, 0, id, (u32)(j >> 1), w);
                word = (j & 1) ? (((u64)w[2] << 32) | w[3]) : (((u64)w[0] << 32) | w[1]);
            } else {
                block(seed, purpose, a, id, (u32)j, w);
                word = ((u64)w[0] << 32) | w[1];
            }
            if (rso_lemire64(word, r, &v)) return v;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* CANON C0: logarithms from + - * / only (bit-identical on any IEEE host).  */
/* rso_log transcribes the classic fdlibm e_log.c algorithm (argument        */
/* reduction to [sqrt(2)/2, sqrt(2)), Remez polynomial in s = f/(2+f)).       */
/* ------------------------------------------------------------------------- */
static u64 dbits(double x) { u64 u; memcpy(&u, &x, 8); return u; }
static double bitsd(u64 u) { double x; memcpy(&x, &u, 8); return x; }

double rso_log(double x)
{
    static const double ln2_hi = 0x1.62e42fee00000p-1;
    static const double ln2_lo = 0x1.a39ef35793c76p-33;
    static const double two54  = 0x1p54;
    static const double Lg1 = 0x1.5555555555593p-1, Lg2 = 0x1.999999997fa04p-2,
                        Lg3 = 0x1.2492494229359p-2, Lg4 = 0x1.c71c51d8e78afp-3,
                        Lg5 = 0x1.7466496cb03dep-3, Lg6 = 0x1.39a09d078c69fp-3,
                        Lg7 = 0x1.2f112df3e5244p-3;
    u64 u = dbits(x);
    int32_t hx = (int32_t)(u >> 32);
    u32 lx = (u32)u;
    int k = 0;
    if (hx < 0x00100000) {                      /* x < 2^-1022 */
        if (((hx & 0x7fffffff) | lx) == 0) return -INFINITY;
        if (hx < 0) return NAN;
        k -= 54; x *= two54;
        u = dbits(x); hx = (int32_t)(u >> 32);
    }
    if (hx >= 0x7ff00000) return x + x;
    k += (hx >> 20) - 1023;
    hx &= 0x000fffff;
    int32_t i = (hx + 0x95f64) & 0x100000;
    u = dbits(x);
    u = ((u64)(u32)(hx | (i ^ 0x3ff00000)) << 32) | (u & 0xffffffffull);
    x = bitsd(u);                               /* normalize x or x/2 */
    k += (i >> 20);
    double f = x - 1.0;
    double dk, R, s, z, w, t1, t2, hfsq;
    if ((0x000fffff & (2 + hx)) < 3) {          /* |f| < 2^-20 */
        if (f == 0.0) {
            if (k == 0) return 0.0;
            dk = (double)k;
            return dk * ln2_hi + dk * ln2_lo;
        }
        R = f * f * (0.5 - 0.33333333333333333 * f);
        if (k == 0) return f - R;
        dk = (double)k;
        return dk * ln2_hi - ((R - dk * ln2_lo) - f);
    }
    s = f / (2.0 + f);
    dk = (double)k;
    z = s * s;
    i = hx - 0x6147a;
    w = z * z;
    int32_t j = 0x6b851 - hx;
    t1 = w * (Lg2 + w * (Lg4 + w * Lg6));
    t2 = z * (Lg1 + w * (Lg3 + w * (Lg5 + w * Lg7)));
    i |= j;
    R = t2 + t1;
    if (i > 0) {
        hfsq = 0.5 * f * f;
        if (k == 0) return f - (hfsq - s * (hfsq + R));
        return dk * ln2_hi - ((hfsq - (s * (hfsq + R) + dk * ln2_lo)) - f);
    }
    if (k == 0) return f - s * (f - R);
    return dk * ln2_hi - ((s * (f - R) - dk * ln2_lo) - f);
}

/* log1p by Kahan's correction: u = 1+x; log(u) * x / (u-1). */
double rso_log1p(double x)
{
    double u = 1.0 + x;
    if (u == 1.0) return x;
    return rso_log(u) * x / (u - 1.0);
}

/* ------------------------------------------------------------------------- */
/* CANON C5: hypergeometric deviates.  The paper asks for "a constant time   */
/* algorithm for generating hypergeometric random deviates (e.g.             */
/* [Stad90hyp])" and used stocc.  We use  */
/* Stadlober's ratio-of-uniforms HRUA (numpy-legacy operation order) with a  */
/* numerically stable log-PMF ratio (Loader's saddle-point dbinom, as in R's */
/* dhyper), and the sequential-draw HYP for small samples.                   */
/* ------------------------------------------------------------------------- */

/* stirlerr(n) = log(n!) - log(sqrt(2 pi n) (n/e)^n), integer n >= 1.
 * n <= 15: correctly rounded values (pinned vs mpmath in tests).
 * n > 15: Stirling's series 1/(12n) - 1/(360n^3) + 1/(1260n^5)
 * - 1/(1680n^7) + 1/(1188n^9) in powers of rn = 1/n (one division). */
double rso_stirlerr(double n)
{
    static const double ST[16] = {
        0.0,
        0x1.4c071bcda0a5bp-4, 0x1.52a9b923ea649p-5, 0x1.c579a268d80b3p-6,
        0x1.54a2662fd78a9p-6, 0x1.10b4e513fcbedp-6, 0x1.c6b167bebdf36p-7,
        0x1.85d4d612e4a86p-7, 0x1.552805e7b3076p-7, 0x1.2f4871b12ab64p-7,
        0x1.10f9d4c0743a7p-7, 0x1.f0593088014f8p-8, 0x1.c7018733aa9c6p-8,
        0x1.a40514700f36cp-8, 0x1.86076c002d4a7p-8, 0x1.6c08f6f194a10p-8 };
    static const double S0 = 0x1.5555555555555p-4;   /* 1/12   */
    static const double S1 = 0x1.6c16c16c16c17p-9;   /* 1/360  */
    static const double S2 = 0x1.a01a01a01a01ap-11;  /* 1/1260 */
    static const double S3 = 0x1.3813813813814p-11;  /* 1/1680 */
    static const double S4 = 0x1.b951e2b18ff23p-11;  /* 1/1188 */
    if (n <= 15.0) return ST[(int)n];
    double rn = 1.0 / n;
    double r2 = rn * rn;
    return (S0 - (S1 - (S2 - (S3 - S4 * r2) * r2) * r2) * r2) * rn;
}

/* 1/(2j+1), j = 0..23, correctly rounded (the bd0 series coefficients). */
static const double INV_ODD[24] = {
    0x1p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3,
    0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4,
    0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5,
    0x1.47ae147ae147bp-5, 0x1.2f684bda12f68p-5, 0x1.1a7b9611a7b96p-5, 0x1.0842108421084p-5,
    0x1.f07c1f07c1f08p-6, 0x1.d41d41d41d41dp-6, 0x1.bacf914c1bad0p-6, 0x1.a41a41a41a41ap-6,
    0x1.8f9c18f9c18fap-6, 0x1.7d05f417d05f4p-6, 0x1.6c16c16c16c17p-6, 0x1.5c9882b931057p-6 };

/* bd0(x, np) = x log(x/np) + np - x, evaluated without cancellation
 * (Loader 2000): series 2x sum_j v^(2j+1)/(2j+1) - (x-np) in
 * v = (x-np)/(x+np) when |x-np| < 0.1 (x+np). */
double rso_bd0(double x, double np)
{
    if (fabs(x - np) < 0.1 * (x + np)) {
        double v = (x - np) / (x + np);
        double s = (x - np) * v;
        if (fabs(s) < DBL_MIN) return s;
        double ej = 2 * x * v;
        v = v * v;
        for (int j = 1; j < 1000; j++) {
            ej *= v;
            double s1 = s + (j < 24 ? ej * INV_ODD[j] : ej / ((j << 1) + 1));
            if (s1 == s) return s1;
            s = s1;
        }
    }
    return x * rso_log(x / np) + np - x;
}

static const double LN_2PI = 0x1.d67f1c864beb5p+0;   /* log(2 pi) */

/* log of the binomial density b(x; n, p) (Loader's dbinom_raw). */
double rso_ldbinom(double x, double n, double p, double q)
{
    double lc;
    if (x == 0) {
        if (n == 0) return 0.0;
        lc = (p < 0.1) ? -rso_bd0(n, n * q) - n * p : n * rso_log(q);
        return lc;
    }
    if (x == n) {
        lc = (q < 0.1) ? -rso_bd0(n, n * p) - n * q : n * rso_log(p);
        return lc;
    }
    lc = rso_stirlerr(n) - rso_stirlerr(x) - rso_stirlerr(n - x)
         - rso_bd0(x, n * p) - rso_bd0(n - x, n * q);
    double lf = LN_2PI + rso_log(x * (n - x) / n);   /* log(2 pi x (n-x)/n) */
    return lc - 0.5 * lf;
}

/* log P(X = x) + const for X ~ Hypergeom(kp draws, g successes, R total):
 * b(x; g, pp) b(kp-x; R-g, pp) / b(kp; R, pp), denominator dropped. */
static double ldh(u64 x, u64 kp, u64 g, u64 R, double pp, double qq)
{
    return rso_ldbinom((double)x, (double)g, pp, qq)
         + rso_ldbinom((double)(kp - x), (double)(R - g), pp, qq);
}

/* T(K, M) = log f(K) - log f(M), exported for the accuracy pin. */
double rso_hgd_logratio(u64 kp, u64 g, u64 R, u64 K, u64 M)
{
    double pp = (double)kp / (double)R, qq = (double)(R - kp) / (double)R;
    return ldh(K, kp, g, R, pp, qq) - ldh(M, kp, g, R, pp, qq);
}

static const double HRUA_D1 = 0x1.b72cd3f331398p+0;   /* 2 sqrt(2/e)     */
static const double HRUA_D2 = 0x1.cc3ebd3bc711ap-1;   /* 3 - 2 sqrt(3/e) */

/* HYP: simulate the kp draws one by one (exact; numpy hypergeometric_hyp). */
static u64 hyp(u64 kp, u64 g, u64 R, u64 seed, u64 id)
{
    double d1 = (double)(R - kp);
    double Y = (double)g;
    double K = (double)kp;
    u64 s = 0;
    for (;;) {
        double U = stream_u52(seed, PUR_HGD, id, s++);
        Y = Y - floor(U + Y / (d1 + K));
        K = K - 1.0;
        if (Y == 0.0 || K == 0.0) break;
    }
    return g - (u64)Y;
}

/* HRUA: Stadlober's ratio-of-uniforms with the stable log ratio. */
static u64 hrua(u64 kp, u64 g, u64 R, u64 seed, u64 id)
{
    double p = (double)g / (double)R;
    double q = (double)(R - g) / (double)R;
    double a = (double)kp * p + 0.5;
    double var = (double)(R - kp) * (double)kp * p * q / (double)(R - 1);
    double c = sqrt(var + 0.5);
    double h = HRUA_D1 * c + HRUA_D2;
    u64 M = (u64)(((u128)(kp + 1) * (u128)(g + 1)) / (u128)(R + 2));
    double mn = (double)(kp < g ? kp : g) + 1.0;
    double b16 = floor(a + 16 * c);
    double b = mn < b16 ? mn : b16;
    double pp = (double)kp / (double)R, qq = (double)(R - kp) / (double)R;
    double TM = ldh(M, kp, g, R, pp, qq);
    for (u32 t = 0;; t++) {
        u32 w[4];
        block(seed, PUR_HGD, 0, id, t, w);
        double U = rso_u52(w[0], w[1]);
        double V = rso_u52(w[2], w[3]);
        double X = a + h * (V - 0.5) / U;
        if (X < 0.0 || X >= b) continue;
        u64 K = (u64)floor(X);
        double T = ldh(K, kp, g, R, pp, qq) - TM;
        if (U * (4.0 - U) - 3.0 <= T) return K;
        if (U * (U - T) >= 1.0) continue;
        if (2.0 * rso_log(U) <= T) return K;
    }
}

/* X ~ Hypergeom: number of the k drawn items (out of R) that fall among the
 * L "left" items -- "the number of samples L from the left half ... is
 * distributed hypergeometrically with parameters n, l, N". */
u64 rso_hgd(u64 k, u64 L, u64 R, u64 seed, u64 id)
{
    u64 lo = (k + L > R) ? k + L - R : 0;
    u64 hi = k < L ? k : L;
    if (lo == hi) return lo;
    u64 kp = k < R - k ? k : R - k;
    u64 g  = L < R - L ? L : R - L;
    u64 X = (kp < 16) ? hyp(kp, g, R, seed, id) : hrua(kp, g, R, seed, id);
    if (L > R - L) X = kp - X;
    if (kp < k) X = L - X;
    return X;
}

/* ------------------------------------------------------------------------- */
/* CANON C8: binomial deviates for sampling with replacement ("the           */
/* hypergeometric distribution ... has to be replaced by a binomial          */
/* distribution").  BINV (inversion) when k*p' < 10, else BTRS     */
/* (Hoermann 1993) with the same stable log-density ratio.                   */
/* ------------------------------------------------------------------------- */
static double pow_u64(double b, u64 e)
{
    double r = 1.0;
    while (e) { if (e & 1) r *= b; b *= b; e >>= 1; }
    return r;
}

u64 rso_bin(u64 k, u64 L, u64 R, u64 seed, u64 id)
{
    if (k == 0 || L == 0) return 0;
    if (L == R) return k;
    int flip = L > R - L;
    double p = flip ? (double)(R - L) / (double)R : (double)L / (double)R;
    double q = flip ? (double)L / (double)R : (double)(R - L) / (double)R;
    double n = (double)k;
    u64 X;
    if (n * p < 10.0) {
        /* BINV: sequential search of the CDF from 0 (numpy's inversion). */
        double qn = pow_u64(q, k);
        double np = n * p;
        double bound = np + 10.0 * sqrt(np * q + 1.0);
        if (bound > n) bound = n;
        u64 s = 0;
        double x = 0.0, px = qn;
        double U = stream_u52(seed, PUR_BIN, id, s++);
        while (U > px) {
            x = x + 1.0;
            if (x > bound) { x = 0.0; px = qn; U = stream_u52(seed, PUR_BIN, id, s++); }
            else { U -= px; px = ((n - x + 1.0) * p * px) / (x * q); }
        }
        X = (u64)x;
    } else {
        /* BTRS: transformed rejection with squeeze (Hoermann 1993). */
        double spq = sqrt(n * p * q);
        double b = 1.15 + 2.53 * spq;
        double a = -0.0873 + 0.0248 * b + 0.01 * p;
        double c = n * p + 0.5;
        double alpha = (2.83 + 5.1 / b) * spq;
        double vr = 0.92 - 4.2 / b;
        double m = floor((n + 1.0) * p);
        double lm = rso_ldbinom(m, n, p, q);
        for (u32 t = 0;; t++) {
            u32 w[4];
            block(seed, PUR_BIN, 0, id, t, w);
            double U = rso_u52(w[0], w[1]) - 0.5;
            double V = rso_u52(w[2], w[3]);
            double us = 0.5 - fabs(U);
            double kk = floor((2 * a / us + b) * U + c);
            if (kk < 0.0 || kk > n) continue;
            if (us >= 0.07 && V <= vr) { X = (u64)kk; break; }
            double V2 = V * alpha / (a / (us * us) + b);
            if (rso_log(V2) <= rso_ldbinom(kk, n, p, q) - lm) { X = (u64)kk; break; }
        }
    }
    return flip ? k - X : X;
}

/* CANON C9: geometric skip G = floor(log U / log(1 - rho)). */
double rso_geo(double U, double log1m_rho)
{
    return floor(rso_log(U) / log1m_rho);
}

/* ------------------------------------------------------------------------- */
/* CANON C4: the dyadic split tree.  Node (d, i) covers offsets              */
/* [b(d,i), b(d,i+1)), b(d,i) = floor(i N / 2^d); values are offset + 1.     */
/* Fig. 1 splits at floor(N/2); this equals it at the root and   */
/* everywhere for power-of-two N.  All leaves are at depth D.                */
/* ------------------------------------------------------------------------- */
#define N0_DEFAULT 1024u
#define D_MIN 3

static u64 bnd(u64 N, int d, u64 i) { return (u64)(((u128)i * N) >> d); }

void rso_node(u64 N, int d, u64 i, u64 *lo, u64 *R, u64 *L)
{
    *lo = bnd(N, d, i);
    *R = bnd(N, d, i + 1) - *lo;
    *L = bnd(N, d + 1, 2 * i + 1) - *lo;
}

static int ceil_log2(u64 x) { int d = 0; while (d < 64 && ((u64)1 << d) < x) d++; return d; }

/* D = max(D_MIN, ceil(log2(ceil(m / n0)))). */
int rso_depth(u64 m, u64 n0)
{
    u64 t = m / n0 + (m % n0 != 0);
    int d = ceil_log2(t);
    return d < D_MIN ? D_MIN : d;
}

/* Algorithm R (Fig. 1) with a fixed depth: recurse, splitting the count of
 * node (d,i) between its halves with one deviate keyed by its id. */
typedef struct { u64 N, seed; int D; int wr; u64 *cnt; } tree_t;

static void expand(tree_t *t, int d, u64 i, u64 k)
{
    if (d == t->D) { t->cnt[i] = k; return; }
    u64 lo, R, L;
    rso_node(t->N, d, i, &lo, &R, &L);
    u64 id = ((u64)1 << d) + i;
    u64 x = 0;
    if (k > 0) x = t->wr ? rso_bin(k, L, R, t->seed, id) : rso_hgd(k, L, R, t->seed, id);
    expand(t, d + 1, 2 * i, x);
    expand(t, d + 1, 2 * i + 1, k - x);
}

/* Leaf counts of the tree for m samples (WOR: hypergeometric splits; WR:
 * binomial splits) at depth D.  cnt has 2^D entries. */
void rso_tree_counts(u64 N, u64 m, u64 seed, int D, int wr, u64 *cnt)
{
    tree_t t = { N, seed, D, wr, cnt };
    expand(&t, 0, 0, m);
}

/* Algorithm P (Fig. 2) path replay: the count and global offset of node
 * (d, i) from the root path alone -- each PE draws <= ceil(log p) deviates
 * (P:312), no communication. */
void rso_path(u64 N, u64 m, u64 seed, int wr, int d, u64 i, u64 *count, u64 *offset)
{
    u64 k = m, off = 0;
    for (int e = 0; e < d; e++) {
        u64 anc = i >> (d - e);                 /* ancestor at depth e */
        u64 lo, R, L;
        rso_node(N, e, anc, &lo, &R, &L);
        u64 id = ((u64)1 << e) + anc;
        u64 x = 0;
        if (k > 0) x = wr ? rso_bin(k, L, R, seed, id) : rso_hgd(k, L, R, seed, id);
        if ((i >> (d - e - 1)) & 1) { off += x; k -= x; } else { k = x; }
    }
    *count = k; *offset = off;
}

/* ------------------------------------------------------------------------- */
/* Leaves.                                                                   */
/* ------------------------------------------------------------------------- */
static int cmp_u64(const void *a, const void *b)
{
    u64 x = *(const u64 *)a, y = *(const u64 *)b;
    return (x > y) - (x < y);
}

/* CANON C6, Algorithm H: draw uniform deviates from the leaf
 * range, reject those already in the table, until k distinct; then output
 * sorted.  A plain linear-probing set; values are offsets. */
static void leaf_wor(u64 seed, u64 id, u64 r, u64 k, u64 *vals)
{
    if (k == 0) return;
    u64 cap = 2; while (cap < 2 * k) cap <<= 1;
    u64 *tab = (u64 *)malloc(cap * sizeof(u64));
    for (u64 s = 0; s < cap; s++) tab[s] = UINT64_MAX;
    u64 have = 0;
    for (u64 j = 0; have < k; j++) {
        u64 x = rso_draw(seed, PUR_WOR, id, r, j);
        u64 h = (x * 0x9E3779B97F4A7C15ull) & (cap - 1);
        while (tab[h] != UINT64_MAX && tab[h] != x) h = (h + 1) & (cap - 1);
        if (tab[h] == x) continue;                  /* reject duplicate */
        tab[h] = x;
        vals[have++] = x;
    }
    free(tab);
    qsort(vals, k, sizeof(u64), cmp_u64);
}

/* CANON C8 leaf: k independent draws, sorted with multiplicities. */
static void leaf_wr(u64 seed, u64 id, u64 r, u64 k, u64 *vals)
{
    for (u64 j = 0; j < k; j++) vals[j] = rso_draw(seed, PUR_WR, id, r, j);
    qsort(vals, k, sizeof(u64), cmp_u64);
}

/* ------------------------------------------------------------------------- */
/* Whole samples.                                                            */
/* ------------------------------------------------------------------------- */
enum { RSO_OK = 0, RSO_EINVAL = 1, RSO_ENOMEM = 3, RSO_ECAPACITY = 4 };
enum { MODE_WOR = 0, MODE_WR = 1 };

typedef struct {
    u64 N, seed; int D; int mode; int complement;
    const u64 *cnt, *off;    /* core-tree leaf counts and exclusive offsets */
    u64 *out;                /* NULL: digest only */
    u64 leaf_lo, leaf_hi, next;
    pthread_mutex_t mu;
    u64 digest;
} job_t;

static u64 mix64(u64 z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Order-sensitive, shard-composable digest: sum_i mix64(i ^ mix64(v_i)). */
u64 rso_digest(const u64 *v, u64 count, u64 base_index)
{
    u64 h = 0;
    for (u64 i = 0; i < count; i++) h += mix64((base_index + i) ^ mix64(v[i]));
    return h;
}

/* Values of output leaf i (the values of the final sample lying in
 * [b(D,i), b(D,i+1))), their count and global output offset. */
static u64 leaf_output(u64 N, u64 seed, int D, int mode, int complement,
                       u64 i, u64 k, u64 core_off, u64 *buf, u64 *out_off)
{
    u64 lo, R, L;
    rso_node(N, D, i, &lo, &R, &L);
    u64 id = ((u64)1 << D) + i;
    if (!complement) {
        if (mode == MODE_WR) leaf_wr(seed, id, R, k, buf);
        else leaf_wor(seed, id, R, k, buf);
        for (u64 t = 0; t < k; t++) buf[t] += lo + 1;
        *out_off = core_off;
        return k;
    }
    /* complement: [lo, lo+R) minus the core leaf's k values */
    u64 *ex = (u64 *)malloc((k + 1) * sizeof(u64));
    leaf_wor(seed, id, R, k, ex);
    u64 c = 0, e = 0;
    for (u64 x = 0; x < R; x++) {
        if (e < k && ex[e] == x) { e++; continue; }
        buf[c++] = lo + x + 1;
    }
    free(ex);
    *out_off = lo - core_off;
    return c;
}

static void *worker(void *arg)
{
    job_t *J = (job_t *)arg;
    u64 bufcap = 0; u64 *buf = NULL; u64 dig = 0;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        u64 i = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (i >= J->leaf_hi) break;
        u64 lo, R, L;
        rso_node(J->N, J->D, i, &lo, &R, &L);
        u64 need = J->complement ? R : J->cnt[i];
        if (need + 1 > bufcap) { free(buf); bufcap = need + 1; buf = (u64 *)malloc(bufcap * sizeof(u64)); }
        u64 off;
        u64 c = leaf_output(J->N, J->seed, J->D, J->mode, J->complement,
                            i, J->cnt[i], J->off[i], buf, &off);
        if (J->out) memcpy(J->out + off, buf, c * sizeof(u64));
        else dig += rso_digest(buf, c, off);
    }
    free(buf);
    pthread_mutex_lock(&J->mu); J->digest += dig; pthread_mutex_unlock(&J->mu);
    return NULL;
}

static void run_leaves(job_t *J, int nthreads)
{
    if (nthreads < 1) nthreads = 1;
    pthread_mutex_init(&J->mu, NULL);
    J->next = J->leaf_lo;
    pthread_t th[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, worker, J);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&J->mu);
}

/* Common driver: build the core tree, then fill (or digest) leaves
 * [leaf_lo, leaf_hi).  Returns RSO_* status. */
static int drive(u64 N, u64 n, u64 seed, int mode, u64 *out, int nthreads,
                 u64 leaf_lo, u64 leaf_hi, u64 *digest, int *Dout)
{
    if (mode == MODE_WOR && n > N) return RSO_EINVAL;
    if (mode == MODE_WR && N == 0 && n > 0) return RSO_EINVAL;
    if (N >= ((u64)1 << 63)) return RSO_EINVAL;
    if (n >= ((u64)1 << 40)) return RSO_EINVAL;
    int complement = (mode == MODE_WOR) && (n > N - n);   /* CANON C7: 2n > N */
    u64 m = complement ? N - n : n;
    int D = rso_depth(m, N0_DEFAULT);
    if (Dout) *Dout = D;
    if (n == 0 && !complement) { if (digest) *digest = 0; return RSO_OK; }
    u64 nleaves = (u64)1 << D;
    u64 *cnt = (u64 *)malloc(nleaves * sizeof(u64));
    u64 *off = (u64 *)malloc(nleaves * sizeof(u64));
    if (!cnt || !off) { free(cnt); free(off); return RSO_ENOMEM; }
    rso_tree_counts(N, m, seed, D, mode == MODE_WR, cnt);
    u64 acc = 0;
    for (u64 i = 0; i < nleaves; i++) { off[i] = acc; acc += cnt[i]; }
    job_t J;
    memset(&J, 0, sizeof J);
    J.N = N; J.seed = seed; J.D = D; J.mode = mode; J.complement = complement;
    J.cnt = cnt; J.off = off; J.out = out;
    J.leaf_lo = leaf_lo < nleaves ? leaf_lo : nleaves;
    J.leaf_hi = leaf_hi < nleaves ? leaf_hi : nleaves;
    run_leaves(&J, nthreads);
    if (digest) *digest = J.digest;
    free(cnt); free(off);
    return RSO_OK;
}

/* rs_sample_wor's definition: n distinct values of 1..N, ascending. */
int rso_sample_wor(u64 N, u64 n, u64 seed, u64 *out, int nthreads)
{
    return drive(N, n, seed, MODE_WOR, out, nthreads, 0, UINT64_MAX, NULL, NULL);
}

/* rs_sample_wr's definition: n values of 1..N with repeats, ascending. */
int rso_sample_wr(u64 N, u64 n, u64 seed, u64 *out, int nthreads)
{
    return drive(N, n, seed, MODE_WR, out, nthreads, 0, UINT64_MAX, NULL, NULL);
}

/* Digest of the output restricted to leaves [leaf_lo, leaf_hi) -- the
 * streaming mode used for outputs too large to materialise on the host. */
int rso_digest_range(u64 N, u64 n, u64 seed, int mode, int nthreads,
                     u64 leaf_lo, u64 leaf_hi, u64 *digest)
{
    return drive(N, n, seed, mode, NULL, nthreads, leaf_lo, leaf_hi, digest, NULL);
}

/* Depth and complement decision used for n of N (mode 0 WOR / 1 WR). */
int rso_plan(u64 N, u64 n, int mode, int *D, int *complement, u64 *m)
{
    int c = (mode == MODE_WOR) && (n > N - n);
    *complement = c;
    *m = c ? N - n : n;
    *D = rso_depth(*m, N0_DEFAULT);
    return RSO_OK;
}

/* One output leaf by path replay (D deviates): the sampled-parity check
 * at full sizes.  buf must hold R(leaf) (complement) or count values. */
int rso_leaf(u64 N, u64 n, u64 seed, int mode, u64 leaf, u64 *buf, u64 *count, u64 *offset)
{
    int D, comp; u64 m;
    rso_plan(N, n, mode, &D, &comp, &m);
    if (leaf >= ((u64)1 << D)) return RSO_EINVAL;
    u64 k, off;
    rso_path(N, m, seed, mode == MODE_WR, D, leaf, &k, &off);
    *count = leaf_output(N, seed, D, mode, comp, leaf, k, off, buf, offset);
    return RSO_OK;
}

/* Size of output leaf `leaf` without generating it (for buffer sizing). */
int rso_leaf_size(u64 N, u64 n, u64 seed, int mode, u64 leaf, u64 *count, u64 *range)
{
    int D, comp; u64 m;
    rso_plan(N, n, mode, &D, &comp, &m);
    if (leaf >= ((u64)1 << D)) return RSO_EINVAL;
    u64 k, off, lo, R, L;
    rso_path(N, m, seed, mode == MODE_WR, D, leaf, &k, &off);
    rso_node(N, D, leaf, &lo, &R, &L);
    *count = comp ? R - k : k;
    *range = R;
    return RSO_OK;
}

/* ------------------------------------------------------------------------- */
/* CANON C9: Bernoulli sampling by geometric skips over dyadic chunks       */
/* ("independently apply Bernoulli sampling to subranges";       */
/* skips).                                                        */
/* ------------------------------------------------------------------------- */
int rso_bern_depth(u64 N, double rho)
{
    double t = ceil((double)N * rho / (double)N0_DEFAULT);
    u64 tt = t < 1.0 ? 1 : (t >= 0x1p62 ? ((u64)1 << 62) : (u64)t);
    int d = ceil_log2(tt);
    return d < D_MIN ? D_MIN : d;
}

/* Chunk i at depth Db: emits values into buf (NULL: count only). */
static u64 bern_chunk(u64 N, u64 seed, int Db, u64 i, double lr, u64 *buf)
{
    u64 lo, R, L;
    rso_node(N, Db, i, &lo, &R, &L);
    u64 hi = lo + R, pos = lo, c = 0;
    u64 id = ((u64)1 << Db) + i;
    for (u64 j = 0;; j++) {
        double U = stream_u52(seed, PUR_GEO, id, j);
        double G = rso_geo(U, lr);
        if (G >= 0x1p63) break;
        u64 g = (u64)G;
        if (g >= hi - pos) break;
        pos += g;
        if (buf) buf[c] = pos + 1;
        c++;
        pos += 1;
    }
    return c;
}

int rso_bernoulli(u64 N, double rho, u64 seed, u64 *out, u64 capacity, u64 *count)
{
    if (!(rho >= 0.0 && rho <= 1.0)) return RSO_EINVAL;
    if (N >= ((u64)1 << 63)) return RSO_EINVAL;
    if (rho == 0.0 || N == 0) { *count = 0; return RSO_OK; }
    if (rho == 1.0) {
        for (u64 v = 0; v < N && v < capacity; v++) out[v] = v + 1;
        *count = N;
        return N > capacity ? RSO_ECAPACITY : RSO_OK;
    }
    int Db = rso_bern_depth(N, rho);
    double lr = rso_log1p(-rho);
    u64 total = 0;
    u64 nch = (u64)1 << Db;
    u64 *tmp = NULL; u64 tmpcap = 0;
    for (u64 i = 0; i < nch; i++) {
        u64 c = bern_chunk(N, seed, Db, i, lr, NULL);
        if (c > tmpcap) { free(tmp); tmpcap = c; tmp = (u64 *)malloc(c * sizeof(u64)); }
        bern_chunk(N, seed, Db, i, lr, tmp);
        for (u64 t = 0; t < c; t++) if (total + t < capacity) out[total + t] = tmp[t];
        total += c;
    }
    free(tmp);
    *count = total;
    return total > capacity ? RSO_ECAPACITY : RSO_OK;
}

/* Count (and optionally values) of one Bernoulli chunk. */
u64 rso_bern_chunk(u64 N, double rho, u64 seed, u64 chunk, u64 *buf)
{
    int Db = rso_bern_depth(N, rho);
    return bern_chunk(N, seed, Db, chunk, rso_log1p(-rho), buf);
}

/* ------------------------------------------------------------------------- */
/* Sharding (Algorithm P): rank g of p = 2^s owns node (s, g).    */
/* ------------------------------------------------------------------------- */
int rso_shard_info(u64 N, u64 n, u64 seed, int mode, int world, int rank,
                   u64 *local_count, u64 *global_offset)
{
    int s = 0; while ((1 << s) < world) s++;
    if ((1 << s) != world || rank < 0 || rank >= world || s > D_MIN) return RSO_EINVAL;
    int D, comp; u64 m;
    rso_plan(N, n, mode, &D, &comp, &m);
    u64 k, off;
    rso_path(N, m, seed, mode == MODE_WR, s, (u64)rank, &k, &off);
    if (comp) {
        u64 lo, R, L;
        rso_node(N, s, (u64)rank, &lo, &R, &L);
        *local_count = R - k;
        *global_offset = lo - off;
    } else {
        *local_count = k;
        *global_offset = off;
    }
    return RSO_OK;
}

/* ------------------------------------------------------------------------- */
/* Test hooks (batch loops so the statistical pins run in seconds).          */
/* ------------------------------------------------------------------------- */
/* Exhaustive: hist[v] += 1 for every accepted word (all 2^32 words). */
u64 rso_lemire32_hist(u64 r, u32 *hist)
{
    u64 acc = 0, v;
    for (u64 w = 0; w <= 0xffffffffull; w++)
        if (rso_lemire32((u32)w, r, &v)) { hist[v]++; acc++; }
    return acc;
}

/* Every word w in [w_lo, w_hi) through rso_lemire64: out[0] = accepted words
 * whose value is v, out[1] = accepted words with any other value, out[2] =
 * rejected words.  The caller computes the preimage interval of v with exact
 * integers (tests/test_oracle_primitives.py). */
void rso_lemire64_scan(u64 r, u64 v, u64 w_lo, u64 w_hi, u64 out[3])
{
    out[0] = out[1] = out[2] = 0;
    for (u64 w = w_lo; w != w_hi; w++) {
        u64 x;
        if (rso_lemire64(w, r, &x)) { if (x == v) out[0]++; else out[1]++; }
        else out[2]++;
    }
}

/* count deviates with node ids id0, id0+1, ... */
void rso_hgd_batch(u64 k, u64 L, u64 R, u64 seed, u64 id0, u64 count, u64 *out)
{
    for (u64 t = 0; t < count; t++) out[t] = rso_hgd(k, L, R, seed, id0 + t);
}

void rso_bin_batch(u64 k, u64 L, u64 R, u64 seed, u64 id0, u64 count, u64 *out)
{
    for (u64 t = 0; t < count; t++) out[t] = rso_bin(k, L, R, seed, id0 + t);
}

/* Subset frequencies for tiny N: for seeds s0..s0+count-1, the bitmask of
 * the sample (N <= 63), mode 0 WOR; WR returns the sorted values packed 8
 * bits each (n <= 8). */
void rso_small_samples(u64 N, u64 n, u64 s0, u64 count, int mode, u64 *out)
{
    u64 buf[64];
    for (u64 t = 0; t < count; t++) {
        if (mode == MODE_WR) {
            rso_sample_wr(N, n, s0 + t, buf, 1);
            u64 code = 0;
            for (u64 j = 0; j < n; j++) code |= buf[j] << (8 * j);
            out[t] = code;
        } else {
            rso_sample_wor(N, n, s0 + t, buf, 1);
            u64 mask = 0;
            for (u64 j = 0; j < n; j++) mask |= (u64)1 << (buf[j] - 1);
            out[t] = mask;
        }
    }
}

/* Bounded-sample mode for the CPU baseline: output leaves [leaf_lo, leaf_hi)
 * each found by path replay (no full tree), digested; nthreads workers.
 * Returns the number of values produced in *values. */
typedef struct {
    u64 N, n, seed; int mode;
    u64 next, hi; pthread_mutex_t mu;
    u64 digest, values;
} rjob_t;

static void *rworker(void *arg)
{
    rjob_t *J = (rjob_t *)arg;
    int D, comp; u64 m;
    rso_plan(J->N, J->n, J->mode, &D, &comp, &m);
    u64 *buf = NULL, cap = 0, dig = 0, vals = 0;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        u64 i = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (i >= J->hi) break;
        u64 k, off, lo, R, L;
        rso_path(J->N, m, J->seed, J->mode == MODE_WR, D, i, &k, &off);
        rso_node(J->N, D, i, &lo, &R, &L);
        u64 need = (comp ? R : k) + 1;
        if (need > cap) { free(buf); cap = need; buf = (u64 *)malloc(cap * sizeof(u64)); }
        u64 o;
        u64 c = leaf_output(J->N, J->seed, D, J->mode, comp, i, k, off, buf, &o);
        dig += rso_digest(buf, c, o);
        vals += c;
    }
    free(buf);
    pthread_mutex_lock(&J->mu); J->digest += dig; J->values += vals; pthread_mutex_unlock(&J->mu);
    return NULL;
}

int rso_digest_leaves_replay(u64 N, u64 n, u64 seed, int mode, int nthreads,
                             u64 leaf_lo, u64 leaf_hi, u64 *digest, u64 *values)
{
    int D, comp; u64 m;
    if (mode == MODE_WOR && n > N) return RSO_EINVAL;
    rso_plan(N, n, mode, &D, &comp, &m);
    u64 nl = (u64)1 << D;
    rjob_t J;
    memset(&J, 0, sizeof J);
    J.N = N; J.n = n; J.seed = seed; J.mode = mode;
    J.next = leaf_lo < nl ? leaf_lo : nl;
    J.hi = leaf_hi < nl ? leaf_hi : nl;
    pthread_mutex_init(&J.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, rworker, &J);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&J.mu);
    *digest = J.digest;
    *values = J.values;
    return RSO_OK;
}

/* Bounded-sample Bernoulli: chunks [c_lo, c_hi), digest + count. */
int rso_bern_chunks_digest(u64 N, double rho, u64 seed, u64 c_lo, u64 c_hi, u64 *digest, u64 *values)
{
    int Db = rso_bern_depth(N, rho);
    double lr = rso_log1p(-rho);
    u64 *buf = NULL, cap = 0, dig = 0, vals = 0;
    for (u64 i = c_lo; i < c_hi && i < ((u64)1 << Db); i++) {
        u64 c = bern_chunk(N, seed, Db, i, lr, NULL);
        if (c + 1 > cap) { free(buf); cap = c + 1; buf = (u64 *)malloc(cap * sizeof(u64)); }
        bern_chunk(N, seed, Db, i, lr, buf);
        dig += rso_digest(buf, c, vals);
        vals += c;
    }
    free(buf);
    *digest = dig; *values = vals;
    return RSO_OK;
}

/* The same over chunks [c_lo, c_hi) with nthreads workers, in two passes
 * (counts, then digests at the prefix offsets): the whole-output parity of
 * the roofline-sized Bernoulli run.  Threads only split independent chunks;
 * each chunk is bern_chunk above. */
typedef struct {
    u64 N, seed; int Db; double lr;
    u64 c_lo, c_hi, next; pthread_mutex_t mu;
    u64 *cnt;                 /* per-chunk counts (pass 1) / offsets (pass 2) */
    int pass; u64 digest;
} bjob_t;

static void *bworker(void *arg)
{
    bjob_t *J = (bjob_t *)arg;
    u64 *buf = NULL, cap = 0, dig = 0;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        u64 i0 = J->next; J->next += 64;
        pthread_mutex_unlock(&J->mu);
        if (i0 >= J->c_hi) break;
        for (u64 i = i0; i < i0 + 64 && i < J->c_hi; i++) {
            if (J->pass == 1) { J->cnt[i - J->c_lo] = bern_chunk(J->N, J->seed, J->Db, i, J->lr, NULL); continue; }
            u64 c = bern_chunk(J->N, J->seed, J->Db, i, J->lr, NULL);
            if (c + 1 > cap) { free(buf); cap = c + 1; buf = (u64 *)malloc(cap * sizeof(u64)); }
            bern_chunk(J->N, J->seed, J->Db, i, J->lr, buf);
            dig += rso_digest(buf, c, J->cnt[i - J->c_lo]);
        }
    }
    free(buf);
    pthread_mutex_lock(&J->mu); J->digest += dig; pthread_mutex_unlock(&J->mu);
    return NULL;
}

int rso_bern_chunks_digest_mt(u64 N, double rho, u64 seed, int nthreads, u64 c_lo, u64 c_hi,
                              u64 *digest, u64 *values)
{
    if (!(rho > 0.0 && rho < 1.0)) return RSO_EINVAL;
    bjob_t J;
    memset(&J, 0, sizeof J);
    J.N = N; J.seed = seed; J.Db = rso_bern_depth(N, rho); J.lr = rso_log1p(-rho);
    u64 nch = (u64)1 << J.Db;
    J.c_lo = c_lo < nch ? c_lo : nch;
    J.c_hi = c_hi < nch ? c_hi : nch;
    if (J.c_hi < J.c_lo) J.c_hi = J.c_lo;
    J.cnt = (u64 *)malloc((J.c_hi - J.c_lo + 1) * sizeof(u64));
    if (!J.cnt) return RSO_ENOMEM;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_mutex_init(&J.mu, NULL);
    pthread_t th[256];
    for (J.pass = 1; J.pass <= 2; J.pass++) {
        J.next = J.c_lo;
        for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, bworker, &J);
        for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
        if (J.pass == 1) {                  /* exclusive prefix: offsets */
            u64 acc = 0;
            for (u64 i = 0; i < J.c_hi - J.c_lo; i++) { u64 c = J.cnt[i]; J.cnt[i] = acc; acc += c; }
            *values = acc;
        }
    }
    pthread_mutex_destroy(&J.mu);
    free(J.cnt);
    *digest = J.digest;
    return RSO_OK;
}

/* ------------------------------------------------------------------------
 * NEXT-2: uneven universe (Section 4.3).  PE i owns L[i]
 * elements.  "Arrange the processors into a binomial tree ... At level j we
 * get (maximal) subtrees spanning processors 2^j a .. min(2^j a + 2^j - 1,
 * p - 1)"; the L-values are summed bottom-up and the n samples are split
 * top-down: "an inner node uses a hypergeometric distribution with
 * parameters n [read: its n'], L_l and L_l + L_r to split its n' samples".
 * "The subtree representing processors a..b can use this range as an input
 * for the hash function h": the deviate of the level-j subtree a is keyed
 * by its heap index 2^(J-j) + a (J = ceil log2 p) with bit 62 set (DESIGN
 * R13: disjoint from every node id of the sampling tree).  A subtree whose
 * right half is empty passes n' to the left without a deviate.  Written
 * recursively, exactly as the paper's top-down pass. */
static u64 sum_range(const u64 *L, int lo, int hi)
{
    u64 s = 0;
    for (int i = lo; i < hi; i++) s += L[i];
    return s;
}

static void uneven_rec(int p, int J, int j, u64 a, u64 nprime, const u64 *L, u64 seed, u64 *counts)
{
    const u64 lo = a << j;
    if (j == 0) { counts[lo] = nprime; return; }
    const u64 mid = lo + ((u64)1 << (j - 1));
    if (mid >= (u64)p) { uneven_rec(p, J, j - 1, 2 * a, nprime, L, seed, counts); return; }
    const u64 hi = lo + ((u64)1 << j) < (u64)p ? lo + ((u64)1 << j) : (u64)p;
    const u64 Ll = sum_range(L, (int)lo, (int)mid), Lr = sum_range(L, (int)mid, (int)hi);
    const u64 id = ((u64)1 << 62) | (((u64)1 << (J - j)) + a);
    const u64 x = nprime == 0 ? 0 : rso_hgd(nprime, Ll, Ll + Lr, seed, id);
    uneven_rec(p, J, j - 1, 2 * a, x, L, seed, counts);
    uneven_rec(p, J, j - 1, 2 * a + 1, nprime - x, L, seed, counts);
}

/* counts[0..p) of the n samples; -1 if p < 1, n > sum L or sum L >= 2^63. */
int rso_uneven_counts(int p, const u64 *L, u64 n, u64 seed, u64 *counts)
{
    if (p < 1) return -1;
    u64 tot = 0;
    for (int i = 0; i < p; i++) {
        if (L[i] >= ((u64)1 << 63) - tot) return -1;
        tot += L[i];
    }
    if (n > tot) return -1;
    int J = 0;
    while (((u64)1 << J) < (u64)p) J++;
    uneven_rec(p, J, J, 0, n, L, seed, counts);
    return 0;
}

/* Seed of PE i's local sample (DESIGN R13): mix64(seed + golden * (i + 1)). */
u64 rso_uneven_seed(u64 seed, u64 i)
{
    return mix64(seed + 0x9E3779B97F4A7C15ull * (i + 1));
}

/* NEXT-3: edge index e (0-based, lexicographic over pairs u < v of
 * 0..V-1; row u holds V-1-u edges) -> (u << 32) | v.  The plain definition:
 * u = the largest row with S(u) = u(2V-u-1)/2 <= e, by integer binary search
 * (the SPEC's method), v = e - S(u) + u + 1.  Applied to a 1-based
 * sample over 1..V(V-1)/2 in place of values[i] - 1. */
static unsigned __int128 edge_row_start(u64 V, u64 u)
{
    return (unsigned __int128)u * (2 * (unsigned __int128)V - u - 1) / 2;
}

void rso_edges(u64 V, const u64 *values, u64 count, u64 *out)
{
    for (u64 i = 0; i < count; i++) {
        const u64 e = values[i] - 1;
        u64 lo = 0, hi = V - 2;                  /* largest u in [lo, hi] with S(u) <= e */
        while (lo < hi) {
            const u64 mid = lo + (hi - lo + 1) / 2;
            if (edge_row_start(V, mid) <= e) lo = mid; else hi = mid - 1;
        }
        const u64 v = (u64)(e - edge_row_start(V, lo)) + lo + 1;
        out[i] = (lo << 32) | v;
    }
}

/* NEXT-4: Algorithm B with repair (the paper's GPU variant
 * P:621-637), the comparison baseline.  Step by step:
 *   rho' = min(1, (n + slack*sqrt(n)) / N)        ("rho somewhat larger than
 *          n/N"; reading R14: slack standard deviations)
 *   for attempt a = 0, 1, ...: seed_a = seed + a*0x9E3779B97F4A7C15 (mod 2^64)
 *     S = Bernoulli(N, rho', seed_a) (rso_bernoulli), n' = |S|
 *     if n' >= n stop, else restart ("simply restart")
 *   R = the WOR sample of n' - n positions from 1..n' with seed_a
 *       (rso_sample_wor; "Algorithm R to generate n'-n samples from the range
 *       0..n'-1", P:630-632 -- 1-based here)
 *   out = S without the elements at positions R ("marks the appropriate
 *       positions ... for removal ... compacted").
 * Returns 0, RSO_EINVAL for n > N or a bad slack, -2 past max_attempts. */
int rso_algb(u64 N, u64 n, u64 seed, double slack, u64 *out, u32 max_attempts, u32 *attempts)
{
    if (n > N || !(slack >= 0.0 && slack < 1e300) || N >= ((u64)1 << 63)) return RSO_EINVAL;
    *attempts = 0;
    if (n == 0) return RSO_OK;
    double rho = ((double)n + slack * sqrt((double)n)) / (double)N;
    if (rho > 1.0) rho = 1.0;
    for (u32 a = 0; a < max_attempts; a++) {
        const u64 sa = seed + 0x9E3779B97F4A7C15ull * (u64)a;
        u64 np = 0;
        int st = rso_bernoulli(N, rho, sa, NULL, 0, &np);     /* count only */
        if (st != RSO_OK && st != RSO_ECAPACITY) return st;
        *attempts = a + 1;
        if (np < n) continue;
        u64 *S = (u64 *)malloc((np ? np : 1) * sizeof(u64));
        u64 *R = (u64 *)malloc((np - n ? np - n : 1) * sizeof(u64));
        u64 c2 = 0;
        rso_bernoulli(N, rho, sa, S, np, &c2);
        st = rso_sample_wor(np, np - n, sa, R, 1);
        u64 o = 0, t = 0;
        for (u64 i = 0; i < np; i++) {               /* position i + 1 removed? */
            if (t < np - n && R[t] == i + 1) { t++; continue; }
            out[o++] = S[i];
        }
        free(S); free(R);
        return (st == 0 && c2 == np && o == n && t == np - n) ? RSO_OK : RSO_EINVAL;
    }
    return -2;
}
