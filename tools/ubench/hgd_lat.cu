// Latency of the split tree's deviate pieces on one warp (clock64), sm_100a.
// Dev tool: explains the top CTA's per-level time.
#include <cstdio>
#include "../../paper_1610_05141_b200/csrc/rs_math.cuh"
using namespace rs;

__global__ void k_lat(u64 *out, long long *cyc, double xin)
{
    const u64 k = 1ull << 32, L = 1ull << 47, R = 1ull << 48;
    long long t0, t1;
    double acc = 0;
    u64 X = 0;
    // 1. one IEEE fp64 division chain
    t0 = clock64();
    double d = xin;
    for (int i = 0; i < 16; ++i) d = 1.0 / (d + 1.0);
    t1 = clock64(); cyc[0] = (t1 - t0) / 16; acc += d;
    // 2. log_
    t0 = clock64();
    d = xin;
    for (int i = 0; i < 16; ++i) d = log_(d + 2.0);
    t1 = clock64(); cyc[1] = (t1 - t0) / 16; acc += d;
    // 3. stirlerr
    t0 = clock64();
    d = 1e9;
    for (int i = 0; i < 16; ++i) d = 1e9 + stirlerr(d) * 1e3;
    t1 = clock64(); cyc[2] = (t1 - t0) / 16; acc += d;
    // 4. log_dbinom
    t0 = clock64();
    d = 0;
    for (int i = 0; i < 16; ++i) d += log_dbinom(2147483648.0 + (double)(i + (d > 1e300)), 4294967296.0, 0.5, 0.5, 0.0);
    t1 = clock64(); cyc[3] = (t1 - t0) / 16; acc += d;
    // 4b. log_dbinom_w (straight-line form used by hgd_tp), lane-varying x
    t0 = clock64();
    d = 0;
    for (int i = 0; i < 16; ++i) d += log_dbinom_w(536870912.0 + (double)(threadIdx.x * 977 + i + (d > 1e300)), 1073741824.0, 0.5, 0.5, 0.0);
    t1 = clock64(); cyc[8] = (t1 - t0) / 16; acc += d;
    // 4c. log_dbinom, the same lane-varying x
    t0 = clock64();
    d = 0;
    for (int i = 0; i < 16; ++i) d += log_dbinom(536870912.0 + (double)(threadIdx.x * 977 + i + (d > 1e300)), 1073741824.0, 0.5, 0.5, 0.0);
    t1 = clock64(); cyc[9] = (t1 - t0) / 16; acc += d;
    // 4d. bd0_w / 4e. stirlerr_w chains
    t0 = clock64();
    d = 0;
    for (int i = 0; i < 16; ++i) { bool sl = false; d += bd0_w(536870912.0 + (double)(threadIdx.x * 977 + i + (d > 1e300)), 536870912.0, sl); }
    t1 = clock64(); cyc[10] = (t1 - t0) / 16; acc += d;
    t0 = clock64();
    d = 1e9;
    for (int i = 0; i < 16; ++i) { bool sl = false; d = 1e9 + stirlerr_w(d, sl) * 1e3; }
    t1 = clock64(); cyc[11] = (t1 - t0) / 16; acc += d;
    // 5. whole hgd (thread)
    t0 = clock64();
    for (int i = 0; i < 8; ++i) X += hgd(k, L, R, 1 + X % 3, 1 + i);
    t1 = clock64(); cyc[4] = (t1 - t0) / 8;
    // 6. hgd_grp<32>
    t0 = clock64();
    for (int i = 0; i < 8; ++i) X += hgd_tp(k, L, R, 1 + X % 3, 1 + i);
    t1 = clock64(); cyc[5] = (t1 - t0) / 8;
    // 6b. hgd_tp on cfg0-shaped nodes (k = 2^20 >> l, R = 2^30 >> l)
    t0 = clock64();
    for (int l = 0; l < 10; ++l) X += hgd_tp((1ull << 20) >> l, (1ull << 29) >> l, (1ull << 30) >> l, 1 + X % 3, (1ull << l));
    t1 = clock64(); cyc[7] = (t1 - t0) / 10;
    // 7. hrua_setup
    t0 = clock64();
    Hrua s;
    for (int i = 0; i < 8; ++i) { s = hrua_setup(k + (X & 1) + i, L, R); X += (u64)s.TM; }
    t1 = clock64(); cyc[6] = (t1 - t0) / 8;
    if (threadIdx.x == 0) out[0] = X + (u64)acc;
}


__device__ long long g_ph[8];
__device__ __noinline__ u64 hgd_tp_timed(u64 k, u64 L, u64 R, u64 seed, u64 node_id)
{
    long long t0 = clock64();
    const u64 kp = (R - k) < k ? R - k : k;
    const u64 g = (R - L) < L ? R - L : L;
    const Stream st(seed, P_HGD, node_id);
    const u32 lane = threadIdx.x & 31;
    const double p = (double)g / (double)R;
    const double q = (double)(R - g) / (double)R;
    const double a = (double)kp * p + 0.5;
    const double var = (double)(R - kp) * (double)kp * p * q / (double)(R - 1);
    const double c = sqrt_(var + 0.5);
    const double h = 0x1.b72cd3f331398p+0 * c + 0x1.cc3ebd3bc711ap-1;
    const unsigned __int128 num = (unsigned __int128)(kp + 1) * (unsigned __int128)(g + 1);
    const u64 den = R + 2;
    u64 M = (u64)(((double)(kp + 1) * (double)(g + 1)) / (double)den);
    while ((unsigned __int128)M * den > num) --M;
    while ((unsigned __int128)(M + 1) * den <= num) ++M;
    const double cap = (double)(kp < g ? kp : g) + 1.0;
    const double tail = floor_(a + 16 * c);
    const double b = cap < tail ? cap : tail;
    long long t1 = clock64();
    const HgdCore core{kp, g, R, (double)kp / (double)R, (double)(R - kp) / (double)R,
                       stirlerr((double)g), stirlerr((double)(R - g))};
    long long t2 = clock64();
    const u32 first = 2u;
    const bool mode_lane = lane < first;
    const u32 j = mode_lane ? 0u : (lane - first) >> 1, half = (lane - first) & 1;
    const u32x4 w = st.block(j);
    const double U = u52(w.x, w.y), V = u52(w.z, w.w);
    const double Xc = a + h * (V - 0.5) / U;
    const bool inb = !(Xc < 0.0 || Xc >= b);
    const u64 K = mode_lane ? M : (inb ? (u64)floor_(Xc) : M);
    long long t3 = clock64();
    const u32 hh = mode_lane ? lane : half;
    const double val = log_dbinom_w(hh == 0 ? (double)K : (double)(kp - K), hh == 0 ? (double)g : (double)(R - g),
                                    core.pp, core.qq, hh == 0 ? core.sg : core.sr);
    long long t4 = clock64();
    bool slu = false; const double lu = log_w(U, slu);
    long long t5 = clock64();
    const double TM = __shfl_sync(0xffffffffu, val, 0) + __shfl_sync(0xffffffffu, val, 1);
    const double d1 = __shfl_down_sync(0xffffffffu, val, 1);
    bool acc = false;
    if (!mode_lane && half == 0 && inb) {
        const double T = val + d1 - TM;
        if (U * (4.0 - U) - 3.0 <= T) acc = true;
        else if (!(U * (U - T) >= 1.0)) acc = 2.0 * lu <= T;
    }
    const u32 am = __ballot_sync(0xffffffffu, acc);
    u64 X = am ? __shfl_sync(0xffffffffu, K, __ffs(am) - 1) : 0;
    long long t6 = clock64();
    if (lane == 0) { g_ph[0] = t1 - t0; g_ph[1] = t2 - t1; g_ph[2] = t3 - t2; g_ph[3] = t4 - t3; g_ph[4] = t5 - t4; g_ph[5] = t6 - t5; }
    return X;
}
__global__ void k_phases(u64 *out)
{
    u64 X = 0;
    for (int i = 0; i < 4; ++i) X += hgd_tp_timed(1ull << 20, 1ull << 29, 1ull << 30, 1 + i, 1 + i);
    if (threadIdx.x == 0) out[0] = X;
}

// log_w == log_ bit for bit (NaNs: both NaN) over random bit patterns (every
// class: negative, zero, subnormal, inf, nan) and values near 1 / powers of 2
__device__ unsigned long long g_bad, g_tot, g_slow;
__global__ void k_logcheck(u64 seed)
{
    const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    u64 z = (i + seed) * 0x9E3779B97F4A7C15ull;
    z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 29;
    double xs[6];
    xs[0] = __longlong_as_double((long long)z);                            // any bit pattern
    xs[1] = 1.0 + (double)(long long)(z >> 40) * 0x1p-40;                  // near 1
    xs[2] = __longlong_as_double((long long)(z & 0x000fffffffffffffull));  // subnormal / zero
    xs[3] = ldexp(1.0 + (double)(z >> 44) * 0x1p-20, (int)(z & 63) - 32); // ~powers of two
    xs[4] = (double)(z >> 11) * 0x1p-53;                                   // u52-style uniforms
    xs[5] = (double)(z & 0xffffffffull) / (double)((z >> 32) | 1);         // ratios
    unsigned bad = 0, nslow = 0;
    for (int t = 0; t < 6; ++t) {
        bool slow = false;
        const double a = log_w(xs[t], slow), b = log_(xs[t]);
        const bool same = (a != a && b != b) || __double_as_longlong(a) == __double_as_longlong(b);
        bad += !slow && !same;
        nslow += slow;
    }
    // ddiv_w against the IEEE division (fast cases must agree bit for bit)
    for (int t = 0; t < 6; ++t) {
        bool slow = false;
        const double b = xs[(t + 1) % 6], q = ddiv_w(xs[t], b, slow), r = xs[t] / b;
        const bool same = (q != q && r != r) || __double_as_longlong(q) == __double_as_longlong(r);
        bad += !slow && !same;
        nslow += slow;
    }
    atomicAdd(&g_bad, (unsigned long long)bad);
    atomicAdd(&g_slow, (unsigned long long)nslow);
    atomicAdd(&g_tot, 12ull);
}

int main()
{
    {
        for (int r = 0; r < 16; ++r) k_logcheck<<<4096, 256>>>((u64)r << 40);
        unsigned long long bad = 0, tot = 0, nslow = 0;
        cudaDeviceSynchronize();
        cudaMemcpyFromSymbol(&bad, g_bad, 8);
        cudaMemcpyFromSymbol(&tot, g_tot, 8);
        cudaMemcpyFromSymbol(&nslow, g_slow, 8);
        printf("log_w / ddiv_w vs log_ / IEEE division: %llu mismatches of %llu (%llu slow-flagged)\n", bad, tot, nslow);
    }
    u64 *o; long long *c;
    cudaMalloc(&o, 8); cudaMalloc(&c, 64 * 8);
    cudaMemset(c, 0, 64 * 8);
    for (int rep = 0; rep < 3; ++rep) k_lat<<<1, 32>>>(o, c, 0.5);
    cudaDeviceSynchronize();
    long long h[12] = {0};
    cudaMemcpy(h, c, 12 * 8, cudaMemcpyDeviceToHost);
    const char *nm[] = {"fp64 div (dependent)", "log_", "stirlerr", "log_dbinom (uniform x)", "hgd (1 lane)",
                        "hgd_tp (32 lanes)", "hrua_setup", "hgd_tp cfg0 nodes", "log_dbinom_w (lane x)",
                        "log_dbinom (lane x)", "bd0_w (lane x)", "stirlerr_w"};
    for (int i = 0; i < 12; ++i) printf("%-24s %8lld cycles\n", nm[i], h[i]);
    k_phases<<<1, 32>>>(o);
    cudaDeviceSynchronize();
    long long ph[8];
    cudaMemcpyFromSymbol(ph, g_ph, 8 * 8);
    const char *pn[] = {"setup (p,q,a,var,sqrt,M,b)", "stirlerr(g), stirlerr(R-g)", "Philox + candidate", "log_dbinom (lane)", "log_w(U)", "gather + decide"};
    for (int i = 0; i < 6; ++i) printf("hgd_tp phase %-28s %8lld cycles\n", pn[i], ph[i]);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
