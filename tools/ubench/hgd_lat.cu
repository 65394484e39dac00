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

int main()
{
    u64 *o; long long *c;
    cudaMalloc(&o, 8); cudaMalloc(&c, 64 * 8);
    for (int rep = 0; rep < 3; ++rep) k_lat<<<1, 32>>>(o, c, 0.5);
    cudaDeviceSynchronize();
    long long h[8] = {0};
    cudaMemcpy(h, c, 8 * 8, cudaMemcpyDeviceToHost);
    const char *nm[] = {"fp64 div (dependent)", "log_", "stirlerr", "log_dbinom", "hgd (1 lane)", "hgd_tp (32 lanes)", "hrua_setup", "hgd_tp cfg0 nodes"};
    for (int i = 0; i < 8; ++i) printf("%-24s %8lld cycles\n", nm[i], h[i]);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
