// rs_kernels.cu -- hot-path kernels of the B200 sampler (sm_100a).
// P:n = /root/reference/PAPER.md line n; CANON readings R1-R12: DESIGN.md.
#include "rs_kernels.cuh"
#ifdef RS_SPLIT_PROF
#include <cstdio>
#endif

namespace rs {

__device__ unsigned g_rs_errors = 0;

// ===========================================================================
// Split tree (rows a3/a4).
// ===========================================================================
template <bool WR, int G>
__device__ __forceinline__ void split_top_level(const SplitArgs &a, const u64 *in, u64 *outb, u32 width, int d, u64 base)
{
    for (u32 j = threadIdx.x / G; j < width; j += SPLIT_NT / G) {
        const u64 k = in[j];
        const u64 x = split_node_grp<WR, G>(a.N, d, base + j, k, a.seed);
        if ((threadIdx.x & (G - 1)) == 0) {
            outb[2 * j] = x;
            outb[2 * j + 1] = k - x;
        }
    }
}

template <bool WR>
__device__ __forceinline__ void split_top(const SplitArgs &a)
{
    __shared__ u64 buf[2][SPLIT_WIDTH];
    __shared__ u64 wtmp[SPLIT_NT / 32];
    __shared__ u64 tot;
    const int tid = threadIdx.x;
    const u64 node = a.node0 + blockIdx.x;
    if (tid == 0) buf[0][0] = a.in_cnt ? a.in_cnt[blockIdx.x] : a.root_cnt;
    __syncthreads();
    int cur = 0;
#ifdef RS_SPLIT_PROF
    long long tl[16];
    tl[0] = clock64();
#endif
    for (int l = 0; l < a.nlev; ++l) {
#ifdef RS_SPLIT_PROF
        if (l) tl[l] = clock64();
#endif
        const u32 width = 1u << l;
        const int d = a.ds + l;
        const u64 base = node << l;
        // narrow levels: a group of G lanes per node evaluates G rejection
        // iterations at once (hgd_tpg), so a level costs ~one iteration's latency
        // (a warp per node -- hgd_tp -- up to four nodes per warp)
        if (width * 32 <= 4 * SPLIT_NT) split_top_level<WR, 32>(a, buf[cur], buf[cur ^ 1], width, d, base);
        else if (width * 8 <= SPLIT_NT) split_top_level<WR, 8>(a, buf[cur], buf[cur ^ 1], width, d, base);
        else                            split_top_level<WR, 1>(a, buf[cur], buf[cur ^ 1], width, d, base);
        __syncthreads();
        cur ^= 1;
    }
#ifdef RS_SPLIT_PROF
    if (tid == 0) {
        tl[a.nlev] = clock64();
        for (int l = 0; l < a.nlev; ++l) printf("split level %d: %lld cycles\n", l, tl[l + 1] - tl[l]);
    }
#endif
    // children's offsets: parent offset + exclusive scan of their counts
    const u32 W = 1u << a.nlev;
    const u32 per = (W + SPLIT_NT - 1) / SPLIT_NT;
    const u32 beg = tid * per;
    u64 s = 0;
    for (u32 i = 0; i < per; ++i) if (beg + i < W) s += buf[cur][beg + i];
    u64 ex = block_exclusive_scan<u64, SPLIT_NT>(s, wtmp, &tot) +
             (a.in_off ? a.in_off[blockIdx.x] : a.root_off);
    const u64 obase = (u64)blockIdx.x << a.nlev;
    for (u32 i = 0; i < per; ++i) {
        if (beg + i >= W) break;
        const u64 c = buf[cur][beg + i];
        if (a.leaf_cnt) {
            if (c > 0xffffffffull) atomicOr(&g_rs_errors, 1u);
            a.leaf_cnt[obase + beg + i] = (u32)c;
            a.leaf_off[obase + beg + i] = ex;
        } else {
            a.out_cnt[obase + beg + i] = c;
            a.out_off[obase + beg + i] = ex;
        }
        ex += c;
    }
}

template <bool WR, int G = 1>
__device__ __forceinline__ void split_level(const LevelArgs &a)
{
    const u64 j = ((u64)blockIdx.x * LEVEL_NT + threadIdx.x) / G;
    if (j >= a.width) return;                 // (whole groups: width * G is a multiple of G)
    const u64 k = a.in_cnt[j], off = a.in_off[j];
    const u64 x = split_node_grp<WR, G>(a.N, a.d, a.node0 + j, k, a.seed);
    if ((threadIdx.x & (G - 1)) != 0) return;
    if (a.leaf_cnt) {
        if (k > 0xffffffffull) atomicOr(&g_rs_errors, 1u);
        a.leaf_cnt[2 * j] = (u32)x;
        a.leaf_cnt[2 * j + 1] = (u32)(k - x);
        a.leaf_off[2 * j] = off;
        a.leaf_off[2 * j + 1] = off + x;
    } else {
        a.out_cnt[2 * j] = x;
        a.out_cnt[2 * j + 1] = k - x;
        a.out_off[2 * j] = off;
        a.out_off[2 * j + 1] = off + x;
    }
}

// The last NL levels in one launch: thread j expands node (d, node0 + j)
// through NL levels (2^NL - 1 deviates, breadth-first in registers) and
// writes its 2^NL leaves.  Each lane now runs 2^NL - 1 rejection loops, so a
// warp's slowest lane is close to its average (the divergence of one HRUA
// loop per thread is averaged out), and NL - 1 global round trips and
// launches disappear.
template <int NL, bool WR>
__device__ __forceinline__ void split_deep(const LevelArgs &a)
{
    const u64 j = (u64)blockIdx.x * LEVEL_NT + threadIdx.x;
    if (j >= a.width) return;
    constexpr int W = 1 << NL;
    u64 c[W], o[W];
    c[0] = a.in_cnt[j];
    o[0] = a.in_off[j];
    if (c[0] > 0xffffffffull * (u64)W) atomicOr(&g_rs_errors, 1u);
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        const int d = a.d + l;
#pragma unroll
        for (int i = (1 << l) - 1; i >= 0; --i) {          // in place, from the right
            const u64 k = c[i], off = o[i];
            const u64 x = split_node_t<WR>(a.N, d, ((a.node0 + j) << l) + i, k, a.seed);
            c[2 * i] = x;
            c[2 * i + 1] = k - x;
            o[2 * i] = off;
            o[2 * i + 1] = off + x;
        }
    }
#pragma unroll
    for (int i = 0; i < W; ++i) {
        if (c[i] > 0xffffffffull) atomicOr(&g_rs_errors, 1u);
        a.leaf_cnt[W * j + i] = (u32)c[i];
        a.leaf_off[W * j + i] = o[i];
    }
}

__device__ __forceinline__ u32 ld_acquire_u32(const u32 *p)
{
    u32 v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid-wide barrier of a cooperative launch: every CTA arrives once per level
// (monotone counter); target = (level + 1) * gridDim.x.
__device__ __forceinline__ void coop_barrier(u32 *bar, u32 target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire_u32(bar) < target) __nanosleep(20);
        __threadfence();
    }
    __syncthreads();
}

template <bool WR, int G>
__device__ __forceinline__ void coop_level(const CoopArgs &a, int l, u64 width)
{
    const u32 tid = threadIdx.x;
    const u64 ng = (u64)gridDim.x * COOP_NT / G;
    const int d = a.ds + l;
    const u64 base = a.node0 << l;
    const u64 *icnt = a.buf_cnt[(l + 1) & 1], *ioff = a.buf_off[(l + 1) & 1];   // level l - 1's output
    u64 *ocnt = a.buf_cnt[l & 1], *ooff = a.buf_off[l & 1];
    const bool leaf = a.ds + l + 1 == a.D;
    for (u64 j = ((u64)blockIdx.x * COOP_NT + tid) / G; j < width; j += ng) {
        const u64 k = l ? __ldcg(icnt + j) : a.root_cnt;
        const u64 off = l ? __ldcg(ioff + j) : 0;
        const u64 x = split_node_grp<WR, G>(a.N, d, base + j, k, a.seed);
        if ((tid & (G - 1)) == 0) {
            if (leaf) {
                if (k > 0xffffffffull) atomicOr(&g_rs_errors, 1u);
                a.leaf_cnt[2 * j] = (u32)x;
                a.leaf_cnt[2 * j + 1] = (u32)(k - x);
                a.leaf_off[2 * j] = off;
                a.leaf_off[2 * j + 1] = off + x;
            } else {
                ocnt[2 * j] = x;
                ocnt[2 * j + 1] = k - x;
                ooff[2 * j] = off;
                ooff[2 * j + 1] = off + x;
            }
        }
    }
}

template <bool WR>
__device__ __forceinline__ void split_coop(const CoopArgs &a)
{
    const u64 nw = (u64)gridDim.x * (COOP_NT / 32);      // warps of the grid
#ifdef RS_SPLIT_PROF
    long long tw[24], tb[24];
    long long t_prev = clock64();
#endif
    for (int l = 0; l < a.nlev; ++l) {
        const u64 width = 1ull << l;
        if (width <= 2 * nw)      coop_level<WR, 32>(a, l, width);
        else if (width <= 8 * nw) coop_level<WR, 8>(a, l, width);
        else                      coop_level<WR, 1>(a, l, width);
#ifdef RS_SPLIT_PROF
        const long long t_work = clock64();
#endif
        if (l + 1 < a.nlev) coop_barrier(a.bar, (u32)(l + 1) * gridDim.x);
#ifdef RS_SPLIT_PROF
        const long long t_bar = clock64();
        if (l < 24) { tw[l] = t_work - t_prev; tb[l] = t_bar - t_work; }
        t_prev = t_bar;
#endif
    }
#ifdef RS_SPLIT_PROF
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int l = 0; l < a.nlev && l < 24; ++l) printf("coop level %d: work %lld barrier %lld cycles\n", l, tw[l], tb[l]);
#endif
}

__global__ void __launch_bounds__(COOP_NT, 1) k_split_coop(CoopArgs a) { split_coop<false>(a); }
__global__ void __launch_bounds__(COOP_NT, 1) k_split_coop_wr(CoopArgs a) { split_coop<true>(a); }

// WOR (hypergeometric) and WR (binomial) instantiations are separate
// kernels: each holds only its deviate's code (the split kernels are
// instruction-fetch bound).
__global__ void __launch_bounds__(SPLIT_NT) k_split(SplitArgs a) { split_top<false>(a); }
__global__ void __launch_bounds__(SPLIT_NT) k_split_wr(SplitArgs a) { split_top<true>(a); }
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level(LevelArgs a) { split_level<false>(a); }
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level_wr(LevelArgs a) { split_level<true>(a); }
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level_g32(LevelArgs a) { split_level<false, 32>(a); }
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level_g8(LevelArgs a) { split_level<false, 8>(a); }
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level_wr_g32(LevelArgs a) { split_level<true, 32>(a); }
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level_wr_g8(LevelArgs a) { split_level<true, 8>(a); }
__global__ void __launch_bounds__(LEVEL_NT, RS_D3_MINB) k_split_deep2(LevelArgs a) { split_deep<2, false>(a); }
__global__ void __launch_bounds__(LEVEL_NT, RS_D3_MINB) k_split_deep3(LevelArgs a) { split_deep<3, false>(a); }
__global__ void __launch_bounds__(LEVEL_NT, RS_D3_MINB) k_split_deep4(LevelArgs a) { split_deep<4, false>(a); }
__global__ void __launch_bounds__(LEVEL_NT, 4) k_split_deep2_wr(LevelArgs a) { split_deep<2, true>(a); }
__global__ void __launch_bounds__(LEVEL_NT, RS_D3_MINB) k_split_deep3_wr(LevelArgs a) { split_deep<3, true>(a); }
__global__ void __launch_bounds__(LEVEL_NT, 4) k_split_deep4_wr(LevelArgs a) { split_deep<4, true>(a); }

}  // namespace rs

#include "rs_leaf.cuh"
#include "rs_leaf_warp.cuh"
#include "rs_leaf_lp.cuh"
#include "rs_leaf_wide.cuh"
#include "rs_fused.cuh"
#include "rs_leaf_bitmap.cuh"
#include "rs_algb.cuh"

namespace rs {

// ===========================================================================
// Bernoulli (a9): dyadic chunks, geometric skips G = floor(log U/log1p(-rho))
// (P:199-201), the chain restarted at each chunk start ("independently apply
// Bernoulli sampling to subranges").  ONE WARP PER CHUNK: each
// step a lane turns one Philox block into two skips, and a warp scan of the
// steps G+1 gives 64 consecutive positions (the paper's "prefix sums of
// geometric deviates", without materialising them).  Positions go
// to a shared-memory buffer; the chunk's output offset comes from a
// single-pass decoupled look-back over chunk counts (lane-parallel), then the
// buffer is stored coalesced.
//
// G in fp32 first, CERTIFIED: q' = log2(U') * (ln 2 / lr) with U' = U rounded
// to fp32 and log2 by MUFU; |q' - q| is bounded (U' relative error 2^-24,
// __log2f absolute error <= 2^-22.6 on [0.5, 2] and <= 2 ulp elsewhere, two
// fp32 roundings) far below the margin used here; when [q' - margin,
// q' + margin] contains no integer, floor(q') == floor(q) and that is G;
// otherwise (about 1 draw in 2000 at rho = 0.01) G is evaluated exactly in
// fp64 as CANON defines it (log_, IEEE division, floor).  Bit-exact either way.
// ===========================================================================
// (out of line: rare, and four inlined copies of log_ cost the Bernoulli
// kernels instruction-cache space)
template <typename T>
__device__ __noinline__ T skip_exact(double U, double lr, T r)
{
    const double G = floor_(log_(U) / lr);
    return G >= (double)r ? r + 1 : (T)G + 1;       // any G >= r ends the chain
}

// fp32 candidate for G (see above): sets ok when floor is certain; the
// result saturates at r (any G >= r ends the chain).  Branch-free.
// r is the chunk range saturated at 2^31 - 1; full says it is not saturated
// (otherwise a G at or above the saturation point is not decided here).
__device__ __forceinline__ u32 skip_fast(u32 a, u32 b, float c, float m_abs, u32 r, bool full, bool &ok)
{
    const u64 m = ((((u64)a << 32) | b) >> 11) | 1ull;              // 2 * (u52 mantissa) + 1
    const float U = __ull2float_rn(m) * 0x1p-53f;                   // U rounded to fp32
    const float q = __log2f(U) * c;                                 // ~ log(U) / lr  (> 0)
    const float mg = m_abs + q * 0x1p-20f;
    const float lo = floorf(q - mg), hi = floorf(q + mg);
    const float rf = (float)r;
    ok = (lo >= rf && full) || (lo == hi && lo >= 0.0f && lo < rf);
    return lo >= rf ? r : (u32)fminf(lo, rf);
}

// fp64 candidate for large mean skips (small rho: there the fp32 margin
// m_abs = 2^-19 / |lr| fails often).  log_fast (rs_math.cuh) differs from
// CANON's log_ by a few ulp of |log U| <= 37, i.e. < 2^-44; the margin below
// allows 2^-42 plus 2^-48 relative for the two roundings of q, against
// CANON's IEEE division by lr.  As with skip_fast, an uncertain floor goes to
// skip_exact.
__device__ __forceinline__ u32 skip_fast64(u32 a, u32 b, double il, double m_abs, u32 r, bool full, bool &ok)
{
    const double q = log_fast(u52(a, b)) * il;                      // ~ log(U) / lr  (>= 0)
    const double mg = m_abs + q * 0x1p-48;
    const double lo = floor(q - mg), hi = floor(q + mg);
    const double rf = (double)r;
    ok = (lo >= rf && full) || (lo == hi && lo >= 0.0 && lo < rf);
    return lo >= rf ? r : (u32)fmin(fmax(lo, 0.0), rf);
}

// The u16 path's candidate (chunk ranges <= 2^16, rho >= 2^-6) from 32 bits
// of the draw: U' = w 2^-32 with w = a when a >= 2^24 (b lies below fp32
// precision there), else U' = w 2^-40 with w = (a << 8) | (b >> 24); in both
// cases U' is within a relative 2^-23 of CANON's u52(a, b) (truncation 2^-24
// plus the I2FP rounding 2^-24), inside the margin of skip_fast (whose
// 2^-19 / |lr| term covers relative errors of U up to 2^-19).  32-bit I2FP
// replaces the 64-bit I2F.  a < 2^16 (p = 2^-16) is left to the exact path.
__device__ __forceinline__ u32 skip_fast16(u32 a, u32 b, float c, float m_abs, u32 r, bool &ok)
{
    const bool big = a >= (1u << 24);
    const u32 w = big ? a : __funnelshift_l(b, a, 8);
    const float U = __uint2float_rn(w) * (big ? 0x1p-32f : 0x1p-40f);
    const float q = __log2f(U) * c;                                 // ~ log(U) / lr  (> 0)
    const float mg = m_abs + q * 0x1p-20f;
    const float lo = floorf(q - mg), hi = floorf(q + mg);
    const float rf = (float)r;
    ok = a >= (1u << 16) && (lo >= rf || lo == hi);                 // (lo == hi implies lo >= 0: q > 0)
    return lo >= rf ? r : (u32)lo;
}

struct SkipParams {
    float c, m_abs;          // fp32 path: ln 2 / lr, margin
    double il, m_abs64;      // fp64 path: 1 / lr, margin
};

template <bool F64>
__device__ __forceinline__ u32 skip_cand(u32 a, u32 b, const SkipParams &sp, u32 r, bool full, bool &ok)
{
    return F64 ? skip_fast64(a, b, sp.il, sp.m_abs64, r, full, ok) : skip_fast(a, b, sp.c, sp.m_abs, r, full, ok);
}

__device__ __forceinline__ void st_relaxed(u64 *p, u64 v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_relaxed(const u64 *p)
{
    u64 v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_v4b(u64 *p, u64 a, u64 b, u64 c, u64 d)
{
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d)
                 : "memory");
}

constexpr int BW_WARPS = 4;
// positions buffered per chunk (mean <= n0 = 1024; u64 positions only for
// chunk ranges above 2^24, where the buffer is smaller to fit 48 KB)
// A warp takes a TICKET of G consecutive chunks and buffers their positions
// (type B, relative to each chunk start) in shared memory.  Offsets come
// from a single-pass look-back whose inclusive prefixes are produced IN
// ORDER by one scanner warp (block 0, warp 0): generating warps only publish
// their ticket's count (AGG), and -- double-buffered -- generate their next
// ticket before they wait for the previous one's prefix (INC), so neither a
// slow predecessor nor a long look-back walk stalls them.  T = position
// arithmetic (u32 while a batch's 64 steps fit, else u64).
template <typename T, typename B, int G, u32 CAP, bool F64>
__device__ __forceinline__ u32 bern_ticket(const BernArgs &a, u64 tk, B *bw, u32 (&cnt)[G], const SkipParams &sp,
                                           u32 lane, bool &overflow)
{
    u32 total = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        cnt[g] = 0;
        const u64 ci = tk * G + g;
        if (ci >= a.nchunks) continue;
        const u64 gi = a.chunk0 + ci;
        const u64 lo = bound_at(a.N, a.Db, gi);
        const T r = (T)(bound_at(a.N, a.Db, gi + 1) - lo);
        const u32 r32 = r > (T)0x7fffffffu ? 0x7fffffffu : (u32)r;    // fast path saturation point
        const bool rfull = r <= (T)0x7fffffffu;
        const Stream st(a.seed, P_GEO, ((u64)1 << a.Db) + gi);
        B *bg = bw + total;                        // 4-aligned (vector stores)
        const u32 room = CAP - total;
        // skips in batches of 128 draws: lane l has draws 4(q0 + l) .. +3,
        // i.e. Philox blocks 2(q0 + l) and 2(q0 + l) + 1 (draw j = pair j mod 2
        // of block j / 2, R3)
        T S = 0;
        u32 count = 0;
        for (u32 q0 = 0;; q0 += 32) {
            const u32x4 w0 = philox_rk(2 * (q0 + lane), st, a.rk);
            const u32x4 w1 = philox_rk(2 * (q0 + lane) + 1, st, a.rk);
            bool ok0, ok1, ok2, ok3;
            u32 g0, g1, g2, g3;
            if (sizeof(B) == 2 && !F64) {          // chunk ranges <= 2^16
                g0 = skip_fast16(w0.x, w0.y, sp.c, sp.m_abs, r32, ok0);
                g1 = skip_fast16(w0.z, w0.w, sp.c, sp.m_abs, r32, ok1);
                g2 = skip_fast16(w1.x, w1.y, sp.c, sp.m_abs, r32, ok2);
                g3 = skip_fast16(w1.z, w1.w, sp.c, sp.m_abs, r32, ok3);
            } else {
                g0 = skip_cand<F64>(w0.x, w0.y, sp, r32, rfull, ok0);
                g1 = skip_cand<F64>(w0.z, w0.w, sp, r32, rfull, ok1);
                g2 = skip_cand<F64>(w1.x, w1.y, sp, r32, rfull, ok2);
                g3 = skip_cand<F64>(w1.z, w1.w, sp, r32, rfull, ok3);
            }
            T s0 = (T)g0 + 1, s1 = (T)g1 + 1, s2 = (T)g2 + 1, s3 = (T)g3 + 1;
            if (__any_sync(0xffffffffu, !(ok0 && ok1 && ok2 && ok3))) {   // rare: exact fp64 (CANON)
                if (!ok0) s0 = skip_exact<T>(u52(w0.x, w0.y), a.log1m_rho, r);
                if (!ok1) s1 = skip_exact<T>(u52(w0.z, w0.w), a.log1m_rho, r);
                if (!ok2) s2 = skip_exact<T>(u52(w1.x, w1.y), a.log1m_rho, r);
                if (!ok3) s3 = skip_exact<T>(u52(w1.z, w1.w), a.log1m_rho, r);
            }
            const T l1 = s0 + s1, l2 = l1 + s2, l4 = l2 + s3;       // lane-local prefix
            T incl = l4;                                           // inclusive scan over lanes
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const T y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (u32)o) incl += y;
            }
            const T E = S + incl - l4;                             // before this lane's draws
            const T S0 = E + s0, S1 = E + l1, S2 = E + l2, S3 = E + l4;   // positions + 1
            const u32 j0 = 4 * (q0 + lane);
            if (S3 <= r && j0 + 3 < room) {                        // all four (common)
                if (sizeof(B) == 2) {
                    const u32 lo2 = (u32)(S0 - 1) | ((u32)(S1 - 1) << 16), hi2 = (u32)(S2 - 1) | ((u32)(S3 - 1) << 16);
                    *reinterpret_cast<uint2 *>(bg + j0) = make_uint2(lo2, hi2);
                } else {
                    bg[j0] = (B)(S0 - 1); bg[j0 + 1] = (B)(S1 - 1); bg[j0 + 2] = (B)(S2 - 1); bg[j0 + 3] = (B)(S3 - 1);
                }
            } else {
                if (S0 <= r) { if (j0 < room) bg[j0] = (B)(S0 - 1); else overflow = true; }
                if (S1 <= r) { if (j0 + 1 < room) bg[j0 + 1] = (B)(S1 - 1); else overflow = true; }
                if (S2 <= r) { if (j0 + 2 < room) bg[j0 + 2] = (B)(S2 - 1); else overflow = true; }
                if (S3 <= r) { if (j0 + 3 < room) bg[j0 + 3] = (B)(S3 - 1); else overflow = true; }
            }
            const T tot = __shfl_sync(0xffffffffu, incl, 31);
            if (S + tot <= r) {                    // the whole batch lies in the chunk (common)
                count += 128;
                S += tot;
                continue;
            }
            count += __popc(__ballot_sync(0xffffffffu, S0 <= r)) + __popc(__ballot_sync(0xffffffffu, S1 <= r)) +
                     __popc(__ballot_sync(0xffffffffu, S2 <= r)) + __popc(__ballot_sync(0xffffffffu, S3 <= r));
            break;
        }
        if (__any_sync(0xffffffffu, overflow)) count = min(count, room);
        cnt[g] = count;
        total += (count + 3) & ~3u;                // next chunk starts 4-aligned in the buffer
    }
    return total;
}

// Graph calls (NEXT-3): chunk values -> packed edges (edge_pack), lane-strided
// 8-byte stores (coalesced), not unrolled, so the kernel holds one decode.
template <typename B>
__device__ __noinline__ void bern_store_edges(u64 *d, const B *bw, u32 lim, u64 base, u64 gV, u32 lane)
{
    EdgeCursor cur(gV);
#pragma unroll 1
    for (u32 i = lane; i < lim; i += 32) d[i] = cur.pack(base - 1 + (u64)bw[i]);
}

template <typename B, int G, bool GR>
__device__ __forceinline__ void bern_write(const BernArgs &a, u64 tk, const B *bw, const u32 (&cnt)[G],
                                           u64 excl, u32 lane)
{
    u32 off = 0, boff = 0;                                // output / buffer offsets of chunk g
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const u64 ci = tk * G + g;
        if (ci >= a.nchunks) break;
        const u64 base = bound_at(a.N, a.Db, a.chunk0 + ci) + 1;
        const u64 o0 = excl + off;                        // output index of this chunk's first value
        const u32 n = cnt[g];
        const u64 lim = a.capacity > o0 ? min(a.capacity - o0, (u64)n) : 0;
        // groups of four on the output's 32-byte grid: group q covers chunk
        // values i = 4q - h .. 4q - h + 3
        if (GR) {                                         // graph calls: one decode site
            bern_store_edges(a.out + o0, bw + boff, (u32)lim, base, a.gV, lane);
            off += n;
            boff += (n + 3) & ~3u;
            continue;
        }
        const u32 h = (u32)(reinterpret_cast<uintptr_t>(a.out + o0) >> 3) & 3u;
        u64 *d0 = a.out + (o0 - h);
        const u32 ng = (u32)((h + lim + 3) >> 2);
        const B *bh = bw + boff - (int)h;                 // chunk value 4q - h + t = bh[4q + t]
        for (u32 q = lane; q < ng; q += 32) {
            const int i0 = (int)(4 * q) - (int)h;
            if (i0 >= 0 && (u64)(i0 + 4) <= lim) {        // full group (common): no per-value tests
                st_v4b(d0 + 4 * q, base + (u64)bh[4 * q], base + (u64)bh[4 * q + 1], base + (u64)bh[4 * q + 2],
                       base + (u64)bh[4 * q + 3]);
            } else {
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (i0 + t >= 0 && (u64)(i0 + t) < lim) d0[4 * q + t] = base + (u64)bw[boff + i0 + t];
            }
        }
        off += n;
        boff += (n + 3) & ~3u;
    }
}

constexpr u64 B_AGG = 1ull << 62, B_INC = 2ull << 62, B_VAL = (1ull << 62) - 1;

#ifndef RS_BSC
#define RS_BSC 8
#endif
// The scanner: turns the published ticket counts (AGG) into inclusive
// prefixes (INC) in ticket order, 32 * RS_BSC tickets per step (one L2
// round trip each: the scanner's step rate bounds the kernel when tickets are
// cheap, so each lane takes RS_BSC independent loads).
__device__ __forceinline__ void bern_scanner(const BernArgs &a, u64 ntick, u32 lane)
{
    u64 next = 0, run = 0;
    while (next < ntick) {
        u64 v[RS_BSC];
        u32 fu = RS_BSC;                                    // first unpublished entry of the lane
#pragma unroll
        for (int i = RS_BSC - 1; i >= 0; --i) {
            const u64 idx = next + RS_BSC * lane + i;
            v[i] = idx < ntick ? ld_relaxed(a.status + idx) : 0ull;
            if (idx >= ntick || (v[i] >> 62) == 0) fu = i;
        }
        const u32 first = __reduce_min_sync(0xffffffffu, fu == RS_BSC ? 0xffffffffu : RS_BSC * lane + fu);
        const u32 np = first == 0xffffffffu ? 32u * RS_BSC : first;   // consecutive published tickets
        if (np == 0) { __nanosleep(256); continue; }
        u64 loc = 0;
#pragma unroll
        for (int i = 0; i < RS_BSC; ++i) if (RS_BSC * lane + i < np) loc += v[i] & B_VAL;
        u64 incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u64 y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (u32)o) incl += y;
        }
        u64 pref = run + incl - loc;
#pragma unroll
        for (int i = 0; i < RS_BSC; ++i) {
            if (RS_BSC * lane + i < np) {
                pref += v[i] & B_VAL;
                st_relaxed(a.status + next + RS_BSC * lane + i, B_INC | pref);
            }
        }
        run += __shfl_sync(0xffffffffu, incl, 31);
        next += np;
    }
    if (lane == 0) *a.count_dev = run;
}

__device__ __forceinline__ u64 bern_wait_inc(const BernArgs &a, u64 tk)
{
    u64 v = ld_relaxed(a.status + tk);
    while ((v >> 62) != 2) {
        __nanosleep(128);
        v = ld_relaxed(a.status + tk);
    }
    return v & B_VAL;
}

template <typename T, typename B, int G, u32 CAP, int NW, bool GR, bool F64>
__device__ __forceinline__ void bernoulli_chunks(const BernArgs &a)
{
    __shared__ B buf[NW][2][CAP];
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u64 ntick = (a.nchunks + G - 1) / G;
    if (blockIdx.x == 0 && wid == 0) { bern_scanner(a, ntick, lane); return; }
    SkipParams sp;
    sp.c = (float)(0x1.62e42fefa39efp-1 / a.log1m_rho);            // ln 2 / lr
    sp.m_abs = (float)(0x1p-19 / -a.log1m_rho) + 0x1p-20f;
    sp.il = 1.0 / a.log1m_rho;
    sp.m_abs64 = 0x1p-42 / -a.log1m_rho;
    bool overflow = false, have_prev = false;
    u32 cur = 0, prev_cnt[G], prev_total = 0;
    u64 prev_tk = 0;
    for (;;) {
        u32 tk = 0;
        if (lane == 0) tk = atomicAdd(a.ticket, 1u);
        tk = __shfl_sync(0xffffffffu, tk, 0);
        if (tk < ntick) {
            u32 cnt[G];
            bern_ticket<T, B, G, CAP, F64>(a, tk, buf[wid][cur], cnt, sp, lane, overflow);
            u32 total = 0;
#pragma unroll
            for (int g = 0; g < G; ++g) total += cnt[g];
            if (lane == 0) st_relaxed(a.status + tk, B_AGG | total);
            if (have_prev) {                                       // the previous ticket's prefix
                const u64 excl = bern_wait_inc(a, prev_tk) - prev_total;
                __syncwarp();
                bern_write<B, G, GR>(a, prev_tk, buf[wid][cur ^ 1], prev_cnt, excl, lane);
            }
#pragma unroll
            for (int g = 0; g < G; ++g) prev_cnt[g] = cnt[g];
            prev_total = total;
            prev_tk = tk;
            have_prev = true;
            cur ^= 1;
            __syncwarp();
        } else {
            if (have_prev) {
                const u64 excl = bern_wait_inc(a, prev_tk) - prev_total;
                __syncwarp();
                bern_write<B, G, GR>(a, prev_tk, buf[wid][cur ^ 1], prev_cnt, excl, lane);
            }
            break;
        }
    }
    if (__any_sync(0xffffffffu, overflow) && lane == 0) atomicOr(&g_rs_errors, 2u);
}

#ifndef RS_BG
#define RS_BG 2
#endif
#ifndef RS_B64W
#define RS_B64W 4
#endif
constexpr int BG16 = RS_BG;                                           // chunks per ticket (u16 path)
constexpr u32 BCAP16 = ((BG16 * 1024 + 10 * 32 * (BG16 < 4 ? 2 : BG16 / 2) + 63) / 64) * 64;
constexpr int BNW16 = (BCAP16 * 2 * 2 * 4 <= 48 * 1024) ? 4 : (BCAP16 * 2 * 2 * 2 <= 48 * 1024) ? 2 : 1;
__global__ void __launch_bounds__(32 * BNW16) k_bernoulli(BernArgs a) { bernoulli_chunks<u32, uint16_t, BG16, BCAP16, BNW16, false, false>(a); }
__global__ void __launch_bounds__(32 * BNW16) k_bernoulli_g(BernArgs a) { bernoulli_chunks<u32, uint16_t, BG16, BCAP16, BNW16, true, false>(a); }
// r <= 2^24: u32 positions; 2^24 < r <= 2^32: u64 position arithmetic, u32
// positions buffered; RS_B32G chunks per ticket.  These chunk ranges mean
// rho < 2^-6; the "d" kernels take fp64 skip candidates (chosen for
// rho < BF64_RHO, where the fp32 margin fails too often -- measured
// crossover)
#ifndef RS_B32G
#define RS_B32G 1
#endif
constexpr u32 BCAP32 = RS_B32G * 1024 + 512;
#define RS_BK(name, T, GR, F64) \
    __global__ void __launch_bounds__(32 * RS_B64W) name(BernArgs a) { bernoulli_chunks<T, u32, RS_B32G, BCAP32, RS_B64W, GR, F64>(a); }
RS_BK(k_bernoulli32, u32, false, false)
RS_BK(k_bernoulli32_g, u32, true, false)
RS_BK(k_bernoulli32d, u32, false, true)
RS_BK(k_bernoulli32d_g, u32, true, true)
RS_BK(k_bernoulli64, u64, false, false)
RS_BK(k_bernoulli64_g, u64, true, false)
RS_BK(k_bernoulli64d, u64, false, true)
RS_BK(k_bernoulli64d_g, u64, true, true)
#undef RS_BK
// larger r: u64 positions (1536 x 8 B per warp)
__global__ void __launch_bounds__(32) k_bernoulli64w(BernArgs a) { bernoulli_chunks<u64, u64, 1, 1536, 1, false, true>(a); }
__global__ void __launch_bounds__(32) k_bernoulli64w_g(BernArgs a) { bernoulli_chunks<u64, u64, 1, 1536, 1, true, true>(a); }

// ===========================================================================
// Validation helpers.
// ===========================================================================
__device__ __forceinline__ u64 mix64(u64 z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_digest(const u64 *v, u64 n, u64 base, u64 *acc)
{
    u64 h = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        h += mix64((base + i) ^ mix64(v[i]));
    for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long *)acc, (unsigned long long)h);
}

__global__ void k_validate(const u64 *v, u64 n, u64 N, int strict, u64 *bad)
{
    u64 b = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 x = v[i];
        b += (x < 1 || x > N);
        if (i + 1 < n) {
            const u64 y = v[i + 1];
            b += strict ? (x >= y) : (x > y);
        }
    }
    for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd((unsigned long long *)bad, (unsigned long long)b);
}

__global__ void k_iota(u64 *out, u64 n)
{
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = i + 1;
}

}  // namespace rs
