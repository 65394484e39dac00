// rs_kernels.cu -- hot-path kernels of the B200 sampler (sm_100a).
// P:n = /root/reference/PAPER.md line n; CANON readings R1-R12: DESIGN.md.
#include "rs_kernels.cuh"

namespace rs {

__device__ unsigned g_rs_errors = 0;

// ===========================================================================
// Split tree (rows a3/a4).
// ===========================================================================
__global__ void __launch_bounds__(SPLIT_NT) k_split(SplitArgs a)
{
    __shared__ u64 buf[2][SPLIT_WIDTH];
    __shared__ u64 wtmp[SPLIT_NT / 32];
    __shared__ u64 tot;
    const int tid = threadIdx.x;
    const u64 node = a.node0 + blockIdx.x;
    if (tid == 0) buf[0][0] = a.in_cnt ? a.in_cnt[blockIdx.x] : a.root_cnt;
    __syncthreads();
    int cur = 0;
    for (int l = 0; l < a.nlev; ++l) {
        const u32 width = 1u << l;
        const int d = a.ds + l;
        const u64 base = node << l;
        for (u32 j = tid; j < width; j += SPLIT_NT) {
            const u64 k = buf[cur][j];
            const u64 x = split_node(a.wr != 0, a.N, d, base + j, k, a.seed);
            buf[cur ^ 1][2 * j] = x;
            buf[cur ^ 1][2 * j + 1] = k - x;
        }
        __syncthreads();
        cur ^= 1;
    }
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

__global__ void __launch_bounds__(LEVEL_NT, 8) k_split_level(LevelArgs a)
{
    const u64 j = (u64)blockIdx.x * LEVEL_NT + threadIdx.x;
    if (j >= a.width) return;
    const u64 k = a.in_cnt[j], off = a.in_off[j];
    const u64 x = split_node(a.wr != 0, a.N, a.d, a.node0 + j, k, a.seed);
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

}  // namespace rs

#include "rs_leaf.cuh"
#include "rs_leaf_warp.cuh"
#include "rs_leaf_bitmap.cuh"

namespace rs {

// ===========================================================================
// Bernoulli (a9): dyadic chunks, geometric skips G = floor(log U/log1p(-rho))
// (P:199-201), chunk-local chain restarted at chunk starts ("independently
// apply Bernoulli sampling to subranges").  Each batch of
// 2*BERN_NT skips is prefix-summed in one block scan (the paper's
// "prefix sums of geometric deviates", without materialising them);
// chunk offsets come from a single-pass decoupled look-back.
// ===========================================================================
__device__ __forceinline__ u64 skip_step(double U, double lr, u64 r)
{
    const double G = floor_(log_(U) / lr);
    return G >= (double)r ? r + 1 : (u64)G + 1;   // any G >= r ends the chain
}

__global__ void __launch_bounds__(BERN_NT) k_bernoulli(BernArgs a)
{
    __shared__ u64 vals[BERN_CAP];
    __shared__ u64 wtmp[BERN_NT / 32];
    __shared__ u64 tot;
    __shared__ u64 s_chunk, s_excl;
    const int tid = threadIdx.x;
    if (tid == 0) s_chunk = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const u64 c = s_chunk;
    const u64 gi = a.chunk0 + c;
    const u64 lo = bound_at(a.N, a.Db, gi);
    const u64 r = bound_at(a.N, a.Db, gi + 1) - lo;
    const Stream st(a.seed, P_GEO, ((u64)1 << a.Db) + gi);
    u64 S = 0;          // sum of steps before this batch
    u32 count = 0;
    bool overflow = false;
    for (u64 batch = 0;; ++batch) {
        const u64 q = batch * BERN_NT + tid;            // Philox block: draws 2q, 2q+1
        const u32x4 w = st.block((u32)q);
        const u64 s0 = skip_step(u52(w.x, w.y), a.log1m_rho, r);
        const u64 s1 = skip_step(u52(w.z, w.w), a.log1m_rho, r);
        const u64 pre = block_exclusive_scan<u64, BERN_NT>(s0 + s1, wtmp, &tot);
        const u64 S0 = S + pre + s0, S1 = S0 + s1;     // positions: lo + S - 1
        const u32 e0 = S0 <= r, e1 = S1 <= r;
        const u32 slot = count + 2 * tid;
        if (e0) { if (slot < BERN_CAP) vals[slot] = lo + S0; else overflow = true; }
        if (e1) { if (slot + 1 < BERN_CAP) vals[slot + 1] = lo + S1; else overflow = true; }
        const u32 emitted = __syncthreads_count(e0) + __syncthreads_count(e1);
        count += emitted;
        S += tot;
        if (emitted < 2u * BERN_NT) break;
        __syncthreads();
    }
    if (__syncthreads_or(overflow)) {
        if (tid == 0) atomicOr(&g_rs_errors, 2u);
        count = count < BERN_CAP ? count : BERN_CAP;
    }
    // decoupled look-back: flag bits 63:62 = 1 aggregate, 2 inclusive prefix
    const u64 AGG = 1ull << 62, INC = 2ull << 62, VAL = (1ull << 62) - 1;
    if (tid == 0) {
        volatile u64 *stat = a.status;
        u64 excl = 0;
        if (c == 0) {
            __threadfence();
            stat[0] = INC | count;
        } else {
            stat[c] = AGG | count;
            __threadfence();
            for (u64 p = c - 1;; --p) {
                u64 wv;
                do { wv = stat[p]; } while ((wv >> 62) == 0);
                excl += wv & VAL;
                if ((wv >> 62) == 2) break;
            }
            __threadfence();
            stat[c] = INC | (excl + count);
        }
        s_excl = excl;
        if (c == a.nchunks - 1) *a.count_dev = excl + count;
    }
    __syncthreads();
    const u64 excl = s_excl;
    for (u32 i = tid; i < count; i += BERN_NT) {
        const u64 gpos = excl + i;
        if (gpos < a.capacity) a.out[gpos] = vals[i];
    }
}

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
