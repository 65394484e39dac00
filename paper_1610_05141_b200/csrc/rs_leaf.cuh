// rs_leaf.cuh -- leaf kernels of the B200 sampler (rows a5-a8 of
// SURVEY.md section 8(a)), included by rs_kernels.cu.
// P:n = /root/reference/PAPER.md line n; CANON readings R1-R12: DESIGN.md.
//
// A leaf (D, i) covers offsets [lo, lo + r) and holds k sample values.  WOR:
// the values are the first k DISTINCT values of the leaf's draw stream
// x_0, x_1, ... (Algorithm H: "if X is already in T, reject it"),
// emitted sorted.  WR: the first k draws, sorted with repeats.
//
// On-chip algorithm (one CTA per leaf, draws in registers): a counting sort
// keyed by the monotone hash bucket(x) = x >> (ceil_log2(r) - log2 B), the
// "most significant bits" hash of P:162-164 whose order IS the sort order
// (P:370-374).  B ~ 2J buckets, so buckets hold ~0.5 draws:
//   1. draw -> shared-memory atomicAdd on the bucket's count (arrival slot);
//   2. exclusive scan of the counts -> bucket starts (word = start<<12|count);
//   3. scatter x to keys[start + slot];
//   4. draws in multi-draw buckets compute their rank inside the bucket and
//      move there (WR: ties by position; WOR: an equal value at a lower
//      position marks the draw a duplicate -> Algorithm H's rejection);
//   5. if duplicates were rejected and fewer than k distinct values remain,
//      the next round adds k - |S| draws (R7: rounds == sequential H).
// Three random shared-memory accesses per draw in the common case (1-3), one
// conflict-free 16-byte load per 4 outputs, 32-byte vector stores to HBM.

#include "rs_kernels.cuh"

namespace rs {


// A leaf the kernel cannot complete raises bit `bits` in the sticky device
// flag (rs_device_errors) and in the call's status word (returned as
// RS_ECAPACITY by the synchronous calls, include/rs.h).
__device__ __forceinline__ void leaf_flag(u32 *status, unsigned bits)
{
    atomicOr(&g_rs_errors, bits);
    if (status) atomicOr(status, bits);
}

__device__ __forceinline__ u32 leaf_cap(const LeafArgs &a)
{
    return (a.cap && a.cap < (u32)LEAF_CAP) ? a.cap : (u32)LEAF_CAP;
}

constexpr int LB_LOG_MIN = 10, LB_LOG_MAX = 12;
constexpr u32 LB_MAX = 1u << LB_LOG_MAX;          // buckets (and WR histogram slots)
constexpr u32 CNT_BITS = 12, CNT_MASK = (1u << CNT_BITS) - 1;
static_assert(LEAF_CAP <= (int)CNT_MASK + 1 && LEAF_CAP < (int)LB_MAX, "packing");

template <typename K>
struct SLeaf {
    u32 W[LB_MAX];              // bucket words: start << 12 | count (zero between leaves)
    K keys[LEAF_CAP + 4];       // sorted run at keys[h .. h+k), h = store alignment shift
    u32 bm[128];                // complement: excluded-value bitmap of one window
    u32 wpre[128];              // complement: clear-bit prefix per bitmap word
    u32 wsum[LEAF_NT / 32];
    u32 tot;
    u32 ndup;
};

// Lemire bounded draws from a leaf stream (R3): draw j at attempt 0 is word
// j mod EPB of block j / EPB; a rejected draw retries with block (j, attempt).
template <typename K> struct Drawer;

__device__ __noinline__ u32 lemire_retry32(Stream st, u32 j, u64 r, u32 thresh)
{
    for (u32 att = 1;; ++att) {
        const u64 prod = (u64)st.block(j, att).x * r;
        if ((u32)prod >= thresh) return (u32)(prod >> 32);
    }
}

__device__ __noinline__ u64 lemire_retry64(Stream st, u32 j, u64 r, u64 thresh)
{
    for (u32 att = 1;; ++att) {
        const u32x4 b = st.block(j, att);
        const u64 ww = ((u64)b.x << 32) | b.y;
        if (ww * r >= thresh) return __umul64hi(ww, r);
    }
}

template <> struct Drawer<u32> {
    static constexpr int EPB = 4;
    Stream st; u64 r; u32 thresh;
    __device__ Drawer(const Stream &s, u64 r_) : st(s), r(r_)
    {
        thresh = (r_ & (r_ - 1)) ? (u32)(0u - (u32)r_) % (u32)r_ : 0u;   // 2^32 mod r
    }
    __device__ __forceinline__ u32 fix(u32 w, u32 j) const
    {
        const u64 prod = (u64)w * r;
        if ((u32)prod < thresh) return lemire_retry32(st, j, r, thresh);
        return (u32)(prod >> 32);
    }
    __device__ __forceinline__ void block(u32 q, u32 *v) const
    {
        const u32x4 w = st.block(q);
        v[0] = fix(w.x, 4 * q + 0);
        v[1] = fix(w.y, 4 * q + 1);
        v[2] = fix(w.z, 4 * q + 2);
        v[3] = fix(w.w, 4 * q + 3);
    }
};

template <> struct Drawer<u64> {
    static constexpr int EPB = 2;
    Stream st; u64 r; u64 thresh;
    __device__ Drawer(const Stream &s, u64 r_) : st(s), r(r_)
    {
        thresh = (r_ & (r_ - 1)) ? (0 - r_) % r_ : 0;                    // 2^64 mod r
    }
    __device__ __forceinline__ u64 fix(u64 w, u32 j) const
    {
        if (w * r < thresh) return lemire_retry64(st, j, r, thresh);
        return __umul64hi(w, r);
    }
    __device__ __forceinline__ void block(u32 q, u64 *v) const
    {
        const u32x4 w = st.block(q);
        v[0] = fix(((u64)w.x << 32) | w.y, 2 * q + 0);
        v[1] = fix(((u64)w.z << 32) | w.w, 2 * q + 1);
    }
};

// In-place exclusive scan of the count fields of W[0..B), B in {1024, 2048,
// 4096}: thread t owns the B/LEAF_NT (2, 4 or 8) consecutive buckets from
// t*B/LEAF_NT, read and written as 8-byte pairs.
__device__ __forceinline__ void scan_buckets(u32 *W, u32 B, u32 *wsum, u32 *tot)
{
    constexpr u32 PMAX = (1u << LB_LOG_MAX) / LEAF_NT;
    const u32 per = B / LEAF_NT;
    const u32 beg = threadIdx.x * per;
    u32 v[PMAX];
    u32 s = 0;
#pragma unroll
    for (u32 i = 0; i < PMAX; i += 2) {
        if (i < per) {
            const uint2 q = *reinterpret_cast<const uint2 *>(&W[beg + i]);
            v[i] = q.x & CNT_MASK; v[i + 1] = q.y & CNT_MASK;
            s += v[i] + v[i + 1];
        }
    }
    u32 ex = block_exclusive_scan<u32, LEAF_NT>(s, wsum, tot);
#pragma unroll
    for (u32 i = 0; i < PMAX; i += 2) {
        if (i < per) {
            uint2 q;
            q.x = (ex << CNT_BITS) | v[i];     ex += v[i];
            q.y = (ex << CNT_BITS) | v[i + 1]; ex += v[i + 1];
            *reinterpret_cast<uint2 *>(&W[beg + i]) = q;
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void zero_words(u32 *W, u32 n)
{
    for (u32 i = threadIdx.x * 4; i < n; i += LEAF_NT * 4)
        *reinterpret_cast<uint4 *>(&W[i]) = make_uint4(0u, 0u, 0u, 0u);
}

// Step 5 of leaf_sorted (WOR with rejected duplicates, rare): keep the
// first copy of each value; its rank = number of distinct values below it in
// its bucket.  Driven from shared memory (keys holds every draw at its
// bucket position).  Returns 0 when the k distinct values are placed at
// keys[h..h+k), else the draw count J' = J + k - |S| of the next round
// (R7; W cleared for it).
template <typename K>
__device__ __noinline__ u32 dup_round(SLeaf<K> &sh, u32 J, u32 k, u32 h, int shb, u32 B)
{
    const u32 tid = threadIdx.x;
    K xs[LEAF_EPT];
    u32 dk[LEAF_EPT];
    u32 keep = 0, nd2 = 0;
#pragma unroll 1
    for (int i = 0; i < LEAF_EPT; ++i) {
        const u32 p = tid + (u32)LEAF_NT * i;
        if (p >= J) continue;
        const K xv = sh.keys[h + p];
        const u32 wd = sh.W[(u32)(xv >> shb)], s0 = wd >> CNT_BITS, c = wd & CNT_MASK;
        bool first = true;
        u32 d = 0;
        for (u32 t = 0; t < c; ++t) {
            const K y = sh.keys[h + s0 + t];
            if (y == xv && s0 + t < p) first = false;
            if (y < xv) {
                bool yfirst = true;
                for (u32 t2 = 0; t2 < t; ++t2) yfirst &= (sh.keys[h + s0 + t2] != y);
                d += yfirst;
            }
        }
        if (first) { keep |= 1u << i; xs[i] = xv; dk[i] = d; }
        else ++nd2;
    }
    __syncthreads();                              // all bucket words read before they change
#pragma unroll 1
    for (int i = 0; i < LEAF_EPT; ++i) {
        const u32 p = tid + (u32)LEAF_NT * i;
        if (p < J && !(keep & (1u << i)))
            atomicSub(&sh.W[(u32)(sh.keys[h + p] >> shb)], 1u);   // one value fewer in the bucket
    }
    if (nd2) atomicAdd(&sh.ndup, nd2);
    __syncthreads();
    const u32 d = J - sh.ndup;                    // |S| after this round
    __syncthreads();
    if (tid == 0) sh.ndup = 0;
    if (d < k) {                                  // next round: k - |S| more draws
        zero_words(sh.W, B);
        __syncthreads();
        return J + (k - d);
    }
    scan_buckets(sh.W, B, sh.wsum, &sh.tot);      // starts of the distinct values
#pragma unroll 1
    for (int i = 0; i < LEAF_EPT; ++i)
        if (keep & (1u << i))
            sh.keys[h + (sh.W[(u32)(xs[i] >> shb)] >> CNT_BITS) + dk[i]] = xs[i];
    __syncthreads();
    return 0;
}

// The leaf's sorted sample (relative offsets x in [0, r)) into
// sh.keys[h .. h + k).  On entry sh.W is all zero and sh.ndup == 0; on
// return W is dirty (the caller clears it) and ndup == 0.  Returns false on
// on-chip capacity overflow (more than cap <= LEAF_CAP draws needed; the
// caller raises the flag).
template <typename K, bool WR>
__device__ bool leaf_sorted(SLeaf<K> &sh, const Stream &st, u64 r, u32 k, u32 h, u32 cap)
{
    constexpr int EPB = Drawer<K>::EPB;
    constexpr int BPT = LEAF_EPT / EPB;            // Philox blocks per thread per round
    const u32 tid = threadIdx.x;
    const Drawer<K> dr(st, r);
    const int cr = ceil_log2(r);
    u32 J = k;                                     // draws of the rounds so far
    for (;;) {
        if (J > cap) return false;
        int logB = ceil_log2(J) + 1;
        logB = logB < LB_LOG_MIN ? LB_LOG_MIN : (logB > LB_LOG_MAX ? LB_LOG_MAX : logB);
        const u32 B = 1u << logB;
        const int shb = cr > logB ? cr - logB : 0;

        K x[LEAF_EPT];
        u32 sl[LEAF_EPT];      // arrival slot -> position -> rank
        u32 wv[LEAF_EPT];      // bucket word (start << 12 | count)
#define RS_VALID(i, w) ((tid + (u32)LEAF_NT * (i)) * EPB + (w) < J)
        // 1. draws of this round -> bucket counts (arrival slots)
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            const u32 q = tid + (u32)LEAF_NT * i;
            if (q * EPB < J) {
                K v[EPB];
                dr.block(q, v);
#pragma unroll
                for (int w = 0; w < EPB; ++w) {
                    const int e = i * EPB + w;
                    x[e] = v[w];
                    if (RS_VALID(i, w)) sl[e] = atomicAdd(&sh.W[(u32)(v[w] >> shb)], 1u);
                }
            }
        }
        __syncthreads();
        // 2. bucket starts
        scan_buckets(sh.W, B, sh.wsum, &sh.tot);
        // 3. scatter in bucket order
        bool multi = false;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
#pragma unroll
            for (int w = 0; w < EPB; ++w) {
                const int e = i * EPB + w;
                if (RS_VALID(i, w)) {
                    const u32 wd = sh.W[(u32)(x[e] >> shb)];
                    wv[e] = wd;
                    sl[e] += wd >> CNT_BITS;
                    sh.keys[h + sl[e]] = x[e];
                    multi |= (wd & CNT_MASK) > 1;
                }
            }
        }
        if (!__syncthreads_or(multi)) return true;       // all draws distinct: J == k
        // 4. rank inside multi-draw buckets
        u32 nd = 0;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
#pragma unroll
            for (int w = 0; w < EPB; ++w) {
                const int e = i * EPB + w;
                if (RS_VALID(i, w) && (wv[e] & CNT_MASK) > 1) {
                    const u32 s0 = wv[e] >> CNT_BITS, c = wv[e] & CNT_MASK, me = sl[e];
                    u32 rank = 0;
                    bool first = true;
                    for (u32 t = 0; t < c; ++t) {
                        const K y = sh.keys[h + s0 + t];
                        rank += (y < x[e]);
                        if (y == x[e] && s0 + t < me) {
                            if (WR) ++rank;                   // ties by position
                            else first = false;               // Algorithm H: reject
                        }
                    }
                    sl[e] = s0 + rank;
                    nd += !first;
                }
            }
        }
        if (WR || !__syncthreads_or(nd)) {
            if (WR) __syncthreads();
#pragma unroll
            for (int i = 0; i < BPT; ++i)
#pragma unroll
                for (int w = 0; w < EPB; ++w) {
                    const int e = i * EPB + w;
                    if (RS_VALID(i, w) && (wv[e] & CNT_MASK) > 1) sh.keys[h + sl[e]] = x[e];
                }
            __syncthreads();
            return true;
        }
        // 5. WOR with rejected duplicates (rare): out of line
        J = dup_round<K>(sh, J, k, h, shb, B);
        if (J == 0) return true;                      // else: next round with J draws
#undef RS_VALID
    }
}

__device__ __forceinline__ void st_v4(u64 *p, u64 a, u64 b, u64 c, u64 d)
{
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d)
                 : "memory");
}

__device__ __forceinline__ void load4(const u32 *p, u64 &a, u64 &b, u64 &c, u64 &d)
{
    const uint4 q = *reinterpret_cast<const uint4 *>(p);
    a = q.x; b = q.y; c = q.z; d = q.w;
}
__device__ __forceinline__ void load4(const u64 *p, u64 &a, u64 &b, u64 &c, u64 &d)
{
    const ulonglong2 q0 = *reinterpret_cast<const ulonglong2 *>(p);
    const ulonglong2 q1 = *reinterpret_cast<const ulonglong2 *>(p + 2);
    a = q0.x; b = q0.y; c = q1.x; d = q1.y;
}

// dst[i] = base + keys[h + i], i < k; dst - h is 32-byte aligned, so whole
// groups go out as 32-byte vector stores (row a6).
template <typename K>
__device__ __forceinline__ void store_run(const K *keys, u32 k, u32 h, u64 base, u64 *dst, u64 gV = 0)
{
    u64 *d0 = dst - h;
    const u32 ng = (h + k + 3) >> 2;
    for (u32 g = threadIdx.x; g < ng; g += LEAF_NT) {
        u64 v[4];
        load4(keys + 4 * g, v[0], v[1], v[2], v[3]);
        const int i0 = (int)(4 * g) - (int)h;
        if (i0 >= 0 && i0 + 4 <= (int)k) {
            st_v4(d0 + 4 * g, out_word(base + v[0], gV), out_word(base + v[1], gV), out_word(base + v[2], gV),
                  out_word(base + v[3], gV));
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (i0 + j >= 0 && i0 + j < (int)k) d0[4 * g + j] = out_word(base + v[j], gV);
        }
    }
}

struct LeafGeom { u64 lo, r, id; };

__device__ __forceinline__ LeafGeom leaf_geom(const LeafArgs &a, u64 L)
{
    const u64 gi = a.leaf0 + L;
    LeafGeom g;
    g.lo = bound_at(a.N, a.D, gi);
    g.r = bound_at(a.N, a.D, gi + 1) - g.lo;
    g.id = ((u64)1 << a.D) + gi;
    return g;
}

// WR leaves with more draws than the on-chip capacity (only when leaf
// ranges are tiny, e.g. n >> N): r == 1 -> k copies; r < LB_MAX ->
// histogram of all k draws, scan, emit runs by binary search.
template <typename K>
__device__ bool wr_big_leaf(SLeaf<K> &sh, const Stream &st, u64 lo, u64 r, u32 k, u64 *dst)
{
    const u64 base = lo + 1;
    if (r == 1) {
        for (u32 i = threadIdx.x; i < k; i += LEAF_NT) dst[i] = base;
        return true;
    }
    if (r >= LB_MAX) return false;
    u32 *hist = sh.W;                                  // zero on entry
    const Drawer<K> dr(st, r);
    constexpr int EPB = Drawer<K>::EPB;
    const u32 nblk = (k + EPB - 1) / EPB;
    for (u32 q = threadIdx.x; q < nblk; q += LEAF_NT) {
        K v[EPB];
        dr.block(q, v);
        for (int w = 0; w < EPB; ++w)
            if (q * EPB + w < k) atomicAdd(&hist[(u32)v[w]], 1u);
    }
    __syncthreads();
    block_scan_array<u32, LEAF_NT>(hist, (int)r, sh.wsum, &sh.tot);
    for (u32 t = threadIdx.x; t < k; t += LEAF_NT) {
        u32 a = 0, b = (u32)r;                          // last v with hist[v] <= t
        while (b - a > 1) {
            const u32 mid = (a + b) >> 1;
            if (hist[mid] <= t) a = mid; else b = mid;
        }
        dst[t] = base + a;
    }
    return true;
}

template <typename K>
__device__ __forceinline__ void leaf_init(SLeaf<K> &sh)
{
    zero_words(sh.W, LB_MAX);
    if (threadIdx.x == 0) sh.ndup = 0;
    __syncthreads();
}

// WOR (a5/a6) and WR (a8) leaves: one CTA per leaf, grid-stride over leaves.
// SPILLS: only the leaves of a warp kernel's spill list (a.spill, *a.spill_n),
// by one CTA (the fused kernels' last CTA).
template <typename K, bool WR, bool SPILLS = false>
__device__ __forceinline__ void sample_leaves(const LeafArgs &a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SLeaf<K> &sh = *reinterpret_cast<SLeaf<K> *>(smem_raw);
    leaf_init(sh);
    const u32 *list = SPILLS ? a.spill : a.list;
    const u64 nwork = SPILLS ? (u64)*(volatile const u32 *)a.spill_n : list ? (u64)*a.list_n : a.nleaves;
    const u64 first = SPILLS ? 0 : blockIdx.x, step = SPILLS ? 1 : gridDim.x;
    for (u64 it = first; it < nwork; it += step) {
        const u64 L = list ? (u64)((volatile const u32 *)list)[it] : it;
        const u32 k = a.cnt[L];
        if (k == 0) continue;
        const LeafGeom g = leaf_geom(a, L);
        const Stream st(a.seed, WR ? P_WR : P_WOR, g.id);
        u64 *dst = a.out + a.off[L];
        const u32 cap = leaf_cap(a);
        if (k > cap) {
            const bool ok = WR && wr_big_leaf<K>(sh, st, g.lo, g.r, k, dst);
            if (!ok && threadIdx.x == 0) leaf_flag(a.status, 1u);
        } else {
            const u32 h = (u32)(reinterpret_cast<uintptr_t>(dst) >> 3) & 3u;
            if (leaf_sorted<K, WR>(sh, st, g.r, k, h, cap)) store_run<K>(sh.keys, k, h, g.lo + 1, dst, a.gV);
            else if (threadIdx.x == 0) leaf_flag(a.status, 1u);
        }
        __syncthreads();
        zero_words(sh.W, LB_MAX);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_wor32(LeafArgs a) { sample_leaves<u32, false>(a); }
__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_wor64(LeafArgs a) { sample_leaves<u64, false>(a); }
__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_wr32(LeafArgs a) { sample_leaves<u32, true>(a); }
__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_wr64(LeafArgs a) { sample_leaves<u64, true>(a); }

// Complement leaves (a7): the leaf's output is [lo, lo + r) minus
// the e excluded values of the core leaf.  Work item = (leaf, window of
// COMP_TILE values): mark the window's excluded values in a bitmap, prefix-
// count the clear bits per 32-value word, and let each warp emit its words'
// clear values (lane l <-> value 32w + l: consecutive lanes write consecutive
// output positions, so the stores coalesce).
constexpr u64 COMP_TILE = 4096;
static_assert(COMP_TILE == 32 * 128, "bitmap of 128 words");

template <typename K>
__device__ __forceinline__ u32 lower_bound_s(const K *v, u32 n, u64 x)
{
    u32 a = 0, b = n;
    while (a < b) {
        const u32 m = (a + b) >> 1;
        if ((u64)v[m] < x) a = m + 1; else b = m;
    }
    return a;
}

template <typename K>
__device__ __forceinline__ void complement_leaves(const LeafArgs &a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SLeaf<K> &sh = *reinterpret_cast<SLeaf<K> *>(smem_raw);
    leaf_init(sh);
    const u32 tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const u64 total = a.nleaves * a.tiles_per_leaf;
    for (u64 T = blockIdx.x; T < total; T += gridDim.x) {
        const u64 L = T / a.tiles_per_leaf, tile = T - L * a.tiles_per_leaf;
        const LeafGeom g = leaf_geom(a, L);
        const u64 v0 = tile * COMP_TILE;
        if (v0 >= g.r) continue;
        const u32 nv = (u32)(g.r - v0 < COMP_TILE ? g.r - v0 : COMP_TILE);
        const u32 e = a.cnt[L];
        if (e > 0) {
            const Stream st(a.seed, P_WOR, g.id);
            const bool ok = leaf_sorted<K, false>(sh, st, g.r, e, 0, leaf_cap(a));
            __syncthreads();
            zero_words(sh.W, LB_MAX);
            if (!ok) {
                if (tid == 0) leaf_flag(a.status, 1u);
                __syncthreads();
                continue;
            }
        }
        const u32 i0 = lower_bound_s<K>(sh.keys, e, v0);
        const u32 i1 = lower_bound_s<K>(sh.keys, e, v0 + nv);
        if (tid < 128) sh.bm[tid] = 0;
        __syncthreads();
        for (u32 i = i0 + tid; i < i1; i += LEAF_NT) {
            const u32 o = (u32)((u64)sh.keys[i] - v0);
            atomicOr(&sh.bm[o >> 5], 1u << (o & 31));
        }
        __syncthreads();
        const u32 nw = (nv + 31) >> 5;
        u32 clear = 0;
        if (tid < nw) {
            const u32 valid = (tid + 1) * 32 <= nv ? 0xffffffffu : ((1u << (nv & 31)) - 1u);
            clear = ~sh.bm[tid] & valid;
        }
        const u32 pre = block_exclusive_scan<u32, LEAF_NT>((u32)__popc(clear), sh.wsum, &sh.tot);
        if (tid < nw) sh.wpre[tid] = pre;
        __syncthreads();
        // window output starts at leaf output index v0 - i0
        u64 *dst = a.out + (g.lo - a.out_base - a.off[L]) + (v0 - i0);
        const u64 base = g.lo + v0 + 1;
        for (u32 w = wid; w < nw; w += LEAF_NT / 32) {
            const u32 valid = (w + 1) * 32 <= nv ? 0xffffffffu : ((1u << (nv & 31)) - 1u);
            const u32 cw = ~sh.bm[w] & valid;
            if ((cw >> lane) & 1u)
                dst[sh.wpre[w] + __popc(cw & ((1u << lane) - 1u))] = out_word(base + 32 * w + lane, a.gV);
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_comp32(LeafArgs a) { complement_leaves<u32>(a); }
__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_comp64(LeafArgs a) { complement_leaves<u64>(a); }

}  // namespace rs
