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

// ===========================================================================
// Leaf machinery: sorted first-k-distinct (Algorithm H, sorted
// per P:356-374) or sorted multiset (WR), entirely in shared memory.
//
// Draws are bucketed by their top bits (the monotone "hash" of P:162-164 /
// bucket order IS sort order), counted with shared-memory
// atomics, scattered, and ranked inside their (small) bucket.  Rounds follow
// R7: round 1 = draws [0,k); if only d < k are distinct, the next round adds
// the next k-d draws (J grows) -- equal to sequential Algorithm H.
// ===========================================================================
template <typename K>
struct LeafShared {
    K keys[LEAF_CAP];            // bucket-scattered draws
    K stage[LEAF_CAP];           // sorted result
    u32 bstart[LEAF_CAP + 1];    // bucket counters -> starts
    u32 bdist[LEAF_CAP + 1];     // distinct counts -> starts (duplicate path)
    u32 wtmp[LEAF_NT / 32];
    u32 tot;
};

// Lemire bounded draws from a leaf stream (R3).
template <typename K> struct Drawer;

template <> struct Drawer<u32> {
    static constexpr int EPB = 4;        // draws per Philox block
    Stream st; u64 r; u32 thresh;
    __device__ Drawer(const Stream &s, u64 r_) : st(s), r(r_)
    {
        // 2^32 mod r (0 for powers of two: Lemire never rejects)
        thresh = (r_ & (r_ - 1)) ? (u32)(0u - (u32)r_) % (u32)r_ : 0u;
    }
    __device__ __forceinline__ u32 fix(u32 w, u64 j) const
    {
        u64 prod = (u64)w * r;
        if ((u32)prod < thresh) {
            for (u32 att = 1;; ++att) {
                prod = (u64)st.block((u32)j, att).x * r;
                if ((u32)prod >= thresh) break;
            }
        }
        return (u32)(prod >> 32);
    }
    __device__ __forceinline__ void block(u64 q, u32 *v) const
    {
        const u32x4 w = st.block((u32)q);
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
        thresh = (r_ & (r_ - 1)) ? (0 - r_) % r_ : 0;   // 2^64 mod r
    }
    __device__ __forceinline__ u64 fix(u64 w, u64 j) const
    {
        u64 lo = w * r, hi = __umul64hi(w, r);
        if (lo < thresh) {
            for (u32 att = 1;; ++att) {
                const u32x4 b = st.block((u32)j, att);
                const u64 ww = ((u64)b.x << 32) | b.y;
                lo = ww * r; hi = __umul64hi(ww, r);
                if (lo >= thresh) break;
            }
        }
        return hi;
    }
    __device__ __forceinline__ void block(u64 q, u64 *v) const
    {
        const u32x4 w = st.block((u32)q);
        v[0] = fix(((u64)w.x << 32) | w.y, 2 * q + 0);
        v[1] = fix(((u64)w.z << 32) | w.w, 2 * q + 1);
    }
};

// Result: sh.stage[0..k) sorted (distinct for WOR, with repeats for WR).
// Returns false on capacity overflow (flag raised).
template <typename K, bool WR>
__device__ bool leaf_core(LeafShared<K> &sh, const Stream &st, u64 r, u32 k)
{
    constexpr int EPB = Drawer<K>::EPB;
    constexpr int BPT = LEAF_EPT / EPB;     // Philox blocks per thread
    const int tid = threadIdx.x;
    const Drawer<K> dr(st, r);
    const int cr = ceil_log2(r);
    u32 J = k;
    for (;;) {
        if (J > (u32)LEAF_CAP) {
            if (tid == 0) atomicOr(&g_rs_errors, 1u);
            return false;
        }
        int logB = ceil_log2(J);
        if (logB < 5) logB = 5;
        const u32 B = 1u << logB;
        const int shift = cr > logB ? cr - logB : 0;
        for (u32 i = tid; i <= B; i += LEAF_NT) { sh.bstart[i] = 0; sh.bdist[i] = 0; }
        __syncthreads();

        // draws [0, J) -> registers; bucket histogram with arrival slots
        K x[LEAF_EPT];
        u32 arr[LEAF_EPT];
#pragma unroll
        for (int s = 0; s < BPT; ++s) {
            const u64 q = (u64)tid + (u64)LEAF_NT * s;
            if (q * EPB < J) {
                K v[EPB];
                dr.block(q, v);
#pragma unroll
                for (int w = 0; w < EPB; ++w) {
                    const int e = s * EPB + w;
                    x[e] = v[w];
                    if (q * EPB + w < J) arr[e] = atomicAdd(&sh.bstart[(u32)(v[w] >> shift)], 1u);
                }
            }
        }
        __syncthreads();
        block_scan_array<u32, LEAF_NT>(sh.bstart, (int)B, sh.wtmp, &sh.tot);

#pragma unroll
        for (int s = 0; s < BPT; ++s) {
            const u64 q = (u64)tid + (u64)LEAF_NT * s;
#pragma unroll
            for (int w = 0; w < EPB; ++w) {
                if (q * EPB + w < J) {
                    const int e = s * EPB + w;
                    sh.keys[sh.bstart[(u32)(x[e] >> shift)] + arr[e]] = x[e];
                }
            }
        }
        __syncthreads();

        // rank inside the bucket; optimistic store assuming no duplicates
        int dup = 0;
#pragma unroll
        for (int s = 0; s < BPT; ++s) {
            const u64 q = (u64)tid + (u64)LEAF_NT * s;
#pragma unroll
            for (int w = 0; w < EPB; ++w) {
                if (q * EPB + w < J) {
                    const int e = s * EPB + w;
                    const u32 b = (u32)(x[e] >> shift);
                    const u32 s0 = sh.bstart[b], c = sh.bstart[b + 1] - s0;
                    const u32 me = s0 + arr[e];
                    u32 rank = 0;
                    for (u32 t = s0; t < s0 + c; ++t) {
                        const K y = sh.keys[t];
                        rank += (y < x[e]);
                        if (y == x[e] && t < me) {
                            if (WR) ++rank; else dup = 1;
                        }
                    }
                    sh.stage[s0 + rank] = x[e];
                }
            }
        }
        if (WR) { __syncthreads(); return true; }
        if (!__syncthreads_or(dup)) return true;

        // duplicate path: keep the first copy (lowest slot) of each value
#pragma unroll
        for (int s = 0; s < BPT; ++s) {
            const u64 q = (u64)tid + (u64)LEAF_NT * s;
#pragma unroll
            for (int w = 0; w < EPB; ++w) {
                if (q * EPB + w < J) {
                    const int e = s * EPB + w;
                    const u32 b = (u32)(x[e] >> shift);
                    const u32 s0 = sh.bstart[b], me = s0 + arr[e];
                    bool first = true;
                    for (u32 t = s0; t < me; ++t) first &= (sh.keys[t] != x[e]);
                    if (first) atomicAdd(&sh.bdist[b], 1u);
                }
            }
        }
        __syncthreads();
        block_scan_array<u32, LEAF_NT>(sh.bdist, (int)B, sh.wtmp, &sh.tot);
        const u32 d = sh.bdist[B];
        if (d < k) {                 // next round: k - d more draws
            J += k - d;
            __syncthreads();
            continue;
        }
        __syncthreads();             // stage is rewritten below
#pragma unroll
        for (int s = 0; s < BPT; ++s) {
            const u64 q = (u64)tid + (u64)LEAF_NT * s;
#pragma unroll
            for (int w = 0; w < EPB; ++w) {
                if (q * EPB + w < J) {
                    const int e = s * EPB + w;
                    const u32 b = (u32)(x[e] >> shift);
                    const u32 s0 = sh.bstart[b], c = sh.bstart[b + 1] - s0, me = s0 + arr[e];
                    bool first = true;
                    for (u32 t = s0; t < me; ++t) first &= (sh.keys[t] != x[e]);
                    if (!first) continue;
                    u32 rank = 0;              // distinct values below x in the bucket
                    for (u32 t = s0; t < s0 + c; ++t) {
                        const K y = sh.keys[t];
                        if (!(y < x[e])) continue;
                        bool yfirst = true;
                        for (u32 t2 = s0; t2 < t; ++t2) yfirst &= (sh.keys[t2] != y);
                        rank += yfirst;
                    }
                    sh.stage[sh.bdist[b] + rank] = x[e];
                }
            }
        }
        __syncthreads();
        return true;
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

// WR leaves with more draws than the on-chip capacity.  This happens only
// when N < 2^D (leaf ranges r <= 1) -- e.g. n >> N -- or with probability
// < 1e-100 otherwise.  r == 1: k copies of lo+1 (the draws cannot change
// the value).  r <= WR_HIST: histogram of all k draws (smem atomics), scan,
// emit runs by binary search over the run starts.  Else: capacity flag.
constexpr u32 WR_HIST = 2 * LEAF_CAP - 1;

template <typename K>
__device__ void wr_big_leaf(LeafShared<K> &sh, const Stream &st, u64 lo, u64 r, u32 k, u64 *dst)
{
    const u64 base = lo + 1;
    if (r == 1) {
        for (u32 i = threadIdx.x; i < k; i += LEAF_NT) dst[i] = base;
        return;
    }
    if (r > WR_HIST) {
        if (threadIdx.x == 0) atomicOr(&g_rs_errors, 1u);
        return;
    }
    u32 *hist = reinterpret_cast<u32 *>(sh.keys);        // WR_HIST + 1 counters fit keys+stage
    for (u32 i = threadIdx.x; i <= (u32)r; i += LEAF_NT) hist[i] = 0;
    __syncthreads();
    const Drawer<K> dr(st, r);
    constexpr int EPB = Drawer<K>::EPB;
    const u64 nblk = ((u64)k + EPB - 1) / EPB;
    for (u64 q = threadIdx.x; q < nblk; q += LEAF_NT) {
        K v[EPB];
        dr.block(q, v);
        for (int w = 0; w < EPB; ++w)
            if (q * EPB + w < k) atomicAdd(&hist[(u32)v[w]], 1u);
    }
    __syncthreads();
    block_scan_array<u32, LEAF_NT>(hist, (int)r, sh.wtmp, &sh.tot);
    for (u32 t = threadIdx.x; t < k; t += LEAF_NT) {
        u32 a = 0, b = (u32)r;                          // last v with hist[v] <= t
        while (b - a > 1) {
            const u32 mid = (a + b) >> 1;
            if (hist[mid] <= t) a = mid; else b = mid;
        }
        dst[t] = base + a;
    }
}

// WOR (a5/a6) and WR (a8) leaves: draw, sort, store lo + x + 1 at the offset.
template <typename K, bool WR>
__device__ __forceinline__ void sample_leaves(const LeafArgs &a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LeafShared<K> &sh = *reinterpret_cast<LeafShared<K> *>(smem_raw);
    for (u64 L = blockIdx.x; L < a.nleaves; L += gridDim.x) {
        const u32 k = a.cnt[L];
        if (k == 0) continue;
        const LeafGeom g = leaf_geom(a, L);
        const Stream st(a.seed, WR ? P_WR : P_WOR, g.id);
        u64 *dst = a.out + a.off[L];
        if (WR && k > (u32)LEAF_CAP) {
            wr_big_leaf<K>(sh, st, g.lo, g.r, k, dst);
            __syncthreads();
            continue;
        }
        if (!leaf_core<K, WR>(sh, st, g.r, k)) continue;
        const u64 base = g.lo + 1;
        for (u32 i = threadIdx.x; i < k; i += LEAF_NT) dst[i] = base + (u64)sh.stage[i];
        __syncthreads();
    }
}

// ===========================================================================
// v2 leaf: Algorithm H with the paper's SORTED hash table (P:360-368,
// P:582-594).  The table has M ~ 2k slots plus an overflow area on the right
// ("n additional table entries ... unnecessary to wrap around");
// the hash is the monotone home(x) = floor(x M / 2^cr) ("extracting the most
// significant bits").  Insertion keeps every cluster sorted by
// "skipping elements smaller than k and shifting the cluster elements larger
// than k one position to the right": a thread carrying x walks
// right from home(x) past smaller keys and CAS-swaps x into the first slot
// holding a larger key (or EMPTY), then carries the displaced key onward.
// Slot contents only decrease and keys only move right, so concurrent
// insertion terminates and yields the unique ordered-probing table of the key
// set.  Equal keys: WOR drops the second copy (Algorithm H's rejection);
// WR keeps both.  Scanning the table in order then IS the sorted sample.
// ===========================================================================
constexpr int T_OVF = 256;                          // overflow slots (no wrap-around)
constexpr int T_MAX = 2 * LEAF_CAP + T_OVF;         // slots for k <= LEAF_CAP

template <typename K> struct Empty;
template <> struct Empty<u32> { static constexpr u32 v = 0xffffffffu; };
template <> struct Empty<u64> { static constexpr u64 v = ~0ull; };

template <typename K>
struct TableShared {
    K T[T_MAX];
    u32 wcnt[LEAF_NT / 32];
    u32 wpre[LEAF_NT / 32 + 1];
    u32 ndup;
};

__device__ __forceinline__ u32 cas_(u32 *p, u32 c, u32 v) { return atomicCAS(p, c, v); }
__device__ __forceinline__ u64 cas_(u64 *p, u64 c, u64 v)
{
    return (u64)atomicCAS((unsigned long long *)p, (unsigned long long)c, (unsigned long long)v);
}

// Insert x; returns 1 if x was a duplicate (WOR: dropped), 2 on overflow.
template <typename K, bool WR>
__device__ __forceinline__ int table_insert(K *T, K x, u32 p, u32 limit)
{
    for (;;) {
        const K y = *(volatile K *)&T[p];
        if (!WR && y == x) return 1;
        if (y < x || (WR && y == x)) {           // skip smaller (and equal, WR) keys
            if (++p >= limit) return 2;
            continue;
        }
        const K old = cas_(&T[p], y, x);       // y > x or EMPTY: take the slot
        if (old != y) continue;                // slot changed under us: re-read
        if (y == Empty<K>::v) return 0;
        x = y;                                 // carry the displaced key right
        if (++p >= limit) return 2;
    }
}

template <typename K>
__device__ __forceinline__ u32 home_of(K x, u32 M, int cr);
template <>
__device__ __forceinline__ u32 home_of<u32>(u32 x, u32 M, int cr) { return (u32)(((u64)x * M) >> cr); }
template <>
__device__ __forceinline__ u32 home_of<u64>(u64 x, u32 M, int cr)
{
    return (u32)(((unsigned __int128)x * M) >> cr);
}

// Insert a lane's pending draws q[0..n) with ONE loop, so a lane that
// finishes a short walk starts its next value in the same iteration (the
// warp then runs ~the sum of its lanes' walks, not 4 x the slowest walk).
// q is a register shift-queue (compile-time indices only).  Returns the
// number of duplicates (WOR) and sets *ovf on overflow.
template <typename K, bool WR, int NV>
__device__ __forceinline__ u32 insert_all(K *T, K (&q)[NV], int n, u32 M, int cr, u32 limit, bool *ovf)
{
    u32 dups = 0;
    K x = q[0];
    u32 p = home_of<K>(x, M, cr);
    while (n > 0) {
        bool done = false;
        const K y = *(volatile K *)&T[p];
        if (!WR && y == x) {                       // Algorithm H: reject the duplicate
            ++dups;
            done = true;
        } else if (y < x || (WR && y == x)) {      // skip smaller keys
            if (++p >= limit) { *ovf = true; return dups; }
        } else {
            const K old = cas_(&T[p], y, x);       // y > x or EMPTY: take the slot
            if (old == y) {
                if (y == Empty<K>::v) done = true;
                else { x = y; if (++p >= limit) { *ovf = true; return dups; } }   // carry y right
            }
        }
        if (done) {
#pragma unroll
            for (int t = 0; t + 1 < NV; ++t) q[t] = q[t + 1];
            --n;
            x = q[0];
            p = home_of<K>(x, M, cr);
        }
    }
    return dups;
}

template <typename K, bool WR>
__device__ __forceinline__ void sample_leaves_v2(const LeafArgs &a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TableShared<K> &sh = *reinterpret_cast<TableShared<K> *>(smem_raw);
    constexpr int EPB = Drawer<K>::EPB;
    constexpr int BPT = LEAF_EPT / EPB;               // Philox blocks per thread per round
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (u64 L = blockIdx.x; L < a.nleaves; L += gridDim.x) {
        const u32 k = a.cnt[L];
        if (k == 0) continue;
        const LeafGeom g = leaf_geom(a, L);
        const Stream st(a.seed, WR ? P_WR : P_WOR, g.id);
        u64 *dst = a.out + a.off[L];
        if (k > (u32)LEAF_CAP) {                 // beyond on-chip capacity
            if (WR) wr_big_leaf<K>(*reinterpret_cast<LeafShared<K> *>(smem_raw), st, g.lo, g.r, k, dst);
            else if (tid == 0) atomicOr(&g_rs_errors, 1u);
            __syncthreads();
            continue;
        }
        const u32 M = ((2 * k + 255) / 256) * 256;    // ~2k slots, multiple of 256
        const u32 TS = M + T_OVF;                     // scanned slots (multiple of 256)
        const int cr = ceil_log2(g.r);
        {
            uint4 *T4 = reinterpret_cast<uint4 *>(sh.T);
            const uint4 e4 = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
            for (u32 i = tid; i < TS * sizeof(K) / 16; i += LEAF_NT) T4[i] = e4;
        }
        if (tid == 0) sh.ndup = 0;
        __syncthreads();
        const Drawer<K> dr(st, g.r);
        u32 J0 = 0, J = k, have = 0;
        bool overflow = false;
        for (;;) {                                     // rounds of Algorithm H
            const u32 q0 = J0 / EPB, q1 = (J + EPB - 1) / EPB;
            // this thread's draws of the round, packed into a register queue
            K v[LEAF_EPT];
            int nv = 0;
#pragma unroll
            for (int s = 0; s < BPT; ++s) {
                const u32 q = q0 + tid + LEAF_NT * s;
                K b[EPB];
                if (q < q1) dr.block(q, b);
#pragma unroll
                for (int w = 0; w < EPB; ++w) {
                    const u32 j = q * EPB + w;
                    const bool ok = q < q1 && j >= J0 && j < J;
                    // append b[w] at position nv (unrolled select: no local memory)
#pragma unroll
                    for (int t = 0; t < LEAF_EPT; ++t)
                        if (ok && t == nv) v[t] = b[w];
                    nv += ok;
                }
            }
            const u32 dups = nv ? insert_all<K, WR, LEAF_EPT>(sh.T, v, nv, M, cr, TS, &overflow) : 0u;
            const u32 wd = __reduce_add_sync(0xffffffffu, dups);     // duplicates this round
            if (lane == 0 && wd) atomicAdd(&sh.ndup, wd);
            if (__syncthreads_or(overflow)) break;
            const u32 nd = sh.ndup;
            have += (J - J0) - nd;
            if (WR || have == k) break;
            __syncthreads();                           // all threads have read ndup
            if (tid == 0) sh.ndup = 0;
            __syncthreads();
            J0 = J;
            J += k - have;                             // next round: k - |S| draws
        }
        if (__syncthreads_or(overflow)) {
            if (tid == 0) atomicOr(&g_rs_errors, 1u);
            continue;
        }
        // in-place per-warp compaction of the table (warp w owns TS/8 slots)
        const u32 per = TS / (LEAF_NT / 32);
        K *reg = sh.T + wid * per;
        u32 c = 0;
        for (u32 i = 0; i < per; i += 32) {
            const K v = reg[i + lane];
            const bool occ = v != Empty<K>::v;
            const u32 m = __ballot_sync(0xffffffffu, occ);
            if (occ) reg[c + __popc(m & ((1u << lane) - 1))] = v;
            c += __popc(m);
            __syncwarp();
        }
        if (lane == 0) sh.wcnt[wid] = c;
        __syncthreads();
        if (tid == 0) {
            u32 acc = 0;
            for (int w = 0; w < LEAF_NT / 32; ++w) { sh.wpre[w] = acc; acc += sh.wcnt[w]; }
            sh.wpre[LEAF_NT / 32] = acc;
        }
        __syncthreads();
        const u32 o = sh.wpre[wid];
        const u64 base = g.lo + 1;
        for (u32 t = lane; t < c; t += 32) dst[o + t] = base + (u64)reg[t];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(LEAF_NT, 4) k_leaf_wor32(LeafArgs a) { sample_leaves_v2<u32, false>(a); }
__global__ void __launch_bounds__(LEAF_NT) k_leaf_wor64(LeafArgs a) { sample_leaves_v2<u64, false>(a); }
__global__ void __launch_bounds__(LEAF_NT, 4) k_leaf_wr32(LeafArgs a) { sample_leaves_v2<u32, true>(a); }
__global__ void __launch_bounds__(LEAF_NT) k_leaf_wr64(LeafArgs a) { sample_leaves_v2<u64, true>(a); }

// Complement leaves (a7): emit [lo, lo+r) minus the core leaf's
// e excluded values.  Output index t of the leaf maps to offset t + j(t),
// j(t) = #{i : E_i - i <= t} (E sorted), found by binary search.  Large
// leaves are split into tiles of COMP_TILE outputs across CTAs.
constexpr u64 COMP_TILE = 8192;

template <typename K>
__device__ __forceinline__ void complement_leaves(const LeafArgs &a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LeafShared<K> &sh = *reinterpret_cast<LeafShared<K> *>(smem_raw);
    const u64 total = a.nleaves * a.tiles_per_leaf;
    for (u64 T = blockIdx.x; T < total; T += gridDim.x) {
        const u64 L = T / a.tiles_per_leaf, tile = T - L * a.tiles_per_leaf;
        const u32 e = a.cnt[L];
        const LeafGeom g = leaf_geom(a, L);
        const u64 outc = g.r - e;
        const u64 t0 = tile * COMP_TILE;
        if (t0 >= outc) continue;
        const u64 t1 = t0 + COMP_TILE < outc ? t0 + COMP_TILE : outc;
        if (e > 0) {
            const Stream st(a.seed, P_WOR, g.id);
            if (!leaf_core<K, false>(sh, st, g.r, e)) continue;
        }
        u64 *dst = a.out + (g.lo - a.out_base - a.off[L]);
        const u64 base = g.lo + 1;
        for (u64 t = t0 + threadIdx.x; t < t1; t += LEAF_NT) {
            u32 lo_i = 0, hi_i = e;
            while (lo_i < hi_i) {
                const u32 mid = (lo_i + hi_i) >> 1;
                if ((u64)sh.stage[mid] - mid <= t) lo_i = mid + 1; else hi_i = mid;
            }
            dst[t] = base + t + lo_i;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(LEAF_NT) k_leaf_comp32(LeafArgs a) { complement_leaves<u32>(a); }
__global__ void __launch_bounds__(LEAF_NT) k_leaf_comp64(LeafArgs a) { complement_leaves<u64>(a); }

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
