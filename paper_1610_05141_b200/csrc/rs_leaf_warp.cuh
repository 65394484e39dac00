// rs_leaf_warp.cuh -- the common-path leaf kernel: ONE WARP PER LEAF
// (rows a5, a6, a8 of SURVEY.md section 8(a)); included by rs_kernels.cu
// after rs_leaf.cuh.  P:n = /root/reference/PAPER.md line n.
//
// Same result as leaf_sorted (rs_leaf.cuh): the leaf's first k distinct
// draws (WOR, Algorithm H) or first k draws (WR), sorted
// (P:356-374), value lo + x + 1.  A leaf holds ~n0 = 1024 draws, i.e. 32-44
// per lane, so a warp owns it end to end with no CTA barrier, the draws stay
// in registers, and ~20 independent leaves are in flight per SM.
//
// Per round of J draws (R7), with B = 1024 monotone-hash buckets
// bucket(x) = x >> (ceil_log2(r) - 10) (the hash order is the sort
// order), held as u32 counters:
//   1. Philox blocks (lane l: blocks l + 32m) -> draws -> RED.ADD count[bucket],
//      and the draws are staged in draw order (16-byte stores);
//   2. warp scan of the counts (XOR-swizzled so every access is conflict-free)
//      -> bucket starts; max bucket load P;
//   3. the staged draws come back into registers; ATOMS.ADD on the start ->
//      final position (+ h, the store alignment shift), scatter the draw
//      there: positions are now sorted by bucket;
//   4. lane l loads positions [E l, E l + E) into registers; P phases of
//      odd-even transposition sort the (tiny) buckets -- a bucket of c draws
//      is sorted after c phases, and draws of different buckets never swap;
//   5. WOR: equal neighbours are duplicates (Algorithm H rejects them); if
//      fewer than k distinct values remain the next round draws k - |S| more
//      (J += k - |S|) and restarts; otherwise
//   6. 32-byte vector stores straight from registers (positions are aligned to
//      the output's 32-byte grid by h), or via shared memory after
//      compacting out the duplicates.
// Leaves that do not fit (J + h > 32 * WL_E2, or a bucket load above WL_PMAX)
// are appended to a spill list that the CTA kernel (rs_leaf.cuh) completes.

#ifndef RS_WL_SMEMST_GR
#define RS_WL_SMEMST_GR 1   // the same, for the G(n, m) kernels only (measured gnm leaf 22.38 -> 21.99 ms)
#endif
#ifndef RS_WL_SMEMST
#define RS_WL_SMEMST 0      // base / output pointer through shared memory (measured 14.03 -> 13.74 ms with the plain kernel; with the spill-free top-up kernel off is faster: 12.87 -> 12.64 ms)
#endif
#ifndef RS_WL_RANK
#define RS_WL_RANK 0        // count atomics return the rank in the bucket (u8 per draw); the scatter reads start + rank
#endif
#ifndef RS_WL_TUV4
#define RS_WL_TUV4 0        // top-up merge stored by output slot, 32-byte stores (bit-exact; measured slower: cfg1 leaf 4.99 -> 5.56 ms)
#endif
#ifndef RS_WL_CB
#define RS_WL_CB 2          // Philox blocks per count step (> 2: generic loop)
#endif
#ifndef RS_WL_EXACTP
#define RS_WL_EXACTP 1      // exactly P odd-even phases (not P rounded up to even)
#endif
#ifndef RS_WL_MINB
#define RS_WL_MINB 1          // resident CTAs per SM the register budget is sized for (16 warps)
#endif
#ifndef RS_WL_GB
#define RS_WL_GB 3          // scatter group (blocks); measured: headline leaf 14.06 (1) / 13.66 (3) / 14.09 ms (9)
#endif

namespace rs {

#ifdef RS_EXP_CLOCK
__device__ unsigned long long g_rs_prof[8];
#define RS_TS(var) const long long var = clock64()
#define RS_ACC(i, a, b) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_rs_prof[i], (unsigned long long)((b) - (a))); } while (0)
#else
#define RS_TS(var)
#define RS_ACC(i, a, b)
#endif

constexpr int WL_B = 1024;                 // buckets (u32 counters)
constexpr int WL_LOGB = 10;
constexpr int WL_E1 = 36, WL_E2 = 44;      // positions per lane; E mod 32 in {4, 12}: conflict-free LDS.128
#ifdef RS_WL_TWO_E
constexpr int WL_CAP = 32 * WL_E2;         // 1408 positions per leaf
#else
constexpr int WL_CAP = 32 * WL_E1;         // 1152 positions per leaf
#endif
constexpr u32 WL_PMAX = 48;                // odd-even phases allowed before spilling

constexpr u32 WL_SENT0 = 0xFFFFFFFFu - (u32)WL_CAP;   // sentinel at position p: WL_SENT0 + p (> any key)

struct WarpLeaf {
    u32 cnt[WL_B + WL_B / 32];             // padded bucket counters / starts (33 words per lane)
    unsigned long long pf_off;             // prefetched count / offset of the warp's next leaf
    u32 pf_k, pf_pad;                      //   (in shared memory: not live in registers)
#if RS_WL_SMEMST || RS_WL_SMEMST_GR
    unsigned long long cur_base, cur_dst;  // the current leaf's base value / output pointer
#endif
    u32 keys[WL_CAP];                      // staging (draw order), then positions: pad, draws, sentinels
#if RS_WL_RANK
    u32 rank[WL_CAP / 4];                  // draw j's rank in its bucket: byte j & 3 of word j >> 2
#endif
};

// Word of bucket b's counter.  Lane l owns buckets [32 l, 32 l + 32) for the
// scan; bucket 32 l + i lives at word 33 l + i, so the scan's accesses (fixed
// i across lanes) hit 32 distinct banks and use immediate offsets.
__device__ __forceinline__ u32 wl_word(u32 b)
{
    return b + (b >> 5);
}

__device__ __forceinline__ u32 shr32(u32 v, u32 s)   // v >> s, 0 for s == 32
{
    u32 r;
    asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(s));
    return r;
}

// Four bounded draws of block q (R3): Lemire's multiply-shift, which for a
// power-of-two range is the top ceil_log2(r) bits (never rejects).  The
// Philox round keys come from the kernel arguments (constant bank).
struct WDrawer {
    Drawer<u32> d;
    u32 s;          // 32 - ceil_log2(r)
    bool pow2;
    __device__ WDrawer(const Stream &st, u64 r, int cr) : d(st, r), s(32u - (u32)cr), pow2((r & (r - 1)) == 0) {}
    // power-of-two range: the top cr bits of each word (Lemire never rejects)
    __device__ __forceinline__ void block_pow2(const RoundKeys &K, u32 q, u32 *v) const
    {
        u32 c0 = q, c1 = d.st.tag, c2 = d.st.id_lo, c3 = d.st.id_hi;
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            const u64 p0 = (u64)0xD2511F53u * c0, p1 = (u64)0xCD9E8D57u * c2;
            c0 = (u32)(p1 >> 32) ^ c1 ^ K.k[2 * r];
            c1 = (u32)p1;
            c2 = (u32)(p0 >> 32) ^ c3 ^ K.k[2 * r + 1];
            c3 = (u32)p0;
        }
        v[0] = shr32(c0, s); v[1] = shr32(c1, s); v[2] = shr32(c2, s); v[3] = shr32(c3, s);
    }
    template <bool P2 = false>
    __device__ __forceinline__ void block(const RoundKeys &K, u32 q, u32 *v) const
    {
#ifdef RS_EXP_NOPHILOX
        { const u32 t = q * 0x9E3779B9u ^ d.st.id_lo; v[0] = shr32(t, s); v[1] = shr32(t * 3u, s); v[2] = shr32(t * 5u, s); v[3] = shr32(t * 7u, s); return; }
#endif
        if (P2 || pow2) {          // P2: every leaf range of the launch is a power of two
            u32 c0 = q, c1 = d.st.tag, c2 = d.st.id_lo, c3 = d.st.id_hi;
#pragma unroll
            for (int r = 0; r < 10; ++r) {
                const u64 p0 = (u64)0xD2511F53u * c0, p1 = (u64)0xCD9E8D57u * c2;
                c0 = (u32)(p1 >> 32) ^ c1 ^ K.k[2 * r];
                c1 = (u32)p1;
                c2 = (u32)(p0 >> 32) ^ c3 ^ K.k[2 * r + 1];
                c3 = (u32)p0;
            }
            v[0] = shr32(c0, s); v[1] = shr32(c1, s); v[2] = shr32(c2, s); v[3] = shr32(c3, s);
        } else {
            d.block(q, v);
        }
    }
};

// Compiler fence: memory operations are not moved across it, which keeps
// the scheduler from batching every atomic / store of an unrolled loop
// (and holding all their operands in registers at once).
__device__ __forceinline__ void wl_fence() { asm volatile("" ::: "memory"); }

__device__ __forceinline__ void wl_ce(u32 &a, u32 &b)
{
    const u32 lo = min(a, b), hi = max(a, b);
    a = lo; b = hi;
}

__device__ __forceinline__ u32 warp_excl_scan(u32 v, u32 lane)
{
    u32 incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (u32)o) incl += y;
    }
    return incl - v;
}

__device__ __forceinline__ u32 wl_scan(WarpLeaf &sh, u32 lane);

// Steps 1-2: count the round's J draws per bucket and stage them in draw
// order at keys[0..J); scan the counts into starts.  Returns the largest
// bucket load (0 if a bucket is a single value).
template <bool P2>
__device__ __forceinline__ u32 wl_count(WarpLeaf &sh, const RoundKeys &K, const WDrawer &dr, u32 J, int shb, u32 lane)
{
    RS_TS(tc0);
    const u32 qfull = J >> 2;                    // blocks whose 4 draws all count
    const u32 nq = (J + 3) >> 2;                 // blocks of the round
#if RS_WL_CB > 2
    // RS_WL_CB independent Philox blocks per step (ILP)
#pragma unroll 1
    for (u32 q0 = lane; q0 < nq; q0 += 32 * RS_WL_CB) {
        u32 v[RS_WL_CB][4];
#pragma unroll
        for (int c = 0; c < RS_WL_CB; ++c) dr.block<P2>(K, q0 + 32 * c, v[c]);
        if (q0 + 32 * (RS_WL_CB - 1) < qfull) {
#pragma unroll
            for (int w = 0; w < 4; ++w)
#pragma unroll
                for (int c = 0; c < RS_WL_CB; ++c) atomicAdd(&sh.cnt[wl_word(v[c][w] >> shb)], 1u);
        } else {
#pragma unroll
            for (int w = 0; w < 4; ++w)
#pragma unroll
                for (int c = 0; c < RS_WL_CB; ++c)
                    if (4 * (q0 + 32 * c) + w < J) atomicAdd(&sh.cnt[wl_word(v[c][w] >> shb)], 1u);
        }
#pragma unroll
        for (int c = 0; c < RS_WL_CB; ++c)
            if (q0 + 32 * c < nq)
                *reinterpret_cast<uint4 *>(&sh.keys[4 * (q0 + 32 * c)]) = make_uint4(v[c][0], v[c][1], v[c][2], v[c][3]);
    }
#else
#pragma unroll 1
    for (u32 q = lane; q < nq; q += 64) {        // two independent Philox blocks per step (ILP)
        const u32 q2 = q + 32;
        u32 v[4], v2[4];
        dr.block<P2>(K, q, v);
        dr.block<P2>(K, q2, v2);
#if RS_WL_RANK && !defined(RS_WL_REGEN)
        // ATOMS with return: the old count is the draw's rank in its bucket
        // (ranks above 255 wrap, but then the bucket load exceeds WL_PMAX and
        // the leaf spills before the ranks are read)
        u32 rk = 0, rk2 = 0;
        if (q2 < qfull) {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                rk |= (atomicAdd(&sh.cnt[wl_word(v[w] >> shb)], 1u) & 0xffu) << (8 * w);
                rk2 |= (atomicAdd(&sh.cnt[wl_word(v2[w] >> shb)], 1u) & 0xffu) << (8 * w);
            }
        } else {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                if (4 * q + w < J) rk |= (atomicAdd(&sh.cnt[wl_word(v[w] >> shb)], 1u) & 0xffu) << (8 * w);
                if (4 * q2 + w < J) rk2 |= (atomicAdd(&sh.cnt[wl_word(v2[w] >> shb)], 1u) & 0xffu) << (8 * w);
            }
        }
        sh.rank[q] = rk;
        if (q2 < nq) sh.rank[q2] = rk2;
#else
        if (q2 < qfull) {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
#ifndef RS_EXP_NOCOUNT
                atomicAdd(&sh.cnt[wl_word(v[w] >> shb)], 1u);
                atomicAdd(&sh.cnt[wl_word(v2[w] >> shb)], 1u);
#endif
            }
        } else {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                if (4 * q + w < J) atomicAdd(&sh.cnt[wl_word(v[w] >> shb)], 1u);
                if (4 * q2 + w < J) atomicAdd(&sh.cnt[wl_word(v2[w] >> shb)], 1u);
            }
        }
#endif
#if !defined(RS_WL_REGEN)
        *reinterpret_cast<uint4 *>(&sh.keys[4 * q]) = make_uint4(v[0], v[1], v[2], v[3]);
        if (q2 < nq) *reinterpret_cast<uint4 *>(&sh.keys[4 * q2]) = make_uint4(v2[0], v2[1], v2[2], v2[3]);
#endif
    }
#endif
    __syncwarp();
    RS_TS(tc1);
    const u32 P = wl_scan(sh, lane);
    RS_TS(tc2);
    RS_ACC(0, tc0, tc1);
    RS_ACC(1, tc1, tc2);
    return shb == 0 ? 0u : P;
}

// Step 2: scan the 1024 bucket counts (lane l owns buckets [32 l, 32 l + 32)
// at words 33 l + i: conflict-free) into starts; returns the largest load.
__device__ __forceinline__ u32 wl_scan(WarpLeaf &sh, u32 lane)
{
    u32 *cl = sh.cnt + 33 * lane;
    u32 c[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) c[i] = cl[i];
    u32 seg[4], mx4[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {                // four independent chains (ILP)
        seg[g] = 0; mx4[g] = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) { seg[g] += c[8 * g + i]; mx4[g] = max(mx4[g], c[8 * g + i]); }
    }
    const u32 S = (seg[0] + seg[1]) + (seg[2] + seg[3]);
    const u32 mx = max(max(mx4[0], mx4[1]), max(mx4[2], mx4[3]));
    const u32 run = warp_excl_scan(S, lane);
    const u32 P = __reduce_max_sync(0xffffffffu, mx);
    u32 rg[4];
    rg[0] = run; rg[1] = run + seg[0]; rg[2] = rg[1] + seg[1]; rg[3] = rg[2] + seg[2];
#pragma unroll
    for (int i = 0; i < 8; ++i) {                // starts in place, four chains
#pragma unroll
        for (int g = 0; g < 4; ++g) { cl[8 * g + i] = rg[g]; rg[g] += c[8 * g + i]; }
    }
    __syncwarp();
    return P;
}

#ifndef RS_WL_REG
#define RS_WL_REG 0         // 1: draws stay in registers from the count to the scatter (no staging round trip) in every kernel
#endif
#ifndef RS_WL_GBR
#define RS_WL_GBR RS_WL_GB  // scatter group of the register-resident path (measured 1 / 3 / 9: equal / best / 6 % slower)
#endif
#ifndef RS_WL_REG_WR
#define RS_WL_REG_WR 1      // register-resident count/scatter in the power-of-two WR kernel (measured: 10.91 -> 10.16 ms once the kernels were slimmed; slower before)
#endif
#ifndef RS_WL_REG_P2
#define RS_WL_REG_P2 1      // ... in the power-of-two WOR kernels only (spill-free there)
#endif

// Monotone bucket of a draw x < 2^cr (cr >= 11), 1056 buckets:
// b = floor(33 x / 2^(cr - 5)) = hi(x * M), M = 33 << (37 - cr) -- one
// IMAD.HI.  Bucket b's counter is word b: lane l owns the words
// [33 l, 33 l + 33) in the scan (stride 33: conflict-free).
__device__ __forceinline__ u32 wl_bucket_mult(int cr) { return 33u << (37 - cr); }

// hi(x * M) as an opaque instruction: recomputed at each use (the count and
// the scatter) instead of 36 bucket indices held in registers across the scan.
__device__ __forceinline__ u32 wl_bkt(u32 x, u32 M)
{
    u32 b;
    asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(b) : "r"(x), "r"(M));
    return b;
}

// Steps 1-2 with the round's draws kept in registers: lane l's blocks
// l + 32 m (m < 9) -> x[4 m .. 4 m + 3]; RED.ADD count[bucket]; scan the
// counts into starts.  Returns the largest bucket load.
template <bool POW2>
__device__ __forceinline__ u32 wl_count_reg(WarpLeaf &sh, const RoundKeys &K, const WDrawer &dr, u32 J, u32 M,
                                            u32 lane, u32 (&x)[WL_E1])
{
    constexpr int NB = WL_E1 / 4;
    // group m = draws [128 m, 128 m + 128): full groups straight from the
    // unrolled loop; the one partial group (J mod 128 != 0) after it, its
    // draws selected out of x -- one copy of the per-draw tests (this kernel
    // is instruction-fetch sensitive); groups beyond J are not generated
#pragma unroll
    for (int m = 0; m < NB; ++m) {
        if (128u * m < J) {
            const u32 q = lane + 32u * m;
            if (POW2) dr.block_pow2(K, q, &x[4 * m]);
            else dr.d.block(q, &x[4 * m]);
            if (128u * m + 127u < J) {
#pragma unroll
                for (int t = 0; t < 4; ++t) atomicAdd(&sh.cnt[wl_bkt(x[4 * m + t], M)], 1u);
            }
        }
    }
    const u32 mp = J >> 7;
    if ((J & 127u) && mp < (u32)NB) {
        u32 v[4] = {x[0], x[1], x[2], x[3]};
#pragma unroll
        for (int m = 1; m < NB; ++m)
            if ((u32)m == mp) { v[0] = x[4 * m]; v[1] = x[4 * m + 1]; v[2] = x[4 * m + 2]; v[3] = x[4 * m + 3]; }
        const u32 q = lane + 32u * mp;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (4 * q + t < J) atomicAdd(&sh.cnt[wl_bkt(v[t], M)], 1u);
    }
    __syncwarp();
    u32 *cl = sh.cnt + 33 * lane;
    u32 c[33];
#pragma unroll
    for (int i = 0; i < 33; ++i) c[i] = cl[i];
    u32 seg[3], mx3[3];
#pragma unroll
    for (int g = 0; g < 3; ++g) {                // three independent chains (ILP)
        seg[g] = 0; mx3[g] = 0;
#pragma unroll
        for (int i = 0; i < 11; ++i) { seg[g] += c[11 * g + i]; mx3[g] = max(mx3[g], c[11 * g + i]); }
    }
    const u32 S = seg[0] + seg[1] + seg[2];
    const u32 mx = max(max(mx3[0], mx3[1]), mx3[2]);
    const u32 run = warp_excl_scan(S, lane);
    const u32 P = __reduce_max_sync(0xffffffffu, mx);
    u32 rg[3];
    rg[0] = run; rg[1] = run + seg[0]; rg[2] = rg[1] + seg[1];
#pragma unroll
    for (int i = 0; i < 11; ++i) {               // starts in place, three chains
#pragma unroll
        for (int g = 0; g < 3; ++g) { cl[11 * g + i] = rg[g]; rg[g] += c[11 * g + i]; }
    }
    __syncwarp();
    return P;
}

// Step 3 from registers: every draw to its bucket's next position (+ h).
__device__ __forceinline__ void wl_scatter_reg(WarpLeaf &sh, u32 J, u32 h, u32 M, u32 lane, const u32 (&x)[WL_E1])
{
    u32 *kh = sh.keys + h;
    constexpr int NB = WL_E1 / 4;
    constexpr int GB = RS_WL_GBR;
    static_assert(NB % GB == 0, "group size");
    // full GB-groups of groups from the unrolled loop; the rest (at most GB
    // groups, the last one partial) one group at a time after it, each
    // group's draws selected out of x: one copy of the per-draw tests
    u32 mr0 = 0;                                 // first group not in a full GB-group
#pragma unroll
    for (int m0 = 0; m0 < NB; m0 += GB) {
        if (128u * (m0 + GB - 1) + 127u < J) {   // the GB-group's draws all exist for every lane
            u32 pos[4 * GB];
#pragma unroll
            for (int e = 4 * m0; e < 4 * (m0 + GB); ++e) pos[e - 4 * m0] = atomicAdd(&sh.cnt[wl_bkt(x[e], M)], 1u);
            // atomics first, stores after (smem stores and atomics may alias as far
            // as the compiler knows: interleaving would serialise every round trip)
#pragma unroll
            for (int e = 4 * m0; e < 4 * (m0 + GB); ++e) { RS_CHK(h + pos[e - 4 * m0] < (u32)WL_CAP); kh[pos[e - 4 * m0]] = x[e]; }
            mr0 = m0 + GB;
        }
    }
    // (group mr0 + g: mr0 is a multiple of GB, so a (NB / GB)-way select)
#pragma unroll
    for (int g = 0; g < GB; ++g) {
        const u32 m = mr0 + g;
        if (128u * m >= J) break;
        u32 v[4] = {x[4 * g], x[4 * g + 1], x[4 * g + 2], x[4 * g + 3]};
#pragma unroll
        for (int m0 = GB; m0 < NB; m0 += GB)
            if ((u32)m0 == mr0) { v[0] = x[4 * (m0 + g)]; v[1] = x[4 * (m0 + g) + 1]; v[2] = x[4 * (m0 + g) + 2]; v[3] = x[4 * (m0 + g) + 3]; }
        u32 pos[4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
            pos[t] = 4 * (lane + 32u * m) + t < J ? atomicAdd(&sh.cnt[wl_bkt(v[t], M)], 1u) : (u32)WL_CAP;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (pos[t] != (u32)WL_CAP) { RS_CHK(h + pos[t] < (u32)WL_CAP); kh[pos[t]] = v[t]; }
    }
    __syncwarp();
}

__device__ __forceinline__ void wl_clear(WarpLeaf &sh, u32 lane)
{
    static_assert(WL_B % 128 == 0 && WL_B / 32 <= 32, "clear layout");
#pragma unroll
    for (int i = 0; i < WL_B / 128; ++i)
        *reinterpret_cast<uint4 *>(&sh.cnt[128 * i + 4 * lane]) = make_uint4(0u, 0u, 0u, 0u);
    if (lane < WL_B / 32) sh.cnt[WL_B + lane] = 0u;
}

// 32-byte store of base + {a, b, c, d} (u64 + u32), predicated; the adds
// live inside the asm so the compiler cannot hoist all of a lane's 64-bit
// sums ahead of the stores (which would double the register footprint).
__device__ __forceinline__ void st_v4_base_if(bool pred, u64 *p, u64 base, u32 a, u32 b, u32 c, u32 d)
{
    asm volatile("{\n\t.reg .pred q;\n\t.reg .u32 l0, h0, l1, h1, l2, h2, l3, h3, bl, bh;\n\t"
                 "setp.ne.u32 q, %6, 0;\n\t"
                 "mov.b64 {bl, bh}, %1;\n\t"
                 "add.cc.u32 l0, bl, %2;\n\taddc.u32 h0, bh, 0;\n\t"
                 "add.cc.u32 l1, bl, %3;\n\taddc.u32 h1, bh, 0;\n\t"
                 "add.cc.u32 l2, bl, %4;\n\taddc.u32 h2, bh, 0;\n\t"
                 "add.cc.u32 l3, bl, %5;\n\taddc.u32 h3, bh, 0;\n\t"
                 "@q st.global.v8.u32 [%0], {l0, h0, l1, h1, l2, h2, l3, h3};\n\t}"
                 ::"l"(p), "l"(base), "r"(a), "r"(b), "r"(c), "r"(d), "r"((u32)pred) : "memory");
}

// Step 3: every draw of the round to its bucket's next position (+ h).
template <bool REM = true>   // REM: the partial groups in one after-loop copy (smaller code; WR measured slower)
__device__ __forceinline__ void wl_scatter(WarpLeaf &sh, const RoundKeys &K, const WDrawer &dr, u32 J, u32 h, int shb, u32 lane)
{
    u32 *kh = sh.keys + h;
#if defined(RS_WL_REGEN)
    const u32 qfull = J >> 2;
    // the draws are regenerated (Philox is cheaper than holding them)
#pragma unroll 1
    for (u32 q = lane; 4 * q < J; q += 32) {
        u32 v[4];
        dr.block(K, q, v);
        if (q < qfull) {
#pragma unroll
            for (int w = 0; w < 4; ++w) kh[atomicAdd(&sh.cnt[wl_word(v[w] >> shb)], 1u)] = v[w];
        } else {
#pragma unroll
            for (int w = 0; w < 4; ++w)
                if (4 * q + w < J) kh[atomicAdd(&sh.cnt[wl_word(v[w] >> shb)], 1u)] = v[w];
        }
    }
#else
    // the staged draws (keys[0..J)) come back into registers first: the
    // scatter overwrites the staging area
    constexpr int NB = WL_E1 / 4;
    u32 x[WL_E1];
#if RS_WL_RANK
    u32 rk[NB];
#endif
#pragma unroll
    for (int m = 0; m < NB; ++m) {
        const u32 q = lane + 32u * m;
        if (4 * q < J) {
            const uint4 t = *reinterpret_cast<const uint4 *>(&sh.keys[4 * q]);
            x[4 * m] = t.x; x[4 * m + 1] = t.y; x[4 * m + 2] = t.z; x[4 * m + 3] = t.w;
#if RS_WL_RANK
            rk[m] = sh.rank[q];
#endif
        }
    }
    __syncwarp();
#if RS_WL_RANK
#define WL_POS(e) (sh.cnt[wl_word(x[e] >> shb)] + ((rk[(e) >> 2] >> (8 * ((e) & 3))) & 0xffu))
#else
#define WL_POS(e) atomicAdd(&sh.cnt[wl_word(x[e] >> shb)], 1u)
#endif
    // Atomics first, stores after, in groups of GB blocks: smem stores and
    // atomics may alias as far as the compiler knows, so interleaving them
    // would serialise every atomic's round trip.
    constexpr int GB = RS_WL_GB;
    static_assert(NB % GB == 0, "group size");
    u32 mr0 = 0;                                 // first group not in a full GB-group
#pragma unroll
    for (int m0 = 0; m0 < NB; m0 += GB) {
        // the GB-group's draws all exist for every lane: no per-draw test
        const bool full = 4 * (31u + 32u * (m0 + GB - 1)) + 3 < J;
        if (full) {
            u32 pos[4 * GB];
#pragma unroll
            for (int e = 4 * m0; e < 4 * (m0 + GB); ++e)
#ifdef RS_EXP_NOSCATTER
                pos[e - 4 * m0] = 4 * (lane + 32u * (e >> 2)) + (e & 3);
#else
                pos[e - 4 * m0] = WL_POS(e);
#endif
#pragma unroll
            for (int e = 4 * m0; e < 4 * (m0 + GB); ++e) { RS_CHK(h + pos[e - 4 * m0] < (u32)WL_CAP); kh[pos[e - 4 * m0]] = x[e]; }
            mr0 = m0 + GB;
        }
    }
#if !RS_WL_RANK
    // the rest (at most GB groups, the last partial) one group at a time, its
    // draws selected out of x: one copy of the per-draw tests (code size)
#pragma unroll
    for (int g = 0; g < GB; ++g) {
        const u32 m = mr0 + g;
        if (!REM || 128u * m >= J) break;
        u32 v[4] = {x[4 * g], x[4 * g + 1], x[4 * g + 2], x[4 * g + 3]};
#pragma unroll
        for (int m0 = GB; m0 < NB; m0 += GB)
            if ((u32)m0 == mr0) { v[0] = x[4 * (m0 + g)]; v[1] = x[4 * (m0 + g) + 1]; v[2] = x[4 * (m0 + g) + 2]; v[3] = x[4 * (m0 + g) + 3]; }
        u32 pos[4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
            pos[t] = 4 * (lane + 32u * m) + t < J ? atomicAdd(&sh.cnt[wl_word(v[t] >> shb)], 1u) : (u32)WL_CAP;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (pos[t] != (u32)WL_CAP) { RS_CHK(h + pos[t] < (u32)WL_CAP); kh[pos[t]] = v[t]; }
    }
#endif
#pragma unroll
    for (int m0 = 0; m0 < NB; m0 += GB) {
        if (REM && !RS_WL_RANK) break;          // (handled above)
        if ((u32)m0 < mr0 || !(4 * (lane + 32u * m0) < J)) continue;
        u32 pos[4 * GB];
#pragma unroll
        for (int e = 4 * m0; e < 4 * (m0 + GB); ++e) {
            const u32 j = 4 * (lane + 32u * (e >> 2)) + (e & 3);
            pos[e - 4 * m0] = j < J ? WL_POS(e) : (u32)WL_CAP;
        }
#pragma unroll
        for (int e = 4 * m0; e < 4 * (m0 + GB); ++e)
            if (pos[e - 4 * m0] != (u32)WL_CAP) kh[pos[e - 4 * m0]] = x[e];
    }
#undef WL_POS
#endif
    __syncwarp();
}

// Steps 4-6 for E positions per lane.  Returns 0 (leaf stored) or, for WOR
// with too few distinct values, WL_TOPUP | |S| (the distinct values are
// compacted in sh.keys[h, h + |S|) for wl_topup).
// Graph calls (NEXT-3): positions [h, h + k) of sh.keys hold the leaf's
// sorted offsets; decode each to its packed edge (edge_pack, rs_math.cuh) in a
// non-unrolled loop so the kernel holds a single copy of the decode.
__device__ __noinline__ void wl_store_edges(const WarpLeaf &sh, u64 *d0, u32 h, u32 k, u64 base, u64 gV, u32 lane)
{
    EdgeCursor cur(gV);
#pragma unroll 1
    for (u32 i = h + lane; i < h + k; i += 32) d0[i] = cur.pack(base - 1 + sh.keys[i]);
    __syncwarp();
}

// WOR leaves whose round ended with |S| = dist < k distinct values (R7):
// instead of a new full round over J + (k - dist) draws, the distinct values
// (sorted, sh.keys[h, h + dist)) are topped up draw by draw -- draws J, J+1,
// ... in order, each kept iff it is in neither the sorted set (binary search,
// broadcast loads) nor the new values so far -- until k are distinct: the
// same first-k-distinct set.  The merged run is stored directly (old value i
// moves up by the number of new values below it).  Up to 32 new values (one
// per lane; at most LeafArgs::topup_max); more returns false and the caller
// runs the full round.
template <bool GR, bool P2>
__device__ __forceinline__ bool wl_topup(const WarpLeaf &sh, const RoundKeys &K, const WDrawer &dr, u32 J, u32 k,
                                      u32 dist, u32 h, u64 base, u64 *d0, u32 lane, u64 gV, u32 tmax)
{
    const u32 need = k - dist;
    if (need > tmax) return false;                   // tmax <= 32

    const u32 *ks = sh.keys + h;
    u32 nv = 0, mv = 0xffffffffu, mr = 0;            // lane t < nv: t-th new value and its rank in ks
    for (u32 j0 = J; nv < need; j0 += 32) {
        u32 v[4];
        dr.block<P2>(K, (j0 + lane) >> 2, v);
        const u32 w = (j0 + lane) & 3u;
        const u32 xl = w == 0 ? v[0] : w == 1 ? v[1] : w == 2 ? v[2] : v[3];
#pragma unroll 1
        for (u32 t = 0; t < 32 && nv < need; ++t) {
            const u32 x = __shfl_sync(0xffffffffu, xl, t);
            u32 lo = 0, hi = dist;                       // lower_bound(ks, x)
            while (lo < hi) {
                const u32 mid = (lo + hi) >> 1;
                if (ks[mid] < x) lo = mid + 1; else hi = mid;
            }
            const bool old = lo < dist && ks[lo] == x;
            const bool dup = __any_sync(0xffffffffu, lane < nv && mv == x);
            if (!old && !dup) {
                if (lane == nv) { mv = x; mr = lo; }
                ++nv;
            }
        }
    }
#if RS_WL_TUV4
    if (!GR && nv <= 4) {
        // merged output slot o (0 <= o < k) holds new value t if o == F_t
        // (F_t = rank_t + #{new < value_t}, its final position), else old value
        // ks[o - #{t : F_t < o}].  Output by slot, four per lane: 32-byte
        // stores on the output's 32-byte grid (d0 is aligned, slots start at h).
        u32 F = 0xffffffffu;
        {
            u32 sft = 0;
            for (u32 t = 0; t < nv; ++t) sft += __shfl_sync(0xffffffffu, mv, t) < mv;
            if (lane < nv) F = mr + sft;
        }
        const u32 F0 = __shfl_sync(0xffffffffu, F, 0), F1 = __shfl_sync(0xffffffffu, F, 1);
        const u32 F2 = __shfl_sync(0xffffffffu, F, 2), F3 = __shfl_sync(0xffffffffu, F, 3);
        const u32 m0 = __shfl_sync(0xffffffffu, mv, 0), m1 = __shfl_sync(0xffffffffu, mv, 1);
        const u32 m2 = __shfl_sync(0xffffffffu, mv, 2), m3 = __shfl_sync(0xffffffffu, mv, 3);
        const u32 end = h + k, ng = (end + 3) >> 2;
        for (u32 g = lane; g < ng; g += 32) {
            u64 w[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const u32 o = 4 * g + t - h;       // wraps (huge) below h: F_t < o false
                const u32 c = (F0 < o) + (F1 < o) + (F2 < o) + (F3 < o);
                const u32 v = o == F0 ? m0 : o == F1 ? m1 : o == F2 ? m2 : o == F3 ? m3 : ks[min(o - c, (u32)WL_CAP - 1u - h)];
                w[t] = out_word_t<GR>(base + v, gV);
            }
            if (4 * g >= h && 4 * g + 4 <= end) {
                st_v4(d0 + 4 * g, w[0], w[1], w[2], w[3]);
            } else {
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (4 * g + t >= h && 4 * g + t < end) d0[4 * g + t] = w[t];
            }
        }
        __syncwarp();
        return true;
    }
#endif
    // merged positions: old value i -> i + #{new < ks[i]} = i + #{t : rank_t <= i}
    // (rank_t = lower_bound of new value t in ks); new value t -> rank_t +
    // #{new < value_t}.  The first four ranks are broadcast once.
    const u32 r0 = __shfl_sync(0xffffffffu, lane < nv ? mr : 0xffffffffu, 0);
    const u32 r1 = __shfl_sync(0xffffffffu, lane < nv ? mr : 0xffffffffu, 1);
    const u32 r2 = __shfl_sync(0xffffffffu, lane < nv ? mr : 0xffffffffu, 2);
    const u32 r3 = __shfl_sync(0xffffffffu, lane < nv ? mr : 0xffffffffu, 3);
    if (nv == 1) {                                  // (the common case: one compare per value)
#pragma unroll 1
        for (u32 i = lane; i < dist; i += 32) d0[h + i + (r0 <= i)] = out_word_t<GR>(base + ks[i], gV);
    } else {
#pragma unroll 1
        for (u32 i0 = 0; i0 < dist; i0 += 32) {     // warp-uniform trip count (shuffles inside)
            const u32 i = i0 + lane;
            u32 sft = (r0 <= i) + (r1 <= i) + (r2 <= i) + (r3 <= i);
#pragma unroll 1
            for (u32 t = 4; t < nv; ++t) sft += __shfl_sync(0xffffffffu, mr, t) <= i;
            if (i < dist) d0[h + i + sft] = out_word_t<GR>(base + ks[i], gV);
        }
    }
    u32 sft = 0;
#pragma unroll 1
    for (u32 t = 0; t < nv; ++t) sft += __shfl_sync(0xffffffffu, mv, t) < mv;
    if (lane < nv) d0[h + mr + sft] = out_word_t<GR>(base + mv, gV);
    __syncwarp();
    return true;
}

constexpr u32 WL_TOPUP = 0x80000000u;      // wl_finish: "dist distinct values compacted, top up"

constexpr u32 WL_DUPLIST = 0xfffffffeu;   // wl_finish (SD kernels): "duplicates: to the duplicate list"

template <int E, bool WR, bool GR, bool TU, bool SD = false>
__device__ __forceinline__ u32 wl_finish(WarpLeaf &sh, u32 J, u32 k, u32 h, u32 P_, u64 base,
                                         u64 *dst, u32 lane, u64 gV)   // (base, dst: unused if RS_WL_SMEMST)
{
    u32 P = P_;
    RS_TS(tf0);
    wl_clear(sh, lane);                          // counters are dead: ready for the next round / leaf
    if (lane < h) sh.keys[lane] = 0u;            // pad below the first draw
    {   // sentinels WL_SENT0 + p above the last draw: distinct, larger than any key
        const u32 s0 = h + J, s4 = (s0 + 3) & ~3u;
        if (lane < s4 - s0 && s0 + lane < 32u * E) sh.keys[s0 + lane] = WL_SENT0 + s0 + lane;
#pragma unroll 1
        for (u32 p = s4 + 4 * lane; p < 32u * E; p += 128)
            *reinterpret_cast<uint4 *>(&sh.keys[p]) =
                make_uint4(WL_SENT0 + p, WL_SENT0 + p + 1, WL_SENT0 + p + 2, WL_SENT0 + p + 3);
    }
    __syncwarp();
    // 4. blocked registers + odd-even transposition inside buckets
    u32 y[E];
#pragma unroll
    for (int i = 0; i < E; i += 4) {
        const uint4 t = *reinterpret_cast<const uint4 *>(&sh.keys[E * lane + i]);
        y[i] = t.x; y[i + 1] = t.y; y[i + 2] = t.z; y[i + 3] = t.w;
    }
#ifdef RS_EXP_NOSORT
    P = 0;
#endif
#if RS_WL_EXACTP
    // a bucket of c draws is sorted after c alternating phases (c = 1: none),
    // so exactly P phases: pairs, then a lone even phase if P is odd
    if (P < 2) P = 0;
    for (u32 ph = 0; ph + 1 < P; ph += 2) {      // even + odd phase per step
#else
    for (u32 ph = 0; ph < P; ph += 2) {          // even + odd phase per step (P rounded up)
#endif
#pragma unroll
        for (int i = 0; i < E; i += 2) wl_ce(y[i], y[i + 1]);
        const u32 nxt = __shfl_down_sync(0xffffffffu, y[0], 1);
        const u32 prv = __shfl_up_sync(0xffffffffu, y[E - 1], 1);
#pragma unroll
        for (int i = 1; i < E - 1; i += 2) wl_ce(y[i], y[i + 1]);
        if (lane < 31) y[E - 1] = min(y[E - 1], nxt);
        if (lane > 0) y[0] = max(prv, y[0]);
    }
#if RS_WL_EXACTP
    if (P & 1) {
#pragma unroll
        for (int i = 0; i < E; i += 2) wl_ce(y[i], y[i + 1]);
    }
#endif
    RS_TS(tf1);
    RS_ACC(3, tf0, tf1);
    const u32 p0 = E * lane;
#if RS_WL_SMEMST || RS_WL_SMEMST_GR
    if (RS_WL_SMEMST || GR) {
        // reloaded here (not live in registers through the count/scatter/sort)
        base = sh.cur_base;
        dst = reinterpret_cast<u64 *>(sh.cur_dst);
    }
#endif
    u64 *d0 = dst - h;                           // 32-byte aligned
    if (!WR) {
        // 5. duplicates = equal neighbours (Algorithm H rejects them).  Fast
        // test: the smallest neighbour difference is 0 somewhere.  Pads get
        // distinct values 0, 1, 2 and sentinels are distinct, so a zero
        // difference is a duplicate, or (rarely) the first draw equal to the
        // last pad -- the exact count below sorts that out.
        if (lane == 0) { if (h > 1) y[1] = 1u; if (h > 2) y[2] = 2u; }
        const u32 prv = __shfl_up_sync(0xffffffffu, y[E - 1], 1);
        u32 m4[4] = {lane ? y[0] - prv : 1u, 1u, 1u, 1u};
#pragma unroll
        for (int i = 1; i < E; ++i) m4[i & 3] = min(m4[i & 3], y[i] - y[i - 1]);
        const u32 md = min(min(m4[0], m4[1]), min(m4[2], m4[3]));
        if (SD && __any_sync(0xffffffffu, md == 0u)) return WL_DUPLIST;   // (or the first draw equal to the last pad)
        if (!SD && __any_sync(0xffffffffu, md == 0u)) {
            // exact count: distinct neighbours as min(difference, 1) (sorted:
            // differences >= 0), two per three-input add; the sentinels are
            // distinct and above every key, the pads 0, 1, 2 distinct, so only
            // lane 0's first draw equal to its last pad is not a duplicate
            u32 n4[4] = {lane ? min(y[0] - prv, 1u) : 1u, 0u, 0u, 0u};
#pragma unroll
            for (int i = 1; i < E; i += 2)
                n4[(i >> 1) & 3] += min(y[i] - y[i - 1], 1u) + (i + 1 < E ? min(y[i + 1] - y[i], 1u) : 1u);
            u32 nd = (u32)E + 1u - ((n4[0] + n4[1]) + (n4[2] + n4[3]));
            if (lane == 0 && h) nd -= h == 1 ? y[1] == y[0] : h == 2 ? y[2] == y[1] : y[3] == y[2];
            const u32 ndup = __reduce_add_sync(0xffffffffu, nd);
            if (ndup) {
                const u32 dist = J - ndup;       // |S| after this round
                if (!TU && dist < k) return J + (k - dist);
                // compact the distinct values through shared memory, then store:
                // every position but the duplicates -- the pads stay at [0, h), the
                // distinct draws land at [h, h + |S|), the sentinels above (unread)
                u32 o = warp_excl_scan((u32)E - nd, lane);
                __syncwarp();
#pragma unroll
                for (int i = 0; i < E; ++i)
                    if (!(p0 + i > h && y[i] == (i ? y[i - 1] : prv))) sh.keys[o++] = y[i];
                __syncwarp();
                if (dist < k) return WL_TOPUP | dist;      // the caller tops the set up (wl_topup)
                if (GR) { wl_store_edges(sh, d0, h, k, base, gV, lane); return 0; }
                const u32 ng = (h + k + 3) >> 2;
                for (u32 g = lane; g < ng; g += 32) {
                    const uint4 t = *reinterpret_cast<const uint4 *>(&sh.keys[4 * g]);
                    const u32 vv[4] = {t.x, t.y, t.z, t.w};
                    const u32 i0 = 4 * g;
                    if (i0 >= h && i0 + 4 <= h + k) {
                        st_v4(d0 + i0, out_word_t<GR>(base + vv[0], gV), out_word_t<GR>(base + vv[1], gV),
                              out_word_t<GR>(base + vv[2], gV), out_word_t<GR>(base + vv[3], gV));
                    } else {
#pragma unroll
                        for (int t2 = 0; t2 < 4; ++t2)
                            if (i0 + t2 >= h && i0 + t2 < h + k) d0[i0 + t2] = out_word_t<GR>(base + vv[t2], gV);
                    }
                }
                __syncwarp();
                return 0;
            }
        }
    }
    RS_TS(tf2);
    RS_ACC(4, tf1, tf2);
    // 6. no duplicates (J == k): 32-byte stores straight from registers; the
    // head group (positions 0..3, lane 0) and the tail group are partial.
    const u32 end = h + k;
#ifdef RS_EXP_NOSTORE
    if (y[0] == 0x12345u && y[E-1] == 7u) d0[lane] = y[3];
    return 0;
#endif
    if (GR) {                                      // graph calls: packed edges
        // one decode site: the sorted draws go through shared memory (16-byte
        // stores, lane stride 4 (mod 32) banks: conflict-free per quarter
        // warp), then lane-strided 8-byte stores (coalesced)
        __syncwarp();
#pragma unroll
        for (int m = 0; m < E; m += 4)
            *reinterpret_cast<uint4 *>(&sh.keys[p0 + m]) = make_uint4(y[m], y[m + 1], y[m + 2], y[m + 3]);
        __syncwarp();
        wl_store_edges(sh, d0, h, k, base, gV, lane);
        return 0;
    } else {
#pragma unroll
        for (int m = 0; m < E; m += 4) {
            const u32 p = p0 + m;
            st_v4_base_if(p >= h && p + 4 <= end, d0 + p, base, y[m], y[m + 1], y[m + 2], y[m + 3]);
        }
    }
    if (lane == 0 && (h || end < 4)) {             // head group (positions 0..3) if partial
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if ((u32)t >= h && (u32)t < end) d0[t] = out_word_t<GR>(base + y[t], gV);
    }
    const u32 tg = (end - 1) & ~3u;               // tail group start (if partial, and not the head)
    if ((end & 3u) && tg >= 4 && lane == tg / E) {
        // the group's three values selected first (a select chain), then ONE
        // store sequence: this rarely-run code stays small
        const u32 mt = tg - p0;
        u32 v0 = y[0], v1 = y[1], v2 = y[2];
#pragma unroll
        for (int m = 4; m < E; m += 4)
            if ((u32)m == mt) { v0 = y[m]; v1 = y[m + 1]; v2 = y[m + 2]; }
        d0[tg] = out_word_t<GR>(base + v0, gV);                   // (tg < end: the group is partial)
        if (tg + 1 < end) d0[tg + 1] = out_word_t<GR>(base + v1, gV);
        if (tg + 2 < end) d0[tg + 2] = out_word_t<GR>(base + v2, gV);
    }
    __syncwarp();
    return 0;
}

// CS: CTA-span leaf ranges (fused kernels).  SD: a leaf whose round has an
// equal neighbour goes to the duplicate list (a.dup) instead of the duplicate
// path, which is not compiled in (ranges where duplicates are rare: a smaller
// kernel).  LS: the leaves of the duplicate list (the pass after an SD kernel).
template <bool WR, bool GR, bool TU, bool P2 = false, bool CS = false, int NW = WL_WARPS, bool SD = false,
          bool LS = false>
__device__ __forceinline__ void warp_leaves(const LeafArgs &a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WarpLeaf &sh = reinterpret_cast<WarpLeaf *>(smem_raw)[wid];
    wl_clear(sh, lane);
    __syncwarp();
    const u64 stride = CS ? (u64)NW : (u64)gridDim.x * NW;
    u64 I = CS ? ((u64)blockIdx.x << a.span_log) + wid : (u64)blockIdx.x * NW + wid;   // leaf (LS: list) index
    const u64 Iend = LS ? (u64)*(volatile const u32 *)a.dup_n
                        : CS ? min(a.nleaves, ((u64)blockIdx.x + 1) << a.span_log) : a.nleaves;
    // the next leaf's count / offset arrive by cp.async straight into shared
    // memory while this leaf is processed (no register stays live for them)
    const u32 s_k = (u32)__cvta_generic_to_shared(&sh.pf_k), s_off = (u32)__cvta_generic_to_shared(&sh.pf_off);
    if (lane == 0 && I < Iend) {
        const u64 L0 = LS ? (u64)a.dup[I] : I;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s_k), "l"(a.cnt + L0) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s_off), "l"(a.off + L0) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (; I < Iend; I += stride) {
        const u64 L = LS ? (u64)a.dup[I] : I;
        if (lane == 0) asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        const u32 k = sh.pf_k;
        const u64 off = sh.pf_off;
        __syncwarp();
        if (lane == 0 && I + stride < Iend) {   // prefetch the next leaf's count and offset
            const u64 L1 = LS ? (u64)a.dup[I + stride] : I + stride;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s_k), "l"(a.cnt + L1) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s_off), "l"(a.off + L1) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        if (k == 0) continue;
        if (a.wcap != 0u && k > a.wcap) {               // (tests: force the spill path)
            if (lane == 0) a.spill[atomicAdd(a.spill_n, 1u)] = (u32)L;
            continue;
        }
        const LeafGeom g = leaf_geom(a, L);
        const int cr = ceil_log2(g.r);
        const WDrawer dr(Stream(a.seed, WR ? P_WR : P_WOR, g.id), g.r, cr);
        u64 *dst = a.out + off;
        const u32 h = (u32)(reinterpret_cast<uintptr_t>(dst) >> 3) & 3u;
        const int shb = cr > WL_LOGB ? cr - WL_LOGB : 0;
        const u64 base = g.lo + 1;
#if RS_WL_SMEMST || RS_WL_SMEMST_GR
        if (RS_WL_SMEMST || GR) {
            if (lane == 0) { sh.cur_base = base; sh.cur_dst = reinterpret_cast<unsigned long long>(dst); }
            __syncwarp();
        }
#endif
        constexpr bool SMST = RS_WL_SMEMST || (RS_WL_SMEMST_GR && GR);
        u32 J = k;
        // the register-resident count/scatter: for the power-of-two WOR kernels
        // (no spills there; measured headline 12.45 -> 12.26 ms, cfg1 4.64 ->
        // 4.33) or everywhere with RS_WL_REG (spills elsewhere; WR slower)
        constexpr bool REG = RS_WL_REG || (RS_WL_REG_P2 && P2 && !WR && !GR) || (RS_WL_REG_WR && P2 && WR && !GR);
        const u32 M = REG ? wl_bucket_mult(cr) : 0u;
        for (;;) {
            u32 res = 0xffffffffu;
            if (REG) {
            if (J + h <= (u32)WL_CAP) {
                u32 x[WL_E1];
                const u32 P = (P2 || dr.pow2) ? wl_count_reg<true>(sh, a.rk, dr, J, M, lane, x)
                                              : wl_count_reg<false>(sh, a.rk, dr, J, M, lane, x);
                if (P > WL_PMAX) {              // pathological bucket load
                    wl_clear(sh, lane);
                    __syncwarp();
                } else {
                    wl_scatter_reg(sh, J, h, M, lane, x);
                    res = wl_finish<WL_E1, WR, GR, TU, SD>(sh, J, k, h, P, SMST ? 0 : base, SMST ? nullptr : dst, lane, a.gV);
                }
            }
            } else {
            if (J + h <= (u32)WL_CAP) {
                const u32 P = wl_count<P2>(sh, a.rk, dr, J, shb, lane);
                if (P > WL_PMAX) {              // pathological bucket load
                    wl_clear(sh, lane);
                    __syncwarp();
                } else if (J + h <= 32u * WL_E1) {
                    RS_TS(ts0);
                    wl_scatter<true>(sh, a.rk, dr, J, h, shb, lane);
                    RS_TS(ts1);
                    RS_ACC(2, ts0, ts1);
                    res = wl_finish<WL_E1, WR, GR, TU, SD>(sh, J, k, h, P, SMST ? 0 : base, SMST ? nullptr : dst, lane, a.gV);
                    RS_TS(ts2);
                    RS_ACC(5, ts1, ts2);
                } else {
#ifndef RS_WL_TWO_E
                    wl_clear(sh, lane);         // larger leaves go to the CTA kernel (measured faster than a second, 44-position instantiation)
                    __syncwarp();
#else
                    wl_scatter<true>(sh, a.rk, dr, J, h, shb, lane);
                    res = wl_finish<WL_E2, WR, GR, TU>(sh, J, k, h, P, base, dst, lane, a.gV);
#endif
                }
            }
            }
            if (res == 0) break;
            if (SD && res == WL_DUPLIST) {      // the list pass (a top-up kernel) completes this leaf
                if (lane == 0) a.dup[atomicAdd(a.dup_n, 1u)] = (u32)L;
                break;
            }
            if (res == 0xffffffffu) {           // the CTA kernel completes this leaf
                if (lane == 0) a.spill[atomicAdd(a.spill_n, 1u)] = (u32)L;
                break;
            }
            if (TU && (res & WL_TOPUP)) {       // |S| < k: top up draw by draw, else a full round
                const u32 dist = res & ~WL_TOPUP;
                if (wl_topup<GR, P2>(sh, a.rk, dr, J, k, dist, h, base, dst - h, lane, a.gV, a.topup_max)) break;
                res = J + (k - dist);
            }
            J = res;
        }
    }
}

__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wor(LeafArgs a) { warp_leaves<false, false, false>(a); }
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wr(LeafArgs a) { warp_leaves<true, false, false>(a); }
// small leaf ranges (many duplicates): the top-up instead of full rounds
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wor_tu(LeafArgs a) { warp_leaves<false, false, true>(a); }
// G(n, m) (NEXT-3): the WOR kernel with the edge decode fused into its stores
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_gnm(LeafArgs a) { warp_leaves<false, true, false>(a); }
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_gnm_tu(LeafArgs a) { warp_leaves<false, true, true>(a); }
// every leaf range a power of two (N = 2^a): no Lemire rejection code at all
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wor_tu_p2(LeafArgs a) { warp_leaves<false, false, true, true>(a); }
__global__ void RS_WL_LB(SD_WARPS) k_leaf_warp_wor_sd_p2(LeafArgs a) { warp_leaves<false, false, true, true, false, SD_WARPS, true>(a); }
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wor_tu_p2_ls(LeafArgs a) { warp_leaves<false, false, true, true, false, WL_WARPS, false, true>(a); }
__global__ void RS_WL_LB(WR_WARPS) k_leaf_warp_wr_p2(LeafArgs a) { warp_leaves<true, false, false, true, false, WR_WARPS>(a); }
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wor_p2(LeafArgs a) { warp_leaves<false, false, false, true>(a); }

}  // namespace rs
