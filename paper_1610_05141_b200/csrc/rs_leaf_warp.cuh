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

#ifndef RS_WL_MINB
#define RS_WL_MINB 4          // resident CTAs per SM the register budget is sized for
#endif

namespace rs {

constexpr int WL_B = 1024;                 // buckets (u32 counters)
constexpr int WL_LOGB = 10;
constexpr int WL_E1 = 36, WL_E2 = 44;      // positions per lane; E mod 32 in {4, 12}: conflict-free LDS.128
constexpr int WL_CAP = 32 * WL_E2;         // 1408 positions per leaf
constexpr u32 WL_PMAX = 48;                // odd-even phases allowed before spilling

struct WarpLeaf {
    u32 cnt[WL_B + WL_B / 32];             // padded bucket counters / starts (33 words per lane)
    u32 keys[WL_CAP];                      // staging (draw order), then positions: pad, draws, sentinels
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
// power-of-two range is the top ceil_log2(r) bits (never rejects).
struct WDrawer {
    Drawer<u32> d;
    u32 s;          // 32 - ceil_log2(r)
    bool pow2;
    __device__ WDrawer(const Stream &st, u64 r, int cr) : d(st, r), s(32u - (u32)cr), pow2((r & (r - 1)) == 0) {}
    __device__ __forceinline__ void block(u32 q, u32 *v) const
    {
        if (pow2) {
            const u32x4 w = d.st.block(q);
            v[0] = shr32(w.x, s); v[1] = shr32(w.y, s); v[2] = shr32(w.z, s); v[3] = shr32(w.w, s);
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

// Steps 1-2: count the round's J draws per bucket and stage them in draw
// order at keys[0..J); scan the counts into starts.  Returns the largest
// bucket load (0 if a bucket is a single value).
__device__ __forceinline__ u32 wl_count(WarpLeaf &sh, const WDrawer &dr, u32 J, int shb, u32 lane)
{
    const u32 qfull = J >> 2;                    // blocks whose 4 draws all count
#pragma unroll 1
    for (u32 q = lane; 4 * q < J; q += 32) {
        u32 v[4];
        dr.block(q, v);
        if (q < qfull) {
#pragma unroll
            for (int w = 0; w < 4; ++w) atomicAdd(&sh.cnt[wl_word(v[w] >> shb)], 1u);
        } else {
#pragma unroll
            for (int w = 0; w < 4; ++w)
                if (4 * q + w < J) atomicAdd(&sh.cnt[wl_word(v[w] >> shb)], 1u);
        }
#if !defined(RS_WL_REGEN)
        *reinterpret_cast<uint4 *>(&sh.keys[4 * q]) = make_uint4(v[0], v[1], v[2], v[3]);
#endif
    }
    __syncwarp();
    u32 *cl = sh.cnt + 33 * lane;
    u32 S = 0, mx = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const u32 c = cl[i];
        S += c;
        mx = max(mx, c);
    }
    u32 run = warp_excl_scan(S, lane);
    const u32 P = __reduce_max_sync(0xffffffffu, mx);
#pragma unroll
    for (int i = 0; i < 32; ++i) {               // starts in place (second read)
        const u32 c = cl[i];
        cl[i] = run;
        run += c;
    }
    __syncwarp();
    return shb == 0 ? 0u : P;
}

__device__ __forceinline__ void wl_clear(WarpLeaf &sh, u32 lane)
{
#pragma unroll
    for (int i = 0; i < (WL_B + WL_B / 32) / 32; ++i) sh.cnt[32 * i + lane] = 0u;
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
__device__ __forceinline__ void wl_scatter(WarpLeaf &sh, const WDrawer &dr, u32 J, u32 h, int shb, u32 lane)
{
    u32 *kh = sh.keys + h;
    const u32 qfull = J >> 2;
#if defined(RS_WL_REGEN)
    // the draws are regenerated (Philox is cheaper than holding them)
#pragma unroll 1
    for (u32 q = lane; 4 * q < J; q += 32) {
        u32 v[4];
        dr.block(q, v);
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
#pragma unroll
    for (int m = 0; m < NB; ++m) {
        const u32 q = lane + 32u * m;
        if (4 * q < J) {
            const uint4 t = *reinterpret_cast<const uint4 *>(&sh.keys[4 * q]);
            x[4 * m] = t.x; x[4 * m + 1] = t.y; x[4 * m + 2] = t.z; x[4 * m + 3] = t.w;
        }
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < NB; ++m) {
        const u32 q = lane + 32u * m;
        if (q < qfull) {
#pragma unroll
            for (int w = 0; w < 4; ++w)
                kh[atomicAdd(&sh.cnt[wl_word(x[4 * m + w] >> shb)], 1u)] = x[4 * m + w];
        } else if (4 * q < J) {
#pragma unroll
            for (int w = 0; w < 4; ++w)
                if (4 * q + w < J) kh[atomicAdd(&sh.cnt[wl_word(x[4 * m + w] >> shb)], 1u)] = x[4 * m + w];
        }
    }
#endif
    __syncwarp();
}

// Steps 4-6 for E positions per lane.  Returns 0 (leaf stored) or, for WOR
// with too few distinct values, the next round's draw count J' > J.
template <int E, bool WR>
__device__ __forceinline__ u32 wl_finish(WarpLeaf &sh, u32 J, u32 k, u32 h, u32 P, u64 base,
                                         u64 *dst, u32 lane)
{
    wl_clear(sh, lane);                          // counters are dead: ready for the next round / leaf
    if (lane < h) sh.keys[lane] = 0u;            // pad below the first draw
    for (u32 p = h + J + lane; p < 32u * E; p += 32) sh.keys[p] = 0xffffffffu;   // sentinels
    __syncwarp();
    // 4. blocked registers + odd-even transposition inside buckets
    u32 y[E];
#pragma unroll
    for (int i = 0; i < E; i += 4) {
        const uint4 t = *reinterpret_cast<const uint4 *>(&sh.keys[E * lane + i]);
        y[i] = t.x; y[i + 1] = t.y; y[i + 2] = t.z; y[i + 3] = t.w;
    }
    for (u32 ph = 0; ph < P; ++ph) {
        if ((ph & 1u) == 0) {
#pragma unroll
            for (int i = 0; i < E; i += 2) wl_ce(y[i], y[i + 1]);
        } else {
            const u32 nxt = __shfl_down_sync(0xffffffffu, y[0], 1);
            const u32 prv = __shfl_up_sync(0xffffffffu, y[E - 1], 1);
#pragma unroll
            for (int i = 1; i < E - 1; i += 2) wl_ce(y[i], y[i + 1]);
            if (lane < 31) y[E - 1] = min(y[E - 1], nxt);
            if (lane > 0) y[0] = max(prv, y[0]);
        }
    }
    const u32 p0 = E * lane;
    u64 *d0 = dst - h;                           // 32-byte aligned
    if (!WR) {
        // 5. duplicates = equal neighbours (Algorithm H rejects them).  Count
        // every equality, then remove those of the pad (positions 1..h-1, and
        // position h if the first draw is 0) and of the sentinels.
        const u32 prv = __shfl_up_sync(0xffffffffu, y[E - 1], 1);
        u32 nd = lane ? (u32)(y[0] == prv) : 0u;
#pragma unroll
        for (int i = 1; i < E; ++i) nd += (u32)(y[i] == y[i - 1]);
        u32 ndup = __reduce_add_sync(0xffffffffu, nd);
        const u32 yh = __shfl_sync(0xffffffffu, h == 0 ? y[0] : h == 1 ? y[1] : h == 2 ? y[2] : y[3], 0);
        ndup -= (h ? h - 1 + (u32)(yh == 0u) : 0u) + (32u * E - (h + J)) - (32u * E > h + J ? 1u : 0u);
        if (ndup) {
            const u32 dist = J - ndup;           // |S| after this round
            if (dist < k) return J + (k - dist);
            // compact the k distinct values through shared memory, then store
            u32 keep = 0;
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const u32 p = p0 + i;
                keep += p >= h && p < h + J && !(p > h && y[i] == (i ? y[i - 1] : prv));
            }
            u32 o = h + warp_excl_scan(keep, lane);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const u32 p = p0 + i;
                if (p >= h && p < h + J && !(p > h && y[i] == (i ? y[i - 1] : prv))) sh.keys[o++] = y[i];
            }
            __syncwarp();
            const u32 ng = (h + k + 3) >> 2;
            for (u32 g = lane; g < ng; g += 32) {
                const uint4 t = *reinterpret_cast<const uint4 *>(&sh.keys[4 * g]);
                const u32 vv[4] = {t.x, t.y, t.z, t.w};
                const u32 i0 = 4 * g;
                if (i0 >= h && i0 + 4 <= h + k) {
                    st_v4(d0 + i0, base + vv[0], base + vv[1], base + vv[2], base + vv[3]);
                } else {
#pragma unroll
                    for (int t2 = 0; t2 < 4; ++t2)
                        if (i0 + t2 >= h && i0 + t2 < h + k) d0[i0 + t2] = base + vv[t2];
                }
            }
            __syncwarp();
            return 0;
        }
    }
    // 6. no duplicates (J == k): 32-byte stores straight from registers; the
    // head group (positions 0..3, lane 0) and the tail group are partial.
    const u32 end = h + k;
#pragma unroll
    for (int m = 0; m < E; m += 4) {
        const u32 p = p0 + m;
        st_v4_base_if(p >= h && p + 4 <= end, d0 + p, base, y[m], y[m + 1], y[m + 2], y[m + 3]);
    }
    if (lane == 0 && h) {                          // head: positions h..3 (k >= 1)
#pragma unroll
        for (int t = 1; t < 4; ++t)
            if ((u32)t >= h && (u32)t < end) d0[t] = base + y[t];
    }
    const u32 tg = (end - 1) & ~3u;               // tail group start (if partial)
    if ((end & 3u) && tg >= 4 && lane == tg / E) {
        const u32 mt = tg - p0;
#pragma unroll
        for (int m = 0; m < E; m += 4)
            if ((u32)m == mt) {
#pragma unroll
                for (int t = 0; t < 3; ++t)
                    if (tg + t < end) d0[tg + t] = base + y[m + t];
            }
    }
    __syncwarp();
    return 0;
}

template <bool WR>
__device__ __forceinline__ void warp_leaves(const LeafArgs &a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WarpLeaf &sh = reinterpret_cast<WarpLeaf *>(smem_raw)[wid];
    wl_clear(sh, lane);
    __syncwarp();
    const u64 stride = (u64)gridDim.x * WL_WARPS;
    u64 L = (u64)blockIdx.x * WL_WARPS + wid;
    u32 k_next = L < a.nleaves ? a.cnt[L] : 0u;
    u64 off_next = L < a.nleaves ? a.off[L] : 0ull;
    for (; L < a.nleaves; L += stride) {
        const u32 k = k_next;
        const u64 off = off_next;
        if (L + stride < a.nleaves) {          // prefetch the next leaf's count and offset
            k_next = a.cnt[L + stride];
            off_next = a.off[L + stride];
        }
        if (k == 0) continue;
        const LeafGeom g = leaf_geom(a, L);
        const int cr = ceil_log2(g.r);
        const WDrawer dr(Stream(a.seed, WR ? P_WR : P_WOR, g.id), g.r, cr);
        u64 *dst = a.out + off;
        const u32 h = (u32)(reinterpret_cast<uintptr_t>(dst) >> 3) & 3u;
        const int shb = cr > WL_LOGB ? cr - WL_LOGB : 0;
        const u64 base = g.lo + 1;
        u32 J = k;
        for (;;) {
            u32 res = 0xffffffffu;
            if (J + h <= 32u * WL_E2) {
                const u32 P = wl_count(sh, dr, J, shb, lane);
                if (P > WL_PMAX) {              // pathological bucket load
                    wl_clear(sh, lane);
                    __syncwarp();
                } else if (J + h <= 32u * WL_E1) {
                    wl_scatter(sh, dr, J, h, shb, lane);
                    res = wl_finish<WL_E1, WR>(sh, J, k, h, P, base, dst, lane);
                } else {
#ifndef RS_WL_TWO_E
                    wl_clear(sh, lane);         // larger leaves go to the CTA kernel (measured faster than a second, 44-position instantiation)
                    __syncwarp();
#else
                    wl_scatter(sh, dr, J, h, shb, lane);
                    res = wl_finish<WL_E2, WR>(sh, J, k, h, P, base, dst, lane);
#endif
                }
            }
            if (res == 0) break;
            if (res == 0xffffffffu) {           // the CTA kernel completes this leaf
                if (lane == 0) a.spill[atomicAdd(a.spill_n, 1u)] = (u32)L;
                break;
            }
            J = res;
        }
    }
}

__global__ void __launch_bounds__(32 * WL_WARPS, RS_WL_MINB) k_leaf_warp_wor(LeafArgs a) { warp_leaves<false>(a); }
__global__ void __launch_bounds__(32 * WL_WARPS, RS_WL_MINB) k_leaf_warp_wr(LeafArgs a) { warp_leaves<true>(a); }

}  // namespace rs
