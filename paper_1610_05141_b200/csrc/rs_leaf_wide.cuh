// rs_leaf_wide.cuh -- the warp-per-leaf counting sort (rs_leaf_warp.cuh) for
// WIDE leaf ranges, 2^32 - 4096 < r < 2^63 (rows a5, a6, a8 of SURVEY.md
// section 8(a); the paper-shaped sweep N = 2^50, n <= 2^28).
// Included by rs_kernels.cu after rs_leaf_warp.cuh.  P:n = PAPER.md line n.
//
// A draw x < r (R3: 64-bit Lemire, two Philox words per draw) is split into a
// 31-bit SORT KEY key = x >> sh, sh = ceil_log2(r) - 31 (monotone in x; below
// 2^31, so the warp kernel's sentinels stay above every key), and a PAYLOAD
// low = x mod 2^sh.  The warp kernel's machinery runs on the keys --
// monotone-hash buckets, counting sort, odd-even transposition inside buckets
// -- with the payload moved alongside (a second staging array and
// compare-exchanges that swap both).  Keys are distinct unless two draws share
// their top 32 bits (a tie, or a true duplicate: Algorithm H would reject one,
// P:157-160); both happen for about 1 leaf in 10^4 and then the whole leaf is
// completed exactly by the CTA kernel with 64-bit keys (k_leaf_wor64 /
// k_leaf_wr64) through the spill list.  Output value lo + ((key << sh) | low) + 1.
constexpr int WW_KEYBITS = 31;

namespace rs {

struct WarpLeafW {
    WarpLeaf w;                            // counters, prefetch slots, keys (staging, then sorted)
    u32 lows[WL_CAP + 4];                  // payloads (staging, then sorted alongside)
};

// Steps 1-2: the round's J draws -> (key, low) staged in draw order, bucket
// counts of the keys, scan.  Returns the largest bucket load.
template <bool POW2>
__device__ __forceinline__ u32 ww_count(WarpLeafW &sh, const RoundKeys &K, const Drawer<u64> &dr, u32 J, u32 sh64,
                                        u32 shk, u32 lane)
{
    const u32 nq = (J + 1) >> 1;                 // Philox blocks: two draws each
    const u64 lmask = ((u64)1 << shk) - 1;
#pragma unroll 1
    for (u32 q = lane; q < nq; q += 64) {        // two independent blocks per step (ILP)
        u32 kk[4], ll[4];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const u32 qq = q + 32u * b;
            const u32x4 w = philox_rk_(qq, dr.st.tag, dr.st.id_lo, dr.st.id_hi, K);
            u64 x0 = ((u64)w.x << 32) | w.y, x1 = ((u64)w.z << 32) | w.w;
            if (POW2) { x0 >>= sh64; x1 >>= sh64; }
            else if (qq < nq) { x0 = dr.fix(x0, 2 * qq); x1 = dr.fix(x1, 2 * qq + 1); }
            kk[2 * b] = (u32)(x0 >> shk); ll[2 * b] = (u32)(x0 & lmask);
            kk[2 * b + 1] = (u32)(x1 >> shk); ll[2 * b + 1] = (u32)(x1 & lmask);
        }
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const u32 qq = q + 32u * b;
            if (2 * qq < J) atomicAdd(&sh.w.cnt[wl_word(kk[2 * b] >> (WW_KEYBITS - WL_LOGB))], 1u);
            if (2 * qq + 1 < J) atomicAdd(&sh.w.cnt[wl_word(kk[2 * b + 1] >> (WW_KEYBITS - WL_LOGB))], 1u);
        }
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const u32 qq = q + 32u * b;
            if (qq < nq) {
                *reinterpret_cast<uint2 *>(&sh.w.keys[2 * qq]) = make_uint2(kk[2 * b], kk[2 * b + 1]);
                *reinterpret_cast<uint2 *>(&sh.lows[2 * qq]) = make_uint2(ll[2 * b], ll[2 * b + 1]);
            }
        }
    }
    __syncwarp();
    return wl_scan(sh.w, lane);
}

// Step 3: every staged (key, low) to its bucket's next position (+ h).
__device__ __forceinline__ void ww_scatter(WarpLeafW &sh, u32 J, u32 h, u32 lane)
{
    constexpr int NB = WL_E1 / 4;                // draws j = 4 (lane + 32 m) + t
    u32 x[WL_E1], l[WL_E1];
#pragma unroll
    for (int m = 0; m < NB; ++m) {
        const u32 q = lane + 32u * m;
        if (4 * q < J) {
            const uint4 t = *reinterpret_cast<const uint4 *>(&sh.w.keys[4 * q]);
            const uint4 u = *reinterpret_cast<const uint4 *>(&sh.lows[4 * q]);
            x[4 * m] = t.x; x[4 * m + 1] = t.y; x[4 * m + 2] = t.z; x[4 * m + 3] = t.w;
            l[4 * m] = u.x; l[4 * m + 1] = u.y; l[4 * m + 2] = u.z; l[4 * m + 3] = u.w;
        }
    }
    __syncwarp();
    u32 *kh = sh.w.keys + h, *lh = sh.lows + h;
    // full groups (every lane's four draws exist) unrolled without per-draw
    // tests; the one partial group after the loop, its draws selected out of
    // x / l: one copy of the tests (the warp kernels are instruction-fetch
    // sensitive)
#pragma unroll
    for (int m = 0; m < NB; ++m) {
        if (128u * m + 127u < J) {
            u32 pos[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) pos[t] = atomicAdd(&sh.w.cnt[wl_word(x[4 * m + t] >> (WW_KEYBITS - WL_LOGB))], 1u);
#pragma unroll
            for (int t = 0; t < 4; ++t) { RS_CHK(h + pos[t] < (u32)WL_CAP); kh[pos[t]] = x[4 * m + t]; lh[pos[t]] = l[4 * m + t]; }
        }
    }
    const u32 mp = J >> 7;
    if ((J & 127u) && mp < (u32)NB) {
        u32 v[4] = {x[0], x[1], x[2], x[3]}, w[4] = {l[0], l[1], l[2], l[3]};
#pragma unroll
        for (int m = 1; m < NB; ++m)
            if ((u32)m == mp) {
                v[0] = x[4 * m]; v[1] = x[4 * m + 1]; v[2] = x[4 * m + 2]; v[3] = x[4 * m + 3];
                w[0] = l[4 * m]; w[1] = l[4 * m + 1]; w[2] = l[4 * m + 2]; w[3] = l[4 * m + 3];
            }
        u32 pos[4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
            pos[t] = 4 * (lane + 32u * mp) + t < J ? atomicAdd(&sh.w.cnt[wl_word(v[t] >> (WW_KEYBITS - WL_LOGB))], 1u)
                                                   : (u32)WL_CAP;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (pos[t] != (u32)WL_CAP) { RS_CHK(h + pos[t] < (u32)WL_CAP); kh[pos[t]] = v[t]; lh[pos[t]] = w[t]; }
    }
    __syncwarp();
}

__device__ __forceinline__ void ww_ce(u32 &a, u32 &b, u32 &pa, u32 &pb)
{
    const bool s = a > b;
    const u32 ka = s ? b : a, kb = s ? a : b, qa = s ? pb : pa, qb = s ? pa : pb;
    a = ka; b = kb; pa = qa; pb = qb;
}

// Steps 4-6: blocked registers, P odd-even phases moving the payloads along,
// equal neighbours -> false (the leaf spills), else 32-byte stores.
__device__ __forceinline__ bool ww_finish(WarpLeafW &sh, u32 J, u32 h, u32 P, u64 base, u32 shk, u64 *dst, u32 lane)
{
    constexpr int E = WL_E1;
    wl_clear(sh.w, lane);
    if (lane < h) sh.w.keys[lane] = 0u;          // pads below the first draw (never above a key)
    {   // sentinels WL_SENT0 + p above the last draw: distinct, larger than any key
        const u32 s0 = h + J;
#pragma unroll 1
        for (u32 p = s0 + lane; p < 32u * E; p += 32) sh.w.keys[p] = WL_SENT0 + p;
    }
    __syncwarp();
    u32 y[E], pl[E];
#pragma unroll
    for (int i = 0; i < E; i += 4) {
        const uint4 t = *reinterpret_cast<const uint4 *>(&sh.w.keys[E * lane + i]);
        const uint4 u = *reinterpret_cast<const uint4 *>(&sh.lows[E * lane + i]);
        y[i] = t.x; y[i + 1] = t.y; y[i + 2] = t.z; y[i + 3] = t.w;
        pl[i] = u.x; pl[i + 1] = u.y; pl[i + 2] = u.z; pl[i + 3] = u.w;
    }
    if (P < 2) P = 0;
    for (u32 ph = 0; ph + 1 < P; ph += 2) {      // even + odd phase per step
#pragma unroll
        for (int i = 0; i < E; i += 2) ww_ce(y[i], y[i + 1], pl[i], pl[i + 1]);
        const u32 nxt = __shfl_down_sync(0xffffffffu, y[0], 1), pn = __shfl_down_sync(0xffffffffu, pl[0], 1);
        const u32 prv = __shfl_up_sync(0xffffffffu, y[E - 1], 1), pp = __shfl_up_sync(0xffffffffu, pl[E - 1], 1);
#pragma unroll
        for (int i = 1; i < E - 1; i += 2) ww_ce(y[i], y[i + 1], pl[i], pl[i + 1]);
        if (lane < 31 && nxt < y[E - 1]) { y[E - 1] = nxt; pl[E - 1] = pn; }
        if (lane > 0 && prv > y[0]) { y[0] = prv; pl[0] = pp; }
    }
    if (P & 1) {
#pragma unroll
        for (int i = 0; i < E; i += 2) ww_ce(y[i], y[i + 1], pl[i], pl[i + 1]);
    }
    // a tie or duplicate is an equal pair of neighbours (pads and sentinels are distinct)
    const u32 p0 = E * lane;
    bool eq = false;
    const u32 prv = __shfl_up_sync(0xffffffffu, y[E - 1], 1);
    eq |= lane > 0 && p0 > h && y[0] == prv;            // (sentinels: distinct, above every key)
#pragma unroll
    for (int i = 1; i < E; ++i) eq |= y[i] == y[i - 1] && p0 + i > h;
    if (__any_sync(0xffffffffu, eq)) return false;
    u64 *d0 = dst - h;                           // 32-byte aligned
    const u32 end = h + J;
    // full 32-byte groups from registers; the partial head (positions 0..3,
    // lane 0) and tail groups after, the tail's values selected first: one
    // copy of the per-value stores
#pragma unroll
    for (int m = 0; m < E; m += 4) {
        const u32 p = p0 + m;
        if (p >= h && p + 4 <= end) {
            u64 v[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) v[t] = base + (((u64)y[m + t] << shk) | pl[m + t]);
            st_v4(d0 + p, v[0], v[1], v[2], v[3]);
        }
    }
    if (lane == 0 && (h || end < 4)) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if ((u32)t >= h && (u32)t < end) d0[t] = base + (((u64)y[t] << shk) | pl[t]);
    }
    const u32 tg = (end - 1) & ~3u;
    if ((end & 3u) && tg >= 4 && lane == tg / E) {
        const u32 mt = tg - p0;
        u32 k0 = y[0], k1 = y[1], k2 = y[2], q0 = pl[0], q1 = pl[1], q2 = pl[2];
#pragma unroll
        for (int m = 4; m < E; m += 4)
            if ((u32)m == mt) { k0 = y[m]; k1 = y[m + 1]; k2 = y[m + 2]; q0 = pl[m]; q1 = pl[m + 1]; q2 = pl[m + 2]; }
        d0[tg] = base + (((u64)k0 << shk) | q0);
        if (tg + 1 < end) d0[tg + 1] = base + (((u64)k1 << shk) | q1);
        if (tg + 2 < end) d0[tg + 2] = base + (((u64)k2 << shk) | q2);
    }
    __syncwarp();
    return true;
}

template <bool WR, bool CS = false, int NW = WL_WARPS>
__device__ __forceinline__ void warp_leaves_wide(const LeafArgs &a)   // CS: CTA-span leaf ranges (fused kernels)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WarpLeafW &sh = reinterpret_cast<WarpLeafW *>(smem_raw)[wid];
    wl_clear(sh.w, lane);
    __syncwarp();
    const u64 stride = CS ? (u64)NW : (u64)gridDim.x * NW;
    u64 L = CS ? ((u64)blockIdx.x << a.span_log) + wid : (u64)blockIdx.x * NW + wid;
    const u64 Lend = CS ? min(a.nleaves, ((u64)blockIdx.x + 1) << a.span_log) : a.nleaves;
    const u32 s_k = (u32)__cvta_generic_to_shared(&sh.w.pf_k), s_off = (u32)__cvta_generic_to_shared(&sh.w.pf_off);
    if (lane == 0 && L < Lend) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s_k), "l"(a.cnt + L) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s_off), "l"(a.off + L) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (; L < Lend; L += stride) {
        if (lane == 0) asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        const u32 k = sh.w.pf_k;
        const u64 off = sh.w.pf_off;
        __syncwarp();
        if (lane == 0 && L + stride < Lend) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s_k), "l"(a.cnt + L + stride) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s_off), "l"(a.off + L + stride) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        if (k == 0) continue;
        if (a.wcap != 0u && k > a.wcap) {               // (tests: force the spill path)
            if (lane == 0) a.spill[atomicAdd(a.spill_n, 1u)] = (u32)L;
            continue;
        }
        const LeafGeom g = leaf_geom(a, L);
        const int cr = ceil_log2(g.r);                      // 32 .. 63
        const u32 shk = (u32)cr - (u32)WW_KEYBITS;          // key = x >> shk < 2^31
        const Drawer<u64> dr(Stream(a.seed, WR ? P_WR : P_WOR, g.id), g.r);
        const bool pow2 = (g.r & (g.r - 1)) == 0;
        u64 *dst = a.out + off;
        const u32 h = (u32)(reinterpret_cast<uintptr_t>(dst) >> 3) & 3u;
        bool ok = false;
        if (k + h <= (u32)WL_CAP) {
            const u32 P = pow2 ? ww_count<true>(sh, a.rk, dr, k, 64u - (u32)cr, shk, lane)
                               : ww_count<false>(sh, a.rk, dr, k, 0u, shk, lane);
            if (P <= WL_PMAX) {
                ww_scatter(sh, k, h, lane);
                ok = ww_finish(sh, k, h, P, g.lo + 1, shk, dst, lane);
            } else {
                wl_clear(sh.w, lane);
                __syncwarp();
            }
        }
        if (!ok && lane == 0) a.spill[atomicAdd(a.spill_n, 1u)] = (u32)L;
    }
}

__global__ void RS_WW_LB k_leaf_warp_wide_wor(LeafArgs a) { warp_leaves_wide<false, false, WW_WARPS>(a); }
__global__ void RS_WW_LB k_leaf_warp_wide_wr(LeafArgs a) { warp_leaves_wide<true, false, WW_WARPS>(a); }

}  // namespace rs
