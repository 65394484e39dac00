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
// Per round of J draws (R7), with B = 2048 monotone-hash buckets
// bucket(x) = x >> (ceil_log2(r) - 11) (the hash order is the sort
// order), held as u16 counters two per word:
//   1. Philox blocks (lane l: blocks l + 32m) -> draws -> RED.ADD count[bucket];
//   2. warp scan of the counts (swizzled so every access is conflict-free)
//      -> bucket starts; max bucket load P;
//   3. ATOMS.ADD on the start -> final position (+ h, the store alignment
//      shift), scatter the draw there: positions are now sorted by bucket;
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

namespace rs {

constexpr int WL_B = 2048;                 // buckets (u16 counters, two per word)
constexpr int WL_LOGB = 11;
constexpr int WL_E1 = 36, WL_E2 = 44;      // positions per lane; E mod 32 in {4, 12}: conflict-free LDS.128
constexpr int WL_CAP = 32 * WL_E2;         // 1664 positions per leaf
constexpr u32 WL_PMAX = 48;                // odd-even phases allowed before spilling

struct WarpLeaf {
    u32 cnt[WL_B / 2];                     // swizzled u16 bucket counters / starts
    u32 keys[WL_CAP];                      // positions 0..h-1 pad, h..h+J-1 draws, then sentinels
};

// Word of bucket b's counter (half (b & 1)): lane l owns pairs [32 l, 32 l + 32)
// for the scan, stored so that its 16-byte loads v = 0..7 are at
// v*128 + 4 l -- each 8-lane phase covers all 32 banks.
__device__ __forceinline__ u32 wl_word(u32 b)
{
    const u32 p = b >> 1;
    return ((p & 31) >> 2) * 128 + ((p >> 5) << 2) + (p & 3);
}

// An opaque copy ordered after the preceding memory operations: used to keep
// the compiler from hoisting every Philox block of a lane ahead of the first
// atomics (which would hold all of them in registers at once).
__device__ __forceinline__ u32 wl_fence(u32 v)
{
    asm volatile("" : "+r"(v)::"memory");
    return v;
}

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

// One round of J draws of a leaf with E positions per lane.  Returns
//   0           : leaf stored;
//   J' > J      : WOR, next round with J' draws;
//   0xffffffff  : does not fit on chip (spill).
template <int E, bool WR>
__device__ __forceinline__ u32 wl_round(WarpLeaf &sh, const Drawer<u32> &dr, u32 J, u32 k, u32 h,
                                        int shb, u64 base, u64 *dst, u32 lane)
{
    constexpr int NB = E / 4;                 // Philox blocks per lane
    // 1. draws -> bucket counts
#pragma unroll
    for (int m = 0; m < NB; ++m) {
        const u32 q = wl_fence(lane + 32u * m);
        if (4 * q < J) {
            u32 v[4];
            dr.block(q, v);
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                if (4 * q + w < J) {
                    const u32 b = v[w] >> shb;
                    atomicAdd(&sh.cnt[wl_word(b)], 1u << ((b & 1u) << 4));
                }
            }
        }
    }
    __syncwarp();
    // 2. scan: lane owns pairs [32 lane, 32 lane + 32) = buckets [64 lane, 64 lane + 64)
    u32 S = 0, mx = 0;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
        const uint4 c = *reinterpret_cast<const uint4 *>(&sh.cnt[v * 128 + 4 * lane]);
        S += c.x + c.y + c.z + c.w;                            // halves cannot carry (J < 2^16)
        mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(c.x, c.y), __vmaxu2(c.z, c.w)));
    }
    u32 run = warp_excl_scan((S & 0xffffu) + (S >> 16), lane);
    u32 P = __reduce_max_sync(0xffffffffu, max(mx & 0xffffu, mx >> 16));
    if (shb == 0) P = 0;                      // bucket == value: nothing to order inside
#pragma unroll
    for (int v = 0; v < 8; ++v) {             // second pass (re-read): starts, in place
        const uint4 c = *reinterpret_cast<const uint4 *>(&sh.cnt[v * 128 + 4 * lane]);
        uint4 o;
        o.x = run * 0x10001u + (c.x << 16); run += (c.x & 0xffffu) + (c.x >> 16);
        o.y = run * 0x10001u + (c.y << 16); run += (c.y & 0xffffu) + (c.y >> 16);
        o.z = run * 0x10001u + (c.z << 16); run += (c.z & 0xffffu) + (c.z >> 16);
        o.w = run * 0x10001u + (c.w << 16); run += (c.w & 0xffffu) + (c.w >> 16);
        *reinterpret_cast<uint4 *>(&sh.cnt[v * 128 + 4 * lane]) = o;
    }
    __syncwarp();
    if (P > WL_PMAX) {                        // pathological bucket load: spill
        for (int v = 0; v < 8; ++v)
            *reinterpret_cast<uint4 *>(&sh.cnt[v * 128 + 4 * lane]) = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
        return 0xffffffffu;
    }
    // 3. scatter to the final bucket positions (the draws are regenerated:
    //    cheaper than holding E of them in registers across the scan)
#pragma unroll
    for (int m = 0; m < NB; ++m) {
        const u32 q = wl_fence(lane + 32u * m);
        if (4 * q < J) {
            u32 v[4];
            dr.block(q, v);
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                if (4 * q + w < J) {
                    const u32 b = v[w] >> shb, sft = (b & 1u) << 4;
                    const u32 old = atomicAdd(&sh.cnt[wl_word(b)], 1u << sft);
                    sh.keys[h + ((old >> sft) & 0xffffu)] = v[w];
                }
            }
        }
    }
    __syncwarp();
    // counters are dead: clear them for the next round / leaf; pad and sentinels
#pragma unroll
    for (int v = 0; v < 8; ++v)
        *reinterpret_cast<uint4 *>(&sh.cnt[v * 128 + 4 * lane]) = make_uint4(0u, 0u, 0u, 0u);
    if (lane < h) sh.keys[lane] = 0u;
    for (u32 p = h + J + lane; p < 32u * E; p += 32) sh.keys[p] = 0xffffffffu;
    __syncwarp();
    // 4. blocked registers + odd-even transposition inside buckets
    u32 y[E];
#pragma unroll
    for (int i = 0; i < E; i += 4) {
        const uint4 q = *reinterpret_cast<const uint4 *>(&sh.keys[E * lane + i]);
        y[i] = q.x; y[i + 1] = q.y; y[i + 2] = q.z; y[i + 3] = q.w;
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
    // 5. duplicates (WOR): equal to the previous position
    u64 dupm = 0;
    u32 nd = 0;
    if (!WR) {
        const u32 prv = __shfl_up_sync(0xffffffffu, y[E - 1], 1);
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const u32 p = p0 + i;
            const bool d = p > h && p < h + J && y[i] == (i ? y[i - 1] : prv);
            dupm |= (u64)d << i;
            nd += d;
        }
        const u32 ndup = __reduce_add_sync(0xffffffffu, nd);
        if (ndup) {
            const u32 dist = J - ndup;          // |S| after this round
            if (dist < k) return J + (k - dist);
            // compact the k distinct values through shared memory
            u32 keep = 0;
#pragma unroll
            for (int i = 0; i < E; ++i) keep += (p0 + i >= h && p0 + i < h + J);
            keep -= nd;
            u32 o = h + warp_excl_scan(keep, lane);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < E; ++i) {
                const u32 p = p0 + i;
                if (p >= h && p < h + J && !((dupm >> i) & 1u)) sh.keys[o++] = y[i];
            }
            __syncwarp();
            u64 *d0 = dst - h;
            const u32 ng = (h + k + 3) >> 2;
            for (u32 g = lane; g < ng; g += 32) {
                const uint4 q = *reinterpret_cast<const uint4 *>(&sh.keys[4 * g]);
                const u32 vv[4] = {q.x, q.y, q.z, q.w};
                const u32 i0 = 4 * g;
                if (i0 >= h && i0 + 4 <= h + k) {
                    st_v4(d0 + i0, base + vv[0], base + vv[1], base + vv[2], base + vv[3]);
                } else {
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        if (i0 + t >= h && i0 + t < h + k) d0[i0 + t] = base + vv[t];
                }
            }
            __syncwarp();
            return 0;
        }
    }
    // 6. no duplicates: J == k; 32-byte stores straight from registers
    u64 *d0 = dst - h;
#pragma unroll
    for (int m = 0; m < E; m += 4) {
        const u32 p = p0 + m;
        if (p >= h && p + 4 <= h + k) {
            st_v4(d0 + p, base + y[m], base + y[m + 1], base + y[m + 2], base + y[m + 3]);
        } else {
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (p + t >= h && p + t < h + k) d0[p + t] = base + y[m + t];
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
#pragma unroll
    for (int v = 0; v < 8; ++v)
        *reinterpret_cast<uint4 *>(&sh.cnt[v * 128 + 4 * lane]) = make_uint4(0u, 0u, 0u, 0u);
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
        const Stream st(a.seed, WR ? P_WR : P_WOR, g.id);
        const Drawer<u32> dr(st, g.r);
        u64 *dst = a.out + off;
        const u32 h = (u32)(reinterpret_cast<uintptr_t>(dst) >> 3) & 3u;
        const int cr = ceil_log2(g.r);
        const int shb = cr > WL_LOGB ? cr - WL_LOGB : 0;
        const u64 base = g.lo + 1;
        u32 J = k;
        for (;;) {
            u32 res;
            if (J + h <= 32u * WL_E1) res = wl_round<WL_E1, WR>(sh, dr, J, k, h, shb, base, dst, lane);
            else if (J + h <= 32u * WL_E2) res = wl_round<WL_E2, WR>(sh, dr, J, k, h, shb, base, dst, lane);
            else res = 0xffffffffu;
            if (res == 0) break;
            if (res == 0xffffffffu) {           // the CTA kernel completes this leaf
                if (lane == 0) a.spill[atomicAdd(a.spill_n, 1u)] = (u32)L;
                break;
            }
            J = res;
        }
    }
}

__global__ void __launch_bounds__(32 * WL_WARPS, 4) k_leaf_warp_wor(LeafArgs a) { warp_leaves<false>(a); }
__global__ void __launch_bounds__(32 * WL_WARPS, 4) k_leaf_warp_wr(LeafArgs a) { warp_leaves<true>(a); }

}  // namespace rs
