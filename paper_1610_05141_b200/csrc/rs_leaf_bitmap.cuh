// rs_leaf_bitmap.cuh -- leaves with a small range r (<= BM_RMAX): ONE WARP PER
// LEAF over a bitmap of the range.  Used for the complement (row a7, the
// dense cfg3a case: N = 2^32, n = 0.75 N -> core leaves of r = 4096 with
// e ~ 1024 excluded values) and for WOR leaves whose range is small.
// Included by rs_kernels.cu.  P:n = /root/reference/PAPER.md line n.
//
// Algorithm H with the table replaced by a bitmap of [0, r):
// round t ORs the bits of its draws into the map; the set after draws
// [0, J) is exactly the map (OR is idempotent), so the rounds of R7 -- round
// t+1 adds k - |S| draws -- only touch the NEW draws, and |S| is a popcount.
// The map is already in sorted order (P:370-374 with the identity hash), so
// the leaf's output is its set bits (WOR) or its clear bits (complement,
// "generate the N - n elements not in the sample"), emitted with
// a per-word popcount prefix.  One random shared-memory access per draw.

namespace rs {

constexpr u32 BM_RMAX = 1u << 15;             // largest leaf range on this path
constexpr u32 BM_WORDS = BM_RMAX / 32;        // 1024 words = 4 KB per warp

struct BitmapLeaf {
    u32 bm[BM_WORDS];
};

// Draws [J0, J) of the leaf stream into the map (Lemire / power-of-two
// shift, R3), lane-strided over Philox blocks.
__device__ __forceinline__ void bm_draws(BitmapLeaf &sh, const RoundKeys &K, const WDrawer &dr,
                                         u32 J0, u32 J, u32 lane)
{
#pragma unroll 1
    for (u32 q = (J0 >> 2) + lane; 4 * q < J; q += 32) {
        u32 v[4];
        dr.block(K, q, v);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const u32 j = 4 * q + w;
            if (j >= J0 && j < J) atomicOr(&sh.bm[v[w] >> 5], 1u << (v[w] & 31u));
        }
    }
    __syncwarp();
}

__device__ __forceinline__ u32 bm_valid(u32 w, u32 r)
{
    return (w + 1) * 32 <= r ? 0xffffffffu : ((1u << (r & 31u)) - 1u);
}

template <bool COMP, bool GR>
__device__ __forceinline__ void bitmap_leaves(const LeafArgs &a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    BitmapLeaf &sh = reinterpret_cast<BitmapLeaf *>(smem_raw)[wid];
    const u64 stride = (u64)gridDim.x * WB_WARPS;
    for (u64 L = (u64)blockIdx.x * WB_WARPS + wid; L < a.nleaves; L += stride) {
        const u32 k = a.cnt[L];                     // sample (WOR) or excluded (complement) count
        const LeafGeom g = leaf_geom(a, L);
        const u32 r = (u32)g.r;
        const u32 nw = (r + 31) >> 5;
        const u64 nout = COMP ? g.r - k : k;
        if (nout == 0) continue;
        u64 *dst = COMP ? a.out + (g.lo - a.out_base - a.off[L]) : a.out + a.off[L];
        const u64 base = g.lo + 1;
        EdgeCursor ecur(a.gV);                      // graph calls: per-lane values ascend
        auto ow = [&](u64 x) -> u64 { return GR ? ecur.pack(x - 1) : x; };
        for (u32 w = lane; w < nw; w += 32) sh.bm[w] = 0u;
        __syncwarp();
        if (k > 0) {
            const int cr = ceil_log2(g.r);
            const WDrawer dr(Stream(a.seed, P_WOR, g.id), g.r, cr);
            u32 J0 = 0, J = k;
            for (;;) {                              // rounds (R7): only the new draws
                bm_draws(sh, a.rk, dr, J0, J, lane);
                u32 c = 0;
                for (u32 w = lane; w < nw; w += 32) c += __popc(sh.bm[w]);
                const u32 d = __reduce_add_sync(0xffffffffu, c);
                if (d >= k) break;                  // d == k: the first k distinct draws
                J0 = J;
                J += k - d;
            }
        }
        // emit the output bits in order; dense: one word per step, lane = bit,
        // so consecutive lanes store consecutive outputs
        if (nout * 4 >= (u64)r) {
            // four words per step (16-byte broadcast load): independent
            // prefix chains and stores; the last partial word is masked
            const u32 lm = (1u << lane) - 1u;
            const u32 nfull = r >> 5;               // words with all 32 values in range
            u32 pos = 0;
            u64 vb = base + lane;
            u32 w = 0;
#pragma unroll 1
            for (; w + 4 <= nfull; w += 4, vb += 128) {
                const uint4 W4 = *reinterpret_cast<const uint4 *>(&sh.bm[w]);
                const u32 b0 = COMP ? ~W4.x : W4.x, b1 = COMP ? ~W4.y : W4.y;
                const u32 b2 = COMP ? ~W4.z : W4.z, b3 = COMP ? ~W4.w : W4.w;
                const u32 p0 = pos, p1 = p0 + __popc(b0), p2 = p1 + __popc(b1), p3 = p2 + __popc(b2);
                pos = p3 + __popc(b3);
                if ((b0 >> lane) & 1u) dst[p0 + __popc(b0 & lm)] = ow(vb);
                if ((b1 >> lane) & 1u) dst[p1 + __popc(b1 & lm)] = ow(vb + 32);
                if ((b2 >> lane) & 1u) dst[p2 + __popc(b2 & lm)] = ow(vb + 64);
                if ((b3 >> lane) & 1u) dst[p3 + __popc(b3 & lm)] = ow(vb + 96);
            }
#pragma unroll 1
            for (; w < nw; ++w, vb += 32) {
                const u32 word = sh.bm[w];
                const u32 bits = COMP ? (~word & bm_valid(w, r)) : word;
                if ((bits >> lane) & 1u) dst[pos + __popc(bits & lm)] = ow(vb);
                pos += __popc(bits);
            }
        } else {
            // sparse: lane l owns words [l*per, (l+1)*per); warp scan of counts
            const u32 per = (nw + 31) >> 5;
            const u32 w0 = lane * per, w1 = min(w0 + per, nw);
            u32 c = 0;
            for (u32 w = w0; w < w1; ++w) {
                const u32 word = sh.bm[w];
                c += __popc(COMP ? (~word & bm_valid(w, r)) : word);
            }
            u32 pos = warp_excl_scan(c, lane);
            for (u32 w = w0; w < w1; ++w) {
                const u32 word = sh.bm[w];
                u32 bits = COMP ? (~word & bm_valid(w, r)) : word;
                while (bits) {
                    const u32 b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    dst[pos++] = ow(base + 32u * w + b);
                }
            }
        }
        __syncwarp();
    }
}

__global__ void RS_WB_LB k_leaf_bitmap_wor(LeafArgs a) { bitmap_leaves<false, false>(a); }
__global__ void RS_WB_LB k_leaf_bitmap_comp(LeafArgs a) { bitmap_leaves<true, false>(a); }
__global__ void RS_WB_LB k_leaf_bitmap_wor_g(LeafArgs a) { bitmap_leaves<false, true>(a); }
__global__ void RS_WB_LB k_leaf_bitmap_comp_g(LeafArgs a) { bitmap_leaves<true, true>(a); }

}  // namespace rs
