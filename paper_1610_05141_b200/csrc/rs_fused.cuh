// rs_fused.cuh -- small trees (rows a3-a5): the split and the leaves in ONE
// launch.  Included by rs_kernels.cu after the warp-leaf kernels.
//
// For a tree of at most 2^RS_FUSED_MAXD leaves (n up to ~2^21 at 1024 samples
// per leaf) the split is a chain of D - s dependent deviates per leaf
// (P:218-221), and the level-by-level launches (or grid barriers)
// between them cost as much as the deviates.  Here CTA c owns the subtree of
// WL_WARPS leaves under node c at depth D - LB (LB = log2 WL_WARPS, or less
// for tiny trees): its warp 0 walks the path from the shard root to that
// node -- one warp deviate (hgd_tp / binom_tp) per level, taking the child on
// c's path and adding the left child's count to the offset when it goes
// right -- and then its warps expand the LB levels below in parallel (warp j
// splits node j of the level).  The top of the path is computed redundantly
// by every CTA: the chain is the same D - s deviates either way, and no CTA
// waits for another.  Every count is the tree's (same deviate keyed by the
// same node id), so the output is bit-identical to the split kernels'.  Then
// each warp runs the warp-per-leaf kernel body on its own leaf (the grid
// has exactly one warp per leaf).
#pragma once

namespace rs {

constexpr int FUSED_LB = 4;            // log2(WL_WARPS): one leaf per warp
static_assert((1 << FUSED_LB) == WL_WARPS, "fused kernels: one warp per leaf");

template <bool WR>
__device__ __forceinline__ void fused_split(const FusedArgs &f)
{
    __shared__ u64 fs_cnt[2][WL_WARPS], fs_off[2][WL_WARPS];
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int lb = f.lb;                          // levels expanded inside the CTA
    const int dp = f.D - lb;                      // depth of the CTA's subtree root
    const u64 c = blockIdx.x;                     // its index below the shard root
    if (wid == 0) {
        u64 k = f.root_cnt, off = 0, i = 0;
        for (int d = f.s; d < dp; ++d) {
            const u64 gi = (f.idx << (d - f.s)) + i;
            const u64 x = split_node_grp<WR, 32>(f.N, d, gi, k, f.seed);
            const u64 right = (c >> (dp - 1 - d)) & 1u;
            if (right) { off += x; k -= x; } else { k = x; }
            i = 2 * i + right;
        }
        if (lane == 0) { fs_cnt[0][0] = k; fs_off[0][0] = off; }
    }
    __syncthreads();
    int cur = 0;
    for (int l = 0; l < lb; ++l) {
        const u32 width = 1u << l;
        if (wid < width) {
            const u64 k = fs_cnt[cur][wid], off = fs_off[cur][wid];
            const u64 gi = (((f.idx << (dp - f.s)) + c) << l) + wid;
            const u64 x = split_node_grp<WR, 32>(f.N, dp + l, gi, k, f.seed);
            if (lane == 0) {
                fs_cnt[cur ^ 1][2 * wid] = x;
                fs_cnt[cur ^ 1][2 * wid + 1] = k - x;
                fs_off[cur ^ 1][2 * wid] = off;
                fs_off[cur ^ 1][2 * wid + 1] = off + x;
            }
        }
        __syncthreads();
        cur ^= 1;
    }
    const u32 nl = 1u << lb;
    if (threadIdx.x < nl) {
        const u64 cnt = fs_cnt[cur][threadIdx.x];
        if (cnt > 0xffffffffull) atomicOr(&g_rs_errors, 1u);
        f.leaf_cnt[(c << lb) + threadIdx.x] = (u32)cnt;
        f.leaf_off[(c << lb) + threadIdx.x] = fs_off[cur][threadIdx.x];
    }
    __syncthreads();                              // the leaf body reads them (cp.async, this SM)
}

__global__ void __launch_bounds__(32 * WL_WARPS, RS_WL_MINB) k_fused_wor_tu(FusedArgs f)
{ fused_split<false>(f); warp_leaves<false, false, true>(f.la); }
__global__ void __launch_bounds__(32 * WL_WARPS, RS_WL_MINB) k_fused_wor_tu_p2(FusedArgs f)
{ fused_split<false>(f); warp_leaves<false, false, true, true>(f.la); }
__global__ void __launch_bounds__(32 * WL_WARPS, RS_WL_MINB) k_fused_wr(FusedArgs f)
{ fused_split<true>(f); warp_leaves<true, false, false>(f.la); }
__global__ void __launch_bounds__(32 * WL_WARPS, RS_WL_MINB) k_fused_wr_p2(FusedArgs f)
{ fused_split<true>(f); warp_leaves<true, false, false, true>(f.la); }
__global__ void __launch_bounds__(32 * WL_WARPS, RS_WL_MINB) k_fused_wide_wor(FusedArgs f)
{ fused_split<false>(f); warp_leaves_wide<false>(f.la); }
__global__ void __launch_bounds__(32 * WL_WARPS, RS_WL_MINB) k_fused_wide_wr(FusedArgs f)
{ fused_split<true>(f); warp_leaves_wide<true>(f.la); }

}  // namespace rs
