// rs_fused.cuh -- small trees (rows a3-a5): the split and the leaves in ONE
// launch.  Included by rs_kernels.cu after the warp-leaf kernels.
//
// For a tree of at most 2^RS_FUSED_MAXD leaves (n up to ~2^24 at 1024 samples
// per leaf) the split is a chain of D - s dependent deviates per leaf
// (P:218-221), and the level-by-level launches (or grid barriers)
// between them cost as much as the deviates.  Here CTA c owns the subtree of
// 2^lb leaves under node c at depth D - lb (lb = log2 WL_WARPS, or less for
// tiny trees, or more so that there are at most 2^RS_FUSED_CTA_LOG CTAs): its
// warp 0 walks the path from the shard root to that node -- one warp deviate
// (hgd_tp / binom_tp) per level, taking the child on c's path and adding the
// left child's count to the offset when it goes right -- and then its warps
// expand the lb levels below (a warp or 8 lanes per node as the level
// widens).  The top of the path is computed redundantly
// by every CTA: the chain is the same D - s deviates either way, and no CTA
// waits for another.  Every count is the tree's (same deviate keyed by the
// same node id), so the output is bit-identical to the split kernels'.  Then
// the CTA's warps run the warp-per-leaf kernel body over its own leaves, and
// the last CTA completes the (rare) spilled leaves.
#pragma once

namespace rs {

constexpr int FUSED_LB = 4;            // log2(WL_WARPS)
static_assert((1 << FUSED_LB) == WL_WARPS, "fused kernels: a warp per node of the narrow levels");
static_assert(RS_FUSED_MAXD - RS_FUSED_CTA_LOG <= FUSED_LB + 3, "fused kernels: levels of <= 4 WL_WARPS nodes");

// One node of level l of the CTA's subtree: node j's (count, offset) from
// the level's input (shared memory while the level fits the warps, then the
// ws ping / pong buffers), its split by a group of G lanes, the children to
// the next level's buffer or, at the last level, to the leaf arrays.
template <bool WR, int G>
__device__ __forceinline__ void fused_node(const FusedArgs &f, u64 (*fs_cnt)[WL_WARPS], u64 (*fs_off)[WL_WARPS],
                                           int l, int cur, u32 j, int dp, u64 c)
{
    const u32 width = 1u << l;
    const bool in_sm = width <= (u32)WL_WARPS, out_sm = 2 * width <= (u32)WL_WARPS;
    const u64 k = in_sm ? fs_cnt[cur][j] : f.lv_cnt[cur][(c << l) + j];
    const u64 off = in_sm ? fs_off[cur][j] : f.lv_off[cur][(c << l) + j];
    const u64 gi = (((f.idx << (dp - f.s)) + c) << l) + j;
    const u64 x = split_node_grp<WR, G>(f.N, dp + l, gi, k, f.seed);
    if ((threadIdx.x & (G - 1)) != 0) return;
    const u64 o0 = 2 * (u64)j, o1 = o0 + 1;
    if (l + 1 == f.lb) {
        if (k > 0xffffffffull) atomicOr(&g_rs_errors, 1u);
        const u64 b = (c << f.lb);
        f.leaf_cnt[b + o0] = (u32)x;
        f.leaf_cnt[b + o1] = (u32)(k - x);
        f.leaf_off[b + o0] = off;
        f.leaf_off[b + o1] = off + x;
    } else if (out_sm) {
        fs_cnt[cur ^ 1][o0] = x; fs_cnt[cur ^ 1][o1] = k - x;
        fs_off[cur ^ 1][o0] = off; fs_off[cur ^ 1][o1] = off + x;
    } else {
        const u64 b = c << (l + 1);
        f.lv_cnt[cur ^ 1][b + o0] = x; f.lv_cnt[cur ^ 1][b + o1] = k - x;
        f.lv_off[cur ^ 1][b + o0] = off; f.lv_off[cur ^ 1][b + o1] = off + x;
    }
}

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
    if (lb == 0) {                                // a single leaf
        if (threadIdx.x == 0) {
            if (fs_cnt[0][0] > 0xffffffffull) atomicOr(&g_rs_errors, 1u);
            f.leaf_cnt[c] = (u32)fs_cnt[0][0];
            f.leaf_off[c] = fs_off[0][0];
        }
    }
    int cur = 0;
    for (int l = 0; l < lb; ++l) {
        const u32 width = 1u << l;
        // a warp per node (hgd_tp), or 8 lanes per node (hgd_tpg<8>); wider
        // levels (a lane per node) measured slower than the level kernels
        if (width <= (u32)WL_WARPS) {
            if (wid < width) fused_node<WR, 32>(f, fs_cnt, fs_off, l, cur, wid, dp, c);
        } else {                                  // (width <= 4 WL_WARPS: see the static_assert)
            if (threadIdx.x / 8 < width) fused_node<WR, 8>(f, fs_cnt, fs_off, l, cur, threadIdx.x / 8, dp, c);
        }
        __syncthreads();
        cur ^= 1;
    }
}

// The leaves the warp bodies spilled (usually none): the LAST CTA to finish
// its leaves (a counter in the call's status header, zeroed with it) runs
// them through the CTA-per-leaf routine, in the shared memory the warps no
// longer use -- instead of a second launch.
static_assert(LEAF_NT == 32 * WL_WARPS, "fused kernels: the CTA leaf routine's thread count");
template <typename K, bool WR>
__device__ __forceinline__ void fused_spills(const LeafArgs &a)
{
    __shared__ u32 last;
    __threadfence();                                      // every warp's spill-list entries ...
    __syncthreads();
    if (threadIdx.x == 0) {
        last = atomicAdd(a.status + 3, 1u) == gridDim.x - 1;   // ... before this CTA's arrival
        if (last) __threadfence();
    }
    __syncthreads();
    if (last) sample_leaves<K, WR, true>(a);
}

__global__ void RS_WL_LB(WL_WARPS) k_fused_wor_tu(FusedArgs f)
{ fused_split<false>(f); warp_leaves<false, false, true, false, true>(f.la); fused_spills<u32, false>(f.la); }
__global__ void RS_WL_LB(WL_WARPS) k_fused_wor_tu_p2(FusedArgs f)
{ fused_split<false>(f); warp_leaves<false, false, true, true, true>(f.la); fused_spills<u32, false>(f.la); }
__global__ void RS_WL_LB(WL_WARPS) k_fused_wr(FusedArgs f)
{ fused_split<true>(f); warp_leaves<true, false, false, false, true>(f.la); fused_spills<u32, true>(f.la); }
__global__ void RS_WL_LB(WL_WARPS) k_fused_wr_p2(FusedArgs f)
{ fused_split<true>(f); warp_leaves<true, false, false, true, true>(f.la); fused_spills<u32, true>(f.la); }
// Wide leaves: with the spills in the kernel (one leaf per warp: the saved
// launch matters) or left to a separate CTA launch (more leaves per warp: the
// u64 spill routine inlined costs the leaf body registers, n = 2^24 229 ->
// 245 us; the host picks)
__global__ void RS_WL_LB(WL_WARPS) k_fused_wide_wor(FusedArgs f)
{ fused_split<false>(f); warp_leaves_wide<false, true>(f.la); }
__global__ void RS_WL_LB(WL_WARPS) k_fused_wide_wr(FusedArgs f)
{ fused_split<true>(f); warp_leaves_wide<true, true>(f.la); }
__global__ void RS_WL_LB(WL_WARPS) k_fused_wide_wor_s(FusedArgs f)
{ fused_split<false>(f); warp_leaves_wide<false, true>(f.la); fused_spills<u64, false>(f.la); }
__global__ void RS_WL_LB(WL_WARPS) k_fused_wide_wr_s(FusedArgs f)
{ fused_split<true>(f); warp_leaves_wide<true, true>(f.la); fused_spills<u64, true>(f.la); }

}  // namespace rs
