// rs_kernels.cuh -- the hot-path kernels of the B200 sampler (sm_100a).
// P:n = /root/reference/PAPER.md line n.  CANON readings R1-R12: DESIGN.md.
#pragma once
#include <cuda_runtime.h>
#include "rs_math.cuh"

namespace rs {

// Checked builds (-DRS_CHECKED, tools/checked_suite.sh): shared-memory index
// checks in the leaf kernels' scatter; a violation sets bit 8 of the sticky
// device error word (rs_device_errors), which every parity test asserts is 0.
#ifdef RS_CHECKED
#define RS_CHK(c) do { if (!(c)) atomicOr(&g_rs_errors, 0x100u); } while (0)
#else
#define RS_CHK(c) do { } while (0)
#endif

// Sticky device error flags (rs_device_errors): bit 0 leaf capacity,
// bit 1 Bernoulli chunk capacity.  Defined in rs_kernels.cu (librs.cu is a
// single translation unit).

constexpr int SPLIT_NT = 512;                     // top CTA: narrow levels use lane groups
constexpr int SPLIT_LEVELS = 11;                 // levels expanded per split phase
constexpr int SPLIT_WIDTH = 1 << SPLIT_LEVELS;   // nodes per CTA at the phase's last level

#ifndef RS_LEAF_NT
#define RS_LEAF_NT 512
#endif
constexpr int LEAF_NT = RS_LEAF_NT;              // threads per leaf CTA
#ifndef RS_LEAF_MINB
#define RS_LEAF_MINB 2      // 2 CTAs per SM (64 registers): wide leaves 15 % faster
#endif
constexpr int LEAF_CAP = 2048;                   // draws held on chip per leaf
constexpr int LEAF_EPT = LEAF_CAP / LEAF_NT;     // elements per thread

// ---------------------------------------------------------------------------
// Block-wide exclusive scans (warp shuffles + one smem round).
// ---------------------------------------------------------------------------
template <typename T, int NT>
__device__ __forceinline__ T block_exclusive_scan(T v, T *warp_tmp, T *total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tmp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        T w = lane < NT / 32 ? warp_tmp[lane] : T(0);
        T wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < NT / 32) warp_tmp[lane] = wi - w;
        if (lane == NT / 32 - 1) *total = wi;
    }
    __syncthreads();
    return incl - v + warp_tmp[wid];
}

// In-place exclusive scan of a[0..n) (n <= NT * per-thread chunk); a[n] = total.
template <typename T, int NT>
__device__ __forceinline__ void block_scan_array(T *a, int n, T *warp_tmp, T *total)
{
    const int per = (n + NT - 1) / NT;
    const int beg = threadIdx.x * per;
    T s = 0;
    for (int i = 0; i < per; ++i) if (beg + i < n) s += a[beg + i];
    T ex = block_exclusive_scan<T, NT>(s, warp_tmp, total);
    for (int i = 0; i < per; ++i) {
        if (beg + i < n) { const T v = a[beg + i]; a[beg + i] = ex; ex += v; }
    }
    __syncthreads();
    if (threadIdx.x == 0) a[n] = *total;
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Split kernel (row a3/a4): expand SPLIT_LEVELS levels of the recursion tree
// (Fig. 1) below each input node in shared memory, drawing one
// deviate per node keyed by its id; offsets propagate top-down as an
// exclusive scan of the children's counts under the parent's offset.
// ---------------------------------------------------------------------------
struct SplitArgs {
    u64 N, seed;
    int wr;          // 0: hypergeometric splits (WOR); 1: binomial (WR)
    int ds;          // depth of the input nodes
    u64 node0;       // index (at depth ds) of the node handled by CTA 0
    int nlev;        // levels to expand (<= SPLIT_LEVELS)
    const u64 *in_cnt, *in_off;     // per CTA (nullptr: use root_cnt/root_off)
    u64 root_cnt, root_off;
    u64 *out_cnt, *out_off;         // 2^nlev per CTA (intermediate phase) or
    u32 *leaf_cnt;                  // leaf phase: u32 counts + u64 offsets
    u64 *leaf_off;
};

__global__ void __launch_bounds__(SPLIT_NT) k_split(SplitArgs a);
__global__ void __launch_bounds__(SPLIT_NT) k_split_wr(SplitArgs a);

// The narrow top of the tree in ONE cooperative launch (a CTA per SM, grid
// barrier between levels): each level's nodes are spread over the grid's
// warps -- a warp per node (hgd_tp) while there are few nodes, then 8-lane
// groups, then a thread per node -- so a level costs about one deviate's
// latency plus a barrier, with no launch or cold instruction cache per level.
#ifndef RS_COOP_NT
#define RS_COOP_NT 256
#endif
constexpr int COOP_NT = RS_COOP_NT;          // (256: up to 255 registers -- the deviates spill at 128)
struct CoopArgs {
    u64 N, seed;
    int ds, nlev, D;                 // levels ds .. ds + nlev - 1 are split here
    u64 node0;                       // subtree root index at depth ds
    u64 root_cnt;
    u64 *buf_cnt[2], *buf_off[2];    // level outputs alternate (ping, pong)
    u32 *leaf_cnt;                   // ds + nlev == D: the leaf level's u32 counts + u64 offsets
    u64 *leaf_off;
    u32 *bar;                        // grid barrier counter (zeroed by the call)
};
__global__ void __launch_bounds__(COOP_NT, 1) k_split_coop(CoopArgs a);
__global__ void __launch_bounds__(COOP_NT, 1) k_split_coop_wr(CoopArgs a);

// One tree level across the whole GPU: thread j splits node (d, node0 + j).
constexpr int LEVEL_NT = 128;
#ifndef RS_SPLIT_TOP
#define RS_SPLIT_TOP 7
#endif
constexpr int SPLIT_TOP = RS_SPLIT_TOP;          // levels expanded by the single top CTA (then level kernels)
struct LevelArgs {
    u64 N, seed;
    int wr, d;
    u64 node0, width;
    const u64 *in_cnt, *in_off;
    u64 *out_cnt, *out_off;        // next level (intermediate) or
    u32 *leaf_cnt;                 // leaf level: u32 counts + u64 offsets
    u64 *leaf_off;
};
#ifndef RS_LV_MINB
#define RS_LV_MINB 8        // 64 registers (measured headline step -27 us vs 4)
#endif
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level(LevelArgs a);
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level_wr(LevelArgs a);
// the same with G = 32 / 8 lanes per node (parallel rejection iterations, narrow levels)
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level_g32(LevelArgs a);
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level_g8(LevelArgs a);
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level_wr_g32(LevelArgs a);
__global__ void __launch_bounds__(LEVEL_NT, RS_LV_MINB) k_split_level_wr_g8(LevelArgs a);
#ifndef RS_LV_G32_MAXW
#define RS_LV_G32_MAXW (1u << 12)     // level widths up to this take 32 lanes per node
#endif
#ifndef RS_LV_G8_MAXW
#define RS_LV_G8_MAXW (1u << 14)      // ... then 8 lanes per node
#endif
// The last 2, 3 or 4 levels in one launch, a thread per subtree.
#ifndef RS_D3_MINB
#define RS_D3_MINB 8      // 64 registers: twice the warps (measured: split 1.66 -> 1.49 ms)
#endif
__global__ void __launch_bounds__(LEVEL_NT, RS_D3_MINB) k_split_deep2(LevelArgs a);
__global__ void __launch_bounds__(LEVEL_NT, RS_D3_MINB) k_split_deep3(LevelArgs a);
__global__ void __launch_bounds__(LEVEL_NT, RS_D3_MINB) k_split_deep4(LevelArgs a);
__global__ void __launch_bounds__(LEVEL_NT, 4) k_split_deep2_wr(LevelArgs a);
__global__ void __launch_bounds__(LEVEL_NT, RS_D3_MINB) k_split_deep3_wr(LevelArgs a);
__global__ void __launch_bounds__(LEVEL_NT, 4) k_split_deep4_wr(LevelArgs a);

// ---------------------------------------------------------------------------
// Leaf kernels (rows a5/a6/a7/a8).
// ---------------------------------------------------------------------------
struct LeafArgs {
    u64 N, seed;
    int D;                 // leaf depth
    u64 leaf0;             // global index of the first leaf of this launch
    u64 nleaves;
    const u32 *cnt;        // per-leaf sample (or excluded) counts
    const u64 *off;        // per-leaf output offsets (WOR/WR) / core offsets (complement)
    u64 out_base;          // complement: subtracted from leaf output positions
    u64 tiles_per_leaf;    // complement tiling
    u64 *out;
    u32 *spill;            // warp kernel: leaves it could not hold on chip (appended)
    u32 *spill_n;          //   ... and their count; the CTA kernel then walks this list
    const u32 *list;       // CTA kernel: if set, process only list[0 .. *list_n)
    const u32 *list_n;
    RoundKeys rk;          // Philox round keys of seed (round_keys(seed))
    u64 gV;                // != 0: graph calls, store packed edges of G(gV, .) (NEXT-3)
    u32 topup_max;         // warp *_tu kernels: most new values topped up per leaf (<= 32)
    u32 *status;           // per-call status word (bit 0: a leaf exceeded the on-chip capacity)
    u32 cap;               // CTA kernel draw capacity (0: LEAF_CAP; rs_set_option(RS_OPT_LEAF_CAP), tests)
    u32 lp_cr;             // LP kernels: ceil_log2 of the launch's largest leaf range (generation tag shift)
    u32 span_log;          // fused kernels: CTA c owns leaves [c << span_log, (c + 1) << span_log)
    u32 wcap;              // warp kernels: != 0 spills every leaf of more draws (RS_OPT_WARP_CAP, tests)
    u32 *dup;              // SD warp kernels: leaves whose round drew a duplicate (appended) ...
    u32 *dup_n;            //   ... and their count; the LS kernel then completes them
};

__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_wor32(LeafArgs a);
__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_wor64(LeafArgs a);
__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_wr32(LeafArgs a);
__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_wr64(LeafArgs a);
__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_comp32(LeafArgs a);
__global__ void __launch_bounds__(LEAF_NT, RS_LEAF_MINB) k_leaf_comp64(LeafArgs a);

// Warp-per-leaf kernels (u32 keys): the common path; see rs_leaf.cuh.
#ifndef RS_WL_MINB
#define RS_WL_MINB 1
#endif
#if RS_WL_MINB
#define RS_WL_LB(nw) __launch_bounds__(32 * (nw), RS_WL_MINB)
#else
#define RS_WL_LB(nw) __launch_bounds__(32 * (nw))
#endif
#ifndef RS_WL_WARPS
#define RS_WL_WARPS 16
#endif
// warps (independent leaves) per CTA: measured best at 16 (one 16-warp CTA per
// SM) for the counting-sort kernel and at 8 for the bitmap kernel
constexpr int WL_WARPS = RS_WL_WARPS;
#ifndef RS_WB_WARPS
#define RS_WB_WARPS 8
#endif
#ifndef RS_WB_MINB
#define RS_WB_MINB 0         // 0: no minimum-blocks bound (ptxas' own choice, 80 registers: measured fastest, cfg3a
                             // leaf 6.11 ms; an explicit bound of 1 generated slower code, 6.89; 4: 64 registers, 6.50)
#endif
#if RS_WB_MINB
#define RS_WB_LB __launch_bounds__(32 * WB_WARPS, RS_WB_MINB)
#else
#define RS_WB_LB __launch_bounds__(32 * WB_WARPS)
#endif
constexpr int WB_WARPS = RS_WB_WARPS;
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wor(LeafArgs a);
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wr(LeafArgs a);
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_gnm(LeafArgs a);
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wor_tu(LeafArgs a);
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_gnm_tu(LeafArgs a);
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wor_tu_p2(LeafArgs a);
#ifndef RS_WR_WARPS
#define RS_WR_WARPS 16
#endif
constexpr int WR_WARPS = RS_WR_WARPS;   // warps per CTA of the power-of-two WR kernel
__global__ void RS_WL_LB(WR_WARPS) k_leaf_warp_wr_p2(LeafArgs a);
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wor_p2(LeafArgs a);
// power-of-two WOR for ranges where duplicates are rare: the main kernel without the duplicate
// path (its leaves with a duplicate listed) + the top-up kernel over that list
#ifndef RS_SD_WARPS
#define RS_SD_WARPS 16
#endif
constexpr int SD_WARPS = RS_SD_WARPS;   // warps per CTA of the duplicate-free kernel
__global__ void RS_WL_LB(SD_WARPS) k_leaf_warp_wor_sd_p2(LeafArgs a);
__global__ void RS_WL_LB(WL_WARPS) k_leaf_warp_wor_tu_p2_ls(LeafArgs a);
// wide leaf ranges (> 2^32 - 4096): 31-bit keys + payload (rs_leaf_wide.cuh)
#ifndef RS_WW_WARPS
#define RS_WW_WARPS 12      // 167 registers (16 warps: 128 with 384 B spills; measured n = 2^28 leaf sweep 2.28 -> 1.90 ms)
#endif
#ifndef RS_WW_MINB
#define RS_WW_MINB 1
#endif
#if RS_WW_MINB
#define RS_WW_LB __launch_bounds__(32 * WW_WARPS, RS_WW_MINB)
#else
#define RS_WW_LB __launch_bounds__(32 * WW_WARPS)
#endif
constexpr int WW_WARPS = RS_WW_WARPS;   // warps per CTA of the wide kernels
__global__ void RS_WW_LB k_leaf_warp_wide_wor(LeafArgs a);
__global__ void RS_WW_LB k_leaf_warp_wide_wr(LeafArgs a);
// Small trees: split + leaves in one launch (rs_fused.cuh); CTA c owns the
// WL_WARPS leaves under node c at depth D - lb of the shard rooted at (s, idx).
struct FusedArgs {
    LeafArgs la;           // la.cnt / la.off = leaf_cnt / leaf_off, la.span_log = lb
    u64 N, seed;
    int s, D, lb;
    u64 idx, root_cnt;
    u32 *leaf_cnt;
    u64 *leaf_off;
    u64 *lv_cnt[2], *lv_off[2];   // intermediate levels wider than a CTA's warps (ws ping / pong)
};
#ifndef RS_FUSED_MAXD
#define RS_FUSED_MAXD 14   // shard trees of <= 2^14 leaves (deeper: the per-lane levels are slower than the level kernels)
#endif
#ifndef RS_FUSED_CTA_LOG
#define RS_FUSED_CTA_LOG 7 // at most 2^7 CTAs (one wave of one 16-warp CTA per SM): deeper trees give each CTA more levels
#endif
__global__ void RS_WL_LB(WL_WARPS) k_fused_wor_tu(FusedArgs f);
__global__ void RS_WL_LB(WL_WARPS) k_fused_wor_tu_p2(FusedArgs f);
__global__ void RS_WL_LB(WL_WARPS) k_fused_wr(FusedArgs f);
__global__ void RS_WL_LB(WL_WARPS) k_fused_wr_p2(FusedArgs f);
__global__ void RS_WL_LB(WL_WARPS) k_fused_wide_wor(FusedArgs f);
__global__ void RS_WL_LB(WL_WARPS) k_fused_wide_wr(FusedArgs f);
__global__ void RS_WL_LB(WL_WARPS) k_fused_wide_wor_s(FusedArgs f);
__global__ void RS_WL_LB(WL_WARPS) k_fused_wide_wr_s(FusedArgs f);
// Ordered linear-probing leaf kernels (rs_leaf_lp.cuh): the default WOR / WR path.
#ifndef RS_LP_WARPS
#define RS_LP_WARPS 16
#endif
constexpr int LP_WARPS = RS_LP_WARPS;
__global__ void __launch_bounds__(32 * LP_WARPS, 1) k_leaf_lp_wor(LeafArgs a);
__global__ void __launch_bounds__(32 * LP_WARPS, 1) k_leaf_lp_wr(LeafArgs a);
#ifndef RS_WL_TU_LOG
#define RS_WL_TU_LOG 21
#endif
constexpr u64 WL_TU_RMAX = 1ull << RS_WL_TU_LOG;   // leaf ranges up to this take the top-up kernels
// Warp-per-leaf bitmap kernels for leaf ranges r <= 2^15 (rs_leaf_bitmap.cuh).
__global__ void RS_WB_LB k_leaf_bitmap_wor(LeafArgs a);
__global__ void RS_WB_LB k_leaf_bitmap_comp(LeafArgs a);
__global__ void RS_WB_LB k_leaf_bitmap_wor_g(LeafArgs a);
__global__ void RS_WB_LB k_leaf_bitmap_comp_g(LeafArgs a);

// ---------------------------------------------------------------------------
// Bernoulli (row a9): one chunk per CTA (dynamic ticket order), geometric
// skips + block scan, decoupled look-back over chunk counts, store.
// ---------------------------------------------------------------------------

struct BernArgs {
    u64 N, seed;
    int Db;
    u64 chunk0, nchunks;
    double log1m_rho;
    u64 *status;           // nchunks look-back words (zeroed)
    u32 *ticket;           // zeroed
    u64 *out;
    u64 capacity;
    u64 *count_dev;
    RoundKeys rk;          // Philox round keys of seed
    u64 gV;                // != 0: graph calls, store packed edges (NEXT-3)
};

__global__ void k_bernoulli(BernArgs a);                           // chunk ranges <= 2^16
__global__ void k_bernoulli32(BernArgs a);                         // chunk ranges <= 2^24
__global__ void k_bernoulli64(BernArgs a);                         // chunk ranges <= 2^32
__global__ void k_bernoulli64w(BernArgs a);                        // larger chunk ranges
__global__ void k_bernoulli32d(BernArgs a);                        // fp64 skip candidates (small rho)
__global__ void k_bernoulli64d(BernArgs a);
__global__ void k_bernoulli32d_g(BernArgs a);
__global__ void k_bernoulli64d_g(BernArgs a);
constexpr double BF64_RHO = 0x1p-12;                               // fp64 candidates below this rho
__global__ void k_bernoulli_g(BernArgs a);                         // G(n, p) variants (NEXT-3)
__global__ void k_bernoulli32_g(BernArgs a);
__global__ void k_bernoulli64_g(BernArgs a);
__global__ void k_bernoulli64w_g(BernArgs a);

// NEXT-4 (rs_algb.cuh): Algorithm B's repair -- S[0..np) minus the elements at
// the sorted 1-based positions R[0..nr) -> out (compaction)
constexpr u32 AB_THREADS = 256, AB_PER = 16, AB_TILE = AB_THREADS * AB_PER, AB_SMAX = 256;
__global__ void __launch_bounds__(AB_THREADS) k_algb_compact(const u64 *__restrict__ S, u64 np,
                                                             const u64 *__restrict__ R, u64 nr,
                                                             u64 *__restrict__ out);

// Validation (tests / bench correctness checks).
__global__ void k_digest(const u64 *v, u64 n, u64 base, u64 *acc);
__global__ void k_validate(const u64 *v, u64 n, u64 N, int strict, u64 *bad);
__global__ void k_iota(u64 *out, u64 n);

}  // namespace rs
