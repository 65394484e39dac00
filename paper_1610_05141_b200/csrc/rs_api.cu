// rs_api.cu -- host side of librs.so: argument checks, planning (depth,
// complement, Algorithm P path replay for shards), workspace layout and
// kernel launches.  Declarations and contracts: include/rs.h.
// P:n = /root/reference/PAPER.md line n; CANON readings: DESIGN.md section 2.
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "rs.h"
#include "rs_kernels.cuh"

using namespace rs;

namespace {

thread_local rs_status t_last = RS_OK;
int g_leaf_path = 0;                    // rs_set_option(RS_OPT_LEAF_PATH)
int g_topup_max = 32;                   // rs_set_option(RS_OPT_TOPUP_MAX)
int g_leaf_cap = 0;                     // rs_set_option(RS_OPT_LEAF_CAP) (tests: force overflows)
int g_split_coop = 1;                   // rs_set_option(RS_OPT_SPLIT_COOP): cooperative top of the split tree
int g_fused = 1;                        // rs_set_option(RS_OPT_FUSED): small trees in one launch (rs_fused.cuh)
int g_warp_cap = 0;                     // rs_set_option(RS_OPT_WARP_CAP): warp kernels spill leaves above it (tests)
#ifndef RS_WL_WOR_TU_ALL
#define RS_WL_WOR_TU_ALL 1
#endif
#ifndef RS_WL_SD
#define RS_WL_SD 1          // power-of-two WOR above the top-up cutoff: duplicate leaves to a second pass
#endif
#ifndef RS_WL_P2
#define RS_WL_P2 1
#endif
#ifndef RS_WL_P2_PLAIN
#define RS_WL_P2_PLAIN 0        // 1: large power-of-two ranges take the plain (no top-up) p2 kernel
#endif
#ifndef RS_COOP_LEVELS
#define RS_COOP_LEVELS 15               // input widths 1 .. 2^14
#endif
thread_local uint64_t t_launches = 0;

rs_status ret(rs_status s) { t_last = s; return s; }

cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// ---- benchmark instrumentation (rs_timing_*) ------------------------------
struct TimedSpan { int cls; cudaEvent_t a, b; };
std::mutex g_tmu;
bool g_timing = false;
std::vector<TimedSpan> g_spans;
std::vector<cudaEvent_t> g_free_events;
double g_ms[4];
uint64_t g_cnt[4];

cudaEvent_t get_event()
{
    if (!g_free_events.empty()) {
        cudaEvent_t e = g_free_events.back();
        g_free_events.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// RAII span: records a start event on construction, an end event on end().
struct Span {
    bool on = false; int cls = 0; cudaEvent_t a{}, b{}; cudaStream_t st{};
    Span(int c, cudaStream_t s) : cls(c), st(s)
    {
        std::lock_guard<std::mutex> g(g_tmu);
        if (!g_timing) return;
        on = true;
        a = get_event(); b = get_event();
        cudaEventRecord(a, st);
    }
    void end()
    {
        if (!on) return;
        cudaEventRecord(b, st);
        std::lock_guard<std::mutex> g(g_tmu);
        g_spans.push_back({cls, a, b});
        on = false;
    }
};

rs_status cuda_ok()
{
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RS_OK : RS_ECUDA;
}

bool have_device()
{
    int n = 0;
    return cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
}

int log2_world(int world)
{
    int s = 0;
    while ((1 << s) < world) ++s;
    return ((1 << s) == world && s <= 3) ? s : -1;
}

// ---------------------------------------------------------------------------
// Plans.
// ---------------------------------------------------------------------------
struct TreePlan {
    int mode;               // RS_MODE_WOR / RS_MODE_WR
    u64 N, n, m, seed;
    int D, s;
    u64 idx;                // the subtree root is node (s, idx)
    bool comp;
    u64 root_cnt;           // core count of the subtree root (s, idx)
    u64 root_core_off;      // core offset of that root in the world=1 tree
    u64 shard_lo, shard_hi; // shard's offsets [lo, hi)
    u64 leaf0, nleaves;     // shard's leaves
    u64 r_max;              // largest leaf range
    u64 local_count, global_offset;
    u64 gV;                 // graph calls: vertex count (outputs are packed edges)
    int top;                // levels expanded by the single top CTA
    // workspace layout
    size_t o_ping_cnt, o_ping_off, o_pong_cnt, o_pong_off, o_leaf_cnt, o_leaf_off, o_spill, bytes;
};

// Plan for the subtree rooted at node (s, idx) of the split tree, s <= D:
// Algorithm P's path replay gives its count and its offset in the global
// output ("<= ceil(log p) hypergeometric random deviates").  Shards
// are the nodes at depth log2(world); ranges of leaves are unions of nodes.
rs_status plan_node(int mode, u64 N, u64 n, u64 seed, int s, u64 idx, TreePlan &p)
{
    memset(&p, 0, sizeof p);
    if (N >= (1ull << 63)) return RS_EINVAL;
    if (mode == RS_MODE_WOR && n > N) return RS_EINVAL;
    if (mode == RS_MODE_WR && N == 0 && n > 0) return RS_EINVAL;
    if (n >= (1ull << 40)) return RS_EINVAL;            // > 8 TiB of output
    p.mode = mode; p.N = N; p.n = n; p.seed = seed;
    p.comp = (mode == RS_MODE_WOR) && (n > N - n);      // R8: 2n > N
    p.m = p.comp ? N - n : n;
    p.D = tree_depth(p.m);
    if (s < 0 || s > p.D || s > 62 || idx >= (1ull << s)) return RS_EINVAL;
    p.s = s; p.idx = idx;
    // Algorithm P (Fig. 2): follow the s splits on the root path
    u64 k = p.m, off = 0;
    for (int e = 0; e < s; ++e) {
        const u64 anc = idx >> (s - e);
        const u64 x = split_node(mode == RS_MODE_WR, N, e, anc, k, seed);
        if ((idx >> (s - e - 1)) & 1) { off += x; k -= x; } else { k = x; }
    }
    p.root_cnt = k;
    p.root_core_off = off;
    p.shard_lo = bound_at(N, s, idx);
    p.shard_hi = bound_at(N, s, idx + 1);
    p.local_count = p.comp ? (p.shard_hi - p.shard_lo) - k : k;
    p.global_offset = p.comp ? p.shard_lo - off : off;
    p.nleaves = 1ull << (p.D - s);
    p.leaf0 = idx << (p.D - s);
    p.r_max = (N >> p.D) + ((N & ((1ull << p.D) - 1)) != 0);
    // split: one CTA expands depths s..s+top, then one launch per level
    p.top = (p.D - s) < SPLIT_TOP ? (p.D - s) : SPLIT_TOP;
    const u64 wmax = 1ull << (p.D - s > 0 ? p.D - s - 1 : 0);   // widest intermediate level
    size_t o = 0;
    p.o_ping_cnt = o; o = align256(o + wmax * 8);
    p.o_ping_off = o; o = align256(o + wmax * 8);
    p.o_pong_cnt = o; o = align256(o + wmax * 8);
    p.o_pong_off = o; o = align256(o + wmax * 8);
    p.o_leaf_cnt = o; o = align256(o + p.nleaves * 4);
    p.o_leaf_off = o; o = align256(o + p.nleaves * 8);
    p.o_spill = o; o = align256(o + (2 * p.nleaves + 8) * 4);   // header (8 words), spill list, duplicate list
    p.bytes = o;
    return RS_OK;
}

// Shard rank of world = 2^s (s <= 3): node (s, rank).
rs_status plan_tree(int mode, u64 N, u64 n, u64 seed, int world, int rank, TreePlan &p)
{
    const int s = log2_world(world);
    if (s < 0 || rank < 0 || rank >= world) { memset(&p, 0, sizeof p); return RS_EINVAL; }
    return plan_node(mode, N, n, seed, s, (u64)rank, p);
}

template <typename F>
void set_smem(F *kernel, size_t bytes)
{
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Persistent leaf grid: every resident CTA slot once (occupancy x SMs),
// capped by the number of work items; the kernels grid-stride over leaves.
unsigned leaf_grid(const void *kern, int threads, size_t smem, u64 work)
{
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
#ifndef RS_CARVEOUT
#define RS_CARVEOUT 70      // leaves >= 164 KB of smem (the 16-warp leaf CTA needs 141 KB) and more L1 for spills (measured +0.4 %)
#endif
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, RS_CARVEOUT);
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem) != cudaSuccess || per < 1)
        per = 1;
    const u64 g = (u64)sms * (u64)per;
    return (unsigned)(work < g ? (work ? work : 1) : g);
}

// Small trees on the warp-leaf paths: the split and the leaves in one launch
// (rs_fused.cuh), then the (usually empty) spill pass.  Returns false (nothing
// launched) when the plan is not one.
bool run_fused(const TreePlan &p, u64 *out, unsigned char *ws, cudaStream_t st)
{
    const int depth = p.D - p.s;
    if (!g_fused || depth < 0 || depth > RS_FUSED_MAXD || p.comp || p.gV || g_leaf_path != 0) return false;
    const bool wr = (p.mode == RS_MODE_WR);
    const bool wide = p.r_max > 0xfffff000ull;
    if (p.r_max <= BM_RMAX && !wr) return false;                   // bitmap leaves
    const bool w32 = !wide && (p.N >> p.D) >= (1ull << 11);
    if (!w32 && !wide) return false;
    const bool p2 = (p.N & (p.N - 1)) == 0 && RS_WL_P2;
    const bool tu = p.r_max <= WL_TU_RMAX;
    if (w32 && !wr && !(tu || RS_WL_WOR_TU_ALL)) return false;     // the plain WOR kernel
    if (w32 && !wr && p2 && !tu && RS_WL_P2_PLAIN) return false;
    u32 *status = (u32 *)(ws + p.o_spill);
    u32 *leaf_cnt = (u32 *)(ws + p.o_leaf_cnt);
    u64 *leaf_off = (u64 *)(ws + p.o_leaf_off);
    FusedArgs f;
    memset(&f, 0, sizeof f);
    LeafArgs &la = f.la;
    la.N = p.N; la.seed = p.seed; la.D = p.D;
    la.leaf0 = p.leaf0; la.nleaves = p.nleaves;
    la.cnt = leaf_cnt; la.off = leaf_off; la.out = out;
    la.rk = round_keys(p.seed);
    la.status = status;
    la.cap = (u32)g_leaf_cap;
    la.wcap = (u32)g_warp_cap;
    la.topup_max = (u32)g_topup_max;
    la.spill_n = status + 1;
    la.spill = status + 8;
    f.N = p.N; f.seed = p.seed; f.s = p.s; f.D = p.D;
    f.lb = depth < FUSED_LB ? depth : depth > FUSED_LB + RS_FUSED_CTA_LOG ? depth - RS_FUSED_CTA_LOG : FUSED_LB;
    la.span_log = (u32)f.lb;
    f.idx = p.idx; f.root_cnt = p.root_cnt;
    f.leaf_cnt = leaf_cnt; f.leaf_off = leaf_off;
    f.lv_cnt[0] = (u64 *)(ws + p.o_ping_cnt); f.lv_off[0] = (u64 *)(ws + p.o_ping_off);
    f.lv_cnt[1] = (u64 *)(ws + p.o_pong_cnt); f.lv_off[1] = (u64 *)(ws + p.o_pong_off);
    const bool wide_sep = wide && f.lb > FUSED_LB;            // wide, > 1 leaf per warp: spills launched apart
    void (*fk)(FusedArgs) = wide ? (wide_sep ? (wr ? k_fused_wide_wr : k_fused_wide_wor)
                                             : (wr ? k_fused_wide_wr_s : k_fused_wide_wor_s))
                          : wr ? (p2 ? k_fused_wr_p2 : k_fused_wr)
                               : (p2 ? k_fused_wor_tu_p2 : k_fused_wor_tu);
    const size_t fsm = wide ? sizeof(WarpLeafW) * WL_WARPS : sizeof(WarpLeaf) * WL_WARPS;
    (void)leaf_grid((const void *)fk, 32 * WL_WARPS, fsm, 1);      // (attributes)
    Span sp(1, st);
    static_assert(sizeof(SLeaf<u32>) <= sizeof(WarpLeaf) * WL_WARPS, "fused kernels: spills reuse the warps' smem");
    fk<<<1u << (depth - f.lb), 32 * WL_WARPS, fsm, st>>>(f);   // (spilled leaves: its last CTA, unless wide_sep)
    ++t_launches;
    if (wide_sep) {                                             // the CTA kernel with u64 keys
        LeafArgs lb = la;
        lb.spill = nullptr; lb.spill_n = nullptr;
        lb.list = status + 8; lb.list_n = status + 1;
        void (*kern)(LeafArgs) = wr ? k_leaf_wr64 : k_leaf_wor64;
        const unsigned g2 = leaf_grid((const void *)kern, LEAF_NT, sizeof(SLeaf<u64>),
                                      p.nleaves < 2ull * 148 ? p.nleaves : 2ull * 148);
        kern<<<g2, LEAF_NT, sizeof(SLeaf<u64>), st>>>(lb);
        ++t_launches;
    }
    sp.end();
    return true;
}

// Launch the split phases and the leaf kernel of a tree plan.  The call's
// status word (ws + o_spill) is zeroed here when clear_status is set;
// otherwise it accumulates over several run_tree calls (host-buffer batches).
rs_status run_tree(const TreePlan &p, u64 *out, unsigned char *ws, cudaStream_t st, bool clear_status = true)
{
    if (p.local_count == 0) return RS_OK;
    u32 *status = (u32 *)(ws + p.o_spill);
    const bool warp_path = (!(p.r_max <= BM_RMAX && p.mode == RS_MODE_WOR && g_leaf_path != 1) &&
                            !p.comp && p.r_max <= 0xfffff000ull && g_leaf_path != 1 &&
                            (p.N >> p.D) >= (1ull << 11)) ||
                           (!p.comp && p.r_max > 0xfffff000ull && g_leaf_path != 1 && !p.gV);   // wide warp path
    (void)warp_path;
    if (clear_status)      // the status header (status, spill / duplicate counts, barrier) in one memset
        cudaMemsetAsync(status, 0, 32, st);
    else
        cudaMemsetAsync(status + 1, 0, 28, st);
    if (run_fused(p, out, ws, st)) return cuda_ok();
    u64 *ping_cnt = (u64 *)(ws + p.o_ping_cnt), *ping_off = (u64 *)(ws + p.o_ping_off);
    u64 *pong_cnt = (u64 *)(ws + p.o_pong_cnt), *pong_off = (u64 *)(ws + p.o_pong_off);
    u32 *leaf_cnt = (u32 *)(ws + p.o_leaf_cnt);
    u64 *leaf_off = (u64 *)(ws + p.o_leaf_off);
    Span sp_split(0, st);
    const u64 *in_cnt = ping_cnt, *in_off = ping_off;
    int top = p.top;
#ifndef RS_COOP_MIN_LEVELS
#define RS_COOP_MIN_LEVELS 6            // shallower trees: the single top CTA (no grid barrier, smaller launch)
#endif
    if (g_split_coop && p.D - p.s >= RS_COOP_MIN_LEVELS) {   // the narrow top (input widths <= 2^14) in one cooperative launch
        CoopArgs a;
        memset(&a, 0, sizeof a);
        a.N = p.N; a.seed = p.seed;
        a.ds = p.s; a.D = p.D; a.node0 = p.idx; a.root_cnt = p.root_cnt;
        a.nlev = (p.D - p.s) < RS_COOP_LEVELS ? (p.D - p.s) : RS_COOP_LEVELS;
        a.buf_cnt[0] = ping_cnt; a.buf_off[0] = ping_off; a.buf_cnt[1] = pong_cnt; a.buf_off[1] = pong_off;
        a.leaf_cnt = leaf_cnt; a.leaf_off = leaf_off;
        a.bar = status + 2;                            // zeroed above
        static int sms = 0;
        if (!sms) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (sms <= 0) sms = 148;
        }
        void *args[] = {&a};
        const void *kf = (p.mode == RS_MODE_WR) ? (const void *)k_split_coop_wr : (const void *)k_split_coop;
        if (cudaLaunchCooperativeKernel(kf, dim3(sms), dim3(COOP_NT), args, 0, st) != cudaSuccess) return RS_ECUDA;
        ++t_launches;
        top = a.nlev;
        const int lastbuf = (a.nlev - 1) & 1;          // where level ds + nlev's counts are
        in_cnt = lastbuf ? pong_cnt : ping_cnt;
        in_off = lastbuf ? pong_off : ping_off;
    } else {   // top levels s .. s+top in one CTA
        SplitArgs a;
        memset(&a, 0, sizeof a);
        a.N = p.N; a.seed = p.seed; a.wr = (p.mode == RS_MODE_WR);
        a.ds = p.s; a.nlev = p.top; a.node0 = p.idx;
        a.root_cnt = p.root_cnt; a.root_off = 0;        // offsets local to the shard
        if (p.s + p.top == p.D) { a.leaf_cnt = leaf_cnt; a.leaf_off = leaf_off; }
        else { a.out_cnt = ping_cnt; a.out_off = ping_off; }
        (a.wr ? k_split_wr : k_split)<<<1, SPLIT_NT, 0, st>>>(a);
        ++t_launches;
    }
    // the last NL levels (when there are level kernels at all) in one launch,
    // a thread per depth-(D-NL) subtree
#ifndef RS_SPLIT_DEEP
#define RS_SPLIT_DEEP 3
#endif
    const int below = p.D - p.s - top;                 // levels after the top
    // (only where the deep levels are wide: a narrow subtree per thread is a
    // chain of 2^NL - 1 sequential deviates, slower than NL lane-group levels)
#ifndef RS_SPLIT_DEEP_MINW
#define RS_SPLIT_DEEP_MINW (1ull << 15)
#endif
    const int NL = (below >= RS_SPLIT_DEEP + 1 && (1ull << (p.D - p.s - RS_SPLIT_DEEP)) >= RS_SPLIT_DEEP_MINW)
                       ? RS_SPLIT_DEEP : 0;
    const int flip0 = (in_cnt == pong_cnt) ? 1 : 0;   // the next output goes to the other buffer
    for (int d = p.s + top; d < p.D - NL; ++d) {      // one launch per level
        LevelArgs a;
        memset(&a, 0, sizeof a);
        a.N = p.N; a.seed = p.seed; a.wr = (p.mode == RS_MODE_WR); a.d = d;
        a.width = 1ull << (d - p.s);
        a.node0 = p.idx << (d - p.s);
        a.in_cnt = in_cnt; a.in_off = in_off;
        const bool flip = (((d - p.s - top) & 1) == 0) != (flip0 == 1);
        u64 *oc = flip ? pong_cnt : ping_cnt, *oo = flip ? pong_off : ping_off;
        if (d + 1 == p.D) { a.leaf_cnt = leaf_cnt; a.leaf_off = leaf_off; }
        else { a.out_cnt = oc; a.out_off = oo; }
        const u32 G = a.width <= RS_LV_G32_MAXW ? 32 : a.width <= RS_LV_G8_MAXW ? 8 : 1;
        const u64 grid = (a.width * G + LEVEL_NT - 1) / LEVEL_NT;
        void (*lk)(LevelArgs) = G == 32 ? (a.wr ? k_split_level_wr_g32 : k_split_level_g32)
                              : G == 8  ? (a.wr ? k_split_level_wr_g8 : k_split_level_g8)
                                        : (a.wr ? k_split_level_wr : k_split_level);
        lk<<<(unsigned)grid, LEVEL_NT, 0, st>>>(a);
        ++t_launches;
        in_cnt = oc; in_off = oo;
    }
    if (NL) {
        LevelArgs a;
        memset(&a, 0, sizeof a);
        const int d = p.D - NL;
        a.N = p.N; a.seed = p.seed; a.wr = (p.mode == RS_MODE_WR); a.d = d;
        a.width = 1ull << (d - p.s);
        a.node0 = p.idx << (d - p.s);
        a.in_cnt = in_cnt; a.in_off = in_off;
        a.leaf_cnt = leaf_cnt; a.leaf_off = leaf_off;
        const u64 grid = (a.width + LEVEL_NT - 1) / LEVEL_NT;
        void (*dk)(LevelArgs) = a.wr ? (NL == 2 ? k_split_deep2_wr : NL == 3 ? k_split_deep3_wr : k_split_deep4_wr)
                                     : (NL == 2 ? k_split_deep2 : NL == 3 ? k_split_deep3 : k_split_deep4);
        dk<<<(unsigned)grid, LEVEL_NT, 0, st>>>(a);
        ++t_launches;
    }
    sp_split.end();
    Span sp_leaf(1, st);
    LeafArgs la;
    memset(&la, 0, sizeof la);
    la.N = p.N; la.seed = p.seed; la.D = p.D;
    la.leaf0 = p.leaf0; la.nleaves = p.nleaves;
    la.cnt = leaf_cnt; la.off = leaf_off; la.out = out;
    la.rk = round_keys(p.seed);
    la.gV = p.gV;
    la.status = status;
    la.cap = (u32)g_leaf_cap;
    la.wcap = (u32)g_warp_cap;
    const bool wide = p.r_max > 0xfffff000ull;    // u32 keys (below the warp kernel's sentinels)
    const bool wr = (p.mode == RS_MODE_WR);
    void (*kern)(LeafArgs);
    size_t sm;
    if (p.r_max <= BM_RMAX && p.mode == RS_MODE_WOR && g_leaf_path != 1) {
        // small leaf ranges: warp per leaf over a bitmap (complement or WOR)
        la.out_base = p.shard_lo;
        void (*bk)(LeafArgs) = p.gV ? (p.comp ? k_leaf_bitmap_comp_g : k_leaf_bitmap_wor_g)
                                    : (p.comp ? k_leaf_bitmap_comp : k_leaf_bitmap_wor);
        const size_t bsm = sizeof(BitmapLeaf) * WB_WARPS;
        const unsigned gb = leaf_grid((const void *)bk, 32 * WB_WARPS, bsm, (p.nleaves + WB_WARPS - 1) / WB_WARPS);
        bk<<<gb, 32 * WB_WARPS, bsm, st>>>(la);
        ++t_launches;
        sp_leaf.end();
        return cuda_ok();
    } else if (p.comp) {
        la.out_base = p.shard_lo;
        la.tiles_per_leaf = (p.r_max + COMP_TILE - 1) / COMP_TILE;
        kern = wide ? k_leaf_comp64 : k_leaf_comp32;
    } else if (!wide && g_leaf_path != 1 && (p.N >> p.D) >= (1ull << 11)) {
        // common path (leaf ranges of >= 2^11 values: the warp kernels' bucket
        // function needs ceil_log2(r) >= 11): warp per leaf; leaves it cannot hold go to a spill
        // list that the CTA kernel completes right after (usually empty)
        u32 *spill_n = status + 1;        // zeroed above
        la.spill_n = spill_n;
        la.spill = status + 8;
        // leaves with many duplicates (r <= 2^21: >= 22 % of leaves) top the
        // distinct set up draw by draw instead of re-running a full round
        const bool tu = p.r_max <= WL_TU_RMAX;
        la.topup_max = (u32)g_topup_max;
        // plain WOR takes the top-up kernel at every range: since the exact
        // phase count it needs no spill slots and is faster than the plain
        // kernel (headline leaf 13.64 -> 12.88 ms); G(n, m) keeps the cutoff
        // (its _tu kernel measured slower above 2^21: 21.97 -> 23.64 ms)
#ifndef RS_WL_WOR_TU_ALL
#define RS_WL_WOR_TU_ALL 1
#endif
        // RS_OPT_LEAF_PATH = 3: the ordered linear-probing kernels (rs_leaf_lp.cuh;
        // bit-exact, measured 1.9x slower than the counting-sort warp kernels:
        // DESIGN.md section 6) when every leaf range has >= 2^11 values
        const u64 r_min = p.N >> p.D;
        if (!p.gV && g_leaf_path == 3 && r_min >= (1ull << LP_LOGT)) {
            la.lp_cr = (u32)ceil_log2(p.r_max);
            void (*lk)(LeafArgs) = wr ? k_leaf_lp_wr : k_leaf_lp_wor;
            const size_t lsm = sizeof(LPLeaf) * LP_WARPS;
            const unsigned gl = leaf_grid((const void *)lk, 32 * LP_WARPS, lsm, (p.nleaves + LP_WARPS - 1) / LP_WARPS);
            lk<<<gl, 32 * LP_WARPS, lsm, st>>>(la);
        } else {
            // N a power of two: every leaf range is one (r = N / 2^D) -> the
            // kernels compiled without the Lemire rejection path
            const bool p2 = (p.N & (p.N - 1)) == 0 && RS_WL_P2;
            void (*wk)(LeafArgs) = wr ? (p2 ? k_leaf_warp_wr_p2 : k_leaf_warp_wr)
                                 : p.gV ? (tu ? k_leaf_warp_gnm_tu : k_leaf_warp_gnm)
                                        : ((tu || RS_WL_WOR_TU_ALL)
                                               ? (p2 ? (!tu && RS_WL_P2_PLAIN ? k_leaf_warp_wor_p2 : k_leaf_warp_wor_tu_p2)
                                                     : k_leaf_warp_wor_tu)
                                               : k_leaf_warp_wor);
            // power-of-two WOR with duplicates rare (ranges above the top-up
            // cutoff): the kernel without the duplicate path, then the top-up
            // kernel over the leaves it listed (SD / LS, rs_leaf_warp.cuh)
            // (from r = 2^24: P(duplicate) ~ k^2 / 2r <= 3 %, below the ~3 % the
            // smaller kernel saves on every leaf)
            const bool sd = !wr && p2 && !p.gV && !tu && RS_WL_SD && !(RS_WL_P2_PLAIN) &&
                            (p.N >> p.D) >= (1ull << 24);
            if (sd) wk = k_leaf_warp_wor_sd_p2;
            la.dup = status + 8 + p.nleaves;
            la.dup_n = status + 4;
            const int nw = (wr && p2) ? WR_WARPS : sd ? SD_WARPS : WL_WARPS;
            const size_t wsm = sizeof(WarpLeaf) * nw;
            const u64 wgrid = (p.nleaves + nw - 1) / nw;
            const unsigned g1 = leaf_grid((const void *)wk, 32 * nw, wsm, wgrid);
            wk<<<g1, 32 * nw, wsm, st>>>(la);
            if (sd) {
                ++t_launches;
                const size_t lsm = sizeof(WarpLeaf) * WL_WARPS;
                const unsigned gl = leaf_grid((const void *)k_leaf_warp_wor_tu_p2_ls, 32 * WL_WARPS, lsm, wgrid);
                k_leaf_warp_wor_tu_p2_ls<<<gl, 32 * WL_WARPS, lsm, st>>>(la);
            }
        }
        ++t_launches;
        LeafArgs lb = la;
        lb.spill = nullptr; lb.spill_n = nullptr;
        lb.list = status + 8; lb.list_n = spill_n;
        kern = wr ? k_leaf_wr32 : k_leaf_wor32;
        sm = sizeof(SLeaf<u32>);
        const unsigned g2 = leaf_grid((const void *)kern, LEAF_NT, sm, 2ull * 148);
        kern<<<g2, LEAF_NT, sm, st>>>(lb);
        ++t_launches;
        sp_leaf.end();
        return cuda_ok();
    } else if (wide && g_leaf_path != 1 && !p.gV) {
        // wide leaf ranges: warp per leaf on 31-bit keys + payloads; the CTA
        // kernel with 64-bit keys completes the leaves it spills (ties)
        u32 *spill_n = status + 1;        // zeroed above
        la.spill_n = spill_n;
        la.spill = status + 8;
        void (*wk)(LeafArgs) = wr ? k_leaf_warp_wide_wr : k_leaf_warp_wide_wor;
        const size_t wsm = sizeof(WarpLeafW) * WW_WARPS;
        const unsigned g1 = leaf_grid((const void *)wk, 32 * WW_WARPS, wsm, (p.nleaves + WW_WARPS - 1) / WW_WARPS);
        wk<<<g1, 32 * WW_WARPS, wsm, st>>>(la);
        ++t_launches;
        LeafArgs lb = la;
        lb.spill = nullptr; lb.spill_n = nullptr;
        lb.list = status + 8; lb.list_n = spill_n;
        kern = wr ? k_leaf_wr64 : k_leaf_wor64;
        sm = sizeof(SLeaf<u64>);
        const unsigned g2 = leaf_grid((const void *)kern, LEAF_NT, sm, 2ull * 148);
        kern<<<g2, LEAF_NT, sm, st>>>(lb);
        ++t_launches;
        sp_leaf.end();
        return cuda_ok();
    } else if (wide) {
        kern = wr ? k_leaf_wr64 : k_leaf_wor64;
    } else {
        kern = wr ? k_leaf_wr32 : k_leaf_wor32;
    }
    sm = wide ? sizeof(SLeaf<u64>) : sizeof(SLeaf<u32>);
    const u64 work = p.comp ? p.nleaves * la.tiles_per_leaf : p.nleaves;
    const unsigned grid = leaf_grid((const void *)kern, LEAF_NT, sm, work);
    kern<<<grid, LEAF_NT, sm, st>>>(la);
    ++t_launches;
    sp_leaf.end();
    return cuda_ok();
}

rs_status plan_call(const TreePlan &p, u64 *out, void *ws, size_t ws_bytes, void *stream)
{
    if (!have_device()) return RS_ECUDA;
    if (p.local_count == 0) return RS_OK;
    if (!out) return RS_EINVAL;
    const cudaStream_t cs = S(stream);
    unsigned char *w = (unsigned char *)ws;
    bool own = false;
    if (w == nullptr) {
        if (cudaMallocAsync((void **)&w, p.bytes, cs) != cudaSuccess) return RS_ENOMEM;
        own = true;
    } else if (ws_bytes < p.bytes) {
        return RS_ENOMEM;
    }
    const rs_status st = run_tree(p, out, w, cs);
    if (own) cudaFreeAsync(w, cs);
    return st;
}

rs_status tree_call(int mode, u64 N, u64 n, u64 seed, int world, int rank, u64 *out,
                    void *ws, size_t ws_bytes, void *stream)
{
    if (!have_device()) return RS_ECUDA;
    TreePlan p;
    const rs_status st = plan_tree(mode, N, n, seed, world, rank, p);
    if (st != RS_OK) return st;
    return plan_call(p, out, ws, ws_bytes, stream);
}

// ---------------------------------------------------------------------------
// Bernoulli.
// ---------------------------------------------------------------------------
struct BernPlan {
    int Db, s;
    u64 chunk0, nchunks, shard_lo, shard_hi;
    double lr;
    size_t o_status, o_ticket, bytes;
};

int bern_depth(u64 N, double rho)
{
    const double t = ceil((double)N * rho / 1024.0);
    const u64 tt = t < 1.0 ? 1 : (t >= 0x1p62 ? (1ull << 62) : (u64)t);
    const int d = ceil_log2(tt);
    return d < 3 ? 3 : d;
}

rs_status plan_bern(u64 N, double rho, int world, int rank, BernPlan &p)
{
    memset(&p, 0, sizeof p);
    if (!(rho >= 0.0 && rho <= 1.0)) return RS_EINVAL;
    if (N >= (1ull << 63)) return RS_EINVAL;
    const int s = log2_world(world);
    if (s < 0 || rank < 0 || rank >= world) return RS_EINVAL;
    p.s = s;
    p.Db = bern_depth(N, rho);
    if (p.Db - s > 31) return RS_EINVAL;
    p.nchunks = 1ull << (p.Db - s);
    p.chunk0 = (u64)rank << (p.Db - s);
    p.shard_lo = bound_at(N, s, (u64)rank);
    p.shard_hi = bound_at(N, s, (u64)rank + 1);
    p.lr = log1p_(-rho);
    size_t o = 0;
    p.o_status = o; o = align256(o + p.nchunks * 8);
    p.o_ticket = o; o = align256(o + 8);
    p.bytes = o;
    return RS_OK;
}

__global__ void k_fill_range(u64 *out, u64 lo, u64 n, u64 cap, u64 *count, u64 gV)
{
    const u64 m = n < cap ? n : cap;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += (u64)gridDim.x * blockDim.x)
        out[i] = out_word(lo + i + 1, gV);
    if (blockIdx.x == 0 && threadIdx.x == 0) *count = n;
}

rs_status bern_call(u64 N, double rho, u64 seed, int world, int rank, u64 *out, u64 capacity,
                    u64 *count_dev, void *ws, size_t ws_bytes, void *stream, u64 gV = 0)
{
    if (!have_device()) return RS_ECUDA;
    BernPlan p;
    rs_status st = plan_bern(N, rho, world, rank, p);
    if (st != RS_OK) return st;
    if (!count_dev) return RS_EINVAL;
    const cudaStream_t cs = S(stream);
    if (rho == 0.0 || N == 0 || rho == 1.0) {
        const u64 n = (rho == 0.0 || N == 0) ? 0 : p.shard_hi - p.shard_lo;
        k_fill_range<<<n ? 1184 : 1, 256, 0, cs>>>(out, p.shard_lo, n, capacity, count_dev, gV);
        ++t_launches;
        return cuda_ok();
    }
    unsigned char *w = (unsigned char *)ws;
    bool own = false;
    if (w == nullptr) {
        if (cudaMallocAsync((void **)&w, p.bytes, cs) != cudaSuccess) return RS_ENOMEM;
        own = true;
    } else if (ws_bytes < p.bytes) {
        return RS_ENOMEM;
    }
    cudaMemsetAsync(w, 0, p.bytes, cs);
    BernArgs a;
    a.N = N; a.seed = seed; a.Db = p.Db;
    a.chunk0 = p.chunk0; a.nchunks = p.nchunks;
    a.log1m_rho = p.lr;
    a.status = (u64 *)(w + p.o_status);
    a.ticket = (u32 *)(w + p.o_ticket);
    a.out = out; a.capacity = capacity; a.count_dev = count_dev;
    a.rk = round_keys(seed);
    a.gV = gV;
    Span sp(2, cs);
    {
        const u64 rmax = (N >> p.Db) + ((N & ((1ull << p.Db) - 1)) != 0);   // largest chunk range
        const int cls = rmax <= (1ull << 16) ? 0 : rmax <= (1ull << 24) ? 1 : rmax <= (1ull << 32) ? 2 : 3;
        const bool d = rho < BF64_RHO;
        void (*const plain[4])(BernArgs) = {k_bernoulli, d ? k_bernoulli32d : k_bernoulli32,
                                            d ? k_bernoulli64d : k_bernoulli64, k_bernoulli64w};
        void (*const graph[4])(BernArgs) = {k_bernoulli_g, d ? k_bernoulli32d_g : k_bernoulli32_g,
                                            d ? k_bernoulli64d_g : k_bernoulli64_g, k_bernoulli64w_g};
        void (*bk)(BernArgs) = gV ? graph[cls] : plain[cls];
        const int nt = cls == 0 ? 32 * BNW16 : cls == 3 ? 32 : 32 * RS_B64W;
        int per = 0, dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(bk, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bk, nt, 0) != cudaSuccess || per < 1) per = 1;
        const u64 need = (p.nchunks + nt / 32 - 1) / (nt / 32) + 1, g = (u64)sms * per;   // + the scanner
        bk<<<(unsigned)(need < g ? need : g), nt, 0, cs>>>(a);
    }
    sp.end();
    ++t_launches;
    st = cuda_ok();
    if (own) cudaFreeAsync(w, cs);
    return st;
}

// ---------------------------------------------------------------------------
// NEXT-4: Algorithm B + repair, composed from the
// Bernoulli kernel, the WOR sampler (for the positions to remove) and the
// compaction kernel (rs_algb.cuh).
// ---------------------------------------------------------------------------
double algb_rho(u64 N, u64 n, double slack)          // rho' (R14)
{
    const double rho = ((double)n + slack * sqrt((double)n)) / (double)N;
    return rho > 1.0 ? 1.0 : rho;
}

// workspace: the Bernoulli pass (capacity + count) and the removal positions
// (at most capacity - n)
size_t algb_ws_bytes(u64 N, u64 n, double slack, u64 *cap_out)
{
    const double rho = algb_rho(N, n, slack);
    const u64 cap = rs_bernoulli_capacity(N, rho);
    if (cap_out) *cap_out = cap;
    BernPlan bp;
    const size_t bb = plan_bern(N, rho, 1, 0, bp) == RS_OK ? bp.bytes : 0;
    return align256((cap + 4) * 8) + align256((cap > n ? cap - n : 1) * 8) + align256(bb);
}

rs_status algb_call(u64 N, u64 n, u64 seed, double slack, u32 max_attempts, u64 *out, u32 *attempts,
                    void *ws, size_t ws_bytes, void *stream)
{
    if (attempts) *attempts = 0;
    if (n > N || !(slack >= 0.0 && slack < 1e300) || N >= (1ull << 63)) return RS_EINVAL;
    if (!have_device()) return RS_ECUDA;
    if (n == 0) return RS_OK;
    const double rho = algb_rho(N, n, slack);
    u64 cap = 0;
    const size_t need = algb_ws_bytes(N, n, slack, &cap);
    const cudaStream_t cs = S(stream);
    unsigned char *w = (unsigned char *)ws;
    const bool own = w == nullptr;
    if (own) {
        if (cudaMallocAsync((void **)&w, need, cs) != cudaSuccess) return RS_ENOMEM;
    } else if (ws_bytes < need) {
        return RS_ENOMEM;
    }
    u64 *tmp = (u64 *)w;
    u64 *cnt_dev = tmp + cap + 1;
    u64 *rem = (u64 *)(w + align256((cap + 4) * 8));
    unsigned char *bws = w + align256((cap + 4) * 8) + align256((cap > n ? cap - n : 1) * 8);
    const size_t bws_bytes = need - (size_t)(bws - w);
    rs_status st = RS_EATTEMPTS;
    for (u32 a = 0; a < max_attempts; ++a) {
        const u64 sa = seed + 0x9E3779B97F4A7C15ull * (u64)a;
        st = bern_call(N, rho, sa, 1, 0, tmp, cap, cnt_dev, bws_bytes ? bws : nullptr, bws_bytes, stream);
        if (st != RS_OK) break;
        u64 np = 0;                                        // n' to the host
        if (cudaMemcpyAsync(&np, cnt_dev, 8, cudaMemcpyDeviceToHost, cs) != cudaSuccess ||
            cudaStreamSynchronize(cs) != cudaSuccess) { st = RS_ECUDA; break; }
        if (attempts) *attempts = a + 1;
        if (np > cap) { st = RS_ECAPACITY; break; }
        if (np < n) { st = RS_EATTEMPTS; continue; }     // restart
        const u64 r = np - n;
        if (r == 0) {
            st = cudaMemcpyAsync(out, tmp, n * 8, cudaMemcpyDeviceToDevice, cs) == cudaSuccess ? RS_OK : RS_ECUDA;
            break;
        }
        st = tree_call(RS_MODE_WOR, np, r, sa, 1, 0, rem, nullptr, 0, stream);   // positions to remove
        if (st == RS_OK) {
            Span sp(3, cs);
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const u64 tiles = (np + AB_TILE - 1) / AB_TILE, g = (u64)sms * 8;
            k_algb_compact<<<(unsigned)(tiles < g ? tiles : g), AB_THREADS, 0, cs>>>(tmp, np, rem, r, out);
            sp.end();
            ++t_launches;
            st = cuda_ok();
        }
        break;
    }
    if (own) cudaFreeAsync(w, cs);
    return st;
}

// Staging for the host-buffer calls, cached per device across calls (a
// fresh cudaMallocAsync of ~2 GiB per call cost ~250 ms of page mapping,
// more than the copies of a 2^28-value sample).  One call at a time per
// device holds it; rs_release_cache() frees it.
struct HostStage {
    std::mutex mu;
    u64 *buf[2] = {nullptr, nullptr};
    size_t buf_bytes = 0;
    unsigned char *ws = nullptr;
    size_t ws_bytes = 0;
    cudaStream_t cs = nullptr;
    cudaEvent_t gen_done[2]{}, copy_done[2]{};
    void release()
    {
        if (buf[0]) cudaFree(buf[0]);
        if (buf[1]) cudaFree(buf[1]);
        if (ws) cudaFree(ws);
        buf[0] = buf[1] = nullptr; ws = nullptr; buf_bytes = ws_bytes = 0;
    }
};
constexpr int RS_MAX_DEV = 64;
HostStage g_stage[RS_MAX_DEV];

__global__ void k_deviates(int kind, u64 k, u64 L, u64 R, u64 seed, u64 id0, u64 count, u64 *out)
{
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x)
        out[i] = kind ? binom(k, L, R, seed, id0 + i) : hgd(k, L, R, seed, id0 + i);
}

// The lane-group deviates (hgd_tpg / binom_grp): G lanes per deviate.
template <int G>
__global__ void k_deviates_grp(int kind, u64 k, u64 L, u64 R, u64 seed, u64 id0, u64 count, u64 *out)
{
    const u64 ngrp = (u64)gridDim.x * blockDim.x / G;
    for (u64 i = (blockIdx.x * (u64)blockDim.x + threadIdx.x) / G; i < count; i += ngrp) {
        const u64 x = G == 32 ? (kind ? binom_tp(k, L, R, seed, id0 + i) : hgd_tp(k, L, R, seed, id0 + i))
                              : (kind ? binom_grp<G>(k, L, R, seed, id0 + i) : hgd_tpg<G>(k, L, R, seed, id0 + i));
        if ((threadIdx.x & (G - 1)) == 0) out[i] = x;
    }
}

}  // namespace

// ===========================================================================
// C ABI.
// ===========================================================================
extern "C" {

rs_status rs_sample_wor(uint64_t N, uint64_t n, uint64_t seed, uint64_t *out, void *stream)
{
    return ret(tree_call(RS_MODE_WOR, N, n, seed, 1, 0, out, nullptr, 0, stream));
}

rs_status rs_sample_wr(uint64_t N, uint64_t n, uint64_t seed, uint64_t *out, void *stream)
{
    return ret(tree_call(RS_MODE_WR, N, n, seed, 1, 0, out, nullptr, 0, stream));
}

rs_status rs_bernoulli(uint64_t N, double rho, uint64_t seed, uint64_t *out, uint64_t capacity,
                       uint64_t *count_dev, void *stream)
{
    return ret(bern_call(N, rho, seed, 1, 0, out, capacity, count_dev, nullptr, 0, stream));
}

uint64_t rs_bernoulli_capacity(uint64_t N, double rho)
{
    if (!(rho > 0.0)) return 0;
    const double mu = (double)N * rho;
    const double c = ceil(mu + 10.0 * sqrt(mu * (1.0 - rho))) + 64.0;
    return c >= (double)N ? N : (uint64_t)c;
}

rs_status rs_shard_info(uint64_t N, uint64_t n, uint64_t seed, int mode, int world, int rank,
                        uint64_t *local_count, uint64_t *global_offset)
{
    if (mode != RS_MODE_WOR && mode != RS_MODE_WR) return ret(RS_EINVAL);
    TreePlan p;
    const rs_status st = plan_tree(mode, N, n, seed, world, rank, p);
    if (st != RS_OK) return ret(st);
    if (local_count) *local_count = p.local_count;
    if (global_offset) *global_offset = p.global_offset;
    return ret(RS_OK);
}

rs_status rs_sample_wor_shard(uint64_t N, uint64_t n, uint64_t seed, int world, int rank,
                              uint64_t *out_local, void *stream)
{
    return ret(tree_call(RS_MODE_WOR, N, n, seed, world, rank, out_local, nullptr, 0, stream));
}

rs_status rs_sample_wr_shard(uint64_t N, uint64_t n, uint64_t seed, int world, int rank,
                             uint64_t *out_local, void *stream)
{
    return ret(tree_call(RS_MODE_WR, N, n, seed, world, rank, out_local, nullptr, 0, stream));
}

rs_status rs_bernoulli_shard(uint64_t N, double rho, uint64_t seed, int world, int rank,
                             uint64_t *out_local, uint64_t capacity, uint64_t *count_dev,
                             void *stream)
{
    return ret(bern_call(N, rho, seed, world, rank, out_local, capacity, count_dev, nullptr, 0, stream));
}

rs_status rs_workspace_bytes(int mode, uint64_t N, uint64_t n, double rho, int world,
                             size_t *bytes)
{
    if (!bytes) return ret(RS_EINVAL);
    size_t best = 0;
    for (int rank = 0; rank < (world > 0 ? world : 1); ++rank) {
        if (mode == RS_MODE_BERNOULLI) {
            BernPlan p;
            const rs_status st = plan_bern(N, rho, world, rank, p);
            if (st != RS_OK) return ret(st);
            if (p.bytes > best) best = p.bytes;
        } else {
            TreePlan p;
            const rs_status st = plan_tree(mode, N, n, 0, world, rank, p);
            if (st != RS_OK) return ret(st);
            if (p.bytes > best) best = p.bytes;
        }
    }
    *bytes = best;
    return ret(RS_OK);
}

rs_status rs_sample_wor_ws(uint64_t N, uint64_t n, uint64_t seed, int world, int rank,
                           uint64_t *out_local, void *ws, size_t ws_bytes, void *stream)
{
    if (!ws) return ret(RS_EINVAL);
    return ret(tree_call(RS_MODE_WOR, N, n, seed, world, rank, out_local, ws, ws_bytes, stream));
}

rs_status rs_sample_wr_ws(uint64_t N, uint64_t n, uint64_t seed, int world, int rank,
                          uint64_t *out_local, void *ws, size_t ws_bytes, void *stream)
{
    if (!ws) return ret(RS_EINVAL);
    return ret(tree_call(RS_MODE_WR, N, n, seed, world, rank, out_local, ws, ws_bytes, stream));
}

rs_status rs_bernoulli_ws(uint64_t N, double rho, uint64_t seed, int world, int rank,
                          uint64_t *out_local, uint64_t capacity, uint64_t *count_dev,
                          void *ws, size_t ws_bytes, void *stream)
{
    if (!ws) return ret(RS_EINVAL);
    return ret(bern_call(N, rho, seed, world, rank, out_local, capacity, count_dev, ws, ws_bytes,
                         stream));
}

// NEXT-3: Erdos-Renyi graphs over the V(V-1)/2 possible edges.
static bool edge_count(uint64_t V, uint64_t *N)
{
    if (V < 2 || V > 0xffffffffull) return false;
    *N = (V & 1) ? V * ((V - 1) >> 1) : (V >> 1) * (V - 1);
    return true;
}

rs_status rs_gnm(uint64_t V, uint64_t m, uint64_t seed, uint64_t *edges, void *ws, size_t ws_bytes,
                 void *stream)
{
    u64 N;
    if (!edge_count(V, &N)) return ret(RS_EINVAL);
    if (!have_device()) return ret(RS_ECUDA);
    TreePlan p;
    rs_status st = plan_tree(RS_MODE_WOR, N, m, seed, 1, 0, p);
    if (st != RS_OK) return ret(st);
    p.gV = V;
    return ret(plan_call(p, edges, ws, ws_bytes, stream));
}

rs_status rs_gnp(uint64_t V, double p, uint64_t seed, uint64_t *edges, uint64_t capacity,
                 uint64_t *count_dev, void *ws, size_t ws_bytes, void *stream)
{
    u64 N;
    if (!edge_count(V, &N)) return ret(RS_EINVAL);
    return ret(bern_call(N, p, seed, 1, 0, edges, capacity, count_dev, ws, ws_bytes, stream, V));
}

rs_status rs_sample_wor_algb(uint64_t N, uint64_t n, uint64_t seed, double slack, uint32_t max_attempts,
                             uint64_t *out, uint32_t *attempts, void *ws, size_t ws_bytes, void *stream)
{
    return ret(algb_call(N, n, seed, slack, max_attempts, out, attempts, ws, ws_bytes, stream));
}

uint64_t rs_algb_workspace_bytes(uint64_t N, uint64_t n, double slack)
{
    if (n > N || n == 0 || !(slack >= 0.0 && slack < 1e300)) return 0;
    return algb_ws_bytes(N, n, slack, nullptr);
}

rs_status rs_uneven_counts(int p, const uint64_t *L, uint64_t n, uint64_t seed, uint64_t *counts)
{
    if (p < 1 || !L || !counts) return ret(RS_EINVAL);
    // prefix sums of L (subtree sums are differences)
    std::vector<u64> pre((size_t)p + 1, 0);
    for (int i = 0; i < p; ++i) {
        if (L[i] >= (1ull << 63) - pre[i]) return ret(RS_EINVAL);
        pre[i + 1] = pre[i] + L[i];
    }
    if (n > pre[p]) return ret(RS_EINVAL);
    int J = 0;
    while ((1ull << J) < (u64)p) ++J;
    // top-down, level by level: cur[a] = samples of the level-j subtree a
    std::vector<u64> cur(1, n), nxt;
    for (int j = J; j > 0; --j) {
        nxt.assign(cur.size() * 2, 0);
        for (size_t a = 0; a < cur.size(); ++a) {
            const u64 lo = (u64)a << j, mid = lo + (1ull << (j - 1));
            if (lo >= (u64)p) continue;
            if (mid >= (u64)p) { nxt[2 * a] = cur[a]; continue; }     // no right half
            const u64 hi = (lo + (1ull << j)) < (u64)p ? lo + (1ull << j) : (u64)p;
            const u64 Ll = pre[mid] - pre[lo], Lt = pre[hi] - pre[lo];
            const u64 id = (1ull << 62) | ((1ull << (J - j)) + a);
            const u64 x = cur[a] ? hgd(cur[a], Ll, Lt, seed, id) : 0;
            nxt[2 * a] = x;
            nxt[2 * a + 1] = cur[a] - x;
        }
        cur.swap(nxt);
    }
    for (int i = 0; i < p; ++i) counts[i] = cur[(size_t)i];
    return ret(RS_OK);
}

uint64_t rs_uneven_seed(uint64_t seed, uint64_t pe)
{
    u64 z = seed + 0x9E3779B97F4A7C15ull * (pe + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

rs_status rs_node_info(int mode, uint64_t N, uint64_t n, uint64_t seed, int depth, uint64_t index,
                       uint64_t *count, uint64_t *global_offset)
{
    if (mode != RS_MODE_WOR && mode != RS_MODE_WR) return ret(RS_EINVAL);
    TreePlan p;
    const rs_status st = plan_node(mode, N, n, seed, depth, index, p);
    if (st != RS_OK) return ret(st);
    if (count) *count = p.local_count;
    if (global_offset) *global_offset = p.global_offset;
    return ret(RS_OK);
}

rs_status rs_sample_node(int mode, uint64_t N, uint64_t n, uint64_t seed, int depth,
                         uint64_t index, uint64_t *out, void *stream)
{
    if (mode != RS_MODE_WOR && mode != RS_MODE_WR) return ret(RS_EINVAL);
    TreePlan p;
    const rs_status st = plan_node(mode, N, n, seed, depth, index, p);
    if (st != RS_OK) return ret(st);
    return ret(plan_call(p, out, nullptr, 0, stream));
}

static rs_status shard_host(int mode, uint64_t N, uint64_t n, uint64_t seed, int world,
                            int rank, uint64_t *out_host, uint64_t host_elems, void *stream);

rs_status rs_sample_shard_host(int mode, uint64_t N, uint64_t n, uint64_t seed, int world,
                               int rank, uint64_t *out_host, void *stream)
{
    return ret(shard_host(mode, N, n, seed, world, rank, out_host, ~0ull, stream));
}

rs_status rs_sample_shard_host_stream(int mode, uint64_t N, uint64_t n, uint64_t seed, int world,
                                      int rank, uint64_t *out_host, uint64_t host_elems, void *stream)
{
    return ret(shard_host(mode, N, n, seed, world, rank, out_host, host_elems, stream));
}

rs_status rs_sample_checked(int mode, uint64_t N, uint64_t n, uint64_t seed, int world, int rank,
                            uint64_t *out_local, void *stream)
{
    if (!have_device()) return ret(RS_ECUDA);
    if (mode != RS_MODE_WOR && mode != RS_MODE_WR) return ret(RS_EINVAL);
    TreePlan p;
    rs_status st = plan_tree(mode, N, n, seed, world, rank, p);
    if (st != RS_OK) return ret(st);
    if (p.local_count == 0) return ret(RS_OK);
    if (!out_local) return ret(RS_EINVAL);
    const cudaStream_t cs = S(stream);
    unsigned char *w = nullptr;
    if (cudaMallocAsync((void **)&w, p.bytes, cs) != cudaSuccess) return ret(RS_ENOMEM);
    st = run_tree(p, out_local, w, cs);
    u32 flags = 0;
    if (st == RS_OK && cudaMemcpyAsync(&flags, w + p.o_spill, 4, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
        st = RS_ECUDA;
    cudaFreeAsync(w, cs);
    if (cudaStreamSynchronize(cs) != cudaSuccess) st = RS_ECUDA;
    if (st == RS_OK && flags) st = RS_ECAPACITY;
    return ret(st);
}

static rs_status shard_host(int mode, uint64_t N, uint64_t n, uint64_t seed, int world,
                            int rank, uint64_t *out_host, uint64_t host_elems, void *stream)
{
    if (!have_device()) return (RS_ECUDA);
    if (mode != RS_MODE_WOR && mode != RS_MODE_WR) return (RS_EINVAL);
    TreePlan sp;
    rs_status st = plan_tree(mode, N, n, seed, world, rank, sp);
    if (st != RS_OK) return (st);
    if (sp.local_count == 0) return (RS_OK);
    if (!out_host) return (RS_EINVAL);
    // batches: the shard's descendants at depth s + b, each <= 2^27 values
    int b = 0;
    while (b < sp.D - sp.s && (sp.local_count >> b) > (1ull << 27)) ++b;
    if (b < sp.D - sp.s && b < 20 && sp.local_count > (1ull << 26)) ++b;   // >= 2 batches to overlap
    const u64 nb = 1ull << b;
    std::vector<TreePlan> plans(nb);
    u64 maxc = 0;
    size_t maxws = 0;
    for (u64 i = 0; i < nb; ++i) {
        st = plan_node(mode, N, n, seed, sp.s + b, (sp.idx << b) + i, plans[i]);
        if (st != RS_OK) return (st);
        if (plans[i].local_count > maxc) maxc = plans[i].local_count;
        if (plans[i].bytes > maxws) maxws = plans[i].bytes;
    }
    // host_elems < count: stream the batches through a two-slot host ring
    // (batch i -> out_host + (i & 1) * maxc; for benchmarks of the D2H path
    // with bounded host memory).  Needs host_elems >= 2 * maxc.
    const bool ring = host_elems < sp.local_count;
    if (ring && host_elems < 2 * maxc) return (RS_EINVAL);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= RS_MAX_DEV) return (RS_ECUDA);
    HostStage &H = g_stage[dev];
    std::lock_guard<std::mutex> lock(H.mu);
    if (!H.cs) {
        if (cudaStreamCreateWithFlags(&H.cs, cudaStreamNonBlocking) != cudaSuccess) { H.cs = nullptr; return (RS_ECUDA); }
        for (int i = 0; i < 2; ++i) {
            cudaEventCreateWithFlags(&H.gen_done[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&H.copy_done[i], cudaEventDisableTiming);
        }
    }
    const size_t need_buf = align256(maxc * 8 + 8), need_ws = align256(maxws ? maxws : 1);
    if (H.buf_bytes < need_buf) {
        if (H.buf[0]) cudaFree(H.buf[0]);
        if (H.buf[1]) cudaFree(H.buf[1]);
        H.buf[0] = H.buf[1] = nullptr; H.buf_bytes = 0;
        if (cudaMalloc((void **)&H.buf[0], need_buf) != cudaSuccess ||
            cudaMalloc((void **)&H.buf[1], need_buf) != cudaSuccess) { H.release(); cudaGetLastError(); return (RS_ENOMEM); }
        H.buf_bytes = need_buf;
    }
    if (H.ws_bytes < need_ws) {
        if (H.ws) cudaFree(H.ws);
        H.ws = nullptr; H.ws_bytes = 0;
        if (cudaMalloc((void **)&H.ws, need_ws) != cudaSuccess) { H.release(); cudaGetLastError(); return (RS_ENOMEM); }
        H.ws_bytes = need_ws;
    }
    const cudaStream_t gs = S(stream), cs = H.cs;
    cudaEventRecord(H.copy_done[0], cs);          // the staging buffers are free once earlier copies end
    cudaEventRecord(H.copy_done[1], cs);
    cudaStreamWaitEvent(gs, H.copy_done[0], 0);
    const u64 base_off = sp.global_offset;
    for (u64 i = 0; i < nb && st == RS_OK; ++i) {
        const int j = (int)(i & 1);
        if (i >= 2) cudaStreamWaitEvent(gs, H.copy_done[j], 0);     // buffer j is free again
        st = run_tree(plans[i], H.buf[j], H.ws, gs, i == 0);
        cudaEventRecord(H.gen_done[j], gs);
        cudaStreamWaitEvent(cs, H.gen_done[j], 0);
        if (plans[i].local_count &&
            cudaMemcpyAsync(out_host + (ring ? (u64)j * maxc : plans[i].global_offset - base_off), H.buf[j],
                            plans[i].local_count * 8, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
            st = RS_ECUDA;
        cudaEventRecord(H.copy_done[j], cs);
    }
    cudaStreamWaitEvent(gs, H.copy_done[0], 0);
    cudaStreamWaitEvent(gs, H.copy_done[1], 0);
    u32 flags = 0;     // the batches' status word (every plan shares o_spill's layout)
    if (st == RS_OK && cudaMemcpyAsync(&flags, H.ws + plans[0].o_spill, 4, cudaMemcpyDeviceToHost, gs) != cudaSuccess)
        st = RS_ECUDA;
    if (cudaStreamSynchronize(gs) != cudaSuccess || cudaStreamSynchronize(cs) != cudaSuccess) st = RS_ECUDA;
    if (st == RS_OK && flags) st = RS_ECAPACITY;
    return (st);
}

rs_status rs_deviates(int kind, uint64_t k, uint64_t L, uint64_t R, uint64_t seed, uint64_t id0,
                      uint64_t count, uint64_t *out, void *stream)
{
    if (kind < 0 || kind > 5) return ret(RS_EINVAL);
    if (L > R || ((kind & 1) == 0 && k > R) || R >= (1ull << 63)) return ret(RS_EINVAL);
    if (!have_device()) return ret(RS_ECUDA);
    if (count == 0) return ret(RS_OK);
    const u64 g = (count + 127) / 128;
    const unsigned gg = (unsigned)(g < 4096 ? g : 4096);
    if (kind <= 1) k_deviates<<<gg, 128, 0, S(stream)>>>(kind, k, L, R, seed, id0, count, out);
    else if (kind <= 3) k_deviates_grp<32><<<gg, 128, 0, S(stream)>>>(kind & 1, k, L, R, seed, id0, count, out);
    else k_deviates_grp<8><<<gg, 128, 0, S(stream)>>>(kind & 1, k, L, R, seed, id0, count, out);
    ++t_launches;
    return ret(cuda_ok());
}

rs_status rs_release_cache(void)
{
    for (int d = 0; d < RS_MAX_DEV; ++d) {
        std::lock_guard<std::mutex> lock(g_stage[d].mu);
        if (g_stage[d].buf_bytes || g_stage[d].ws_bytes) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(d);
            g_stage[d].release();
            cudaSetDevice(cur);
        }
    }
    return ret(RS_OK);
}

rs_status rs_sample_wor_host(uint64_t N, uint64_t n, uint64_t seed, uint64_t *out_host,
                             void *stream)
{
    return rs_sample_shard_host(RS_MODE_WOR, N, n, seed, 1, 0, out_host, stream);
}

rs_status rs_digest(const uint64_t *v, uint64_t count, uint64_t base_index, uint64_t *result_dev,
                    void *stream)
{
    if (!have_device()) return ret(RS_ECUDA);
    if (count == 0) return ret(RS_OK);
    const u64 blocks = (count + 255) / 256;
    k_digest<<<(unsigned)(blocks < 4736 ? blocks : 4736), 256, 0, S(stream)>>>(v, count, base_index,
                                                                              result_dev);
    ++t_launches;
    return ret(cuda_ok());
}

rs_status rs_validate(const uint64_t *v, uint64_t count, uint64_t N, int strict, uint64_t *bad_dev,
                      void *stream)
{
    if (!have_device()) return ret(RS_ECUDA);
    if (count == 0) return ret(RS_OK);
    const u64 blocks = (count + 255) / 256;
    k_validate<<<(unsigned)(blocks < 4736 ? blocks : 4736), 256, 0, S(stream)>>>(v, count, N, strict,
                                                                                bad_dev);
    ++t_launches;
    return ret(cuda_ok());
}

rs_status rs_plan(int mode, uint64_t N, uint64_t n, double rho, int *depth, int *complement,
                  uint64_t *core_count)
{
    if (mode == RS_MODE_BERNOULLI) {
        BernPlan p;
        const rs_status st = plan_bern(N, rho, 1, 0, p);
        if (st != RS_OK) return ret(st);
        if (depth) *depth = p.Db;
        if (complement) *complement = 0;
        if (core_count) *core_count = 0;
        return ret(RS_OK);
    }
    TreePlan p;
    const rs_status st = plan_tree(mode, N, n, 0, 1, 0, p);
    if (st != RS_OK) return ret(st);
    if (depth) *depth = p.D;
    if (complement) *complement = p.comp ? 1 : 0;
    if (core_count) *core_count = p.m;
    return ret(RS_OK);
}

rs_status rs_device_errors(int clear, unsigned *flags)
{
    if (!have_device()) return ret(RS_ECUDA);
    if (cudaDeviceSynchronize() != cudaSuccess) return ret(RS_ECUDA);
    unsigned f = 0;
    if (cudaMemcpyFromSymbol(&f, g_rs_errors, sizeof f) != cudaSuccess) return ret(RS_ECUDA);
    if (flags) *flags = f;
    if (clear) {
        const unsigned z = 0;
        if (cudaMemcpyToSymbol(g_rs_errors, &z, sizeof z) != cudaSuccess) return ret(RS_ECUDA);
    }
    return ret(RS_OK);
}

rs_status rs_set_option(int option, int value)
{
    if (option == RS_OPT_LEAF_PATH && value >= 0 && value <= 3) {
        g_leaf_path = value;
        return ret(RS_OK);
    }
    if (option == RS_OPT_TOPUP_MAX && value >= 0 && value <= 32) {
        g_topup_max = value;
        return ret(RS_OK);
    }
    if (option == RS_OPT_SPLIT_COOP && (value == 0 || value == 1)) {
        g_split_coop = value;
        return ret(RS_OK);
    }
    if (option == RS_OPT_FUSED && (value == 0 || value == 1)) {
        g_fused = value;
        return ret(RS_OK);
    }
    if (option == RS_OPT_WARP_CAP && value >= 0 && value <= WL_CAP) {
        g_warp_cap = value;
        return ret(RS_OK);
    }
    if (option == RS_OPT_LEAF_CAP && value >= 0 && value <= LEAF_CAP) {
        g_leaf_cap = value;
        return ret(RS_OK);
    }
    return ret(RS_EINVAL);
}

uint64_t rs_launch_count(int reset)
{
    const uint64_t v = t_launches;
    if (reset) t_launches = 0;
    return v;
}

rs_status rs_timing_enable(int on)
{
    std::lock_guard<std::mutex> g(g_tmu);
    g_timing = on != 0;
    return ret(RS_OK);
}

rs_status rs_timing_read(int reset, double *ms, uint64_t *launches)
{
    std::lock_guard<std::mutex> g(g_tmu);
    for (const TimedSpan &t : g_spans) {
        float f = 0.f;
        if (cudaEventSynchronize(t.b) != cudaSuccess) return ret(RS_ECUDA);
        if (cudaEventElapsedTime(&f, t.a, t.b) != cudaSuccess) return ret(RS_ECUDA);
        g_ms[t.cls] += f;
        g_cnt[t.cls] += 1;
        g_free_events.push_back(t.a);
        g_free_events.push_back(t.b);
    }
    g_spans.clear();
    for (int i = 0; i < 4; ++i) {
        if (ms) ms[i] = g_ms[i];
        if (launches) launches[i] = g_cnt[i];
        if (reset) { g_ms[i] = 0; g_cnt[i] = 0; }
    }
    return ret(RS_OK);
}

const char *rs_status_string(rs_status s)
{
    switch (s) {
    case RS_OK: return "ok";
    case RS_EINVAL: return "invalid argument";
    case RS_ECUDA: return "CUDA error or no device";
    case RS_ENOMEM: return "workspace allocation failed or too small";
    case RS_ECAPACITY: return "capacity exceeded";
    case RS_EATTEMPTS: return "restart budget exhausted (Algorithm B)";
    }
    return "unknown status";
}

rs_status rs_last_status(void) { return t_last; }

const char *rs_version(void) { return "rs 0.1 (CANON v1, sm_100a)"; }

#ifdef RS_EXP_CLOCK
// dev: per-phase cycle totals of the warp leaf kernel (RS_EXP_CLOCK builds)
int rs_debug_prof(unsigned long long *out8, int reset)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out8, g_rs_prof, 8 * sizeof(unsigned long long));
    if (reset) { unsigned long long z[8] = {0}; cudaMemcpyToSymbol(g_rs_prof, z, sizeof z); }
    return 0;
}
#endif

}  // extern "C"
