/*
 * rs.h -- C ABI of librs.so, the B200 (sm_100a) divide-and-conquer random
 * sampler of Sanders, Lamm, Huebschle-Schneider, Schrade and Dachsbacher,
 * "Efficient Random Sampling -- Parallel, Vectorized, Cache-Efficient, and
 * Online" (arXiv 1610.05141).  P:n = /root/reference/PAPER.md line n.
 *
 * Conventions (all entry points):
 *  - Values are 1-based uint64, little-endian, ascending; "sorted sample of
 *    n numbers out of the range 1..N".
 *  - Pointers named *_dev / out are DEVICE pointers owned by the caller
 *    (e.g. allocated by torch); the library owns only its transient
 *    workspace (stream-ordered cudaMallocAsync, or the caller's via *_ws).
 *  - Calls are asynchronous on `stream` (cudaStream_t passed as void*;
 *    NULL = legacy default stream).  Argument errors are detected on the
 *    host before any launch and nothing is written.
 *  - Results are a pure function of (N, n or rho, seed): identical for any
 *    world size and bit-exact with the CANON v1 definition.
 *  - No CPU fallback: without a CUDA device every call returns RS_ECUDA.
 *  - Thread-safe and reentrant; no global RNG state (the seed is an
 *    argument).  rs_last_status() is thread-local.
 *  - Device-side capacity overflows (a leaf needing more than the
 *    on-chip capacity -- probability < 1e-100 at every supported shape,
 *    DESIGN.md 5) leave that leaf unwritten and raise bit 0 of the call's
 *    status word (in its workspace) and of a sticky device flag
 *    (rs_device_errors()).  The synchronous calls (rs_sample_checked, the
 *    host-buffer calls) read the status word and return RS_ECAPACITY.
 */
#ifndef RS_H
#define RS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RS_OK = 0,
    RS_EINVAL = 1,     /* invalid argument (n > N, rho not in [0,1], ...) */
    RS_ECUDA = 2,      /* CUDA runtime error / no device                  */
    RS_ENOMEM = 3,     /* workspace allocation failed / too small         */
    RS_ECAPACITY = 4,  /* output capacity exceeded (Bernoulli) / a leaf
                          exceeded the on-chip capacity (checked calls)   */
    RS_EATTEMPTS = 5   /* Algorithm B: restart budget exhausted           */
} rs_status;

enum { RS_MODE_WOR = 0, RS_MODE_WR = 1, RS_MODE_BERNOULLI = 2 };

/* ---- sampling without replacement: Algorithm R / P ----------
 * Writes the n distinct values of a uniform random n-subset of 1..N to
 * out[0..n), ascending.  out: device, capacity >= n.  n > N -> RS_EINVAL;
 * n == 0 -> no-op; N >= 2^63 -> RS_EINVAL.  If 2n > N the N-n values NOT in
 * the sample are generated and the complement is emitted. */
rs_status rs_sample_wor(uint64_t N, uint64_t n, uint64_t seed, uint64_t *out, void *stream);

/* ---- sampling with replacement: binomial splits ------------
 * n values of 1..N with repeats (iid uniform), ascending.  N == 0 && n > 0
 * -> RS_EINVAL. */
rs_status rs_sample_wr(uint64_t N, uint64_t n, uint64_t seed, uint64_t *out, void *stream);

/* ---- Bernoulli sampling by geometric skips -------
 * Each of 1..N independently with probability rho, ascending.  Writes
 * min(count, capacity) values to out and the true count to *count_dev
 * (device, stream-ordered).  The count is random, so overflow is known only
 * after the stream completes: the caller checks *count_dev <= capacity; a
 * re-call with a larger buffer returns the identical sample.  rho must be in
 * [0,1] (NaN -> RS_EINVAL). */
rs_status rs_bernoulli(uint64_t N, double rho, uint64_t seed, uint64_t *out,
                       uint64_t capacity, uint64_t *count_dev, void *stream);

/* A capacity exceeded with probability < 1e-23 (10-sigma + 64), <= N. */
uint64_t rs_bernoulli_capacity(uint64_t N, double rho);

/* ---- sharding: Algorithm P over p = world GPUs -------------
 * Rank g of world = 2^s (s <= 3) owns the dyadic range
 * [floor(g N / world), floor((g+1) N / world)).  rs_shard_info replays the
 * s hypergeometric (binomial for WR) splits on the root path on the host
 * -- "each PE generates <= ceil(log p) hypergeometric random deviates"
 * -- giving the rank's output count and its offset in the global
 * output.  No communication.  mode: RS_MODE_WOR or RS_MODE_WR. */
rs_status rs_shard_info(uint64_t N, uint64_t n, uint64_t seed, int mode, int world,
                        int rank, uint64_t *local_count, uint64_t *global_offset);

/* The rank's slice of rs_sample_wor / rs_sample_wr output, written to
 * out_local[0..local_count).  Concatenating all ranks' slices in rank
 * order gives exactly the world = 1 output. */
rs_status rs_sample_wor_shard(uint64_t N, uint64_t n, uint64_t seed, int world, int rank,
                              uint64_t *out_local, void *stream);
rs_status rs_sample_wr_shard(uint64_t N, uint64_t n, uint64_t seed, int world, int rank,
                             uint64_t *out_local, void *stream);

/* The rank's slice of rs_bernoulli: values in its dyadic range, local
 * count to *count_dev.  Global offsets need an exclusive scan of the
 * ranks' counts (the one collective; done by the Python layer over NCCL). */
rs_status rs_bernoulli_shard(uint64_t N, double rho, uint64_t seed, int world, int rank,
                             uint64_t *out_local, uint64_t capacity, uint64_t *count_dev,
                             void *stream);

/* ---- any node of the split tree: range-addressable sampling (NEXT-1) -----
 * The online / "sorted output in batches" use of Algorithm R:
 * node (depth, index), 0 <= depth <= D (the tree depth, rs_plan), index <
 * 2^depth, covers the dyadic value range [floor(index N / 2^depth),
 * floor((index+1) N / 2^depth)) (+1 for the 1-based values).
 * rs_node_info: the node's output count and its offset in the full output,
 * by host path replay of the depth splits above it (no device; same
 * arithmetic as the kernels).  rs_sample_node: the node's slice of
 * rs_sample_wor (mode RS_MODE_WOR, complement rule included) or rs_sample_wr
 * (RS_MODE_WR) into out[0..count) (device).  The slices of the nodes of any
 * partition of the leaf range, in order, concatenate to the full output.
 * depth > D or index out of range -> RS_EINVAL. */
rs_status rs_node_info(int mode, uint64_t N, uint64_t n, uint64_t seed, int depth, uint64_t index,
                       uint64_t *count, uint64_t *global_offset);
rs_status rs_sample_node(int mode, uint64_t N, uint64_t n, uint64_t seed, int depth,
                         uint64_t index, uint64_t *out, void *stream);

/* ---- Erdos-Renyi random graphs (NEXT-3) -----------------------
 * "Generating a random graph in the G(n,m) and G(n,p) model ... is equivalent
 * to sampling from the n(n-1)/2 possible edges": the WOR / Bernoulli sample
 * over edge indices, with the index -> (u, v) decode fused into the leaf
 * stores.  Vertices 0..V-1, 2 <= V < 2^32; edge index e (lexicographic over
 * pairs u < v) is stored as (u << 32) | v, so the output is the edge list in
 * lexicographic order.  rs_gnm: m distinct edges into edges[0..m) (m > V(V-1)/2
 * -> RS_EINVAL).  rs_gnp: each edge independently with probability p;
 * capacity / count_dev as rs_bernoulli (capacity from
 * rs_bernoulli_capacity(V(V-1)/2, p)).  Outputs equal the decoded
 * rs_sample_wor / rs_bernoulli samples over 1..V(V-1)/2 with the same seed.
 * ws: NULL (cudaMallocAsync on the stream) or a device workspace of ws_bytes
 * >= rs_workspace_bytes(RS_MODE_WOR / RS_MODE_BERNOULLI, V(V-1)/2, m, p, 1). */
rs_status rs_gnm(uint64_t V, uint64_t m, uint64_t seed, uint64_t *edges, void *ws, size_t ws_bytes,
                 void *stream);
rs_status rs_gnp(uint64_t V, double p, uint64_t seed, uint64_t *edges, uint64_t capacity,
                 uint64_t *count_dev, void *ws, size_t ws_bytes, void *stream);

/* ---- Algorithm B + repair (NEXT-4, the comparison baseline) -------------
 * The paper's own GPU design B_GPU, composed from the
 * kernels above: a Bernoulli sample with rho' = min(1, (n + slack sqrt(n)) /
 * N) ("rho somewhat larger than n/N"), restarted with seed_a = seed + a *
 * 0x9E3779B97F4A7C15 (a = 1, 2, ...) while its size n' < n ("simply restart"),
 * then repaired by removing the elements at the n' - n positions of the WOR
 * sample rs_sample_wor(n', n' - n, seed_a) ("Algorithm R to generate n'-n
 * samples from the range 0..n'-1"), with a compaction kernel.  out: device,
 * capacity >= n; receives n distinct values of 1..N, ascending -- a uniform
 * n-subset, but NOT the same one as rs_sample_wor.  attempts (host, may be
 * NULL): Bernoulli passes used.  Synchronous: n' goes to the host after every
 * pass (as in the paper).  Workspace: ws (device, caller-owned)
 * of ws_bytes >= rs_algb_workspace_bytes(N, n, slack) -- the Bernoulli buffer
 * of rs_bernoulli_capacity(N, rho') values and the removal positions -- or
 * ws = NULL: cudaMallocAsync / cudaFreeAsync on the stream.  n > N, slack < 0
 * or not finite, N >= 2^63 -> RS_EINVAL; too small ws -> RS_ENOMEM; more
 * than max_attempts passes -> RS_EATTEMPTS. */
rs_status rs_sample_wor_algb(uint64_t N, uint64_t n, uint64_t seed, double slack,
                             uint32_t max_attempts, uint64_t *out, uint32_t *attempts,
                             void *ws, size_t ws_bytes, void *stream);
uint64_t rs_algb_workspace_bytes(uint64_t N, uint64_t n, double slack);   /* 0 if invalid or n == 0 */

/* ---- uneven universe (NEXT-2) ---------------------------------
 * p PEs (GPUs, ranks) own L[0..p) elements ("owner computes"); the n
 * samples of their union are assigned to the PEs by the paper's binomial
 * tree: subtree sums of L bottom-up, then hypergeometric splits of the count
 * top-down, the deviate of the subtree over PEs 2^j a .. keyed by that
 * range (R13).  Host only (no device); every rank computes the
 * same counts from the all-gathered L, so the paper's tree messages become
 * one all-gather of p words.  n > sum L or sum L >= 2^63 -> RS_EINVAL.
 * rs_uneven_seed: the seed of PE i's local sample, rs_sample_wor(L[i],
 * counts[i], rs_uneven_seed(seed, i)) (values are local element indices). */
rs_status rs_uneven_counts(int p, const uint64_t *L, uint64_t n, uint64_t seed, uint64_t *counts);
uint64_t rs_uneven_seed(uint64_t seed, uint64_t pe);

/* ---- caller-provided workspace variants --------------------------------
 * rs_workspace_bytes: bytes of device workspace the *_ws calls need for
 * (mode, N, n or rho, world).  ws must be 256-byte aligned.  Too small ->
 * RS_ENOMEM (nothing launched). */
rs_status rs_workspace_bytes(int mode, uint64_t N, uint64_t n, double rho, int world,
                             size_t *bytes);
rs_status rs_sample_wor_ws(uint64_t N, uint64_t n, uint64_t seed, int world, int rank,
                           uint64_t *out_local, void *ws, size_t ws_bytes, void *stream);
rs_status rs_sample_wr_ws(uint64_t N, uint64_t n, uint64_t seed, int world, int rank,
                          uint64_t *out_local, void *ws, size_t ws_bytes, void *stream);
rs_status rs_bernoulli_ws(uint64_t N, double rho, uint64_t seed, int world, int rank,
                          uint64_t *out_local, uint64_t capacity, uint64_t *count_dev,
                          void *ws, size_t ws_bytes, void *stream);

/* ---- host-buffer end-to-end call ----------------------------------------
 * rs_sample_wor into a HOST buffer out_host[0..n): generates on the device
 * in leaf-range batches and copies each batch device->host (pinned host
 * memory recommended) while the next batch is generated. */
rs_status rs_sample_wor_host(uint64_t N, uint64_t n, uint64_t seed, uint64_t *out_host,
                             void *stream);

/* Host-buffer call for any mode/shard: the rank's slice of rs_sample_wor
 * (mode RS_MODE_WOR) or rs_sample_wr (RS_MODE_WR) into out_host[0..count),
 * count = rs_shard_info's local_count.  Generates the slice node by node
 * (rs_sample_node; batches of <= 2^27 values) into two device staging
 * buffers, copying batch i to the host on an internal stream while batch
 * i+1 is generated on `stream`.  Synchronous (returns after the last copy).
 * out_host should be pinned for full copy bandwidth.  The two staging
 * buffers (<= 1 GiB each), the tree workspace and the copy stream are kept
 * per device across calls (calls on one device are serialised by a lock);
 * rs_release_cache frees them. */
rs_status rs_sample_shard_host(int mode, uint64_t N, uint64_t n, uint64_t seed, int world,
                               int rank, uint64_t *out_host, void *stream);

/* The same with a bounded host buffer of host_elems values: if host_elems <
 * count, batch i is copied to out_host + (i mod 2) * B (B = the largest
 * batch, <= 2^27 values), i.e. the host sees the slice streamed through a
 * two-slot ring (bench.py's end-to-end leg at N > 1: bounded pinned memory
 * per rank).  host_elems < 2 B -> RS_EINVAL; host_elems >= count is
 * rs_sample_shard_host. */
rs_status rs_sample_shard_host_stream(int mode, uint64_t N, uint64_t n, uint64_t seed, int world,
                                      int rank, uint64_t *out_host, uint64_t host_elems,
                                      void *stream);

/* ---- checked device call ---------------------------------------------------
 * rs_sample_wor_shard / rs_sample_wr_shard (mode RS_MODE_WOR / RS_MODE_WR;
 * world = 1, rank = 0 for the whole sample) followed by a synchronisation of
 * `stream` and a read of the call's own status word: RS_ECAPACITY if a leaf
 * could not be completed on chip (that leaf's output span is then
 * unspecified), without touching the process-wide sticky flag's state.
 * out_local: device, capacity >= rs_shard_info's local_count. */
rs_status rs_sample_checked(int mode, uint64_t N, uint64_t n, uint64_t seed, int world, int rank,
                            uint64_t *out_local, void *stream);
rs_status rs_release_cache(void);

/* ---- split deviates (diagnostics / tests) ----------------------------------
 * out[t] = the split tree's deviate for node id id0 + t (the device code the
 * split kernels run): kind 0 = hypergeometric X ~ Hyp(k draws, L of R)
 * (R6), kind 1 = binomial X ~ Bin(k, L/R) (R9);
 * kinds 2/3 (4/5) = the same deviates computed by groups of 32 (8) lanes:
 * hypergeometric with 32 lanes splits the work by density term (hgd_tp),
 * otherwise the lanes evaluate rejection iterations in parallel -- all must
 * be bit-identical to kinds 0/1.
 * out: device, count values.  L > R, (kind 0) k > R, R >= 2^63 -> RS_EINVAL. */
rs_status rs_deviates(int kind, uint64_t k, uint64_t L, uint64_t R, uint64_t seed, uint64_t id0,
                      uint64_t count, uint64_t *out, void *stream);

/* ---- validation helpers (tests / benchmarks; not on the hot path) ------
 * rs_digest: *result_dev += sum_i mix64((base_index + i) ^ mix64(v[i]))
 * (mod 2^64; order-sensitive, shard-composable; caller zeroes result_dev).
 * rs_validate: *bad_dev += number of i with v[i] outside [1, N] or
 * v[i] >= v[i+1] (strict) / v[i] > v[i+1] (non-strict). */
rs_status rs_digest(const uint64_t *v, uint64_t count, uint64_t base_index,
                    uint64_t *result_dev, void *stream);
rs_status rs_validate(const uint64_t *v, uint64_t count, uint64_t N, int strict,
                      uint64_t *bad_dev, void *stream);

/* Planning info: depth D of the split tree (WOR/WR) or D_b (Bernoulli),
 * complement flag and core count m.  Pure host function. */
rs_status rs_plan(int mode, uint64_t N, uint64_t n, double rho, int *depth,
                  int *complement, uint64_t *core_count);

/* Sticky device error flags (bit 0: leaf capacity, bit 1: Bernoulli chunk
 * capacity).  Synchronises the device; clear != 0 resets them. */
rs_status rs_device_errors(int clear, unsigned *flags);

/* Test hook: select the leaf implementation (process-wide).
 * RS_OPT_LEAF_PATH: 0 = automatic (default: warp-per-leaf kernels, bitmap
 * kernels for leaf ranges <= 2^15, CTA kernel for leaves that do not fit);
 * 1 = the CTA-per-leaf kernels for every leaf (so tests cover that path);
 * 2 = as 0; 3 = the ordered linear-probing warp kernels (rs_leaf_lp.cuh:
 * a measured alternative, slower; kept selectable and tested) where every
 * leaf range has >= 2^11 values.
 * RS_OPT_TOPUP_MAX: 0..32, most duplicates the warp kernels for small leaf
 * ranges top up draw by draw before running a full extra round (default 32;
 * tests lower it to cover the fallback).
 * RS_OPT_SPLIT_COOP: 1 (default) = the narrow top of the split tree in one
 * cooperative launch; 0 = a single top CTA then one launch per level.
 * RS_OPT_LEAF_CAP: 0 (default) or 1..2048, the CTA leaf kernel's draw
 * capacity; small values force capacity overflows so that tests can check
 * that they are reported (RS_ECAPACITY from the checked calls).
 * RS_OPT_FUSED: 1 (default) = trees of <= 2^11 leaves (the shard's depth
 * D - s <= 11) on the warp-leaf paths run split and leaves in one launch,
 * each CTA walking the path from the shard root to its 16-leaf subtree
 * (n up to ~2^21; rs_fused.cuh); 0 = the separate split and leaf launches.
 * RS_OPT_WARP_CAP: 0 (default) or 1..1152: the warp-per-leaf kernels hand
 * every leaf of more draws to the CTA kernel's spill pass (tests: covers
 * that path, normally taken by ~1 leaf in 10^4).
 * Results are identical for every setting of LEAF_PATH, TOPUP_MAX,
 * SPLIT_COOP, FUSED and WARP_CAP (LEAF_CAP changes which leaves fail).  Unknown option
 * or value -> RS_EINVAL. */
enum { RS_OPT_LEAF_PATH = 1, RS_OPT_TOPUP_MAX = 2, RS_OPT_LEAF_CAP = 3, RS_OPT_SPLIT_COOP = 4, RS_OPT_FUSED = 5,
       RS_OPT_WARP_CAP = 6 };
rs_status rs_set_option(int option, int value);

/* Number of kernel launches issued by this thread since the last reset. */
uint64_t rs_launch_count(int reset);

/* Device-time instrumentation for benchmarks: while enabled, every call
 * records CUDA events on its launch stream around each kernel class
 * (0 split tree, 1 leaf, 2 Bernoulli, 3 other: Algorithm B's compaction).  rs_timing_read
 * synchronises on the recorded events and returns the accumulated
 * milliseconds and launch counts per class (arrays of 4); reset != 0
 * clears them.  Disabled by default (no events recorded). */
rs_status rs_timing_enable(int on);
rs_status rs_timing_read(int reset, double *ms, uint64_t *launches);

const char *rs_status_string(rs_status s);
rs_status rs_last_status(void);
const char *rs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RS_H */
