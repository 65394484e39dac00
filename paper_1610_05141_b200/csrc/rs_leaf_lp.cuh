// rs_leaf_lp.cuh -- the common-path WOR / WR leaf kernel (rows a5, a6, a8 of
// SURVEY.md section 8(a)): ONE WARP PER LEAF over an ORDERED LINEAR-PROBING
// TABLE in shared memory.  Included by rs_kernels.cu after rs_leaf_warp.cuh.
// P:n = /root/reference/PAPER.md line n.
//
// Same result as leaf_sorted (rs_leaf.cuh): the leaf's first k distinct draws
// (WOR, Algorithm H) or its first k draws with repeats (WR), sorted
// (P:356-374), value lo + x + 1.
//
// The paper's base case is a hash table with a MONOTONE hash, "so that
// sorting the hash table ... is easy".  Here the hash
// is h(x) = x >> (ceil_log2(r) - 11) (2048 home slots for ~1024 draws) and the
// table is kept in sorted order during insertion (ordered linear probing):
// inserting a key c at slot s is `old = atomicMin(T[s], c)`; if old was empty
// the key is placed; if old == c it is a duplicate (WOR: rejected, Algorithm
// H); otherwise the larger of the two (max(old, c)) moves on to slot s + 1.
// Keys only move right and every slot keeps the minimum of the keys that
// reach it, so the final table is the same for every insertion order (the
// warp's lanes insert concurrently) and reading the slots left to right
// gives the keys in ascending order, each duplicate dropped exactly once.
// WR keeps equal keys (an equal key moves on), so repeats end up adjacent.
//
// Per leaf, per round of draws (R7: round t+1 draws k - |S| more):
//   1. Philox blocks (lane l: blocks l + 32 m, two per step) -> draws -> one
//      atomicMin each at the home slot (the only random shared-memory access
//      most draws make); the ~21 % that must move on are appended to a
//      per-warp carry queue (ballot-compacted);
//   2. the queue is drained by the warp's lanes, each taking a new entry when
//      its chain ends;
// then the table is read row by row (32 slots per row, conflict-free): a
// ballot of the filled slots gives each key's output position, and each row
// is one coalesced store of ~16 consecutive u64 values straight to HBM.
//
// Entries carry a generation tag (x + (gen << CR), CR = ceil_log2 of the
// launch's largest leaf range): the table is cleared only every 2^(32-CR) - 1
// leaves; entries >= (gen + 1) << CR are empty or stale.  CR > 28: clear per leaf.
// Leaves the table cannot hold (more than LP_JMAX draws, or a chain running
// past the overflow slots) go to the spill list that the CTA kernel completes.

namespace rs {

constexpr int LP_LOGT = 11;
constexpr u32 LP_T = 1u << LP_LOGT;          // home slots
constexpr u32 LP_TO = 128;                   // overflow slots past the last home slot
constexpr u32 LP_TCAP = LP_T + LP_TO;        // 68 rows of 32 slots
constexpr u32 LP_QCAP = 512;                 // carry queue (circular) entries per warp
constexpr u32 LP_JMAX = 1408;                // draws per leaf held here (load <= 0.69)
constexpr u32 LP_EMPTY = 0xFFFFFFFFu;
static_assert((LP_TCAP / 32) % 4 == 0, "rows are read four at a time");

struct LPLeaf {
    u32 T[LP_TCAP];                          // ordered table
    uint2 Q[LP_QCAP];                        // carries: (entry, next slot)
    unsigned long long pf_off;               // prefetched count / offset of the next leaf
    u32 pf_k, pf_pad;
};
static_assert(sizeof(LPLeaf) % 16 == 0, "LPLeaf alignment");

__device__ __forceinline__ u32 lp_lanemask_lt()
{
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Predicated 8-byte global store of base + t at dst[idx] (IMAD.WIDE for the
// value and the address: the FMA pipe, not the ALU pipe).
__device__ __forceinline__ void lp_store_if(bool p, u64 *dst, u32 idx, u64 base, u32 t)
{
    asm volatile("{\n\t.reg .pred q;\n\t.reg .u64 a, v;\n\t"
                 "setp.ne.u32 q, %4, 0;\n\t"
                 "mad.wide.u32 a, %1, 8, %0;\n\t"
                 "mad.wide.u32 v, %3, 1, %2;\n\t"
                 "@q st.global.u64 [a], v;\n\t}"
                 ::"l"(dst), "r"(idx), "l"(base), "r"(t), "r"((u32)p) : "memory");
}

// Drain the circular carry queue Q[rd, wr): each pass takes up to 32 entries
// (one per lane) in FIFO order, probes once, and appends the chains that must
// move on (the larger key, next slot) at the tail -- until the queue is empty.
// A chain that runs past the overflow slots sets ovf (the leaf spills).
template <bool WR>
__device__ __forceinline__ void lp_drain(LPLeaf &sh, u32 wr, u32 limit, u32 lane, u32 lt, u32 &ndup, bool &ovf)
{
    u32 rd = 0;
#pragma unroll 1
    while (rd != wr) {
        const u32 n = min(wr - rd, 32u);
        const bool has = lane < n;
        uint2 e = make_uint2(0u, 0u);
        if (has) e = sh.Q[(rd + lane) & (LP_QCAP - 1)];
        const bool inb = has && e.y < LP_TCAP;
        ovf |= has && !inb;
        u32 old = LP_EMPTY;
        if (inb) old = atomicMin(&sh.T[e.y], e.x);
        const bool dup = !WR && inb && old == e.x;
        ndup += dup;
        const bool cont = inb && old < limit && !dup;
        const u32 m = __ballot_sync(0xffffffffu, cont);
        __syncwarp();
        if (cont) sh.Q[(wr + __popc(m & lt)) & (LP_QCAP - 1)] = make_uint2(max(old, e.x), e.y + 1);
        rd += n;
        wr += __popc(m);
    }
    __syncwarp();
}

// One round: insert draws [j0, j1) of the leaf (R3 Lemire draws; power-of-two
// ranges are the top cr bits of a word): one atomicMin per draw at its home
// slot, the chains that must move on go to the carry queue, then the drain.
template <bool WR>
__device__ __forceinline__ void lp_insert(LPLeaf &sh, const RoundKeys &K, const Drawer<u32> &dr, bool pow2,
                                          u32 cr, u32 j0, u32 j1, u32 G, u32 limit, u32 lane, u32 lt,
                                          u32 &ndup, bool &ovf)
{
    const u32 sc = pow2 ? (1u << (cr & 31)) : 0u;                // x = hi(w * 2^cr)
    const u32 hsh = (u32)cr - LP_LOGT;                            // home = x >> hsh
    u32 qn = 0;
    const u32 qlo = j0 >> 2, qhi = (j1 + 3) >> 2;
#pragma unroll 1
    for (u32 qb = qlo; qb < qhi; qb += 64) {
        if (qn + 256 > LP_QCAP) {                 // room for this step's carries
            lp_drain<WR>(sh, qn, limit, lane, lt, ndup, ovf);
            qn = 0;
        }
        u32 e[8], hm[8], old[8];
        bool v[8];
        const bool full = 4 * qb >= j0 && 4 * (qb + 64) <= j1;   // every draw of the step counts
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const u32 q = qb + lane + 32u * b;
            const u32x4 w = philox_rk_(q, dr.st.tag, dr.st.id_lo, dr.st.id_hi, K);
            const u32 ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const u32 j = 4 * q + t;
                v[4 * b + t] = full || (j >= j0 && j < j1);
                u32 x;
                if (pow2) {
                    x = __umulhi(ws[t], sc);
                    hm[4 * b + t] = ws[t] >> (32 - LP_LOGT);         // == x >> hsh
                } else {
                    x = v[4 * b + t] ? dr.fix(ws[t], j) : 0u;
                    hm[4 * b + t] = x >> hsh;
                }
                e[4 * b + t] = x + G;
            }
        }
        // all eight probes first (no store between them: they issue back to back)
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            old[t] = LP_EMPTY;
            if (v[t]) old[t] = atomicMin(&sh.T[hm[t]], e[t]);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const bool dup = !WR && v[t] && old[t] == e[t];
            ndup += dup;
            const bool carry = v[t] && old[t] < limit && !dup;
            const u32 m = __ballot_sync(0xffffffffu, carry);
            if (carry) sh.Q[qn + __popc(m & lt)] = make_uint2(max(old[t], e[t]), hm[t] + 1);
            qn += __popc(m);
        }
    }
    __syncwarp();
    lp_drain<WR>(sh, qn, limit, lane, lt, ndup, ovf);
}

template <bool WR>
__device__ __forceinline__ void lp_leaves(const LeafArgs &a)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    LPLeaf &sh = reinterpret_cast<LPLeaf *>(smem_raw)[wid];
    const u32 lt = lp_lanemask_lt();
    const u32 CR = a.lp_cr;                                   // launch-uniform tag shift
    const bool gens = CR <= 28;
    const u32 NG = gens ? (1u << (32 - CR)) - 1u : 1u;        // generations per clear
    u32 gleft = 0;                                            // generations left before a clear
    const u64 stride = (u64)gridDim.x * LP_WARPS;
    u64 L = (u64)blockIdx.x * LP_WARPS + wid;
    const u32 s_k = (u32)__cvta_generic_to_shared(&sh.pf_k), s_off = (u32)__cvta_generic_to_shared(&sh.pf_off);
    if (lane == 0 && L < a.nleaves) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s_k), "l"(a.cnt + L) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s_off), "l"(a.off + L) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
#pragma unroll 1
    for (; L < a.nleaves; L += stride) {
        if (lane == 0) asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        const u32 k = sh.pf_k;
        const u64 off = sh.pf_off;
        __syncwarp();
        if (lane == 0 && L + stride < a.nleaves) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s_k), "l"(a.cnt + L + stride) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s_off), "l"(a.off + L + stride) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        if (k == 0) continue;
        if (k > LP_JMAX) {                                    // the CTA kernel completes it
            if (lane == 0) a.spill[atomicAdd(a.spill_n, 1u)] = (u32)L;
            continue;
        }
        if (gleft == 0) {                                     // clear: every slot empty
#pragma unroll 1
            for (u32 i = 4 * lane; i < LP_TCAP; i += 128)
                *reinterpret_cast<uint4 *>(&sh.T[i]) = make_uint4(LP_EMPTY, LP_EMPTY, LP_EMPTY, LP_EMPTY);
            gleft = NG;
            __syncwarp();
        }
        --gleft;
        const u32 G = gens ? gleft << CR : 0u;                // this leaf's generation tag
        const u32 limit = gens ? (gleft + 1u) << CR : LP_EMPTY;
        const LeafGeom g = leaf_geom(a, L);
        const u32 cr = (u32)ceil_log2(g.r);
        const Drawer<u32> dr(Stream(a.seed, WR ? P_WR : P_WOR, g.id), g.r);
        const bool pow2 = (g.r & (g.r - 1)) == 0;
        u32 ndup = 0, J0 = 0, J = k;
        bool ovf = false;
        for (;;) {                                            // rounds (R7)
            lp_insert<WR>(sh, a.rk, dr, pow2, cr, J0, J, G, limit, lane, lt, ndup, ovf);
            if (WR || __any_sync(0xffffffffu, ovf)) break;
            const u32 dist = J - __reduce_add_sync(0xffffffffu, ndup);
            if (dist >= k) break;
            J0 = J;
            J += k - dist;
            if (J > LP_JMAX) { ovf = true; break; }
        }
        if (__any_sync(0xffffffffu, ovf)) {
            if (lane == 0) a.spill[atomicAdd(a.spill_n, 1u)] = (u32)L;
            continue;                                          // (its entries are stale from here on)
        }
        // rows: each filled slot's output index is the number of filled slots before it
        const u64 base = g.lo + 1 - (u64)G;                   // value = base + entry
        u64 *dst = a.out + off;
        u32 pos = 0;
#pragma unroll 1
        for (u32 i = 0; i < LP_TCAP / 32; i += 4) {
            u32 t[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) t[r] = sh.T[32 * (i + r) + lane];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const bool f = t[r] < limit;
                const u32 m = __ballot_sync(0xffffffffu, f);
                lp_store_if(f, dst, pos + __popc(m & lt), base, t[r]);
                pos += __popc(m);
            }
            if (pos >= k) break;
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(32 * LP_WARPS, 1) k_leaf_lp_wor(LeafArgs a) { lp_leaves<false>(a); }
__global__ void __launch_bounds__(32 * LP_WARPS, 1) k_leaf_lp_wr(LeafArgs a) { lp_leaves<true>(a); }

}  // namespace rs
