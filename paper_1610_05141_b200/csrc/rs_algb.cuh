// rs_algb.cuh -- NEXT-4: the repair step of Algorithm B as the
// paper's GPU variant does it ("marks the appropriate positions in
// the sample array for removal.  Finally, the sample array is compacted"),
// fused into one pass: S[0..n') minus the elements at the sorted 1-based
// positions R[0..nr) -> out[0..n' - nr).  Included by rs_kernels.cu.
//
// Element i (0-based) moves to i - #{R <= i}; it is dropped iff i + 1 is in R.
// One CTA per tile of AB_TILE elements: two binary searches give the tile's
// first and last removal, the few removals inside the tile (expected
// AB_TILE (n'-n)/n' << 1) go to shared memory.  HBM-bound: 8 B read per
// input element, 8 B written per output element.

namespace rs {

__device__ __forceinline__ u64 ab_count_le(const u64 *R, u64 nr, u64 x)   // #{R[t] <= x}
{
    u64 lo = 0, hi = nr;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (R[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(AB_THREADS) k_algb_compact(const u64 *__restrict__ S, u64 np,
                                                             const u64 *__restrict__ R, u64 nr,
                                                             u64 *__restrict__ out)
{
    __shared__ u64 c01[2];
    __shared__ u64 rs_[AB_SMAX];
    const u32 tid = threadIdx.x;
    for (u64 lo = (u64)blockIdx.x * AB_TILE; lo < np; lo += (u64)gridDim.x * AB_TILE) {
        const u64 hi = lo + AB_TILE < np ? lo + AB_TILE : np;
        if (tid == 0) c01[0] = ab_count_le(R, nr, lo);
        if (tid == 32) c01[1] = ab_count_le(R, nr, hi);
        __syncthreads();
        const u64 c0 = c01[0], nin = c01[1] - c0;
        if (nin <= AB_SMAX)
            for (u32 t = tid; t < nin; t += AB_THREADS) rs_[t] = R[c0 + t];
        __syncthreads();
        u64 v[AB_PER];
#pragma unroll
        for (int j = 0; j < AB_PER; ++j) {
            const u64 i = lo + (u64)j * AB_THREADS + tid;
            v[j] = i < hi ? S[i] : 0ull;
        }
#pragma unroll
        for (int j = 0; j < AB_PER; ++j) {
            const u64 i = lo + (u64)j * AB_THREADS + tid;
            if (i >= hi) break;
            if (nin == 0) { out[i - c0] = v[j]; continue; }
            u64 s;
            bool rm;
            if (nin <= AB_SMAX) {
                s = c0; rm = false;
                for (u32 t = 0; t < (u32)nin; ++t) { s += rs_[t] <= i; rm |= rs_[t] == i + 1; }
            } else {
                s = ab_count_le(R, nr, i);
                rm = s < nr && R[s] == i + 1;
            }
            if (!rm) out[i - s] = v[j];
        }
        __syncthreads();
    }
}

}  // namespace rs
