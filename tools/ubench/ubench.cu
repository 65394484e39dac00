// Microbenchmarks of the primitives the leaf kernel is built from (sm_100a):
// Philox4x32-10 blocks, shared-memory atomics / loads / stores at random
// addresses, and the global write ceiling.  Dev tool: numbers go to DESIGN.md.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef uint32_t u32; typedef uint64_t u64;

__device__ __forceinline__ uint4 philox(u32 c0, u32 c1, u32 c2, u32 c3, u32 k0, u32 k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    u32 h0 = __umulhi(0xD2511F53u, c0), l0 = 0xD2511F53u * c0;
    u32 h1 = __umulhi(0xCD9E8D57u, c2), l1 = 0xCD9E8D57u * c2;
    c0 = h1 ^ c1 ^ k0; c1 = l1; c2 = h0 ^ c3 ^ k1; c3 = l0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

__global__ void k_philox(u32 iters, u32 *out, u32 seed) {
  u32 acc = 0;
  u32 t = blockIdx.x * blockDim.x + threadIdx.x;
  for (u32 i = 0; i < iters; ++i) {
    uint4 w = philox(i, 2u << 24, t, 0, seed, 7);
    acc ^= w.x ^ w.y ^ w.z ^ w.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

// random smem ops: each thread does iters ops at pseudo-random addresses in a 16 KB table
template <int OP>
__global__ void k_smem(u32 iters, u32 *out) {
  __shared__ u32 T[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) T[i] = i;
  __syncthreads();
  u32 x = threadIdx.x * 0x9E3779B9u + blockIdx.x, acc = 0;
  for (u32 i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    u32 a = x >> 20;  // 0..4095
    if (OP == 0) acc += atomicAdd(&T[a], 1u);
    else if (OP == 1) acc += atomicOr(&T[a], 1u << (x & 31));
    else if (OP == 2) acc += T[a];
    else if (OP == 3) T[a] = x;
    else if (OP == 4) atomicAdd(&T[a], 1u);   // no return (RED)
    else if (OP == 5) acc += atomicCAS(&T[a], acc, x);
  }
  __syncthreads();
  if (acc == 0x12345678 || T[threadIdx.x] == 0x12345679) out[0] = acc;
}

// issue ceiling: 8 independent chains of one-instruction steps per thread
// (inline PTX: lop3.b32 -> one LOP3 on the ALU pipe; mul.wide.u32 -> one
// IMAD.WIDE on the FMA pipe), 16 steps unrolled per loop trip.
__global__ void k_lop3(u32 iters, u32 *out) {
  u32 a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = threadIdx.x * (c + 3) + blockIdx.x;
  for (u32 i = 0; i < iters; i += 16) {
#pragma unroll
    for (int s = 0; s < 16; ++s)
#pragma unroll
      for (int c = 0; c < 8; ++c) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(a[(c + 1) & 7]), "r"(i));
  }
  u32 acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc ^= a[c];
  if (acc == 0x12345678) out[0] = acc;
}
__global__ void k_imadw(u32 iters, u32 *out) {
  u64 a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = threadIdx.x * (c + 3) + blockIdx.x;
  for (u32 i = 0; i < iters; i += 16) {
#pragma unroll
    for (int s = 0; s < 16; ++s)
#pragma unroll
      for (int c = 0; c < 8; ++c) asm volatile("mul.wide.u32 %0, %1, 0xD2511F53;" : "=l"(a[c]) : "r"((u32)(a[c] >> 32) + (u32)a[c]));
  }
  u64 acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc ^= a[c];
  if (acc == 0x12345678) out[0] = (u32)acc;
}
// conflict-free LDS (lane-strided) for the wavefront rate
__global__ void k_lds_cf(u32 iters, u32 *out) {
  __shared__ u32 T[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) T[i] = i;
  __syncthreads();
  u32 acc = 0, b = threadIdx.x & 31;
  for (u32 i = 0; i < iters; ++i) { acc += T[(b + 32 * (i & 127))]; b ^= acc & 0; }
  if (acc == 0x12345678) out[0] = acc;
}

// baseline: the LCG loop alone
__global__ void k_lcg(u32 iters, u32 *out) {
  u32 x = threadIdx.x * 0x9E3779B9u + blockIdx.x, acc = 0;
  for (u32 i = 0; i < iters; ++i) { x = x * 1664525u + 1013904223u; acc += x >> 20; }
  if (acc == 0x12345678) out[0] = acc;
}

template <int V>
__global__ void k_fill(u64 *out, u64 n) {
  u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x, st = (u64)gridDim.x * blockDim.x;
  if (V == 1) { for (u64 i = i0; i < n; i += st) out[i] = i + 1; }
  if (V == 2) { for (u64 i = i0; i < n / 2; i += st) { ulonglong2 v = make_ulonglong2(2*i+1, 2*i+2); reinterpret_cast<ulonglong2*>(out)[i] = v; } }
  if (V == 4) { for (u64 i = i0; i < n / 4; i += st) {
      u64 a = 4*i+1, b = a+1, c = a+2, d = a+3; u64 *p = out + 4*i;
      asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" :: "l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory"); } }
}


// ---- cycle-accurate issue / smem rates (clock-frequency independent) -----
// Each block records its SM-clock duration; rate = warp-ops per SM per cycle
// = (warps per SM x ops per warp) / cycles.  Launched with exactly `per`
// resident blocks per SM so every SM runs the same load.
__device__ long long g_cyc[4096];

template <int OP>
__global__ void k_rate(u32 iters, u32 *out) {
  __shared__ u32 T[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) T[i] = i * 7u;
  __syncthreads();
  const long long t0 = clock64();
  u32 a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = threadIdx.x * (c + 3) + blockIdx.x;
  u32 x = threadIdx.x * 0x9E3779B9u + blockIdx.x, acc = 0;
  const u32 lane = threadIdx.x & 31;
  for (u32 i = 0; i < iters; i += 16) {
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      if (OP == 0) {            // 8 LOP3 per step (ALU pipe)
#pragma unroll
        for (int c = 0; c < 8; ++c) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(a[(c + 1) & 7]), "r"(i));
      } else if (OP == 1) {     // 8 IMAD (FMA pipe)
#pragma unroll
        for (int c = 0; c < 8; ++c) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(a[(c + 1) & 7]), "r"(i));
      } else if (OP == 2) {     // 4 LOP3 + 4 IMAD interleaved
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(a[(c + 1) & 7]), "r"(i));
          asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c + 1]) : "r"(a[(c + 2) & 7]), "r"(i));
        }
      } else if (OP == 3) {     // 8 IMAD.WIDE (mul.wide.u32)
#pragma unroll
        for (int c = 0; c < 8; ++c) { u64 p; asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a[c]), "r"(a[(c+1)&7])); a[c] = (u32)(p >> 32); }
      } else if (OP == 4) {     // 1 conflict-free LDS (lane stride)
        acc += T[lane + 32 * ((i + s) & 127)];
      } else if (OP == 5) {     // 1 random LDS
        x = x * 1664525u + 1013904223u; acc += T[x >> 20];
      } else if (OP == 6) {     // 1 random ATOMS.ADD (no return)
        x = x * 1664525u + 1013904223u; atomicAdd(&T[x >> 20], 1u);
      } else if (OP == 7) {     // 1 conflict-free STS
        T[lane + 32 * ((i + s) & 127)] = x; x += 3;
      } else if (OP == 8) {     // 1 SHFL
        acc += __shfl_sync(0xffffffffu, acc + s, (lane + 1 + s) & 31);
      } else if (OP == 9) {     // 1 random ATOMS.MIN with return
        x = x * 1664525u + 1013904223u; acc += atomicMin(&T[x >> 20], x);
      } else if (OP == 10) {    // 1 random ATOMS.ADD of a variable with return
        x = x * 1664525u + 1013904223u; acc += atomicAdd(&T[x >> 20], x & 7u);
      } else if (OP == 11) {    // 1 random ATOMS.ADD(1) with return (POPC.INC form)
        x = x * 1664525u + 1013904223u; acc += atomicAdd(&T[x >> 20], 1u);
      } else if (OP == 12) {    // 1 random STS
        x = x * 1664525u + 1013904223u; T[x >> 20] = x;
      } else if (OP == 13) {    // 1 random ATOMS.MIN, no return
        x = x * 1664525u + 1013904223u; atomicMin(&T[x >> 20], x);
      } else if (OP == 14) {    // ATOMS.MIN, lane-distinct banks (conflict-free)
        x = x * 1664525u + 1013904223u; acc += atomicMin(&T[lane + 32 * ((x >> 20) & 127)], x);
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  u32 r = acc;
#pragma unroll
  for (int c = 0; c < 8; ++c) r ^= a[c];
  if (r == 0x12345678 || T[threadIdx.x] == 0x12345679) out[0] = r;
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

#define TIME(label, launch, work, unit) do { \
  launch; cudaDeviceSynchronize(); cudaEventRecord(e0); for (int r = 0; r < 3; ++r) { launch; } cudaEventRecord(e1); \
  cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3; \
  printf("%-28s %9.3f ms  %10.3f %s\n", label, ms, (double)(work) / (ms * 1e-3) / 1e9, unit); } while (0)

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  printf("%s SMs=%d\n", p.name, sms);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  u32 *o; cudaMalloc(&o, 64);
  int grid = sms * 8, nt = 256; u32 it = 4096;
  double threads = (double)grid * nt;
  TIME("philox blocks", (k_philox<<<grid, nt>>>(it, o, 1)), threads * it, "G blocks/s");
  TIME("lcg loop", (k_lcg<<<grid, nt>>>(it * 4, o)), threads * it * 4, "G it/s");
  TIME("lop3 chains (1 LOP3/step)", (k_lop3<<<grid, nt>>>(it, o)), threads * it * 8, "G thread-inst/s");
  TIME("imad.wide+iadd3 (2/step)", (k_imadw<<<grid, nt>>>(it, o)), threads * it * 8 * 2, "G thread-inst/s");
  TIME("smem LDS conflict-free", (k_lds_cf<<<grid, nt>>>(it, o)), threads * it, "G ops/s");
  TIME("smem atomicAdd ret", (k_smem<0><<<grid, nt>>>(it, o)), threads * it, "G ops/s");
  TIME("smem atomicOr ret", (k_smem<1><<<grid, nt>>>(it, o)), threads * it, "G ops/s");
  TIME("smem LDS random", (k_smem<2><<<grid, nt>>>(it, o)), threads * it, "G ops/s");
  TIME("smem STS random", (k_smem<3><<<grid, nt>>>(it, o)), threads * it, "G ops/s");
  TIME("smem atomicAdd noret", (k_smem<4><<<grid, nt>>>(it, o)), threads * it, "G ops/s");
  TIME("smem atomicCAS", (k_smem<5><<<grid, nt>>>(it, o)), threads * it, "G ops/s");
  {   // warm the clocks up (~1 s of work) before the cycle-based rates
    for (int r = 0; r < 40; ++r) k_philox<<<grid, nt>>>(it, o, 1);
    cudaDeviceSynchronize();
    const char *names[] = {"LOP3 (8/step)", "IMAD (8/step)", "LOP3+IMAD (4+4/step)", "IMAD.WIDE (8/step)",
                           "LDS conflict-free (1/step)", "LDS random (1/step)", "ATOMS.ADD random (1/step)",
                           "STS conflict-free (1/step)", "SHFL (1/step)", "ATOMS.MIN random ret", "ATOMS.ADD var random ret",
                           "ATOMS.ADD 1 random ret", "STS random", "ATOMS.MIN random noret", "ATOMS.MIN conflict-free ret"};
    const double ops[] = {8, 8, 8, 8, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
    const int W = 16;                // warps per SM (one 512-thread block per SM)
    void (*const ks[])(u32, u32 *) = {k_rate<0>, k_rate<1>, k_rate<2>, k_rate<3>, k_rate<4>, k_rate<5>, k_rate<6>,
                                       k_rate<7>, k_rate<8>, k_rate<9>, k_rate<10>, k_rate<11>, k_rate<12>, k_rate<13>, k_rate<14>};
    for (int op = 0; op < 15; ++op) {
      void (*k)(u32, u32 *) = ks[op];
      const u32 iters = 8192;
      k<<<sms, 32 * W>>>(iters, o);
      cudaDeviceSynchronize();
      k<<<sms, 32 * W>>>(iters, o);
      cudaDeviceSynchronize();
      long long cyc[4096];
      cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(long long) * sms);
      double mean = 0; for (int b = 0; b < sms; ++b) mean += (double)cyc[b]; mean /= sms;
      const double wops = (double)W * iters * ops[op];       // warp-level ops per SM
      printf("%-28s %8.3f warp-ops/SM/cycle (%6.1f thread-ops/SM/cycle)  [16 warps/SM, %.0f cycles]\n",
             names[op], wops / mean, 32 * wops / mean, mean);
    }
  }
  u64 n = 1ull << 32; u64 *buf; cudaMalloc(&buf, n * 8);
  for (int g : {sms * 4, sms * 8, sms * 16}) {
    char l[64];
    snprintf(l, 64, "fill u64 v1 grid=%d", g); TIME(l, (k_fill<1><<<g, 256>>>(buf, n)), n * 8.0, "GB/s");
    snprintf(l, 64, "fill u64 v2 grid=%d", g); TIME(l, (k_fill<2><<<g, 256>>>(buf, n)), n * 8.0, "GB/s");
    snprintf(l, 64, "fill u64 v4 grid=%d", g); TIME(l, (k_fill<4><<<g, 256>>>(buf, n)), n * 8.0, "GB/s");
  }
  TIME("cudaMemsetAsync 32GiB", (cudaMemsetAsync(buf, 0, n * 8)), n * 8.0, "GB/s");
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
