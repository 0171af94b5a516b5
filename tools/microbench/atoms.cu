// Shared-memory atomic throughput microbenchmark (B200 design probe).
// Measures warp-wide ATOMS/RED on spread addresses, with/without return,
// u32 vs packed-u16x2, and match_any aggregation cost.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_atoms(int iters, uint32_t span_mask, unsigned long long* out) {
  extern __shared__ uint32_t cnt[];
  for (int i = threadIdx.x; i <= span_mask; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  uint32_t seed = hsh(blockIdx.x * 1024 + threadIdx.x);
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    seed = seed * 1664525u + 1013904223u;
    uint32_t a = (seed >> 8) & span_mask;
    if (MODE == 0) {            // red (no return)
      atomicAdd(&cnt[a], 1u);
    } else if (MODE == 1) {     // atom with return
      acc += atomicAdd(&cnt[a], (seed & 1) ? 1u : 0x10000u);
    } else if (MODE == 2) {     // plain ld+st (non-atomic upper bound)
      cnt[a] += 1u;
    } else if (MODE == 3) {     // match_any + leader atomic with return
      uint32_t peers = __match_any_sync(0xffffffffu, a);
      int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if ((threadIdx.x & 31) == leader) old = atomicAdd(&cnt[a], __popc(peers));
      acc += old;
    } else if (MODE == 4) {     // 64-bit atomic with return
      acc += atomicAdd((unsigned long long*)&cnt[a & ~1u], 1ull);
    }
  }
  __syncthreads();
  if (acc == 0x123456789ull) out[0] = acc;
  if (threadIdx.x == 0) out[1 + blockIdx.x] = cnt[0];
}

__global__ void k_stream(const int4* __restrict__ p, size_t n, unsigned long long* out) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(p + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x7fffffff) out[0] = 1;
}

template <int MODE>
float run(int sms, int threads, int iters, uint32_t span, unsigned long long* out) {
  size_t smem = span * 4;
  cudaFuncSetAttribute(k_atoms<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_atoms<MODE><<<sms, threads, smem>>>(iters, span - 1, out);
  cudaEventRecord(a);
  k_atoms<MODE><<<sms, threads, smem>>>(iters, span - 1, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  return ms;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("dev %s sms %d l2 %d MB smem/blk optin %zu clock %d kHz\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, p.clockRate);
  int sms = p.multiProcessorCount;
  unsigned long long* out; CK(cudaMalloc(&out, 8 * 4096));
  const char* names[] = {"red.u32", "atom.ret.u32", "plain ld/st", "match+atom", "atom.ret.u64"};
  for (uint32_t span : {4096u, 32768u}) for (int threads : {256, 1024}) {
    int iters = 4096;
    double n = (double)sms * threads * iters;
    float t0 = run<0>(sms, threads, iters, span, out);
    float t1 = run<1>(sms, threads, iters, span, out);
    float t2 = run<2>(sms, threads, iters, span, out);
    float t3 = run<3>(sms, threads, iters, span, out);
    float t4 = run<4>(sms, threads, iters, span, out);
    float ts[] = {t0, t1, t2, t3, t4};
    for (int m = 0; m < 5; ++m)
      printf("span %6u thr %4d %-14s %8.3f ms  %.3e ops/s  %.2f cyc/warp-instr/SM\n", span, threads, names[m], ts[m], n / (ts[m] * 1e-3),
             (ts[m] * 1e-3 * p.clockRate * 1e3) / (n / 32 / sms));
  }
  size_t bytes = (size_t)8 << 30; int4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a); k_stream<<<sms * 8, 256>>>(buf, bytes / 16, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); printf("stream read %.1f GB/s\n", bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
