// Global-memory atomic throughput probe: atomicAdd with return on random u32 addresses
// inside a region of R bytes (L2-resident vs HBM), and no-return RED, plus per-CTA
// private regions (each CTA hits only its own 1 MB slab) like per-block counter arrays.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template <int RET>
__global__ void k(uint32_t* a, uint64_t words_per_cta, int iters, unsigned long long* out) {
  uint32_t s = hsh(blockIdx.x * 977 + threadIdx.x);
  uint32_t* base = a + (uint64_t)blockIdx.x * words_per_cta;
  unsigned long long acc = 0;
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    s = s * 1664525u + 1013904223u;
    uint32_t idx = (uint32_t)(((uint64_t)(s >> 4) * words_per_cta) >> 28);
    if (RET) acc += atomicAdd(base + idx, 1u); else atomicAdd(base + idx, 1u);
  }
  if (acc == 12345) out[0] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out; cudaMalloc(&out, 64);
  size_t total = (size_t)2 << 30; uint32_t* a; cudaMalloc(&a, total); cudaMemset(a, 0, total);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocks_per_sm : {4, 8}) for (uint64_t slab_kb : {16ull, 128ull, 1024ull}) for (int ret : {0, 1}) {
    int grid = sms * blocks_per_sm, thr = 256, iters = 2048;
    uint64_t wpc = slab_kb * 256;
    if ((uint64_t)grid * wpc * 4 > total) continue;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (ret) k<1><<<grid, thr>>>(a, wpc, iters, out); else k<0><<<grid, thr>>>(a, wpc, iters, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)grid * thr * iters;
      if (rep) printf("grid %5d slab %5llu KB (total %6.1f MB) %s: %.3e atomics/s\n", grid, (unsigned long long)slab_kb,
                      grid * wpc * 4 / 1e6, ret ? "atom.ret" : "red     ", ops / (ms * 1e-3));
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
