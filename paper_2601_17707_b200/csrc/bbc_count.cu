// Wedge-enumeration + closing kernel (G-BBC static / G-BBC++ dynamic).
//
// Reference mechanisms restated (paths under /root/reference):
//   pkg/src/bbcount/buckets.py:166-197   per-anchor wedge buckets, filter, closing
//   pkg/src/bbcount/tiled.py:107-168     G-BBC: static round-robin blocks, end-vertex
//                                        tiles of bounded span (TileConfig.tile_size)
//   pkg/src/bbcount/tiled.py:182-292     G-BBC++: fanout-sorted tasks claimed from a
//                                        shared counter by persistent workers
//   PAPER.md:873-912 (Alg. 3), 1190-1253 (Alg. 4)
//
// One CTA processes one anchor (start vertex) u at a time.  For every record
// (u, c) it walks the admitted suffix of centre c's rank-sorted list, i.e. the
// wedges u -> c -> w with rank(w) > rank(u), and adds 1 to the positive or
// negative half of w's packed u16x2 counter in a shared-memory tile over the
// end-vertex rank range [lo, lo + span).  Parity = sign bit of (word ^ s(u,c)).
// A tile is closed either by a sweep (balanced += C(p,2)+C(q,2), unbalanced +=
// p*q, counter := 0) or, for sparse tiles, inline from the atomic's return value
// (a + wedge adds the old positive count to balanced and the old negative count
// to unbalanced, and vice versa; summed over all increments this equals the
// sweep) followed by a re-walk that zeroes only the touched counters.
#include <algorithm>
#include <string>

#include "bbc_internal.cuh"

namespace bbc {

namespace {

constexpr int kCountThreads = 1024;
constexpr int kWarps = kCountThreads / 32;
constexpr int kRB = 2048;  // records per batch held in shared memory
constexpr uint32_t kFull = 0xffffffffu;

enum Mode { kDense = 0, kSparse = 1, kZero = 2, kWide = 3 };

struct Params {
  const uint32_t* __restrict__ adj;
  const uint2* __restrict__ rec;
  const uint32_t* __restrict__ aoff;
  const unsigned long long* __restrict__ awork;
  const uint32_t* __restrict__ order;
  uint32_t n;
  uint32_t ntasks;
  uint32_t part_index;
  uint32_t part_count;
  uint32_t span16;  // endpoint span of a packed tile
  uint32_t span32;  // endpoint span of a wide (2 x u32) tile
  uint32_t cap_words;
  int dynamic;
  unsigned long long* acc;
  unsigned int* queue;
  unsigned long long* block_work;
};

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// first position in [lo, hi) whose rank is >= x (lists are rank-sorted)
__device__ __forceinline__ uint32_t lower_bound_rank(const uint32_t* __restrict__ adj, uint32_t lo, uint32_t hi,
                                                     uint32_t x) {
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if ((__ldg(adj + mid) & 0x7fffffffu) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// exclusive scan of a[0..nb) in place; returns the total.  All threads call.
__device__ uint32_t block_exclusive_scan(uint32_t* a, int nb, uint32_t* s_warp) {
  constexpr int per = kRB / kCountThreads;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int base = threadIdx.x * per;
  uint32_t v[per];
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < per; ++i) {
    v[i] = (base + i < nb) ? a[base + i] : 0u;
    sum += v[i];
  }
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;
  }
  __syncthreads();
  uint32_t excl = x - sum + (warp > 0 ? s_warp[warp - 1] : 0u);
#pragma unroll
  for (int i = 0; i < per; ++i) {
    if (base + i < nb) a[base + i] = excl;
    excl += v[i];
  }
  uint32_t total = s_warp[kWarps - 1];
  __syncthreads();
  return total;
}

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long x, unsigned long long* s_red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  if (lane == 0) s_red[warp] = x;
  __syncthreads();
  unsigned long long t = 0;
#pragma unroll 4
  for (int w = 0; w < kWarps; ++w) t += s_red[w];
  __syncthreads();
  return t;
}

// largest k in [0, nb) with pfx[k] <= ch
__device__ __forceinline__ int find_record(const uint32_t* pfx, int nb, uint32_t ch) {
  int lo = 0, hi = nb;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (pfx[mid] <= ch)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// Walk all chunks of the current record batch.  A chunk is 32 aligned int4
// groups (128 adjacency words) of one record's sub-slice, one group per lane.
template <int M>
__device__ __forceinline__ void run_chunks(const Params& P, uint32_t* cnt, const uint32_t* s_sb,
                                           const uint32_t* s_se, const uint32_t* s_pfx, int nb, uint32_t nchunks,
                                           uint32_t lo, unsigned long long& tb, unsigned long long& tu) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint4* adj4 = reinterpret_cast<const uint4*>(P.adj);
  for (uint32_t ch = warp; ch < nchunks; ch += kWarps) {
    const int k = find_record(s_pfx, nb, ch);
    const uint32_t sbx = s_sb[k];
    const uint32_t sb = sbx & 0x7fffffffu, sgn = sbx & 0x80000000u, se = s_se[k];
    const uint32_t grp = (sb >> 2) + (ch - s_pfx[k]) * 32u + (uint32_t)lane;
    const uint32_t p0 = grp * 4u;
    if (p0 < se) {
      const uint4 q = ld_stream(adj4 + grp);
      const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t p = p0 + (uint32_t)j;
        if (p >= sb && p < se) {
          const uint32_t word = wv[j];
          const uint32_t idx = (word & 0x7fffffffu) - lo;
          const uint32_t par = (word ^ sgn) >> 31;  // 1: asymmetric (negative) wedge
          if (M == kDense) {
            atomicAdd(&cnt[idx], par ? 0x10000u : 1u);
          } else if (M == kWide) {
            atomicAdd(&cnt[2u * idx + par], 1u);
          } else if (M == kSparse) {
            const uint32_t old = atomicAdd(&cnt[idx], par ? 0x10000u : 1u);
            const uint32_t lo16 = old & 0xffffu, hi16 = old >> 16;
            tb += par ? hi16 : lo16;
            tu += par ? lo16 : hi16;
          } else {  // kZero
            cnt[idx] = 0u;
          }
        }
      }
    }
  }
}

// closing sweep of a packed tile: balanced += C(p,2)+C(q,2), unbalanced += p*q
__device__ __forceinline__ void sweep16(uint32_t* cnt, uint32_t span, unsigned long long& tb,
                                        unsigned long long& tu) {
  uint4* c4 = reinterpret_cast<uint4*>(cnt);
  const uint32_t nq = (span + 3) >> 2;
  for (uint32_t i = threadIdx.x; i < nq; i += kCountThreads) {
    uint4 x = c4[i];
    if ((x.x | x.y | x.z | x.w) == 0u) continue;
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t p = xs[j] & 0xffffu, q = xs[j] >> 16;
      tb += (unsigned long long)((p * (p - (p > 0))) >> 1) + (unsigned long long)((q * (q - (q > 0))) >> 1);
      tu += (unsigned long long)(p * q);
    }
    c4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// closing sweep of a wide tile (interleaved u32 positive / negative counts)
__device__ __forceinline__ void sweep32(uint32_t* cnt, uint32_t span, unsigned long long& tb,
                                        unsigned long long& tu) {
  uint4* c4 = reinterpret_cast<uint4*>(cnt);
  const uint32_t nq = (2u * span + 3) >> 2;
  for (uint32_t i = threadIdx.x; i < nq; i += kCountThreads) {
    uint4 x = c4[i];
    if ((x.x | x.y | x.z | x.w) == 0u) continue;
    const unsigned long long p0 = x.x, q0 = x.y, p1 = x.z, q1 = x.w;
    tb += p0 * (p0 - (p0 > 0)) / 2 + q0 * (q0 - (q0 > 0)) / 2 + p1 * (p1 - (p1 > 0)) / 2 + q1 * (q1 - (q1 > 0)) / 2;
    tu += p0 * q0 + p1 * q1;
    c4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
}

__device__ __forceinline__ void add128(unsigned long long& lo, unsigned long long& hi, unsigned long long x) {
  lo += x;
  hi += (lo < x) ? 1ull : 0ull;
}

__global__ void __launch_bounds__(kCountThreads, 1) k_count(Params P) {
  extern __shared__ uint4 smem4[];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem4);
  uint32_t* s_sb = cnt + P.cap_words;
  uint32_t* s_se = s_sb + kRB;
  uint32_t* s_pfx = s_se + kRB;
  __shared__ uint32_t s_warp[32];
  __shared__ unsigned long long s_red[kWarps];
  __shared__ uint32_t s_task;

  for (uint32_t i = threadIdx.x; i < P.cap_words / 4; i += kCountThreads) smem4[i] = make_uint4(0u, 0u, 0u, 0u);

  unsigned long long bal_lo = 0, bal_hi = 0, unb_lo = 0, unb_hi = 0, work = 0;
  uint32_t next = blockIdx.x;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_task = P.dynamic ? atomicAdd(P.queue, 1u) : next;
    __syncthreads();
    const uint32_t t = s_task;
    next += gridDim.x;
    if (t >= P.ntasks) break;
    const uint32_t gidx = P.part_index + t * P.part_count;
    const uint32_t r = P.dynamic ? P.order[gidx] : gidx;
    if (P.awork[r] == 0ull) continue;
    const uint32_t rb = P.aoff[r], re = P.aoff[r + 1];
    const bool wide = (re - rb) > 65535u;  // counts are bounded by deg(u); u16 halves suffice below
    const uint32_t span_cap = wide ? P.span32 : P.span16;
    unsigned long long tb = 0, tu = 0;
    for (uint32_t lo = r + 1; lo < P.n; lo += span_cap) {
      const uint32_t hi = min(P.n, lo + span_cap);
      const uint32_t span = hi - lo;
      const bool first = lo == r + 1, last = hi == P.n;
      int mode = -1;
      unsigned long long tile_w = 0;
      for (uint32_t b0 = rb; b0 < re; b0 += kRB) {
        const int nb = (int)min((uint32_t)kRB, re - b0);
        unsigned long long myw = 0;
        for (int k = threadIdx.x; k < nb; k += kCountThreads) {
          const uint2 rr = P.rec[b0 + k];
          uint32_t sb = rr.x & 0x7fffffffu, se = rr.y;
          if (!first) sb = lower_bound_rank(P.adj, sb, se, lo);
          if (!last) se = lower_bound_rank(P.adj, sb, se, hi);
          uint32_t nq = 0;
          if (se > sb) {
            nq = ((se + 3u) >> 2) - (sb >> 2);
            myw += se - sb;
          }
          s_sb[k] = sb | (rr.x & 0x80000000u);
          s_se[k] = se;
          s_pfx[k] = (nq + 31u) >> 5;
        }
        __syncthreads();
        const uint32_t nchunks = block_exclusive_scan(s_pfx, nb, s_warp);
        const unsigned long long bw = block_sum_u64(myw, s_red);
        work += myw;
        tile_w += bw;
        if (mode < 0) {
          if (wide)
            mode = kWide;
          else if (re - rb > (uint32_t)kRB || 2ull * bw >= span)
            mode = kDense;
          else
            mode = kSparse;
        }
        if (nchunks == 0) continue;
        if (mode == kDense) {
          run_chunks<kDense>(P, cnt, s_sb, s_se, s_pfx, nb, nchunks, lo, tb, tu);
        } else if (mode == kWide) {
          run_chunks<kWide>(P, cnt, s_sb, s_se, s_pfx, nb, nchunks, lo, tb, tu);
        } else {
          run_chunks<kSparse>(P, cnt, s_sb, s_se, s_pfx, nb, nchunks, lo, tb, tu);
          __syncthreads();
          run_chunks<kZero>(P, cnt, s_sb, s_se, s_pfx, nb, nchunks, lo, tb, tu);
        }
        __syncthreads();
      }
      if (tile_w == 0) continue;
      if (mode == kDense) {
        sweep16(cnt, span, tb, tu);
        __syncthreads();
      } else if (mode == kWide) {
        sweep32(cnt, span, tb, tu);
        __syncthreads();
      }
    }
    add128(bal_lo, bal_hi, tb);
    add128(unb_lo, unb_hi, tu);
  }

  // exact 128-bit reduction: warp shuffle, then one pair of global atomics per warp
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    unsigned long long l2 = __shfl_xor_sync(kFull, bal_lo, o), h2 = __shfl_xor_sync(kFull, bal_hi, o);
    unsigned long long l3 = __shfl_xor_sync(kFull, unb_lo, o), h3 = __shfl_xor_sync(kFull, unb_hi, o);
    bal_lo += l2;
    bal_hi += h2 + (bal_lo < l2 ? 1ull : 0ull);
    unb_lo += l3;
    unb_hi += h3 + (unb_lo < l3 ? 1ull : 0ull);
  }
  if (lane == 0) {
    unsigned long long old = atomicAdd(&P.acc[0], bal_lo);
    atomicAdd(&P.acc[1], bal_hi + (old + bal_lo < old ? 1ull : 0ull));
    old = atomicAdd(&P.acc[2], unb_lo);
    atomicAdd(&P.acc[3], unb_hi + (old + unb_lo < old ? 1ull : 0ull));
  }
  const unsigned long long bw = block_sum_u64(work, s_red);
  if (threadIdx.x == 0) P.block_work[blockIdx.x] = bw;
}

int configure(Graph& g, int& cap_words, int& smem_bytes) {
  cudaFuncAttributes fa;
  BBC_CK(cudaFuncGetAttributes(&fa, k_count));
  int avail = g.max_smem - (int)fa.sharedSizeBytes - 3 * kRB * 4 - 64;
  cap_words = (avail / 16) * 4;
  smem_bytes = cap_words * 4 + 3 * kRB * 4 + 16;
  BBC_CK(cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
  return BBC_OK;
}

}  // namespace

int count_graph(Graph& g, const bbc_opts* o, uint64_t out[2], bbc_stats* st) {
  bbc_opts opts{};
  if (o) opts = *o;
  if (opts.algo != BBC_ALGO_GBBC && opts.algo != BBC_ALGO_GBBCPP) {
    set_error("algo must be 0 (G-BBC) or 1 (G-BBC++)");
    return BBC_ERR_ARG;
  }
  if (opts.tile_span < 0 || opts.blocks < 0) {
    set_error("tile_span and blocks must be >= 0");
    return BBC_ERR_ARG;
  }
  int part_count = opts.part_count <= 0 ? 1 : opts.part_count;
  if (opts.part_index < 0 || opts.part_index >= part_count) {
    set_error("part_index must lie in [0, part_count)");
    return BBC_ERR_ARG;
  }
  BBC_CK(cudaSetDevice(g.device));
  int cap_words = 0, smem_bytes = 0;
  int rc = configure(g, cap_words, smem_bytes);
  if (rc) return rc;
  uint32_t span16 = (uint32_t)cap_words - 4u;
  uint32_t span32 = (uint32_t)cap_words / 2u - 4u;
  if (opts.tile_span > 0) {
    span16 = std::min<uint32_t>(span16, (uint32_t)opts.tile_span);
    span32 = std::min<uint32_t>(span32, (uint32_t)opts.tile_span);
  }
  int blocks = opts.blocks > 0 ? opts.blocks : g.num_sms;
  if (blocks > g.block_work_cap) {
    cudaFree(g.block_work);
    g.block_work = nullptr;
    BBC_CK(cudaMalloc(&g.block_work, (size_t)blocks * 8));
    g.block_work_cap = blocks;
  }
  const uint32_t n = (uint32_t)g.n;
  const uint32_t ntasks = n > (uint32_t)opts.part_index ? (n - (uint32_t)opts.part_index + part_count - 1) / part_count : 0u;

  Params P;
  P.adj = g.adj;
  P.rec = g.rec;
  P.aoff = g.aoff;
  P.awork = g.awork;
  P.order = g.order;
  P.n = n;
  P.ntasks = ntasks;
  P.part_index = (uint32_t)opts.part_index;
  P.part_count = (uint32_t)part_count;
  P.span16 = span16;
  P.span32 = span32;
  P.cap_words = (uint32_t)cap_words;
  P.dynamic = opts.algo == BBC_ALGO_GBBCPP;
  P.acc = g.acc;
  P.queue = g.queue;
  P.block_work = g.block_work;

  BBC_CK(cudaMemsetAsync(g.acc, 0, 32, g.stream));
  BBC_CK(cudaMemsetAsync(g.queue, 0, 4, g.stream));
  BBC_CK(cudaEventRecord(g.ev0, g.stream));
  k_count<<<blocks, kCountThreads, smem_bytes, g.stream>>>(P);
  BBC_CK(cudaGetLastError());
  BBC_CK(cudaEventRecord(g.ev1, g.stream));
  unsigned long long h_acc[4];
  BBC_CK(cudaMemcpyAsync(h_acc, g.acc, 32, cudaMemcpyDeviceToHost, g.stream));
  BBC_CK(cudaStreamSynchronize(g.stream));
  g.last_blocks = blocks;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, g.ev0, g.ev1);
  out[0] = h_acc[0];
  out[1] = h_acc[2];
  if (st) {
    unsigned long long* bw = new unsigned long long[blocks];
    cudaMemcpy(bw, g.block_work, (size_t)blocks * 8, cudaMemcpyDeviceToHost);
    unsigned long long w = 0;
    for (int b = 0; b < blocks; ++b) w += bw[b];
    delete[] bw;
    st->wedges = w;
    st->wedges_total = g.w_s;
    st->w_u = g.w_u;
    st->w_v = g.w_v;
    st->balanced_hi = h_acc[1];
    st->unbalanced_hi = h_acc[3];
    st->anchor_side = g.side;
    st->blocks = blocks;
    st->threads = kCountThreads;
    st->tile_span = (int32_t)span16;
    st->tasks = (int32_t)ntasks;
    st->preprocess_ms = g.preprocess_ms;
    st->count_ms = ms;
  }
  if (h_acc[1] || h_acc[3]) {
    set_error("balanced/unbalanced count exceeded 64-bit range");
    return BBC_ERR_OVERFLOW;
  }
  return BBC_OK;
}

}  // namespace bbc
