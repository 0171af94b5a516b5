// SURVEY.md 8(f) row 1 on the same device CSR as the count kernel: six-way butterfly
// classification -- reference oracle.classify_butterflies (pkg/src/bbcount/oracle.py:
// 172-197, ButterflyClassCounts :31-64).  Anchors are U vertices, centres V (the classes
// are not side-symmetric, oracle.py:176-178), so the graph must be built with BBC_SIDE_U.
// For every anchor pair (u, w) the wedges through the common centres c split into pp (both
// edges +), mm (both -) and pm (signs differ); the classes are C(pp,2), pp*mm, C(mm,2),
// C(pm,2), pp*pm, mm*pm.  (Row 2, (2,k)-bicliques, runs in the count kernel itself with
// C(., k) closings: bbc_count.cu.)
//
// Structure (one CTA per anchor, persistent CTAs over the G-BBC++ queue or static
// round-robin): the anchor's end-vertex ranks are cut into bands from the top (one band
// table column per band when the table exists); per band and per batch of <= T records,
// each record's admitted sub-slice comes from the table or a galloping search, a block
// scan lays the 32-byte chunks out and the chunk walker (bbc_walk.cuh) increments a
// shared-memory counter per end vertex:
//   C10: pp | mm << 10 | pm << 20 (deg u <= 1023), closed inline from the atomic's return
//        value (adding a pp wedge to (a, b, d) adds a to C(pp,2), b to pp*mm and d to
//        pp*pm, likewise for mm and pm), or -- dense bands -- by no-return increments and
//        a sweep;
//   C32 (deg u > 1023): three words, no-return increments and a closing sweep.
// Totals are exact 128-bit per thread, reduced with one pair of atomics per warp.
#include <cstring>

#include "bbc_internal.cuh"
#include "bbc_walk.cuh"

namespace bbc {

namespace {

enum ExtMode { kClassify = 0 };

struct ExtParams {
  const uint32_t* __restrict__ adj;
  const uint2* __restrict__ rec;
  const uint32_t* __restrict__ coff;
  const uint32_t* __restrict__ aoff;
  const unsigned long long* __restrict__ awork;
  const uint32_t* __restrict__ order;
  const uint32_t* __restrict__ bnd;   // band table (nullptr: searches only)
  const uint32_t* __restrict__ brow;
  uint32_t nbands, t16;
  uint32_t hash_target;  // wedges per hash round over sparse column ranges (0: bands only)
  uint32_t n, ntasks, part_index, part_count;
  uint32_t cap_words;
  int dynamic;
  unsigned long long* acc;  // 6 x (lo, hi) + [12] overflow flag
  unsigned int* queue;
  unsigned long long* block_work;
};

__device__ __forceinline__ void add128(unsigned long long& lo, unsigned long long& hi, unsigned long long x) {
  lo += x;
  hi += (lo < x) ? 1ull : 0ull;
}

// wedge class: 0 pp, 1 mm, 2 pm (sg = s(u, c) in bit 31, word bit 31 = s(c, w))
__device__ __forceinline__ uint32_t wedge_class(uint32_t w, uint32_t sg) {
  return ((w ^ sg) >> 31) ? 2u : (sg >> 31);
}

// the inline closing of one wedge of class t on an end vertex that held (a, b, d):
// C(t,t) += own count, (t, t') += the other counts -- branch-free (selects)
__device__ __forceinline__ void add_class(uint32_t t, uint32_t a, uint32_t b, uint32_t d, unsigned long long& c0,
                                          unsigned long long& c1, unsigned long long& c2, unsigned long long& c3,
                                          unsigned long long& c4, unsigned long long& c5) {
  const bool p = t == 0u, m = t == 1u, x = t == 2u;
  c0 += p ? a : 0u;
  c2 += m ? b : 0u;
  c3 += x ? d : 0u;
  c1 += p ? b : (m ? a : 0u);
  c4 += p ? d : (x ? a : 0u);
  c5 += m ? d : (x ? b : 0u);
}

// classification, pp | mm << 10 | pm << 20 per end vertex (deg u <= 1023)
struct OpClsC10 {
  uint32_t rb;
  unsigned long long c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0;
  __device__ __forceinline__ void wedge(uint32_t w, uint32_t sg, int) {
    const uint32_t t = wedge_class(w, sg);
    const uint32_t old = s_atom_add(rb + (w << 2), 1u << (10u * t));
    const uint32_t a = old & 1023u, b = (old >> 10) & 1023u, d = old >> 20;
    add_class(t, a, b, d, c0, c1, c2, c3, c4, c5);
  }
  __device__ __forceinline__ void chunk(const uint32_t (&wv)[8], uint32_t sg, uint32_t m) {
    chunk_by_wedge(*this, wv, sg, m);
  }
  __device__ __forceinline__ void flush() {}
};

// dense packed bands (>= 2 wedges per counter word): no-return increments of
// pp | mm << 10 | pm << 20, closed by the sweep
struct OpPackedDense {
  uint32_t rb;
  __device__ __forceinline__ void wedge(uint32_t w, uint32_t sg, int) {
    s_red_add(rb + (w << 2), 1u << (10u * wedge_class(w, sg)));
  }
  __device__ __forceinline__ void chunk(const uint32_t (&wv)[8], uint32_t sg, uint32_t m) {
    chunk_by_wedge(*this, wv, sg, m);
  }
  __device__ __forceinline__ void flush() {}
};

// classification, three u32 words per end vertex, closed by the sweep; rb rebased by
// lo_rank * 12
struct OpClsC32 {
  uint32_t rb;
  __device__ __forceinline__ void wedge(uint32_t w, uint32_t sg, int) {
    s_red_add(rb + (w & 0x7fffffffu) * 12u + 4u * wedge_class(w, sg), 1u);
  }
  __device__ __forceinline__ void chunk(const uint32_t (&wv)[8], uint32_t sg, uint32_t m) {
    chunk_by_wedge(*this, wv, sg, m);
  }
  __device__ __forceinline__ void flush() {}
};

// sparse column ranges: a linear-probing hash of K slots, key = rank + 1 in word 2h,
// packed pp | mm << 10 | pm << 20 counts in word 2h + 1, closed inline from the add's
// return value like OpClsC10 (a round's wedge count is known before its walk and kept
// at or below K / 2, so the table never fills)
struct OpClsHash {
  uint32_t* tab;
  uint32_t K;
  unsigned long long c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0;
  __device__ __forceinline__ void wedge(uint32_t w, uint32_t sg, int) {
    const uint32_t t = wedge_class(w, sg);
    const uint32_t key = (w & 0x7fffffffu) + 1u;
    uint32_t h = (uint32_t)(((unsigned long long)(key * 0x9E3779B1u) * K) >> 32);
    for (;;) {
      const uint32_t k = atomicCAS(&tab[2u * h], 0u, key);
      if (k == 0u || k == key) break;
      h = (h + 1u == K) ? 0u : h + 1u;
    }
    const uint32_t old = atomicAdd(&tab[2u * h + 1u], 1u << (10u * t));
    const uint32_t a = old & 1023u, b = (old >> 10) & 1023u, d = old >> 20;
    add_class(t, a, b, d, c0, c1, c2, c3, c4, c5);
  }
  __device__ __forceinline__ void chunk(const uint32_t (&wv)[8], uint32_t sg, uint32_t m) {
    chunk_by_wedge(*this, wv, sg, m);
  }
  __device__ __forceinline__ void flush() {}
};

struct ExtSmem {
  uint32_t* cnt;
  uint32_t *lo, *hi, *pfx;
  uint32_t* v;
  unsigned long long* w;
};

// One anchor: bands from the top, record batches of T.  Packed layouts use table-column
// bands when the band table exists (bounds from the table, or a galloping search from the
// previous band's bound).  A band holding >= 2 wedges per counter word (estimated from its
// first batch) is counted with no-return increments and swept, others close inline from
// the atomics' return values and are cleared with vector stores.  For single-batch anchors
// the bands after the first (the high-degree end vertices) are widened adaptively to hold
// about K / 2 wedges in a shared-memory hash (OpClsHash): few rounds over sparse ranges.
template <int T, int MODE>
__device__ void ext_anchor(const ExtParams& P, const ExtSmem& S, uint32_t r, uint32_t rb, uint32_t re,
                           unsigned long long w_a, unsigned long long (&acc)[12], uint32_t& ovf,
                           unsigned long long& work) {
  const uint32_t deg = re - rb;
  const bool wide = deg > 1023u;
  const uint32_t wpv = wide ? 3u : 1u;  // words per end vertex
  const bool cols = !wide && P.bnd != nullptr && P.t16 > 0u && P.t16 <= P.cap_words;
  const uint32_t span = cols ? P.t16 : P.cap_words / wpv;
  const uint32_t nbands = (P.n - 1u - r) / span + 1u;  // unit bands 0..nbands-1 hold ranks > r
  const uint32_t nbatch = (deg + T - 1u) / (uint32_t)T;
  const bool single = nbatch == 1u;
  const bool hashing = cols && single && P.hash_target > 0u;
  const uint32_t K = (P.cap_words / 2u) & ~3u, target = min(P.hash_target, K / 2u);
  const uint32_t base = sptr(S.cnt);
  uint32_t scan_buf = 0;
  uint32_t carry = 0;  // single batch: this record's upper bound for the next band
  uint32_t width = 1;  // unit bands per band (hash rounds)
  unsigned long long part[6] = {0, 0, 0, 0, 0, 0};
  for (uint32_t b = 0; b < nbands;) {
    const uint32_t nbw = (hashing && b > 0) ? min(width, nbands - b) : 1u;
    const long long top = (long long)P.n - (long long)b * span;
    const long long bot = top - (long long)nbw * span;
    const uint32_t lo_rank = bot > 0 ? (uint32_t)bot : 0u;
    const uint32_t band_words = (uint32_t)(top - (long long)lo_rank) * wpv;
    unsigned long long band_w = 0;
    int dense = -1;
    bool redo = false, hashed = false;
    for (uint32_t b0 = rb; b0 < re; b0 += T) {
      const int nb = (int)min((uint32_t)T, re - b0);
      uint32_t ng = 0;
      unsigned long long myw = 0;
      uint32_t nlo = 0;
      if ((int)threadIdx.x < nb) {
        const uint2 rr = P.rec[b0 + threadIdx.x];
        const uint32_t begin = rr.x & 0x7fffffffu;
        const uint32_t bi = cols ? __ldg(P.brow + rr.y) : 0xffffffffu;
        uint32_t hi, lo;
        if (bi != 0xffffffffu) {
          const uint32_t* row = P.bnd + (size_t)bi * P.nbands;
          hi = __ldg(row + b);
          lo = b + nbw < P.nbands ? __ldg(row + b + nbw) : 0u;
        } else {
          if (b == 0)
            hi = __ldg(P.coff + rr.y + 1);
          else if (single)
            hi = carry;
          else
            hi = lower_bound_rank(P.adj, begin, __ldg(P.coff + rr.y + 1), top);
          lo = single ? lower_bound_gallop(P.adj, begin, hi, bot) : lower_bound_rank(P.adj, begin, hi, bot);
        }
        lo = max(lo, begin);
        hi = max(hi, lo);
        nlo = lo;
        if (hi > lo) {
          ng = unit_count(lo, hi);
          myw = hi - lo;
        }
        S.lo[threadIdx.x] = lo | (rr.x & 0x80000000u);
        S.hi[threadIdx.x] = hi;
      }
      uint32_t ngroups;
      unsigned long long bw;
      const uint32_t ex = scan_sum<T>(ng, myw, ngroups, bw, S.v, S.w, scan_buf++);
      if ((int)threadIdx.x < nb) S.pfx[threadIdx.x] = ex;
      block_sync();
      if (hashing && b > 0 && bw > target && nbw > 1u) {  // too many wedges: narrower, no walk
        width = max(1u, min(nbw / 2u, (uint32_t)((unsigned long long)nbw * target / bw)));
        redo = true;
        break;  // (single batch: the record arrays are not reused before the next scan)
      }
      carry = nlo;
      work += myw;
      band_w += bw;
      if (hashing && b > 0 && bw <= target) {
        hashed = true;
        if (ngroups) {
          OpClsHash op;
          op.tab = S.cnt;
          op.K = K;
          walk_chunks<T>(P.adj, S.lo, S.hi, S.pfx, nb, ngroups, op);
          part[0] += op.c0;
          part[1] += op.c1;
          part[2] += op.c2;
          part[3] += op.c3;
          part[4] += op.c4;
          part[5] += op.c5;
        }
        if (2ull * bw < target) width = min(2u * width, nbands);
        block_sync();
        break;
      }
      if (dense < 0) dense = wide || bw * nbatch >= 2ull * band_words;
      if (ngroups) {
        if (dense && !wide) {
          OpPackedDense op{base - (lo_rank << 2)};
          walk_chunks<T>(P.adj, S.lo, S.hi, S.pfx, nb, ngroups, op);
        } else if (!wide) {
          OpClsC10 op;
          op.rb = base - (lo_rank << 2);
          walk_chunks<T>(P.adj, S.lo, S.hi, S.pfx, nb, ngroups, op);
          part[0] += op.c0;
          part[1] += op.c1;
          part[2] += op.c2;
          part[3] += op.c3;
          part[4] += op.c4;
          part[5] += op.c5;
        } else {
          OpClsC32 op{base - lo_rank * 12u};
          walk_chunks<T>(P.adj, S.lo, S.hi, S.pfx, nb, ngroups, op);
        }
      }
      block_sync();  // the next batch overwrites the record arrays
    }
    if (redo) {
      block_sync();  // every warp is done with this set-up's record arrays
      continue;
    }
    if (b == 0u && hashing && nbands > 1u) {
      // first hash-round width from the remaining wedges' average density (instead of
      // doubling up from one column)
      const unsigned long long rest = w_a > band_w ? w_a - band_w : 0ull, span_c = nbands - 1u;
      width = (uint32_t)max(1ull, min(span_c, (unsigned long long)target * span_c / max(rest, 1ull)));
    }
    b += nbw;
    if (band_w == 0ull) continue;
    uint4* c4 = reinterpret_cast<uint4*>(S.cnt);
    if (hashed) {
#pragma unroll 4
      for (uint32_t i = threadIdx.x; i < K / 2u; i += T) c4[i] = make_uint4(0u, 0u, 0u, 0u);
      block_sync();
      continue;
    }
    const uint32_t nq = (band_words + 3u) / 4u;
    if (dense) {
      if (wide) {
        // closing sweep over (pp, mm, pm) triples
        for (uint32_t i = threadIdx.x; i < (band_words / 3u); i += T) {
          const unsigned long long a = S.cnt[3u * i], bb = S.cnt[3u * i + 1u], d = S.cnt[3u * i + 2u];
          part[0] += a * (a - (a > 0)) / 2;
          part[1] += a * bb;
          part[2] += bb * (bb - (bb > 0)) / 2;
          part[3] += d * (d - (d > 0)) / 2;
          part[4] += a * d;
          part[5] += bb * d;
        }
      } else {
        for (uint32_t i = threadIdx.x; i < band_words; i += T) {
          const uint32_t x = S.cnt[i];
          if (x == 0u) continue;
          const unsigned long long a = x & 1023u, bb = (x >> 10) & 1023u, d = x >> 20;
          part[0] += a * (a - (a > 0)) / 2;
          part[1] += a * bb;
          part[2] += bb * (bb - (bb > 0)) / 2;
          part[3] += d * (d - (d > 0)) / 2;
          part[4] += a * d;
          part[5] += bb * d;
        }
      }
      block_sync();
    }
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < nq; i += T) c4[i] = make_uint4(0u, 0u, 0u, 0u);
    block_sync();
  }
  for (int i = 0; i < 6; ++i) add128(acc[2 * i], acc[2 * i + 1], part[i]);
}

template <int T, int MINB, int MODE>
__global__ void __launch_bounds__(T, MINB) k_ext(ExtParams P) {
  extern __shared__ uint4 smem4[];
  __shared__ uint32_t s_v[64];
  __shared__ unsigned long long s_w[64];
  __shared__ uint32_t s_task;
  __shared__ uint32_t s_ovf;
  ExtSmem S;
  S.cnt = reinterpret_cast<uint32_t*>(smem4);
  S.lo = S.cnt + P.cap_words;
  S.hi = S.lo + T;
  S.pfx = S.hi + T;
  S.v = s_v;
  S.w = s_w;
  for (uint32_t i = threadIdx.x; i < P.cap_words / 4; i += T) smem4[i] = make_uint4(0u, 0u, 0u, 0u);
  if (threadIdx.x == 0) s_ovf = 0u;

  unsigned long long acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long work = 0;
  uint32_t ovf = 0;
  uint32_t next = blockIdx.x;
  if (threadIdx.x == 0) s_task = P.dynamic ? atomicAdd(P.queue, 1u) : next;
  block_sync();
  for (;;) {
    const uint32_t t = s_task;
    next += gridDim.x;
    block_sync();
    if (t >= P.ntasks) break;
    if (threadIdx.x == 0) s_task = P.dynamic ? atomicAdd(P.queue, 1u) : next;
    const uint32_t gidx = P.part_index + t * P.part_count;
    const uint32_t r = P.dynamic ? P.order[gidx] : gidx;
    const unsigned long long w_a = P.awork[r];
    if (w_a != 0ull) ext_anchor<T, MODE>(P, S, r, P.aoff[r], P.aoff[r + 1], w_a, acc, ovf, work);
    block_sync();
  }
  // exact reduction: warp shuffle of the 128-bit values, one pair of atomics per warp
  const int lane = threadIdx.x & 31;
  constexpr int kVals = 6;
#pragma unroll
  for (int i = 0; i < kVals; ++i) {
    unsigned long long lo = acc[2 * i], hi = acc[2 * i + 1];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long l2 = __shfl_xor_sync(kFull, lo, o), h2 = __shfl_xor_sync(kFull, hi, o);
      lo += l2;
      hi += h2 + (lo < l2 ? 1ull : 0ull);
    }
    if (lane == 0) {
      const unsigned long long old = atomicAdd(&P.acc[2 * i], lo);
      atomicAdd(&P.acc[2 * i + 1], hi + (old + lo < old ? 1ull : 0ull));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) work += __shfl_xor_sync(kFull, work, o);
  if (ovf) atomicOr(&s_ovf, 1u);
  if (lane == 0) s_w[threadIdx.x >> 5] = work;
  block_sync();
  if (threadIdx.x == 0) {
    unsigned long long tw = 0;
    for (int w = 0; w < T / 32; ++w) tw += s_w[w];
    P.block_work[blockIdx.x] = tw;
    if (s_ovf) atomicOr(&P.acc[12], 1ull);
  }
}

template <int MODE>
int ext_launch(Graph& g, const bbc_opts& opts, uint32_t k, unsigned long long* h_acc, float* ms, int* blocks_out) {
  constexpr int T = 128, MINB = 8;
  cudaFuncAttributes fa;
  BBC_CK(cudaFuncGetAttributes(&fa, k_ext<T, MINB, MODE>));
  int per_sm = 0;
  BBC_CK(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, g.device));
  const int budget = std::min(g.max_smem, per_sm / MINB - 1024);
  const int avail = budget - (int)fa.sharedSizeBytes - (3 * T * 4 + 64);
  const int cap_words = (avail / 16) * 4;  // as the count kernel: the band table columns fit
  const int smem_bytes = cap_words * 4 + 3 * T * 4 + 16;
  BBC_CK(cudaFuncSetAttribute(k_ext<T, MINB, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
  const int blocks = opts.blocks > 0 ? opts.blocks : g.num_sms * MINB;
  if (blocks > g.block_work_cap) {
    cudaFree(g.block_work);
    g.block_work = nullptr;
    BBC_CK(cudaMalloc(&g.block_work, (size_t)blocks * 16));
    g.block_work_cap = blocks;
  }
  const int part_count = opts.part_count <= 0 ? 1 : opts.part_count;
  const uint32_t n = (uint32_t)g.n;
  ExtParams P;
  P.adj = g.adj;
  P.rec = g.rec;
  P.coff = g.coff;
  P.aoff = g.aoff;
  P.awork = g.awork;
  P.order = g.order;
  P.bnd = (opts.flags & 1024) ? nullptr : g.bnd;  // flags bit 10: searches only (tests)
  P.brow = g.brow;
  P.nbands = g.nbands;
  P.t16 = g.t16;
  P.hash_target = (opts.flags & 2) ? 0u : 1024u;  // flags bit 1: table-column bands only
  P.n = n;
  P.ntasks = n > (uint32_t)opts.part_index ? (n - (uint32_t)opts.part_index + part_count - 1) / part_count : 0u;
  P.part_index = (uint32_t)opts.part_index;
  P.part_count = (uint32_t)part_count;
  P.cap_words = (uint32_t)cap_words;
  P.dynamic = opts.algo == BBC_ALGO_GBBCPP;
  P.acc = g.acc;
  P.queue = g.queue;
  P.block_work = g.block_work;
  BBC_CK(cudaMemsetAsync(g.acc, 0, 128, g.stream));
  BBC_CK(cudaMemsetAsync(g.queue, 0, 8, g.stream));
  BBC_CK(cudaEventRecord(g.ev0, g.stream));
  if (n > 0) {
    k_ext<T, MINB, MODE><<<blocks, T, smem_bytes, g.stream>>>(P);
    BBC_CK(cudaGetLastError());
  }
  BBC_CK(cudaEventRecord(g.ev1, g.stream));
  BBC_CK(cudaMemcpyAsync(h_acc, g.acc, 13 * 8, cudaMemcpyDeviceToHost, g.stream));
  BBC_CK(cudaStreamSynchronize(g.stream));
  cudaEventElapsedTime(ms, g.ev0, g.ev1);
  g.last_blocks = blocks;
  *blocks_out = blocks;
  return BBC_OK;
}

int ext_check_opts(const bbc_opts& opts) {
  if (opts.algo != BBC_ALGO_GBBC && opts.algo != BBC_ALGO_GBBCPP) {
    set_error("algo must be 0 (G-BBC) or 1 (G-BBC++)");
    return BBC_ERR_ARG;
  }
  const int part_count = opts.part_count <= 0 ? 1 : opts.part_count;
  if (opts.blocks < 0 || opts.part_index < 0 || opts.part_index >= part_count) {
    set_error("blocks must be >= 0 and part_index in [0, part_count)");
    return BBC_ERR_ARG;
  }
  return BBC_OK;
}

void ext_stats(Graph& g, bbc_stats* st, int blocks, float ms) {
  if (!st) return;
  std::memset(st, 0, sizeof(*st));
  unsigned long long* bw = new unsigned long long[blocks];
  cudaMemcpy(bw, g.block_work, (size_t)blocks * 8, cudaMemcpyDeviceToHost);
  unsigned long long w = 0;
  for (int b = 0; b < blocks; ++b) w += bw[b];
  delete[] bw;
  st->wedges = w;
  st->wedges_total = g.w_s;
  st->w_u = g.w_u;
  st->w_v = g.w_v;
  st->anchor_side = g.side;
  st->blocks = blocks;
  st->threads = 128;
  st->tasks = (int32_t)g.n;
  st->preprocess_ms = g.preprocess_ms;
  st->count_ms = ms;
}

}  // namespace

int classify_graph(Graph& g, const bbc_opts* o, uint64_t out[12], bbc_stats* st) {
  bbc_opts opts{};
  if (o) opts = *o;
  if (int rc = ext_check_opts(opts)) return rc;
  if (g.side != 0) {
    set_error("classification anchors U-pairs over V-centres (oracle.py:176-178): build the graph with BBC_SIDE_U");
    return BBC_ERR_ARG;
  }
  BBC_CK(cudaSetDevice(g.device));
  unsigned long long h[13];
  float ms = 0.f;
  int blocks = 0;
  if (int rc = ext_launch<kClassify>(g, opts, 2u, h, &ms, &blocks)) return rc;
  for (int i = 0; i < 12; ++i) out[i] = h[i];
  ext_stats(g, st, blocks, ms);
  return BBC_OK;
}

}  // namespace bbc
