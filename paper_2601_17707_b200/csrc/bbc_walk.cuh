// Device building blocks shared by the count kernel (bbc_count.cu) and the SURVEY.md 8(f)
// kernels (bbc_ext.cu): streaming loads, rank search, the one-barrier block scan, record
// search, 32-bit shared-memory atomics and the pair-of-groups wedge walker.
#pragma once

#include <stdint.h>

namespace bbc {

constexpr uint32_t kFull = 0xffffffffu;

// Block barrier for code whose warps may reach it diverged.  __syncthreads() is bar.sync,
// i.e. barrier.sync.aligned, which requires every warp to arrive converged; the count
// kernel's warps are routinely split by data-dependent loops (galloping record searches,
// per-lane queue loops) when they reach a barrier, and on config 4 (1 B edges) that broke
// the CTA's barrier pairing (warps walking one round while others set up the next: wrong
// bounds, out-of-range shared-memory atomics; compute-sanitizer synccheck reported
// "divergent thread(s) in warp").  The non-aligned form counts arrivals per thread.
__device__ __forceinline__ void block_sync() { asm volatile("barrier.sync 0;" ::: "memory"); }

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// first position in [lo, hi) whose rank is >= x (lists are rank-sorted)
__device__ __forceinline__ uint32_t lower_bound_rank(const uint32_t* __restrict__ adj, uint32_t lo, uint32_t hi,
                                                     long long x) {
  if (x <= 0) return lo;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if ((long long)(__ldg(adj + mid) & 0x7fffffffu) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// The same when the answer is known to be <= hi and usually close to it (successive round
// boundaries of a record move down its list by a few positions): gallop down from hi,
// then binary-search the last jump.  Typically one or two loads instead of log2(len).
__device__ __forceinline__ uint32_t lower_bound_gallop(const uint32_t* __restrict__ adj, uint32_t lo, uint32_t hi,
                                                       long long x) {
  if (x <= 0) return lo;
  uint32_t b = hi, step = 1;  // invariant: every position in [b, hi) has rank >= x
  while (b > lo) {
    const uint32_t p = b - min(step, b - lo);
    if ((long long)(__ldg(adj + p) & 0x7fffffffu) >= x) {
      b = p;
      step <<= 1;
    } else {
      return lower_bound_rank(adj, p + 1u, b, x);
    }
  }
  return lo;
}

// Block-wide exclusive scan of one u32 per thread fused with a u64 sum, with ONE barrier:
// each warp publishes its totals, then every warp scans the (<= 32) warp totals itself.
// The totals are double-buffered by `buf` (callers alternate it), since consecutive scans
// may have no other barrier between them and a warp can be one scan ahead.
template <int T>
__device__ __forceinline__ uint32_t scan_sum(uint32_t v, unsigned long long w, uint32_t& total,
                                             unsigned long long& wtotal, uint32_t* s_v, unsigned long long* s_w,
                                             uint32_t buf) {
  constexpr int kWarps = T / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(kFull, w, o);
  uint32_t* sv = s_v + (buf & 1u) * 32u;
  unsigned long long* sw = s_w + (buf & 1u) * 32u;
  if (lane == 31) sv[warp] = x;
  if (lane == 0) sw[warp] = w;
  block_sync();
  uint32_t a = lane < kWarps ? sv[lane] : 0u;
  unsigned long long bsum = lane < kWarps ? sw[lane] : 0ull;
#pragma unroll
  for (int o = 1; o < kWarps; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, a, o);
    if (lane >= o) a += y;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) bsum += __shfl_xor_sync(kFull, bsum, o);
  total = __shfl_sync(kFull, a, kWarps - 1);
  wtotal = bsum;
  const uint32_t before = __shfl_sync(kFull, a, (warp + 31) & 31);  // inclusive prefix of warp - 1
  return x - v + (warp > 0 ? before : 0u);
}

// largest k in [0, nb) with pfx[k] <= g
__device__ __forceinline__ int find_record(const uint32_t* pfx, int nb, uint32_t g) {
  int lo = 0, hi = nb;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (pfx[mid] <= g)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// the same for nb <= N (a power of two): fixed-depth, branch-free (no divergence
// between lanes whose searches would take different numbers of steps); pfx[0] = 0 <= g
template <int N>
__device__ __forceinline__ int find_record_fixed(const uint32_t* pfx, int nb, uint32_t g) {
  int k = 0;
#pragma unroll
  for (int s = N / 2; s >= 1; s >>= 1) {
    const int c = k + s;
    if (c < nb && pfx[c] <= g) k = c;
  }
  return k;
}

// ---- shared-memory primitives on 32-bit shared addresses ------------------------------
// (generic pointers make the compiler re-derive the shared window base per access)
// (the move is opaque to the compiler, so a base address stays in one register instead of
// being re-derived from the CTA's shared window before every atomic)
__device__ __forceinline__ uint32_t sptr(const void* p) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t s_atom_add(uint32_t a, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ uint32_t s_atom_or(uint32_t a, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ void s_red_add(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void s_st(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// C(c, j) exactly, ~0 (an overflow marker) from 2^64 - 1 on
__device__ __forceinline__ unsigned long long binom_sat(unsigned long long c, uint32_t j) {
  if ((unsigned long long)j > c) return 0ull;
  if ((unsigned long long)j > c - j) j = (uint32_t)(c - j);
  unsigned __int128 r = 1;
  for (uint32_t i = 1; i <= j; ++i) {
    r = r * (unsigned __int128)(c - j + i) / i;
    if (r >> 64) return ~0ull;
  }
  return r == (unsigned __int128)~0ull ? ~0ull : (unsigned long long)r;
}

// C(c, k) with closed forms for k = 1, 2, 3 (exact below 2^21 for k = 3)
__device__ __forceinline__ unsigned long long binom_k(unsigned long long c, uint32_t k) {
  if (c < k) return 0ull;
  if (k == 1u) return c;
  if (k == 2u) return (c * (c - 1ull)) >> 1;
  if (k == 3u && c < (1ull << 21)) return c * (c - 1ull) * (c - 2ull) / 6ull;
  return binom_sat(c, k);
}

// 128-bit accumulation (lo, hi) of a binom_k value; the overflow marker adds 2^64, so any
// total that passed 2^64 - 1 shows in the high word
__device__ __forceinline__ void add_k(unsigned long long& lo, unsigned long long& hi, unsigned long long x) {
  if (x == ~0ull) {
    hi += 1ull;
    return;
  }
  lo += x;
  hi += (lo < x) ? 1ull : 0ull;
}

// 256-bit streaming load (sm_100: LDG.E.NA.ENL2.256), no L1 allocation
__device__ __forceinline__ void ld_stream8(const uint32_t* p, uint32_t (&r)[8]) {
  // not volatile: a pure load of read-only data, free to be scheduled early
  asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}

// default chunk handler: op.wedge(word, sign, slot) for every valid slot
template <class Op>
__device__ __forceinline__ void chunk_by_wedge(Op& op, const uint32_t (&wv)[8], uint32_t sg, uint32_t m) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (m & (1u << j)) op.wedge(wv[j], sg, j);
}

// The walk unit: an aligned 32-byte chunk of 8 adjacency words.  A sub-slice [lo, hi)
// covers chunks lo / 8 .. (hi - 1) / 8.  (adj is 256-byte aligned and padded by 8 words.)
__device__ __forceinline__ uint32_t unit_count(uint32_t lo, uint32_t hi) { return ((hi + 7u) >> 3) - (lo >> 3); }

// valid slots (bits 0..7) of the chunk starting at word position p0 for [lo, hi)
__device__ __forceinline__ uint32_t slot_mask8(uint32_t p0, uint32_t lo, uint32_t hi) {
  const int a = max((int)(lo - p0), 0);
  const int b = min((int)(hi - p0), 8);
  return b <= a ? 0u : (((1u << b) - 1u) & (0xffu << a));
}

// Walk the 32-byte chunks of the round's sub-slices, one chunk (8 wedges) per thread per
// iteration.  Interleaved order (default, the fast path's short rounds): one fixed-depth
// record search and one 256-bit load per chunk; consecutive threads take consecutive
// chunks of a record (a warp reads 1 KB contiguous).  BLOCKED order (the general path's
// long sub-slices): each thread takes a contiguous run of chunks.
// op.chunk(words, sign, valid-slot mask) handles the chunk (ops that can are branch-free:
// an invalid slot becomes a no-op atomic on a dummy word, so all eight shared-memory
// atomics issue back to back); op.flush() after each chunk.
template <int T, bool BLOCKED = false, class Op>
__device__ __forceinline__ void walk_chunks(const uint32_t* adj, const uint32_t* s_lo, const uint32_t* s_hi,
                                            const uint32_t* s_pfx, int nb, uint32_t nunits, Op& op) {
  if (BLOCKED) {
    // blocked distribution (general path: batches of up to T records, long sub-slices):
    // thread t takes the contiguous chunks [t * per, (t + 1) * per), so its record changes
    // only at record boundaries -- one record search per thread, then a compare per chunk
    // (measured: config 5 218 -> 206 ms; on the fast path's short rounds the interleaved
    // order below is faster, config 2 12.9 vs 14.6 ms)
    const uint32_t per = (nunits + T - 1u) / (uint32_t)T;
    uint32_t g = threadIdx.x * per;
    const uint32_t g1 = min(g + per, nunits);
    if (g >= g1) return;
    int k = find_record(s_pfx, nb, g);
    uint32_t nxt = k + 1 < nb ? s_pfx[k + 1] : 0xffffffffu;
    uint32_t lx = s_lo[k], hi = s_hi[k], base = s_pfx[k];
    for (; g < g1; ++g) {
      if (g >= nxt) {
        do {
          ++k;
          nxt = k + 1 < nb ? s_pfx[k + 1] : 0xffffffffu;
        } while (g >= nxt);
        lx = s_lo[k];
        hi = s_hi[k];
        base = s_pfx[k];
      }
      const uint32_t lo = lx & 0x7fffffffu, sg = lx & 0x80000000u;
      const uint32_t p0 = ((lo >> 3) + (g - base)) << 3;
      uint32_t wv[8];
      ld_stream8(adj + p0, wv);
      const uint32_t m = slot_mask8(p0, lo, hi);
      op.chunk(wv, sg, m);
      op.flush();
    }
  } else {
    for (uint32_t g = threadIdx.x; g < nunits; g += T) {
      // search depth by the batch's record count (block-uniform branch): most anchors have
      // few records
      const int k = nb <= 32 ? find_record_fixed<32>(s_pfx, nb, g)
                             : (nb <= 64 || T <= 64 ? find_record_fixed<(T < 64 ? T : 64)>(s_pfx, nb, g)
                                                    : find_record_fixed<T>(s_pfx, nb, g));
      const uint32_t lx = s_lo[k], hi = s_hi[k];
      const uint32_t lo = lx & 0x7fffffffu, sg = lx & 0x80000000u;
      const uint32_t p0 = ((lo >> 3) + (g - s_pfx[k])) << 3;
      uint32_t wv[8];
      ld_stream8(adj + p0, wv);
      const uint32_t m = slot_mask8(p0, lo, hi);
      op.chunk(wv, sg, m);
      op.flush();
    }
  }
}

}  // namespace bbc
