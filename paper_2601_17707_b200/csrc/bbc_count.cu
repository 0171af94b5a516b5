// Wedge-enumeration + closing kernel (G-BBC static / G-BBC++ dynamic).
//
// Reference mechanisms restated (paths under /root/reference):
//   pkg/src/bbcount/buckets.py:166-197   per-anchor wedge buckets, filter, closing
//   pkg/src/bbcount/tiled.py:107-168     G-BBC: static round-robin blocks, end-vertex
//                                        tiles of bounded span (TileConfig.tile_size)
//   pkg/src/bbcount/tiled.py:182-292     G-BBC++: work-sorted tasks claimed from a
//                                        shared counter by persistent workers
//   PAPER.md:873-912 (Alg. 3), 1190-1253 (Alg. 4)
//
// One CTA processes one anchor (start vertex) u at a time; several CTAs share an SM so
// one anchor's barrier and load latency is covered by the others.  The wedges
// u -> c -> w (rank(w) > rank(u)) are the admitted suffixes of the centres' rank-sorted
// lists.  The end-vertex rank range is cut into bands of S ranks counted from the top
// (band b = [n - (b+1) S, n - b S)), so the heavy high-degree end vertices share band 0.
// Per band a shared-memory tile holds one packed counter per end vertex:
//   W8  (deg u <= 255):   u8 positive | u8 negative, two end vertices per u32 word
//   W16 (deg u <= 65535): u16 positive | u16 negative, one end vertex per word
//   W32 (larger):         separate u32 positive / negative words
// (a pair (u, w) has at most deg u common centres, so the halves never carry).  Each
// wedge adds 1 to the positive or negative half, parity = sign bit of (word ^ s(u,c)).
// A band is closed either by a sweep (balanced += C(p,2)+C(q,2), unbalanced += p*q,
// counter := 0) when it holds at least as many wedges as counter words, or -- the usual
// case -- inline from the atomic's return value (a + wedge adds the old positive count
// to balanced and the old negative count to unbalanced, a - wedge the reverse; summed
// over all increments this is exactly the sweep) followed by zeroing the touched words.
// Sub-slices of each record within a band come from the band table (one load per edge
// of the band) or, without a table, from a binary search.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "bbc_internal.cuh"
#include "bbc_walk.cuh"

namespace bbc {

namespace {


enum Mode { kDense = 0, kSparse = 1 };

struct Params {
  const uint32_t* __restrict__ adj;
  const uint2* __restrict__ rec;
  const uint32_t* __restrict__ coff;
  const uint32_t* __restrict__ aoff;
  const unsigned long long* __restrict__ awork;
  const uint32_t* __restrict__ order;
  const uint32_t* __restrict__ bnd;   // nullptr: binary search
  const uint32_t* __restrict__ brow;  // row of each centre in bnd (~0: binary search)
  uint32_t nbands;
  uint32_t n;
  uint32_t ntasks;
  uint32_t part_index;
  uint32_t part_count;
  uint32_t span8;   // band spans (end vertices per band) of the three layouts; with a
  uint32_t span16;  // band table, span16 == table granularity and span8 == 2 * span16
  uint32_t span32;
  uint32_t cap_words;
  int fast;         // 0: always the general banded path (flags bit 0)
  uint32_t hash_thr;  // cold range in key-hash rounds when bitmap rounds would average fewer wedges
  uint32_t t16;     // band-table granularity (ranks per column)
  uint32_t bcols8;  // this launch's tile band in table columns (W8 / W16 layouts)
  uint32_t bcols16;
  int phase;        // 0: every band; 1: hub band only; 2: cold range only
  uint32_t bm_cols;    // cold seen-bitmap round width in table columns (0: off)
  uint32_t bm_words;   // bitmap words of the widest round
  uint32_t bm_cols0;   // first bitmap round width in table columns
  uint32_t rep_slots;  // repeat-queue entries left by the widest bitmap round
  uint32_t bits_thr;   // cold range in bitmap rounds when tile rounds would average fewer wedges
  uint32_t sweep_min;  // tile rounds with >= sweep_min wedges per counter word close by sweep
  uint32_t fast_max;  // largest degree on the fast path (same for every launch of a count)
  int debug;        // flags bits 2 / 3: skip band 0 / skip the cold range (timing only)
  uint32_t k;       // (2,k)-bicliques (k > 2: the KG kernel); 2 = balanced / unbalanced
  int dynamic;
  unsigned long long* acc;
  unsigned int* queue;
  unsigned long long* block_work;
  unsigned long long* block_busy;  // per-CTA busy time (ns), accumulated like block_work
};

// The tile / bitmap ops address their words from a REBASED shared address: rb = base -
// (lo_rank / ranks-per-word) * 4 (mod 2^32), so a wedge's word is rb + (rank / per-word) * 4
// with no subtraction; lo_rank is aligned to the ranks per word (tiles are sized with the
// slack).  Ranks are < 2^30 on the fast path, so (w >> s) keeps no sign bit after masking.

// counter-tile increments without return (closed later by the sweep)
template <int W, bool BF = false>
struct OpTileDense {
  uint32_t rb;
  uint32_t dummy;  // a tile word of this lane (BF chunks add 0 to it)
  __device__ __forceinline__ void wedge(uint32_t w, uint32_t sg, int) {
    const uint32_t v = w ^ sg;  // bit 31: parity (1 = negative wedge)
#ifdef BBC_MATCH
    // north_star (2) match aggregation (experiment): lanes incrementing the same
    // counter byte combine, the lowest one adds the group's size
    if (W == 8) {
      const uint32_t sh = ((w & 1u) << 4) | ((v >> 28) & 8u);
      const uint32_t a = rb + ((w << 1) & 0xfffffffcu);
      const uint32_t peers = __match_any_sync(__activemask(), (a << 3) | (sh >> 3));
      if ((threadIdx.x & 31u) == (uint32_t)(__ffs(peers) - 1)) s_red_add(a, (uint32_t)__popc(peers) << sh);
      return;
    }
#endif
    if (W == 8)
      s_red_add(rb + ((w << 1) & 0xfffffffcu), 1u << (((w & 1u) << 4) | ((v >> 28) & 8u)));
    else
      s_red_add(rb + ((w << 2) & 0xfffffffcu), 1u << ((v >> 27) & 16u));
  }
  // BF (the fast path's dense tile rounds): branch-free chunk -- an invalid slot adds 0 to
  // this lane's own tile word (a no-op; per-lane words, so the no-ops do not serialise on
  // one address) and the eight adds issue back to back.  Measured: config 2 12.78 ->
  // 12.58 ms; on the general path's dense W16 bands (config 5) the branchy form is faster
  // (206 vs 229 ms).
  __device__ __forceinline__ void chunk(const uint32_t (&wv)[8], uint32_t sg, uint32_t m) {
    if (!BF) {
      chunk_by_wedge(*this, wv, sg, m);
      return;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t w = wv[j], v = w ^ sg;
      const bool ok = (m >> j) & 1u;
      uint32_t a, inc;
      if (W == 8) {
        a = rb + ((w << 1) & 0xfffffffcu);
        inc = 1u << (((w & 1u) << 4) | ((v >> 28) & 8u));
      } else {
        a = rb + ((w << 2) & 0xfffffffcu);
        inc = 1u << ((v >> 27) & 16u);
      }
      s_red_add(ok ? a : dummy, ok ? inc : 0u);
    }
  }
  __device__ __forceinline__ void flush() {}
};

// W32 tile: separate u32 positive / negative words per end vertex; rb rebased by lo_rank * 8
struct OpTileDense32 {
  uint32_t rb;
  __device__ __forceinline__ void wedge(uint32_t w, uint32_t sg, int) {
    s_red_add(rb + (w << 3) + (((w ^ sg) >> 29) & 4u), 1u);
  }
  __device__ __forceinline__ void chunk(const uint32_t (&wv)[8], uint32_t sg, uint32_t m) {
    chunk_by_wedge(*this, wv, sg, m);
  }
  __device__ __forceinline__ void flush() {}
};

// counter-tile increments closed inline from the return value (a + wedge adds the old
// positive count to balanced and the old negative count to unbalanced, a - wedge the
// reverse); 32-bit partial sums per pair (8 x 65535 < 2^32), flushed to 64 bits.  With
// KEEP the touched word of each slot is kept (single-iteration rounds zero from it).
template <int W, bool KEEP, bool KG = false, bool BF = false>
struct OpTileClose {
  uint32_t rb;
  unsigned long long *tb, *tu;
  uint32_t k = 2;  // KG: (2,k)-bicliques, a wedge on a bucket holding c adds C(c, k-1)
  uint32_t b32 = 0, u32 = 0;
  uint32_t touched[8];
  uint32_t dummy = 0;  // BF: a tile word of this lane (invalid slots add 0 to it)
  __device__ __forceinline__ void add(uint32_t c, uint32_t other) {
    if (KG) {
      if (c >= k - 1u) add_k(*tb, *tu, binom_k(c, k - 1u));
    } else {
      b32 += c;
      u32 += other;
    }
  }
  __device__ __forceinline__ void wedge(uint32_t w, uint32_t sg, int j) {
    const uint32_t v = w ^ sg;
#ifdef BBC_MATCH
    if (W == 8 && !KG) {
      // match aggregation (experiment): a group of g lanes adding to one counter byte that
      // held c adds c + (c+1) + ... + (c+g-1) = g*c + g(g-1)/2 to the own sum and g times
      // the other byte to the other sum -- exactly the sum of the g single increments
      const uint32_t hs = (w & 1u) << 4;
      const uint32_t sh = hs | ((v >> 28) & 8u);
      const uint32_t a = rb + ((w << 1) & 0xfffffffcu);
      const uint32_t peers = __match_any_sync(__activemask(), (a << 3) | (sh >> 3));
      if ((threadIdx.x & 31u) == (uint32_t)(__ffs(peers) - 1)) {
        const uint32_t g = (uint32_t)__popc(peers);
        const uint32_t old = s_atom_add(a, g << sh);
        const uint32_t own = (old >> sh) & 0xffu, oth = (old >> (sh ^ 8u)) & 0xffu;
        b32 += g * own + ((g * (g - 1u)) >> 1);
        u32 += g * oth;
      }
      if (KEEP) touched[j] = a;
      return;
    }
#endif
    if (W == 8 && !KG) {
      // the increment selects this wedge's own byte; a byte dot product (IDP4A) of the old
      // word with it adds the own count, with the end vertex's other byte the other count
      const uint32_t hs = (w & 1u) << 4;
      const uint32_t inc = 1u << (hs | ((v >> 28) & 8u));
      const uint32_t a = rb + ((w << 1) & 0xfffffffcu);
      const uint32_t old = s_atom_add(a, inc);
      b32 = __dp4a(old, inc, b32);
      u32 = __dp4a(old, (0x101u << hs) ^ inc, u32);
      if (KEEP) touched[j] = a;
    } else if (W == 8) {
      const uint32_t sh = ((w & 1u) << 4) | ((v >> 28) & 8u);
      const uint32_t a = rb + ((w << 1) & 0xfffffffcu);
      const uint32_t old = s_atom_add(a, 1u << sh);
      add((old >> sh) & 0xffu, (old >> (sh ^ 8u)) & 0xffu);
      if (KEEP) touched[j] = a;
    } else {
      const uint32_t sh = (v >> 27) & 16u;
      const uint32_t a = rb + ((w << 2) & 0xfffffffcu);
      const uint32_t old = s_atom_add(a, 1u << sh);
      add((old >> sh) & 0xffffu, (old >> (sh ^ 16u)) & 0xffffu);
      if (KEEP) touched[j] = a;
    }
  }
  // BF (the fast path's tile rounds, k = 2): branch-free chunk -- an invalid slot adds 0 to
  // the lane's own tile word and its return value is masked out of the sums
  __device__ __forceinline__ void chunk(const uint32_t (&wv)[8], uint32_t sg, uint32_t m) {
    if (BF && !KG) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t w = wv[j], v = w ^ sg;
        const bool ok = (m >> j) & 1u;
        if (W == 8) {
          const uint32_t hs = (w & 1u) << 4;
          const uint32_t inc = ok ? 1u << (hs | ((v >> 28) & 8u)) : 0u;
          const uint32_t a = ok ? rb + ((w << 1) & 0xfffffffcu) : dummy;
          const uint32_t old = s_atom_add(a, inc);
          b32 = __dp4a(old, inc, b32);
          u32 = __dp4a(old, ok ? (0x101u << hs) ^ inc : 0u, u32);
          if (KEEP) touched[j] = ok ? a : touched[j];
        } else {
          const uint32_t sh = (v >> 27) & 16u;
          const uint32_t a = ok ? rb + ((w << 2) & 0xfffffffcu) : dummy;
          const uint32_t old = s_atom_add(a, ok ? 1u << sh : 0u);
          b32 += ok ? (old >> sh) & 0xffffu : 0u;
          u32 += ok ? (old >> (sh ^ 16u)) & 0xffffu : 0u;
          if (KEEP) touched[j] = ok ? a : touched[j];
        }
      }
      return;
    }
    chunk_by_wedge(*this, wv, sg, m);
  }
  __device__ __forceinline__ void flush() {
    if (!KG) {
      *tb += b32;
      *tu += u32;
      b32 = u32 = 0u;
    }
  }
};

// closing of one end vertex with p symmetric and q asymmetric wedges: k = 2 adds
// C(p,2)+C(q,2) to balanced (tb) and p*q to unbalanced (tu); KG adds C(p,k)+C(q,k) to the
// 128-bit (tb, tu)
template <bool KG>
__device__ __forceinline__ void close_pq(unsigned long long p, unsigned long long q, uint32_t k,
                                         unsigned long long& tb, unsigned long long& tu) {
  if (KG) {
    add_k(tb, tu, binom_k(p, k));
    add_k(tb, tu, binom_k(q, k));
  } else {
    tb += ((p * (p - (p > 0))) >> 1) + ((q * (q - (q > 0))) >> 1);
    tu += p * q;
  }
}

// ---- very wide cold ranges: key hash + repeat queue ------------------------------------
// When the cold range spans so many ranks that bitmap rounds would hold only a few hundred
// wedges each (config 4: tens of millions of end-vertex ranks), a round instead covers as
// many table columns as hold about K / 2 wedges, in a linear-probing hash of K keys
// (rank + 1, with the parity of the end vertex's FIRST wedge in bit 31).  The first wedge
// of an end vertex inserts its key; a later one finds it and queues (slot, own parity).
// After the walk the queue is counted per key slot in a small secondary set of packed u16
// counts and every repeated slot is closed once (first wedge's parity from the key).  The round's wedge
// count is known before the walk (block scan), so the hash never fills; a queue overflow
// redoes the round narrower.
struct OpKeys {
  uint32_t* keys;
  uint32_t K, queue, count, Q;
  __device__ __forceinline__ void wedge(uint32_t w, uint32_t sg, int) {
    const uint32_t key = (w & 0x7fffffffu) + 1u, par = (w ^ sg) >> 31;
    uint32_t h = (uint32_t)(((unsigned long long)(key * 0x9E3779B1u) * K) >> 32);
    for (;;) {
      const uint32_t old = atomicCAS(&keys[h], 0u, key | (par << 31));
      if (old == 0u) break;
      if ((old & 0x7fffffffu) == key) {
        const uint32_t idx = s_atom_add(count, 1u);
        if (idx < Q) s_st(queue + (idx << 2), h | (par << 31));
        break;
      }
      h = (h + 1u == K) ? 0u : h + 1u;
    }
  }
  __device__ __forceinline__ void chunk(const uint32_t (&wv)[8], uint32_t sg, uint32_t m) {
    chunk_by_wedge(*this, wv, sg, m);
  }
  __device__ __forceinline__ void flush() {}
};

// ---- cold bands: two-bit seen/parity bitmap + repeat queue -----------------------------
// In the cold end-vertex range almost every (anchor, end vertex) pair has one common
// centre (config 2: 2.7 % of the cold wedges land on a repeated end vertex), and a pair
// with one wedge contributes nothing.  A cold round therefore keeps two bits per end
// vertex (8x denser than a u8x2 counter tile, so one round spans 8x more ranks): word
// bit i = seen, bit 16 + i = parity (1 = negative) of the FIRST wedge, for 16 end vertices.
// Every wedge ORs in its seen bit and, when negative, the parity bit, in ONE atomic.  A
// wedge that finds the seen bit already set is a repeat and is appended to a queue as
// (rank, counted parity): a negative repeat that turned the parity bit from 0 to 1 is
// queued as POSITIVE -- it stands for the positive first wedge, the parity bit now for
// itself.  After the walk the queue is counted in a small hash (no divergence in the
// walk) and every repeated end vertex is closed (first wedge from the parity bit), so the
// adjacency is read once.  A round whose queue overflows is redone narrower.
struct OpBits {
  uint32_t rb, queue, count, Q, dummy;  // dummy: a bitmap word of this lane (ORed with 0)
  // bits = (1 | neg << 16) << i with neg = parity of (w ^ sg); (sg >> 15) | 1 is the same
  // for the whole chunk.  The eight atomics issue back to back (an invalid slot ORs 0 into
  // the dummy word); the rare repeats are queued afterwards.
  __device__ __forceinline__ void chunk(const uint32_t (&wv)[8], uint32_t sg, uint32_t m) {
    const uint32_t sgs1 = (sg >> 15) | 1u;
    uint32_t old[8], bits[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t w = wv[j];
      const bool ok = (m >> j) & 1u;
      bits[j] = ok ? (((w >> 15) & 0x10000u) ^ sgs1) << (w & 15u) : 0u;
      old[j] = s_atom_or(ok ? rb + ((w >> 2) & 0x0ffffffcu) : dummy, bits[j]);
    }
    // one LOP3 per wedge: any seen bit that was already set (a repeat) shows in `any`
    uint32_t any = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) any |= old[j] & bits[j];
    if (any & 0xffffu) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (!(old[j] & bits[j] & 0xffffu)) continue;
        // counted as negative only if it is negative and the parity bit was already set
        const uint32_t cneg = ((old[j] & bits[j]) >> 16) != 0u;
        const uint32_t idx = s_atom_add(count, 1u);
        if (idx < Q) s_st(queue + (idx << 2), (wv[j] & 0x7fffffffu) | (cneg << 31));
      }
    }
  }
  __device__ __forceinline__ void flush() {}
};

// slot of key (rank + 1) in a linear-probing set of K slots that never fills; bit 31 set
// when this call inserted it
__device__ __forceinline__ uint32_t rep_insert(uint32_t* keys, uint32_t K, uint32_t key) {
  volatile uint32_t* vk = keys;
  uint32_t h = (uint32_t)(((unsigned long long)(key * 0x9E3779B1u) * K) >> 32);
  for (;;) {
    uint32_t k = vk[h];
    if (k == key) return h;
    if (k == 0u) {
      k = atomicCAS(&keys[h], 0u, key);
      if (k == 0u) return h | 0x80000000u;
      if (k == key) return h;
    }
    h = (h + 1u == K) ? 0u : h + 1u;
  }
}

__device__ __forceinline__ unsigned long long c2(unsigned long long x) { return x * (x - (x > 0)) >> 1; }

// closing sweep over `words` counter words of layout W
template <int T, int W, bool KG = false>
__device__ __forceinline__ void sweep(uint32_t* cnt, uint32_t words, unsigned long long& tb, unsigned long long& tu,
                                      uint32_t k = 2) {
  uint4* c4 = reinterpret_cast<uint4*>(cnt);
  const uint32_t nq = (words + 3) >> 2;
  for (uint32_t i = threadIdx.x; i < nq; i += T) {
    const uint4 x = c4[i];
    if ((x.x | x.y | x.z | x.w) == 0u) continue;
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
    if (KG) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (W == 8) {
          close_pq<true>(xs[j] & 0xffu, (xs[j] >> 8) & 0xffu, k, tb, tu);
          close_pq<true>((xs[j] >> 16) & 0xffu, xs[j] >> 24, k, tb, tu);
        } else if (W == 16) {
          close_pq<true>(xs[j] & 0xffffu, xs[j] >> 16, k, tb, tu);
        } else {
          add_k(tb, tu, binom_k(xs[j], k));
        }
      }
    } else if (W == 8) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t p0 = xs[j] & 0xffu, q0 = (xs[j] >> 8) & 0xffu, p1 = (xs[j] >> 16) & 0xffu, q1 = xs[j] >> 24;
        tb += (p0 * (p0 - (p0 > 0)) + q0 * (q0 - (q0 > 0)) + p1 * (p1 - (p1 > 0)) + q1 * (q1 - (q1 > 0))) >> 1;
        tu += p0 * q0 + p1 * q1;
      }
    } else if (W == 16) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t p = xs[j] & 0xffffu, q = xs[j] >> 16;
        tb += (unsigned long long)((p * (p - (p > 0))) >> 1) + (unsigned long long)((q * (q - (q > 0))) >> 1);
        tu += (unsigned long long)(p * q);
      }
    } else {
      tb += c2(xs[0]) + c2(xs[1]) + c2(xs[2]) + c2(xs[3]);
      tu += (unsigned long long)xs[0] * xs[1] + (unsigned long long)xs[2] * xs[3];
    }
    c4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
}

__device__ __forceinline__ void add128(unsigned long long& lo, unsigned long long& hi, unsigned long long x) {
  lo += x;
  hi += (lo < x) ? 1ull : 0ull;
}

struct Smem {
  uint32_t* cnt;
  uint32_t* lo;
  uint32_t* hi;
  uint32_t* pfx;
  uint32_t* v;
  unsigned long long* w;
  uint32_t* ins;  // repeat-set insertions of the current cold round
};

// General path: any degree (records in batches of T), table or binary search, layout W.
template <int T, int W, bool KG>
__device__ void process_anchor(const Params& P, const Smem& S, uint32_t r, uint32_t rb, uint32_t re,
                               unsigned long long& tb, unsigned long long& tu, unsigned long long& work) {
  const uint32_t span = W == 8 ? P.span8 : (W == 16 ? P.span16 : P.span32);
  const uint32_t step = W == 8 ? 2u : 1u;  // table columns per band
  // band b = table columns [b * step, (b + 1) * step) only when the band span is the
  // table granularity (the 128 x 8 configuration); otherwise bounds by search
  const bool table = P.bnd != nullptr && W != 32 && P.span16 == P.t16;
  const uint32_t nbands_u = (P.n - 1u - r) / span + 1u;  // bands 0..nbands_u-1 hold ranks > r
  const uint32_t nbatch = (re - rb + T - 1u) / (uint32_t)T;
  uint32_t scan_buf = 0;  // alternates the scan's total buffers
  for (uint32_t b = 0; b < nbands_u; ++b) {
    const long long top = (long long)P.n - (long long)b * span;
    const long long bot = top - (long long)span;
    // lo_rank aligned to the ranks per word (W8: 2) for the rebased ops
    const uint32_t lo_rank = (bot > 0 ? (uint32_t)bot : 0u) & (W == 8 ? ~1u : ~0u);
    const uint32_t band_span = (uint32_t)(top - (long long)lo_rank);
    const uint32_t band_words = W == 8 ? (band_span + 1u) / 2u : (W == 16 ? band_span : 2u * band_span);
    const uint32_t base =
        sptr(S.cnt) - (W == 8 ? (lo_rank >> 1) << 2 : (W == 16 ? lo_rank << 2 : lo_rank << 3));
    int mode = -1;
    unsigned long long band_w = 0;
    for (uint32_t b0 = rb; b0 < re; b0 += T) {
      const int nb = (int)min((uint32_t)T, re - b0);
      uint32_t ng = 0;
      unsigned long long myw = 0;
      if ((int)threadIdx.x < nb) {
        const uint2 rr = P.rec[b0 + threadIdx.x];
        const uint32_t begin = rr.x & 0x7fffffffu, c = rr.y;
        uint32_t lo, hi;
        const uint32_t bi = table ? __ldg(P.brow + c) : 0xffffffffu;
        if (bi != 0xffffffffu) {
          const uint32_t* row = P.bnd + (size_t)bi * P.nbands;
          const uint32_t j0 = b * step, j1 = (b + 1u) * step;
          hi = __ldg(row + j0);
          lo = j1 < P.nbands ? __ldg(row + j1) : 0u;
        } else {
          const uint32_t end = __ldg(P.coff + c + 1);
          hi = b == 0 ? end : lower_bound_rank(P.adj, begin, end, top);
          lo = lower_bound_rank(P.adj, begin, hi, bot);
        }
        lo = max(lo, begin);
        hi = max(hi, lo);
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
      work += myw;
      band_w += bw;
      // the closing of a band is chosen once, from its first batch: the sweep when the band
      // will hold >= sweep_min wedges per counter word (and always for W32), else inline
      // closing from the atomics' return values and a vector clear
      if (mode < 0)
        mode = (W == 32 || bw * nbatch >= (unsigned long long)P.sweep_min * band_words || (P.debug & 2048)) ? kDense
                                                                                                          : kSparse;
      if (ngroups) {
        if (mode == kDense) {
          if (W == 32) {
            OpTileDense32 op{base};
            walk_chunks<T, true>(P.adj, S.lo, S.hi, S.pfx, nb, ngroups, op);
          } else {
            OpTileDense<W> op{base, 0u};
            walk_chunks<T, true>(P.adj, S.lo, S.hi, S.pfx, nb, ngroups, op);
          }
        } else {
          OpTileClose<W == 32 ? 16 : W, false, KG> op{base, &tb, &tu, P.k};
          walk_chunks<T, true>(P.adj, S.lo, S.hi, S.pfx, nb, ngroups, op);
        }
      }
      block_sync();  // the next batch overwrites the record arrays
    }
    if (band_w > 0) {
      if (mode == kDense) {
        sweep<T, W, KG>(S.cnt, band_words, tb, tu, P.k);
      } else {
        uint4* c4 = reinterpret_cast<uint4*>(S.cnt);
#pragma unroll 4
        for (uint32_t i = threadIdx.x; i < (band_words + 3u) / 4u; i += T) c4[i] = make_uint4(0u, 0u, 0u, 0u);
      }
      block_sync();
    }
  }
}

// Anchors with deg <= T and a band table (layouts W8 / W16).  Work is done in rounds;
// a round covers a range of table columns [ca, cb) = end-vertex ranks
// [n - cb * t16, n - ca * t16) and walks every record's sub-slice of that range once:
//   * the hub band (the top `hstep` columns: the high-degree end vertices that receive
//     most wedges) is a tile round (phase 1);
//   * the colder columns (phase 2) go through the hash table in one round when they fit
//     at load <= 2/3, else one tile round per band of `bstep` columns.
// Phase 0 runs both in one launch.  Tile rounds with <= 2 groups per thread close inline
// and zero from registers; larger ones use no-return increments and the closing sweep.
// Records stay in registers across rounds.
template <int T, int W, bool KG>
__device__ void process_anchor_fast(const Params& P, const Smem& S, uint32_t r, uint32_t rb, uint32_t re,
                                    unsigned long long w_a, unsigned long long& tb, unsigned long long& tu,
                                    unsigned long long& work) {
  const uint32_t step = W == 8 ? P.bcols8 : P.bcols16;     // this launch's tile band: columns
  // hub band: the phase-1 tile (128 x 8 configuration = table granularity), or this
  // launch's tile when one launch does every band
  const uint32_t hstep = P.phase == 0 ? step : (W == 8 ? 2u : 1u);
  const uint32_t t16 = P.t16;
  const uint32_t ncols = min(P.nbands, (P.n - 1u - r) / t16 + 1u);  // columns holding ranks > r
  const int nb = (int)(re - rb);
  const bool mine = (int)threadIdx.x < nb;
  uint32_t recx = 0u, lend = 0u;
  const uint32_t* row = nullptr;
  if (mine) {
    const uint2 rr = P.rec[rb + threadIdx.x];
    recx = rr.x;
    const uint32_t bi = P.bnd ? __ldg(P.brow + rr.y) : 0xffffffffu;
    if (bi != 0xffffffffu)
      row = P.bnd + (size_t)bi * P.nbands;
    else
      lend = __ldg(P.coff + rr.y + 1);
  }
  // column j of this thread's record: first position of its list with rank >= n - j * t16
  // (0 past the last column: start of the list), from the band table or, without one
  // (end-vertex ranges too wide for a table), by a galloping search down from `from`, a
  // position known to be at or above it (the previous round's boundary)
  auto col = [&](uint32_t j, uint32_t from) -> uint32_t {
    if (!mine || j >= P.nbands) return 0u;
    if (row) return __ldg(row + j);
    if (j == 0u) return lend;
    return lower_bound_gallop(P.adj, recx & 0x7fffffffu, from, (long long)P.n - (long long)j * t16);
  };
  // columns needed up front are loaded together (one latency)
  const uint32_t c0 = P.phase == 2 ? 0u : col(0u, lend), c1 = col(hstep, lend);
  const uint32_t c2 = P.phase == 1 ? 0u : col(min(hstep + step, ncols), c1);
  const uint32_t cn = (P.phase == 1 || !(P.debug & 4)) ? 0u : col(ncols, c1);
  // sub-slices [lo, hi) (positions of two table columns) -> S arrays, block scan;
  // returns total groups, bw = total wedges
  // One barrier per round set-up: each thread publishes its record's sub-slice, then EVERY
  // warp scans all (<= T) records itself (T / 32 per lane) and writes the same prefix
  // values to S.pfx -- a benign race, and a warp only reads pfx after writing it.  A round
  // without chunks adds a barrier so that no warp overwrites S.lo / S.hi while another
  // still scans them.
  auto setup = [&](uint32_t hi, uint32_t lo, unsigned long long& bw) -> uint32_t {
    if (mine) {
      lo = max(lo, recx & 0x7fffffffu);
      hi = max(hi, lo);
      S.lo[threadIdx.x] = lo | (recx & 0x80000000u);
      S.hi[threadIdx.x] = hi;
    }
    block_sync();
    constexpr int R = T / 32;
    const int lane = threadIdx.x & 31;
    uint32_t ng[R], run = 0;
    unsigned long long wsum = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int k = lane * R + i;
      ng[i] = 0u;
      if (k < nb) {
        const uint32_t a = S.lo[k] & 0x7fffffffu, b = S.hi[k];
        ng[i] = unit_count(a, b) & (b > a ? 0xffffffffu : 0u);
        wsum += b - a;
      }
      run += ng[i];
    }
    uint32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(kFull, wsum, o);
    uint32_t ex = incl - run;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int k = lane * R + i;
      if (k < nb) S.pfx[k] = ex;
      ex += ng[i];
    }
    const uint32_t ngroups = __shfl_sync(kFull, incl, 31);
    bw = wsum;
    __syncwarp();
#ifdef BBC_ROUND_STATS
    if ((P.debug & 4096) && threadIdx.x == 0) {
      atomicAdd(P.acc + 8, (unsigned long long)ngroups);
      atomicAdd(P.acc + 9, bw);
      atomicAdd(P.acc + 10, 1ull);
    }
#endif
    if (ngroups == 0u) block_sync();
    return ngroups;
  };
  // one tile round over band columns [ca, ca + cols)
  auto tile_round = [&](uint32_t ca, uint32_t cols, uint32_t ngroups, unsigned long long bw) {
#ifdef BBC_ROUND_STATS
    if ((P.debug & 4096) && threadIdx.x == 0) atomicAdd(P.acc + 6, 1ull);
#endif
    const long long top = (long long)P.n - (long long)ca * t16;
    const long long bot = top - (long long)cols * t16;
    // lo_rank aligned to the ranks per word (W8: 2), see the rebased ops
    const uint32_t lo_rank = (bot > 0 ? (uint32_t)bot : 0u) & (W == 8 ? ~1u : ~0u);
    const uint32_t band_span = (uint32_t)(top - (long long)lo_rank);
    const uint32_t band_words = W == 8 ? (band_span + 1u) / 2u : band_span;
    const uint32_t base = sptr(S.cnt) - (W == 8 ? (lo_rank >> 1) << 2 : lo_rank << 2);
    if (ngroups <= (uint32_t)T) {
      // at most one chunk per thread: close inline and zero the touched words
      // from registers (no second pass over the tile or the adjacency)
      OpTileClose<W, true, KG, true> op{base, &tb, &tu, P.k};
      op.dummy = sptr(S.cnt) + ((threadIdx.x & 31u) << 2);
#pragma unroll
      for (int j = 0; j < 8; ++j) op.touched[j] = 0xffffffffu;
      walk_chunks<T>(P.adj, S.lo, S.hi, S.pfx, nb, ngroups, op);
      block_sync();
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (op.touched[j] != 0xffffffffu) s_st(op.touched[j], 0u);
    } else if (bw < (unsigned long long)P.sweep_min * band_words && !(P.debug & 2048)) {
      // medium rounds: inline closing, then the tile is cleared with vector stores (a
      // closing sweep costs ~9 instructions per counter word, inline closing ~4 per wedge)
      OpTileClose<W, false, KG, true> op{base, &tb, &tu, P.k};
      op.dummy = sptr(S.cnt) + ((threadIdx.x & 31u) << 2);
      walk_chunks<T>(P.adj, S.lo, S.hi, S.pfx, nb, ngroups, op);
      block_sync();
      uint4* c4 = reinterpret_cast<uint4*>(S.cnt);
      for (uint32_t i = threadIdx.x; i < (band_words + 3u) / 4u; i += T) c4[i] = make_uint4(0u, 0u, 0u, 0u);
    } else {
      // dense rounds: no-return increments and the shared-memory closing sweep
      OpTileDense<W, true> op{base, sptr(S.cnt) + ((threadIdx.x & 31u) << 2)};
      walk_chunks<T>(P.adj, S.lo, S.hi, S.pfx, nb, ngroups, op);
      block_sync();
      sweep<T, W, KG>(S.cnt, band_words, tb, tu, P.k);
    }
    // no trailing barrier: every caller's next tile use comes after a setup (two barriers)
    // or after the end of the anchor (one barrier)
  };
  // band-by-band tile rounds over columns [ca, cb); a band is `step` columns starting at
  // any column (the table has every boundary), the last one truncated at cb
  // (work is a per-thread partial summed over the CTA at the end: thread 0 adds totals)
  const bool t0 = threadIdx.x == 0;
  // tiles over columns [step, ncols): the column values are carried from band to band and
  // the next band's lower column is prefetched while the current band runs
  auto tiles = [&]() {
    uint32_t hi = c1, lo = c2;
    for (uint32_t c = hstep; c < ncols; c += step) {
      const uint32_t nxt = c + step < ncols ? col(min(c + 2u * step, ncols), lo) : 0u;
      unsigned long long bw;
      const uint32_t ng = setup(hi, lo, bw);
      if (t0) work += bw;
      if (ng) tile_round(c, step, ng, bw);
      hi = lo;
      lo = nxt;
    }
  };

  // the hub band
  unsigned long long hub_w = 0;
  if (P.phase != 2 && !(P.debug & 4)) {
    const uint32_t ng = setup(c0, c1, hub_w);
    if (t0) work += hub_w;
    if (ng) tile_round(0u, hstep, ng, hub_w);
  }
  if (P.phase == 1 || ncols <= hstep || (P.debug & 8)) return;
  // cold range in two-bit bitmap rounds (see OpBits).  A round of `cols` columns uses
  // cols * t16 / 16 bitmap words and gives the rest of the tile to the repeat queue and
  // its hash, so narrow rounds tolerate many repeats.  Repeats are densest just below the
  // hub band (higher-degree end vertices), so rounds start narrow and double while the
  // queue stays under 1/4 full; an overflowing round is redone at half the width (one
  // column: a counter tile).
  auto bitmap_rounds = [&]() {
    uint32_t cols = P.bm_cols0;
    uint32_t hi = c1;
    uint32_t parity = 0;  // the queue counter of a round alternates between S.ins[0] / [1]
    for (uint32_t c = hstep; c < ncols;) {
      const uint32_t cb = min(c + cols, ncols);
      const uint32_t lo = col(cb, hi);
      uint32_t* cnt = S.ins + (parity++ & 1u);
      // reset and read of the repeat counter are volatile: the walk increments it through
      // inline-asm atomics the compiler cannot see
      if (t0) *(volatile uint32_t*)cnt = 0u;  // its last reader finished before the previous round's barriers
      unsigned long long bw;
      const uint32_t ng = setup(hi, lo, bw);
      if (ng == 0u) {
        hi = lo;
        c = cb;
        continue;
      }
      const long long top = (long long)P.n - (long long)c * t16;
      const long long bot = (long long)P.n - (long long)cb * t16;
      const uint32_t lo_rank = (bot > 0 ? (uint32_t)bot : 0u) & ~15u;  // rebased ops: 16 per word
      const uint32_t span_words = (uint32_t)((top - (long long)lo_rank + 15) / 16 + 3) & ~3u;
      // queue of Q repeats, then a 2Q-slot key set and its packed counts (never fills)
      const uint32_t Q = ((P.cap_words - span_words) / 5u) & ~3u;
      const uint32_t K = 2u * Q;
      uint32_t* bm = S.cnt;
      uint32_t* queue = S.cnt + span_words;
      uint32_t* keys = queue + Q;
      uint32_t* vals = keys + K;
      OpBits op{sptr(bm) - ((lo_rank >> 4) << 2), sptr(queue), sptr(cnt), Q, sptr(bm) + ((threadIdx.x & 31u) << 2)};
      walk_chunks<T>(P.adj, S.lo, S.hi, S.pfx, nb, ng, op);
      block_sync();
      const uint32_t nq = *(volatile const uint32_t*)cnt;
      const bool ovf = nq > Q;
      if (nq != 0u && !ovf) {
        // count the repeats per end vertex; the inserting entry becomes the closer and
        // carries the parity bit of the end vertex's first wedge
        for (uint32_t i = threadIdx.x; i < nq; i += T) {
          const uint32_t e = queue[i];
          const uint32_t rank = e & 0x7fffffffu;
          const uint32_t h = rep_insert(keys, K, rank + 1u);
          atomicAdd(&vals[h & 0x7fffffffu], (e >> 31) ? 0x10000u : 1u);
          const uint32_t rel = rank - lo_rank;
          const uint32_t neg = (bm[rel >> 4] >> (16u + (rel & 15u))) & 1u;
          queue[i] = (h >> 31) ? (h | (neg << 30)) : 0u;
        }
        block_sync();
        // close every repeated end vertex (first wedge from the parity bit + the counts)
        for (uint32_t i = threadIdx.x; i < nq; i += T) {
          const uint32_t e = queue[i];
          if (e == 0u) continue;
          const uint32_t h = e & 0x3fffffffu, neg = (e >> 30) & 1u;
          const uint32_t v = vals[h];
          close_pq<KG>((v & 0xffffu) + (neg ^ 1u), (v >> 16) + neg, P.k, tb, tu);
          keys[h] = 0u;
          vals[h] = 0u;
          queue[i] = 0u;
        }
      } else if (ovf) {
        uint4* q4 = reinterpret_cast<uint4*>(queue);
        for (uint32_t i = threadIdx.x; i < Q / 4u; i += T) q4[i] = make_uint4(0u, 0u, 0u, 0u);
      }
      // the bitmap is no longer read (closing uses the queue's parity bits); the next
      // round's setup barriers order this clearing before its walk
      uint4* c4 = reinterpret_cast<uint4*>(bm);
#pragma unroll 4
      for (uint32_t i = threadIdx.x; i < span_words / 4u; i += T) c4[i] = make_uint4(0u, 0u, 0u, 0u);
#ifdef BBC_ROUND_STATS
      if (P.debug & 4096) {
        if (t0) atomicAdd(P.acc + 4, 1ull);
        if (t0 && ovf) atomicAdd(P.acc + 5, 1ull);
      }
#endif
      if (!ovf) {
        if (t0) work += bw;
        hi = lo;
        c = cb;
        if (nq < Q / 4u) cols = min(2u * cols, P.bm_cols);
      } else if (cols > 1u) {
        cols = (cols + 1u) / 2u;  // redo [c, c + cols)
      } else {
        // a single column with too many repeats: one counter-tile round
        unsigned long long tbw;
        const uint32_t tng = setup(hi, lo, tbw);
        if (t0) work += tbw;
        if (tng) tile_round(c, 1u, tng, tbw);
        hi = lo;
        c = cb;
      }
    }
  };

  // cold range in key-hash rounds over adaptive column ranges (see OpKeys): a round aims
  // at `target` wedges; the first width comes from the cold range's average density
  auto hash_rounds = [&](unsigned long long wc) {
    // keys (K words: rank + 1 with the first wedge's parity), the repeat queue (Q), and a
    // small secondary set (2Q slots) counting repeats per key slot -- only repeated keys
    // need counts, so the primary set spends one word per slot and holds more wedges
    const uint32_t Q = (P.cap_words / 16u) & ~3u;
    const uint32_t SS = 2u * Q;
    const uint32_t K = (P.cap_words - Q - 2u * SS) & ~3u;
    const uint32_t target = K / 2u;
    const uint32_t span = ncols - hstep;
    uint32_t cols = (uint32_t)max(1ull, min((unsigned long long)span, (unsigned long long)target * span / max(wc, 1ull)));
    uint32_t hi = c1;
    uint32_t parity = 0;
    uint32_t* keys = S.cnt;
    uint32_t* queue = keys + K;
    uint32_t* skeys = queue + Q;
    uint32_t* svals = skeys + SS;
    for (uint32_t c = hstep; c < ncols;) {
      const uint32_t cb = min(c + cols, ncols);
      const uint32_t lo = col(cb, hi);
      uint32_t* cnt = S.ins + (parity++ & 1u);
      if (t0) *(volatile uint32_t*)cnt = 0u;
      unsigned long long bw;
      const uint32_t ng = setup(hi, lo, bw);
      if (ng == 0u) {
        hi = lo;
        c = cb;
        cols = min(2u * cols, span);
        continue;
      }
      if (bw > target && cols > 1u) {  // too many wedges for the hash: narrower, no walk
        cols = max(1u, min(cols / 2u, (uint32_t)((unsigned long long)cols * target / bw)));
        block_sync();  // every warp is done with this set-up's record arrays
        continue;
      }
      if (bw > target) {  // a single column denser than the hash: one counter-tile round
        if (t0) work += bw;
        tile_round(c, 1u, ng, bw);
        hi = lo;
        c = cb;
        continue;
      }
#ifdef BBC_ROUND_STATS
      if ((P.debug & 4096) && t0) atomicAdd(P.acc + 7, 1ull);
#endif
      OpKeys op{keys, K, sptr(queue), sptr(cnt), Q};
      walk_chunks<T>(P.adj, S.lo, S.hi, S.pfx, nb, ng, op);
      block_sync();
      const uint32_t nq = *(volatile const uint32_t*)cnt;
      const bool ovf = nq > Q;
      if (nq != 0u && !ovf) {
        // count the repeats per key slot in the secondary set; the entry that inserted the
        // slot becomes its closer and carries the first wedge's parity
        for (uint32_t i = threadIdx.x; i < nq; i += T) {
          const uint32_t e = queue[i], h = e & 0x7fffffffu;
          const uint32_t r = rep_insert(skeys, SS, h + 1u);
          atomicAdd(&svals[r & 0x7fffffffu], (e >> 31) ? 0x10000u : 1u);
          queue[i] = (r >> 31) ? ((r & 0x3fffffffu) | 0x80000000u | ((keys[h] >> 31) << 30)) : 0u;
        }
        block_sync();
        for (uint32_t i = threadIdx.x; i < nq; i += T) {
          const uint32_t e = queue[i];
          if (e == 0u) continue;
          queue[i] = 0u;
          const uint32_t slot = e & 0x3fffffffu, v = svals[slot];
          const unsigned long long neg = (e >> 30) & 1u;
          close_pq<KG>((v & 0xffffu) + (neg ^ 1ull), (v >> 16) + neg, P.k, tb, tu);
          skeys[slot] = 0u;
          svals[slot] = 0u;
        }
      } else if (ovf) {
        uint4* q4 = reinterpret_cast<uint4*>(queue);
        for (uint32_t i = threadIdx.x; i < Q / 4u; i += T) q4[i] = make_uint4(0u, 0u, 0u, 0u);
      }
      // keys are no longer read (parities travelled with the queue entries)
      uint4* k4 = reinterpret_cast<uint4*>(keys);
#pragma unroll 4
      for (uint32_t i = threadIdx.x; i < K / 4u; i += T) k4[i] = make_uint4(0u, 0u, 0u, 0u);
      if (!ovf) {
        if (t0) work += bw;
        hi = lo;
        c = cb;
        if (2ull * bw < target) cols = min(2u * cols, span);
      } else if (cols > 1u) {
        cols = (cols + 1u) / 2u;
      } else {
        unsigned long long tbw;
        const uint32_t tng = setup(hi, lo, tbw);
        if (t0) work += tbw;
        if (tng) tile_round(c, 1u, tng, tbw);
        hi = lo;
        c = cb;
      }
    }
  };

  // cold range: key-hash rounds when bitmap rounds would average fewer than hash_thr (256)
  // wedges (very wide, sparse rank ranges); else two-bit bitmap rounds (8x the span of a
  // counter tile) unless counter tiles would average at least bits_thr wedges per round
  // (dense cold ranges, where repeats are common); else counter tiles band by band.
  // (flags bit 13 forces hash rounds, bit 9 bitmap rounds, bit 7 disables both)
  if (P.bm_cols != 0u) {
    // cold wedges: the anchor's work minus the hub band's (a block scan only when the hub
    // round was skipped)
    unsigned long long wc = w_a - hub_w;
    if (P.debug & 4) setup(c1, cn, wc);
    const unsigned long long bm_rounds = (ncols - hstep + P.bm_cols - 1u) / P.bm_cols;
    if ((P.debug & 8192) || wc < (unsigned long long)P.hash_thr * bm_rounds) {
      hash_rounds(wc);
      return;
    }
    const unsigned long long tile_rounds = (ncols - hstep + step - 1u) / step;
    if (P.bm_cols != 0u && (wc < (unsigned long long)P.bits_thr * tile_rounds || (P.debug & 512))) {
      bitmap_rounds();
      return;
    }
  }
  tiles();
}

template <int T, int MINB, bool KG>
__global__ void __launch_bounds__(T, MINB) k_count(Params P) {
  constexpr int kWarps = T / 32;
  extern __shared__ uint4 smem4[];
  __shared__ uint32_t s_v[64];
  __shared__ unsigned long long s_w[64];
  __shared__ uint32_t s_task;
  __shared__ uint32_t s_ins[2];
  Smem S;
  S.cnt = reinterpret_cast<uint32_t*>(smem4);
  S.lo = S.cnt + P.cap_words;
  S.hi = S.lo + T;
  S.pfx = S.hi + T;
  S.v = s_v;
  S.w = s_w;
  S.ins = s_ins;

  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  for (uint32_t i = threadIdx.x; i < P.cap_words / 4; i += T) smem4[i] = make_uint4(0u, 0u, 0u, 0u);

  unsigned long long bal_lo = 0, bal_hi = 0, unb_lo = 0, unb_hi = 0, work = 0;
  uint32_t next = blockIdx.x;
  if (threadIdx.x == 0) s_task = P.dynamic ? atomicAdd(P.queue, 1u) : next;
  block_sync();
  for (;;) {
    const uint32_t t = s_task;
    next += gridDim.x;
    block_sync();  // every thread holds t before s_task is overwritten
    if (t >= P.ntasks) break;
    // claim the following task now so the queue round trip overlaps this anchor
    if (threadIdx.x == 0) s_task = P.dynamic ? atomicAdd(P.queue, 1u) : next;
    const uint32_t gidx = P.part_index + t * P.part_count;
    const uint32_t r = P.dynamic ? P.order[gidx] : gidx;
    const unsigned long long w_a = P.awork[r];
    if (w_a == 0ull) {
      block_sync();  // publish the claimed task
      continue;
    }
    const uint32_t rb = P.aoff[r], re = P.aoff[r + 1];
    const uint32_t deg = re - rb;
    unsigned long long tb = 0, tu = 0;
    // fast path: every record held by one thread; the bound is the same for all launches of
    // a count so that phases agree on which anchors they split
    const bool fast = P.fast && deg <= min((uint32_t)T, P.fast_max);
    if (!fast && P.phase == 2) {  // general-path anchors are done entirely in phase 1
      block_sync();
      continue;
    }
    if (fast && deg <= 255u)
      process_anchor_fast<T, 8, KG>(P, S, r, rb, re, w_a, tb, tu, work);
    else if (fast)
      process_anchor_fast<T, 16, KG>(P, S, r, rb, re, w_a, tb, tu, work);
    else if (deg <= 255u)
      process_anchor<T, 8, KG>(P, S, r, rb, re, tb, tu, work);
    else if (deg <= 65535u)
      process_anchor<T, 16, KG>(P, S, r, rb, re, tb, tu, work);
    else
      process_anchor<T, 32, KG>(P, S, r, rb, re, tb, tu, work);
    add128(bal_lo, bal_hi, tb);
    add128(unb_lo, unb_hi, tu);
    block_sync();  // publish the claimed task
  }

  // exact 128-bit reduction: warp shuffle, then one pair of global atomics per warp
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    unsigned long long l2 = __shfl_xor_sync(kFull, bal_lo, o), h2 = __shfl_xor_sync(kFull, bal_hi, o);
    unsigned long long l3 = __shfl_xor_sync(kFull, unb_lo, o), h3 = __shfl_xor_sync(kFull, unb_hi, o);
    unsigned long long w2 = __shfl_xor_sync(kFull, work, o);
    bal_lo += l2;
    bal_hi += h2 + (bal_lo < l2 ? 1ull : 0ull);
    unb_lo += l3;
    unb_hi += h3 + (unb_lo < l3 ? 1ull : 0ull);
    work += w2;
  }
  if (lane == 0) {
    unsigned long long old = atomicAdd(&P.acc[0], bal_lo);
    atomicAdd(&P.acc[1], bal_hi + (old + bal_lo < old ? 1ull : 0ull));
    old = atomicAdd(&P.acc[2], unb_lo);
    atomicAdd(&P.acc[3], unb_hi + (old + unb_lo < old ? 1ull : 0ull));
    s_w[threadIdx.x >> 5] = work;
  }
  block_sync();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kWarps; ++w) t += s_w[w];
    P.block_work[blockIdx.x] += t;  // launches of one count accumulate (zeroed per count)
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    P.block_busy[blockIdx.x] += t_end - t_start;
  }
}

struct Launch {
  int threads = 0;
  int blocks_per_sm = 0;
  int cap_words = 0;
  int smem_bytes = 0;
  void (*kernel)(Params) = nullptr;
};

// T threads per CTA, MINB CTAs per SM: shared memory is split evenly between the CTAs of
// an SM (1 KB per CTA is reserved by the driver) and registers are capped accordingly.
template <int T, int MINB, bool KG = false>
int configure_t(Graph& g, Launch& L) {
  cudaFuncAttributes fa;
  BBC_CK(cudaFuncGetAttributes(&fa, k_count<T, MINB, KG>));
  int per_sm = 0;
  BBC_CK(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, g.device));
  int budget = std::min(g.max_smem, per_sm / MINB - 1024);
  int avail = budget - (int)fa.sharedSizeBytes - (3 * T * 4 + 64);
  L.threads = T;
  L.blocks_per_sm = MINB;
  L.cap_words = (avail / 16) * 4;
  L.smem_bytes = L.cap_words * 4 + 3 * T * 4 + 16;
  L.kernel = k_count<T, MINB, KG>;
  BBC_CK(cudaFuncSetAttribute(k_count<T, MINB, KG>, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem_bytes));
  return BBC_OK;
}

// single-launch configuration (all phases): 128 x 8 per SM.  Measured on config 2 and
// removed: 128 x {4, 6, 10, 12} (19.6 / 16.0 / 17.7 / 20.0 ms vs 15.4 ms at the time),
// 256 x 4, 512 x 2 and 1024 x 1.
int configure(Graph& g, Launch& L) { return configure_t<128, 8>(g, L); }

// two-phase configuration: hub band with 128 x 8, cold range with 256 x 2 (big hash)
int configure_cold(Graph& g, Launch& L) { return configure_t<256, 2>(g, L); }

}  // namespace

// Table granularity: the W16 span of the 128-thread configuration in use (hub band).
int count_span16(Graph& g) {
  Launch L;
  BBC_CK(cudaSetDevice(g.device));
  if (configure(g, L)) return -1;
  return L.cap_words - 8;
}

// k = 2: balanced / unbalanced butterflies; k > 2: balanced (2,k)-bicliques (out[0] = the
// count, out[1] = 0) with the same rounds and C(., k) closings (the KG kernel)
int count_graph(Graph& g, const bbc_opts* o, uint64_t out[2], bbc_stats* st, int32_t k) {
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
  if (k < 2) {
    set_error("k must be >= 2, got " + std::to_string(k));
    return BBC_ERR_ARG;
  }
  const bool kg = k > 2;
  BBC_CK(cudaSetDevice(g.device));
  Launch L, Lc;
  int rc = kg ? configure_t<128, 8, true>(g, L) : configure(g, L);
  if (rc) return rc;
  bool use_table = g.bnd != nullptr && !(opts.flags & 1024);  // 1024: binary search (tests)
  const bool tile_override = opts.tile_span > 0 && (uint32_t)opts.tile_span < 2u * ((uint32_t)L.cap_words - 8u);
  if (tile_override) use_table = false;
  // flags bit 6 (experimental, measured slower on config 2): hub band and cold range in
  // two launches with different CTA shapes
  const bool two_phase = !kg && use_table && (opts.flags & 64) && (opts.flags & 1) == 0;
  if (two_phase) {
    rc = configure_cold(g, Lc);
    if (rc) return rc;
  }
  const int blocks1 = opts.blocks > 0 ? opts.blocks : g.num_sms * L.blocks_per_sm;
  const int blocks2 = two_phase ? (opts.blocks > 0 ? opts.blocks : g.num_sms * Lc.blocks_per_sm) : 0;
  const int blocks = std::max(blocks1, blocks2);
  if (blocks > g.block_work_cap) {
    cudaFree(g.block_work);
    g.block_work = nullptr;
    BBC_CK(cudaMalloc(&g.block_work, (size_t)blocks * 16));
    g.block_work_cap = blocks;
  }
  const uint32_t n = (uint32_t)g.n;
  const uint32_t ntasks =
      n > (uint32_t)opts.part_index ? (n - (uint32_t)opts.part_index + part_count - 1) / part_count : 0u;

  // tuning constants (measured on configs 2-5)
  constexpr struct {
    uint32_t rep_slots = 128, bits_thr = 4096, sweep_min = 4, bm_cols0 = 8, hash_thr = 256;
  } tune;

  auto params = [&](const Launch& X, int phase) {
    Params P;
    uint32_t span16 = (uint32_t)X.cap_words - 8u;
    uint32_t span8 = 2u * span16, span32 = span16 / 2u;
    if (tile_override) {
      // TileConfig.tile_size: bands of at most tile_span end vertices in every layout
      const uint32_t t = (uint32_t)opts.tile_span;
      span8 = t;
      span16 = std::min(span16, t);
      span32 = std::min(span32, t);
    }
    P.adj = g.adj;
    P.rec = g.rec;
    P.coff = g.coff;
    P.aoff = g.aoff;
    P.awork = g.awork;
    P.order = g.order;
    P.bnd = use_table ? g.bnd : nullptr;
    P.brow = g.brow;
    P.nbands = g.nbands;
    P.t16 = g.t16;
    P.bcols16 = std::max(1u, span16 / std::max(1u, g.t16));
    P.bcols8 = std::max(2u, span8 / std::max(1u, g.t16));
    P.phase = phase;
    P.n = n;
    P.ntasks = ntasks;
    P.part_index = (uint32_t)opts.part_index;
    P.part_count = (uint32_t)part_count;
    P.span8 = span8;
    P.span16 = span16;
    P.span32 = span32;
    P.cap_words = (uint32_t)X.cap_words;
    // the fast path needs the fixed column grid (not with TileConfig.tile_size spans) and
    // ranks < 2^30 (rebased word addressing)
    P.fast = ((opts.flags & 1) || tile_override || g.t16 == 0 || n >= (1u << 30) ||
              (uint32_t)X.cap_words < g.t16 + 8u)  // this configuration's tile must hold a column
                 ? 0
                 : 1;
    P.fast_max = two_phase ? (uint32_t)std::min(L.threads, Lc.threads) : (uint32_t)X.threads;
    P.hash_thr = (opts.flags & 2) ? 0u : tune.hash_thr;  // flags bit 1: no key-hash rounds
    // cold two-bit bitmap rounds (flags bit 7 disables): the widest round leaves room for
    // a queue of rep_slots repeats (flags bit 8: 16, and rounds start at that width, so
    // that tests exercise the overflow / narrowing path)
    const uint32_t rep = (opts.flags & 256) ? 16u : tune.rep_slots;
    P.rep_slots = std::max(16u, std::min(rep, (uint32_t)X.cap_words / 10u) & ~3u);
    P.bm_words = ((uint32_t)X.cap_words - 5u * P.rep_slots) & ~3u;
    P.bm_cols = (opts.flags & 128) ? 0u : (16u * P.bm_words) / std::max(1u, g.t16);
    P.bm_cols0 = std::max(1u, std::min(P.bm_cols, (opts.flags & 256) ? P.bm_cols : tune.bm_cols0));
    P.bits_thr = tune.bits_thr;
    P.sweep_min = tune.sweep_min;
    P.debug = opts.flags;
    P.dynamic = opts.algo == BBC_ALGO_GBBCPP;
    P.k = (uint32_t)k;
    P.acc = g.acc;
    P.queue = g.queue + (phase == 2 ? 1 : 0);
    P.block_work = g.block_work;
    P.block_busy = g.block_work + g.block_work_cap;
    return P;
  };

  BBC_CK(cudaMemsetAsync(g.acc, 0, 128, g.stream));
  BBC_CK(cudaMemsetAsync(g.queue, 0, 8, g.stream));
  BBC_CK(cudaMemsetAsync(g.block_work, 0, (size_t)blocks * 8, g.stream));
  BBC_CK(cudaMemsetAsync(g.block_work + g.block_work_cap, 0, (size_t)blocks * 8, g.stream));
  BBC_CK(cudaEventRecord(g.ev0, g.stream));
  const Params P1 = params(L, two_phase ? 1 : 0);
  L.kernel<<<blocks1, L.threads, L.smem_bytes, g.stream>>>(P1);
  BBC_CK(cudaGetLastError());
  if (two_phase) {
    const Params P2 = params(Lc, 2);
    Lc.kernel<<<blocks2, Lc.threads, Lc.smem_bytes, g.stream>>>(P2);
    BBC_CK(cudaGetLastError());
  }
  BBC_CK(cudaEventRecord(g.ev1, g.stream));
  const uint32_t span16 = P1.span16;
  unsigned long long h_acc[16];
  BBC_CK(cudaMemcpyAsync(h_acc, g.acc, 128, cudaMemcpyDeviceToHost, g.stream));
  BBC_CK(cudaStreamSynchronize(g.stream));
  g.last_blocks = blocks;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, g.ev0, g.ev1);
  for (int i = 0; i < 8; ++i) g.rounds[i] = h_acc[4 + i];
  if (kg) {
    // per-thread (tb, tu) were the low / high words of one 128-bit sum: total =
    // bal + unb * 2^64 (as 128-bit values); the low 64 bits and whether it overflowed
    const bool ovf = h_acc[1] != 0ull || h_acc[2] != 0ull || h_acc[3] != 0ull;
    h_acc[1] = ovf ? 1ull : 0ull;
    h_acc[2] = h_acc[3] = 0ull;
  }
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
    st->threads = L.threads;
    st->tile_span = (int32_t)span16;
    st->tasks = (int32_t)ntasks;
    st->preprocess_ms = g.preprocess_ms;
    st->count_ms = ms;
  }
  if (h_acc[1] || h_acc[3]) {
    set_error(kg ? "balanced (2,k) count exceeded 64-bit range" : "balanced/unbalanced count exceeded 64-bit range");
    return BBC_ERR_OVERFLOW;
  }
  return BBC_OK;
}

}  // namespace bbc
