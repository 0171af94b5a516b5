// Device-side edge-list ingestion: the reference loader
// pipeline load_graph = parse_edge_list -> apply_sign_policy -> dedup_latest -> to_graph
// (pkg/src/bbcount/ingest.py:80-191) on the GPU, for ASCII text.
//
// Behaviour restated (ingest.py line numbers):
//   * lines end at '\n'; a line is stripped of whitespace, skipped when empty or when it
//     starts with '%' or '#'; it must then hold 2-4 whitespace-separated tokens
//     ``u v [value] [timestamp]`` (MalformedLineError with the 1-based line, :80-115);
//   * labels map to dense ids per side in first-occurrence order over the parsed edges
//     (:113-114), independent of later deduplication;
//   * ExplicitSign: value 1 -> +, 0 or -1 -> -, anything else InvalidSignValueError, no
//     value MissingValueError; RatingThreshold: value >= t (or > t) is +; RandomBernoulli:
//     positive iff blake2b(ordinal, key=seed, digest 8 bytes) / 2^64 < p (:118-158), the
//     first failing edge in input order raising;
//   * dedup_latest: per (u, v) the maximal (has timestamp, timestamp, position) wins,
//     output in the pair's first-occurrence order (:161-175).
// Anything outside the exact fast paths -- non-ASCII bytes, value tokens that are not a
// plain decimal exactly representable by Clinger's fast path (mantissa < 2^53, |exp10| <=
// 22), timestamps that are not [+-]digits{1,18}, or a 64-bit label-hash collision --
// returns BBC_ERR_UNSUPPORTED with the first such line, and the Python layer runs the
// host loader (ingest.py semantics) on the whole text instead.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "bbc_internal.cuh"

namespace bbc {

namespace {

constexpr int kT = 256;

// temporaries are stream-ordered allocations from the device's (cached) default pool, so
// repeated ingestions do not pay cudaMalloc / cudaFree round trips
thread_local cudaStream_t t_stream = nullptr;

struct Buf {
  void* p = nullptr;
  ~Buf() {
    if (p) cudaFreeAsync(p, t_stream);
  }
  template <typename X>
  X* as() {
    return static_cast<X*>(p);
  }
};

#define ING_ALLOC(buf, bytes)                                                             \
  do {                                                                                    \
    cudaError_t _e = cudaMallocAsync(&(buf).p, (bytes) ? (size_t)(bytes) : 16, t_stream); \
    if (_e != cudaSuccess) return cuda_fail(_e, "cudaMallocAsync (ingest)");             \
  } while (0)

inline int grid(int64_t n) {
  int64_t b = (n + kT - 1) / kT;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

// Python's str.isspace() over ASCII: \t \n \v \f \r, 0x1c-0x1f, space
__device__ __forceinline__ bool is_ws(uint8_t c) { return (c >= 9 && c <= 13) || (c >= 28 && c <= 32); }

struct IsNewline {
  const uint8_t* t;
  __device__ __forceinline__ bool operator()(const int64_t& i) const { return t[i] == '\n'; }
};

// line status
enum { kSkip = 0, kEdge = 1, kMalformed = 2, kUnsupported = 3 };

__device__ const double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                      1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

// Plain decimal -> double, exact (Clinger's fast path); false when outside it
__device__ bool parse_double(const uint8_t* s, int n, double& out) {
  int i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  unsigned long long mant = 0;
  int digits = 0, frac = 0, sig = 0;
  bool dot = false;
  for (; i < n; ++i) {
    const uint8_t c = s[i];
    if (c >= '0' && c <= '9') {
      ++digits;
      if (dot) ++frac;
      if (mant == 0 && c == '0') continue;  // leading zeros
      if (++sig > 19) return false;
      mant = mant * 10ull + (c - '0');
    } else if (c == '.' && !dot) {
      dot = true;
    } else {
      break;
    }
  }
  if (digits == 0) return false;
  int e10 = 0;
  if (i < n && (s[i] == 'e' || s[i] == 'E')) {
    ++i;
    bool eneg = false;
    if (i < n && (s[i] == '+' || s[i] == '-')) eneg = s[i++] == '-';
    int ed = 0;
    for (; i < n && s[i] >= '0' && s[i] <= '9'; ++i) {
      if (++ed > 4) return false;
      e10 = e10 * 10 + (s[i] - '0');
    }
    if (ed == 0) return false;
    if (eneg) e10 = -e10;
  }
  if (i != n) return false;
  e10 -= frac;
  if (mant == 0) {
    out = neg ? -0.0 : 0.0;
    return true;
  }
  if (mant >= (1ull << 53) || e10 < -22 || e10 > 22) return false;
  double v = (double)mant;
  v = e10 >= 0 ? v * kPow10[e10] : v / kPow10[-e10];
  out = neg ? -v : v;
  return true;
}

// [+-]digits{1,18} -> int64
__device__ bool parse_int(const uint8_t* s, int n, long long& out) {
  int i = 0;
  bool neg = false;
  if (i < n && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  if (i == n || n - i > 18) return false;
  long long v = 0;
  for (; i < n; ++i) {
    if (s[i] < '0' || s[i] > '9') return false;
    v = v * 10 + (s[i] - '0');
  }
  out = neg ? -v : v;
  return true;
}

struct Line {
  int64_t tok[4];   // token starts (absolute byte offsets)
  int32_t len[4];   // token lengths
  double value;
  long long ts;
  int32_t ntok;
};

// one thread per line: strip, comment check, tokens, numeric fields
__global__ void k_parse_lines(const uint8_t* __restrict__ t, int64_t nbytes, const int64_t* __restrict__ nl,
                              int64_t nlines, uint8_t* __restrict__ status, Line* __restrict__ lines) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nlines; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = k == 0 ? 0 : nl[k - 1] + 1;
    const int64_t e = nl[k];  // the line's '\n' (or the end of the text)
    Line L;
    L.ntok = 0;
    L.value = 0.0;
    L.ts = 0;
    uint8_t st = kSkip;
    int64_t i = s;
    bool first = true;
    while (i < e) {
      const uint8_t c = t[i];
      if (c >= 0x80) {
        st = kUnsupported;
        break;
      }
      if (is_ws(c)) {
        ++i;
        continue;
      }
      if (first && (c == '%' || c == '#')) break;  // comment line
      first = false;
      int64_t j = i;
      bool ascii = true;
      while (j < e && !is_ws(t[j])) {
        if (t[j] >= 0x80) ascii = false;
        ++j;
      }
      if (!ascii) {
        st = kUnsupported;
        break;
      }
      if (L.ntok < 4) {
        L.tok[L.ntok] = i;
        L.len[L.ntok] = (int32_t)(j - i);
      }
      ++L.ntok;
      i = j;
    }
    if (st != kUnsupported && L.ntok > 0) {
      if (L.ntok < 2 || L.ntok > 4) {
        st = kMalformed;
      } else {
        st = kEdge;
        if (L.ntok >= 3 && !parse_double(t + L.tok[2], L.len[2], L.value)) st = kUnsupported;
        if (st == kEdge && L.ntok == 4 && !parse_int(t + L.tok[3], L.len[3], L.ts)) st = kUnsupported;
      }
    }
    status[k] = st;
    lines[k] = L;
  }
}

__global__ void k_first_problem(const uint8_t* __restrict__ status, int64_t nlines, unsigned long long* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nlines; k += (int64_t)gridDim.x * blockDim.x)
    if (status[k] >= kMalformed) atomicMin(out, ((unsigned long long)k << 2) | status[k]);
}

struct IsEdgeLine {
  const uint8_t* status;
  __device__ __forceinline__ bool operator()(const int64_t& k) const { return status[k] == kEdge; }
};

// 64-bit FNV-1a of a token's bytes
__device__ __forceinline__ unsigned long long hash_token(const uint8_t* p, int n) {
  unsigned long long h = 1469598103934665603ull;
  for (int i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
  return h;
}

__global__ void k_label_hashes(const uint8_t* __restrict__ t, const Line* __restrict__ lines,
                               const int64_t* __restrict__ eline, int64_t m, int side,
                               unsigned long long* __restrict__ h, uint32_t* __restrict__ ord) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const Line& L = lines[eline[e]];
    h[e] = hash_token(t + L.tok[side], L.len[side]);
    ord[e] = (uint32_t)e;
  }
}

// after a stable sort by hash: run heads, collision check against the run head's bytes
__global__ void k_label_runs(const uint8_t* __restrict__ t, const Line* __restrict__ lines,
                             const int64_t* __restrict__ eline, int64_t m, int side,
                             const unsigned long long* __restrict__ h, const uint32_t* __restrict__ ord,
                             uint32_t* __restrict__ head, unsigned long long* __restrict__ collision) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const bool is_head = i == 0 || h[i] != h[i - 1];
    head[i] = is_head ? 1u : 0u;
    if (!is_head) {
      // compare with the previous element (same hash): equal strings chain to the head
      const Line& a = lines[eline[ord[i]]];
      const Line& b = lines[eline[ord[i - 1]]];
      bool same = a.len[side] == b.len[side];
      for (int c = 0; same && c < a.len[side]; ++c) same = t[a.tok[side] + c] == t[b.tok[side] + c];
      if (!same) atomicMin(collision, (unsigned long long)eline[ord[i]]);
    }
  }
}

// run j's first ordinal (heads are the first element of each run: stable sort)
__global__ void k_run_firsts(const uint32_t* __restrict__ head, const uint32_t* __restrict__ run_idx,
                             const uint32_t* __restrict__ ord, int64_t m, uint32_t* __restrict__ first,
                             uint32_t* __restrict__ runs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    if (head[i]) {
      first[run_idx[i] - 1] = ord[i];
      runs[run_idx[i] - 1] = run_idx[i] - 1;
    }
}

__global__ void k_scatter_u32(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ val, int64_t n,
                              uint32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[idx[i]] = val[i];
}

__global__ void k_iota32(uint32_t* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (uint32_t)i;
}

// label id of every edge: id_of_run[run of its sorted position]
__global__ void k_label_ids(const uint32_t* __restrict__ ord, const uint32_t* __restrict__ run_idx,
                            const uint32_t* __restrict__ id_of_run, int64_t m, int32_t* __restrict__ ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    ids[ord[i]] = (int32_t)id_of_run[run_idx[i] - 1];
}

// ---- blake2b (RFC 7693), one keyed 8-byte message, 8-byte digest ----------------------
__device__ const unsigned long long kB2IV[8] = {
    0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull, 0xa54ff53a5f1d36f1ull,
    0x510e527fade682d1ull, 0x9b05688c2b3e6c1full, 0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
__device__ const uint8_t kB2Sigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

__device__ __forceinline__ unsigned long long rotr64(unsigned long long x, int n) { return (x >> n) | (x << (64 - n)); }

__device__ void b2_compress(unsigned long long h[8], const unsigned long long m[16], unsigned long long t, bool last) {
  unsigned long long v[16];
  for (int i = 0; i < 8; ++i) {
    v[i] = h[i];
    v[i + 8] = kB2IV[i];
  }
  v[12] ^= t;
  if (last) v[14] = ~v[14];
#define B2G(a, b, c, d, x, y)     \
  a = a + b + x;                  \
  d = rotr64(d ^ a, 32);          \
  c = c + d;                      \
  b = rotr64(b ^ c, 24);          \
  a = a + b + y;                  \
  d = rotr64(d ^ a, 16);          \
  c = c + d;                      \
  b = rotr64(b ^ c, 63);
  for (int r = 0; r < 12; ++r) {
    const uint8_t* s = kB2Sigma[r];
    B2G(v[0], v[4], v[8], v[12], m[s[0]], m[s[1]]);
    B2G(v[1], v[5], v[9], v[13], m[s[2]], m[s[3]]);
    B2G(v[2], v[6], v[10], v[14], m[s[4]], m[s[5]]);
    B2G(v[3], v[7], v[11], v[15], m[s[6]], m[s[7]]);
    B2G(v[0], v[5], v[10], v[15], m[s[8]], m[s[9]]);
    B2G(v[1], v[6], v[11], v[12], m[s[10]], m[s[11]]);
    B2G(v[2], v[7], v[8], v[13], m[s[12]], m[s[13]]);
    B2G(v[3], v[4], v[9], v[14], m[s[14]], m[s[15]]);
  }
#undef B2G
  for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
}

// blake2b(msg = ordinal as 8 little-endian bytes, key = seed as 8 little-endian bytes,
// digest_size = 8) read as a little-endian u64 (ingest.py:118-123)
__device__ unsigned long long blake2b_ordinal(unsigned long long seed, unsigned long long ordinal) {
  unsigned long long h[8];
  for (int i = 0; i < 8; ++i) h[i] = kB2IV[i];
  h[0] ^= 0x01010000ull ^ (8ull << 8) ^ 8ull;  // digest 8, key 8, fanout 1, depth 1
  unsigned long long m[16];
  for (int i = 0; i < 16; ++i) m[i] = 0ull;
  m[0] = seed;  // key block (padded to 128 bytes)
  b2_compress(h, m, 128ull, false);
  m[0] = ordinal;  // message block
  b2_compress(h, m, 136ull, true);
  return h[0];
}

// sign of every parsed edge; first failing edge in order (code = ordinal << 2 | kind)
__global__ void k_signs(const Line* __restrict__ lines, const int64_t* __restrict__ eline, int64_t m,
                        bbc_sign_policy pol, int8_t* __restrict__ sign, unsigned long long* __restrict__ err) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const Line& L = lines[eline[e]];
    int8_t s = 1;
    unsigned long long code = ~0ull;
    if (pol.kind == 2) {
      const double unit = __ull2double_rn(blake2b_ordinal(pol.seed, (unsigned long long)e)) * 5.421010862427522e-20;
      s = unit < pol.p_positive ? 1 : -1;
    } else if (L.ntok < 3) {
      code = ((unsigned long long)e << 2) | 1ull;  // MissingValueError
    } else if (pol.kind == 1) {
      s = (pol.at_or_above ? L.value >= pol.threshold : L.value > pol.threshold) ? 1 : -1;
    } else if (L.value == 1.0) {
      s = 1;
    } else if (L.value == 0.0 || L.value == -1.0) {
      s = -1;
    } else {
      code = ((unsigned long long)e << 2) | 2ull;  // InvalidSignValueError
    }
    sign[e] = s;
    if (code != ~0ull) atomicMin(err, code);
  }
}

__global__ void k_pair_keys(const int32_t* __restrict__ uid, const int32_t* __restrict__ vid, int64_t m, int bv,
                            unsigned long long* __restrict__ key, uint32_t* __restrict__ ord) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    key[e] = ((unsigned long long)(uint32_t)uid[e] << bv) | (uint32_t)vid[e];
    ord[e] = (uint32_t)e;
  }
}

// per (u, v) run (stable order = ascending position): the winner is the maximal
// (has timestamp, timestamp, position); first = the run head's position
__global__ void k_dedup_runs(const unsigned long long* __restrict__ key, const uint32_t* __restrict__ ord, int64_t m,
                             const Line* __restrict__ lines, const int64_t* __restrict__ eline,
                             uint32_t* __restrict__ first, uint32_t* __restrict__ winner, uint32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    if (i > 0 && key[i] == key[i - 1]) {
      flag[i] = 0u;
      continue;
    }
    flag[i] = 1u;
    uint32_t best = ord[i];
    const Line& L0 = lines[eline[best]];
    int best_has = L0.ntok == 4;
    long long best_ts = L0.ts;
    for (int64_t j = i + 1; j < m && key[j] == key[i]; ++j) {
      const uint32_t e = ord[j];  // later position than every previous one
      const Line& L = lines[eline[e]];
      const int has = L.ntok == 4;
      if (has > best_has || (has == best_has && (!has || L.ts >= best_ts))) {
        best = e;
        best_has = has;
        best_ts = L.ts;
      }
    }
    first[i] = ord[i];
    winner[i] = best;
  }
}

__global__ void k_final_edges(const uint32_t* __restrict__ win_sorted, int64_t mf, const int32_t* __restrict__ uid,
                              const int32_t* __restrict__ vid, const int8_t* __restrict__ sign,
                              int32_t* __restrict__ ou, int32_t* __restrict__ ov, int8_t* __restrict__ os) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < mf; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t e = win_sorted[i];
    ou[i] = uid[e];
    ov[i] = vid[e];
    os[i] = sign[e];
  }
}

int bits(uint64_t x) {
  int b = 1;
  while ((1ull << b) <= x && b < 64) ++b;
  return b;
}

}  // namespace

struct Ingest {
  int device = 0;
  int64_t n_u = 0, n_v = 0, m = 0;
  int32_t* u = nullptr;
  int32_t* v = nullptr;
  int8_t* s = nullptr;
  ~Ingest() {
    cudaFree(u);
    cudaFree(v);
    cudaFree(s);
  }
};

namespace {

// dense first-occurrence ids of one side's labels; returns the number of labels
int label_ids(cudaStream_t st, const uint8_t* t, const Line* lines, const int64_t* eline, int64_t m, int side,
              int32_t* ids, int64_t* n_labels, unsigned long long* d_collision) {
  Buf h, h2, ord, ord2, head, run_idx, first, runs, first2, runs2, id_of_run, pos, temp, nrun;
  ING_ALLOC(h, m * 8);
  ING_ALLOC(h2, m * 8);
  ING_ALLOC(ord, m * 4);
  ING_ALLOC(ord2, m * 4);
  ING_ALLOC(head, m * 4);
  ING_ALLOC(run_idx, m * 4);
  k_label_hashes<<<grid(m), kT, 0, st>>>(t, lines, eline, m, side, h.as<unsigned long long>(), ord.as<uint32_t>());
  size_t t1 = 0, t2 = 0, t3 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (uint32_t*)nullptr, (uint32_t*)nullptr, (int)m, 0, 64, st);
  cub::DeviceScan::InclusiveSum(nullptr, t2, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)m, st);
  cub::DeviceRadixSort::SortPairs(nullptr, t3, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)m, 0, 32, st);
  const size_t tb = std::max(t1, std::max(t2, t3));
  ING_ALLOC(temp, tb);
  size_t x = tb;
  BBC_CK(cub::DeviceRadixSort::SortPairs(temp.p, x, h.as<unsigned long long>(), h2.as<unsigned long long>(),
                                         ord.as<uint32_t>(), ord2.as<uint32_t>(), (int)m, 0, 64, st));
  k_label_runs<<<grid(m), kT, 0, st>>>(t, lines, eline, m, side, h2.as<unsigned long long>(), ord2.as<uint32_t>(),
                                       head.as<uint32_t>(), d_collision);
  x = tb;
  BBC_CK(cub::DeviceScan::InclusiveSum(temp.p, x, head.as<uint32_t>(), run_idx.as<uint32_t>(), (int)m, st));
  uint32_t nr = 0;
  BBC_CK(cudaMemcpyAsync(&nr, run_idx.as<uint32_t>() + m - 1, 4, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  ING_ALLOC(first, (int64_t)nr * 4);
  ING_ALLOC(runs, (int64_t)nr * 4);
  ING_ALLOC(first2, (int64_t)nr * 4);
  ING_ALLOC(runs2, (int64_t)nr * 4);
  ING_ALLOC(id_of_run, (int64_t)nr * 4);
  ING_ALLOC(pos, (int64_t)nr * 4);
  k_run_firsts<<<grid(m), kT, 0, st>>>(head.as<uint32_t>(), run_idx.as<uint32_t>(), ord2.as<uint32_t>(), m,
                                       first.as<uint32_t>(), runs.as<uint32_t>());
  // runs in first-occurrence order -> dense ids
  x = tb;
  BBC_CK(cub::DeviceRadixSort::SortPairs(temp.p, x, first.as<uint32_t>(), first2.as<uint32_t>(), runs.as<uint32_t>(),
                                         runs2.as<uint32_t>(), (int)nr, 0, bits((uint64_t)m), st));
  k_iota32<<<grid(nr), kT, 0, st>>>(pos.as<uint32_t>(), nr);
  k_scatter_u32<<<grid(nr), kT, 0, st>>>(runs2.as<uint32_t>(), pos.as<uint32_t>(), nr, id_of_run.as<uint32_t>());
  k_label_ids<<<grid(m), kT, 0, st>>>(ord2.as<uint32_t>(), run_idx.as<uint32_t>(), id_of_run.as<uint32_t>(), m, ids);
  BBC_CK(cudaGetLastError());
  BBC_CK(cudaStreamSynchronize(st));
  *n_labels = nr;
  return BBC_OK;
}

int ingest_text(int device, const char* text, int64_t nbytes, const bbc_sign_policy& pol, Ingest& out) {
  BBC_CK(cudaSetDevice(device));
  cudaStream_t st;
  BBC_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
      t_stream = nullptr;
    }
  } guard{st};
  t_stream = st;
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  out.device = device;
  if (nbytes <= 0) return BBC_OK;
  Buf t, nl, nnl, temp, status, lines, scal, eline, ne;
  ING_ALLOC(t, nbytes + 1);
  BBC_CK(cudaMemcpyAsync(t.p, text, (size_t)nbytes, cudaMemcpyHostToDevice, st));
  // newline positions
  ING_ALLOC(nl, (nbytes + 1) * 8);
  ING_ALLOC(nnl, 8);
  thrust::counting_iterator<int64_t> it(0);
  size_t tb = 0;
  cub::DeviceSelect::If(nullptr, tb, it, nl.as<int64_t>(), nnl.as<int64_t>(), nbytes, IsNewline{t.as<uint8_t>()}, st);
  ING_ALLOC(temp, tb);
  BBC_CK(cub::DeviceSelect::If(temp.p, tb, it, nl.as<int64_t>(), nnl.as<int64_t>(), nbytes, IsNewline{t.as<uint8_t>()},
                               st));
  int64_t n_nl = 0;
  char last = 0;
  BBC_CK(cudaMemcpyAsync(&n_nl, nnl.p, 8, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  last = text[nbytes - 1];
  const int64_t nlines = n_nl + (last != '\n' ? 1 : 0);
  if (last != '\n') BBC_CK(cudaMemcpyAsync(nl.as<int64_t>() + n_nl, &nbytes, 8, cudaMemcpyHostToDevice, st));
  // parse
  ING_ALLOC(status, nlines);
  ING_ALLOC(lines, nlines * (int64_t)sizeof(Line));
  ING_ALLOC(scal, 64);
  unsigned long long* d_problem = scal.as<unsigned long long>();
  BBC_CK(cudaMemsetAsync(scal.p, 0xff, 64, st));
  k_parse_lines<<<grid(nlines), kT, 0, st>>>(t.as<uint8_t>(), nbytes, nl.as<int64_t>(), nlines, status.as<uint8_t>(),
                                             lines.as<Line>());
  k_first_problem<<<grid(nlines), kT, 0, st>>>(status.as<uint8_t>(), nlines, d_problem);
  unsigned long long problem = ~0ull;
  BBC_CK(cudaMemcpyAsync(&problem, d_problem, 8, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  if (problem != ~0ull) {
    const int64_t line = (int64_t)(problem >> 2) + 1;
    if ((problem & 3ull) == kMalformed) {
      set_error("line " + std::to_string(line) + ": expected 2-4 tokens", line);
      return BBC_ERR_PARSE;
    }
    set_error("line " + std::to_string(line) + " needs the host loader", line);
    return BBC_ERR_UNSUPPORTED;
  }
  // edges in input order
  ING_ALLOC(eline, nlines * 8);
  ING_ALLOC(ne, 8);
  thrust::counting_iterator<int64_t> lit(0);
  size_t tb2 = 0;
  cub::DeviceSelect::If(nullptr, tb2, lit, eline.as<int64_t>(), ne.as<int64_t>(), nlines, IsEdgeLine{status.as<uint8_t>()},
                        st);
  Buf temp2;
  ING_ALLOC(temp2, tb2);
  BBC_CK(cub::DeviceSelect::If(temp2.p, tb2, lit, eline.as<int64_t>(), ne.as<int64_t>(), nlines,
                               IsEdgeLine{status.as<uint8_t>()}, st));
  int64_t m = 0;
  BBC_CK(cudaMemcpyAsync(&m, ne.p, 8, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  if (m == 0) return BBC_OK;
  if (m >= (1ll << 31)) {
    set_error("more than 2^31 - 1 edges");
    return BBC_ERR_ARG;
  }
  // labels -> dense ids (both sides), collision check
  Buf uid, vid, sign;
  ING_ALLOC(uid, m * 4);
  ING_ALLOC(vid, m * 4);
  ING_ALLOC(sign, m);
  unsigned long long* d_coll = d_problem + 1;
  if (int rc = label_ids(st, t.as<uint8_t>(), lines.as<Line>(), eline.as<int64_t>(), m, 0, uid.as<int32_t>(), &out.n_u,
                         d_coll))
    return rc;
  if (int rc = label_ids(st, t.as<uint8_t>(), lines.as<Line>(), eline.as<int64_t>(), m, 1, vid.as<int32_t>(), &out.n_v,
                         d_coll))
    return rc;
  // signs (policy errors: first failing edge in order)
  unsigned long long* d_err = d_problem + 2;
  k_signs<<<grid(m), kT, 0, st>>>(lines.as<Line>(), eline.as<int64_t>(), m, pol, sign.as<int8_t>(), d_err);
  unsigned long long h2[2];
  BBC_CK(cudaMemcpyAsync(h2, d_problem + 1, 16, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  if (h2[0] != ~0ull) {
    const int64_t line = (int64_t)h2[0] + 1;
    set_error("label hash collision at line " + std::to_string(line) + ": needs the host loader", line);
    return BBC_ERR_UNSUPPORTED;
  }
  if (h2[1] != ~0ull) {
    int64_t eline_h = 0;
    BBC_CK(cudaMemcpy(&eline_h, eline.as<int64_t>() + (h2[1] >> 2), 8, cudaMemcpyDeviceToHost));
    const int64_t line = eline_h + 1;
    if ((h2[1] & 3ull) == 1ull) {
      set_error("edge at line " + std::to_string(line) + " has no value", line);
      return BBC_ERR_MISSING;
    }
    set_error("edge at line " + std::to_string(line) + " has an invalid sign value", line);
    return BBC_ERR_SIGNVAL;
  }
  // dedup_latest: runs of equal (u, v) in position order
  Buf key, key2, ord, ord2, first, winner, flag, firstc, winc, nsel, fsort, wsort, temp3;
  ING_ALLOC(key, m * 8);
  ING_ALLOC(key2, m * 8);
  ING_ALLOC(ord, m * 4);
  ING_ALLOC(ord2, m * 4);
  ING_ALLOC(first, m * 4);
  ING_ALLOC(winner, m * 4);
  ING_ALLOC(flag, m * 4);
  ING_ALLOC(firstc, m * 4);
  ING_ALLOC(winc, m * 4);
  ING_ALLOC(fsort, m * 4);
  ING_ALLOC(wsort, m * 4);
  ING_ALLOC(nsel, 8);
  const int bv = bits((uint64_t)out.n_v);
  k_pair_keys<<<grid(m), kT, 0, st>>>(uid.as<int32_t>(), vid.as<int32_t>(), m, bv, key.as<unsigned long long>(),
                                      ord.as<uint32_t>());
  const int kb = bv + bits((uint64_t)out.n_u);  // compact pair key u << bv | v
  size_t s1 = 0, s2 = 0, s3 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, s1, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                  (uint32_t*)nullptr, (uint32_t*)nullptr, (int)m, 0, 64, st);
  cub::DeviceSelect::Flagged(nullptr, s2, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr, (int*)nullptr,
                             (int)m, st);
  cub::DeviceRadixSort::SortPairs(nullptr, s3, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)m, 0, 32, st);
  const size_t ts = std::max(s1, std::max(s2, s3));
  ING_ALLOC(temp3, ts);
  size_t x = ts;
  BBC_CK(cub::DeviceRadixSort::SortPairs(temp3.p, x, key.as<unsigned long long>(), key2.as<unsigned long long>(),
                                         ord.as<uint32_t>(), ord2.as<uint32_t>(), (int)m, 0, kb, st));
  k_dedup_runs<<<grid(m), kT, 0, st>>>(key2.as<unsigned long long>(), ord2.as<uint32_t>(), m, lines.as<Line>(),
                                       eline.as<int64_t>(), first.as<uint32_t>(), winner.as<uint32_t>(),
                                       flag.as<uint32_t>());
  x = ts;
  BBC_CK(cub::DeviceSelect::Flagged(temp3.p, x, first.as<uint32_t>(), flag.as<uint32_t>(), firstc.as<uint32_t>(),
                                    nsel.as<int>(), (int)m, st));
  x = ts;
  BBC_CK(cub::DeviceSelect::Flagged(temp3.p, x, winner.as<uint32_t>(), flag.as<uint32_t>(), winc.as<uint32_t>(),
                                    nsel.as<int>(), (int)m, st));
  int mf = 0;
  BBC_CK(cudaMemcpyAsync(&mf, nsel.p, 4, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  // first-occurrence order of the surviving pairs
  x = ts;
  BBC_CK(cub::DeviceRadixSort::SortPairs(temp3.p, x, firstc.as<uint32_t>(), fsort.as<uint32_t>(), winc.as<uint32_t>(),
                                         wsort.as<uint32_t>(), mf, 0, bits((uint64_t)m), st));
  BBC_CK(cudaMalloc(&out.u, (size_t)mf * 4 + 16));
  BBC_CK(cudaMalloc(&out.v, (size_t)mf * 4 + 16));
  BBC_CK(cudaMalloc(&out.s, (size_t)mf + 16));
  k_final_edges<<<grid(mf), kT, 0, st>>>(wsort.as<uint32_t>(), mf, uid.as<int32_t>(), vid.as<int32_t>(),
                                         sign.as<int8_t>(), out.u, out.v, out.s);
  BBC_CK(cudaGetLastError());
  BBC_CK(cudaStreamSynchronize(st));
  out.m = mf;
  return BBC_OK;
}

}  // namespace

}  // namespace bbc

struct bbc_ingest {
  bbc::Ingest in;
};

extern "C" {

int bbc_ingest_text(int device, const char* text, int64_t nbytes, const bbc_sign_policy* policy, int64_t counts[3],
                    bbc_ingest** out) {
  if (!out || !counts || (nbytes > 0 && !text) || nbytes < 0) {
    bbc::set_error("bad arguments to bbc_ingest_text");
    return BBC_ERR_ARG;
  }
  *out = nullptr;
  bbc_sign_policy pol{};
  if (policy) pol = *policy;
  if (pol.kind < 0 || pol.kind > 2 || (pol.kind == 2 && !(pol.p_positive >= 0.0 && pol.p_positive <= 1.0))) {
    bbc::set_error("bad sign policy");
    return BBC_ERR_ARG;
  }
  bbc_ingest* h = new bbc_ingest;
  int rc = bbc::ingest_text(device, text, nbytes, pol, h->in);
  if (rc) {
    delete h;
    return rc;
  }
  counts[0] = h->in.n_u;
  counts[1] = h->in.n_v;
  counts[2] = h->in.m;
  *out = h;
  return BBC_OK;
}

int bbc_ingest_edges(bbc_ingest* h, int32_t* u, int32_t* v, int8_t* sign) {
  if (!h || (h->in.m > 0 && (!u || !v || !sign))) {
    bbc::set_error("bad arguments to bbc_ingest_edges");
    return BBC_ERR_ARG;
  }
  if (h->in.m == 0) return BBC_OK;
  BBC_CK(cudaSetDevice(h->in.device));
  BBC_CK(cudaMemcpy(u, h->in.u, (size_t)h->in.m * 4, cudaMemcpyDeviceToHost));
  BBC_CK(cudaMemcpy(v, h->in.v, (size_t)h->in.m * 4, cudaMemcpyDeviceToHost));
  BBC_CK(cudaMemcpy(sign, h->in.s, (size_t)h->in.m, cudaMemcpyDeviceToHost));
  return BBC_OK;
}

int bbc_ingest_graph(bbc_ingest* h, int32_t side_rule, bbc_graph** out) {
  if (!h || !out) {
    bbc::set_error("bad arguments to bbc_ingest_graph");
    return BBC_ERR_ARG;
  }
  return bbc_graph_create_device(h->in.device, h->in.n_u, h->in.n_v, h->in.m, h->in.u, h->in.v, h->in.s, side_rule,
                                 out);
}

void bbc_ingest_destroy(bbc_ingest* h) { delete h; }

}  // extern "C"
