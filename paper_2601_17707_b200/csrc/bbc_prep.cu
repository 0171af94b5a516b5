// Device-side preprocessing: validation, degrees, anchor-side choice, priority
// ranks, signed CSR with the sign packed into the adjacency word, per-edge
// admitted-suffix records, per-anchor work and the G-BBC++ task order.
//
// Reference behaviour restated (paths under /root/reference/pkg/src/bbcount):
//   graph.py:109-114  range check per edge, u before v, first offending edge
//   graph.py:114      EdgeSign(sign): only +1 / -1 are valid signs
//   graph.py:116-121  sort by (u, v); DuplicateEdgeError(u, v) at the first equal
//                     pair in that order, regardless of sign
//   graph.py:230-235  priority rank = position in ascending (degree, id) order
//   graph.py:174-176  min_side (smaller partition, ties to U)
//   buckets.py:53-57  wedge_scan_bound; admitted wedges W_S = sum_c C(deg c, 2)
//   tiled.py:213-214  G-BBC++ order: descending work estimate, ties by id
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "bbc_internal.cuh"

namespace bbc {

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n, int num_sms) {
  int64_t b = (n + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)num_sms * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

inline int bits_for(uint64_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

// First failing edge in input order: code = edge * 4 + kind, kind 0 u-range,
// 1 v-range, 2 sign.  Degrees of valid edges are accumulated.
__device__ __forceinline__ void validate_edge(int64_t i, int32_t uu, int32_t vv, int32_t ss, int64_t n_u, int64_t n_v,
                                              unsigned int* __restrict__ deg_u, unsigned int* __restrict__ deg_v,
                                              unsigned long long* __restrict__ err) {
  unsigned long long code = ~0ull;
  if (uu < 0 || uu >= n_u)
    code = (unsigned long long)i * 4ull;
  else if (vv < 0 || vv >= n_v)
    code = (unsigned long long)i * 4ull + 1ull;
  else if (ss != 1 && ss != -1)
    code = (unsigned long long)i * 4ull + 2ull;
  if (code != ~0ull) {
    atomicMin(err, code);
  } else {
    atomicAdd(&deg_u[uu], 1u);
    atomicAdd(&deg_v[vv], 1u);
  }
}

// Four edges per thread with 16-byte loads of u / v and one 4-byte load of signs when the
// arrays are 16-byte aligned (the tail and unaligned inputs go edge by edge).
__global__ void k_validate_degrees(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                                   const int8_t* __restrict__ s, int64_t m, int64_t base, int64_t n_u, int64_t n_v,
                                   unsigned int* __restrict__ deg_u, unsigned int* __restrict__ deg_v,
                                   unsigned long long* __restrict__ err) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(v)) & 15u) == 0 &&
                   (reinterpret_cast<uintptr_t>(s) & 3u) == 0;
  int64_t done = 0;
  if (vec) {
    const int64_t m4 = m / 4;
    for (int64_t q = tid; q < m4; q += nt) {
      const int4 u4 = reinterpret_cast<const int4*>(u)[q], v4 = reinterpret_cast<const int4*>(v)[q];
      const int32_t s4 = reinterpret_cast<const int32_t*>(s)[q];
      validate_edge(base + 4 * q + 0, u4.x, v4.x, (int8_t)(s4 & 0xff), n_u, n_v, deg_u, deg_v, err);
      validate_edge(base + 4 * q + 1, u4.y, v4.y, (int8_t)((s4 >> 8) & 0xff), n_u, n_v, deg_u, deg_v, err);
      validate_edge(base + 4 * q + 2, u4.z, v4.z, (int8_t)((s4 >> 16) & 0xff), n_u, n_v, deg_u, deg_v, err);
      validate_edge(base + 4 * q + 3, u4.w, v4.w, (int8_t)(s4 >> 24), n_u, n_v, deg_u, deg_v, err);
    }
    done = m4 * 4;
  }
  for (int64_t i = done + tid; i < m; i += nt)
    validate_edge(base + i, u[i], v[i], s[i], n_u, n_v, deg_u, deg_v, err);
}

// sum C(d, 2) and max d over one degree array
__global__ void k_wedge_sum(const unsigned int* __restrict__ deg, int64_t n, unsigned long long* __restrict__ out_sum,
                            unsigned int* __restrict__ out_max) {
  unsigned long long acc = 0;
  unsigned int mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long d = deg[i];
    acc += d * (d - (d > 0)) / 2;
    mx = max(mx, (unsigned int)d);
  }
  for (int o = 16; o; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out_sum, acc);
    atomicMax(out_max, mx);
  }
}

__global__ void k_iota(uint32_t* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (uint32_t)i;
}

__global__ void k_scatter_rank(const uint32_t* __restrict__ rank_to_id, int64_t n, uint32_t* __restrict__ rank) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    rank[rank_to_id[i]] = (uint32_t)i;
}

// centre-major key: c << cs | rank(a) << 1 | neg, cs = rank bits + 1 (the radix sort then
// needs only bits(nc) + cs bits: 40 instead of 52 passes' worth on config 2)
__global__ void k_centre_keys(const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                              const int8_t* __restrict__ s, int64_t m, int side, int cs,
                              const uint32_t* __restrict__ rank, unsigned long long* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t a = side == 0 ? (uint32_t)u[i] : (uint32_t)v[i];
    uint32_t c = side == 0 ? (uint32_t)v[i] : (uint32_t)u[i];
    keys[i] = ((unsigned long long)c << cs) | ((unsigned long long)rank[a] << 1) | (s[i] < 0 ? 1ull : 0ull);
  }
}

// adjacency words + duplicate detection + keys for the anchor-major regroup
__global__ void k_adj_dup(const unsigned long long* __restrict__ keys, int64_t m, int side, int cs,
                          const uint32_t* __restrict__ rank_to_id, uint32_t* __restrict__ adj,
                          uint32_t* __restrict__ akey, uint32_t* __restrict__ aval,
                          unsigned long long* __restrict__ dup) {
  const unsigned long long rmask = (1ull << (cs - 1)) - 1ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long k = keys[i];
    uint32_t r = (uint32_t)((k >> 1) & rmask);
    adj[i] = r | ((uint32_t)(k & 1ull) << 31);
    akey[i] = r;
    aval[i] = (uint32_t)i;
    if (i > 0 && (keys[i - 1] >> 1) == (k >> 1)) {
      unsigned long long c = k >> cs, a = rank_to_id[r];
      unsigned long long pair = side == 0 ? ((a << 32) | c) : ((c << 32) | a);
      atomicMin(dup, pair);
    }
  }
}

// records in anchor-rank order: rec[j] = {(i + 1) | neg << 31, c}; the admitted suffix of
// centre c's list is [i + 1, coff[c + 1])
// (and awork: the records' admitted wedges coff[c + 1] - (i + 1) summed per anchor rank
// r = akey[j]; records of one anchor are contiguous, so a warp segmented scan leaves one
// 64-bit atomic per anchor segment and warp)
__global__ void k_records(const uint32_t* __restrict__ pos_sorted, const uint32_t* __restrict__ akey,
                          const unsigned long long* __restrict__ keys, int64_t m, int cs,
                          const uint32_t* __restrict__ coff, uint2* __restrict__ rec,
                          unsigned long long* __restrict__ awork) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; base < m; base += stride) {
    const int64_t j = base + lane;
    unsigned long long w = 0;
    uint32_t r = 0xffffffffu;
    if (j < m) {
      const uint32_t i = pos_sorted[j];
      const unsigned long long k = keys[i];
      const uint32_t c = (uint32_t)(k >> cs);
      rec[j] = make_uint2((i + 1u) | ((uint32_t)(k & 1ull) << 31), c);
      w = coff[c + 1] - (i + 1u);
      r = akey[j];
    }
    // inclusive segmented sum over lanes with equal r (contiguous)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
      const uint32_t ry = __shfl_up_sync(0xffffffffu, r, o);
      if (lane >= o && ry == r) w += y;
    }
    const uint32_t rn = __shfl_down_sync(0xffffffffu, r, 1);
    if (j < m && (lane == 31 || rn != r)) atomicAdd(&awork[r], w);
  }
}

// centres with list length > {0, 4, 16, 64, 256, 1024, 4096, 16384}
__global__ void k_count_rows(const uint32_t* __restrict__ coff, int64_t nc, unsigned int* __restrict__ cnt) {
  unsigned int c8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t d = coff[c + 1] - coff[c];
    c8[0] += d > 0u;
    c8[1] += d > 4u;
    c8[2] += d > 16u;
    c8[3] += d > 64u;
    c8[4] += d > 256u;
    c8[5] += d > 1024u;
    c8[6] += d > 4096u;
    c8[7] += d > 16384u;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    unsigned int v = c8[i];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&cnt[i], v);
  }
}

// table rows for centres with lists longer than min_deg (row order is arbitrary)
__global__ void k_table_rows(const uint32_t* __restrict__ coff, int64_t nc, uint32_t min_deg,
                             uint32_t* __restrict__ brow, unsigned int* __restrict__ rows) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x)
    brow[c] = (coff[c + 1] - coff[c] > min_deg) ? atomicAdd(rows, 1u) : 0xffffffffu;
}

// band table: row brow[c] holds, for j in [0, nbands), the first position of c's list
// whose rank is >= n - j * t (j = 0: the list end).  Lists are rank-sorted.
__global__ void k_band_table(const uint32_t* __restrict__ adj, const uint32_t* __restrict__ coff,
                             const uint32_t* __restrict__ brow, int64_t nc, uint32_t nbands, uint32_t t, uint32_t n,
                             uint32_t* __restrict__ bnd) {
  const int64_t total = nc * (int64_t)nbands;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / nbands;
    const uint32_t row = brow[c];
    if (row == 0xffffffffu) continue;
    const uint32_t j = (uint32_t)(e - c * nbands);
    uint32_t lo = coff[c], hi = coff[c + 1];
    if (j > 0) {
      const int64_t x = (int64_t)n - (int64_t)j * t;
      if (x <= 0) {
        hi = lo;
      } else {
        while (lo < hi) {
          uint32_t mid = (lo + hi) >> 1;
          if ((int64_t)(adj[mid] & 0x7fffffffu) < x)
            lo = mid + 1;
          else
            hi = mid;
        }
      }
    }
    bnd[(size_t)row * nbands + j] = hi;
  }
}

// All device memory of a handle is stream-ordered (cudaMallocAsync on the handle's
// stream) from the device's default pool, which keeps freed blocks cached: the
// preprocessing temporaries of repeated graph builds (bench e2e) then cost no
// cudaMalloc / cudaFree round trips.
thread_local cudaStream_t t_alloc_stream = nullptr;

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, t_alloc_stream);
  }
  template <typename T>
  T* as() {
    return static_cast<T*>(p);
  }
};

int alloc(void** p, size_t bytes) {
  cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 16, t_alloc_stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("device allocation of ") + std::to_string(bytes) + " bytes failed: " +
              cudaGetErrorString(e));
    return BBC_ERR_NOMEM;
  }
  return BBC_OK;
}

#define BBC_ALLOC(ptr, bytes)                                  \
  do {                                                         \
    int _r = alloc((void**)&(ptr), (bytes));                   \
    if (_r) return _r;                                         \
  } while (0)

void free_graph_arrays(Graph& g) {
  void* ptrs[] = {g.adj, g.coff, g.rec, g.aoff, g.awork, g.order, g.rank_to_id, g.acc, g.queue, g.bnd, g.brow};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, g.stream);
  cudaFree(g.block_work);  // (re)allocated with cudaMalloc by the count
  cudaStreamSynchronize(g.stream);
  g.bnd = nullptr;
  g.brow = nullptr;
  g.adj = g.coff = g.aoff = g.order = g.rank_to_id = nullptr;
  g.rec = nullptr;
  g.awork = g.acc = g.block_work = nullptr;
  g.queue = nullptr;
}

// Full pipeline on device arrays.  Returns a bbc_status.
// Host edge arrays to upload into the device buffers during the build (chunked, each
// chunk validated while the next one is copied).
struct Upload {
  const int32_t* u;
  const int32_t* v;
  const int8_t* s;
};

int build_on_device(Graph& g, const int32_t* du, const int32_t* dv, const int8_t* ds, int side_rule,
                    const Upload* up = nullptr) {
  cudaStream_t st = g.stream;
  const int64_t m = g.m, n_u = g.n_u, n_v = g.n_v;
  const int sms = g.num_sms;

  // ---- K1: validation + degrees ------------------------------------------------
  DevBuf deg_u, deg_v, scal;
  BBC_ALLOC(deg_u.p, (size_t)(n_u + 1) * 4);
  BBC_ALLOC(deg_v.p, (size_t)(n_v + 1) * 4);
  BBC_ALLOC(scal.p, 64);
  unsigned long long* d_err = scal.as<unsigned long long>();      // [0] err, [1] dup
  unsigned long long* d_wsum = d_err + 2;                          // [2] W_U, [3] W_V
  unsigned int* d_max = reinterpret_cast<unsigned int*>(d_err + 4);  // [0] max deg_u, [1] max deg_v
  BBC_CK(cudaMemsetAsync(deg_u.p, 0, (size_t)(n_u + 1) * 4, st));
  BBC_CK(cudaMemsetAsync(deg_v.p, 0, (size_t)(n_v + 1) * 4, st));
  BBC_CK(cudaMemsetAsync(scal.p, 0, 64, st));
  BBC_CK(cudaMemsetAsync(scal.p, 0xff, 16, st));
  if (m > 0 && up) {
    // the upload runs on a copy stream in chunks; chunk i is validated on the build stream
    // as soon as it has landed, overlapping the copy of chunk i + 1
    cudaStream_t cs;
    BBC_CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaEvent_t ready;
    BBC_CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    BBC_CK(cudaEventRecord(ready, st));  // the upload buffers were allocated on st
    BBC_CK(cudaStreamWaitEvent(cs, ready, 0));
    cudaEventDestroy(ready);
    const int64_t nch = m >= (1ll << 22) ? 8 : 1;
    const int64_t chunk = ((m + nch - 1) / nch + 3) & ~3ll;  // multiples of 4 keep the vector loads aligned
    for (int64_t off = 0; off < m; off += chunk) {
      const int64_t len = std::min(chunk, m - off);
      BBC_CK(cudaMemcpyAsync((void*)(du + off), up->u + off, (size_t)len * 4, cudaMemcpyHostToDevice, cs));
      BBC_CK(cudaMemcpyAsync((void*)(dv + off), up->v + off, (size_t)len * 4, cudaMemcpyHostToDevice, cs));
      BBC_CK(cudaMemcpyAsync((void*)(ds + off), up->s + off, (size_t)len, cudaMemcpyHostToDevice, cs));
      cudaEvent_t ev;
      BBC_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      BBC_CK(cudaEventRecord(ev, cs));
      BBC_CK(cudaStreamWaitEvent(st, ev, 0));
      cudaEventDestroy(ev);
      k_validate_degrees<<<grid_for(len, sms), kThreads, 0, st>>>(du + off, dv + off, ds + off, len, off, n_u, n_v,
                                                                  deg_u.as<unsigned int>(), deg_v.as<unsigned int>(),
                                                                  d_err);
    }
    cudaStreamDestroy(cs);
  } else if (m > 0) {
    k_validate_degrees<<<grid_for(m, sms), kThreads, 0, st>>>(du, dv, ds, m, 0, n_u, n_v, deg_u.as<unsigned int>(),
                                                              deg_v.as<unsigned int>(), d_err);
  }
  // W_U = sum over V of C(deg_v, 2) (anchoring U), W_V = sum over U of C(deg_u, 2)
  k_wedge_sum<<<grid_for(n_v, sms), kThreads, 0, st>>>(deg_v.as<unsigned int>(), n_v, d_wsum + 0, d_max + 1);
  k_wedge_sum<<<grid_for(n_u, sms), kThreads, 0, st>>>(deg_u.as<unsigned int>(), n_u, d_wsum + 1, d_max + 0);
  BBC_CK(cudaGetLastError());
  unsigned long long h_scal[8];
  BBC_CK(cudaMemcpyAsync(h_scal, scal.p, 64, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  if (h_scal[0] != ~0ull) {
    unsigned long long code = h_scal[0];
    int64_t edge = (int64_t)(code >> 2);
    int kind = (int)(code & 3ull);
    int32_t val_u = 0, val_v = 0;
    int8_t val_s = 0;
    cudaMemcpy(&val_u, du + edge, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&val_v, dv + edge, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&val_s, ds + edge, 1, cudaMemcpyDeviceToHost);
    if (kind == 0) {
      set_error("u index " + std::to_string(val_u) + " out of range [0, " + std::to_string(n_u) + ")", edge * 2);
      return BBC_ERR_RANGE;
    }
    if (kind == 1) {
      set_error("v index " + std::to_string(val_v) + " out of range [0, " + std::to_string(n_v) + ")", edge * 2 + 1);
      return BBC_ERR_RANGE;
    }
    set_error(std::to_string((int)val_s) + " is not a valid EdgeSign", edge);
    return BBC_ERR_ARG;
  }
  g.w_u = h_scal[2];
  g.w_v = h_scal[3];
  uint32_t maxdeg[2];
  std::memcpy(maxdeg, &h_scal[4], 8);

  // ---- K3: side choice ------------------------------------------------------------
  int side;
  if (side_rule == BBC_SIDE_U)
    side = 0;
  else if (side_rule == BBC_SIDE_V)
    side = 1;
  else if (side_rule == BBC_SIDE_MIN)
    side = n_u <= n_v ? 0 : 1;
  else
    side = (g.w_u < g.w_v || (g.w_u == g.w_v && n_u <= n_v)) ? 0 : 1;
  g.side = side;
  g.n = side == 0 ? n_u : n_v;
  g.nc = side == 0 ? n_v : n_u;
  g.w_s = side == 0 ? g.w_u : g.w_v;
  g.max_anchor_deg = maxdeg[side];
  const int64_t n = g.n, nc = g.nc;
  unsigned int* deg_s = side == 0 ? deg_u.as<unsigned int>() : deg_v.as<unsigned int>();
  unsigned int* deg_c = side == 0 ? deg_v.as<unsigned int>() : deg_u.as<unsigned int>();

  BBC_ALLOC(g.adj, (size_t)(m + 8) * 4);
  BBC_ALLOC(g.coff, (size_t)(nc + 1) * 4);
  BBC_ALLOC(g.rec, (size_t)(m + 1) * 8);
  BBC_ALLOC(g.aoff, (size_t)(n + 1) * 4);
  BBC_ALLOC(g.awork, (size_t)(n + 1) * 8);
  BBC_ALLOC(g.order, (size_t)(n + 1) * 4);
  BBC_ALLOC(g.rank_to_id, (size_t)(n + 1) * 4);
  BBC_CK(cudaMemsetAsync(g.adj + m, 0, 8 * 4, st));

  // ---- K2: priority ranks: stable sort of ids by degree ------------------------------
  DevBuf ids, sorted_deg, rank, keys_a, keys_b, akey_a, akey_b, aval_a, aval_b, temp;
  BBC_ALLOC(ids.p, (size_t)(n + 1) * 4);
  BBC_ALLOC(sorted_deg.p, (size_t)(n + 1) * 4);
  BBC_ALLOC(rank.p, (size_t)(n + 1) * 4);
  BBC_ALLOC(keys_a.p, (size_t)(m + 1) * 8);
  BBC_ALLOC(keys_b.p, (size_t)(m + 1) * 8);
  BBC_ALLOC(akey_a.p, (size_t)(m + 1) * 4);
  BBC_ALLOC(akey_b.p, (size_t)(m + 1) * 4);
  BBC_ALLOC(aval_a.p, (size_t)(m + 1) * 4);
  BBC_ALLOC(aval_b.p, (size_t)(m + 1) * 4);

  const int deg_bits = std::max(1, bits_for(maxdeg[side]));
  const int rank_bits = std::max(1, bits_for((uint64_t)n));
  const int cs = rank_bits + 1;  // centre shift of the centre-major keys
  const int key_bits = cs + std::max(1, bits_for((uint64_t)nc));
  size_t t1 = 0, t2 = 0, t3 = 0, t4 = 0, t5 = 0, t6 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, (unsigned int*)nullptr, (unsigned int*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)n, 0, deg_bits, st);
  cub::DeviceRadixSort::SortKeys(nullptr, t2, (unsigned long long*)nullptr, (unsigned long long*)nullptr, (int)m, 0,
                                 key_bits, st);
  cub::DeviceRadixSort::SortPairs(nullptr, t3, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)m, 0, rank_bits, st);
  cub::DeviceScan::ExclusiveSum(nullptr, t4, (unsigned int*)nullptr, (uint32_t*)nullptr, (int)(std::max(n, nc) + 1), st);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, t5, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                            (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, 0, 64, st);
  t6 = std::max(std::max(std::max(t1, t2), std::max(t3, t4)), t5);
  BBC_ALLOC(temp.p, t6);

  if (n > 0) {
    k_iota<<<grid_for(n, sms), kThreads, 0, st>>>(ids.as<uint32_t>(), n);
    size_t tb = t6;
    BBC_CK(cub::DeviceRadixSort::SortPairs(temp.p, tb, deg_s, sorted_deg.as<unsigned int>(), ids.as<uint32_t>(),
                                           g.rank_to_id, (int)n, 0, deg_bits, st));
    k_scatter_rank<<<grid_for(n, sms), kThreads, 0, st>>>(g.rank_to_id, n, rank.as<uint32_t>());
  }

  // ---- K4: signed centre CSR ------------------------------------------------------------
  {
    size_t tb = t6;
    BBC_CK(cub::DeviceScan::ExclusiveSum(temp.p, tb, deg_c, g.coff, (int)(nc + 1), st));
  }
  if (m > 0) {
    k_centre_keys<<<grid_for(m, sms), kThreads, 0, st>>>(du, dv, ds, m, side, cs, rank.as<uint32_t>(),
                                                         keys_a.as<unsigned long long>());
    size_t tb = t6;
    BBC_CK(cub::DeviceRadixSort::SortKeys(temp.p, tb, keys_a.as<unsigned long long>(),
                                          keys_b.as<unsigned long long>(), (int)m, 0, key_bits, st));
    k_adj_dup<<<grid_for(m, sms), kThreads, 0, st>>>(keys_b.as<unsigned long long>(), m, side, cs, g.rank_to_id, g.adj,
                                                     akey_a.as<uint32_t>(), aval_a.as<uint32_t>(), d_err + 1);
    BBC_CK(cudaGetLastError());
    unsigned long long dup = ~0ull;
    BBC_CK(cudaMemcpyAsync(&dup, d_err + 1, 8, cudaMemcpyDeviceToHost, st));
    BBC_CK(cudaStreamSynchronize(st));
    if (dup != ~0ull) {
      int64_t uu = (int64_t)(dup >> 32), vv = (int64_t)(dup & 0xffffffffull);
      set_error("duplicate edge (" + std::to_string(uu) + ", " + std::to_string(vv) + ")", (int64_t)dup);
      return BBC_ERR_DUP;
    }
    // ---- records grouped by anchor rank ----
    tb = t6;
    BBC_CK(cub::DeviceRadixSort::SortPairs(temp.p, tb, akey_a.as<uint32_t>(), akey_b.as<uint32_t>(),
                                           aval_a.as<uint32_t>(), aval_b.as<uint32_t>(), (int)m, 0, rank_bits, st));
    BBC_CK(cudaMemsetAsync(g.awork, 0, (size_t)(n + 1) * 8, st));
    k_records<<<grid_for(m, sms), kThreads, 0, st>>>(aval_b.as<uint32_t>(), akey_b.as<uint32_t>(),
                                                     keys_b.as<unsigned long long>(), m, cs, g.coff, g.rec, g.awork);
  }
  // anchor offsets from degrees in rank order
  if (n > 0) {
    BBC_CK(cudaMemsetAsync(sorted_deg.as<unsigned int>() + n, 0, 4, st));
    size_t tb = t6;
    BBC_CK(cub::DeviceScan::ExclusiveSum(temp.p, tb, sorted_deg.as<unsigned int>(), g.aoff, (int)(n + 1), st));
  } else {
    BBC_CK(cudaMemsetAsync(g.aoff, 0, 4, st));
  }

  // ---- K5: per-anchor work and the G-BBC++ dispatch order ---------------------------------
  if (n > 0) {
    if (m == 0) BBC_CK(cudaMemsetAsync(g.awork, 0, (size_t)n * 8, st));
    k_iota<<<grid_for(n, sms), kThreads, 0, st>>>(ids.as<uint32_t>(), n);
    // descending work; LSD radix descending sort is stable -> ties in ascending rank
    unsigned long long* work_sorted = keys_a.as<unsigned long long>();
    size_t tb = t6;
    BBC_CK(cub::DeviceRadixSort::SortPairsDescending(temp.p, tb, g.awork, work_sorted, ids.as<uint32_t>(), g.order,
                                                     (int)n, 0, 64, st));
  }
  BBC_CK(cudaGetLastError());

  // band table: rows only for centres whose list is longer than
  // kTableMinDeg (short lists are binary-searched within one or two cache lines), and
  // only when the rows fit a memory budget; brow[c] = row of c or ~0.
  {
    int span16 = count_span16(g);
    if (span16 <= 0) return BBC_ERR_CUDA;
    g.t16 = (uint32_t)span16;
    g.nbands = (uint32_t)((n + span16 - 1) / span16);
    if (g.nbands == 0) g.nbands = 1;
    if (nc > 0 && n > 0) {
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      size_t budget = (size_t)8192 << 20;  // beyond it the kernel searches
      budget = std::min<size_t>(budget, free_b / 4);
      // smallest list-length threshold whose rows fit the budget (0: every centre)
      DevBuf rowcnt;
      BBC_ALLOC(rowcnt.p, 64);
      const uint32_t thresholds[8] = {0u, 4u, 16u, 64u, 256u, 1024u, 4096u, 16384u};
      BBC_CK(cudaMemsetAsync(rowcnt.p, 0, 64, st));
      k_count_rows<<<grid_for(nc, sms), kThreads, 0, st>>>(g.coff, nc, rowcnt.as<unsigned int>());
      unsigned int cnt[8];
      BBC_CK(cudaMemcpyAsync(cnt, rowcnt.p, 32, cudaMemcpyDeviceToHost, st));
      BBC_CK(cudaStreamSynchronize(st));
      int pick = -1;
      for (int i = 0; i < 8 && pick < 0; ++i)
        if ((size_t)cnt[i] * g.nbands * 4 <= budget) pick = i;
      unsigned int rows = 0;
      if (pick >= 0 && cnt[pick] > 0) {
        BBC_ALLOC(g.brow, (size_t)(nc + 1) * 4);
        BBC_CK(cudaMemsetAsync(rowcnt.p, 0, 16, st));
        k_table_rows<<<grid_for(nc, sms), kThreads, 0, st>>>(g.coff, nc, thresholds[pick], g.brow,
                                                             rowcnt.as<unsigned int>());
        BBC_CK(cudaMemcpyAsync(&rows, rowcnt.p, 4, cudaMemcpyDeviceToHost, st));
        BBC_CK(cudaStreamSynchronize(st));
      }
      const size_t need = (size_t)rows * g.nbands * 4;
      if (rows > 0 && need <= budget) {
        BBC_ALLOC(g.bnd, need);
        k_band_table<<<grid_for(nc * (int64_t)g.nbands, sms), kThreads, 0, st>>>(
            g.adj, g.coff, g.brow, nc, g.nbands, g.t16, (uint32_t)n, g.bnd);
        BBC_CK(cudaGetLastError());
      }
    }
  }

  BBC_ALLOC(g.acc, 128);
  BBC_ALLOC(g.queue, 64);
  g.block_work_cap = std::max(1, sms * 32);
  BBC_ALLOC(g.block_work, (size_t)g.block_work_cap * 16);
  BBC_CK(cudaStreamSynchronize(st));
  return BBC_OK;
}

int init_handle(Graph& g, int device, int64_t n_u, int64_t n_v, int64_t m) {
  if (n_u < 0 || n_v < 0 || m < 0) {
    set_error("sizes must be non-negative");
    return BBC_ERR_ARG;
  }
  if (n_u >= (1ll << 31) || n_v >= (1ll << 31) || m >= (1ll << 31) - 16) {
    set_error("graph too large: vertex counts and edge count must be below 2^31");
    return BBC_ERR_ARG;
  }
  int ndev = 0;
  BBC_CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) {
    set_error("device " + std::to_string(device) + " not available (" + std::to_string(ndev) + " visible)");
    return BBC_ERR_ARG;
  }
  BBC_CK(cudaSetDevice(device));
  g.device = device;
  g.n_u = n_u;
  g.n_v = n_v;
  g.m = m;
  BBC_CK(cudaDeviceGetAttribute(&g.num_sms, cudaDevAttrMultiProcessorCount, device));
  BBC_CK(cudaDeviceGetAttribute(&g.max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  BBC_CK(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;  // keep freed blocks for the next build
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
  BBC_CK(cudaEventCreate(&g.ev0));
  BBC_CK(cudaEventCreate(&g.ev1));
  return BBC_OK;
}

int create_common(int device, int64_t n_u, int64_t n_v, int64_t m, const int32_t* u, const int32_t* v,
                  const int8_t* s, int32_t side_rule, bool host, bbc_graph** out) {
  if (!out) {
    set_error("out must not be null");
    return BBC_ERR_ARG;
  }
  *out = nullptr;
  if (side_rule < -1 || side_rule > 2) {
    set_error("side_rule must be -1, 0, 1 or 2");
    return BBC_ERR_ARG;
  }
  if (m > 0 && (!u || !v || !s)) {
    set_error("edge arrays must not be null");
    return BBC_ERR_ARG;
  }
  bbc_graph* h = new bbc_graph();
  Graph& g = h->g;
  int rc = init_handle(g, device, n_u, n_v, m);
  if (rc) {
    delete h;
    return rc;
  }
  t_alloc_stream = g.stream;
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  {  // upload buffers are released (stream-ordered) before any error teardown
  DevBuf du, dv, ds;
  const int32_t* pu = u;
  const int32_t* pv = v;
  const int8_t* ps = s;
  if (host && m > 0) {
    rc = alloc(&du.p, (size_t)m * 4);
    if (!rc) rc = alloc(&dv.p, (size_t)m * 4);
    if (!rc) rc = alloc(&ds.p, (size_t)m);
    pu = du.as<int32_t>();
    pv = dv.as<int32_t>();
    ps = ds.as<int8_t>();
  }
  if (!rc) {
    // device time of the build; with host arrays it includes their (overlapped) upload
    cudaEventRecord(t0, g.stream);
    const Upload up{u, v, s};
    rc = build_on_device(g, pu, pv, ps, side_rule, host && m > 0 ? &up : nullptr);
    cudaEventRecord(t1, g.stream);
    cudaEventSynchronize(t1);
    cudaEventElapsedTime(&g.preprocess_ms, t0, t1);
  }
  }
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  if (rc) {
    bbc_graph_destroy(h);
    return rc;
  }
  *out = h;
  return BBC_OK;
}

}  // namespace

int create_graph(int device, int64_t n_u, int64_t n_v, int64_t m, const int32_t* u, const int32_t* v,
                 const int8_t* s, int32_t side_rule, bool host, bbc_graph** out) {
  return create_common(device, n_u, n_v, m, u, v, s, side_rule, host, out);
}

void destroy_graph(Graph& g) {
  if (g.stream) {
    cudaSetDevice(g.device);
    cudaStreamSynchronize(g.stream);
  }
  free_graph_arrays(g);
  if (g.ev0) cudaEventDestroy(g.ev0);
  if (g.ev1) cudaEventDestroy(g.ev1);
  if (g.stream) cudaStreamDestroy(g.stream);
  g.stream = nullptr;
  g.ev0 = g.ev1 = nullptr;
}

}  // namespace bbc

extern "C" {

int bbc_graph_create(int device, int64_t n_u, int64_t n_v, int64_t m, const int32_t* u, const int32_t* v,
                     const int8_t* sign, int32_t side_rule, bbc_graph** out) {
  return bbc::create_common(device, n_u, n_v, m, u, v, sign, side_rule, true, out);
}

int bbc_graph_create_device(int device, int64_t n_u, int64_t n_v, int64_t m, const int32_t* d_u, const int32_t* d_v,
                            const int8_t* d_sign, int32_t side_rule, bbc_graph** out) {
  return bbc::create_common(device, n_u, n_v, m, d_u, d_v, d_sign, side_rule, false, out);
}

void bbc_graph_destroy(bbc_graph* h) {
  if (!h) return;
  bbc::destroy_graph(h->g);
  delete h;
}

}  // extern "C"
