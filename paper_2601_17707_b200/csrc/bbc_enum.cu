// Device enumeration of every butterfly, replacing oracle.enumerate_butterflies
// (pkg/src/bbcount/oracle.py:73-107): each 4-cycle once, canonical (u1 < u2, v1 < v2),
// in (u1, u2, v1, v2) lexicographic order, signs in the order (u1v1, u1v2, u2v1, u2v2).
//
// The reference pivots on vertex pairs of the smaller side and intersects neighbour sets
// (:85-104).  Here the pairs come from wedges instead:
//   1. centre lists: edges sorted by (centre, pivot) -- CUB radix sort;
//   2. every wedge (a < b) through centre c, generated in ascending c (one thread per
//      list entry a, looping over the later entries b);
//   3. stable radix sort of the wedges by (a, b): ties keep ascending c, so a run of
//      equal (a, b) lists the pair's common centres in order;
//   4. a run of r centres yields C(r, 2) butterflies (c_i, c_j), i < j -- the exclusive
//      scan of C(r, 2) over runs gives every wedge its output slots;
//   5. pivot V: outputs are (u_i, u_j, a, b) already ordered by (v1, v2); one stable
//      sort by (u1, u2) makes the order (u1, u2, v1, v2), as the reference's final sort
//      (:104).
// Test-scale API (the reference calls it for desk-scale validation): wedges and outputs
// are materialised.
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "bbc_internal.cuh"

namespace bbc {
namespace {

constexpr int kT = 256;

inline unsigned grid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, 1 << 20)); }

__global__ void k_enum_check(const int32_t* u, const int32_t* v, const int8_t* s, int64_t m, int64_t n_u, int64_t n_v,
                             unsigned long long* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long code = ~0ull;
    if (u[i] < 0 || u[i] >= n_u)
      code = (unsigned long long)i * 4ull;
    else if (v[i] < 0 || v[i] >= n_v)
      code = (unsigned long long)i * 4ull + 1ull;
    else if (s[i] != 1 && s[i] != -1)
      code = (unsigned long long)i * 4ull + 2ull;
    if (code != ~0ull) atomicMin(err, code);
  }
}

// key = centre << 32 | pivot, payload = edge index; degree of each centre
__global__ void k_enum_keys(const int32_t* u, const int32_t* v, int64_t m, int pivot_v, unsigned long long* key,
                            uint32_t* idx, unsigned int* deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = (uint32_t)(pivot_v ? v[i] : u[i]), c = (uint32_t)(pivot_v ? u[i] : v[i]);
    key[i] = (unsigned long long)c << 32 | p;
    idx[i] = (uint32_t)i;
    atomicAdd(&deg[c], 1u);
  }
}

__global__ void k_enum_wcount(const unsigned int* deg, int64_t nc, unsigned long long* wc) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long d = deg[c];
    wc[c] = d * (d - (d > 0)) / 2;
  }
}

// one thread per sorted list entry (position i in centre c's list): wedges (entry i, entry j > i)
// at woff[c] + (pairs before i) + (j - i - 1)
__global__ void k_enum_wedges(const unsigned long long* skey, const uint32_t* sidx, const unsigned long long* coff,
                              const unsigned long long* woff, const unsigned int* deg, const uint32_t* ecent, int64_t m,
                              unsigned long long* wkey, uint32_t* wa, uint32_t* wb) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = ecent[e];
    const unsigned long long d = deg[c], i = (unsigned long long)e - coff[c];
    unsigned long long o = woff[c] + i * (d - 1) - i * (i - (i > 0)) / 2;
    // pairs before i: sum_{i' < i} (d - 1 - i') = i (d - 1) - i (i - 1) / 2
    const uint32_t a = (uint32_t)(skey[e] & 0xffffffffu);
    for (unsigned long long j = i + 1; j < d; ++j, ++o) {
      const int64_t f = (int64_t)(coff[c] + j);
      wkey[o] = (unsigned long long)a << 32 | (skey[f] & 0xffffffffu);
      wa[o] = sidx[e];  // edge (a, c)
      wb[o] = sidx[f];  // edge (b, c)
    }
  }
}

__global__ void k_enum_centres(const unsigned long long* skey, int64_t m, uint32_t* ecent) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
    ecent[e] = (uint32_t)(skey[e] >> 32);
}

// per sorted wedge: 1 at the head of its (a, b) run
__global__ void k_enum_heads(const unsigned long long* k, int64_t w, uint32_t* head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < w; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || k[i] != k[i - 1]) ? 1u : 0u;
}

__global__ void k_enum_runid(const uint32_t* incl, int64_t w, uint32_t* rid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < w; i += (int64_t)gridDim.x * blockDim.x)
    rid[i] = incl[i] - 1u;
}

__global__ void k_enum_runstart(const uint32_t* head, const uint32_t* rid, int64_t w, uint32_t* rstart, uint32_t nruns) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < w; i += (int64_t)gridDim.x * blockDim.x)
    if (head[i]) rstart[rid[i]] = (uint32_t)i;
  if (blockIdx.x == 0 && threadIdx.x == 0) rstart[nruns] = (uint32_t)w;
}

__global__ void k_enum_runpairs(const uint32_t* rstart, uint32_t nruns, unsigned long long* rp) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nruns; r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long c = rstart[r + 1] - rstart[r];
    rp[r] = c * (c - (c > 0)) / 2;
  }
}

// one thread per sorted wedge (position i in its run of c): butterflies (i, j > i)
__global__ void k_enum_emit(const unsigned long long* wkey, const uint32_t* wa, const uint32_t* wb,
                            const uint32_t* rid, const uint32_t* rstart, const unsigned long long* roff,
                            const int32_t* u, const int32_t* v, const int8_t* s, int64_t w, int pivot_v,
                            int32_t* ids, uint8_t* sg, unsigned long long* okey) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < w; x += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = rid[x];
    const unsigned long long c = rstart[r + 1] - rstart[r], i = (unsigned long long)x - rstart[r];
    unsigned long long o = roff[r] + i * (c - 1) - i * (i - (i > 0)) / 2;
    const uint32_t a = (uint32_t)(wkey[x] >> 32), b = (uint32_t)(wkey[x] & 0xffffffffu);
    const uint32_t ea_i = wa[x], eb_i = wb[x];
    const uint32_t ci = (uint32_t)(pivot_v ? u[ea_i] : v[ea_i]);
    for (unsigned long long j = i + 1; j < c; ++j, ++o) {
      const int64_t y = (int64_t)rstart[r] + (int64_t)j;
      const uint32_t ea_j = wa[y], eb_j = wb[y];
      const uint32_t cj = (uint32_t)(pivot_v ? u[ea_j] : v[ea_j]);
      uint32_t q[4], e4[4];
      if (!pivot_v) {  // (u1, u2, v1, v2) = (a, b, c_i, c_j); edges a-ci, a-cj, b-ci, b-cj
        q[0] = a; q[1] = b; q[2] = ci; q[3] = cj;
        e4[0] = ea_i; e4[1] = ea_j; e4[2] = eb_i; e4[3] = eb_j;
      } else {  // (u1, u2, v1, v2) = (c_i, c_j, a, b); edges ci-a, ci-b, cj-a, cj-b
        q[0] = ci; q[1] = cj; q[2] = a; q[3] = b;
        e4[0] = ea_i; e4[1] = eb_i; e4[2] = ea_j; e4[3] = eb_j;
      }
      uint8_t bits = 0;
      for (int t = 0; t < 4; ++t) {
        ids[4 * o + t] = (int32_t)q[t];
        bits |= (uint8_t)((s[e4[t]] < 0 ? 1u : 0u) << t);
      }
      sg[o] = bits;
      if (okey) okey[o] = (unsigned long long)q[0] << 32 | q[1];
    }
  }
}

__global__ void k_enum_permute(const uint32_t* perm, const int32_t* ids, const uint8_t* sg, int64_t n, int32_t* ids2,
                               uint8_t* sg2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[i];
    for (int t = 0; t < 4; ++t) ids2[4 * i + t] = ids[4 * (int64_t)p + t];
    sg2[i] = sg[p];
  }
}

__global__ void k_widen(const unsigned int* x, int64_t n, unsigned long long* y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i];
}

__global__ void k_gather2(const uint32_t* perm, const uint32_t* a, const uint32_t* b, int64_t n, uint32_t* a2,
                          uint32_t* b2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    a2[i] = a[perm[i]];
    b2[i] = b[perm[i]];
  }
}

__global__ void k_iota(uint32_t* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (uint32_t)i;
}

// scoped device allocations (stream-ordered frees)
struct Pool {
  cudaStream_t st;
  std::vector<void*> ptrs;
  ~Pool() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
  }
  template <class T>
  int get(T** p, size_t n) {
    void* q = nullptr;
    if (cudaMallocAsync(&q, std::max<size_t>(n * sizeof(T), 16), st) != cudaSuccess) {
      cudaGetLastError();
      set_error("device allocation of " + std::to_string(n * sizeof(T)) + " bytes failed (butterfly enumeration)");
      return BBC_ERR_NOMEM;
    }
    ptrs.push_back(q);
    *p = static_cast<T*>(q);
    return BBC_OK;
  }
};

#define BBC_GET(pool, ptr, n)          \
  do {                                 \
    int _r = (pool).get(&(ptr), (n));  \
    if (_r) return _r;                 \
  } while (0)

template <class F>
int cub_call(Pool& pool, F f) {
  size_t bytes = 0;
  BBC_CK(f(nullptr, bytes));
  void* tmp = nullptr;
  BBC_GET(pool, *(char**)&tmp, bytes);
  BBC_CK(f(tmp, bytes));
  return BBC_OK;
}

int enumerate(int device, int64_t n_u, int64_t n_v, int64_t m, const int32_t* hu, const int32_t* hv, const int8_t* hs,
              uint64_t* count, int32_t* out_ids, uint8_t* out_signs, uint64_t max_out) {
  if (!count || n_u < 0 || n_v < 0 || m < 0 || (m > 0 && (!hu || !hv || !hs))) {
    set_error("bbc_enumerate_butterflies: bad arguments");
    return BBC_ERR_ARG;
  }
  if (n_u >= (1ll << 31) || n_v >= (1ll << 31) || m >= (1ll << 31)) {
    set_error("bbc_enumerate_butterflies: graph too large");
    return BBC_ERR_ARG;
  }
  *count = 0;
  if (m == 0) return BBC_OK;
  BBC_CK(cudaSetDevice(device));
  cudaStream_t st;
  BBC_CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg_{st};
  Pool pool{st, {}};
  const int pivot_v = n_u <= n_v ? 0 : 1;  // reference min_side (oracle.py:106)
  const int64_t nc = pivot_v ? n_u : n_v;
  int32_t *u, *v;
  int8_t* s;
  unsigned long long* err;
  BBC_GET(pool, u, m);
  BBC_GET(pool, v, m);
  BBC_GET(pool, s, m);
  BBC_GET(pool, err, 1);
  BBC_CK(cudaMemcpyAsync(u, hu, m * 4, cudaMemcpyHostToDevice, st));
  BBC_CK(cudaMemcpyAsync(v, hv, m * 4, cudaMemcpyHostToDevice, st));
  BBC_CK(cudaMemcpyAsync(s, hs, m, cudaMemcpyHostToDevice, st));
  BBC_CK(cudaMemsetAsync(err, 0xff, 8, st));
  k_enum_check<<<grid(m), kT, 0, st>>>(u, v, s, m, n_u, n_v, err);
  unsigned long long herr;
  BBC_CK(cudaMemcpyAsync(&herr, err, 8, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  if (herr != ~0ull) {
    set_error("bbc_enumerate_butterflies: edge out of range or bad sign", (int64_t)(herr >> 2));
    return (herr & 3) == 2 ? BBC_ERR_ARG : BBC_ERR_RANGE;
  }
  // 1. centre lists
  unsigned long long *key, *skey, *coff, *wc, *woff;
  uint32_t *idx, *sidx, *ecent;
  unsigned int* deg;
  BBC_GET(pool, key, m);
  BBC_GET(pool, skey, m);
  BBC_GET(pool, idx, m);
  BBC_GET(pool, sidx, m);
  BBC_GET(pool, ecent, m);
  BBC_GET(pool, deg, nc + 1);
  BBC_GET(pool, coff, nc + 1);
  BBC_GET(pool, wc, nc + 1);
  BBC_GET(pool, woff, nc + 1);
  BBC_CK(cudaMemsetAsync(deg, 0, (nc + 1) * 4, st));
  k_enum_keys<<<grid(m), kT, 0, st>>>(u, v, m, pivot_v, key, idx, deg);
  if (int r = cub_call(pool, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, key, skey, idx, sidx, (int)m, 0, 64, st);
      }))
    return r;
  k_enum_centres<<<grid(m), kT, 0, st>>>(skey, m, ecent);
  k_enum_wcount<<<grid(nc + 1), kT, 0, st>>>(deg, nc + 1, wc);  // deg[nc] = 0
  // coff = exclusive scan of degrees (as u64), woff = exclusive scan of C(deg, 2)
  {
    unsigned long long* deg64;
    BBC_GET(pool, deg64, nc + 1);
    k_widen<<<grid(nc + 1), kT, 0, st>>>(deg, nc + 1, deg64);
    if (int r = cub_call(pool, [&](void* t, size_t& b) {
          return cub::DeviceScan::ExclusiveSum(t, b, deg64, coff, (int)(nc + 1), st);
        }))
      return r;
  }
  if (int r = cub_call(pool, [&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, wc, woff, (int)(nc + 1), st);
      }))
    return r;
  unsigned long long W = 0;
  BBC_CK(cudaMemcpyAsync(&W, woff + nc, 8, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  if (W >= (1ull << 31)) {
    set_error("bbc_enumerate_butterflies: too many wedges for enumeration (" + std::to_string(W) + ")");
    return BBC_ERR_ARG;
  }
  if (W == 0) return BBC_OK;
  const int64_t w = (int64_t)W;
  // 2-3. wedges in ascending centre order, stable-sorted by (a, b)
  unsigned long long *wkey, *wkey2;
  uint32_t *wa, *wb, *wid, *wid2, *swa, *swb;
  BBC_GET(pool, wkey, w);
  BBC_GET(pool, wkey2, w);
  BBC_GET(pool, wa, w);
  BBC_GET(pool, wb, w);
  BBC_GET(pool, wid, w);
  BBC_GET(pool, wid2, w);
  BBC_GET(pool, swa, w);
  BBC_GET(pool, swb, w);
  k_enum_wedges<<<grid(m), kT, 0, st>>>(skey, sidx, coff, woff, deg, ecent, m, wkey, wa, wb);
  k_iota<<<grid(w), kT, 0, st>>>(wid, w);
  if (int r = cub_call(pool, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, wkey, wkey2, wid, wid2, (int)w, 0, 64, st);
      }))
    return r;
  k_gather2<<<grid(w), kT, 0, st>>>(wid2, wa, wb, w, swa, swb);
  // 4. runs of equal (a, b) and their butterfly offsets
  uint32_t *head, *rid, *rstart;
  BBC_GET(pool, head, w);
  BBC_GET(pool, rid, w);
  k_enum_heads<<<grid(w), kT, 0, st>>>(wkey2, w, head);
  if (int r = cub_call(pool, [&](void* t, size_t& b) {
        return cub::DeviceScan::InclusiveSum(t, b, head, rid, (int)w, st);
      }))
    return r;
  uint32_t nruns = 0;
  BBC_CK(cudaMemcpyAsync(&nruns, rid + (w - 1), 4, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  // run ids from the inclusive scan are 1-based: shift
  uint32_t* rid0;
  BBC_GET(pool, rid0, w);
  k_enum_runid<<<grid(w), kT, 0, st>>>(rid, w, rid0);
  BBC_GET(pool, rstart, (size_t)nruns + 1);
  k_enum_runstart<<<grid(w), kT, 0, st>>>(head, rid0, w, rstart, nruns);
  unsigned long long *rp, *roff;
  BBC_GET(pool, rp, (size_t)nruns + 1);
  BBC_GET(pool, roff, (size_t)nruns + 1);
  BBC_CK(cudaMemsetAsync(rp + nruns, 0, 8, st));
  k_enum_runpairs<<<grid(nruns), kT, 0, st>>>(rstart, nruns, rp);
  if (int r = cub_call(pool, [&](void* t, size_t& b) {
        return cub::DeviceScan::ExclusiveSum(t, b, rp, roff, (int)(nruns + 1), st);
      }))
    return r;
  unsigned long long B = 0;
  BBC_CK(cudaMemcpyAsync(&B, roff + nruns, 8, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  *count = B;
  if (!out_ids || B == 0) return BBC_OK;
  if (B > max_out || !out_signs) {
    set_error("bbc_enumerate_butterflies: output buffer holds " + std::to_string(max_out) + " of " +
              std::to_string(B) + " butterflies");
    return BBC_ERR_ARG;
  }
  if (B >= (1ull << 31)) {
    set_error("bbc_enumerate_butterflies: too many butterflies to materialise");
    return BBC_ERR_ARG;
  }
  const int64_t nb = (int64_t)B;
  // 5. emit (and, pivoting on V, restore the (u1, u2, v1, v2) order)
  int32_t* ids;
  uint8_t* sg;
  unsigned long long* okey = nullptr;
  BBC_GET(pool, ids, 4 * nb);
  BBC_GET(pool, sg, nb);
  if (pivot_v) BBC_GET(pool, okey, nb);
  k_enum_emit<<<grid(w), kT, 0, st>>>(wkey2, swa, swb, rid0, rstart, roff, u, v, s, w, pivot_v, ids, sg, okey);
  if (pivot_v) {
    unsigned long long* okey2;
    uint32_t *perm, *perm2;
    int32_t* ids2;
    uint8_t* sg2;
    BBC_GET(pool, okey2, nb);
    BBC_GET(pool, perm, nb);
    BBC_GET(pool, perm2, nb);
    BBC_GET(pool, ids2, 4 * nb);
    BBC_GET(pool, sg2, nb);
    k_iota<<<grid(nb), kT, 0, st>>>(perm, nb);
    if (int r = cub_call(pool, [&](void* t, size_t& b) {
          return cub::DeviceRadixSort::SortPairs(t, b, okey, okey2, perm, perm2, (int)nb, 0, 64, st);
        }))
      return r;
    k_enum_permute<<<grid(nb), kT, 0, st>>>(perm2, ids, sg, nb, ids2, sg2);
    ids = ids2;
    sg = sg2;
  }
  BBC_CK(cudaMemcpyAsync(out_ids, ids, (size_t)nb * 16, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaMemcpyAsync(out_signs, sg, (size_t)nb, cudaMemcpyDeviceToHost, st));
  BBC_CK(cudaStreamSynchronize(st));
  return BBC_OK;
}

}  // namespace
}  // namespace bbc

extern "C" int bbc_enumerate_butterflies(int32_t device, int64_t n_u, int64_t n_v, int64_t m, const int32_t* u,
                                         const int32_t* v, const int8_t* sign, uint64_t* count, int32_t* ids,
                                         uint8_t* signs, uint64_t max_out) {
  return bbc::enumerate(device, n_u, n_v, m, u, v, sign, count, ids, signs, max_out);
}
