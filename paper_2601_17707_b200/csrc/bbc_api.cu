// C-ABI glue: error state, counting entry point, schedule-report accessors.
#include <cstring>
#include <string>
#include <vector>

#include "bbc_internal.cuh"

namespace bbc {

int count_graph(Graph& g, const bbc_opts* o, uint64_t out[2], bbc_stats* st, int32_t k = 2);
int classify_graph(Graph& g, const bbc_opts* o, uint64_t out[12], bbc_stats* st);

namespace {
thread_local std::string t_err;
thread_local int64_t t_info = 0;
}  // namespace

void set_error(const std::string& msg, int64_t info) {
  t_err = msg;
  t_info = info;
}

int cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e));
  cudaGetLastError();
  return e == cudaErrorMemoryAllocation ? BBC_ERR_NOMEM : BBC_ERR_CUDA;
}

}  // namespace bbc

extern "C" {

int bbc_count(bbc_graph* h, const bbc_opts* opts, uint64_t out[2], bbc_stats* stats) {
  if (!h || !out) {
    bbc::set_error("graph handle and out must not be null");
    return BBC_ERR_ARG;
  }
  if (stats) std::memset(stats, 0, sizeof(*stats));
  return bbc::count_graph(h->g, opts, out, stats);
}

int bbc_classify(bbc_graph* h, const bbc_opts* opts, uint64_t out[12], bbc_stats* stats) {
  if (!h || !out) {
    bbc::set_error("graph handle and out must not be null");
    return BBC_ERR_ARG;
  }
  return bbc::classify_graph(h->g, opts, out, stats);
}

int bbc_count_2k(bbc_graph* h, int32_t k, const bbc_opts* opts, uint64_t out[2], bbc_stats* stats) {
  if (!h || !out) {
    bbc::set_error("graph handle and out must not be null");
    return BBC_ERR_ARG;
  }
  // the count kernel with C(., k) closings (hub tiles, cold bitmap / hash rounds)
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (k != 2) return bbc::count_graph(h->g, opts, out, stats, k);
  // k = 2: the balanced butterfly count (its high word in out[1])
  bbc_stats st{};
  uint64_t o2[2] = {0, 0};
  int rc = bbc::count_graph(h->g, opts, o2, &st, 2);
  if (stats) *stats = st;
  out[0] = o2[0];
  out[1] = st.balanced_hi;
  if (rc == BBC_ERR_OVERFLOW && st.balanced_hi == 0) rc = BBC_OK;  // only unbalanced overflowed
  return rc;
}

int bbc_block_work(bbc_graph* h, uint64_t* out, int32_t n) {
  if (!h || !out || n < 0) {
    bbc::set_error("bad arguments to bbc_block_work");
    return BBC_ERR_ARG;
  }
  bbc::Graph& g = h->g;
  int k = n < g.last_blocks ? n : g.last_blocks;
  if (k > 0) {
    BBC_CK(cudaSetDevice(g.device));
    BBC_CK(cudaMemcpy(out, g.block_work, (size_t)k * 8, cudaMemcpyDeviceToHost));
  }
  for (int i = k; i < n; ++i) out[i] = 0;
  return BBC_OK;
}

int bbc_block_busy_ns(bbc_graph* h, uint64_t* out, int32_t n) {
  if (!h || !out || n < 0) {
    bbc::set_error("bad arguments to bbc_block_busy_ns");
    return BBC_ERR_ARG;
  }
  bbc::Graph& g = h->g;
  int k = n < g.last_blocks ? n : g.last_blocks;
  if (k > 0) {
    BBC_CK(cudaSetDevice(g.device));
    BBC_CK(cudaMemcpy(out, g.block_work + g.block_work_cap, (size_t)k * 8, cudaMemcpyDeviceToHost));
  }
  for (int i = k; i < n; ++i) out[i] = 0;
  return BBC_OK;
}

int bbc_round_counters(bbc_graph* h, uint64_t out[8]) {
  if (!h || !out) {
    bbc::set_error("bad arguments to bbc_round_counters");
    return BBC_ERR_ARG;
  }
  for (int i = 0; i < 8; ++i) out[i] = h->g.rounds[i];
  return BBC_OK;
}

int bbc_task_order(bbc_graph* h, int32_t algo, int32_t* out, uint64_t* work, int64_t n) {
  if (!h || !out || n < 0) {
    bbc::set_error("bad arguments to bbc_task_order");
    return BBC_ERR_ARG;
  }
  bbc::Graph& g = h->g;
  int64_t k = n < g.n ? n : g.n;
  if (k <= 0) return BBC_OK;
  BBC_CK(cudaSetDevice(g.device));
  std::vector<uint32_t> ids((size_t)g.n), ord((size_t)g.n);
  std::vector<unsigned long long> aw((size_t)g.n);
  BBC_CK(cudaMemcpy(ids.data(), g.rank_to_id, (size_t)g.n * 4, cudaMemcpyDeviceToHost));
  BBC_CK(cudaMemcpy(aw.data(), g.awork, (size_t)g.n * 8, cudaMemcpyDeviceToHost));
  if (algo == BBC_ALGO_GBBCPP) {
    BBC_CK(cudaMemcpy(ord.data(), g.order, (size_t)g.n * 4, cudaMemcpyDeviceToHost));
  } else {
    for (int64_t i = 0; i < g.n; ++i) ord[i] = (uint32_t)i;
  }
  for (int64_t i = 0; i < k; ++i) {
    out[i] = (int32_t)ids[ord[i]];
    if (work) work[i] = aw[ord[i]];
  }
  return BBC_OK;
}

int bbc_graph_info(bbc_graph* h, int64_t* info, int32_t n) {
  if (!h || !info) {
    bbc::set_error("bad arguments to bbc_graph_info");
    return BBC_ERR_ARG;
  }
  const bbc::Graph& g = h->g;
  int64_t v[8] = {g.n_u, g.n_v, g.m, g.side, g.n, (int64_t)g.w_s, (int64_t)g.w_u, (int64_t)g.w_v};
  for (int i = 0; i < n && i < 8; ++i) info[i] = v[i];
  return BBC_OK;
}

int bbc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void* bbc_graph_stream(bbc_graph* h) { return h ? (void*)h->g.stream : nullptr; }

const char* bbc_last_error(void) { return bbc::t_err.c_str(); }

int64_t bbc_last_error_info(void) { return bbc::t_info; }

}  // extern "C"
