// Multi-GPU counting in one process (SURVEY.md 8(b) bbc_count_multi, 8(e)).
//
// Reference analogue: count_balanced_parallel (pkg/src/bbcount/buckets.py:213-246) --
// a pool of workers, each counting a range of anchors over the same read-only graph,
// and an exact integer sum of the subtotals (:236-243).  Here the workers are GPUs:
//
//   1. sharded upload: device d copies edge slice d (ceil(m / N) edges) of the host
//      arrays into its own buffers -- N PCIe links in parallel instead of N full copies;
//   2. one grouped ncclAllGather per array over NVLink / NVSwitch gives every device the
//      whole edge list (9 B per edge);
//   3. every device builds the replicated CSR from its device arrays (the same kernels as
//      bbc_graph_create_device, all devices concurrently);
//   4. device d counts the dispatch-order tasks d, d + N, ... (bbc_opts.part_index /
//      part_count; the descending-work order interleaves the heavy anchors);
//   5. one grouped ncclAllReduce (sum) of the 128-bit (balanced, unbalanced) pairs as
//      32-bit limbs in u64 lanes -- exact for any N -- read back from the first device.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": in-process it resolves to the copy
// torch already loaded, if any), so libbbc.so itself has no link-time NCCL dependency.
// Each device is driven by its own host thread for steps 1, 3 and 4.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "bbc_internal.cuh"

namespace bbc {

int count_graph(Graph& g, const bbc_opts* o, uint64_t out[2], bbc_stats* st, int32_t k);
int create_graph(int device, int64_t n_u, int64_t n_v, int64_t m, const int32_t* u, const int32_t* v,
                 const int8_t* s, int32_t side_rule, bool host, bbc_graph** out);

namespace {

struct Nccl {
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.init_all = (decltype(n.init_all))dlsym(h, "ncclCommInitAll");
    n.destroy = (decltype(n.destroy))dlsym(h, "ncclCommDestroy");
    n.all_gather = (decltype(n.all_gather))dlsym(h, "ncclAllGather");
    n.all_reduce = (decltype(n.all_reduce))dlsym(h, "ncclAllReduce");
    n.group_start = (decltype(n.group_start))dlsym(h, "ncclGroupStart");
    n.group_end = (decltype(n.group_end))dlsym(h, "ncclGroupEnd");
    n.error_string = (decltype(n.error_string))dlsym(h, "ncclGetErrorString");
    n.ok = n.init_all && n.destroy && n.all_gather && n.all_reduce && n.group_start && n.group_end &&
           n.error_string;
  });
  return n;
}

int nccl_fail(ncclResult_t r, const char* where) {
  set_error(std::string("NCCL error in ") + where + ": " + nccl().error_string(r));
  return BBC_ERR_NCCL;
}

#define BBC_NCCL(call)                                          \
  do {                                                          \
    ncclResult_t _r = (call);                                   \
    if (_r != ncclSuccess) return nccl_fail(_r, #call);         \
  } while (0)

// run fn(i) for every device on its own host thread; the first failure's code and message
// (set_error is thread-local) are re-raised on the caller's thread
template <class Fn>
int per_device(int ndev, Fn fn) {
  std::vector<int> rc(ndev, BBC_OK);
  std::vector<std::string> msg(ndev);
  std::vector<int64_t> info(ndev, 0);
  std::vector<std::thread> th;
  for (int i = 0; i < ndev; ++i)
    th.emplace_back([&, i] {
      rc[i] = fn(i);
      if (rc[i]) {
        msg[i] = bbc_last_error();
        info[i] = bbc_last_error_info();
      }
    });
  for (auto& t : th) t.join();
  for (int i = 0; i < ndev; ++i)
    if (rc[i]) {
      set_error(msg[i], info[i]);
      return rc[i];
    }
  return BBC_OK;
}

}  // namespace
}  // namespace bbc

struct bbc_multi {
  int ndev = 0;
  std::vector<int> devices;
  std::vector<bbc_graph*> graphs;
  std::vector<ncclComm_t> comms;
  std::vector<cudaStream_t> streams;
  std::vector<unsigned long long*> limbs;  // 8 u64 lanes per device
  float build_ms = 0.f;
};

namespace bbc {
namespace {

void destroy_multi(bbc_multi* h) {
  if (!h) return;
  for (int i = 0; i < h->ndev; ++i) {
    cudaSetDevice(h->devices[i]);
    if (i < (int)h->graphs.size() && h->graphs[i]) bbc_graph_destroy(h->graphs[i]);
    if (i < (int)h->limbs.size() && h->limbs[i]) cudaFree(h->limbs[i]);
    if (i < (int)h->streams.size() && h->streams[i]) cudaStreamDestroy(h->streams[i]);
  }
  if (nccl().ok)
    for (ncclComm_t c : h->comms)
      if (c) nccl().destroy(c);
  delete h;
}

int multi_create(int ndev, const int* devices, int64_t n_u, int64_t n_v, int64_t m, const int32_t* u,
                 const int32_t* v, const int8_t* s, int32_t side_rule, bbc_multi** out) {
  if (!out || ndev < 1 || !devices) {
    set_error("bbc_multi_create: ndev >= 1, a device list and out are required");
    return BBC_ERR_ARG;
  }
  *out = nullptr;
  int visible = 0;
  BBC_CK(cudaGetDeviceCount(&visible));
  for (int i = 0; i < ndev; ++i) {
    if (devices[i] < 0 || devices[i] >= visible) {
      set_error("device " + std::to_string(devices[i]) + " not available (" + std::to_string(visible) + " visible)");
      return BBC_ERR_ARG;
    }
    for (int j = 0; j < i; ++j)
      if (devices[j] == devices[i]) {
        set_error("bbc_multi_create: devices must be distinct (one partition per GPU)");
        return BBC_ERR_ARG;
      }
  }
  if (m < 0 || (m > 0 && (!u || !v || !s))) {
    set_error("edge arrays must not be null");
    return BBC_ERR_ARG;
  }
  if (!nccl().ok) {
    set_error("libnccl.so.2 could not be loaded (needed for multi-GPU counting)");
    return BBC_ERR_NCCL;
  }
  bbc_multi* h = new bbc_multi();
  h->ndev = ndev;
  h->devices.assign(devices, devices + ndev);
  h->graphs.assign(ndev, nullptr);
  h->comms.assign(ndev, nullptr);
  h->streams.assign(ndev, nullptr);
  h->limbs.assign(ndev, nullptr);
  ncclResult_t nr = nccl().init_all(h->comms.data(), ndev, devices);
  if (nr != ncclSuccess) {
    h->comms.assign(ndev, nullptr);
    destroy_multi(h);
    return nccl_fail(nr, "ncclCommInitAll");
  }
  const int64_t chunk = (m + ndev - 1) / ndev;  // edges per shard (the last one may be short)
  const int64_t cap = chunk * ndev;
  std::vector<int32_t*> du(ndev, nullptr), dv(ndev, nullptr);
  std::vector<int8_t*> ds(ndev, nullptr);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // 1. sharded upload, one host thread per device
  int rc = per_device(ndev, [&](int i) -> int {
    BBC_CK(cudaSetDevice(devices[i]));
    BBC_CK(cudaStreamCreateWithFlags(&h->streams[i], cudaStreamNonBlocking));
    BBC_CK(cudaMalloc(&h->limbs[i], 64));
    if (i == 0) {
      BBC_CK(cudaEventCreate(&e0));
      BBC_CK(cudaEventCreate(&e1));
      BBC_CK(cudaEventRecord(e0, h->streams[0]));
    }
    if (cap == 0) return BBC_OK;
    BBC_CK(cudaMalloc(&du[i], (size_t)cap * 4 + 64));
    BBC_CK(cudaMalloc(&dv[i], (size_t)cap * 4 + 64));
    BBC_CK(cudaMalloc(&ds[i], (size_t)cap + 64));
    const int64_t lo = std::min(m, (int64_t)i * chunk), hi = std::min(m, lo + chunk);
    if (hi > lo) {
      BBC_CK(cudaMemcpyAsync(du[i] + lo, u + lo, (size_t)(hi - lo) * 4, cudaMemcpyHostToDevice, h->streams[i]));
      BBC_CK(cudaMemcpyAsync(dv[i] + lo, v + lo, (size_t)(hi - lo) * 4, cudaMemcpyHostToDevice, h->streams[i]));
      BBC_CK(cudaMemcpyAsync(ds[i] + lo, s + lo, (size_t)(hi - lo), cudaMemcpyHostToDevice, h->streams[i]));
    }
    return BBC_OK;
  });
  auto release = [&] {
    for (int i = 0; i < ndev; ++i) {
      cudaSetDevice(devices[i]);
      if (h->streams[i]) cudaStreamSynchronize(h->streams[i]);
      cudaFree(du[i]);
      cudaFree(dv[i]);
      cudaFree(ds[i]);
    }
  };
  // 2. every device receives the other shards over NVLink (in place: shard i sits at i * chunk)
  if (!rc && cap > 0 && ndev > 1) {
    nr = nccl().group_start();
    for (int i = 0; i < ndev && nr == ncclSuccess; ++i) {
      nr = nccl().all_gather(du[i] + i * chunk, du[i], (size_t)chunk, ncclInt32, h->comms[i], h->streams[i]);
      if (nr == ncclSuccess)
        nr = nccl().all_gather(dv[i] + i * chunk, dv[i], (size_t)chunk, ncclInt32, h->comms[i], h->streams[i]);
      if (nr == ncclSuccess)
        nr = nccl().all_gather(ds[i] + i * chunk, ds[i], (size_t)chunk, ncclInt8, h->comms[i], h->streams[i]);
    }
    ncclResult_t ne = nccl().group_end();
    if (nr == ncclSuccess) nr = ne;
    if (nr != ncclSuccess) rc = nccl_fail(nr, "ncclAllGather (edge shards)");
  }
  // 3. replicated CSR build on every device (its own stream inside the handle)
  if (!rc)
    rc = per_device(ndev, [&](int i) -> int {
      BBC_CK(cudaSetDevice(devices[i]));
      BBC_CK(cudaStreamSynchronize(h->streams[i]));
      return create_graph(devices[i], n_u, n_v, m, du[i], dv[i], ds[i], side_rule, false, &h->graphs[i]);
    });
  if (!rc) {
    cudaSetDevice(devices[0]);
    cudaEventRecord(e1, h->streams[0]);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    h->build_ms = ms;
  }
  release();
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (rc) {
    destroy_multi(h);
    return rc;
  }
  *out = h;
  return BBC_OK;
}

int multi_count(bbc_multi* h, const bbc_opts* o, uint64_t out[2], bbc_stats* st) {
  if (!h || !out) {
    set_error("multi handle and out must not be null");
    return BBC_ERR_ARG;
  }
  bbc_opts opts{};
  if (o) opts = *o;
  if (opts.part_count > 1) {
    set_error("bbc_multi_count partitions the anchors itself (part_count must be 0 or 1)");
    return BBC_ERR_ARG;
  }
  const int ndev = h->ndev;
  std::vector<bbc_stats> sts(ndev);
  std::vector<uint64_t> res(2 * ndev, 0);
  // 4. per-device partition counts, concurrently
  int rc = per_device(ndev, [&](int i) -> int {
    bbc_opts p = opts;
    p.part_index = i;
    p.part_count = ndev;
    std::memset(&sts[i], 0, sizeof(bbc_stats));
    int r = count_graph(h->graphs[i]->g, &p, &res[2 * i], &sts[i], 2);
    if (r && r != BBC_ERR_OVERFLOW) return r;
    // 128-bit (balanced, unbalanced) as eight 32-bit limbs in u64 lanes
    const uint64_t w[4] = {res[2 * i], sts[i].balanced_hi, res[2 * i + 1], sts[i].unbalanced_hi};
    unsigned long long lanes[8];
    for (int j = 0; j < 4; ++j) {
      lanes[2 * j] = w[j] & 0xffffffffull;
      lanes[2 * j + 1] = w[j] >> 32;
    }
    BBC_CK(cudaSetDevice(h->devices[i]));
    BBC_CK(cudaMemcpyAsync(h->limbs[i], lanes, 64, cudaMemcpyHostToDevice, h->streams[i]));
    BBC_CK(cudaStreamSynchronize(h->streams[i]));
    return BBC_OK;
  });
  if (rc) return rc;
  // 5. one all-reduce of the limbs
  BBC_NCCL(nccl().group_start());
  ncclResult_t nr = ncclSuccess;
  for (int i = 0; i < ndev && nr == ncclSuccess; ++i)
    nr = nccl().all_reduce(h->limbs[i], h->limbs[i], 8, ncclUint64, ncclSum, h->comms[i], h->streams[i]);
  ncclResult_t ne = nccl().group_end();
  if (nr == ncclSuccess) nr = ne;
  if (nr != ncclSuccess) return nccl_fail(nr, "ncclAllReduce (counts)");
  unsigned long long lanes[8];
  BBC_CK(cudaSetDevice(h->devices[0]));
  BBC_CK(cudaMemcpyAsync(lanes, h->limbs[0], 64, cudaMemcpyDeviceToHost, h->streams[0]));
  for (int i = 0; i < ndev; ++i) {
    BBC_CK(cudaSetDevice(h->devices[i]));
    BBC_CK(cudaStreamSynchronize(h->streams[i]));
  }
  // limbs back to 128-bit values (carries across lanes)
  unsigned __int128 v[2];
  for (int j = 0; j < 2; ++j) {
    unsigned __int128 x = 0;
    for (int l = 3; l >= 0; --l) x = (x << 32) + (unsigned __int128)lanes[4 * j + l];
    v[j] = x;
  }
  out[0] = (uint64_t)v[0];
  out[1] = (uint64_t)v[1];
  const uint64_t bhi = (uint64_t)(v[0] >> 64), uhi = (uint64_t)(v[1] >> 64);
  if (st) {
    std::memset(st, 0, sizeof(*st));
    *st = sts[0];
    st->wedges = 0;
    st->tasks = 0;
    st->count_ms = 0.f;
    st->preprocess_ms = h->build_ms;
    for (int i = 0; i < ndev; ++i) {
      st->wedges += sts[i].wedges;
      st->tasks += sts[i].tasks;
      st->count_ms = std::max(st->count_ms, sts[i].count_ms);  // the slowest device bounds the step
    }
    st->balanced_hi = bhi;
    st->unbalanced_hi = uhi;
    st->blocks = sts[0].blocks * ndev;
  }
  if (bhi || uhi) {
    set_error("balanced/unbalanced count exceeded 64-bit range");
    return BBC_ERR_OVERFLOW;
  }
  return BBC_OK;
}

}  // namespace
}  // namespace bbc

extern "C" {

int bbc_multi_create(int32_t ndev, const int32_t* devices, int64_t n_u, int64_t n_v, int64_t m, const int32_t* u,
                     const int32_t* v, const int8_t* sign, int32_t side_rule, bbc_multi** out) {
  return bbc::multi_create(ndev, devices, n_u, n_v, m, u, v, sign, side_rule, out);
}

int bbc_multi_count(bbc_multi* h, const bbc_opts* opts, uint64_t out[2], bbc_stats* stats) {
  return bbc::multi_count(h, opts, out, stats);
}

int bbc_multi_devices(bbc_multi* h, int32_t* devices, int32_t n) {
  if (!h) return 0;
  for (int i = 0; i < n && i < h->ndev; ++i) devices[i] = h->devices[i];
  return h->ndev;
}

bbc_graph* bbc_multi_graph(bbc_multi* h, int32_t i) {
  return (h && i >= 0 && i < h->ndev) ? h->graphs[i] : nullptr;
}

void bbc_multi_destroy(bbc_multi* h) { bbc::destroy_multi(h); }

int bbc_count_multi(int32_t ndev, const int32_t* devices, int64_t n_u, int64_t n_v, int64_t m, const int32_t* u,
                    const int32_t* v, const int8_t* sign, int32_t side_rule, const bbc_opts* opts, uint64_t out[2],
                    bbc_stats* stats) {
  bbc_multi* h = nullptr;
  int rc = bbc::multi_create(ndev, devices, n_u, n_v, m, u, v, sign, side_rule, &h);
  if (rc) return rc;
  rc = bbc::multi_count(h, opts, out, stats);
  bbc::destroy_multi(h);
  return rc;
}

}  // extern "C"
