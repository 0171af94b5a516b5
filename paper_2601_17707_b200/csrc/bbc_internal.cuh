// Internal definitions shared by the preprocessing and counting translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/bbc.h"

namespace bbc {

// Device-resident signed CSR for one anchor side.
//
//  adj   u32[m + 4]  centre-side lists, each sorted by ascending anchor rank;
//                    word = rank(w) | neg(c, w) << 31  (sign packed in bit 31)
//  coff  u32[nc + 1] centre offsets into adj
//  rec   uint2[m]    one record per anchor-side edge (a, c), grouped by rank(a):
//                    x = begin | neg(a, c) << 31, y = c; [begin, coff[c+1]) is the
//                    admitted suffix of c's list (ranks > rank(a))
//  bnd   u32[nc * nbands] (optional) band table: bnd[c * nbands + j] = first position
//                    of c's list with rank >= n - j * t16 (j = 0: list end)
//  aoff  u32[n + 1]  anchor offsets into rec (by rank)
//  awork u64[n]      admitted wedges per anchor (= sum of end - begin)
//  order u32[n]      anchor ranks by descending awork (G-BBC++ dispatch order)
//  rank_to_id u32[n] anchor-side vertex id of each rank
struct Graph {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t n_u = 0, n_v = 0, m = 0;
  int side = 0;       // anchor side: 0 = U, 1 = V
  int64_t n = 0;      // anchors
  int64_t nc = 0;     // centres
  uint64_t w_u = 0, w_v = 0, w_s = 0;
  uint32_t max_anchor_deg = 0;
  uint32_t* adj = nullptr;
  uint32_t* coff = nullptr;
  uint2* rec = nullptr;
  uint32_t* aoff = nullptr;
  unsigned long long* awork = nullptr;
  uint32_t* order = nullptr;
  uint32_t* rank_to_id = nullptr;
  uint32_t* bnd = nullptr;   // band-table rows (long centre lists only)
  uint32_t* brow = nullptr;  // brow[c]: row of centre c in bnd, or ~0 (binary search)
  uint32_t nbands = 0;
  uint32_t t16 = 0;
  // count scratch
  unsigned long long* acc = nullptr;        // [4]: bal lo, bal hi, unb lo, unb hi
  unsigned int* queue = nullptr;            // [1]
  unsigned long long* block_work = nullptr; // [2 * block_work_cap]: per-CTA admitted wedges,
                                            // then per-CTA busy ns (globaltimer)
  int block_work_cap = 0;
  int last_blocks = 0;
  uint64_t rounds[8] = {};  // last count with flags bit 12: bitmap, overflowed, tile, hash rounds;
                           // walked groups, walked wedges, round setups
  int num_sms = 0;
  int max_smem = 0;
  float preprocess_ms = 0.f;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

void set_error(const std::string& msg, int64_t info = 0);
int count_span16(Graph& g);  // endpoint span of a packed u16x2 tile on g.device
int cuda_fail(cudaError_t e, const char* where);

#define BBC_CK(call)                                              \
  do {                                                            \
    cudaError_t _e = (call);                                      \
    if (_e != cudaSuccess) return ::bbc::cuda_fail(_e, #call);    \
  } while (0)

}  // namespace bbc

struct bbc_graph {
  bbc::Graph g;
};
