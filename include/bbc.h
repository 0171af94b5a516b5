/*
 * bbc.h -- C ABI of the B200 balanced-butterfly counter (libbbc.so).
 *
 * The reference (/root/reference/pkg, pure Python) has no FFI: its engines are
 * Python functions `engine(g, ...) -> int | (int, ScheduleReport)` exported from
 * pkg/src/bbcount/__init__.py:10-63 and selected by name in the CLI
 * (pkg/src/bbcount/cli.py:34, 216-233).  These entry points are what a binding
 * of those engines binds (see INTEGRATION.md for the ctypes stub):
 *
 *   bbc_graph_create / bbc_graph_create_device
 *       replaces SignedBipartiteGraph.build (graph.py:99-129): range check
 *       (IndexOutOfRangeError, graph.py:109-114), duplicate rejection
 *       (DuplicateEdgeError(u, v), graph.py:116-121), degrees (graph.py:91-92),
 *       priority ranks (graph.py:93-97, 230-235), anchor-side choice
 *       (min_side graph.py:174-176 / cheaper side by admitted wedges), and the
 *       centre lists of _center_pairs (buckets.py:60-61), all on the device.
 *   bbc_count
 *       replaces the k = 2 hot kernel and its drivers:
 *       _pair_subtotal (buckets.py:166-197), count_balanced_parallel
 *       (buckets.py:213-246), count_balanced_tiled (tiled.py:107-168, algo
 *       BBC_ALGO_GBBC) and count_balanced_dynamic (tiled.py:182-292, algo
 *       BBC_ALGO_GBBCPP); also returns the unbalanced count the reference only
 *       has through count_balanced_bruteforce (oracle.py:116-124).
 *   bbc_block_work / bbc_task_order
 *       the device side of ScheduleReport.per_block_work / task_order
 *       (tiled.py:62-89).
 *
 * Conventions: plain pointers and sizes; host arrays are read during the call
 * only; the library owns all device memory inside a handle.  One handle per
 * device; a handle is not re-entrant.  Return codes map onto the reference's
 * exceptions (errors.py:4-55); the message is in bbc_last_error() and the
 * payload (edge index, duplicate pair) in bbc_last_error_info().
 */
#ifndef BBC_H
#define BBC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bbc_graph bbc_graph;

enum bbc_status {
  BBC_OK = 0,
  BBC_ERR_RANGE = 1,    /* IndexOutOfRangeError; info = edge*2 + (0: u, 1: v)   */
  BBC_ERR_DUP = 2,      /* DuplicateEdgeError;  info = (u << 32) | v            */
  BBC_ERR_OVERFLOW = 3, /* CountOverflowError (a total exceeds 2^64 - 1)        */
  BBC_ERR_ARG = 4,      /* ValueError (bad sizes, options, sign not +-1)        */
  BBC_ERR_CUDA = 5,     /* BBCountError                                         */
  BBC_ERR_NCCL = 6,     /* BBCountError (NCCL unavailable / collective failed)  */
  BBC_ERR_NOMEM = 7,    /* BBCountError (device allocation failed)              */
  BBC_ERR_PARSE = 8,    /* MalformedLineError; info = 1-based line               */
  BBC_ERR_MISSING = 9,  /* MissingValueError; info = 1-based line of the edge    */
  BBC_ERR_SIGNVAL = 10, /* InvalidSignValueError; info = 1-based line            */
  BBC_ERR_UNSUPPORTED = 11 /* input outside the device loader's exact fast paths:
                              use the host loader; info = 1-based line           */
};

enum bbc_algo {
  BBC_ALGO_GBBC = 0,   /* G-BBC: static round-robin CTAs over anchors in rank order */
  BBC_ALGO_GBBCPP = 1  /* G-BBC++: persistent CTAs, global atomic queue, descending work */
};

enum bbc_side_rule {
  BBC_SIDE_CHEAPER = -1, /* fewer admitted wedges W_S (north_star (1))          */
  BBC_SIDE_U = 0,
  BBC_SIDE_V = 1,
  BBC_SIDE_MIN = 2       /* reference min_side: smaller partition, ties to U    */
};

typedef struct {
  int32_t algo;         /* bbc_algo                                                 */
  int32_t tile_span;    /* endpoint-tile span (TileConfig.tile_size); 0 = max smem  */
  int32_t blocks;       /* CTAs; 0 = one persistent wave (SMs x occupancy)          */
  int32_t warp_max;     /* regime bands (tiled.py:171-179); 0 = defaults 32 / 512   */
  int32_t partial_max;
  int32_t part_index;   /* start-vertex partition [part_index of part_count]        */
  int32_t part_count;   /* 0 or 1 = whole graph                                     */
  int32_t flags;        /* 0 in production; testing / measurement switches:         */
                        /*  bit 0  general banded path only                           */
                        /*  bit 1  no cold key-hash rounds                            */
                        /*  bit 2  skip the hub band, bit 3 skip the cold range       */
                        /*         (timing only: the counts are then partial)         */
                        /*  bit 6  hub / cold range in two launches (experimental)    */
                        /*  bit 7  cold range in counter tiles only                   */
                        /*  bit 8  tiny repeat queue (exercises overflow + narrowing) */
                        /*  bit 9  force cold bitmap rounds                           */
                        /*  bit 10 band bounds by search (ignore the band table)      */
                        /*  bit 11 closing sweep for every tile round                 */
                        /*  bit 12 record round counters (bbc_round_counters; only in */
                        /*         a -DBBC_ROUND_STATS diagnostic build)              */
                        /*  bit 13 force cold key-hash rounds                         */
} bbc_opts;

typedef struct {
  uint64_t wedges;        /* admitted wedges processed by this call (partition)     */
  uint64_t wedges_total;  /* W_S of the processed side over the whole graph        */
  uint64_t w_u, w_v;      /* W if anchoring U / V                                   */
  uint64_t balanced_hi;   /* high 64 bits of the exact 128-bit totals               */
  uint64_t unbalanced_hi;
  int32_t anchor_side;    /* 0 = U, 1 = V                                           */
  int32_t blocks;
  int32_t threads;
  int32_t tile_span;
  int32_t tasks;          /* anchors dispatched by this call                        */
  int32_t reserved;
  float preprocess_ms;    /* device time of bbc_graph_create's device work          */
  float count_ms;         /* device time of the count kernels (incl. closing)       */
} bbc_stats;

/* Build from HOST arrays (u:int32[m], v:int32[m], sign:int8[m] in {+1,-1}). */
int bbc_graph_create(int device, int64_t n_u, int64_t n_v, int64_t m, const int32_t* u,
                     const int32_t* v, const int8_t* sign, int32_t side_rule, bbc_graph** out);

/* Same, from arrays already resident in device memory on `device` (not modified;
 * the caller keeps ownership and must have finished writing them). */
int bbc_graph_create_device(int device, int64_t n_u, int64_t n_v, int64_t m, const int32_t* d_u,
                            const int32_t* d_v, const int8_t* d_sign, int32_t side_rule,
                            bbc_graph** out);

/* Count balanced / unbalanced butterflies: out[0] = balanced, out[1] = unbalanced
 * (low 64 bits; BBC_ERR_OVERFLOW when either exceeds 2^64-1, high words in stats).
 * With part_count > 1 the result is this partition's share; partial results of all
 * partitions sum (mod 2^128) to the graph's counts. */
int bbc_count(bbc_graph* g, const bbc_opts* opts, uint64_t out[2], bbc_stats* stats);

/* six-way butterfly classification, replacing
 * oracle.classify_butterflies (pkg/src/bbcount/oracle.py:172-197).  Anchors U-pairs over
 * V-centres, so the graph must have been built with side_rule BBC_SIDE_U (else
 * BBC_ERR_ARG).  out[2i], out[2i+1] = low / high 64 bits of class i in
 * ButterflyClassCounts.as_dict() order (oracle.py:56-64): coherent_pp_pp, coherent_pp_mm,
 * coherent_mm_mm, incoherent_pm_pm, mixed_pp_pm, mixed_pm_mm.  opts: algo, blocks,
 * part_index / part_count as for bbc_count (partial results sum). */
int bbc_classify(bbc_graph* g, const bbc_opts* opts, uint64_t out[12], bbc_stats* stats);

/* balanced (2,k)-bicliques, k >= 2, replacing
 * count_balanced_2k_serial (pkg/src/bbcount/buckets.py:64-154): the size-2 side is the
 * graph's anchor side (build with BBC_SIDE_U / BBC_SIDE_V to choose it).
 * out[0], out[1] = low / high 64 bits; BBC_ERR_ARG for k < 2 (InvalidKError);
 * BBC_ERR_OVERFLOW above 2^64-1 (CountOverflowError). */
int bbc_count_2k(bbc_graph* g, int32_t k, const bbc_opts* opts, uint64_t out[2], bbc_stats* stats);

/* device-side ingestion, replacing load_graph =
 * parse_edge_list -> apply_sign_policy -> dedup_latest -> to_graph
 * (pkg/src/bbcount/ingest.py:80-191) for ASCII edge-list text ('\n' line ends; tokens
 * "u v [value] [timestamp]"; '%' / '#' comments).  Labels become dense ids per side in
 * first-occurrence order; the deduplicated edges keep the pairs' first-occurrence order. */
typedef struct {
  int32_t kind;         /* 0 ExplicitSign, 1 RatingThreshold, 2 RandomBernoulli        */
  int32_t at_or_above;  /* RatingThreshold.at_or_above_is_positive                    */
  double threshold;     /* RatingThreshold.threshold                                  */
  double p_positive;    /* RandomBernoulli.p_positive                                 */
  uint64_t seed;        /* RandomBernoulli.seed & (2^64 - 1)                          */
} bbc_sign_policy;

typedef struct bbc_ingest bbc_ingest;

/* counts = {n_u, n_v, m (deduplicated edges)}; errors BBC_ERR_PARSE / _MISSING /
 * _SIGNVAL (first offending line, as the reference raises them) or _UNSUPPORTED. */
int bbc_ingest_text(int device, const char* text, int64_t nbytes, const bbc_sign_policy* policy,
                    int64_t counts[3], bbc_ingest** out);
/* The m edges to host arrays (u:int32, v:int32, sign:int8 in {+1,-1}). */
int bbc_ingest_edges(bbc_ingest* h, int32_t* u, int32_t* v, int8_t* sign);
/* Build the counting graph straight from the ingested device arrays. */
int bbc_ingest_graph(bbc_ingest* h, int32_t side_rule, bbc_graph** out);
void bbc_ingest_destroy(bbc_ingest* h);

/* several GPUs of this process as the workers of
 * count_balanced_parallel (buckets.py:213-246: anchors split over workers, exact sum of
 * the subtotals at :236-243).  bbc_multi_create uploads edge shard i (ceil(m / ndev)
 * edges) to devices[i] only, all-gathers the shards over NVLink (ncclAllGather), and
 * builds the replicated CSR on every device; bbc_multi_count counts start-vertex
 * partition i on devices[i] concurrently and sums the 128-bit (balanced, unbalanced)
 * with one ncclAllReduce.  Same validation errors as bbc_graph_create; BBC_ERR_NCCL when
 * libnccl.so.2 is unavailable or a collective fails.  opts.part_count must be 0 / 1. */
typedef struct bbc_multi bbc_multi;
int bbc_multi_create(int32_t ndev, const int32_t* devices, int64_t n_u, int64_t n_v, int64_t m,
                     const int32_t* u, const int32_t* v, const int8_t* sign, int32_t side_rule,
                     bbc_multi** out);
int bbc_multi_count(bbc_multi* h, const bbc_opts* opts, uint64_t out[2], bbc_stats* stats);
/* the handle's devices (returns ndev) and the graph replica on devices[i] */
int bbc_multi_devices(bbc_multi* h, int32_t* devices, int32_t n);
bbc_graph* bbc_multi_graph(bbc_multi* h, int32_t i);
void bbc_multi_destroy(bbc_multi* h);
/* one-shot create + count + destroy (the SURVEY.md 8(b) proposal, plus side_rule) */
int bbc_count_multi(int32_t ndev, const int32_t* devices, int64_t n_u, int64_t n_v, int64_t m,
                    const int32_t* u, const int32_t* v, const int8_t* sign, int32_t side_rule,
                    const bbc_opts* opts, uint64_t out[2], bbc_stats* stats);

/* Every butterfly, replacing oracle.enumerate_butterflies (pkg/src/bbcount/oracle.py:73-107):
 * canonical (u1 < u2, v1 < v2) in (u1, u2, v1, v2) order, from HOST edge arrays, on
 * `device`.  *count receives the number of butterflies; with ids != NULL the first
 * call's output is written: ids[4i..4i+3] = u1, u2, v1, v2 and signs[i] bit j set when
 * sign j (order u1v1, u1v2, u2v1, u2v2) is negative.  BBC_ERR_ARG when max_out is too
 * small or the graph's wedges / butterflies exceed 2^31 (a test-scale API, as the
 * reference's). */
int bbc_enumerate_butterflies(int32_t device, int64_t n_u, int64_t n_v, int64_t m, const int32_t* u,
                              const int32_t* v, const int8_t* sign, uint64_t* count, int32_t* ids,
                              uint8_t* signs, uint64_t max_out);

/* Per-CTA admitted wedges of the last bbc_count (ScheduleReport.per_block_work). */
int bbc_block_work(bbc_graph* g, uint64_t* out, int32_t n);

/* Per-CTA busy time (ns, %globaltimer from the CTA's start to its exit) of the last
 * bbc_count: with persistent CTAs the spread of these is the schedule's real load
 * imbalance (a CTA that finishes early idles until the slowest one is done). */
int bbc_block_busy_ns(bbc_graph* g, uint64_t* out, int32_t n);

/* Diagnostics: rounds of the last bbc_count run with opts.flags bit 12 (BBC_FLAG_ROUNDS):
 * out[0] bitmap rounds, out[1] of them overflowed and redone, out[2] counter-tile rounds,
 * out[3] hash rounds (the per-anchor round kinds of DESIGN.md section 4), out[4] int4
 * groups walked, out[5] wedges walked, out[6] round set-ups (block scans), out[7] 0. */
int bbc_round_counters(bbc_graph* g, uint64_t out[8]);

/* Anchor dispatch order of `algo` as anchor-side vertex ids (ScheduleReport.task_order);
 * `work` (nullable) receives each task's admitted wedges in the same order. */
int bbc_task_order(bbc_graph* g, int32_t algo, int32_t* ids, uint64_t* work, int64_t n);

/* info[0..7] = n_u, n_v, m, anchor_side, n_anchors, W_S, W_U, W_V */
int bbc_graph_info(bbc_graph* g, int64_t* info, int32_t n);

/* Stream the handle launches on (cudaStream_t as void*), for external timing. */
void* bbc_graph_stream(bbc_graph* g);

void bbc_graph_destroy(bbc_graph* g);

/* Number of visible CUDA devices (0 when the driver reports none). */
int bbc_device_count(void);

const char* bbc_last_error(void);
int64_t bbc_last_error_info(void);

#ifdef __cplusplus
}
#endif

#endif /* BBC_H */
