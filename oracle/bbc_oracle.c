/*
 * bbc_oracle.c -- CPU restatement of the reference bucket engine.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path and the CPU baseline timed by bench.py (`cpu_baseline`, kind "port",
 * and `--impl reference`).  Only tests/, __graft_entry__.smoke() and bench.py
 * may load it; the product package never links or calls it.
 *
 * What it restates (paths relative to /root/reference):
 *   - graph build / validation: pkg/src/bbcount/graph.py:99-129
 *       range check per edge in input order, u before v (:109-114); sort by
 *       (u, v) and reject the first duplicate pair in that order (:116-121);
 *       adjacency lists sorted by neighbour id (:122-128).
 *   - priority ranks: graph.py:230-235 (position in ascending (deg, id)).
 *   - anchor side: graph.py:174-176 (min_side, ties to U) unless forced.
 *   - the k = 2 hot kernel _pair_subtotal: pkg/src/bbcount/buckets.py:166-197
 *       filter prank[w] < prank[u] (:178), stamp-versioned reset (:179-183),
 *       symmetric/asymmetric buckets b1/b2 (:184-187), closing
 *       sum C(b1,2)+C(b2,2) over touched endpoints (:188-193).
 *   - unbalanced = sum b1*b2 over the same (u, w) pairs: equals
 *       total - balanced of count_balanced_bruteforce (oracle.py:116-124),
 *       pinned against the reference by tests/golden.
 *   - totals are exact 128-bit; > 2^64-1 is the reference's
 *       CountOverflowError (buckets.py:195-196).
 * Two SURVEY.md 8(f) extensions of the same wedge loop (mode argument):
 *   - balanced (2,k)-bicliques, k >= 2: closing sum C(b1,k) + C(b2,k) over the
 *       touched endpoints (buckets.py:64-154, math.comb at :146), anchor side fixed
 *       by the caller; a total > 2^64-1 is CountOverflowError.
 *   - six-way classification (oracle.py:172-197): U anchors, V centres; per (u, w)
 *       the wedge counts n_pp, n_mm, n_pm give C(pp,2), pp*mm, C(mm,2), C(pm,2),
 *       pp*pm, mm*pm (ButterflyClassCounts.as_dict order).
 * Multithreading mirrors count_balanced_parallel (buckets.py:205-246): anchor
 * ranges pulled dynamically by workers, exact integer sum.
 *
 * Parity pinned: the tests/golden JSON vectors were produced by the reference package
 * itself (tests/golden/make_golden.py) and tests/test_oracle_golden.py checks
 * this file against every vector.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

typedef struct {
  int64_t n_u, n_v, m;
  /* CSR both directions, lists sorted by neighbour id; sign +1/-1 */
  int64_t *off_u, *off_v;
  int32_t *adj_u, *adj_v;
  int8_t *sgn_u, *sgn_v;
  int64_t *deg_u, *deg_v;
  int64_t *prank_u, *prank_v;
} og_graph;

enum { OK = 0, E_RANGE = 1, E_DUP = 2, E_OVERFLOW = 3, E_ARG = 4, E_NOMEM = 7 };

/* LSD radix sort of (key, payload) pairs over the low `bits` bits; stable */
static void radix_sort_pairs(uint64_t* a, uint32_t* pa, uint64_t* tmp, uint32_t* ptmp, int64_t n, int bits) {
  static int64_t cnt[65536];
  for (int shift = 0; shift < bits; shift += 16) {
    memset(cnt, 0, sizeof(cnt));
    for (int64_t i = 0; i < n; ++i) cnt[(a[i] >> shift) & 0xFFFF]++;
    int64_t s = 0;
    for (int b = 0; b < 65536; ++b) { int64_t c = cnt[b]; cnt[b] = s; s += c; }
    for (int64_t i = 0; i < n; ++i) {
      int64_t d = cnt[(a[i] >> shift) & 0xFFFF]++;
      tmp[d] = a[i]; ptmp[d] = pa[i];
    }
    memcpy(a, tmp, (size_t)n * sizeof(uint64_t));
    memcpy(pa, ptmp, (size_t)n * sizeof(uint32_t));
  }
}

/* graph.py:230-235: rank = position in ascending (degree, index) order */
static int priority_ranks(const int64_t* deg, int64_t n, int64_t* rank) {
  int64_t maxd = 0;
  for (int64_t i = 0; i < n; ++i) if (deg[i] > maxd) maxd = deg[i];
  int64_t* cnt = (int64_t*)calloc((size_t)maxd + 2, sizeof(int64_t));
  if (!cnt) return E_NOMEM;
  for (int64_t i = 0; i < n; ++i) cnt[deg[i] + 1]++;
  for (int64_t d = 0; d <= maxd; ++d) cnt[d + 1] += cnt[d];
  for (int64_t i = 0; i < n; ++i) rank[i] = cnt[deg[i]]++; /* stable: ascending id within a degree */
  free(cnt);
  return OK;
}

void bbc_oracle_graph_free(og_graph* g) {
  if (!g) return;
  free(g->off_u); free(g->off_v); free(g->adj_u); free(g->adj_v); free(g->sgn_u); free(g->sgn_v);
  free(g->deg_u); free(g->deg_v); free(g->prank_u); free(g->prank_v);
  free(g);
}

static int bits_for(uint64_t x) { int b = 0; while (x) { ++b; x >>= 1; } return b; }

/*
 * Build + validate.  err_info receives: E_RANGE -> edge index * 2 + (0: u, 1: v);
 * E_DUP -> (u << 32) | v of the first duplicate in (u, v) order; E_ARG -> edge index.
 */
int bbc_oracle_graph_build(int64_t n_u, int64_t n_v, int64_t m, const int32_t* u, const int32_t* v,
                           const int8_t* s, og_graph** out, int64_t* err_info) {
  *out = NULL;
  if (n_u < 0 || n_v < 0 || m < 0 || n_u >= (1ll << 31) || n_v >= (1ll << 31) || m >= (1ll << 32)) return E_ARG;
  for (int64_t i = 0; i < m; ++i) {
    if (u[i] < 0 || u[i] >= n_u) { *err_info = i * 2; return E_RANGE; }
    if (v[i] < 0 || v[i] >= n_v) { *err_info = i * 2 + 1; return E_RANGE; }
    if (s[i] != 1 && s[i] != -1) { *err_info = i; return E_ARG; }
  }
  og_graph* g = (og_graph*)calloc(1, sizeof(og_graph));
  if (!g) return E_NOMEM;
  g->n_u = n_u; g->n_v = n_v; g->m = m;
  uint64_t* key = (uint64_t*)malloc((size_t)(m + 1) * 8);
  uint64_t* tmp = (uint64_t*)malloc((size_t)(m + 1) * 8);
  g->off_u = (int64_t*)calloc((size_t)n_u + 1, 8);
  g->off_v = (int64_t*)calloc((size_t)n_v + 1, 8);
  g->adj_u = (int32_t*)malloc((size_t)(m + 1) * 4);
  g->adj_v = (int32_t*)malloc((size_t)(m + 1) * 4);
  g->sgn_u = (int8_t*)malloc((size_t)m + 1);
  g->sgn_v = (int8_t*)malloc((size_t)m + 1);
  g->deg_u = (int64_t*)calloc((size_t)n_u + 1, 8);
  g->deg_v = (int64_t*)calloc((size_t)n_v + 1, 8);
  g->prank_u = (int64_t*)malloc(((size_t)n_u + 1) * 8);
  g->prank_v = (int64_t*)malloc(((size_t)n_v + 1) * 8);
  if (!key || !tmp || !g->off_u || !g->off_v || !g->adj_u || !g->adj_v || !g->sgn_u || !g->sgn_v ||
      !g->deg_u || !g->deg_v || !g->prank_u || !g->prank_v) {
    free(key); free(tmp); bbc_oracle_graph_free(g); return E_NOMEM;
  }
  /* sort edge indices by (u, v) (graph.py:116), then reject the first equal neighbour pair */
  uint32_t* idx = (uint32_t*)malloc((size_t)(m + 1) * 4);
  uint32_t* itmp = (uint32_t*)malloc((size_t)(m + 1) * 4);
  if (!idx || !itmp) { free(idx); free(itmp); free(key); free(tmp); bbc_oracle_graph_free(g); return E_NOMEM; }
  for (int64_t i = 0; i < m; ++i) { key[i] = ((uint64_t)u[i] << 32) | (uint64_t)v[i]; idx[i] = (uint32_t)i; }
  radix_sort_pairs(key, idx, tmp, itmp, m, 32 + bits_for((uint64_t)n_u));
  free(itmp);
  uint64_t prev = UINT64_MAX;
  for (int64_t i = 0; i < m; ++i) {
    uint64_t pair = key[i];
    if (pair == prev) {
      *err_info = (int64_t)pair;
      free(idx); free(key); free(tmp); bbc_oracle_graph_free(g); return E_DUP;
    }
    prev = pair;
    g->adj_u[i] = (int32_t)(pair & 0xFFFFFFFFull);
    g->sgn_u[i] = s[idx[i]];
    g->deg_u[pair >> 32]++;
  }
  free(idx);
  free(key); free(tmp);
  for (int64_t x = 0; x < n_u; ++x) g->off_u[x + 1] = g->off_u[x] + g->deg_u[x];
  /* V side: filled in ascending u order, so already sorted (graph.py:124-128) */
  for (int64_t i = 0; i < m; ++i) g->deg_v[g->adj_u[i]]++;
  for (int64_t y = 0; y < n_v; ++y) g->off_v[y + 1] = g->off_v[y] + g->deg_v[y];
  int64_t* cur = (int64_t*)malloc(((size_t)n_v + 1) * 8);
  memcpy(cur, g->off_v, ((size_t)n_v + 1) * 8);
  for (int64_t x = 0; x < n_u; ++x)
    for (int64_t i = g->off_u[x]; i < g->off_u[x + 1]; ++i) {
      int64_t p = cur[g->adj_u[i]]++;
      g->adj_v[p] = (int32_t)x;
      g->sgn_v[p] = g->sgn_u[i];
    }
  free(cur);
  if (priority_ranks(g->deg_u, n_u, g->prank_u) || priority_ranks(g->deg_v, n_v, g->prank_v)) {
    bbc_oracle_graph_free(g); return E_NOMEM;
  }
  *out = g;
  return OK;
}

typedef struct {
  const og_graph* g;
  int side;
  int64_t n;
  int64_t stride;
  int64_t next;         /* shared chunk cursor */
  pthread_mutex_t lock;
  int64_t chunk;
  int mode; /* 0: balanced / unbalanced, 1: (2,k), 2: classification */
  int k;
} job;

typedef struct { job* j; u128 bal, unb; u128 cls[6]; uint64_t admitted, scanned; int err, ovf; } worker_arg;

/* C(b, k) exactly; sets *ovf (and returns 2^64) once it exceeds 2^64 - 1 */
static u128 binom_sat(u128 b, int k, int* ovf) {
  if ((u128)k > b) return 0;
  u128 kk = (u128)k;
  if (kk > b - kk) kk = b - kk;
  u128 r = 1;
  const u128 lim = (u128)1 << 64;
  for (u128 i = 1; i <= kk; ++i) {
    r = r * (b - kk + i) / i;
    if (r >= lim) { *ovf = 1; return lim; }
  }
  return r;
}

/* buckets.py:166-197 (+ unbalanced = sum b1*b2) over anchors [lo, hi) step stride */
static void* worker(void* p) {
  worker_arg* wa = (worker_arg*)p;
  job* j = wa->j;
  const og_graph* g = j->g;
  const int64_t *off_s, *off_o, *prank;
  const int32_t *adj_s, *adj_o;
  const int8_t *sgn_s, *sgn_o;
  if (j->side == 0) { off_s = g->off_u; adj_s = g->adj_u; sgn_s = g->sgn_u; off_o = g->off_v; adj_o = g->adj_v; sgn_o = g->sgn_v; prank = g->prank_u; }
  else { off_s = g->off_v; adj_s = g->adj_v; sgn_s = g->sgn_v; off_o = g->off_u; adj_o = g->adj_u; sgn_o = g->sgn_u; prank = g->prank_v; }
  int64_t n = j->n;
  int64_t* b1 = (int64_t*)calloc((size_t)n + 1, 8);
  int64_t* b2 = (int64_t*)calloc((size_t)n + 1, 8);
  int64_t* b3 = j->mode == 2 ? (int64_t*)calloc((size_t)n + 1, 8) : NULL;
  int64_t* stamp = (int64_t*)malloc(((size_t)n + 1) * 8);
  int64_t* touched = (int64_t*)malloc(((size_t)n + 1) * 8);
  if (!b1 || !b2 || !stamp || !touched || (j->mode == 2 && !b3)) {
    wa->err = E_NOMEM; free(b1); free(b2); free(b3); free(stamp); free(touched); return NULL;
  }
  for (int64_t i = 0; i < n; ++i) stamp[i] = -1;
  u128 bal = 0, unb = 0, cls[6] = {0, 0, 0, 0, 0, 0};
  int ovf = 0;
  uint64_t admitted = 0, scanned = 0;
  for (;;) {
    pthread_mutex_lock(&j->lock);
    int64_t lo = j->next;
    j->next += j->chunk;
    pthread_mutex_unlock(&j->lock);
    if (lo >= n) break;
    int64_t hi = lo + j->chunk < n ? lo + j->chunk : n;
    for (int64_t a = lo; a < hi; ++a) {
      if (a % j->stride) continue;
      int64_t pu = prank[a], nt = 0;
      for (int64_t e = off_s[a]; e < off_s[a + 1]; ++e) {
        int32_t c = adj_s[e];
        int8_t suv = sgn_s[e];
        int64_t cb = off_o[c], ce = off_o[c + 1];
        scanned += (uint64_t)(ce - cb);
        for (int64_t f = cb; f < ce; ++f) {
          int32_t w = adj_o[f];
          if (prank[w] < pu) {
            ++admitted;
            if (stamp[w] != a) { stamp[w] = a; b1[w] = 0; b2[w] = 0; if (b3) b3[w] = 0; touched[nt++] = w; }
            if (j->mode == 2) {
              /* wedge through centre c: pp (both +), mm (both -), pm (signs differ) */
              if (sgn_o[f] != suv) b3[w]++; else if (suv > 0) b1[w]++; else b2[w]++;
            } else if (sgn_o[f] == suv) b1[w]++; else b2[w]++;
          }
        }
      }
      for (int64_t t = 0; t < nt; ++t) {
        u128 c1 = (u128)b1[touched[t]], c2 = (u128)b2[touched[t]];
        if (j->mode == 0) {
          bal += c1 * (c1 - (c1 > 0)) / 2 + c2 * (c2 - (c2 > 0)) / 2;
          unb += c1 * c2;
        } else if (j->mode == 1) {
          bal += binom_sat(c1, j->k, &ovf) + binom_sat(c2, j->k, &ovf);
          if (bal >= ((u128)1 << 64)) ovf = 1;
        } else {
          u128 c3 = (u128)b3[touched[t]];
          cls[0] += c1 * (c1 - (c1 > 0)) / 2;  /* coherent_pp_pp */
          cls[1] += c1 * c2;                   /* coherent_pp_mm */
          cls[2] += c2 * (c2 - (c2 > 0)) / 2;  /* coherent_mm_mm */
          cls[3] += c3 * (c3 - (c3 > 0)) / 2;  /* incoherent_pm_pm */
          cls[4] += c1 * c3;                   /* mixed_pp_pm */
          cls[5] += c2 * c3;                   /* mixed_pm_mm */
        }
      }
    }
  }
  free(b1); free(b2); free(b3); free(stamp); free(touched);
  wa->bal = bal; wa->unb = unb; wa->admitted = admitted; wa->scanned = scanned; wa->ovf = ovf;
  for (int i = 0; i < 6; ++i) wa->cls[i] = cls[i];
  return NULL;
}

/* the wedge loop over all anchors of `side` in the given mode (see the header) */
static int run(const og_graph* g, int side, int threads, int64_t stride, int mode, int k, uint64_t* out) {
  if (side < 0) side = g->n_u <= g->n_v ? 0 : 1;
  if (threads < 1 || stride < 1) return E_ARG;
  job j;
  memset(&j, 0, sizeof(j));
  j.g = g; j.side = side; j.n = side == 0 ? g->n_u : g->n_v; j.stride = stride; j.mode = mode; j.k = k;
  pthread_mutex_init(&j.lock, NULL);
  int64_t target = (int64_t)threads * 64;
  j.chunk = j.n / (target > 0 ? target : 1);
  if (j.chunk < 1) j.chunk = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  worker_arg* wa = (worker_arg*)calloc((size_t)threads, sizeof(worker_arg));
  for (int t = 0; t < threads; ++t) { wa[t].j = &j; }
  for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, worker, &wa[t]);
  worker(&wa[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  u128 bal = 0, unb = 0, cls[6] = {0, 0, 0, 0, 0, 0};
  uint64_t adm = 0, scn = 0;
  int err = OK, ovf = 0;
  for (int t = 0; t < threads; ++t) {
    bal += wa[t].bal; unb += wa[t].unb; adm += wa[t].admitted; scn += wa[t].scanned;
    for (int i = 0; i < 6; ++i) cls[i] += wa[t].cls[i];
    if (wa[t].err) err = wa[t].err;
    ovf |= wa[t].ovf;
  }
  free(th); free(wa);
  pthread_mutex_destroy(&j.lock);
  out[0] = (uint64_t)bal; out[1] = (uint64_t)(bal >> 64);
  out[2] = (uint64_t)unb; out[3] = (uint64_t)(unb >> 64);
  out[4] = adm; out[5] = scn; out[6] = (uint64_t)side;
  if (mode == 2)
    for (int i = 0; i < 6; ++i) { out[8 + 2 * i] = (uint64_t)cls[i]; out[9 + 2 * i] = (uint64_t)(cls[i] >> 64); }
  if (err) return err;
  if (mode == 1) return (ovf || out[1]) ? E_OVERFLOW : OK;
  return (out[1] || out[3]) ? E_OVERFLOW : OK;
}

/*
 * Count balanced / unbalanced butterflies.  side: 0 = U anchors, 1 = V,
 * -1 = reference min_side (graph.py:174-176).  stride > 1 processes the
 * deterministic anchor sample {a : a % stride == 0} (CPU-baseline sampling).
 * out: [bal_lo, bal_hi, unb_lo, unb_hi, admitted, scanned, side_used].
 */
int bbc_oracle_count(const og_graph* g, int side, int threads, int64_t stride, uint64_t* out) {
  return run(g, side, threads, stride, 0, 2, out);
}

/* Balanced (2,k)-bicliques with the size-2 side `side` (0 = U, 1 = V): out[0..1] = the
 * total (lo, hi); E_OVERFLOW once it exceeds 2^64 - 1 (out then saturated / partial). */
int bbc_oracle_count_2k(const og_graph* g, int side, int k, int threads, uint64_t* out) {
  if (k < 2 || side < 0 || side > 1) return E_ARG;
  return run(g, side, threads, 1, 1, k, out);
}

/* Six-way classification (U anchors): out[8 + 2i], out[9 + 2i] = lo, hi of class i in
 * ButterflyClassCounts.as_dict order; out must hold 20 words. */
int bbc_oracle_classify(const og_graph* g, int threads, uint64_t* out) {
  return run(g, 0, threads, 1, 2, 2, out);
}

/*
 * The reference's sort_neighbors traversal (count_balanced_2k_serial, buckets.py:87-111):
 * each centre's list is iterated in ascending priority rank and the scan stops at the
 * first rank >= prank[u] (:106-107), so scanned = admitted + one stop per record instead
 * of sum deg(c)^2.  Same b1/b2 buckets and closing as _pair_subtotal (buckets.py:166-197);
 * buckets are addressed by prank[w] instead of w (a bijection of the end vertices, so the
 * touched set and the sum over it are unchanged) which turns a scan of a sorted list into
 * ascending bucket addresses.  b1/b2 are u32 (they are bounded by deg u < 2^32).  Used
 * for the full-size BASELINE goldens (configs 3-5), where the scan-everything loop above
 * would take days on the build container.  out as bbc_oracle_count.
 */
typedef struct { uint32_t stamp, b1, b2, pad; } sbucket;

typedef struct {
  const og_graph* g;
  int side;
  int64_t n;
  const uint32_t* lst; /* per centre: prank << 1 | neg, ascending */
  int64_t next, chunk;
  pthread_mutex_t lock;
} sjob;

typedef struct { sjob* j; u128 bal, unb; uint64_t admitted, scanned; int err; } sworker_arg;

static void* sworker(void* p) {
  sworker_arg* wa = (sworker_arg*)p;
  sjob* j = wa->j;
  const og_graph* g = j->g;
  const int64_t *off_s = j->side ? g->off_v : g->off_u, *off_o = j->side ? g->off_u : g->off_v;
  const int32_t* adj_s = j->side ? g->adj_v : g->adj_u;
  const int8_t* sgn_s = j->side ? g->sgn_v : g->sgn_u;
  const int64_t* prank = j->side ? g->prank_v : g->prank_u;
  int64_t n = j->n;
  sbucket* b = (sbucket*)calloc((size_t)n + 1, sizeof(sbucket));
  uint32_t* touched = (uint32_t*)malloc(((size_t)n + 1) * 4);
  if (!b || !touched) { wa->err = E_NOMEM; free(b); free(touched); return NULL; }
  u128 bal = 0, unb = 0;
  uint64_t admitted = 0, scanned = 0;
  for (;;) {
    pthread_mutex_lock(&j->lock);
    int64_t lo = j->next;
    j->next += j->chunk;
    pthread_mutex_unlock(&j->lock);
    if (lo >= n) break;
    int64_t hi = lo + j->chunk < n ? lo + j->chunk : n;
    for (int64_t a = lo; a < hi; ++a) {
      uint32_t st = (uint32_t)a + 1, pu = (uint32_t)prank[a];
      int64_t nt = 0;
      for (int64_t e = off_s[a]; e < off_s[a + 1]; ++e) {
        const uint32_t* l = j->lst + off_o[adj_s[e]];
        uint32_t neg = sgn_s[e] < 0;
        int64_t f = 0;
        for (;; ++f) {
          uint32_t x = l[f], r = x >> 1;
          if (r >= pu) break; /* u itself is in the list: the scan always stops */
          sbucket* q = &b[r];
          if (q->stamp != st) { q->stamp = st; q->b1 = 0; q->b2 = 0; touched[nt++] = r; }
          if ((x & 1) == neg) q->b1++; else q->b2++;
        }
        admitted += (uint64_t)f;
        scanned += (uint64_t)f + 1;
      }
      uint64_t sb = 0, su = 0;
      for (int64_t t = 0; t < nt; ++t) {
        uint64_t c1 = b[touched[t]].b1, c2 = b[touched[t]].b2;
        sb += c1 * (c1 - (c1 > 0)) / 2 + c2 * (c2 - (c2 > 0)) / 2;
        su += c1 * c2;
      }
      bal += sb; unb += su; /* per anchor < 2^64: sum over w of deg(u)^2 */
    }
  }
  free(b); free(touched);
  wa->bal = bal; wa->unb = unb; wa->admitted = admitted; wa->scanned = scanned;
  return NULL;
}

int bbc_oracle_count_sorted(const og_graph* g, int side, int threads, uint64_t* out) {
  if (side < 0) side = g->n_u <= g->n_v ? 0 : 1;
  if (threads < 1 || side > 1) return E_ARG;
  int64_t n = side ? g->n_v : g->n_u, no = side ? g->n_u : g->n_v;
  const int64_t *off_s = side ? g->off_v : g->off_u, *off_o = side ? g->off_u : g->off_v;
  const int32_t* adj_s = side ? g->adj_v : g->adj_u;
  const int8_t* sgn_s = side ? g->sgn_v : g->sgn_u;
  const int64_t* prank = side ? g->prank_v : g->prank_u;
  /* centre lists in ascending anchor rank: append anchors in rank order */
  uint32_t* lst = (uint32_t*)malloc(((size_t)g->m + 1) * 4);
  int64_t* cur = (int64_t*)malloc(((size_t)no + 1) * 8);
  int64_t* inv = (int64_t*)malloc(((size_t)n + 1) * 8);
  if (!lst || !cur || !inv) { free(lst); free(cur); free(inv); return E_NOMEM; }
  memcpy(cur, off_o, ((size_t)no + 1) * 8);
  for (int64_t a = 0; a < n; ++a) inv[prank[a]] = a;
  for (int64_t r = 0; r < n; ++r) {
    int64_t a = inv[r];
    for (int64_t e = off_s[a]; e < off_s[a + 1]; ++e)
      lst[cur[adj_s[e]]++] = (uint32_t)r << 1 | (uint32_t)(sgn_s[e] < 0);
  }
  free(cur); free(inv);
  sjob j;
  memset(&j, 0, sizeof(j));
  j.g = g; j.side = side; j.n = n; j.lst = lst;
  pthread_mutex_init(&j.lock, NULL);
  j.chunk = n / ((int64_t)threads * 256);
  if (j.chunk < 1) j.chunk = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  sworker_arg* wa = (sworker_arg*)calloc((size_t)threads, sizeof(sworker_arg));
  for (int t = 0; t < threads; ++t) wa[t].j = &j;
  for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, sworker, &wa[t]);
  sworker(&wa[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  u128 bal = 0, unb = 0;
  uint64_t adm = 0, scn = 0;
  int err = OK;
  for (int t = 0; t < threads; ++t) {
    bal += wa[t].bal; unb += wa[t].unb; adm += wa[t].admitted; scn += wa[t].scanned;
    if (wa[t].err) err = wa[t].err;
  }
  free(th); free(wa); free(lst);
  pthread_mutex_destroy(&j.lock);
  out[0] = (uint64_t)bal; out[1] = (uint64_t)(bal >> 64);
  out[2] = (uint64_t)unb; out[3] = (uint64_t)(unb >> 64);
  out[4] = adm; out[5] = scn; out[6] = (uint64_t)side;
  if (err) return err;
  return (out[1] || out[3]) ? E_OVERFLOW : OK;
}

int64_t bbc_oracle_graph_info(const og_graph* g, int what) {
  switch (what) {
    case 0: return g->n_u;
    case 1: return g->n_v;
    case 2: return g->m;
    default: return -1;
  }
}

/* W_S = sum over the centre side of C(deg, 2): side 0 -> U anchors */
uint64_t bbc_oracle_admitted_total(const og_graph* g, int side) {
  const int64_t* d = side == 0 ? g->deg_v : g->deg_u;
  int64_t n = side == 0 ? g->n_v : g->n_u;
  uint64_t w = 0;
  for (int64_t i = 0; i < n; ++i) w += (uint64_t)(d[i] * (d[i] - 1) / 2);
  return w;
}
