/*
 * Deterministic synthetic signed bipartite graphs (BASELINE.json configs 1-5).
 *
 * Workload generator, not part of the counting path: it produces the host edge
 * arrays (u:int32, v:int32, sign:int8 = +1/-1) that both the CUDA path and the
 * CPU oracle consume, so every consumer sees identical, duplicate-free inputs
 * (SignedBipartiteGraph.build rejects duplicates, reference graph.py:117-121).
 *
 * Counter-based randomness: draw(seed, stream, i) = splitmix64 finaliser of
 * (base(seed, stream) + (i+1) * golden).  Candidate i of an ER graph is
 * (u, v) = (floor(r0 * n_u), floor(r1 * n_v)) with r = draw(seed, {0,1}, i);
 * a Chung-Lu candidate inverts the continuous power-law CDF with density
 * (x+1)^-beta, beta = 1/(gamma-1).  Candidates are deduplicated keeping the
 * first occurrence in candidate order; the first m survivors are the edges.
 * Edge j is negative iff draw(seed, 2, j) < p_neg * 2^64.
 * Planted hubs (config 3) append, for hub h on a side, partners drawn
 * uniformly from the other side (stream 3 + 2h / 4 + 2h), deduplicated the
 * same way, before the Chung-Lu tail fills the edge budget.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint64_t draw(uint64_t seed, uint32_t stream, uint64_t i) {
  uint64_t base = mix64(seed * 0x100ull + stream);
  return mix64(base + i * 0x9E3779B97F4A7C15ull);
}

static inline int64_t uniform_index(uint64_t r, int64_t n) {
  return (int64_t)(((unsigned __int128)r * (uint64_t)n) >> 64);
}

typedef struct {
  int64_t n;
  double beta; /* <= 0 -> uniform */
  double a;    /* (n+1)^(1-beta) - 1 */
  double inv;  /* 1/(1-beta) */
} sampler;

static void sampler_init(sampler* s, int64_t n, double gamma) {
  s->n = n;
  if (gamma <= 0.0) { s->beta = 0.0; return; }
  s->beta = 1.0 / (gamma - 1.0);
  double e = 1.0 - s->beta;
  s->a = pow((double)n + 1.0, e) - 1.0;
  s->inv = 1.0 / e;
}

static inline int64_t sample(const sampler* s, uint64_t r) {
  if (s->beta <= 0.0) return uniform_index(r, s->n);
  double x = (double)(r >> 11) * (1.0 / 9007199254740992.0);
  double y = pow(1.0 + x * s->a, s->inv) - 1.0;
  int64_t i = (int64_t)y;
  if (i < 0) i = 0;
  if (i >= s->n) i = s->n - 1;
  return i;
}

typedef struct {
  uint64_t* slots;
  uint64_t mask;
} hset;

static int hset_init(hset* h, int64_t m) {
  uint64_t cap = 1;
  while (cap < (uint64_t)m * 2 + 16) cap <<= 1;
  h->slots = (uint64_t*)calloc(cap, sizeof(uint64_t));
  h->mask = cap - 1;
  return h->slots ? 0 : -1;
}

/* returns 1 when newly inserted */
static inline int hset_insert(hset* h, uint64_t key) {
  uint64_t k = key + 1, i = mix64(key) & h->mask;
  for (;;) {
    uint64_t cur = h->slots[i];
    if (cur == 0) { h->slots[i] = k; return 1; }
    if (cur == k) return 0;
    i = (i + 1) & h->mask;
  }
}

#define CHUNK 4096

/*
 * Generate m distinct edges.  gamma_u/gamma_v <= 0 selects uniform (ER)
 * endpoints.  hubs_u/hubs_v planted hubs of degree hub_deg on each side (the
 * lowest ids, which are also the Chung-Lu heavy heads).  Returns 0 on
 * success, -1 on allocation failure, -2 if the candidate stream cannot reach
 * m distinct edges within 64*m draws (graph too dense for its shape).
 */
int bbc_synth_generate(int64_t n_u, int64_t n_v, int64_t m, double gamma_u, double gamma_v,
                       double p_neg, uint64_t seed, int32_t hubs_u, int32_t hubs_v, int64_t hub_deg,
                       int32_t* out_u, int32_t* out_v, int8_t* out_s) {
  if (m < 0 || n_u <= 0 || n_v <= 0) return m == 0 ? 0 : -3;
  hset h;
  if (hset_init(&h, m)) return -1;
  sampler su, sv;
  sampler_init(&su, n_u, gamma_u);
  sampler_init(&sv, n_v, gamma_v);
  int64_t got = 0;
  /* planted hubs first: hub k on U is u=k, partners uniform over V */
  for (int side = 0; side < 2; ++side) {
    int32_t hubs = side == 0 ? hubs_u : hubs_v;
    int64_t other = side == 0 ? n_v : n_u;
    for (int32_t k = 0; k < hubs && got < m; ++k) {
      int64_t want = hub_deg < other ? hub_deg : other;
      int64_t placed = 0;
      uint32_t stream = (uint32_t)(3 + 2 * k + side) + 16u;
      for (uint64_t i = 0; placed < want && got < m && i < (uint64_t)want * 64; ++i) {
        int64_t p = uniform_index(draw(seed, stream, i), other);
        int64_t uu = side == 0 ? k : p, vv = side == 0 ? p : k;
        if (hset_insert(&h, ((uint64_t)uu << 32) | (uint64_t)vv)) {
          out_u[got] = (int32_t)uu; out_v[got] = (int32_t)vv; ++got; ++placed;
        }
      }
    }
  }
  int64_t limit = m * 64 + 1024;
  int64_t cu[CHUNK], cv[CHUNK];
  for (int64_t base = 0; got < m; base += CHUNK) {
    if (base > limit) { free(h.slots); return -2; }
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < CHUNK; ++j) {
      cu[j] = sample(&su, draw(seed, 0, (uint64_t)(base + j)));
      cv[j] = sample(&sv, draw(seed, 1, (uint64_t)(base + j)));
    }
    for (int64_t j = 0; j < CHUNK && got < m; ++j) {
      if (hset_insert(&h, ((uint64_t)cu[j] << 32) | (uint64_t)cv[j])) {
        out_u[got] = (int32_t)cu[j]; out_v[got] = (int32_t)cv[j]; ++got;
      }
    }
  }
  free(h.slots);
  uint64_t thr = (uint64_t)(p_neg * 18446744073709551616.0);
  if (p_neg >= 1.0) thr = UINT64_MAX;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < m; ++j)
    out_s[j] = (p_neg > 0.0 && draw(seed, 2, (uint64_t)j) < thr) ? (int8_t)-1 : (int8_t)1;
  return 0;
}
