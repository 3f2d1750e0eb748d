/* ORACLE / TEST INFRASTRUCTURE ONLY — see dwdp_oracle.h for scope and
 * pinning. Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj). */
#include "dwdp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ===================================================================== */
/* RNG: std::mt19937_64 + the hand-written transforms of rng.hpp:17-70.  */

typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) +
               (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    const uint64_t lower = (1ULL << 31) - 1, upper = ~lower;
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:29-31 */
static double rng_u01(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

/* rng.hpp:34-43 */
static uint64_t rng_below(mt64* g, uint64_t n) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = mt64_next(g);
  } while (x >= limit);
  return x % n;
}

/* rng.hpp:51-58 */
static double rng_normal(mt64* g, double mean, double sd) {
  double u1 = rng_u01(g);
  while (u1 <= 0.0) u1 = rng_u01(g);
  const double u2 = rng_u01(g);
  const double z = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
  return mean + sd * z;
}

/* rng.hpp:60-69 */
uint64_t oracle_mix(uint64_t a, uint64_t b) {
  uint64_t x = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

void oracle_rng_u64(uint64_t seed, int n, uint64_t* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int i = 0; i < n; ++i) out[i] = mt64_next(&g);
}

void oracle_rng_normal(uint64_t seed, int n, double mean, double sd, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int i = 0; i < n; ++i) out[i] = rng_normal(&g, mean, sd);
}

/* Walker alias table, rng.hpp:77-123 (stack discipline kept identical). */
typedef struct {
  int n;
  double* prob;
  uint32_t* alias;
} alias_table;

static void alias_build(alias_table* t, const double* w, int n) {
  double total = 0.0;
  for (int i = 0; i < n; ++i) total += w[i];
  t->n = n;
  t->prob = calloc((size_t)n, sizeof(double));
  t->alias = calloc((size_t)n, sizeof(uint32_t));
  double* scaled = malloc(sizeof(double) * (size_t)n);
  uint32_t* small = malloc(sizeof(uint32_t) * (size_t)n);
  uint32_t* large = malloc(sizeof(uint32_t) * (size_t)n);
  int ns = 0, nl = 0;
  for (int i = 0; i < n; ++i) {
    scaled[i] = w[i] * (double)n / total;
    if (scaled[i] < 1.0)
      small[ns++] = (uint32_t)i;
    else
      large[nl++] = (uint32_t)i;
  }
  while (ns > 0 && nl > 0) {
    const uint32_t s = small[--ns];
    const uint32_t l = large[nl - 1];
    t->prob[s] = scaled[s];
    t->alias[s] = l;
    scaled[l] -= 1.0 - scaled[s];
    if (scaled[l] < 1.0) {
      --nl;
      small[ns++] = l;
    }
  }
  for (int i = 0; i < nl; ++i) t->prob[large[i]] = 1.0;
  for (int i = 0; i < ns; ++i) t->prob[small[i]] = 1.0;
  free(scaled);
  free(small);
  free(large);
}

static int alias_sample(const alias_table* t, mt64* g) {
  const int i = (int)rng_below(g, (uint64_t)t->n);
  return rng_u01(g) < t->prob[i] ? i : (int)t->alias[i];
}

/* ===================================================================== */
/* Placement: src/placement.cpp:47-111.                                  */

int oracle_build_placement(int E, int N, int extra, int* local_count,
                           int* redundancy, int* local_sets, int* fetch_expert,
                           int* fetch_src, int capacity) {
  if (N < 2 || E < N || extra < 0) return 2; /* placement.cpp:77-81 */
  const int base = (E + N - 1) / N;
  const int c = base + extra < E ? base + extra : E;
  *local_count = c;
  *redundancy = N * c - E;
  if (capacity < N * E) return 0;
  int stride = E / N; /* placement.cpp:89-94 */
  if ((N - 1) * stride + c < E) stride = c;
  char* holds = calloc((size_t)N * (size_t)E, 1);
  for (int r = 0; r < N; ++r) {
    const int start = (r * stride) % E;
    for (int i = 0; i < c; ++i) holds[(size_t)r * E + (size_t)((start + i) % E)] = 1;
    int k = 0; /* sorted local set = ascending scan of the membership row */
    for (int e = 0; e < E; ++e)
      if (holds[(size_t)r * E + e]) local_sets[r * c + k++] = e;
  }
  /* assign_fetch_sources, placement.cpp:47-73: per destination, greedy
   * least-loaded holder, ties to the lowest rank (holders ascend). */
  int* load = malloc(sizeof(int) * (size_t)N);
  for (int r = 0; r < N; ++r) {
    memset(load, 0, sizeof(int) * (size_t)N);
    int k = 0;
    for (int e = 0; e < E; ++e) {
      if (holds[(size_t)r * E + e]) continue;
      int best = -1;
      for (int h = 0; h < N; ++h) {
        if (h == r || !holds[(size_t)h * E + e]) continue;
        if (best < 0 || load[h] < load[best]) best = h;
      }
      if (best < 0) {
        free(load);
        free(holds);
        return 3;
      }
      load[best]++;
      fetch_expert[r * (E - c) + k] = e;
      fetch_src[r * (E - c) + k] = best;
      ++k;
    }
  }
  free(load);
  free(holds);
  return 0;
}

/* ===================================================================== */
/* Copy plan: src/copyplan.cpp:25-80 (Listing 1 of the paper).          */

int oracle_build_copy_plan(const int64_t* sh, int n, uint64_t slice, int dst,
                           int64_t* out, int64_t* n_out) {
  if (slice == 0) return 2;
  for (int i = 0; i < n; ++i) {
    if (sh[4 * i + 2] <= 0) return 2;
    if (sh[4 * i] == dst) return 2;
    for (int j = 0; j < i; ++j)
      if (sh[4 * j] == sh[4 * i] && sh[4 * j + 1] == sh[4 * i + 1]) return 2;
  }
  int64_t* params = malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* peers = malloc(sizeof(int64_t) * (size_t)(n + 1));
  int np = 0, npe = 0;
  for (int i = 0; i < n; ++i) {
    int seen = 0;
    for (int j = 0; j < np; ++j) seen |= params[j] == sh[4 * i + 1];
    if (!seen) params[np++] = sh[4 * i + 1];
    seen = 0;
    for (int j = 0; j < npe; ++j) seen |= peers[j] == sh[4 * i];
    if (!seen) peers[npe++] = sh[4 * i];
  }
  /* sort peers ascending, then rotate left by dst mod #peers */
  for (int i = 1; i < npe; ++i)
    for (int j = i; j > 0 && peers[j - 1] > peers[j]; --j) {
      const int64_t t = peers[j];
      peers[j] = peers[j - 1];
      peers[j - 1] = t;
    }
  int64_t* rot = malloc(sizeof(int64_t) * (size_t)(npe + 1));
  const int phase = npe ? (int)((uint64_t)dst % (uint64_t)npe) : 0;
  for (int i = 0; i < npe; ++i) rot[i] = peers[(i + phase) % npe];
  const int64_t cap = *n_out;
  int64_t cnt = 0;
  for (int pi = 0; pi < np; ++pi) {
    uint64_t max_m = 0;
    for (int i = 0; i < n; ++i)
      if (sh[4 * i + 1] == params[pi] && (uint64_t)sh[4 * i + 2] > max_m)
        max_m = (uint64_t)sh[4 * i + 2];
    for (uint64_t off = 0; off < max_m; off += slice)
      for (int q = 0; q < npe; ++q)
        for (int i = 0; i < n; ++i) {
          if (sh[4 * i + 1] != params[pi] || sh[4 * i] != rot[q]) continue;
          const uint64_t size = (uint64_t)sh[4 * i + 2];
          if (off >= size) continue;
          const uint64_t chunk = slice < size - off ? slice : size - off;
          if (out && cnt < cap) {
            int64_t* o = out + 5 * cnt;
            o[0] = params[pi];
            o[1] = rot[q];
            o[2] = sh[4 * i + 3] + (int64_t)off;
            o[3] = (int64_t)off;
            o[4] = (int64_t)chunk;
          }
          ++cnt;
        }
  }
  *n_out = cnt;
  free(params);
  free(peers);
  free(rot);
  return 0;
}

/* ===================================================================== */
/* Workload: src/workload.cpp:85-173.                                    */

int oracle_route_tokens(int64_t tokens, int E, int k, double skew, uint64_t seed,
                        int64_t* counts) {
  if (tokens < 0 || k < 1 || k > E) return 2;
  for (int e = 0; e < E; ++e) counts[e] = 0;
  const int64_t a = tokens * k;
  if (a == 0) return 0;
  if (skew == 0.0) { /* workload.cpp:95-101 */
    for (int e = 0; e < E; ++e) counts[e] = a / E + (e < a % E ? 1 : 0);
    return 0;
  }
  double* w = malloc(sizeof(double) * (size_t)E);
  for (int e = 0; e < E; ++e) w[e] = pow((double)(e + 1), -skew);
  alias_table t;
  alias_build(&t, w, E);
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < a; ++i) counts[alias_sample(&t, &g)]++;
  free(t.prob);
  free(t.alias);
  free(w);
  return 0;
}

/* workload.cpp:115-133 */
static int64_t draw_length(int kind, double len, double ratio, double sd,
                           mt64* g, int64_t mnt) {
  double raw = len;
  if (kind == 1) raw = ratio * len + (len - ratio * len) * rng_u01(g);
  if (kind == 2) raw = rng_normal(g, len, sd);
  double c = raw < 1.0 ? 1.0 : raw;
  if (c > (double)mnt) c = (double)mnt;
  return (int64_t)llround(c);
}

int oracle_sample_batches(int kind, double len, double ratio, double sd,
                          int64_t mnt, int bpr, double skew, uint64_t seed,
                          int E, int k, int N, int iters, int64_t* tokens,
                          int64_t* requests, int64_t* routed) {
  if (len < 1 || bpr < 1 || skew < 0 || N < 1 || iters < 1) return 2;
  if (mnt < (int64_t)len) return 2;
  const int64_t qcap = (int64_t)iters * bpr + 1;
  int64_t* q = malloc(sizeof(int64_t) * (size_t)qcap);
  for (int r = 0; r < N; ++r) {
    mt64 g;
    mt64_seed(&g, oracle_mix(seed, 0x10000ULL + (uint64_t)r));
    int64_t head = 0, tail = 0;
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < bpr; ++j) q[tail++] = draw_length(kind, len, ratio, sd, &g, mnt);
      int64_t used = 0, reqs = 0;
      while (head < tail && used + q[head] <= mnt) {
        used += q[head++];
        ++reqs;
      }
      tokens[it * N + r] = used;
      requests[it * N + r] = reqs;
      const uint64_t rs = oracle_mix(oracle_mix(seed, 0x20000ULL + (uint64_t)r), (uint64_t)it);
      if (routed) oracle_route_tokens(used, E, k, skew, rs, routed + ((int64_t)it * N + r) * E);
    }
  }
  free(q);
  return 0;
}

/* ===================================================================== */
/* Cost formulas: src/modelspec.cpp:32-86.                               */

double oracle_expert_shard_bytes(int64_t h, int64_t f, double wb) {
  return 3.0 * (double)h * (double)f * wb;
}

void oracle_moe_entries(int64_t h, int64_t f, int64_t fs, double wb, double ab,
                        double tokens, double pairs, int touched, double* o) {
  o[0] = 2.0 * pairs * 3.0 * (double)h * (double)f;
  o[1] = (double)touched * oracle_expert_shard_bytes(h, f, wb) + 2.0 * pairs * (double)h * ab;
  o[2] = o[3] = 0.0;
  if (fs > 0) {
    o[2] = 2.0 * tokens * 3.0 * (double)h * (double)fs;
    o[3] = 3.0 * (double)h * (double)fs * wb + tokens * (double)h * ab;
  }
}

/* ===================================================================== */
/* MoE numerics (north-star semantics; DeepSeek-V3 routing).             */

static inline float bf16_to_f32(uint16_t v) {
  union {
    uint32_t u;
    float f;
  } c;
  c.u = (uint32_t)v << 16;
  return c.f;
}

static inline uint16_t f32_to_bf16(float f) { /* round to nearest even */
  union {
    uint32_t u;
    float f;
  } c;
  c.f = f;
  if ((c.u & 0x7f800000u) == 0x7f800000u && (c.u & 0x7fffffu)) return (uint16_t)((c.u >> 16) | 0x40);
  const uint32_t lsb = (c.u >> 16) & 1u;
  return (uint16_t)((c.u + 0x7fffu + lsb) >> 16);
}

float oracle_expf(float x) {
  if (x < -87.0f) return 0.0f;
  if (x > 88.0f) return INFINITY;
  const float n = rintf(x * 1.44269504088896341f);
  float r = fmaf(n, -0.693145751953125f, x);
  r = fmaf(n, -1.428606765330187e-06f, r);
  float p = 1.38888889e-3f;
  p = fmaf(p, r, 8.33333333e-3f);
  p = fmaf(p, r, 4.16666667e-2f);
  p = fmaf(p, r, 1.66666667e-1f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  return ldexpf(p, (int)n);
}

float oracle_sigmoidf(float x) { return 1.0f / (1.0f + oracle_expf(-x)); }

uint64_t oracle_tensor_seed(uint64_t base, int layer, int expert, int t) {
  return oracle_mix(oracle_mix(base, 0x1000ULL + (uint64_t)layer),
                    (uint64_t)expert * 8ULL + (uint64_t)t);
}

static inline float hash_val(uint64_t seed, int64_t i, float scale) {
  const uint32_t u = (uint32_t)(oracle_mix(seed, (uint64_t)i) >> 40);
  const float v = (float)u * 0x1.0p-23f - 1.0f;
  return v * scale;
}

typedef struct {
  uint64_t seed;
  int64_t n;
  float scale;
  uint16_t* out;
} fill_arg;

static void fill_chunk(void* p, int64_t c) {
  const fill_arg* a = (const fill_arg*)p;
  const int64_t lo = c << 20, hi = lo + (1 << 20) < a->n ? lo + (1 << 20) : a->n;
  for (int64_t i = lo; i < hi; ++i) a->out[i] = f32_to_bf16(hash_val(a->seed, i, a->scale));
}

static void parallel_for(int64_t n, int nthreads, void (*fn)(void*, int64_t), void* arg);

void oracle_fill_bf16(uint64_t seed, int64_t n, float scale, uint16_t* out) {
  fill_arg a = {seed, n, scale, out};
  parallel_for((n + (1 << 20) - 1) >> 20, 0, fill_chunk, &a);
}

/* ---- tiny parallel-for ------------------------------------------------ */
typedef struct {
  void (*fn)(void*, int64_t);
  void* arg;
  int64_t n;
  int64_t* next;
  pthread_mutex_t* mu;
} pf_job;

static void* pf_worker(void* p) {
  pf_job* j = (pf_job*)p;
  for (;;) {
    pthread_mutex_lock(j->mu);
    const int64_t i = (*j->next)++;
    pthread_mutex_unlock(j->mu);
    if (i >= j->n) break;
    j->fn(j->arg, i);
  }
  return NULL;
}

static void parallel_for(int64_t n, int nthreads, void (*fn)(void*, int64_t), void* arg) {
  if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (nthreads > n) nthreads = (int)(n > 0 ? n : 1);
  int64_t next = 0;
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  pf_job job = {fn, arg, n, &next, &mu};
  pthread_t* th = malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int i = 1; i < nthreads; ++i) pthread_create(&th[i], NULL, pf_worker, &job);
  pf_worker(&job);
  for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
}

/* ---- router ------------------------------------------------------------ */

/* better(a, ia, b, ib): a outranks b (higher value, ties to lower index). */
static inline int better(float a, int ia, float b, int ib) {
  return a > b || (a == b && ia < ib);
}

/* One token: scores -> selection. choice[e] = selection key, sc[e] = weight
 * source (sigmoid score, or exp(l - max) for softmax). */
static void select_token(const oracle_moe_config* cfg, const float* logit,
                         const float* bias, int32_t* idx, float* wts) {
  const int E = cfg->num_experts, k = cfg->top_k;
  float choice[1024], score[1024];
  int keep[1024];
  for (int e = 0; e < E; ++e) {
    if (cfg->scoring == 1) {
      score[e] = oracle_sigmoidf(logit[e]);
      choice[e] = score[e] + (bias ? bias[e] : 0.0f);
    } else {
      choice[e] = logit[e];
    }
    keep[e] = 1;
  }
  const int G = cfg->n_group > 0 ? cfg->n_group : 1;
  if (G > 1 && cfg->topk_group < G) {
    const int gs = E / G;
    float gscore[64];
    int gsel[64];
    for (int g = 0; g < G; ++g) { /* sum of the top-2 choice values */
      int b1 = -1, b2 = -1;
      for (int e = g * gs; e < (g + 1) * gs; ++e) {
        if (b1 < 0 || better(choice[e], e, choice[b1], b1)) {
          b2 = b1;
          b1 = e;
        } else if (b2 < 0 || better(choice[e], e, choice[b2], b2)) {
          b2 = e;
        }
      }
      gscore[g] = gs >= 2 ? choice[b1] + choice[b2] : choice[b1];
      gsel[g] = 0;
    }
    for (int s = 0; s < cfg->topk_group; ++s) {
      int b = -1;
      for (int g = 0; g < G; ++g)
        if (!gsel[g] && (b < 0 || better(gscore[g], g, gscore[b], b))) b = g;
      gsel[b] = 1;
    }
    /* HF masked_fill(~mask, 0.0): masked experts compete with value 0. */
    for (int e = 0; e < E; ++e)
      if (!gsel[e / gs]) {
        choice[e] = 0.0f;
        keep[e] = 0;
      }
  }
  (void)keep;
  int taken[1024] = {0};
  for (int j = 0; j < k; ++j) {
    int b = -1;
    for (int e = 0; e < E; ++e)
      if (!taken[e] && (b < 0 || better(choice[e], e, choice[b], b))) b = e;
    taken[b] = 1;
    idx[j] = b;
  }
  if (cfg->scoring == 1) {
    for (int j = 0; j < k; ++j) wts[j] = score[idx[j]];
    if (cfg->norm_topk) {
      float s = 0.0f;
      for (int j = 0; j < k; ++j) s += wts[j];
      s += 1e-20f;
      for (int j = 0; j < k; ++j) wts[j] = wts[j] / s;
    }
  } else {
    const float m = logit[idx[0]]; /* top-1 logit is the max */
    for (int j = 0; j < k; ++j) wts[j] = oracle_expf(logit[idx[j]] - m);
    float s = 0.0f;
    if (cfg->norm_topk)
      for (int j = 0; j < k; ++j) s += wts[j];
    else
      for (int e = 0; e < E; ++e) s += oracle_expf(logit[e] - m);
    for (int j = 0; j < k; ++j) wts[j] = wts[j] / s;
  }
  for (int j = 0; j < k; ++j) wts[j] = wts[j] * cfg->routed_scale;
}

/* Router logits (north-star semantics of x . Wr^T in fp32, made exactly
 * reproducible): every bf16 row is put on a 22-bit fixed-point grid relative
 * to its largest exponent field emax (value = Q * 2^(emax - 148); elements
 * more than 14 binades below the row maximum are truncated to the grid), the
 * dot product of two rows is the exact int64 sum of Q_x * Q_w, rounded ONCE to
 * fp32 and scaled by 2^(emax_x + emax_w - 296). Order-free, so the device
 * computes it bit-identically with int8 tensor cores (three digit planes). */
static inline uint16_t f32_bits_bf16(float f) { /* exact for bf16 values */
  union {
    float f;
    uint32_t u;
  } c;
  c.f = f;
  return (uint16_t)(c.u >> 16);
}

static void quant_row(const uint16_t* b, const float* f, int64_t K, int32_t* q, int* emax) {
  int m = 0;
  for (int64_t i = 0; i < K; ++i) {
    const uint16_t v = b ? b[i] : f32_bits_bf16(f[i]);
    const int E = (v >> 7) & 0xFF, M = v & 0x7F;
    const int mant = E ? (M | 0x80) : M, eb = E ? E : 1;
    if (mant && eb > m) m = eb;
  }
  if (m == 0) m = 1;
  for (int64_t i = 0; i < K; ++i) {
    const uint16_t v = b ? b[i] : f32_bits_bf16(f[i]);
    const int E = (v >> 7) & 0xFF, M = v & 0x7F;
    const int mant = E ? (M | 0x80) : M, eb = E ? E : 1;
    const int sh = eb - m + 14;
    const int qq = sh >= 0 ? (mant << sh) : (sh > -8 ? (mant >> -sh) : 0);
    q[i] = (v & 0x8000) ? -qq : qq;
  }
  *emax = m;
}

typedef struct {
  const oracle_moe_config* cfg;
  const uint16_t* x16;
  const float* x32;
  const int32_t* wq; /* [E][h] quantised router rows */
  const int* we;     /* [E] their exponents */
  const float* bias;
  float* logits;
  int32_t* idx;
  float* wts;
  int64_t T;
} route_arg;

/* Tokens are routed in blocks of RB so each quantised router row is reused
 * from cache across the block; every logit is still one exact int64 sum. */
#define RB 8
static void route_one(void* p, int64_t blk) {
  route_arg* a = (route_arg*)p;
  const int64_t h = a->cfg->hidden;
  const int E = a->cfg->num_experts;
  const int64_t t0 = blk * RB;
  const int n = (int)(a->T - t0 < RB ? a->T - t0 : RB);
  int32_t* xq = malloc(sizeof(int32_t) * (size_t)(h * RB));
  int ex[RB];
  for (int r = 0; r < n; ++r) {
    const int64_t t = t0 + r;
    quant_row(a->x16 ? a->x16 + t * h : NULL, a->x32 ? a->x32 + t * h : NULL, h, xq + r * h,
              &ex[r]);
  }
  for (int e = 0; e < E; ++e) {
    const int32_t* wr = a->wq + (int64_t)e * h;
    for (int r = 0; r < n; ++r) {
      const int32_t* xr = xq + r * h;
      int64_t z = 0;
      for (int64_t i = 0; i < h; ++i) z += (int64_t)xr[i] * (int64_t)wr[i];
      a->logits[(t0 + r) * E + e] = ldexpf((float)z, ex[r] + a->we[e] - 296);
    }
  }
  free(xq);
  for (int r = 0; r < n; ++r) {
    const int64_t t = t0 + r;
    select_token(a->cfg, a->logits + t * E, a->bias, a->idx + t * a->cfg->top_k,
                 a->wts + t * a->cfg->top_k);
  }
}

/* Quantise the router rows once, route every token, release. */
static void route_all(const oracle_moe_config* cfg, const uint16_t* x16, const float* x32,
                      int64_t T, const uint16_t* w16, const float* w32, const float* bias,
                      float* logits, int32_t* idx, float* wts, int nthreads) {
  const int64_t h = cfg->hidden;
  const int E = cfg->num_experts;
  int32_t* wq = malloc(sizeof(int32_t) * (size_t)(E * h));
  int* we = malloc(sizeof(int) * (size_t)E);
  for (int e = 0; e < E; ++e)
    quant_row(w16 ? w16 + (int64_t)e * h : NULL, w32 ? w32 + (int64_t)e * h : NULL, h,
              wq + (int64_t)e * h, &we[e]);
  route_arg a = {cfg, x16, x32, wq, we, bias, logits, idx, wts, T};
  parallel_for((T + RB - 1) / RB, nthreads, route_one, &a);
  free(wq);
  free(we);
}

void oracle_route(const oracle_moe_config* cfg, const uint16_t* x, int64_t T,
                  const uint16_t* w_router, const float* bias, float* logits,
                  int32_t* idx, float* wts) {
  route_all(cfg, x, NULL, T, w_router, NULL, bias, logits, idx, wts, 0);
}

int64_t oracle_permute(const int32_t* idx, int64_t T, int E, int k, int align,
                       int32_t* counts, int64_t* row_of) {
  int64_t* cursor = calloc((size_t)E, sizeof(int64_t));
  for (int e = 0; e < E; ++e) counts[e] = 0;
  for (int64_t p = 0; p < T * k; ++p) counts[idx[p]]++;
  int64_t off = 0;
  for (int e = 0; e < E; ++e) {
    cursor[e] = off;
    off += (counts[e] + align - 1) / align * align;
  }
  /* stable: pairs visited in (t, k) order */
  for (int64_t p = 0; p < T * k; ++p) row_of[p] = cursor[idx[p]]++;
  free(cursor);
  return off;
}

/* ---- expert FFN -------------------------------------------------------- */

static inline float dotf(const float* a, const float* b, int64_t n) {
  float acc[16] = {0};
  int64_t i = 0;
  for (; i + 16 <= n; i += 16)
    for (int j = 0; j < 16; ++j) acc[j] += a[i + j] * b[i + j];
  float s = 0.0f;
  for (int j = 0; j < 16; ++j) s += acc[j];
  for (; i < n; ++i) s += a[i] * b[i];
  return s;
}

static inline float siluf(float g) { return g / (1.0f + expf(-g)); }

static inline float dot_bf16(const float* a, const uint16_t* w, int64_t n) {
  float acc[16] = {0};
  int64_t i = 0;
  for (; i + 16 <= n; i += 16)
    for (int j = 0; j < 16; ++j) acc[j] += a[i + j] * bf16_to_f32(w[i + j]);
  float s = 0.0f;
  for (int j = 0; j < 16; ++j) s += acc[j];
  for (; i < n; ++i) s += a[i] * bf16_to_f32(w[i]);
  return s;
}

/* ---- W8A8 emulation ---------------------------------------------------
 * Follows the device W8A8 path (paper_2604_01621_b200/csrc/kernels.cu
 * fp8 helpers + gemm_sm100.cu FP8 epilogues): weights and activations are
 * e4m3 with per-row fp32 scales; GEMM products are exact, sums fp32; GEMM1
 * output = acc * (sx * sw), H = bf16(silu(g) * u) re-quantised per row;
 * GEMM2 output = acc * (sh * sd). */
uint8_t oracle_f32_to_e4m3(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  const uint32_t s = (u >> 24) & 0x80u;
  const uint32_t a = u & 0x7fffffffu;
  if (a > 0x7f800000u) return (uint8_t)(s | 0x7f);
  if (a >= 0x43e00000u) return (uint8_t)(s | 0x7e);
  const int e = (int)(a >> 23) - 127;
  if (e < -6) {
    float av;
    memcpy(&av, &a, 4);
    const float q = rintf(av * 512.0f);
    return (uint8_t)(s | (uint32_t)q);
  }
  const uint32_t m = a & 0x7fffffu;
  uint32_t m3 = m >> 20;
  const uint32_t rem = m & 0xfffffu;
  if (rem > 0x80000u || (rem == 0x80000u && (m3 & 1u))) ++m3;
  uint32_t code = ((uint32_t)(e + 7) << 3) + m3;
  if (code > 0x7e) code = 0x7e;
  return (uint8_t)(s | code);
}

float oracle_e4m3_to_f32(uint8_t b) {
  const uint32_t e = (b >> 3) & 0xf, m = b & 7;
  float v;
  if (e) {
    const uint32_t bits = ((e + 120) << 23) | (m << 20);
    memcpy(&v, &bits, 4);
  } else {
    v = (float)m * 0.001953125f;
  }
  return (b & 0x80) ? -v : v;
}

void oracle_e4m3_encode(const float* x, int64_t n, uint8_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = oracle_f32_to_e4m3(x[i]);
}

void oracle_quant_row_e4m3(const float* v, int64_t K, uint8_t* q, float* s) {
  float amax = 0.0f;
  for (int64_t i = 0; i < K; ++i) amax = fmaxf(amax, fabsf(v[i]));
  const float sc = amax > 0.0f ? amax / 448.0f : 1.0f;
  for (int64_t i = 0; i < K; ++i) q[i] = oracle_f32_to_e4m3(v[i] / sc);
  *s = sc;
}

/* ---- NVFP4 (W4A4) ------------------------------------------------------
 * Follows kernels.cu nvfp4_block / nvfp4_fill_rows_kernel / the permute's
 * NVFP4 branch and the kind::mxf4nvf4 GEMM (gemm_sm100.cu): products of
 * e2m1 codes times their e4m3 block scales are exact in fp32, sums fp32,
 * epilogue acc * (s_a * s_b). */
uint8_t oracle_f32_to_e2m1(float x) {
  const float a = fabsf(x);
  const uint8_t c = a <= 0.25f ? 0 : a < 0.75f ? 1 : a <= 1.25f ? 2 : a < 1.75f ? 3
                  : a <= 2.5f ? 4 : a < 3.5f ? 5 : a <= 5.0f ? 6 : 7;
  return (uint8_t)(signbit(x) ? (c | 8) : c); /* sign kept, as cvt.rn.satfinite.e2m1x2 */
}

float oracle_e2m1_to_f32(uint8_t code) {
  static const float mag[8] = {0.0f, 0.5f, 1.0f, 1.5f, 2.0f, 3.0f, 4.0f, 6.0f};
  const float v = mag[code & 7];
  return (code & 8) ? -v : v;
}

void oracle_nvfp4_quant_row(const float* v, int64_t K, uint8_t* codes, uint8_t* sf, float* s) {
  float amax = 0.0f;
  for (int64_t i = 0; i < K; ++i) amax = fmaxf(amax, fabsf(v[i]));
  const float rs = amax > 0.0f ? amax / 2688.0f : 1.0f;
  for (int64_t b = 0; b < K / 16; ++b) {
    float bmax = 0.0f;
    for (int i = 0; i < 16; ++i) bmax = fmaxf(bmax, fabsf(v[b * 16 + i]));
    const uint8_t code = oracle_f32_to_e4m3(bmax / (6.0f * rs));
    const float ds = oracle_e4m3_to_f32(code) * rs;
    const float inv = ds > 0.0f ? 1.0f / ds : 0.0f;
    sf[b] = code;
    for (int i = 0; i < 8; ++i) {
      uint8_t lo = 0, hi = 0;
      if (ds > 0.0f) {
        lo = oracle_f32_to_e2m1(v[b * 16 + 2 * i] * inv);
        hi = oracle_f32_to_e2m1(v[b * 16 + 2 * i + 1] * inv);
      }
      codes[b * 8 + i] = (uint8_t)(lo | (hi << 4));
    }
  }
  *s = rs;
}

int64_t oracle_nvfp4_sf_offset(int64_t row, int64_t block, int64_t K) {
  return ((row >> 7) * (K >> 6) + (block >> 2)) * 512 + (row & 31) * 16 + ((row >> 5) & 3) * 4 +
         (block & 3);
}

/* Quantise n rows of length K into dequantised-grid floats (q values times
 * their block scales for nvfp4; not multiplied by the row scale) + scales. */
static void quant_rows_grid_mode(int mode, const float* src, int64_t n, int64_t K, float* grid,
                                 float* scales, uint8_t* tmp) {
  for (int64_t r = 0; r < n; ++r) {
    if (mode == 2) {
      uint8_t* sf = tmp + K / 2;
      oracle_nvfp4_quant_row(src + r * K, K, tmp, sf, scales + r);
      for (int64_t i = 0; i < K; ++i)
        grid[r * K + i] = oracle_e2m1_to_f32((uint8_t)((tmp[i / 2] >> (4 * (i & 1))) & 15)) *
                          oracle_e4m3_to_f32(sf[i / 16]);
    } else {
      oracle_quant_row_e4m3(src + r * K, K, tmp, scales + r);
      for (int64_t i = 0; i < K; ++i) grid[r * K + i] = oracle_e4m3_to_f32(tmp[i]);
    }
  }
}

static void ffn_rows_w8a8(int mode, const float* gate, const float* up, const float* down, int64_t h,
                          int64_t f, const float* const* xr, const float* scale,
                          float* const* yr, int n) {
#define quant_rows_grid(...) quant_rows_grid_mode(mode, __VA_ARGS__)
  const int64_t mx = h > f ? h : f;
  uint8_t* tmp = malloc((size_t)mx);
  float* gq = malloc(sizeof(float) * (size_t)(f * h));
  float* uq = malloc(sizeof(float) * (size_t)(f * h));
  float* dq = malloc(sizeof(float) * (size_t)(h * f));
  float* gs = malloc(sizeof(float) * (size_t)f);
  float* us = malloc(sizeof(float) * (size_t)f);
  float* ds = malloc(sizeof(float) * (size_t)h);
  quant_rows_grid(gate, f, h, gq, gs, tmp);
  quant_rows_grid(up, f, h, uq, us, tmp);
  quant_rows_grid(down, h, f, dq, ds, tmp);
  float* xq = malloc(sizeof(float) * (size_t)h);
  float* hb = malloc(sizeof(float) * (size_t)f);
  float* hq = malloc(sizeof(float) * (size_t)f);
  for (int r = 0; r < n; ++r) {
    float sx, sh;
    quant_rows_grid(xr[r], 1, h, xq, &sx, tmp);
    for (int64_t j = 0; j < f; ++j) {
      const float g = dotf(xq, gq + j * h, h) * (sx * gs[j]);
      const float u = dotf(xq, uq + j * h, h) * (sx * us[j]);
      hb[j] = bf16_to_f32(f32_to_bf16(siluf(g) * u));
    }
    quant_rows_grid(hb, 1, f, hq, &sh, tmp);
    for (int64_t i = 0; i < h; ++i)
      yr[r][i] += scale[r] * bf16_to_f32(f32_to_bf16(dotf(hq, dq + i * f, f) * (sh * ds[i])));
  }
  free(tmp); free(gq); free(uq); free(dq); free(gs); free(us); free(ds);
  free(xq); free(hb); free(hq);
#undef quant_rows_grid
}

static void ffn_rows_bf16(const uint16_t* gate, const uint16_t* up, const uint16_t* down,
                          int64_t h, int64_t f, const float* const* xr, const float* scale,
                          float* const* yr, int n, float* hbuf) {
  /* weight rows outer, token rows inner: each weight row is streamed once
   * and widened to fp32 once (dotf over the widened row is the same sum as
   * dot_bf16 over the bf16 row) */
  const int64_t mx = h > f ? h : f;
  float* wg = malloc(sizeof(float) * (size_t)mx);
  float* wu = malloc(sizeof(float) * (size_t)mx);
  for (int64_t j = 0; j < f; ++j) {
    for (int64_t i = 0; i < h; ++i) {
      wg[i] = bf16_to_f32(gate[j * h + i]);
      wu[i] = bf16_to_f32(up[j * h + i]);
    }
    for (int r = 0; r < n; ++r)
      hbuf[(int64_t)r * f + j] = siluf(dotf(xr[r], wg, h)) * dotf(xr[r], wu, h);
  }
  for (int64_t i = 0; i < h; ++i) {
    for (int64_t j = 0; j < f; ++j) wg[j] = bf16_to_f32(down[i * f + j]);
    for (int r = 0; r < n; ++r) yr[r][i] += scale[r] * dotf(hbuf + (int64_t)r * f, wg, f);
  }
  free(wg);
  free(wu);
}

/* y_rows[r] += scale[r] * FFN(x_rows[r]) for n rows of one expert. Weight
 * rows outer, token rows inner (each weight row streamed once); every output
 * is the same dotf as a row-at-a-time loop. hbuf: [n][f]. */
static void ffn_rows(const float* gate, const float* up, const float* down,
                     int64_t h, int64_t f, const float* const* xr,
                     const float* scale, float* const* yr, int n, float* hbuf) {
  for (int64_t j = 0; j < f; ++j)
    for (int r = 0; r < n; ++r) {
      const float g = dotf(xr[r], gate + j * h, h);
      const float u = dotf(xr[r], up + j * h, h);
      hbuf[(int64_t)r * f + j] = siluf(g) * u;
    }
  for (int64_t i = 0; i < h; ++i)
    for (int r = 0; r < n; ++r)
      yr[r][i] += scale[r] * dotf(hbuf + (int64_t)r * f, down + i * f, f);
}

typedef struct {
  const oracle_moe_config* cfg;
  uint64_t base;
  int layer;
  const float* x; /* [T][h] fp32 */
  int64_t T;
  const int32_t* idx;
  const float* wts;
  /* explicit weights (NULL for seeded) */
  const float *wg, *wu, *wd, *sg, *su, *sd;
  const uint16_t *const *bg, *const *bu, *const *bd; /* resident bf16 weights */
  float* part; /* [E+1][T][h] partial outputs when needed */
  int64_t* pairs_of; /* per expert: list of (t, j) pair ids; CSR */
  int64_t* pair_start;
  pthread_mutex_t mu;
} ffn_arg;

static void load_expert(ffn_arg* a, int e, int64_t f, float* g, float* u, float* d) {
  const int64_t h = a->cfg->hidden;
  const int E = a->cfg->num_experts;
  if (a->wg) {
    if (e < E) {
      memcpy(g, a->wg + (int64_t)e * f * h, sizeof(float) * (size_t)(f * h));
      memcpy(u, a->wu + (int64_t)e * f * h, sizeof(float) * (size_t)(f * h));
      memcpy(d, a->wd + (int64_t)e * h * f, sizeof(float) * (size_t)(h * f));
    } else {
      memcpy(g, a->sg, sizeof(float) * (size_t)(f * h));
      memcpy(u, a->su, sizeof(float) * (size_t)(f * h));
      memcpy(d, a->sd, sizeof(float) * (size_t)(h * f));
    }
    return;
  }
  const float sk = 1.0f / sqrtf((float)h), sf = 1.0f / sqrtf((float)f);
  const uint64_t s0 = oracle_tensor_seed(a->base, a->layer, e, 0);
  const uint64_t s1 = oracle_tensor_seed(a->base, a->layer, e, 1);
  const uint64_t s2 = oracle_tensor_seed(a->base, a->layer, e, 2);
  for (int64_t i = 0; i < f * h; ++i) {
    g[i] = bf16_to_f32(f32_to_bf16(hash_val(s0, i, sk)));
    u[i] = bf16_to_f32(f32_to_bf16(hash_val(s1, i, sk)));
    d[i] = bf16_to_f32(f32_to_bf16(hash_val(s2, i, sf)));
  }
}

static void expert_job(void* p, int64_t e64) {
  ffn_arg* a = (ffn_arg*)p;
  const int e = (int)e64;
  const int E = a->cfg->num_experts;
  const int64_t h = a->cfg->hidden;
  const int64_t f = e < E ? a->cfg->ffn : a->cfg->shared_ffn;
  const int64_t n = e < E ? a->pair_start[e + 1] - a->pair_start[e] : a->T;
  if (n == 0) return;
  const int resident = a->bg != NULL;
  float* g = resident ? NULL : malloc(sizeof(float) * (size_t)(f * h));
  float* u = resident ? NULL : malloc(sizeof(float) * (size_t)(f * h));
  float* d = resident ? NULL : malloc(sizeof(float) * (size_t)(h * f));
  float* hb = malloc(sizeof(float) * (size_t)(f * n));
  float* out = calloc((size_t)(n * h), sizeof(float));
  const float** xr = malloc(sizeof(float*) * (size_t)n);
  float** yr = malloc(sizeof(float*) * (size_t)n);
  float* sc = malloc(sizeof(float) * (size_t)n);
  if (!resident) load_expert(a, e, f, g, u, d);
  for (int64_t r = 0; r < n; ++r) {
    const int64_t pid = e < E ? a->pairs_of[a->pair_start[e] + r] : r * a->cfg->top_k;
    const int64_t t = pid / a->cfg->top_k;
    xr[r] = a->x + t * h;
    yr[r] = out + r * h;
    sc[r] = e < E ? a->wts[pid] : 1.0f;
  }
  if (a->cfg->w8a8) {
    if (resident) {
      g = malloc(sizeof(float) * (size_t)(f * h));
      u = malloc(sizeof(float) * (size_t)(f * h));
      d = malloc(sizeof(float) * (size_t)(h * f));
      for (int64_t i = 0; i < f * h; ++i) {
        g[i] = bf16_to_f32(a->bg[e][i]);
        u[i] = bf16_to_f32(a->bu[e][i]);
        d[i] = bf16_to_f32(a->bd[e][i]);
      }
    }
    ffn_rows_w8a8(a->cfg->w8a8, g, u, d, h, f, xr, sc, yr, (int)n);
  } else if (resident)
    ffn_rows_bf16(a->bg[e], a->bu[e], a->bd[e], h, f, xr, sc, yr, (int)n, hb);
  else
    ffn_rows(g, u, d, h, f, xr, sc, yr, (int)n, hb);
  /* scatter into the per-pair partial buffer (deterministic reduction later) */
  for (int64_t r = 0; r < n; ++r) {
    const int64_t pid = e < E ? a->pairs_of[a->pair_start[e] + r] : -1 - (r);
    float* dst = pid >= 0 ? a->part + pid * h
                          : a->part + (a->T * a->cfg->top_k + r) * h;
    memcpy(dst, out + r * h, sizeof(float) * (size_t)h);
  }
  free(g);
  free(u);
  free(d);
  free(hb);
  free(out);
  free(xr);
  free(yr);
  free(sc);
}

static void moe_forward_common(const oracle_moe_config* cfg, uint64_t base,
                               int layer, const float* x, int64_t T,
                               const int32_t* idx, const float* wts,
                               const float* wg, const float* wu,
                               const float* wd, const float* sg,
                               const float* su, const float* sd,
                               const uint16_t* const* bg, const uint16_t* const* bu,
                               const uint16_t* const* bd, float* y, int nthreads) {
  const int E = cfg->num_experts, k = cfg->top_k;
  const int64_t h = cfg->hidden;
  ffn_arg a;
  memset(&a, 0, sizeof a);
  a.cfg = cfg;
  a.base = base;
  a.layer = layer;
  a.x = x;
  a.T = T;
  a.idx = idx;
  a.wts = wts;
  a.wg = wg;
  a.wu = wu;
  a.wd = wd;
  a.sg = sg;
  a.su = su;
  a.sd = sd;
  a.bg = bg;
  a.bu = bu;
  a.bd = bd;
  const int64_t npart = T * k + (cfg->shared_ffn > 0 ? T : 0);
  a.part = calloc((size_t)(npart * h), sizeof(float));
  a.pair_start = calloc((size_t)E + 1, sizeof(int64_t));
  a.pairs_of = malloc(sizeof(int64_t) * (size_t)(T * k + 1));
  for (int64_t p = 0; p < T * k; ++p) a.pair_start[idx[p] + 1]++;
  for (int e = 0; e < E; ++e) a.pair_start[e + 1] += a.pair_start[e];
  int64_t* cur = malloc(sizeof(int64_t) * (size_t)E);
  for (int e = 0; e < E; ++e) cur[e] = a.pair_start[e];
  for (int64_t p = 0; p < T * k; ++p) a.pairs_of[cur[idx[p]]++] = p;
  free(cur);
  parallel_for(E + (cfg->shared_ffn > 0 ? 1 : 0), nthreads, expert_job, &a);
  /* combine in fixed k order, then the shared expert */
  for (int64_t t = 0; t < T; ++t)
    for (int64_t i = 0; i < h; ++i) {
      float s = 0.0f;
      for (int j = 0; j < k; ++j) s += a.part[(t * k + j) * h + i];
      if (cfg->shared_ffn > 0) s += a.part[(T * k + t) * h + i];
      y[t * h + i] = s;
    }
  free(a.part);
  free(a.pair_start);
  free(a.pairs_of);
}

void oracle_moe_forward_seeded(const oracle_moe_config* cfg, uint64_t base,
                               int layer, const uint16_t* x, int64_t T,
                               const float* bias, float* y, int32_t* idx,
                               float* wts, int nthreads) {
  const int64_t h = cfg->hidden;
  const int E = cfg->num_experts;
  uint16_t* wr = malloc(sizeof(uint16_t) * (size_t)(E * h));
  oracle_fill_bf16(oracle_tensor_seed(base, layer, E + 1, 0), E * h, 1.0f / sqrtf((float)h), wr);
  float* logits = malloc(sizeof(float) * (size_t)(T * E + 1));
  route_all(cfg, x, NULL, T, wr, NULL, bias, logits, idx, wts, nthreads);
  float* xf = malloc(sizeof(float) * (size_t)(T * h + 1));
  for (int64_t i = 0; i < T * h; ++i) xf[i] = bf16_to_f32(x[i]);
  moe_forward_common(cfg, base, layer, xf, T, idx, wts, NULL, NULL, NULL, NULL,
                     NULL, NULL, NULL, NULL, NULL, y, nthreads);
  free(xf);
  free(logits);
  free(wr);
}

void oracle_moe_forward_explicit(const oracle_moe_config* cfg, const float* x,
                                 int64_t T, const float* w_router,
                                 const float* bias, const float* w_gate,
                                 const float* w_up, const float* w_down,
                                 const float* s_gate, const float* s_up,
                                 const float* s_down, float* y, int32_t* idx,
                                 float* wts) {
  const int E = cfg->num_experts;
  float* logits = malloc(sizeof(float) * (size_t)(T * E + 1));
  route_all(cfg, NULL, x, T, NULL, w_router, bias, logits, idx, wts, 0);
  moe_forward_common(cfg, 0, 0, x, T, idx, wts, w_gate, w_up, w_down, s_gate,
                     s_up, s_down, NULL, NULL, NULL, y, 0);
  free(logits);
}

void oracle_moe_forward_bf16w(const oracle_moe_config* cfg, const uint16_t* x,
                              int64_t T, const uint16_t* w_router,
                              const float* bias, const uint16_t* const* gate,
                              const uint16_t* const* up,
                              const uint16_t* const* down, float* y,
                              int32_t* idx, float* wts, int nthreads) {
  const int64_t h = cfg->hidden;
  const int E = cfg->num_experts;
  float* logits = malloc(sizeof(float) * (size_t)(T * E + 1));
  route_all(cfg, x, NULL, T, w_router, NULL, bias, logits, idx, wts, nthreads);
  float* xf = malloc(sizeof(float) * (size_t)(T * h + 1));
  for (int64_t i = 0; i < T * h; ++i) xf[i] = bf16_to_f32(x[i]);
  moe_forward_common(cfg, 0, 0, xf, T, idx, wts, NULL, NULL, NULL, NULL, NULL, NULL, gate, up,
                     down, y, nthreads);
  free(xf);
  free(logits);
}
