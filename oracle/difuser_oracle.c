/*
 * difuser_oracle.c — TEST INFRASTRUCTURE ONLY: the parity CHECKER.
 *
 * A plain-C restatement of the DiFuseR reference's sketch-IM hot path
 * (/root/reference/proj).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; the product library never
 * does.  Each function cites the reference file:line it restates.  The
 * restatement is pinned against the reference's golden vectors and against
 * fixtures produced by the compiled reference itself (see difuser_oracle.h).
 */
#include "difuser_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9e3779b97f4a7c15ULL
#define FIXED_ONE (1u << 31)
#define HASH_MASK (FIXED_ONE - 1u)
#define VISITED ((int8_t)-1)
#define PHI 0.77351

static inline uint64_t rotl64(uint64_t x, int r) {
  return (x << r) | (x >> (64 - r));
}

/* proj/include/difuser/hash.hpp:9-16 */
uint64_t dor_fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

/* proj/include/difuser/hash.hpp:22-30 (counter-form splitmix64) */
uint64_t dor_splitmix64_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * GOLDEN;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* proj/include/difuser/hash.hpp:50-82: MurmurHash3_x64_128 of the 16-byte
 * block (a, b), seed 0 — one body round, no tail, len = 16. */
void dor_murmur3_pair(uint64_t a, uint64_t b, uint64_t out[2]) {
  const uint64_t c1 = 0x87c37b91114253d5ULL, c2 = 0x4cf5ad432745937fULL;
  uint64_t h1 = 0, h2 = 0;
  uint64_t k1 = rotl64(a * c1, 31) * c2;
  h1 = rotl64(h1 ^ k1, 27) + h2;
  h1 = h1 * 5 + 0x52dce729;
  uint64_t k2 = rotl64(b * c2, 33) * c1;
  h2 = rotl64(h2 ^ k2, 31) + h1;
  h2 = h2 * 5 + 0x38495ab5;
  h1 ^= 16;
  h2 ^= 16;
  h1 += h2;
  h2 += h1;
  h1 = dor_fmix64(h1);
  h2 = dor_fmix64(h2);
  h1 += h2;
  h2 += h1;
  out[0] = h1;
  out[1] = h2;
}

/* proj/include/difuser/hash.hpp:91-93 */
uint32_t dor_edge_hash(uint64_t u, uint64_t v) {
  uint64_t h[2];
  dor_murmur3_pair(u, v, h);
  return (uint32_t)h[0] & HASH_MASK;
}

/* proj/include/difuser/hash.hpp:101-103 */
uint64_t dor_register_hash(uint64_t jkey, uint64_t v) {
  return dor_fmix64(jkey + v * GOLDEN);
}

/* proj/include/difuser/sampling.hpp:23-25 */
uint32_t dor_random_value_at(uint64_t seed, uint32_t r) {
  return (uint32_t)(dor_splitmix64_at(seed, r) >> 33);
}

/* proj/src/graph.cpp:30-35 (range-checked by callers) */
uint32_t dor_to_fixed_point(double w) {
  return (uint32_t)llround(w * (double)FIXED_ONE);
}

/* proj/src/graph.cpp:250-253 */
void dor_weights_const(double p, uint64_t m, uint32_t *w) {
  uint32_t f = dor_to_fixed_point(p);
  for (uint64_t e = 0; e < m; ++e) w[e] = f;
}

/* proj/src/graph.cpp:255-258 (in_degree counted as in graph.cpp:337-341) */
void dor_weights_wc(uint32_t n, uint64_t m, const uint64_t *offsets,
                    const uint32_t *adj, uint32_t *w) {
  uint32_t *indeg = calloc(n ? n : 1, sizeof *indeg);
  (void)offsets;
  for (uint64_t e = 0; e < m; ++e) indeg[adj[e]]++;
  for (uint64_t e = 0; e < m; ++e)
    w[e] = dor_to_fixed_point(1.0 / indeg[adj[e]]);
  free(indeg);
}

/* ---- FASST plan: proj/src/sampling.cpp:7-14 + proj/src/fasst.cpp:21-48 -- */
static const uint32_t *g_sort_vals;
static int cmp_stable(const void *pa, const void *pb) {
  uint32_t a = *(const uint32_t *)pa, b = *(const uint32_t *)pb;
  uint32_t va = g_sort_vals[a], vb = g_sort_vals[b];
  if (va != vb) return va < vb ? -1 : 1;
  return a < b ? -1 : (a > b); /* index tie-break == std::stable_sort */
}

int dor_make_plan(uint32_t r, uint32_t mu, int fasst, uint64_t seed,
                  uint32_t *x_sorted, uint32_t *order, int *degraded) {
  if (r == 0 || mu == 0 || r % mu != 0) return -1;
  uint32_t *x = malloc(sizeof *x * r);
  const uint64_t s = dor_splitmix64_at(seed, 1); /* derive_seed(seed, kSeedTagSamples) */
  for (uint32_t i = 0; i < r; ++i) {
    x[i] = dor_random_value_at(s, i);
    order[i] = i;
  }
  *degraded = 0;
  if (fasst) {
    g_sort_vals = x;
    qsort(order, r, sizeof *order, cmp_stable);
    *degraded = (r / mu) < 32;
  }
  for (uint32_t i = 0; i < r; ++i) x_sorted[i] = x[order[i]];
  free(x);
  return 0;
}

/* proj/src/fasst.cpp:50-88 */
uint64_t dor_device_graph(uint32_t n, const uint64_t *offsets,
                          const uint32_t *adj, const uint32_t *ehash,
                          const uint32_t *w, const uint32_t *xs,
                          uint32_t j_local, uint64_t *d_offsets,
                          uint32_t *d_adj, uint64_t *d_mask) {
  const uint32_t words = (j_local + 63) / 64;
  uint64_t md = 0;
  for (uint32_t u = 0; u < n; ++u) {
    d_offsets[u] = md;
    for (uint64_t e = offsets[u]; e < offsets[u + 1]; ++e) {
      if (w[e] == 0) continue;
      uint64_t *mk = d_mask + md * words;
      int any = 0;
      memset(mk, 0, words * sizeof *mk);
      for (uint32_t j = 0; j < j_local; ++j)
        if ((xs[j] ^ ehash[e]) < w[e]) {
          mk[j >> 6] |= 1ULL << (j & 63);
          any = 1;
        }
      if (!any) continue;
      d_adj[md++] = adj[e];
    }
  }
  d_offsets[n] = md;
  return md;
}

/* proj/src/sketch.cpp:55-66 — register j of u gets
 * clz64(register_hash(splitmix64_at(key, j_offset + j), u)) unless VISITED. */
void dor_fill(uint32_t n, uint32_t j_local, uint32_t j_offset, uint64_t key,
              int8_t *regs) {
  uint64_t *jkey = malloc(sizeof *jkey * j_local);
  for (uint32_t j = 0; j < j_local; ++j)
    jkey[j] = dor_splitmix64_at(key, (uint64_t)j_offset + j);
  for (uint32_t u = 0; u < n; ++u) {
    int8_t *row = regs + (size_t)u * j_local;
    for (uint32_t j = 0; j < j_local; ++j) {
      if (row[j] == VISITED) continue;
      uint64_t h = dor_register_hash(jkey[j], u);
      row[j] = (int8_t)(h ? __builtin_clzll(h) : 64);
    }
  }
  free(jkey);
}

/* proj/src/sketch.cpp:119-131 — sequential, ascending-j double sum. */
double dor_row_score(const int8_t *row, uint32_t j_local) {
  double denom = 0;
  uint32_t live = 0;
  for (uint32_t j = 0; j < j_local; ++j)
    if (row[j] != VISITED) {
      denom += ldexp(1.0, -row[j]);
      ++live;
    }
  if (live == 0) return 0.0;
  return (double)live * live / (denom * PHI);
}

/* proj/src/engine.cpp:9-15, 22-53, 57-96 — Jacobi sweeps over u's out-edges
 * reading the previous-sweep snapshot, edges filtered by changed_prev[v]. */
int dor_simulate(uint32_t n, const uint64_t *d_offsets, const uint32_t *d_adj,
                 const uint64_t *d_mask, uint32_t j_local, int8_t *regs,
                 int cap) {
  const uint32_t words = (j_local + 63) / 64;
  const size_t total = (size_t)n * j_local;
  int8_t *snap = malloc(total ? total : 1);
  uint8_t *chg = malloc(n ? n : 1), *chg_prev = malloc(n ? n : 1);
  memcpy(snap, regs, total);
  memset(chg_prev, 1, n);
  int result = -1;
  for (int it = 1; it <= cap; ++it) {
    memset(chg, 0, n);
    int any = 0;
    for (uint32_t u = 0; u < n; ++u) {
      int8_t *dst = regs + (size_t)u * j_local;
      for (uint64_t e = d_offsets[u]; e < d_offsets[u + 1]; ++e) {
        const uint32_t v = d_adj[e];
        if (!chg_prev[v]) continue;
        const int8_t *src = snap + (size_t)v * j_local;
        const uint64_t *mk = d_mask + e * words;
        for (uint32_t j = 0; j < j_local; ++j) {
          if (!((mk[j >> 6] >> (j & 63)) & 1)) continue;
          if (dst[j] >= 0 && src[j] > dst[j]) {
            dst[j] = src[j];
            chg[u] = 1;
          }
        }
      }
      any |= chg[u];
    }
    for (uint32_t u = 0; u < n; ++u)
      if (chg[u])
        memcpy(snap + (size_t)u * j_local, regs + (size_t)u * j_local, j_local);
    uint8_t *t = chg;
    chg = chg_prev;
    chg_prev = t;
    if (!any) {
      result = it;
      break;
    }
  }
  free(snap);
  free(chg);
  free(chg_prev);
  return result;
}

/* proj/src/sketch.cpp:39-53 */
static uint64_t mark_word(int8_t *regs, uint64_t *vis, uint32_t j_local,
                          uint32_t words, uint32_t u, uint32_t w,
                          uint64_t bits) {
  uint64_t *word = vis + (size_t)u * words + w;
  uint64_t fresh = bits & ~*word;
  if (!fresh) return 0;
  *word |= fresh;
  int8_t *r = regs + (size_t)u * j_local + (size_t)w * 64;
  for (uint64_t b = fresh; b; b &= b - 1) r[__builtin_ctzll(b)] = VISITED;
  return fresh;
}

/* proj/src/engine.cpp:106-144 — commit s, then level-synchronous unified
 * frontier over u's out-edges: cand = fresh_u & mask_e & ~vis_v. */
uint64_t dor_commit_cascade(uint32_t n, const uint64_t *d_offsets,
                            const uint32_t *d_adj, const uint64_t *d_mask,
                            uint32_t j_local, int8_t *regs, uint64_t *vis,
                            uint32_t seed) {
  const uint32_t words = (j_local + 63) / 64;
  uint64_t *fresh = calloc((size_t)n * words + 1, sizeof *fresh);
  uint64_t *fresh_next = calloc((size_t)n * words + 1, sizeof *fresh_next);
  uint32_t *q = malloc(sizeof *q * (n + 1)), *qn = malloc(sizeof *qn * (n + 1));
  uint8_t *inq = calloc(n + 1, 1);
  uint32_t nq = 0, nqn = 0;
  uint64_t marked = 0;
  int any = 0;
  for (uint32_t w = 0; w < words; ++w) {
    uint32_t rem = j_local - w * 64;
    uint64_t tail = rem >= 64 ? ~0ULL : ((1ULL << rem) - 1);
    uint64_t bits = tail & ~vis[(size_t)seed * words + w];
    if (!bits) continue;
    marked += (uint64_t)__builtin_popcountll(
        mark_word(regs, vis, j_local, words, seed, w, bits));
    fresh[(size_t)seed * words + w] |= bits;
    any = 1;
  }
  if (any) q[nq++] = seed;
  while (nq) {
    for (uint32_t i = 0; i < nq; ++i) {
      const uint32_t u = q[i];
      const uint64_t *fu = fresh + (size_t)u * words;
      for (uint64_t e = d_offsets[u]; e < d_offsets[u + 1]; ++e) {
        const uint32_t v = d_adj[e];
        for (uint32_t w = 0; w < words; ++w) {
          uint64_t cand = fu[w] & d_mask[e * words + w] &
                          ~vis[(size_t)v * words + w];
          if (!cand) continue;
          marked += (uint64_t)__builtin_popcountll(
              mark_word(regs, vis, j_local, words, v, w, cand));
          fresh_next[(size_t)v * words + w] |= cand;
          if (!inq[v]) {
            inq[v] = 1;
            qn[nqn++] = v;
          }
        }
      }
    }
    for (uint32_t i = 0; i < nq; ++i)
      memset(fresh + (size_t)q[i] * words, 0, words * sizeof *fresh);
    for (uint32_t i = 0; i < nqn; ++i) inq[qn[i]] = 0;
    uint64_t *tf = fresh;
    fresh = fresh_next;
    fresh_next = tf;
    uint32_t *tq = q;
    q = qn;
    qn = tq;
    nq = nqn;
    nqn = 0;
  }
  free(fresh);
  free(fresh_next);
  free(q);
  free(qn);
  free(inq);
  return marked;
}

/* ---- full run: proj/src/runtime.cpp:37-179 ------------------------------- */
typedef struct {
  uint64_t *off, *mask;
  uint32_t *adj;
  int8_t *regs;
  uint64_t *vis;
  uint64_t visited;
  double *scores;
} rank_t;

static uint32_t ceil_log2(uint32_t mu) {
  uint32_t l = 0;
  for (uint32_t s = 1; s < mu; s <<= 1) ++l;
  return l;
}

int dor_run(uint32_t n, uint64_t m, const uint64_t *offsets,
            const uint32_t *adj, const uint32_t *w, uint32_t k, uint32_t r,
            uint32_t mu, int fasst, double rebuild_eps, uint64_t seed,
            int sim_cap, uint32_t *seeds_dense, double *traj,
            uint32_t *rebuild_rounds, uint32_t *n_rebuilds, int *saturated,
            int *degraded, uint64_t counters[3]) {
  /* runtime.cpp:38-42, sampling.cpp:8, fasst.cpp:23-26 */
  if (k == 0 || k > n || mu == 0 || !(rebuild_eps >= 0.0)) return -1;
  if (r == 0 || r % mu != 0) return -1;
  uint32_t *x = malloc(sizeof *x * r), *order = malloc(sizeof *order * r);
  dor_make_plan(r, mu, fasst, seed, x, order, degraded);
  const uint64_t reg_key = dor_splitmix64_at(seed, 2); /* kSeedTagRegisters */
  const uint32_t J = r / mu, words = (J + 63) / 64;
  uint32_t *ehash = malloc(sizeof *ehash * (m ? m : 1));
  for (uint32_t u = 0; u < n; ++u)
    for (uint64_t e = offsets[u]; e < offsets[u + 1]; ++e)
      ehash[e] = dor_edge_hash(u, adj[e]);
  rank_t *rk = calloc(mu, sizeof *rk);
  int rc = 0;
  for (uint32_t t = 0; t < mu && rc == 0; ++t) {
    rk[t].off = malloc(sizeof(uint64_t) * (n + 1));
    rk[t].adj = malloc(sizeof(uint32_t) * (m ? m : 1));
    rk[t].mask = malloc(sizeof(uint64_t) * (m ? m : 1) * words);
    rk[t].regs = calloc((size_t)n * J + 1, 1);
    rk[t].vis = calloc((size_t)n * words + 1, sizeof(uint64_t));
    rk[t].scores = malloc(sizeof(double) * n);
    if (!rk[t].off || !rk[t].adj || !rk[t].mask || !rk[t].regs ||
        !rk[t].vis || !rk[t].scores) {
      rc = -3;
      break;
    }
    dor_device_graph(n, offsets, adj, ehash, w, x + (size_t)t * J, J,
                     rk[t].off, rk[t].adj, rk[t].mask);
    dor_fill(n, J, t * J, reg_key, rk[t].regs);
    if (dor_simulate(n, rk[t].off, rk[t].adj, rk[t].mask, J, rk[t].regs,
                     sim_cap) < 0)
      rc = -2;
  }
  uint8_t *committed = calloc(n + 1, 1);
  double oldscore = 0.0;
  *n_rebuilds = 0;
  *saturated = 0;
  counters[0] = counters[1] = counters[2] = 0;
  for (uint32_t step = 0; step < k && rc == 0; ++step) {
    for (uint32_t t = 0; t < mu; ++t)
      for (uint32_t v = 0; v < n; ++v)
        rk[t].scores[v] = dor_row_score(rk[t].regs + (size_t)v * J, J);
    /* binomial-tree reduce, collectives.cpp:44-64 */
    for (uint32_t s = 1; s < mu; s <<= 1)
      for (uint32_t t = 0; t + s < mu; t += 2 * s)
        for (uint32_t v = 0; v < n; ++v) rk[t].scores[v] += rk[t + s].scores[v];
    /* root argmax: strict >, best from 0.0, committed skipped (runtime.cpp:95-119) */
    double best = 0.0;
    uint32_t arg = n;
    for (uint32_t v = 0; v < n; ++v) {
      if (committed[v]) continue;
      if (rk[0].scores[v] > best) {
        best = rk[0].scores[v];
        arg = v;
      }
    }
    if (arg == n) {
      *saturated = 1;
      for (uint32_t v = 0; v < n; ++v)
        if (!committed[v]) {
          arg = v;
          break;
        }
    }
    committed[arg] = 1;
    uint64_t covered = 0;
    for (uint32_t t = 0; t < mu; ++t) {
      rk[t].visited += dor_commit_cascade(n, rk[t].off, rk[t].adj, rk[t].mask,
                                          J, rk[t].regs, rk[t].vis, arg);
      covered += rk[t].visited;
    }
    const double score = (double)covered / r;
    seeds_dense[step] = arg;
    traj[step] = score;
    /* counters: collectives.cpp:19,62,76,107 as scheduled per round */
    counters[0] += ((uint64_t)n + 1) * (mu - 1);
    counters[1] += 2ULL * (mu - 1);
    counters[2] += 8 + ceil_log2(mu);
    if (step + 1 < k && (score - oldscore) > rebuild_eps * score) {
      for (uint32_t t = 0; t < mu && rc == 0; ++t) {
        dor_fill(n, J, t * J, reg_key, rk[t].regs);
        if (dor_simulate(n, rk[t].off, rk[t].adj, rk[t].mask, J, rk[t].regs,
                         sim_cap) < 0)
          rc = -2;
      }
      oldscore = score;
      rebuild_rounds[(*n_rebuilds)++] = step;
    }
  }
  for (uint32_t t = 0; t < mu; ++t) {
    free(rk[t].off);
    free(rk[t].adj);
    free(rk[t].mask);
    free(rk[t].regs);
    free(rk[t].vis);
    free(rk[t].scores);
  }
  free(rk);
  free(committed);
  free(ehash);
  free(x);
  free(order);
  return rc;
}

/* ---- FASST analytics (proj/src/fasst.cpp:90-168) -------------------------
 * xs: the plan's slot values (chunk tau = xs[tau*J, (tau+1)*J)); xfill: the
 * X values in fill-rate order (sorted for FASST, generation order for naive).
 * dup_count[mu+1]: edges sampled by exactly k chunks (W = 0 edges count as
 * k = 0, fasst.cpp:107-109); loads[mu]: per-chunk sampled edges
 * (fasst.cpp:128-138); fill: live lanes and counted (edge, 32-lane batch)
 * pairs (fasst.cpp:140-168, R % 32 == 0). */
static int chunk_hits(const uint32_t *xs, uint32_t J, uint32_t h, uint32_t w) {
  for (uint32_t j = 0; j < J; ++j) /* fasst.cpp:93-97 */
    if ((xs[j] ^ h) < w) return 1;
  return 0;
}

void dor_fasst_stats(uint64_t m, const uint32_t *ehash, const uint32_t *w,
                     const uint32_t *xs, const uint32_t *xfill, uint32_t r,
                     uint32_t mu, uint64_t *dup_count, uint64_t *loads,
                     uint64_t *live_lanes, uint64_t *batches) {
  const uint32_t J = r / mu;
  memset(dup_count, 0, (mu + 1) * sizeof *dup_count);
  memset(loads, 0, mu * sizeof *loads);
  *live_lanes = 0;
  *batches = 0;
  for (uint64_t e = 0; e < m; ++e) {
    uint32_t k = 0;
    if (w[e] != 0)
      for (uint32_t t = 0; t < mu; ++t) {
        const int hit = chunk_hits(xs + (uint64_t)t * J, J, ehash[e], w[e]);
        k += hit;
        loads[t] += hit;
      }
    dup_count[k]++;
    if (w[e] == 0 || r % 32 != 0) continue;
    for (uint32_t b = 0; b < r / 32; ++b) { /* fasst.cpp:154-163 */
      uint32_t c = 0;
      for (uint32_t t = 0; t < 32; ++t) c += (xfill[b * 32 + t] ^ ehash[e]) < w[e];
      if (c) {
        *live_lanes += c;
        ++*batches;
      }
    }
  }
}
