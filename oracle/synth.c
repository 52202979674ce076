/*
 * synth.c — TEST INFRASTRUCTURE ONLY: synthetic input graphs for the checker.
 *
 * The bench's reference arm (bench.py --impl reference) and the large parity
 * tests must hand the UNMODIFIED reference (oracle/_ref) exactly the graph the
 * product benchmarks, without loading the product library.  This file writes
 * that graph as a DFSG0001 cache (layout of proj/src/graph.cpp:293-305, the
 * format the reference's load_graph reads) from the same deterministic
 * candidate stream the product generator uses:
 *
 *   candidate c = a pure function of (seed, c) via the counter-form splitmix64
 *                 (proj/include/difuser/hash.hpp:22-30);
 *   R-MAT      : `scale` quadrant draws with (a,b,c,d) = (.57,.19,.19,.05)
 *                 (proj/tests/testutil.hpp:67-86);
 *   ER         : u, v = multiply-shift of two draws into [0, n);
 *   edge set   : self-loops dropped, the first m distinct (u, v) in candidate
 *                 order; then the reference's dense relabel by sorted ids
 *                 (proj/src/graph.cpp:131-142) and (u, v)-sorted CSR.
 *
 * tests/test_host.py checks that this file's caches are byte-identical to the
 * product's save_cache(generate(...)) output.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "difuser_oracle.h"

typedef struct {
  uint64_t key, c;
} kc_t;

static uint64_t rmat_key(uint64_t seed, uint32_t scale, uint64_t c) {
  uint64_t u = 0, v = 0;
  for (uint32_t b = 0; b < scale; ++b) {
    const double p = (double)(dor_splitmix64_at(seed, c * scale + b) >> 11) * 0x1.0p-53;
    u = (u << 1) | (uint64_t)(p >= 0.76);
    v = (v << 1) | (uint64_t)((p >= 0.57 && p < 0.76) || p >= 0.95);
  }
  return (u << 32) | v;
}

static uint64_t er_key(uint64_t seed, uint32_t n, uint64_t c) {
  const uint64_t u = (uint64_t)(((unsigned __int128)dor_splitmix64_at(seed, 2 * c) * n) >> 64);
  const uint64_t v = (uint64_t)(((unsigned __int128)dor_splitmix64_at(seed, 2 * c + 1) * n) >> 64);
  return (u << 32) | v;
}

/* Stable LSD radix sort of kc by key over 16-bit digits of the live key bits. */
static int radix_kc(kc_t *a, size_t n, uint64_t maxkey) {
  kc_t *tmp = (kc_t *)malloc(n * sizeof(kc_t) + 1);
  size_t *cnt = (size_t *)malloc(65536 * sizeof(size_t));
  if (!tmp || !cnt) {
    free(tmp);
    free(cnt);
    return -1;
  }
  kc_t *src = a, *dst = tmp;
  for (int sh = 0; sh < 64 && (maxkey >> sh); sh += 16) {
    memset(cnt, 0, 65536 * sizeof(size_t));
    for (size_t i = 0; i < n; ++i) cnt[(src[i].key >> sh) & 0xFFFF]++;
    size_t run = 0;
    for (int d = 0; d < 65536; ++d) {
      const size_t t = cnt[d];
      cnt[d] = run;
      run += t;
    }
    for (size_t i = 0; i < n; ++i) dst[cnt[(src[i].key >> sh) & 0xFFFF]++] = src[i];
    kc_t *t = src;
    src = dst;
    dst = t;
  }
  if (src != a) memcpy(a, src, n * sizeof(kc_t));
  free(tmp);
  free(cnt);
  return 0;
}

/* Writes the cache; returns 0, -1 bad argument, -2 out of memory, -3 I/O. */
int dor_generate_cache(int kind, uint64_t a, uint64_t m, uint64_t seed, const char *path,
                       uint32_t *n_out) {
  if (m == 0 || (kind == 0 && (a < 1 || a > 31)) || (kind == 1 && a < 2) || kind < 0 || kind > 1)
    return -1;
  const uint64_t id_space = kind == 0 ? (1ull << a) : a;
  uint64_t N = m + m / 4 + 1024;
  uint64_t *keys = NULL;
  for (;;) {
    kc_t *kc = (kc_t *)malloc(N * sizeof(kc_t) + 1);
    if (!kc) return -2;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < (int64_t)N; ++c) {
      kc[c].key = kind == 0 ? rmat_key(seed, (uint32_t)a, (uint64_t)c)
                            : er_key(seed, (uint32_t)a, (uint64_t)c);
      kc[c].c = (uint64_t)c;
    }
    size_t w = 0, maxkey = 0;
    for (uint64_t i = 0; i < N; ++i)  /* drop self-loops, keep candidate order */
      if ((kc[i].key >> 32) != (kc[i].key & 0xFFFFFFFFu)) {
        kc[w++] = kc[i];
        if (kc[i].key > maxkey) maxkey = kc[i].key;
      }
    if (radix_kc(kc, w, maxkey)) {
      free(kc);
      return -2;
    }
    size_t u = 0;  /* first occurrence (smallest c) of each key */
    for (size_t i = 0; i < w; ++i)
      if (u == 0 || kc[u - 1].key != kc[i].key) kc[u++] = kc[i];
    if (u >= m) {
      /* the m distinct keys with the smallest candidate index */
      uint8_t *take = (uint8_t *)calloc(N, 1);
      uint64_t *keyat = (uint64_t *)malloc(N * sizeof(uint64_t) + 1);
      keys = (uint64_t *)malloc(m * sizeof(uint64_t) + 1);
      if (!take || !keyat || !keys) {
        free(take), free(keyat), free(keys), free(kc);
        return -2;
      }
      for (size_t i = 0; i < u; ++i) {
        take[kc[i].c] = 1;
        keyat[kc[i].c] = kc[i].key;
      }
      uint64_t got = 0;
      for (uint64_t c = 0; c < N && got < m; ++c)
        if (take[c]) keys[got++] = keyat[c];
      free(take);
      free(keyat);
      /* keys ascending (u, v): reuse the kc sort on a fresh buffer */
      for (uint64_t i = 0; i < m; ++i) {
        kc[i].key = keys[i];
        kc[i].c = i;
      }
      if (radix_kc(kc, m, maxkey)) {
        free(kc), free(keys);
        return -2;
      }
      for (uint64_t i = 0; i < m; ++i) keys[i] = kc[i].key;
      free(kc);
      break;
    }
    free(kc);
    if (N > (1ull << 40)) return -1;
    N = N + N / 2;
  }
  /* dense relabel over the ids that occur (proj/src/graph.cpp:131-142) */
  uint32_t *dense = (uint32_t *)calloc(id_space + 1, sizeof(uint32_t));
  if (!dense) {
    free(keys);
    return -2;
  }
  for (uint64_t i = 0; i < m; ++i) {
    dense[keys[i] >> 32] = 1;
    dense[keys[i] & 0xFFFFFFFFu] = 1;
  }
  uint64_t n = 0;
  for (uint64_t id = 0; id < id_space; ++id)
    if (dense[id]) ++n;
  uint64_t *orig = (uint64_t *)malloc(n * sizeof(uint64_t) + 1);
  uint64_t *off = (uint64_t *)calloc(n + 1, sizeof(uint64_t));
  uint32_t *adj = (uint32_t *)malloc(m * sizeof(uint32_t) + 1);
  if (!orig || !off || !adj) {
    free(dense), free(keys), free(orig), free(off), free(adj);
    return -2;
  }
  uint32_t next = 0;
  for (uint64_t id = 0; id < id_space; ++id)
    if (dense[id]) {
      orig[next] = id;
      dense[id] = next++;
    }
  for (uint64_t i = 0; i < m; ++i) {
    off[dense[keys[i] >> 32] + 1]++;
    adj[i] = dense[keys[i] & 0xFFFFFFFFu];
  }
  for (uint64_t v = 0; v < n; ++v) off[v + 1] += off[v];
  int rc = 0;
  FILE *f = fopen(path, "wb");
  if (!f) {
    rc = -3;
  } else {
    static const char magic[8] = {'D', 'F', 'S', 'G', '0', '0', '0', '1'};
    uint32_t zero[4096];
    memset(zero, 0, sizeof zero);
    int ok = fwrite(magic, 1, 8, f) == 8 && fwrite(&n, 8, 1, f) == 1 && fwrite(&m, 8, 1, f) == 1 &&
             fwrite(off, 8, n + 1, f) == n + 1 && fwrite(adj, 4, m, f) == m;
    for (uint64_t i = 0; ok && i < m; i += 4096) {  /* weights u32[m]: zero (apply_weights later) */
      const size_t c = (size_t)(m - i < 4096 ? m - i : 4096);
      ok = fwrite(zero, 4, c, f) == c;
    }
    ok = ok && fwrite(orig, 8, n, f) == n;
    if (fclose(f) != 0 || !ok) rc = -3;
  }
  if (n_out) *n_out = (uint32_t)n;
  free(dense), free(keys), free(orig), free(off), free(adj);
  return rc;
}
