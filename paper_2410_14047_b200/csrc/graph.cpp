// graph.cpp — host graph substrate (ingestion is not the hot path, but the
// format must be bit-identical to the reference's: proj/src/graph.cpp).
#include "graph.h"

#include <omp.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <parallel/algorithm>
#include <random>
#include <sstream>
#include <thread>

#include "dfs.h"
#include "hash.cuh"

namespace dfs {

namespace {

constexpr char kCacheMagic[8] = {'D', 'F', 'S', 'G', '0', '0', '0', '1'};

[[noreturn]] void parse_fail(size_t line, const std::string& why) {
  throw Error(kRuntime, "edge list parse error at line " + std::to_string(line) + ": " + why);
}

const char* skip_ws(const char* p, const char* end) {
  while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
  return p;
}

struct RawEdge {
  uint64_t u, v;
  double w;  // < 0: no explicit probability
};

int hw_threads() {
  unsigned t = std::thread::hardware_concurrency();
  return t ? int(std::min(t, 64u)) : 1;
}

}  // namespace

uint32_t to_fixed_point(double w) {
  if (!(w >= 0.0 && w <= 1.0))
    throw Error(kInvalid, "probability out of [0, 1]: " + std::to_string(w));
  return static_cast<uint32_t>(std::llround(w * static_cast<double>(kFixedOne)));
}

// Text format of proj/src/graph.cpp:41-75: "u v [p]" lines, '#' comments.
static std::vector<RawEdge> parse_edges(std::string_view text, bool directed) {
  std::vector<RawEdge> out;
  const char* p = text.data();
  const char* end = p + text.size();
  size_t line = 0;
  while (p < end) {
    ++line;
    const char* eol = static_cast<const char*>(memchr(p, '\n', size_t(end - p)));
    const char* stop = eol ? eol : end;
    const char* q = skip_ws(p, stop);
    p = eol ? eol + 1 : end;
    if (q == stop || *q == '#') continue;
    RawEdge e{0, 0, -1.0};
    auto [pu, ecu] = std::from_chars(q, stop, e.u);
    if (ecu != std::errc{}) parse_fail(line, "expected source id");
    q = skip_ws(pu, stop);
    auto [pv, ecv] = std::from_chars(q, stop, e.v);
    if (ecv != std::errc{}) parse_fail(line, "expected target id");
    q = skip_ws(pv, stop);
    if (q != stop) {
      auto [pw, ecw] = std::from_chars(q, stop, e.w);
      if (ecw != std::errc{}) parse_fail(line, "expected edge probability");
      if (!(e.w >= 0.0 && e.w <= 1.0)) parse_fail(line, "probability out of [0, 1]");
      q = skip_ws(pw, stop);
      if (q != stop) parse_fail(line, "trailing tokens");
    }
    out.push_back(e);
    if (!directed && e.u != e.v) out.push_back({e.v, e.u, e.w});
  }
  if (out.empty()) throw Error(kRuntime, "edge list is empty");
  return out;
}

void ensure_graph_fields(const HostGraph& g) {
  if (g.ehash.size() == g.m && g.in_degree.size() == g.n) return;
  g.ehash.resize(g.m);
  g.in_degree.assign(g.n, 0);
  const int T = hw_threads();
  // ehash in parallel over rows; in_degree serially (cheap).
#pragma omp parallel for schedule(dynamic, 4096) num_threads(T)
  for (int64_t u = 0; u < int64_t(g.n); ++u)
    for (uint64_t e = g.offsets[u]; e < g.offsets[u + 1]; ++e)
      g.ehash[e] = edge_hash(uint64_t(u), g.adj[e]);
  for (uint64_t e = 0; e < g.m; ++e) g.in_degree[g.adj[e]]++;
}

// proj/src/graph.cpp:128-183: dense relabel by sorted unique ids, (u, v) sort,
// duplicate collapse (compound probability 1 - prod(1 - w) when weighted).
static HostGraph build_graph(std::vector<RawEdge>& raw) {
  if (raw.empty()) throw Error(kRuntime, "graph has no edges");
  std::vector<uint64_t> ids;
  ids.reserve(raw.size() * 2);
  for (const RawEdge& e : raw) {
    ids.push_back(e.u);
    ids.push_back(e.v);
  }
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  auto dense = [&](uint64_t id) {
    return uint32_t(std::lower_bound(ids.begin(), ids.end(), id) - ids.begin());
  };
  struct DEdge {
    uint32_t u, v;
    double w;
  };
  std::vector<DEdge> es;
  es.reserve(raw.size());
  for (const RawEdge& e : raw) es.push_back({dense(e.u), dense(e.v), e.w});
  // std::sort (not stable) as the reference: duplicate order feeds the compound product.
  std::sort(es.begin(), es.end(), [](const DEdge& a, const DEdge& b) {
    return a.u != b.u ? a.u < b.u : a.v < b.v;
  });
  HostGraph g;
  g.n = uint32_t(ids.size());
  g.orig_id = std::move(ids);
  g.offsets.assign(size_t(g.n) + 1, 0);
  std::vector<DEdge> merged;
  merged.reserve(es.size());
  size_t i = 0;
  while (i < es.size()) {
    size_t j = i;
    const bool weighted = es[i].w >= 0.0;
    double keep = 1.0;
    while (j < es.size() && es[j].u == es[i].u && es[j].v == es[i].v) {
      if ((es[j].w >= 0.0) != weighted)
        throw Error(kRuntime, "parallel edges mix explicit and implicit probabilities");
      if (weighted) keep *= 1.0 - es[j].w;
      ++j;
    }
    merged.push_back({es[i].u, es[i].v, weighted ? 1.0 - keep : -1.0});
    g.offsets[size_t(es[i].u) + 1]++;
    i = j;
  }
  for (uint32_t u = 0; u < g.n; ++u) g.offsets[size_t(u) + 1] += g.offsets[u];
  g.m = merged.size();
  g.adj.resize(g.m);
  g.weights.resize(g.m);
  for (uint64_t k = 0; k < g.m; ++k) {
    g.adj[k] = merged[k].v;
    g.weights[k] = merged[k].w >= 0.0 ? to_fixed_point(merged[k].w) : 0;
  }
  return g;
}

HostGraph graph_from_text(std::string_view text, bool directed) {
  std::vector<RawEdge> raw = parse_edges(text, directed);
  return build_graph(raw);
}

HostGraph graph_from_csr(uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* adj,
                         const uint64_t* orig_ids) {
  HostGraph g;
  g.n = n;
  g.m = m;
  g.offsets.assign(offsets, offsets + size_t(n) + 1);
  if (g.offsets[0] != 0 || g.offsets[n] != m)
    throw Error(kInvalid, "graph_from_csr: offsets must start at 0 and end at m");
  for (uint32_t u = 0; u < n; ++u)
    if (g.offsets[u + 1] < g.offsets[u]) throw Error(kInvalid, "graph_from_csr: offsets decrease");
  g.adj.assign(adj, adj + m);
  for (uint64_t e = 0; e < m; ++e)
    if (g.adj[e] >= n) throw Error(kInvalid, "graph_from_csr: target id out of range");
  g.weights.assign(m, 0);
  if (orig_ids) {
    g.orig_id.assign(orig_ids, orig_ids + n);
  } else {
    g.orig_id.resize(n);
    for (uint32_t u = 0; u < n; ++u) g.orig_id[u] = u;
  }
  return g;
}

// proj/src/graph.cpp:185-226
WeightSetting WeightSetting::parse(std::string_view spec) {
  auto bad = [&]() { return Error(kRuntime, "bad weight setting: " + std::string(spec)); };
  auto num = [&](std::string_view s) {
    double v = 0;
    auto [p, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
    if (ec != std::errc{} || p != s.data() + s.size()) throw bad();
    return v;
  };
  WeightSetting w;
  if (spec == "wc") {
    w.kind = WeightKind::WeightedCascade;
    return w;
  }
  const size_t colon = spec.find(':');
  if (colon == std::string_view::npos) throw bad();
  const std::string_view head = spec.substr(0, colon), args = spec.substr(colon + 1);
  const size_t comma = args.find(',');
  if (head == "const") {
    if (comma != std::string_view::npos) throw bad();
    w.kind = WeightKind::Constant;
    w.a = num(args);
    if (!(w.a >= 0.0 && w.a <= 1.0)) throw bad();
    return w;
  }
  if (comma == std::string_view::npos) throw bad();
  w.a = num(args.substr(0, comma));
  w.b = num(args.substr(comma + 1));
  if (head == "normal") {
    w.kind = WeightKind::Normal;
    if (w.b < 0.0) throw bad();
    return w;
  }
  if (head == "uniform") {
    w.kind = WeightKind::Uniform;
    if (w.a > w.b) throw bad();
    return w;
  }
  throw bad();
}

std::string WeightSetting::to_string() const {
  std::ostringstream ss;  // default stream formatting, as the reference
  switch (kind) {
    case WeightKind::Constant: ss << "const:" << a; break;
    case WeightKind::WeightedCascade: ss << "wc"; break;
    case WeightKind::Normal: ss << "normal:" << a << "," << b; break;
    case WeightKind::Uniform: ss << "uniform:" << a << "," << b; break;
  }
  return ss.str();
}

void assign_weights(const HostGraph& g, const WeightSetting& s, uint64_t seed,
                    std::vector<uint32_t>& w) {
  auto clamp01 = [](double x) { return std::min(1.0, std::max(0.0, x)); };
  w.resize(g.m);
  switch (s.kind) {
    case WeightKind::Constant: std::fill(w.begin(), w.end(), to_fixed_point(s.a)); break;
    case WeightKind::WeightedCascade:
      ensure_graph_fields(g);
      for (uint64_t e = 0; e < g.m; ++e) w[e] = to_fixed_point(1.0 / g.in_degree[g.adj[e]]);
      break;
    case WeightKind::Normal: {
      std::mt19937_64 rng(seed);
      std::normal_distribution<double> d(s.a, s.b);
      for (uint64_t e = 0; e < g.m; ++e) w[e] = to_fixed_point(clamp01(d(rng)));
      break;
    }
    case WeightKind::Uniform: {
      std::mt19937_64 rng(seed);
      std::uniform_real_distribution<double> d(s.a, s.b);
      for (uint64_t e = 0; e < g.m; ++e) w[e] = to_fixed_point(clamp01(d(rng)));
      break;
    }
  }
}

// ---------------------------------------------------------------- cache
// DFSG0001 layout (proj/src/graph.cpp:293-305): magic, n, m (u64), offsets
// u64[n+1], adj u32[m], weights u32[m], orig_id u64[n]; ehash/in_degree are
// recomputed on load (:337-341).
void save_graph_cache(const HostGraph& g, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw Error(kRuntime, "cannot write " + path);
  out.write(kCacheMagic, sizeof kCacheMagic);
  uint64_t n = g.n, m = g.m;
  out.write(reinterpret_cast<const char*>(&n), 8);
  out.write(reinterpret_cast<const char*>(&m), 8);
  out.write(reinterpret_cast<const char*>(g.offsets.data()), std::streamsize(g.offsets.size() * 8));
  out.write(reinterpret_cast<const char*>(g.adj.data()), std::streamsize(g.adj.size() * 4));
  std::vector<uint32_t> wz;
  const std::vector<uint32_t>* wp = &g.weights;
  if (g.weights.size() != g.m) {
    wz.assign(g.m, 0);
    wp = &wz;
  }
  out.write(reinterpret_cast<const char*>(wp->data()), std::streamsize(g.m * 4));
  out.write(reinterpret_cast<const char*>(g.orig_id.data()), std::streamsize(g.orig_id.size() * 8));
  if (!out) throw Error(kRuntime, "write failed: " + path);
}

static bool is_graph_cache(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  char magic[8] = {};
  in.read(magic, 8);
  return in && memcmp(magic, kCacheMagic, 8) == 0;
}

static HostGraph load_graph_cache(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(kRuntime, "cannot open " + path);
  char magic[8] = {};
  in.read(magic, 8);
  if (!in || memcmp(magic, kCacheMagic, 8) != 0) throw Error(kRuntime, "not a graph cache: " + path);
  uint64_t n = 0, m = 0;
  in.read(reinterpret_cast<char*>(&n), 8);
  in.read(reinterpret_cast<char*>(&m), 8);
  HostGraph g;
  g.n = uint32_t(n);
  g.m = m;
  g.offsets.resize(n + 1);
  g.adj.resize(m);
  g.weights.resize(m);
  g.orig_id.resize(n);
  in.read(reinterpret_cast<char*>(g.offsets.data()), std::streamsize((n + 1) * 8));
  in.read(reinterpret_cast<char*>(g.adj.data()), std::streamsize(m * 4));
  in.read(reinterpret_cast<char*>(g.weights.data()), std::streamsize(m * 4));
  in.read(reinterpret_cast<char*>(g.orig_id.data()), std::streamsize(n * 8));
  if (!in) throw Error(kRuntime, "truncated graph cache: " + path);
  if (g.offsets.back() != m) throw Error(kRuntime, "corrupt graph cache: " + path);
  return g;
}

HostGraph load_graph(const std::string& path, bool directed) {
  if (is_graph_cache(path)) return load_graph_cache(path);
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(kRuntime, "cannot open " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return graph_from_text(ss.str(), directed);
}

// ---------------------------------------------------------------- generators
// Candidate stream: candidate c is a pure function of (seed, c) via the
// counter-form splitmix64, so the selected edge set — the first m distinct
// (u, v) pairs in candidate order — does not depend on thread count or on how
// many candidates were drawn.
namespace {

inline uint64_t rmat_key(uint64_t seed, uint32_t scale, uint64_t c) {
  uint64_t u = 0, v = 0;
  for (uint32_t b = 0; b < scale; ++b) {
    const double p = double(splitmix64_at(seed, c * scale + b) >> 11) * 0x1.0p-53;
    u = (u << 1) | (p >= 0.76);  // quadrants a=.57 b=.19 c=.19 d=.05 (tests/testutil.hpp:67-86)
    v = (v << 1) | ((p >= 0.57 && p < 0.76) || p >= 0.95);
  }
  return (u << 32) | v;
}

inline uint64_t er_key(uint64_t seed, uint32_t n, uint64_t c) {
  const uint64_t u = uint64_t((unsigned __int128)splitmix64_at(seed, 2 * c) * n >> 64);
  const uint64_t v = uint64_t((unsigned __int128)splitmix64_at(seed, 2 * c + 1) * n >> 64);
  return (u << 32) | v;
}

template <class KeyFn>
HostGraph generate(uint64_t m, uint64_t id_space, KeyFn key) {
  if (m == 0) throw Error(kInvalid, "generator: m must be >= 1");
  const int T = hw_threads();
  uint64_t N = m + m / 4 + 1024;
  std::vector<uint64_t> keys;
  for (;;) {
    struct KC {
      uint64_t key, c;
    };
    std::vector<KC> kc(N);
#pragma omp parallel for schedule(static) num_threads(T)
    for (int64_t c = 0; c < int64_t(N); ++c) kc[c] = {key(uint64_t(c)), uint64_t(c)};
    // drop self-loops
    kc.erase(std::remove_if(kc.begin(), kc.end(),
                            [](const KC& x) { return (x.key >> 32) == (x.key & 0xFFFFFFFFu); }),
             kc.end());
    __gnu_parallel::sort(kc.begin(), kc.end(), [](const KC& a, const KC& b) {
      return a.key != b.key ? a.key < b.key : a.c < b.c;
    });
    size_t w = 0;  // keep the first occurrence of each key
    for (size_t i = 0; i < kc.size(); ++i)
      if (w == 0 || kc[w - 1].key != kc[i].key) kc[w++] = kc[i];
    kc.resize(w);
    if (w >= m) {
      std::nth_element(kc.begin(), kc.begin() + (m - 1), kc.end(),
                       [](const KC& a, const KC& b) { return a.c < b.c; });
      kc.resize(m);
      keys.resize(m);
      for (uint64_t i = 0; i < m; ++i) keys[i] = kc[i].key;
      break;
    }
    if (N > (uint64_t(1) << 40)) throw Error(kInvalid, "generator: m exceeds the id space");
    N = N + N / 2;
  }
  __gnu_parallel::sort(keys.begin(), keys.end());
  // dense relabel over the ids that occur (graph.cpp:131-142)
  std::vector<uint32_t> dense(id_space + 1, 0);
  for (uint64_t k : keys) {
    dense[k >> 32] = 1;
    dense[k & 0xFFFFFFFFu] = 1;
  }
  HostGraph g;
  uint32_t next = 0;
  for (uint64_t id = 0; id < id_space; ++id)
    if (dense[id]) {
      dense[id] = next++;
      g.orig_id.push_back(id);
    }
  g.n = next;
  g.m = m;
  g.offsets.assign(size_t(g.n) + 1, 0);
  g.adj.resize(m);
  for (uint64_t i = 0; i < m; ++i) {
    const uint32_t u = dense[keys[i] >> 32], v = dense[keys[i] & 0xFFFFFFFFu];
    g.offsets[size_t(u) + 1]++;
    g.adj[i] = v;
  }
  for (uint32_t u = 0; u < g.n; ++u) g.offsets[size_t(u) + 1] += g.offsets[u];
  g.weights.assign(m, 0);
  return g;
}

}  // namespace

HostGraph generate_rmat(uint32_t scale, uint64_t m, uint64_t seed) {
  if (scale < 1 || scale > 31) throw Error(kInvalid, "rmat: scale must be in [1, 31]");
  return generate(m, uint64_t(1) << scale, [=](uint64_t c) { return rmat_key(seed, scale, c); });
}

HostGraph generate_er(uint32_t n, uint64_t m, uint64_t seed) {
  if (n < 2) throw Error(kInvalid, "er: n must be >= 2");
  return generate(m, n, [=](uint64_t c) { return er_key(seed, n, c); });
}

// ---------------------------------------------------------------- oracle (host)
// proj/src/oracle.cpp:14-79 semantics: liveness of edge e in trial t is
// (mt19937_64(trial_seed)() >> 33) < W[e] drawn in edge order; BFS from seeds.
void influence_stats(const HostGraph& g, const std::vector<uint32_t>& w,
                     const std::vector<uint32_t>& seeds, uint32_t trials, uint64_t seed,
                     uint32_t runs, double* mean, double* std_error) {
  if (trials == 0 || runs == 0) throw Error(kInvalid, "oracle: trials and runs must be >= 1");
  for (uint32_t s : seeds)
    if (s >= g.n) throw Error(kInvalid, "oracle: seed id out of range");
  const uint64_t base = derive_seed(seed, kSeedTagOracle);
  std::vector<uint8_t> live(g.m);
  std::vector<uint32_t> mark(g.n, 0), queue;
  uint32_t epoch = 0;
  double sum = 0, sumsq = 0;
  for (uint32_t run = 0; run < runs; ++run)
    for (uint32_t t = 0; t < trials; ++t) {
      std::mt19937_64 rng(splitmix64_at(splitmix64_at(base, run), t));
      for (uint64_t e = 0; e < g.m; ++e) live[e] = uint32_t(rng() >> 33) < w[e];
      ++epoch;
      queue.clear();
      for (uint32_t s : seeds)
        if (mark[s] != epoch) {
          mark[s] = epoch;
          queue.push_back(s);
        }
      for (size_t h = 0; h < queue.size(); ++h) {
        const uint32_t u = queue[h];
        for (uint64_t e = g.offsets[u]; e < g.offsets[u + 1]; ++e) {
          const uint32_t v = g.adj[e];
          if (live[e] && mark[v] != epoch) {
            mark[v] = epoch;
            queue.push_back(v);
          }
        }
      }
      const double reached = double(queue.size());
      sum += reached;
      sumsq += reached * reached;
    }
  const double T = double(trials) * runs;
  *mean = sum / T;
  *std_error = 0.0;
  if (T > 1) {
    const double var = (sumsq - sum * sum / T) / (T - 1);
    *std_error = std::sqrt(std::max(0.0, var) / T);
  }
}

// Tarjan SCC over a live CSR (iterative, roots in id order, edges in CSR
// order); components numbered in pop order, i.e. reverse topological.
namespace {
struct Tarjan {
  std::vector<int32_t> idx, low, comp;
  std::vector<uint32_t> stk;
  std::vector<uint8_t> on;
  struct Frame {
    uint32_t v;
    uint64_t e;
  };
  std::vector<Frame> call;
  int32_t run(uint32_t n, const std::vector<uint64_t>& off, const std::vector<uint32_t>& tg) {
    idx.assign(n, -1);
    low.assign(n, 0);
    comp.assign(n, -1);
    on.assign(n, 0);
    stk.clear();
    call.clear();
    int32_t counter = 0, ncomp = 0;
    for (uint32_t root = 0; root < n; ++root) {
      if (idx[root] != -1) continue;
      idx[root] = low[root] = counter++;
      stk.push_back(root);
      on[root] = 1;
      call.push_back({root, off[root]});
      while (!call.empty()) {
        const uint32_t v = call.back().v;
        if (call.back().e < off[v + 1]) {
          const uint32_t w = tg[call.back().e++];
          if (idx[w] == -1) {
            idx[w] = low[w] = counter++;
            stk.push_back(w);
            on[w] = 1;
            call.push_back({w, off[w]});
          } else if (on[w]) {
            low[v] = std::min(low[v], idx[w]);
          }
          continue;
        }
        if (low[v] == idx[v]) {
          uint32_t w;
          do {
            w = stk.back();
            stk.pop_back();
            on[w] = 0;
            comp[w] = ncomp;
          } while (w != v);
          ++ncomp;
        }
        call.pop_back();
        if (!call.empty()) low[call.back().v] = std::min(low[call.back().v], low[v]);
      }
    }
    return ncomp;
  }
};
}  // namespace

// proj/src/oracle.cpp:152-250 semantics, including its component-bitset
// closure that ORs target rows in vertex order over the live edges (the gains
// it yields are what the reference reports, so they are reproduced as is).
std::vector<uint32_t> greedy_exact(const HostGraph& g, const std::vector<uint32_t>& w, uint32_t k,
                                   uint32_t trials, uint64_t seed) {
  if (k == 0 || k > g.n) throw Error(kInvalid, "greedy_exact: k must be in [1, n]");
  if (trials == 0) throw Error(kInvalid, "greedy_exact: trials must be >= 1");
  const uint64_t base = derive_seed(seed, kSeedTagOracle);
  std::vector<uint32_t> committed;
  std::vector<uint64_t> gains(g.n), loff(size_t(g.n) + 1), reach, covered, comp_gain;
  std::vector<uint32_t> ltg, comp_size;
  std::vector<uint8_t> live(g.m);
  Tarjan scc;
  for (uint32_t step = 0; step < k; ++step) {
    std::fill(gains.begin(), gains.end(), 0);
    for (uint32_t t = 0; t < trials; ++t) {
      std::mt19937_64 rng(splitmix64_at(splitmix64_at(base, 1000 + step), t));
      for (uint64_t e = 0; e < g.m; ++e) live[e] = uint32_t(rng() >> 33) < w[e];
      std::fill(loff.begin(), loff.end(), 0);
      ltg.clear();
      for (uint32_t u = 0; u < g.n; ++u) {
        for (uint64_t e = g.offsets[u]; e < g.offsets[u + 1]; ++e)
          if (live[e]) ltg.push_back(g.adj[e]);
        loff[size_t(u) + 1] = ltg.size();
      }
      const int32_t nc = scc.run(g.n, loff, ltg);
      const uint32_t words = uint32_t((nc + 63) / 64);
      comp_size.assign(nc, 0);
      for (uint32_t v = 0; v < g.n; ++v) comp_size[scc.comp[v]]++;
      reach.assign(size_t(nc) * words, 0);
      for (int32_t c = 0; c < nc; ++c) reach[size_t(c) * words + (c >> 6)] |= 1ull << (c & 63);
      for (uint32_t u = 0; u < g.n; ++u) {
        const int32_t cu = scc.comp[u];
        for (uint64_t e = loff[u]; e < loff[size_t(u) + 1]; ++e) {
          const int32_t cv = scc.comp[ltg[e]];
          if (cv == cu) continue;
          for (uint32_t x = 0; x < words; ++x)
            reach[size_t(cu) * words + x] |= reach[size_t(cv) * words + x];
        }
      }
      covered.assign(words, 0);
      for (uint32_t s : committed)
        for (uint32_t x = 0; x < words; ++x) covered[x] |= reach[size_t(scc.comp[s]) * words + x];
      comp_gain.assign(nc, 0);
      for (int32_t c = 0; c < nc; ++c) {
        uint64_t gain = 0;
        for (uint32_t x = 0; x < words; ++x)
          for (uint64_t bits = reach[size_t(c) * words + x] & ~covered[x]; bits; bits &= bits - 1)
            gain += comp_size[x * 64 + __builtin_ctzll(bits)];
        comp_gain[c] = gain;
      }
      for (uint32_t v = 0; v < g.n; ++v) gains[v] += comp_gain[scc.comp[v]];
    }
    uint32_t best = 0;
    uint64_t best_gain = 0;
    bool found = false;
    for (uint32_t v = 0; v < g.n; ++v) {
      if (std::find(committed.begin(), committed.end(), v) != committed.end()) continue;
      if (!found || gains[v] > best_gain) {
        found = true;
        best = v;
        best_gain = gains[v];
      }
    }
    committed.push_back(best);
  }
  return committed;
}

}  // namespace dfs
