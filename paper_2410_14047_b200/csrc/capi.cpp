// capi.cpp — extern "C" boundary (include/difuser_b200.h).  Every entry point
// converts exceptions into status codes + a thread-local message.
#include "difuser_b200.h"

#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "graph.h"
#include "hash.cuh"
#include "runtime.h"

struct dfs_graph {
  dfs::HostGraph g;
  bool pinned = false;
  ~dfs_graph() {
    if (pinned) {
      cudaHostUnregister(g.offsets.data());
      if (g.m) cudaHostUnregister(g.adj.data());
    }
  }
};
struct dfs_ctx {
  std::unique_ptr<dfs::Context> c;
  dfs::Report last;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return DFS_OK;
  } catch (const dfs::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return DFS_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DFS_ERUNTIME;
  } catch (...) {
    g_err = "unknown error";
    return DFS_ERUNTIME;
  }
}

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

void need(const void* p, const char* what) {
  if (!p) throw dfs::Error(dfs::kInvalid, std::string("null argument: ") + what);
}

// make_config of proj/bindings/pymodule.cpp:16-28
dfs::RunConfig to_config(const dfs_config* c) {
  need(c, "config");
  dfs::RunConfig r;
  r.k = c->k;
  r.r = c->r;
  r.mu = c->devices;
  const std::string mode = c->mode ? c->mode : "fasst";
  if (mode == "fasst") r.fasst = true;
  else if (mode == "naive") r.fasst = false;
  else throw dfs::Error(dfs::kRuntime, "bad partition mode: " + mode + " (expected naive|fasst)");
  r.weights = dfs::WeightSetting::parse(c->weights ? c->weights : "const:0.1");
  r.rebuild_eps = c->rebuild_eps;
  r.seed = c->seed;
  r.sim_cap = c->sim_cap > 0 ? c->sim_cap : 256;
  r.jacobi = c->jacobi;
  r.count = c->jacobi ? c->count : 0;
  return r;
}
}  // namespace

extern "C" {

const char* dfs_last_error(void) { return g_err.c_str(); }
int dfs_version(void) { return 1; }
void dfs_free(void* p) { std::free(p); }

uint32_t dfs_edge_hash(uint64_t u, uint64_t v) { return dfs::edge_hash(u, v); }
uint32_t dfs_random_value_at(uint64_t seed, uint32_t r) { return dfs::random_value_at(seed, r); }
int dfs_to_fixed_point(double w, uint32_t* out) {
  return guard([&] {
    need(out, "out");
    *out = dfs::to_fixed_point(w);
  });
}
int dfs_is_sampled(uint32_t x, uint32_t h, double w, int* out) {
  return guard([&] {
    need(out, "out");
    *out = (x ^ h) < dfs::to_fixed_point(w);  // sampling.hpp:37-39
  });
}

int dfs_graph_from_text(const char* text, size_t len, int directed, dfs_graph** out) {
  return guard([&] {
    need(out, "out");
    auto g = std::make_unique<dfs_graph>();
    g->g = dfs::graph_from_text(std::string_view(text ? text : "", text ? len : 0), directed != 0);
    *out = g.release();
  });
}
int dfs_graph_load(const char* path, int directed, dfs_graph** out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    auto g = std::make_unique<dfs_graph>();
    g->g = dfs::load_graph(path, directed != 0);
    *out = g.release();
  });
}
int dfs_graph_save_cache(const dfs_graph* g, const char* path) {
  return guard([&] {
    need(g, "graph");
    need(path, "path");
    dfs::save_graph_cache(g->g, path);
  });
}
int dfs_graph_from_csr(uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* adj,
                       const uint64_t* orig_ids, dfs_graph** out) {
  return guard([&] {
    need(offsets, "offsets");
    if (m) need(adj, "adj");
    need(out, "out");
    auto g = std::make_unique<dfs_graph>();
    g->g = dfs::graph_from_csr(n, m, offsets, adj, orig_ids);
    *out = g.release();
  });
}
int dfs_graph_generate(const char* kind, uint32_t a, uint64_t m, uint64_t seed, dfs_graph** out) {
  return guard([&] {
    need(kind, "kind");
    need(out, "out");
    auto g = std::make_unique<dfs_graph>();
    const std::string k = kind;
    if (k == "rmat") g->g = dfs::generate_rmat(a, m, seed);
    else if (k == "er") g->g = dfs::generate_er(a, m, seed);
    else throw dfs::Error(dfs::kInvalid, "unknown generator: " + k);
    *out = g.release();
  });
}
void dfs_graph_free(dfs_graph* g) { delete g; }
uint32_t dfs_graph_n(const dfs_graph* g) { return g ? g->g.n : 0; }
uint64_t dfs_graph_m(const dfs_graph* g) { return g ? g->g.m : 0; }
int dfs_graph_arrays(const dfs_graph* g, const uint64_t** offsets, const uint32_t** adj,
                     const uint64_t** orig_ids, const uint32_t** ehash,
                     const uint32_t** in_degree) {
  return guard([&] {
    need(g, "graph");
    if (offsets) *offsets = g->g.offsets.data();
    if (adj) *adj = g->g.adj.data();
    if (orig_ids) *orig_ids = g->g.orig_id.data();
    if (ehash || in_degree) dfs::ensure_graph_fields(g->g);
    if (ehash) *ehash = g->g.ehash.data();
    if (in_degree) *in_degree = g->g.in_degree.data();
  });
}
int dfs_graph_weights(const dfs_graph* g, const char* spec, uint64_t seed, uint32_t* out) {
  return guard([&] {
    need(g, "graph");
    need(spec, "spec");
    need(out, "out");
    std::vector<uint32_t> w;
    dfs::assign_weights(g->g, dfs::WeightSetting::parse(spec),
                        dfs::derive_seed(seed, dfs::kSeedTagWeights), w);
    std::memcpy(out, w.data(), w.size() * 4);
  });
}
int dfs_weight_string(const char* spec, char** out) {
  return guard([&] {
    need(spec, "spec");
    need(out, "out");
    *out = dup_string(dfs::WeightSetting::parse(spec).to_string());
  });
}

int dfs_ctx_create(int device, dfs_ctx** out) {
  return guard([&] {
    need(out, "out");
    auto c = std::make_unique<dfs_ctx>();
    c->c = std::make_unique<dfs::Context>(device);
    *out = c.release();
  });
}
void dfs_ctx_destroy(dfs_ctx* ctx) { delete ctx; }

int dfs_upload(dfs_ctx* ctx, const dfs_graph* g) {
  return guard([&] {
    need(ctx, "ctx");
    need(g, "graph");
    ctx->c->upload(g->g);
  });
}

int dfs_ctx_stream(dfs_ctx* ctx, void** stream) {
  return guard([&] {
    need(ctx, "ctx");
    need(stream, "stream");
    *stream = ctx->c->stream();
  });
}
int dfs_graph_pin(dfs_graph* g) {
  return guard([&] {
    need(g, "graph");
    if (g->pinned) return;
    dfs::cuda_check(cudaHostRegister(g->g.offsets.data(), g->g.offsets.size() * 8,
                                     cudaHostRegisterDefault),
                    "cudaHostRegister(offsets)");
    if (g->g.m)
      dfs::cuda_check(cudaHostRegister(g->g.adj.data(), g->g.m * 4, cudaHostRegisterDefault),
                      "cudaHostRegister(adj)");
    g->pinned = true;
  });
}

int dfs_run_json(dfs_ctx* ctx, const dfs_graph* g, const dfs_config* cfg, int timings,
                 char** json_out) {
  return guard([&] {
    need(ctx, "ctx");
    need(g, "graph");
    need(json_out, "json_out");
    dfs::RunConfig rc = to_config(cfg);
    ctx->c->upload(g->g);
    ctx->last = ctx->c->run(rc, &g->g);
    *json_out = dup_string(dfs::report_to_json(ctx->last, timings != 0));
  });
}
int dfs_run_resident_json(dfs_ctx* ctx, const dfs_graph* g, const dfs_config* cfg, int timings,
                          char** json_out) {
  return guard([&] {
    need(ctx, "ctx");
    need(json_out, "json_out");
    dfs::RunConfig rc = to_config(cfg);
    ctx->last = ctx->c->run(rc, g ? &g->g : nullptr);
    *json_out = dup_string(dfs::report_to_json(ctx->last, timings != 0));
  });
}
int dfs_last_stats(const dfs_ctx* ctx, dfs_stats* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    const dfs::Report& r = ctx->last;
    out->build = r.timings.build;
    out->fill = r.timings.fill;
    out->simulate = r.timings.simulate;
    out->select = r.timings.select;
    out->cascade = r.timings.cascade;
    out->total = r.timings.total;
    out->upload = r.timings.upload;
    out->sketch_edge_updates = r.sketch_edge_updates;
    out->items_processed = r.items_processed;
    out->sweeps_total = r.sweeps_total;
    out->items_fwd = r.items_fwd;
    out->items_rev = r.items_rev;
    out->cnt_edges = r.cnt_edges;
    out->cnt_batches = r.cnt_batches;
    out->cnt_touched = r.cnt_touched;
    out->cnt_sweeps = r.cnt_sweeps;
    out->cnt_convergences = r.cnt_convergences;
    out->launches = r.launches;
    out->sim_active = r.sim_active;
    out->sim_launches = r.sim_launches;
    out->n = uint32_t(r.n);
    out->m = r.m;
    out->cnt_cas_rows = r.cnt_cas_rows;
    out->cnt_cas_edges = r.cnt_cas_edges;
    out->cnt_cascades = r.cnt_cascades;
    out->run_kernel = r.run_kernel;
    out->item_density = r.item_density;
    out->max_sweeps = r.max_sweeps;
    out->rerun_jacobi = r.rerun_jacobi ? 1u : 0u;
    out->rescored_rows = r.rescored_rows;
  });
}

int dfs_prepare(dfs_ctx* ctx, const dfs_graph* g, const dfs_config* cfg) {
  return guard([&] {
    need(ctx, "ctx");
    need(g, "graph");
    dfs::RunConfig rc = to_config(cfg);
    ctx->c->upload(g->g);
    ctx->c->prepare(rc, &g->g);
  });
}
int dfs_prepare_partition(dfs_ctx* ctx, const dfs_graph* g, const dfs_config* cfg,
                          uint32_t rank, uint32_t world) {
  return guard([&] {
    need(ctx, "ctx");
    dfs::RunConfig rc = to_config(cfg);
    if (g) ctx->c->upload(g->g);  // g == NULL: use the resident graph
    ctx->c->prepare(rc, g ? &g->g : nullptr, rank, world);
  });
}
int dfs_mc_influence(dfs_ctx* ctx, const dfs_graph* g, int resident, const uint32_t* seeds,
                     uint32_t nseeds, uint32_t trials, uint64_t seed, uint32_t runs,
                     const char* weights, double* mean, double* std_error, uint32_t* reached) {
  return guard([&] {
    need(ctx, "ctx");
    need(mean, "mean");
    need(std_error, "std_error");
    if (nseeds) need(seeds, "seeds");
    if (!resident) {
      need(g, "graph");
      ctx->c->upload(g->g);
    }
    const std::vector<uint32_t> s(seeds, seeds + nseeds);
    const std::vector<uint32_t> r = ctx->c->mc_influence(
        s, trials, seed, runs, dfs::WeightSetting::parse(weights ? weights : "const:0.1"),
        g ? &g->g : nullptr, mean, std_error);
    if (reached) std::memcpy(reached, r.data(), r.size() * 4);
  });
}

int dfs_fasst_stats(dfs_ctx* ctx, const dfs_graph* g, const dfs_config* cfg,
                    uint64_t* dup_count, uint64_t* loads, uint64_t fill[2]) {
  return guard([&] {
    need(ctx, "ctx");
    need(dup_count, "dup_count");
    need(loads, "loads");
    need(fill, "fill");
    dfs::RunConfig rc = to_config(cfg);
    const std::vector<uint64_t> h = ctx->c->fasst_stats(rc, g ? &g->g : nullptr);
    const uint32_t mu = rc.mu;
    std::memcpy(dup_count, h.data(), (size_t(mu) + 1) * 8);
    std::memcpy(loads, h.data() + mu + 1, size_t(mu) * 8);
    fill[0] = h[2 * size_t(mu) + 1];
    fill[1] = h[2 * size_t(mu) + 2];
  });
}

static_assert(DFS_PEER_HANDLE_BYTES == dfs::kPeerHandleBytes, "peer handle size");
int dfs_peer_export(dfs_ctx* ctx, void* handle_out) {
  return guard([&] {
    need(ctx, "ctx");
    need(handle_out, "handle_out");
    ctx->c->peer_export(handle_out);
  });
}
int dfs_peer_open(dfs_ctx* ctx, uint32_t rank, uint32_t world, const void* handles) {
  return guard([&] {
    need(ctx, "ctx");
    need(handles, "handles");
    ctx->c->peer_open(rank, world, handles);
  });
}
int dfs_peer_link(dfs_ctx* const* ctxs, uint32_t world) {
  return guard([&] {
    need(ctxs, "ctxs");
    std::vector<dfs::Context*> v;
    for (uint32_t i = 0; i < world; ++i) {
      need(ctxs[i], "ctx");
      v.push_back(ctxs[i]->c.get());
    }
    dfs::Context::peer_link(v);
  });
}
int dfs_peer_run_json(dfs_ctx* ctx, const dfs_graph* g, const dfs_config* cfg, int timings,
                      int resident, char** json_out) {
  return guard([&] {
    need(ctx, "ctx");
    need(json_out, "json_out");
    dfs::RunConfig rc = to_config(cfg);
    if (!resident) {
      need(g, "graph");
      ctx->c->upload(g->g);
    }
    ctx->last = ctx->c->run_peer(rc, g ? &g->g : nullptr);
    *json_out = dup_string(dfs::report_to_json(ctx->last, timings != 0));
  });
}
int dfs_scores_device(dfs_ctx* ctx, uint32_t tau, int full, void* dst) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->stage_scores_device(tau, full, static_cast<double*>(dst));
  });
}
int dfs_rebuild(dfs_ctx* ctx, uint32_t tau) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->stage_rebuild(tau);
  });
}
int dfs_plan(const dfs_ctx* ctx, uint32_t* x_sorted, uint32_t* order, int* degraded) {
  return guard([&] {
    need(ctx, "ctx");
    std::vector<uint32_t> x, o;
    bool d = false;
    ctx->c->stage_plan(x, o, &d);
    if (x_sorted) std::memcpy(x_sorted, x.data(), x.size() * 4);
    if (order) std::memcpy(order, o.data(), o.size() * 4);
    if (degraded) *degraded = d;
  });
}
int dfs_device_graph_size(dfs_ctx* ctx, uint32_t tau, uint64_t* m_tau, uint32_t* words) {
  return guard([&] {
    need(ctx, "ctx");
    std::vector<uint64_t> off, mask;
    std::vector<uint32_t> adj;
    uint32_t w = 0;
    ctx->c->stage_device_graph(tau, off, adj, mask, &w);
    if (m_tau) *m_tau = adj.size();
    if (words) *words = w;
  });
}
int dfs_device_graph(dfs_ctx* ctx, uint32_t tau, uint64_t* offsets, uint32_t* adj,
                     uint64_t* mask) {
  return guard([&] {
    need(ctx, "ctx");
    std::vector<uint64_t> o, mk;
    std::vector<uint32_t> a;
    uint32_t w = 0;
    ctx->c->stage_device_graph(tau, o, a, mk, &w);
    if (offsets) std::memcpy(offsets, o.data(), o.size() * 8);
    if (adj) std::memcpy(adj, a.data(), a.size() * 4);
    if (mask) std::memcpy(mask, mk.data(), mk.size() * 8);
  });
}
int dfs_fill(dfs_ctx* ctx, uint32_t tau) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->stage_fill(tau);
  });
}
int dfs_simulate(dfs_ctx* ctx, uint32_t tau, int cap, int jacobi, int* sweeps) {
  return guard([&] {
    need(ctx, "ctx");
    // jacobi: bit 0 = Jacobi schedule, bit 1 = count reference-schedule units
    const int s = ctx->c->stage_simulate(tau, cap > 0 ? cap : 256, jacobi & 1, (jacobi >> 1) & 1);
    if (sweeps) *sweeps = s;
    if (s < 0)
      throw dfs::Error(dfs::kRuntime, "simulate did not converge within " +
                                          std::to_string(cap > 0 ? cap : 256) +
                                          " iterations; register monotonicity must be broken");
  });
}
int dfs_scores(dfs_ctx* ctx, uint32_t tau, double* out_n) {
  return guard([&] {
    need(ctx, "ctx");
    need(out_n, "out");
    ctx->c->stage_scores(tau, out_n);
  });
}
int dfs_commit_cascade(dfs_ctx* ctx, uint32_t tau, uint32_t seed, uint64_t* visited) {
  return guard([&] {
    need(ctx, "ctx");
    const uint64_t v = ctx->c->stage_commit_cascade(tau, seed);
    if (visited) *visited = v;
  });
}
int dfs_visited_count(dfs_ctx* ctx, uint32_t tau, uint64_t* out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    *out = ctx->c->stage_visited(tau);
  });
}
int dfs_get_registers(dfs_ctx* ctx, uint32_t tau, int8_t* out_nJ) {
  return guard([&] {
    need(ctx, "ctx");
    need(out_nJ, "out");
    ctx->c->stage_get_registers(tau, out_nJ);
  });
}
int dfs_get_visited(dfs_ctx* ctx, uint32_t tau, uint64_t* out_words) {
  return guard([&] {
    need(ctx, "ctx");
    need(out_words, "out");
    ctx->c->stage_get_visited(tau, out_words);
  });
}
int dfs_set_registers(dfs_ctx* ctx, uint32_t tau, const int8_t* in_nJ) {
  return guard([&] {
    need(ctx, "ctx");
    need(in_nJ, "in");
    ctx->c->stage_set_registers(tau, in_nJ);
  });
}

int dfs_rank_counters(dfs_ctx* ctx, uint32_t tau, uint64_t out[8]) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    ctx->c->stage_counters(tau, out);
  });
}

int dfs_format_report(const dfs_report_fields* f, char** json_out) {
  return guard([&] {
    need(f, "fields");
    need(json_out, "json_out");
    dfs::Report rep;
    dfs_config c{f->k, f->r, f->devices, f->mode, f->weights, f->rebuild_eps, f->seed, 256, 0, 0};
    rep.config = to_config(&c);
    rep.n = f->n;
    rep.m = f->m;
    rep.seeds.assign(f->seeds, f->seeds + f->steps);
    rep.seeds_dense.assign(f->seeds_dense, f->seeds_dense + f->steps);
    rep.score_trajectory.assign(f->traj, f->traj + f->steps);
    rep.rebuilds = f->rebuilds;
    if (f->rebuilds) rep.rebuild_rounds.assign(f->rebuild_rounds, f->rebuild_rounds + f->rebuilds);
    rep.saturated = f->saturated != 0;
    rep.degraded_plan = f->degraded != 0;
    rep.reduced_elements = f->reduced_elements;
    rep.broadcast_elements = f->broadcast_elements;
    rep.barriers = f->barriers;
    rep.timings = {f->t_build, f->t_fill, f->t_simulate, f->t_select, f->t_cascade, f->t_total, 0};
    *json_out = dup_string(dfs::report_to_json(rep, f->with_timings != 0));
  });
}

int dfs_influence(const dfs_graph* g, const uint32_t* seeds, uint32_t nseeds, uint32_t trials,
                  uint64_t seed, uint32_t runs, const char* weights, double* mean,
                  double* std_error) {
  return guard([&] {
    need(g, "graph");
    need(mean, "mean");
    need(std_error, "std_error");
    std::vector<uint32_t> w;
    dfs::assign_weights(g->g, dfs::WeightSetting::parse(weights ? weights : "const:0.1"),
                        dfs::derive_seed(seed, dfs::kSeedTagWeights), w);
    std::vector<uint32_t> s(seeds, seeds + nseeds);
    dfs::influence_stats(g->g, w, s, trials, seed, runs, mean, std_error);
  });
}
int dfs_greedy_exact(const dfs_graph* g, uint32_t k, uint32_t trials, uint64_t seed,
                     const char* weights, uint32_t* out_k) {
  return guard([&] {
    need(g, "graph");
    need(out_k, "out");
    std::vector<uint32_t> w;
    dfs::assign_weights(g->g, dfs::WeightSetting::parse(weights ? weights : "const:0.1"),
                        dfs::derive_seed(seed, dfs::kSeedTagWeights), w);
    std::vector<uint32_t> r = dfs::greedy_exact(g->g, w, k, trials, seed);
    std::memcpy(out_k, r.data(), r.size() * 4);
  });
}

}  // extern "C"
