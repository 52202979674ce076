/*
 * difuser_b200.h — C-ABI of the B200-native sketch-IM hot path
 * (DiFuseR, arxiv 2410.14047).  Drop-in boundary for the reference's
 * `difuser::run` (proj/include/difuser/runtime.hpp:56) and its Python binding
 * `_difuser.run_json` (proj/bindings/pymodule.cpp:75-90).
 *
 * Conventions:
 *  - every entry point returns an int status (0 = ok) and never throws;
 *    dfs_last_error() returns the thread-local message of the last failure;
 *    status classes mirror the reference's exceptions: DFS_EINVAL =
 *    std::invalid_argument (ValueError), DFS_ERUNTIME = std::runtime_error
 *    (RuntimeError), DFS_ECUDA = CUDA failure, DFS_ENOMEM, DFS_EINDEX;
 *  - plain pointers and sizes only; host pointers are caller-owned and only
 *    read during the call; library-allocated outputs are released with
 *    dfs_free();
 *  - a context is bound to one CUDA device and is not re-entrant; distinct
 *    contexts may run concurrently.  There is no CPU fallback: without a GPU
 *    dfs_ctx_create fails with DFS_ECUDA.
 */
#ifndef DIFUSER_B200_H
#define DIFUSER_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFS_OK 0
#define DFS_EINVAL 1
#define DFS_ERUNTIME 2
#define DFS_ECUDA 3
#define DFS_ENOMEM 4
#define DFS_EINDEX 5

typedef struct dfs_graph dfs_graph; /* host WeightedGraph (graph.hpp:44-58) */
typedef struct dfs_ctx dfs_ctx;     /* device context (one GPU)            */

/* RunConfig (proj/include/difuser/runtime.hpp:13-22) + pybind kwargs
 * (proj/bindings/pymodule.cpp:86-89).  mode: "fasst" | "naive";
 * weights: "const:p" | "wc" | "normal:m,s" | "uniform:lo,hi". */
typedef struct dfs_config {
  uint32_t k;
  uint32_t r;
  uint32_t devices; /* mu: sample-space partitions (FASST devices) */
  const char *mode;
  const char *weights;
  double rebuild_eps;
  uint64_t seed;
  int32_t sim_cap; /* default 256 (runtime.hpp:21) */
  int32_t jacobi;  /* 0: in-place async schedule; 1: the reference's Jacobi schedule */
  int32_t count;   /* 1 (with jacobi): tally the reference-schedule work units */
} dfs_config;

/* Phase timings (runtime.hpp:24-27) plus instrumentation of the last run. */
typedef struct dfs_stats {
  double build, fill, simulate, select, cascade, total, upload;
  uint64_t sketch_edge_updates; /* live (item, sim) pairs merged by simulate */
  uint64_t items_processed;
  uint64_t sweeps_total;
  uint64_t items_fwd, items_rev;
  /* reference-schedule work units (count mode) */
  uint64_t cnt_edges, cnt_batches, cnt_touched, cnt_sweeps, cnt_convergences;
  uint64_t launches;     /* kernels launched by the run */
  double sim_active;     /* seconds of the simulate launches that ran */
  uint32_t sim_launches; /* simulate launches that ran */
  uint32_t n;
  uint64_t m;
  /* cascade work units (count mode): frontier rows over all levels, their
   * device-graph out-edges, cascades started */
  uint64_t cnt_cas_rows, cnt_cas_edges, cnt_cascades;
  double run_kernel; /* seconds of the whole-loop kernel launch (CUDA events) */
  double item_density; /* live simulations per sampled item (sets the pull switch points) */
  uint32_t max_sweeps;   /* most simulate sweeps of one convergence */
  uint32_t rerun_jacobi; /* 1: a convergence came near sim_cap; the run was decided by the
                            reference's Jacobi schedule (engine.cpp:88-96) */
  uint64_t rescored_rows; /* rows actually rescored (full passes after fills + dirty rows) */
} dfs_stats;

const char *dfs_last_error(void);
int dfs_version(void);
void dfs_free(void *p);

/* ---- hash / sampling helpers (hash.hpp:91-93, sampling.hpp:23-39,
 *      pymodule.cpp:123-133) ------------------------------------------------ */
uint32_t dfs_edge_hash(uint64_t u, uint64_t v);
uint32_t dfs_random_value_at(uint64_t seed, uint32_t r);
int dfs_to_fixed_point(double w, uint32_t *out);
int dfs_is_sampled(uint32_t x, uint32_t h, double w, int *out);

/* ---- host graph (graph.cpp:41-348; pymodule.cpp:35-73) ------------------- */
int dfs_graph_from_text(const char *text, size_t len, int directed, dfs_graph **out);
int dfs_graph_load(const char *path, int directed, dfs_graph **out);
int dfs_graph_save_cache(const dfs_graph *g, const char *path);
int dfs_graph_from_csr(uint32_t n, uint64_t m, const uint64_t *offsets, const uint32_t *adj,
                       const uint64_t *orig_ids /* nullable */, dfs_graph **out);
/* Deterministic synthetic inputs: kind "rmat" (a = scale) or "er" (a = n). */
int dfs_graph_generate(const char *kind, uint32_t a, uint64_t m, uint64_t seed, dfs_graph **out);
void dfs_graph_free(dfs_graph *g);
uint32_t dfs_graph_n(const dfs_graph *g);
uint64_t dfs_graph_m(const dfs_graph *g);
/* Borrowed views valid until dfs_graph_free. */
int dfs_graph_arrays(const dfs_graph *g, const uint64_t **offsets, const uint32_t **adj,
                     const uint64_t **orig_ids, const uint32_t **ehash,
                     const uint32_t **in_degree);
/* apply_weights (runtime.cpp:15-17) on the host: out has m entries. */
int dfs_graph_weights(const dfs_graph *g, const char *spec, uint64_t seed, uint32_t *out);
/* Weight-spec canonical string (WeightSetting::to_string, graph.cpp:228-245). */
int dfs_weight_string(const char *spec, char **out);

/* ---- device context ------------------------------------------------------ */
int dfs_ctx_create(int device, dfs_ctx **out);
void dfs_ctx_destroy(dfs_ctx *ctx);
/* H2D of the CSR + on-device ehash/in-degree/transpose (resident graph). */
int dfs_upload(dfs_ctx *ctx, const dfs_graph *g);
/* The context's CUDA stream (cudaStream_t), e.g. for timing with events. */
int dfs_ctx_stream(dfs_ctx *ctx, void **stream);
/* Page-lock the graph's CSR arrays so uploads are DMA from pinned memory. */
int dfs_graph_pin(dfs_graph *g);

/* ---- hot path ------------------------------------------------------------
 * dfs_run_json: run_json (pymodule.cpp:75-90): uploads g, applies weights,
 * runs the greedy loop, returns the report JSON (report.cpp:9-41).
 * dfs_run_resident_json: same on the graph already uploaded by dfs_upload
 * (g is still needed for randomized normal/uniform weights, else nullable). */
int dfs_run_json(dfs_ctx *ctx, const dfs_graph *g, const dfs_config *cfg, int timings,
                 char **json_out);
int dfs_run_resident_json(dfs_ctx *ctx, const dfs_graph *g, const dfs_config *cfg, int timings,
                          char **json_out);
int dfs_last_stats(const dfs_ctx *ctx, dfs_stats *out);

/* ---- stage entry points (parity harness; engine.hpp / fasst.hpp / sketch.hpp)
 * dfs_prepare = make_plan + apply_weights + build_device_graph for all tau. */
int dfs_prepare(dfs_ctx *ctx, const dfs_graph *g, const dfs_config *cfg);
int dfs_plan(const dfs_ctx *ctx, uint32_t *x_sorted, uint32_t *order, int *degraded);
/* One FASST partition per process (multi-GPU): this context builds only
 * partition `rank` of `world` (= cfg->devices); stage calls then use tau 0.
 * g == NULL reuses the resident graph (dfs_upload) instead of uploading.
 * Replaces the per-thread worker setup of proj/src/runtime.cpp:64-82. */
int dfs_prepare_partition(dfs_ctx *ctx, const dfs_graph *g, const dfs_config *cfg, uint32_t rank,
                          uint32_t world);
/* Row scores into a DEVICE buffer of n doubles (full = all rows, else the rows
 * dirtied by the last cascade) — the send buffer of the score exchange. */
int dfs_scores_device(dfs_ctx *ctx, uint32_t tau, int full, void *dst_device);
/* Rebuild: fill + simulate + full rescore (runtime.cpp:139-153). */
int dfs_rebuild(dfs_ctx *ctx, uint32_t tau);
int dfs_device_graph_size(dfs_ctx *ctx, uint32_t tau, uint64_t *m_tau, uint32_t *words);
int dfs_device_graph(dfs_ctx *ctx, uint32_t tau, uint64_t *offsets, uint32_t *adj,
                     uint64_t *mask);
int dfs_fill(dfs_ctx *ctx, uint32_t tau);                                   /* sketch.cpp:55-66 */
/* engine.cpp:88-96; jacobi bit 0: Jacobi schedule, bit 1: count work units */
int dfs_simulate(dfs_ctx *ctx, uint32_t tau, int cap, int jacobi, int *sweeps);
int dfs_scores(dfs_ctx *ctx, uint32_t tau, double *out_n);                  /* sketch.cpp:119-137 */
int dfs_commit_cascade(dfs_ctx *ctx, uint32_t tau, uint32_t seed, uint64_t *visited); /* engine.cpp:106-144 */
int dfs_visited_count(dfs_ctx *ctx, uint32_t tau, uint64_t *out);          /* sketch.cpp:139 */
int dfs_get_registers(dfs_ctx *ctx, uint32_t tau, int8_t *out_nJ);
/* VISITED bitset of partition tau in the reference layout (SketchMatrix::vis_row,
 * sketch.hpp:35-87): n rows of ceil(J/64) u64 words, bit j = register j VISITED. */
int dfs_get_visited(dfs_ctx *ctx, uint32_t tau, uint64_t *out_words);
int dfs_set_registers(dfs_ctx *ctx, uint32_t tau, const int8_t *in_nJ);
/* {updates, items, edges, batches, touched, sweeps, convergences, visited} */
int dfs_rank_counters(dfs_ctx *ctx, uint32_t tau, uint64_t out[8]);

/* ---- Monte-Carlo influence on the GPU (oracle.cpp:30-79, the binding's
 * influence(), pymodule.cpp:92-107): (mean, std_error) bit-identical to the
 * reference; reached (nullable) receives the trials*runs per-trial reached
 * counts in the reference's trial order.  resident != 0 uses the graph
 * uploaded by dfs_upload (g still needed for normal/uniform weights). */
int dfs_mc_influence(dfs_ctx *ctx, const dfs_graph *g, int resident, const uint32_t *seeds,
                     uint32_t nseeds, uint32_t trials, uint64_t seed, uint32_t runs,
                     const char *weights, double *mean, double *std_error, uint32_t *reached);

/* ---- FASST analytics (proj/src/fasst.cpp:101-168; CLI partition-stats /
 * fillrate, tools/difuser.cpp:116-159) on the resident graph (g: for
 * normal/uniform weights, else nullable).  cfg: r, devices (= mu), mode,
 * weights, seed.  Outputs (exact integer counts; fractions are count / m):
 * dup_count[mu+1] edges sampled by exactly k chunks (duplication_stats),
 * loads[mu] per-chunk sampled edges (device_edge_loads), fill[2] = {live
 * lanes, counted batches} over 32-lane batches of X (fill_rate; {0, 0} and
 * return DFS_OK when r % 32 != 0 — the reference throws there). */
int dfs_fasst_stats(dfs_ctx *ctx, const dfs_graph *g, const dfs_config *cfg,
                    uint64_t *dup_count, uint64_t *loads, uint64_t fill[2]);

/* ---- peer (multi-GPU) mode ----------------------------------------------
 * One FASST partition per GPU (one process per GPU, or one context per
 * partition in one process).  Replaces the per-device worker threads and the
 * in-process CollectiveGroup of proj/src/runtime.cpp:64-172 and
 * proj/src/collectives.cpp:44-113: the per-round reduce_to_root (binomial
 * order), root argmax, seed broadcast and visited-count allreduce run inside
 * the persistent kernel over peer memory (NVLink P2P; CUDA IPC between
 * processes) — the host does not participate between rounds.
 * Setup, per rank: dfs_prepare_partition(ctx, g, cfg{devices = world}, rank,
 * world) -> dfs_peer_export -> exchange the handles out of band (e.g.
 * torch.distributed all_gather) -> dfs_peer_open.  Same-process contexts on
 * distinct devices: dfs_peer_link instead.  Then every rank calls dfs_peer_run_json
 * concurrently; each returns the same report (= reference run with
 * devices = world).  A rank that never arrives makes the others fail with
 * DFS_ERUNTIME after 120 s instead of hanging. */
#define DFS_PEER_HANDLE_BYTES 216
int dfs_peer_export(dfs_ctx *ctx, void *handle_out /* DFS_PEER_HANDLE_BYTES */);
int dfs_peer_open(dfs_ctx *ctx, uint32_t rank, uint32_t world,
                  const void *handles /* world * DFS_PEER_HANDLE_BYTES, rank order */);
int dfs_peer_link(dfs_ctx *const *ctxs, uint32_t world);
/* resident != 0: use the graph uploaded by dfs_upload/dfs_prepare_partition
 * (g may be NULL for const/wc weights); else upload g first. */
int dfs_peer_run_json(dfs_ctx *ctx, const dfs_graph *g, const dfs_config *cfg, int timings,
                      int resident, char **json_out);

/* ---- report formatting (report.cpp:9-41) for drivers that assemble the
 * greedy loop themselves (multi-process path): same nlohmann dump(2) output. */
typedef struct dfs_report_fields {
  uint32_t k, r, devices;
  const char *mode;
  const char *weights;
  double rebuild_eps;
  uint64_t seed;
  uint64_t n, m;
  uint32_t steps; /* entries in seeds / seeds_dense / traj */
  const uint64_t *seeds;
  const uint32_t *seeds_dense;
  const double *traj;
  uint32_t rebuilds;
  const uint32_t *rebuild_rounds;
  int32_t saturated, degraded;
  uint64_t reduced_elements, broadcast_elements, barriers;
  int32_t with_timings;
  double t_build, t_fill, t_simulate, t_select, t_cascade, t_total;
} dfs_report_fields;
int dfs_format_report(const dfs_report_fields *f, char **json_out);

/* ---- verification oracles (oracle.cpp; host, not the hot path) ----------- */
int dfs_influence(const dfs_graph *g, const uint32_t *seeds, uint32_t nseeds, uint32_t trials,
                  uint64_t seed, uint32_t runs, const char *weights, double *mean,
                  double *std_error);
int dfs_greedy_exact(const dfs_graph *g, uint32_t k, uint32_t trials, uint64_t seed,
                     const char *weights, uint32_t *out_k);

#ifdef __cplusplus
}
#endif
#endif /* DIFUSER_B200_H */
