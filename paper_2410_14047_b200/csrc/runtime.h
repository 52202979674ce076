// runtime.h — host runtime: device context, resident graph, sample-space
// partitions ("ranks", FASST, proj/src/fasst.cpp:21-88) and the greedy loop
// of proj/src/runtime.cpp:37-179 driven entirely from the device (no host
// round-trips between rounds).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "dfs.h"
#include "graph.h"

namespace dfs {

// Grow-only named device buffers: repeated runs at the same sizes reuse them.
class Arena {
 public:
  ~Arena();
  void* get(const std::string& name, size_t bytes);
  // Already holds a buffer of at least `bytes` under `name`?
  bool has(const std::string& name, size_t bytes) const {
    auto it = bufs_.find(name);
    return it != bufs_.end() && it->second.bytes >= bytes;
  }
  size_t bytes() const { return total_; }
  // Scratch that may be freed whenever an allocation would otherwise fail
  // (no work in flight uses it: its users synchronise before returning).
  void set_reclaimable(const std::string& name) {
    for (const std::string& x : reclaimable_)
      if (x == name) return;
    reclaimable_.push_back(name);
  }
  bool reclaim();  // frees the reclaimable buffers; true if any bytes were freed
  void release();

 private:
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
  };
  std::unordered_map<std::string, Buf> bufs_;
  std::vector<std::string> reclaimable_;
  size_t total_ = 0;
};

struct RunConfig {  // proj/include/difuser/runtime.hpp:13-22
  uint32_t k = 1, r = 256, mu = 1;
  bool fasst = true;
  WeightSetting weights{};
  double rebuild_eps = 0.01;
  uint64_t seed = 0;
  int sim_cap = 256;
  int jacobi = 0;  // 1: exact reference sweep schedule (parity/debug)
  int count = 0;   // 1 (with jacobi): tally reference-schedule work units
};

struct PhaseTimings {  // runtime.hpp:24-27 (seconds; device-event based)
  double build = 0, fill = 0, simulate = 0, select = 0, cascade = 0, total = 0;
  double upload = 0;  // H2D + graph preparation (outside run() scope)
};

struct Report {  // runtime.hpp:29-41
  RunConfig config;
  uint64_t n = 0, m = 0;
  std::vector<uint64_t> seeds;
  std::vector<uint32_t> seeds_dense;
  std::vector<double> score_trajectory;
  std::vector<uint32_t> rebuild_rounds;
  uint32_t rebuilds = 0;
  bool saturated = false, degraded_plan = false;
  uint64_t reduced_elements = 0, broadcast_elements = 0, barriers = 0;
  PhaseTimings timings;
  // instrumentation (not part of the JSON contract)
  uint64_t sketch_edge_updates = 0, items_processed = 0, sweeps_total = 0;
  uint64_t items_fwd = 0, items_rev = 0, device_edges = 0;
  // reference-schedule units (count mode), summed over ranks and convergences
  uint64_t cnt_edges = 0, cnt_batches = 0, cnt_touched = 0, cnt_sweeps = 0, cnt_convergences = 0;
  uint64_t cnt_cas_rows = 0, cnt_cas_edges = 0, cnt_cascades = 0;
  uint64_t rescored_rows = 0;   // rows actually rescored (all partitions)
  double run_kernel = 0;        // seconds of the k_run launch (CUDA events on the stream)
  double item_density = 0;      // live simulations per forward item (partition 0)
  uint64_t launches = 0;        // kernels launched by run()
  double sim_active = 0;        // seconds of simulate launches that ran (not gated off)
  uint32_t sim_launches = 0;    // simulate launches that ran
  uint32_t max_sweeps = 0;      // most sweeps of one convergence (any partition)
  bool rerun_jacobi = false;    // decided by a Jacobi re-run (near sim_cap)
};

std::string report_to_json(const Report& rep, bool include_timings);

// Peer (multi-GPU) session of one context: which partition it holds, the
// mapped mailboxes / partial-score vectors of every rank, and the share of
// the GPU its persistent kernel may occupy (> 1 when several ranks' contexts
// live on one device, e.g. the single-GPU tests of the peer protocol).
struct PeerState {
  uint32_t world = 0, rank = 0;
  int grid_share = 1;
  PeerView view{};
  PeerBox* box = nullptr;
  std::vector<void*> opened;  // IPC mappings (closed on re-setup / destruction)
  unsigned long long timeouts_seen = 0;
};
// Exported handle: IPC handles of the mailbox, the partial-score vector and
// the dirty-row list, the device UUID and the process id.
constexpr size_t kPeerHandleBytes = 3 * 64 + 16 + 8;

class Context {
 public:
  explicit Context(int device);
  ~Context();
  int device() const { return device_; }
  cudaStream_t stream() const { return stream_; }

  // H2D of the CSR (offsets, adj) + on-device ehash, in-degree, transpose.
  void upload(const HostGraph& g);
  bool has_graph() const { return g_.n > 0; }

  // Plan + weights + per-rank sampled items (the reference's "build" phase).
  // part_world > 0: this context holds only partition part_rank of
  // part_world (= cfg.mu) — one FASST partition per GPU/process.
  void prepare(const RunConfig& cfg, const HostGraph* host_w_src = nullptr,
               uint32_t part_rank = 0, uint32_t part_world = 0);
  // Full greedy run on the resident graph.
  Report run(const RunConfig& cfg, const HostGraph* host_w_src = nullptr);

  // ---- stage API (parity harness), rank tau of the prepared session
  uint32_t ranks() const { return uint32_t(ranks_.size()); }
  void stage_fill(uint32_t tau);
  int stage_simulate(uint32_t tau, int cap, int jacobi, int count = 0);
  void stage_scores(uint32_t tau, double* out);
  uint64_t stage_commit_cascade(uint32_t tau, uint32_t seed);
  uint64_t stage_visited(uint32_t tau);
  void stage_counters(uint32_t tau, uint64_t out[8]);
  // Multi-process round pieces (device pointers; no host round-trip).
  void stage_scores_device(uint32_t tau, int full, double* dst);
  void stage_rebuild(uint32_t tau);
  void stage_get_visited(uint32_t tau, uint64_t* out);
  void stage_get_registers(uint32_t tau, int8_t* out);
  void stage_set_registers(uint32_t tau, const int8_t* in);
  void stage_device_graph(uint32_t tau, std::vector<uint64_t>& off, std::vector<uint32_t>& adj,
                          std::vector<uint64_t>& mask, uint32_t* words);
  void stage_plan(std::vector<uint32_t>& x, std::vector<uint32_t>& order, bool* degraded) const {
    x = x_;
    order = order_;
    *degraded = degraded_;
  }
  const PhaseTimings& last_timings() const { return last_; }
  void sync();

  // FASST analytics (fasst.cpp:101-168) of a plan on the resident graph:
  // out = [dup counts 0..mu | per-chunk loads | fill live lanes | batches].
  std::vector<uint64_t> fasst_stats(const RunConfig& cfg, const HostGraph* host_w_src);

  // Monte-Carlo influence (oracle.cpp:30-79) on the resident graph: per-trial
  // reached counts (run-major), mean and standard error bit-identical to the
  // reference's influence_stats.
  std::vector<uint32_t> mc_influence(const std::vector<uint32_t>& seeds, uint32_t trials,
                                     uint64_t seed, uint32_t runs, const WeightSetting& ws,
                                     const HostGraph* host_w_src, double* mean,
                                     double* std_error);

  // ---- peer mode (one FASST partition per GPU; exchange inside k_run)
  // After prepare(cfg, host, rank, world): write this rank's handle.
  void peer_export(void* out);
  // Map every rank's exported buffers (handles: world * kPeerHandleBytes).
  void peer_open(uint32_t rank, uint32_t world, const void* handles);
  // Same-process peers (one context per partition, distinct devices): direct pointers.
  static void peer_link(const std::vector<Context*>& ctxs);
  void peer_close();
  Report run_peer(const RunConfig& cfg, const HostGraph* host_w_src = nullptr);
  const PeerState& peer() const { return peer_; }

 private:
  Report run_impl(const RunConfig& cfg, const HostGraph* host_w_src, bool peer);
  void plan_weights(const RunConfig& cfg, const HostGraph* host_w_src);
  PeerBox* peer_box();
  void build_items(RankDev& r);
  void finish_items(RankDev& r, int dir, uint64_t cap_items, uint64_t* meta);
  void alloc_rank(RankDev& r, uint32_t tau);
  void reset_rank_state(RankDev& r);

  int device_ = 0;
  cudaStream_t stream_ = nullptr;
  Arena arena_;
  DevGraph g_{};
  std::vector<uint64_t> orig_id_;
  uint32_t* w_ = nullptr;   // weights of the prepared config (CSR order)
  uint32_t* tw_ = nullptr;  // the same in transposed order
  RunConfig cfg_{};
  std::vector<uint32_t> x_, order_;
  bool degraded_ = false;
  std::vector<RankDev> ranks_;
  PhaseTimings last_{};
  double prep_seconds_ = 0;
  PeerState peer_{};
};

}  // namespace dfs
