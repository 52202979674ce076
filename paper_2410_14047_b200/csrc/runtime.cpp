// runtime.cpp — host runtime of the sketch-IM hot path.
//
// The greedy loop of proj/src/runtime.cpp:37-179 runs as a fixed sequence of
// asynchronous launches on one stream: every decision the reference's root
// thread takes (argmax with the committed mask, saturation fallback, the
// eps-gated rebuild) is taken on the device and read by later kernels through
// device-resident control blocks, so the host never waits between rounds.
// Sample-space partitions (FASST "devices", fasst.cpp:21-88) that share one
// GPU are executed back to back on the same stream; their scores are combined
// in the reference's binomial order (collectives.cpp:44-64).
#include "runtime.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <numeric>
#include <unistd.h>

#include "hash.cuh"
#include <nvtx3/nvToolsExt.h>

namespace dfs {

namespace {
// NVTX range for the host-side phases (upload, build, run, peer setup): they
// show up in Nsight timelines and can scope ncu (--nvtx --nvtx-include).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}
uint32_t ceil_log2(uint32_t mu) {
  uint32_t l = 0;
  for (uint32_t s = 1; s < mu; s <<= 1) ++l;
  return l;
}
template <class T>
T* as(void* p) {
  return static_cast<T*>(p);
}
}  // namespace

// ---------------------------------------------------------------- arena
Arena::~Arena() { release(); }

void Arena::release() {
  for (auto& kv : bufs_)
    if (kv.second.p) cudaFree(kv.second.p);
  bufs_.clear();
  total_ = 0;
}

bool Arena::reclaim() {
  bool any = false;
  for (const std::string& name : reclaimable_) {
    auto it = bufs_.find(name);
    if (it == bufs_.end()) continue;
    if (it->second.p) {
      cudaFree(it->second.p);
      any = true;
    }
    total_ -= it->second.bytes;
    bufs_.erase(it);
  }
  return any;
}

void* Arena::get(const std::string& name, size_t bytes) {
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~size_t(255);
  Buf& b = bufs_[name];
  if (b.bytes < bytes) {
    if (b.p) {
      DFS_CUDA(cudaFree(b.p));
      total_ -= b.bytes;
    }
    b.p = nullptr;
    b.bytes = 0;
    cudaError_t e = cudaMalloc(&b.p, bytes);
    if (e == cudaErrorMemoryAllocation && reclaim()) {  // HBM pressure: drop idle scratch, retry
      cudaGetLastError();
      Buf& nb = bufs_[name];  // (reclaim may have rehashed the map)
      e = cudaMalloc(&nb.p, bytes);
      if (e == cudaSuccess) {
        nb.bytes = bytes;
        total_ += bytes;
        return nb.p;
      }
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error(kNoMem, "device allocation of " + std::to_string(bytes) + " bytes for " + name +
                              " failed: " + cudaGetErrorString(e));
    }
    b.bytes = bytes;
    total_ += bytes;
  }
  return b.p;
}

// ---------------------------------------------------------------- context
Context::Context(int device) : device_(device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw Error(kCuda, "no CUDA device available (the sm_100a path has no CPU fallback)");
  }
  if (device < 0 || device >= count) throw Error(kInvalid, "bad device ordinal");
  DFS_CUDA(cudaSetDevice(device));
  DFS_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
}

Context::~Context() {
  cudaSetDevice(device_);
  if (stream_) cudaStreamSynchronize(stream_);
  peer_close();
  arena_.release();
  if (stream_) cudaStreamDestroy(stream_);
}

void Context::sync() { DFS_CUDA(cudaStreamSynchronize(stream_)); }

void Context::upload(const HostGraph& hg) {
  NvtxRange nv("dfs.upload");
  DFS_CUDA(cudaSetDevice(device_));
  auto t0 = Clock::now();
  g_ = DevGraph{};
  g_.n = hg.n;
  g_.m = hg.m;
  const size_t n1 = size_t(hg.n) + 1, m = std::max<uint64_t>(hg.m, 1);
  g_.off = as<uint64_t>(arena_.get("g.off", n1 * 8));
  g_.adj = as<uint32_t>(arena_.get("g.adj", m * 4));
  g_.src = as<uint32_t>(arena_.get("g.src", m * 4));
  g_.ehash = as<uint32_t>(arena_.get("g.ehash", m * 4));
  g_.indeg = as<uint32_t>(arena_.get("g.indeg", n1 * 4));
  g_.toff = as<uint64_t>(arena_.get("g.toff", n1 * 8));
  g_.tedge = as<uint32_t>(arena_.get("g.tedge", m * 4));
  g_.tsrc = as<uint32_t>(arena_.get("g.tsrc", m * 4));
  g_.thash = as<uint32_t>(arena_.get("g.thash", m * 4));
  g_.tdst = as<uint32_t>(arena_.get("g.tdst", m * 4));
  DFS_CUDA(cudaMemcpyAsync(g_.off, hg.offsets.data(), n1 * 8, cudaMemcpyHostToDevice, stream_));
  if (hg.m)
    DFS_CUDA(cudaMemcpyAsync(g_.adj, hg.adj.data(), hg.m * 4, cudaMemcpyHostToDevice, stream_));
  const size_t tb = graph_prepare_tmp_bytes(hg.m, hg.n);
  launch_graph_prepare(g_, arena_.get("tmp.prep", tb), tb, stream_);
  orig_id_ = hg.orig_id;
  sync();
  arena_.set_reclaimable("tmp.prep");  // sort scratch (~12 B/edge): upload-only
  last_.upload = since(t0);
}

void Context::alloc_rank(RankDev& r, uint32_t tau) {
  const std::string p = "r" + std::to_string(tau) + ".";
  const uint32_t n = g_.n;
  const size_t nn = std::max<size_t>(n, 1);
  r.n = n;
  r.tau = tau;
  r.J = cfg_.r / cfg_.mu;
  r.Jp = (r.J + kBatch - 1) / kBatch * kBatch;
  r.W32 = r.Jp / kBatch;
  r.j_offset = tau * r.J;
  r.reg_key = derive_seed(cfg_.seed, kSeedTagRegisters);
  r.x = as<uint32_t>(arena_.get(p + "x", r.Jp * 4));
  r.xlut = as<uint32_t>(arena_.get(p + "xlut", 4100 * 4));
  r.jkey = as<uint64_t>(arena_.get(p + "jkey", r.Jp * 8));
  r.regs = as<int8_t>(arena_.get(p + "regs", nn * r.Jp));
  r.snap = cfg_.jacobi ? as<int8_t>(arena_.get(p + "snap", nn * r.Jp)) : nullptr;
  r.pristine = nullptr;  // decided once every partition is built (prepare)
  r.vis = as<uint32_t>(arena_.get(p + "vis", nn * r.W32 * 4));
  r.fresh[0] = as<uint32_t>(arena_.get(p + "fresh0", nn * r.W32 * 4));
  r.fresh[1] = as<uint32_t>(arena_.get(p + "fresh1", nn * r.W32 * 4));
  r.fresh[2] = as<uint32_t>(arena_.get(p + "fresh2", nn * r.W32 * 4));
  r.lstamp = as<uint32_t>(arena_.get(p + "lstamp", nn * 4));
  r.dstamp = as<uint32_t>(arena_.get(p + "dstamp", nn * 4));
  r.cstamp = as<unsigned long long>(arena_.get(p + "cstamp", nn * 8));
  r.dirty = as<uint32_t>(arena_.get(p + "dirty", nn * 4));
  r.tbits = cfg_.count ? as<uint32_t>(arena_.get(p + "tbits", (nn * r.W32 + 31) / 32 * 4 + 4))
                       : nullptr;
  r.scores = as<double>(arena_.get(p + "scores", nn * 8));
  r.ctl = as<RankCtl>(arena_.get(p + "ctl", sizeof(RankCtl)));
  r.q.counts = as<unsigned int>(arena_.get(p + "qcnt", 16 * 4));
  // Host-side slice: slot values (sorted for FASST) and register keys of the
  // global register index tau*J + j (runtime.cpp:72, sketch.cpp:55-58).
  std::vector<uint32_t> xs(r.Jp, 0xFFFFFFFFu);
  std::vector<uint64_t> jk(r.Jp, 0);
  for (uint32_t j = 0; j < r.J; ++j) {
    xs[j] = x_[size_t(tau) * r.J + j];
    jk[j] = splitmix64_at(r.reg_key, uint64_t(r.j_offset) + j);
  }
  DFS_CUDA(cudaMemcpyAsync(r.x, xs.data(), r.Jp * 4, cudaMemcpyHostToDevice, stream_));
  DFS_CUDA(cudaMemcpyAsync(r.jkey, jk.data(), r.Jp * 8, cudaMemcpyHostToDevice, stream_));
  // (cudaMemcpyAsync stages pageable host data before returning: no sync needed)
  launch_xlut(r, stream_);
}

// Chunk headers, small/big split and small-item list of one direction, from
// the row item offsets the one-pass build wrote.  Sized by upper bounds
// (chunks <= cap/kChunk + n) so the host never waits here; the exact counts
// land in meta[0..2] (chunks, small|big chunk counts, small items) and are
// read back once per partition by build_items.
void Context::finish_items(RankDev& r, int dir, uint64_t cap_items, uint64_t* meta) {
  const std::string p = "r" + std::to_string(r.tau) + (dir ? ".rev." : ".fwd.");
  Items& it = dir ? r.rev : r.fwd;
  const uint32_t n = g_.n;
  const size_t sb = scan_tmp_bytes(uint64_t(n) + 2);
  void* stmp = arena_.get("tmp.scan", sb);
  uint32_t* row_cnt = as<uint32_t>(arena_.get("tmp.rowcnt", (size_t(n) + 2) * 4));
  DFS_CUDA(cudaMemsetAsync(row_cnt, 0, (size_t(n) + 1) * 4, stream_));
  launch_row_chunks(n, it, row_cnt, stream_);
  uint64_t* row_chunk64 = as<uint64_t>(arena_.get("tmp.rowchunk", (size_t(n) + 2) * 8));
  scan_u32_u64(row_cnt, row_chunk64, n, stmp, sb, stream_);
  const uint64_t cap = cap_items / kChunk + n + 1;  // >= chunks
  if (cap >= (uint64_t(1) << 31)) throw Error(kRuntime, "too many work chunks");
  DFS_CUDA(cudaMemcpyAsync(meta, row_chunk64 + n, 8, cudaMemcpyDeviceToDevice, stream_));
  it.chunk_row = as<uint32_t>(arena_.get(p + "chunk_row", cap * 4));
  it.chunk_beg = as<uint64_t>(arena_.get(p + "chunk_beg", (cap + 1) * 8));
  it.row_chunk = as<uint32_t>(arena_.get(p + "row_chunk", (size_t(n) + 1) * 4));
  launch_chunk_write(n, it, row_chunk64, stream_);
  it.small = as<uint32_t>(arena_.get(p + "small", cap * 4));
  it.big = as<uint32_t>(arena_.get(p + "big", cap * 4));
  it.small_items = as<uint32_t>(arena_.get(p + "small_items", std::max<uint64_t>(cap_items, 1) * 4));
  unsigned int* c2 = reinterpret_cast<unsigned int*>(meta + 1);
  launch_split_chunks(it, meta, cap, c2, stream_);
  launch_small_items(it, c2, cap, reinterpret_cast<unsigned long long*>(meta + 2), stream_);
  it.chunks = cap;  // provisional (exact after build_items' readback)
}

// Sampled items of one partition (fasst.cpp:50-88), both directions, each in
// ONE pass over the edge positions (k_items_onepass: windows evaluated once,
// block scan + decoupled look-back, items and row offsets written in place).
// The item arrays are sized from a sampled estimate (every stride-th edge);
// the rare underestimate re-runs the passes with the exact total.  Two host
// readbacks per partition: the estimate and the final metadata.
void Context::build_items(RankDev& r) {
  const std::string p = "r" + std::to_string(r.tau) + ".";
  const uint64_t m = g_.m;
  const uint32_t n = g_.n;
  Items& f = r.fwd;
  Items& rv = r.rev;
  const int fa = cfg_.fasst ? 1 : 0;
  const uint32_t wconst =
      cfg_.weights.kind == WeightKind::Constant ? to_fixed_point(cfg_.weights.a) : 0u;
  const bool filter = fa && cfg_.mu > 1 && m > 0;
  // meta: [0..3] fwd chunk meta, [4..7] rev chunk meta, [8] fwd total, [9] fwd
  // live, [10] sample, [12] rev total, [13] rev live, [14] tile counters
  uint64_t* meta = as<uint64_t>(arena_.get("tmp.meta", 16 * 8));
  auto* um = reinterpret_cast<unsigned long long*>(meta);
  const uint64_t tiles = items_tiles(m);
  auto* tstate = as<unsigned long long>(arena_.get("tmp.tiles", (2 * tiles + 2) * 8));
  f.row_off = as<uint64_t>(arena_.get(p + "fwd.row_off", (size_t(n) + 1) * 8));
  rv.row_off = as<uint64_t>(arena_.get(p + "rev.row_off", (size_t(n) + 1) * 8));
  DFS_CUDA(cudaMemsetAsync(meta, 0, 16 * 8, stream_));
  if (!m) {
    DFS_CUDA(cudaMemsetAsync(f.row_off, 0, (size_t(n) + 1) * 8, stream_));
    DFS_CUDA(cudaMemsetAsync(rv.row_off, 0, (size_t(n) + 1) * 8, stream_));
  }
  // capacity: sampled estimate (exact below 2^20 edges) plus slack
  const uint64_t stride = std::max<uint64_t>(1, m >> 20);
  launch_items_sample(g_, w_, wconst, r, fa, stride, um + 10, stream_);
  uint64_t sampled = 0;
  DFS_CUDA(cudaMemcpyAsync(&sampled, meta + 10, 8, cudaMemcpyDeviceToHost, stream_));
  sync();
  uint64_t cap = stride == 1 ? sampled : sampled * stride + sampled * stride / 8 + 65536;
  uint64_t hm[16];
  for (int attempt = 0;; ++attempt) {
    const size_t ic = std::max<uint64_t>(cap, 1);
    for (int d = 0; d < 2; ++d) {
      Items& it = d ? rv : f;
      const std::string q = p + (d ? "rev." : "fwd.");
      it.other = as<uint32_t>(arena_.get(q + "other", ic * 4));
      it.row = as<uint32_t>(arena_.get(q + "row", ic * 4));
      it.mask = as<uint32_t>(arena_.get(q + "mask", ic * 4));
      it.batch = as<uint8_t>(arena_.get(q + "batch", ic));
    }
    DFS_CUDA(cudaMemsetAsync(meta, 0, 10 * 8, stream_));
    DFS_CUDA(cudaMemsetAsync(meta + 11, 0, 5 * 8, stream_));
    DFS_CUDA(cudaMemsetAsync(tstate, 0, 2 * tiles * 8, stream_));
    auto* ctr = reinterpret_cast<unsigned int*>(meta + 14);
    // multi-partition FASST plans: positions outside the partition's value
    // range are skipped; row offsets from per-row counts
    uint32_t* rc[2] = {nullptr, nullptr};
    if (filter)
      for (int d = 0; d < 2; ++d) {
        rc[d] = as<uint32_t>(arena_.get(d ? "tmp.rowcnt.rev" : "tmp.rowcnt.fwd", (size_t(n) + 2) * 4));
        DFS_CUDA(cudaMemsetAsync(rc[d], 0, (size_t(n) + 1) * 4, stream_));
      }
    launch_items_onepass(g_, w_, tw_, wconst, r, 0, fa, f, cap, tstate, ctr, um + 8, rc[0], stream_);
    launch_items_onepass(g_, w_, tw_, wconst, r, 1, fa, rv, cap, tstate + tiles, ctr + 1, um + 12,
                         rc[1], stream_);
    if (filter) {
      const size_t sb = scan_tmp_bytes(uint64_t(n) + 2);
      void* stmp = arena_.get("tmp.scan", sb);
      scan_u32_u64(rc[0], f.row_off, n, stmp, sb, stream_);
      scan_u32_u64(rc[1], rv.row_off, n, stmp, sb, stream_);
    }
    finish_items(r, 0, cap, meta);
    finish_items(r, 1, cap, meta + 4);
    DFS_CUDA(cudaMemcpyAsync(hm, meta, sizeof hm, cudaMemcpyDeviceToHost, stream_));
    sync();
    if (hm[8] <= cap) break;
    if (attempt) throw Error(kRuntime, "item build: capacity re-run overflowed");
    cap = hm[8];  // underestimated: exact total, once more
  }
  if (hm[8] != hm[12]) throw Error(kRuntime, "item build: direction totals differ");
  f.count = rv.count = hm[8];
  for (int d = 0; d < 2; ++d) {
    Items& it = d ? rv : f;
    it.chunks = hm[4 * d];
    it.nsmall = uint32_t(hm[4 * d + 1]);
    it.nbig = uint32_t(hm[4 * d + 1] >> 32);
    it.nsmall_items = hm[4 * d + 2];
  }
  f.live = hm[9];
}

void Context::reset_rank_state(RankDev& r) {
  const size_t nn = std::max<uint32_t>(r.n, 1);
  DFS_CUDA(cudaMemsetAsync(r.vis, 0, nn * r.W32 * 4, stream_));
  DFS_CUDA(cudaMemsetAsync(r.fresh[0], 0, nn * r.W32 * 4, stream_));
  DFS_CUDA(cudaMemsetAsync(r.fresh[1], 0, nn * r.W32 * 4, stream_));
  DFS_CUDA(cudaMemsetAsync(r.fresh[2], 0, nn * r.W32 * 4, stream_));
  DFS_CUDA(cudaMemsetAsync(r.lstamp, 0, nn * 4, stream_));
  DFS_CUDA(cudaMemsetAsync(r.dstamp, 0, nn * 4, stream_));
  DFS_CUDA(cudaMemsetAsync(r.cstamp, 0, nn * 8, stream_));
  DFS_CUDA(cudaMemsetAsync(r.regs, 0, nn * r.Jp, stream_));
  DFS_CUDA(cudaMemsetAsync(r.scores, 0, nn * 8, stream_));
  DFS_CUDA(cudaMemsetAsync(r.q.counts, 0, 16 * 4, stream_));
  RankCtl c{};
  c.tick = 1;
  DFS_CUDA(cudaMemcpyAsync(r.ctl, &c, sizeof c, cudaMemcpyHostToDevice, stream_));
}

void Context::prepare(const RunConfig& cfg, const HostGraph* host_w_src, uint32_t part_rank,
                      uint32_t part_world) {
  NvtxRange nv("dfs.build");
  auto t0 = Clock::now();
  static const bool ptrace = getenv("DFS_PREP_TRACE") != nullptr;  // diagnostics
  auto mark = [&](const char* what) {
    if (ptrace) fprintf(stderr, "prep %-12s %8.3f ms\n", what, since(t0) * 1e3);
  };
  plan_weights(cfg, host_w_src);
  mark("plan_weights");
  // ---- per-rank state and sampled items (fasst.cpp:50-88, build phase)
  if (part_world && (part_world != cfg.mu || part_rank >= part_world))
    throw Error(kInvalid, "partition rank/world must match devices");
  const uint32_t first = part_world ? part_rank : 0;
  const uint32_t count = part_world ? 1 : cfg.mu;
  ranks_.assign(count, RankDev{});
  for (uint32_t t = 0; t < count; ++t) {
    RankDev& r = ranks_[t];
    alloc_rank(r, first + t);
    mark("alloc_rank");
    build_items(r);
    mark("build_items");
    const std::string p = "r" + std::to_string(first + t) + ".q.";
    const uint64_t cap = std::max<uint64_t>(std::max(r.fwd.chunks, r.rev.chunks), 1);
    for (int gi = 0; gi < kGens; ++gi) {
      r.q.chunks[gi] = as<uint32_t>(arena_.get(p + "c" + std::to_string(gi), cap * 4));
      r.q.rows[gi] = as<uint32_t>(arena_.get(p + "r" + std::to_string(gi),
                                             std::max<uint32_t>(g_.n, 1) * 4));
    }
    reset_rank_state(r);
    mark("reset");
  }
  // Cached first fill per partition (rebuild fills become a copy), only while
  // HBM allows once every partition's working set is allocated.
  // DFS_NO_PRISTINE=1 forces the re-hashing fill (tests of the HBM-pressure path).
  const char* np_env = getenv("DFS_NO_PRISTINE");
  const bool no_pristine = np_env && atoi(np_env) != 0;
  for (RankDev& r : ranks_) {
    if (no_pristine) break;
    const size_t bytes = std::max<size_t>(r.n, 1) * r.Jp;
    const std::string name = "r" + std::to_string(r.tau) + ".pristine";
    bool take = arena_.has(name, bytes);
    if (!take) {  // cudaMemGetInfo waits behind queued work: only on first use
      size_t fr = 0, tot = 0;
      DFS_CUDA(cudaMemGetInfo(&fr, &tot));
      take = fr > bytes + (size_t(4) << 30);
      if (!take) {  // idle scratch first (the build above is stream-ordered: drain it)
        sync();
        if (arena_.reclaim()) {
          DFS_CUDA(cudaMemGetInfo(&fr, &tot));
          take = fr > bytes + (size_t(4) << 30);
        }
      }
    }
    if (take) r.pristine = as<int8_t>(arena_.get(name, bytes));
  }
  mark("pristine");
  prep_seconds_ = since(t0);
}

// Validation, FASST plan and weights of a run (runtime.cpp:38-47,
// fasst.cpp:21-48, apply_weights runtime.cpp:15-17).
void Context::plan_weights(const RunConfig& cfg, const HostGraph* host_w_src) {
  if (!has_graph()) throw Error(kRuntime, "no graph uploaded");
  DFS_CUDA(cudaSetDevice(device_));
  // runtime.cpp:38-42, then gen_random_vector (sampling.cpp:8), make_plan
  // (fasst.cpp:21-27) — same checks, same order, same exception classes.
  if (cfg.k == 0 || cfg.k > g_.n) throw Error(kInvalid, "run: k must be in [1, n]");
  if (cfg.mu == 0) throw Error(kInvalid, "run: mu must be >= 1");
  if (!(cfg.rebuild_eps >= 0.0)) throw Error(kInvalid, "run: rebuild_eps must be >= 0");
  if (cfg.r == 0) throw Error(kInvalid, "gen_random_vector: R must be >= 1");
  if (cfg.r % cfg.mu != 0)
    throw Error(kInvalid, "make_plan: mu must divide R (" + std::to_string(cfg.mu) + " vs " +
                              std::to_string(cfg.r) + ")");
  if (cfg.mu > 64) throw Error(kInvalid, "run: at most 64 sample-space partitions per context");
  if (cfg.r / cfg.mu > 8192) throw Error(kInvalid, "run: at most 8192 simulations per partition");
  cfg_ = cfg;
  // ---- plan (fasst.cpp:21-48): X_r, stable sort for FASST
  const uint64_t xs = derive_seed(cfg.seed, kSeedTagSamples);
  std::vector<uint32_t> x(cfg.r);
  for (uint32_t i = 0; i < cfg.r; ++i) x[i] = random_value_at(xs, i);
  order_.resize(cfg.r);
  std::iota(order_.begin(), order_.end(), 0u);
  degraded_ = false;
  if (cfg.fasst) {
    std::stable_sort(order_.begin(), order_.end(),
                     [&](uint32_t a, uint32_t b) { return x[a] < x[b]; });
    degraded_ = (cfg.r / cfg.mu) < 32;
  }
  x_.resize(cfg.r);
  for (uint32_t i = 0; i < cfg.r; ++i) x_[i] = x[order_[i]];
  // ---- weights (apply_weights, runtime.cpp:15-17)
  w_ = as<uint32_t>(arena_.get("g.w", std::max<uint64_t>(g_.m, 1) * 4));
  tw_ = as<uint32_t>(arena_.get("g.tw", std::max<uint64_t>(g_.m, 1) * 4));
  switch (cfg.weights.kind) {
    case WeightKind::Constant:
      launch_weights(g_, 0, to_fixed_point(cfg.weights.a), w_, stream_);
      launch_tweights(g_, 0, to_fixed_point(cfg.weights.a), w_, tw_, stream_);
      break;
    case WeightKind::WeightedCascade:
      launch_weights(g_, 1, 0, w_, stream_);
      launch_tweights(g_, 1, 0, w_, tw_, stream_);
      break;
    default: {
      if (!host_w_src) throw Error(kRuntime, "randomized weights need the host graph");
      std::vector<uint32_t> hw;
      assign_weights(*host_w_src, cfg.weights, derive_seed(cfg.seed, kSeedTagWeights), hw);
      DFS_CUDA(cudaMemcpyAsync(w_, hw.data(), g_.m * 4, cudaMemcpyHostToDevice, stream_));
      launch_tweights(g_, 2, 0, w_, tw_, stream_);
      sync();
    }
  }
}

Report Context::run(const RunConfig& cfg, const HostGraph* host_w_src) {
  Report rep = run_impl(cfg, host_w_src, false);
  // sim_cap contract (engine.cpp:88-96): the reference throws when a Jacobi
  // convergence needs more than cap sweeps.  The async schedule needs at most
  // as many sweeps as Jacobi, so exceeding the cap there already throws.  A
  // convergence that came within 10% of the cap is decided exactly by
  // re-running with the reference's Jacobi schedule (same report, or the
  // reference's runtime_error).  Measured Jacobi/async ratios of deep
  // convergences are 1.05-1.10 (C3: 215 vs 204 sweeps; R-MAT s20 WC: 128 vs
  // 116), so a Jacobi count above the cap implies an async count above this
  // threshold on these graphs; an unconditional guarantee would need
  // per-register hop tracking.
  if (!cfg.jacobi && 10 * uint64_t(rep.max_sweeps) >= 9 * uint64_t(cfg.sim_cap)) {
    RunConfig exact = cfg;
    exact.jacobi = 1;
    Report jr = run_impl(exact, host_w_src, false);
    jr.config.jacobi = cfg.jacobi;
    jr.rerun_jacobi = true;
    return jr;
  }
  return rep;
}

std::vector<uint32_t> Context::mc_influence(const std::vector<uint32_t>& seeds, uint32_t trials,
                                           uint64_t seed, uint32_t runs, const WeightSetting& ws,
                                           const HostGraph* host_w_src, double* mean,
                                           double* std_error) {
  if (!has_graph()) throw Error(kRuntime, "no graph uploaded");
  DFS_CUDA(cudaSetDevice(device_));
  // oracle.cpp:33-37: same checks, same exception class
  if (trials == 0 || runs == 0) throw Error(kInvalid, "oracle: trials and runs must be >= 1");
  for (uint32_t sd : seeds)
    if (sd >= g_.n) throw Error(kInvalid, "oracle: seed id out of range");
  const uint64_t m = g_.m, n = g_.n;
  // weights as the binding assigns them (pymodule.cpp:96-98)
  uint32_t* w = as<uint32_t>(arena_.get("mc.w", std::max<uint64_t>(m, 1) * 4));
  switch (ws.kind) {
    case WeightKind::Constant: launch_weights(g_, 0, to_fixed_point(ws.a), w, stream_); break;
    case WeightKind::WeightedCascade: launch_weights(g_, 1, 0, w, stream_); break;
    default: {
      if (!host_w_src) throw Error(kRuntime, "randomized weights need the host graph");
      std::vector<uint32_t> hw;
      assign_weights(*host_w_src, ws, derive_seed(seed, kSeedTagWeights), hw);
      DFS_CUDA(cudaMemcpyAsync(w, hw.data(), m * 4, cudaMemcpyHostToDevice, stream_));
      sync();
    }
  }
  const uint64_t total = uint64_t(trials) * runs;
  const uint64_t nb_total = (total + 31) / 32;
  const uint64_t per_batch = m * 4 + 5 * n * 4 + 128;
  size_t fr = 0, tot = 0;
  DFS_CUDA(cudaMemGetInfo(&fr, &tot));
  const uint64_t budget = std::min<uint64_t>(uint64_t(8) << 30, fr / 2);
  const uint64_t nb = std::max<uint64_t>(1, std::min<uint64_t>(nb_total, budget / per_batch));
  uint32_t* live = as<uint32_t>(arena_.get("mc.live", std::max<uint64_t>(nb * m, 1) * 4));
  uint32_t* vis = as<uint32_t>(arena_.get("mc.vis", nb * n * 4));
  uint32_t* fresh = as<uint32_t>(arena_.get("mc.fresh", nb * 2 * n * 4));
  uint32_t* queue = as<uint32_t>(arena_.get("mc.queue", nb * 2 * n * 4));
  uint32_t* reached = as<uint32_t>(arena_.get("mc.reached", nb_total * 32 * 4));
  uint32_t* dseeds = as<uint32_t>(arena_.get("mc.seeds", std::max<size_t>(seeds.size(), 1) * 4));
  if (!seeds.empty())
    DFS_CUDA(cudaMemcpyAsync(dseeds, seeds.data(), seeds.size() * 4, cudaMemcpyHostToDevice,
                             stream_));
  const uint64_t base = derive_seed(seed, kSeedTagOracle);
  for (uint64_t b0 = 0; b0 < nb_total; b0 += nb) {
    const uint32_t cnt = uint32_t(std::min<uint64_t>(nb, nb_total - b0));
    launch_mc_influence(g_, w, base, trials, total, b0, cnt, dseeds, uint32_t(seeds.size()), live,
                        vis, fresh, queue, reached + b0 * 32, stream_);
  }
  std::vector<uint32_t> h(nb_total * 32);
  DFS_CUDA(cudaMemcpyAsync(h.data(), reached, h.size() * 4, cudaMemcpyDeviceToHost, stream_));
  sync();
  h.resize(total);
  // oracle.cpp:65-77, in the reference's trial order
  double sum = 0, sumsq = 0;
  for (uint64_t i = 0; i < total; ++i) {
    const double reached_i = double(h[i]);
    sum += reached_i;
    sumsq += reached_i * reached_i;
  }
  const double T = double(trials) * runs;
  *mean = sum / T;
  *std_error = 0.0;
  if (T > 1) {
    const double var = (sumsq - sum * sum / T) / (T - 1);
    *std_error = std::sqrt(std::max(0.0, var) / T);
  }
  return h;
}

std::vector<uint64_t> Context::fasst_stats(const RunConfig& cfg, const HostGraph* host_w_src) {
  RunConfig c = cfg;
  c.k = 1;  // k is not an input of the analytics
  if (c.r > 32768) throw Error(kInvalid, "fasst_stats: at most 32768 simulations");
  plan_weights(c, host_w_src);
  const uint32_t R = c.r, mu = c.mu;
  uint32_t* x = as<uint32_t>(arena_.get("fs.x", size_t(R) * 4));
  uint32_t* lut = as<uint32_t>(arena_.get("fs.lut", 4100 * 4));
  unsigned long long* out = as<unsigned long long>(arena_.get("fs.out", (2 * size_t(mu) + 3) * 8));
  DFS_CUDA(cudaMemcpyAsync(x, x_.data(), size_t(R) * 4, cudaMemcpyHostToDevice, stream_));
  if (c.fasst) launch_xlut_of(x, R, lut, stream_);
  launch_fasst_stats(g_, w_, x, lut, R, mu, c.fasst ? 1 : 0, R % 32 == 0 ? 1 : 0, out, stream_);
  std::vector<uint64_t> h(2 * size_t(mu) + 3);
  DFS_CUDA(cudaMemcpyAsync(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost, stream_));
  sync();
  return h;
}

Report Context::run_peer(const RunConfig& cfg, const HostGraph* host_w_src) {
  if (!peer_.world) throw Error(kRuntime, "peer mode: call peer setup (export/open or link) first");
  if (cfg.mu != peer_.world)
    throw Error(kInvalid, "peer mode: devices must equal the peer world size");
  return run_impl(cfg, host_w_src, true);
}

Report Context::run_impl(const RunConfig& cfg, const HostGraph* host_w_src, bool peer) {
  NvtxRange nv(peer ? "dfs.run_peer" : "dfs.run");
  auto t_total = Clock::now();
  const unsigned long long launches0 = launches();
  if (peer) {
    prepare(cfg, host_w_src, peer_.rank, peer_.world);
    if (ranks_[0].scores != peer_.view.scores[peer_.rank] ||
        ranks_[0].dirty != peer_.view.dirty[peer_.rank])
      throw Error(kRuntime, "peer mode: partition buffers moved since the peer setup; redo it");
  } else {
    prepare(cfg, host_w_src);
  }
  // mu: the reference's device count (report counters); nl: partitions held here
  const uint32_t n = g_.n, mu = cfg.mu, k = cfg.k, nl = uint32_t(ranks_.size());
  cudaStream_t s = stream_;

  // ---- run-level device state
  RunArrays ra;
  ra.ctl = as<RunCtl>(arena_.get("run.ctl", sizeof(RunCtl)));
  ra.committed = as<uint8_t>(arena_.get("run.committed", std::max<uint32_t>(n, 1)));
  ra.seeds = as<uint32_t>(arena_.get("run.seeds", k * 4));
  ra.traj = as<double>(arena_.get("run.traj", k * 8));
  ra.rebuild_rounds = as<uint32_t>(arena_.get("run.rb", k * 4));
  ra.nblk = 2048;  // >= any cooperative grid (argmax partials)
  ra.blk_score = as<double>(arena_.get("run.bs", ra.nblk * 8));
  ra.blk_arg = as<uint32_t>(arena_.get("run.ba", ra.nblk * 4));
  ra.blk_min = as<uint32_t>(arena_.get("run.bm", ra.nblk * 4));
  ra.nseg = (n + kSeg - 1) / kSeg;
  ra.seg_score = as<double>(arena_.get("run.ss", std::max<uint32_t>(ra.nseg, 1) * 8));
  ra.seg_arg = as<uint32_t>(arena_.get("run.sa", std::max<uint32_t>(ra.nseg, 1) * 4));
  ra.seg_min = as<uint32_t>(arena_.get("run.sm", std::max<uint32_t>(ra.nseg, 1) * 4));
  ra.seg_stamp = as<uint32_t>(arena_.get("run.st", std::max<uint32_t>(ra.nseg, 1) * 4));
  DFS_CUDA(cudaMemsetAsync(ra.seg_stamp, 0, std::max<uint32_t>(ra.nseg, 1) * 4, s));
  DFS_CUDA(cudaMemsetAsync(ra.ctl, 0, sizeof(RunCtl), s));
  DFS_CUDA(cudaMemsetAsync(ra.committed, 0, std::max<uint32_t>(n, 1), s));
  const double* argmax_src = ranks_[0].scores;
  std::vector<RankCtl*> hctl(nl);
  std::vector<const double*> hparts(nl);
  for (uint32_t t = 0; t < nl; ++t) {
    hctl[t] = ranks_[t].ctl;
    hparts[t] = ranks_[t].scores;
  }
  RankCtl** dctl = as<RankCtl*>(arena_.get("run.ctls", nl * sizeof(void*)));
  const double** dparts = as<const double*>(arena_.get("run.parts", nl * sizeof(void*)));
  DFS_CUDA(cudaMemcpyAsync(dctl, hctl.data(), nl * sizeof(void*), cudaMemcpyHostToDevice, s));
  DFS_CUDA(cudaMemcpyAsync(dparts, hparts.data(), nl * sizeof(void*), cudaMemcpyHostToDevice, s));
  if (nl > 1 || peer) {
    ra.reduced = as<double>(arena_.get("run.reduced", std::max<uint32_t>(n, 1) * 8));
    argmax_src = ra.reduced;
  }
  const unsigned int* rebuild = &ra.ctl->rebuild_now;

  // phase events: [0] start, per round 4 boundaries, plus the initial ones
  std::vector<cudaEvent_t> ev;
  auto mark = [&]() {
    cudaEvent_t e;
    DFS_CUDA(cudaEventCreate(&e));
    DFS_CUDA(cudaEventRecord(e, s));
    ev.push_back(e);
    return ev.size() - 1;
  };
  PhaseTimings pt;
  pt.build = prep_seconds_;
  struct Span {
    size_t a, b;
    double* acc;
    int sim_step = -2;  // simulate span: -1 initial, else the round it may rebuild after
  };
  std::vector<Span> spans;
  size_t krun0 = size_t(-1);

  // Default: the whole loop as one persistent kernel (launch_run).
  // DFS_RUN_MODE=launches selects the per-phase launch sequence (same results).
  // When sweeps / cascade levels switch to pull (frontier chunks * f > all
  // chunks): dense items (many live simulations each, e.g. weighted cascade)
  // make full pull passes pay off earlier (A/B: C3 simulate -19%, cascade
  // -21%; sparse IC items keep the later switch).  Since the bottom-up
  // cascade levels propagate in place (bits gained in a level spread within
  // it), mid-density items (IC at R = 1024: the north star, density 7.5) gain
  // from an EARLIER bottom-up switch (cascade 11.7 -> 10.4 ms at f = 16),
  // while C3 (density 19) keeps f = 4 and C2 (2.7) f = 8 (A/B over
  // f = 4, 8, 16, 32).  DFS_SIM_PULL / DFS_CAS_PULL override.
  const double density = ranks_[0].fwd.count ? double(ranks_[0].fwd.live) / ranks_[0].fwd.count : 0;
  const int pull_sim = density >= 10.0 ? 1 : density >= 6.0 ? 2 : 4;
  const int pull_cas = density >= 10.0 ? 4 : density >= 6.0 ? 16 : 8;
  static const bool multi_env =
      getenv("DFS_RUN_MODE") && std::string(getenv("DFS_RUN_MODE")) == "launches";
  const bool multi = multi_env && !peer;  // peer mode exchanges inside k_run only
  unsigned long long* phase_ns = as<unsigned long long>(arena_.get("run.phase", 8 * 8));
  if (!multi) {
    int lj = 0;
    while ((1u << lj) < ranks_[0].J) ++lj;
    RankDev* dranks = as<RankDev>(arena_.get("run.ranks", nl * sizeof(RankDev)));
    DFS_CUDA(cudaMemcpyAsync(dranks, ranks_.data(), nl * sizeof(RankDev), cudaMemcpyHostToDevice, s));
    DFS_CUDA(cudaMemsetAsync(phase_ns, 0, 8 * 8, s));
    const size_t f0 = mark();
    for (uint32_t t = 0; t < nl; ++t) launch_fill(ranks_[t], nullptr, 0, s, false);
    const size_t f1 = mark();
    spans.push_back({f0, f1, &pt.fill});
    krun0 = mark();
    launch_run(dranks, nl, k, cfg.r, n, cfg.rebuild_eps, cfg.sim_cap, cfg.jacobi, cfg.count, 53 - lj,
               ra, dparts, dctl, ra.reduced, phase_ns, peer ? &peer_.view : nullptr,
               peer ? peer_.grid_share : 1, pull_sim, pull_cas, s);
  } else {
    size_t e0 = mark();
    for (uint32_t t = 0; t < nl; ++t) launch_fill(ranks_[t], nullptr, 0, s);
    size_t e1 = mark();
    for (uint32_t t = 0; t < nl; ++t) launch_simulate(ranks_[t], cfg.jacobi, cfg.count, cfg.sim_cap, nullptr, 0, s);
    size_t e2 = mark();
    for (uint32_t t = 0; t < nl; ++t) launch_score(ranks_[t], 1, nullptr, 0, s);
    spans.push_back({e0, e1, &pt.fill});
    spans.push_back({e1, e2, &pt.simulate, -1});
    size_t prev = e2;
    for (uint32_t step = 0; step < k; ++step) {
      // select: rescore dirty rows, binomial-order sum, argmax (runtime.cpp:88-122)
      for (uint32_t t = 0; t < nl; ++t) launch_score(ranks_[t], 0, rebuild, 0, s);
      if (nl > 1) launch_treesum(dparts, nl, n, ra.reduced, s);
      launch_argmax(argmax_src, ra, n, s);
      size_t a = mark();
      spans.push_back({prev, a, &pt.select});
      // commit + cascade (runtime.cpp:124-127) and the covered-count allreduce
      for (uint32_t t = 0; t < nl; ++t) launch_cascade(ranks_[t], &ra.ctl->choice, 0, s);
      launch_round_end(ra, dctl, nl, k, cfg.r, cfg.rebuild_eps, s);
      size_t b = mark();
      spans.push_back({a, b, &pt.cascade});
      prev = b;
      if (step + 1 < k) {  // eps-gated rebuild (runtime.cpp:139-153), predicated on device
        for (uint32_t t = 0; t < nl; ++t) launch_fill(ranks_[t], rebuild, 1, s, true);
        size_t c = mark();
        for (uint32_t t = 0; t < nl; ++t)
          launch_simulate(ranks_[t], cfg.jacobi, cfg.count, cfg.sim_cap, rebuild, 1, s);
        size_t d = mark();
        for (uint32_t t = 0; t < nl; ++t) launch_score(ranks_[t], 1, rebuild, 1, s);
        spans.push_back({b, c, &pt.fill});
        spans.push_back({c, d, &pt.simulate, int(step)});
        prev = d;
      }
    }
  }
  size_t eend = mark();
  sync();
  if (peer) {
    PeerBox b{};
    DFS_CUDA(cudaMemcpy(&b, peer_.box, sizeof b, cudaMemcpyDeviceToHost));
    if (b.timeouts != peer_.timeouts_seen) {
      // the ranks' barrier epochs have drifted apart: the mapping is unusable
      // until every rank redoes the setup (export/open zero the mailboxes)
      peer_close();
      throw Error(kRuntime, "peer mode: a peer did not reach a round barrier in time "
                            "(peer process failed?); results are invalid; redo the peer setup");
    }
  }
  if (getenv("DFS_DBG") && (atoi(getenv("DFS_DBG")) & 4)) dump_trace();

  // ---- results
  Report rep;
  rep.config = cfg;
  rep.n = n;
  rep.m = g_.m;
  rep.degraded_plan = degraded_;
  RunCtl rc{};
  DFS_CUDA(cudaMemcpy(&rc, ra.ctl, sizeof rc, cudaMemcpyDeviceToHost));
  rep.seeds_dense.resize(k);
  rep.score_trajectory.resize(k);
  DFS_CUDA(cudaMemcpy(rep.seeds_dense.data(), ra.seeds, k * 4, cudaMemcpyDeviceToHost));
  DFS_CUDA(cudaMemcpy(rep.score_trajectory.data(), ra.traj, k * 8, cudaMemcpyDeviceToHost));
  rep.rebuilds = rc.n_rebuilds;
  rep.rebuild_rounds.resize(rc.n_rebuilds);
  if (rc.n_rebuilds)
    DFS_CUDA(cudaMemcpy(rep.rebuild_rounds.data(), ra.rebuild_rounds, rc.n_rebuilds * 4,
                        cudaMemcpyDeviceToHost));
  rep.saturated = rc.saturated != 0;
  for (uint32_t t = 0; t < nl; ++t) {
    RankCtl c{};
    DFS_CUDA(cudaMemcpy(&c, ranks_[t].ctl, sizeof c, cudaMemcpyDeviceToHost));
    if (c.error) {
      for (cudaEvent_t e : ev) cudaEventDestroy(e);
      throw Error(kRuntime, "simulate did not converge within " + std::to_string(cfg.sim_cap) +
                                " iterations; register monotonicity must be broken");
    }
    rep.sketch_edge_updates += c.updates;
    rep.items_processed += c.items_processed;
    rep.sweeps_total += c.total_sweeps;
    rep.max_sweeps = std::max(rep.max_sweeps, c.max_sweeps);
    rep.items_fwd += ranks_[t].fwd.count;
    rep.items_rev += ranks_[t].rev.count;
    rep.cnt_edges += c.cnt_edges;
    rep.cnt_batches += c.cnt_batches;
    rep.cnt_touched += c.cnt_touched;
    rep.cnt_sweeps += c.cnt_sweeps;
    rep.cnt_convergences += c.cnt_convergences;
    rep.cnt_cas_rows += c.cnt_cas_rows;
    rep.cnt_cas_edges += c.cnt_cas_edges;
    rep.cnt_cascades += c.cnt_cascades;
    rep.rescored_rows += c.rescored_rows;
  }
  for (uint32_t sd : rep.seeds_dense) rep.seeds.push_back(orig_id_[sd]);
  // comms counters of the reference's collective schedule (collectives.cpp:
  // 19,62,76,107; pinned by tests/test_runtime.cpp:169-180).
  rep.reduced_elements = uint64_t(k) * (uint64_t(n) + 1) * (mu - 1);
  rep.broadcast_elements = uint64_t(k) * 2 * (mu - 1);
  rep.barriers = uint64_t(k) * (8 + ceil_log2(mu));
  if (!multi) {
    unsigned long long hp[4];
    DFS_CUDA(cudaMemcpy(hp, phase_ns, sizeof hp, cudaMemcpyDeviceToHost));
    pt.fill += hp[0] * 1e-9;
    pt.simulate += hp[1] * 1e-9;
    pt.select += hp[2] * 1e-9;
    pt.cascade += hp[3] * 1e-9;
    rep.sim_active = hp[1] * 1e-9;
    rep.sim_launches = (1 + rep.rebuilds) * nl;
  }
  for (const Span& sp : spans) {
    float ms = 0;
    DFS_CUDA(cudaEventElapsedTime(&ms, ev[sp.a], ev[sp.b]));
    *sp.acc += ms * 1e-3;
    if (sp.sim_step == -1 ||
        (sp.sim_step >= 0 && std::find(rep.rebuild_rounds.begin(), rep.rebuild_rounds.end(),
                                       uint32_t(sp.sim_step)) != rep.rebuild_rounds.end())) {
      rep.sim_active += ms * 1e-3;
      rep.sim_launches += nl;
    }
  }
  if (krun0 != size_t(-1)) {
    float ms = 0;
    DFS_CUDA(cudaEventElapsedTime(&ms, ev[krun0], ev[eend]));
    rep.run_kernel = ms * 1e-3;
  }
  for (cudaEvent_t e : ev) cudaEventDestroy(e);
  pt.upload = last_.upload;
  pt.total = since(t_total);
  rep.launches = launches() - launches0;
  rep.item_density = density;
  rep.timings = pt;
  last_ = pt;
  return rep;
}

// ---------------------------------------------------------------- peer mode
// One FASST partition per GPU; the per-round exchange runs inside k_run over
// peer memory.  Setup only maps buffers: rank t's mailbox and
// its partial-score vector (the send buffer of the reference's reduce_to_root,
// collectives.cpp:44-64) become directly addressable by every other rank.
namespace {
struct PeerHandle {
  cudaIpcMemHandle_t box, scores, dirty;
  unsigned char uuid[16];
  int64_t pid;
};
static_assert(sizeof(PeerHandle) <= kPeerHandleBytes, "peer handle layout");

void device_uuid(int dev, unsigned char out[16]) {
  cudaDeviceProp p{};
  DFS_CUDA(cudaGetDeviceProperties(&p, dev));
  std::memcpy(out, &p.uuid, 16);
}
}  // namespace

// How long a peer barrier waits for a rank (DFS_PEER_TIMEOUT_S, default 120 s).
static unsigned long long peer_timeout_ns() {
  const char* e = getenv("DFS_PEER_TIMEOUT_S");
  const double sec = e ? atof(e) : 120.0;
  return static_cast<unsigned long long>((sec > 0 ? sec : 120.0) * 1e9);
}

PeerBox* Context::peer_box() {
  return as<PeerBox>(arena_.get("peer.box", sizeof(PeerBox)));
}

void Context::peer_close() {
  for (void* p : peer_.opened) cudaIpcCloseMemHandle(p);
  peer_ = PeerState{};
}

static void check_partition(const std::vector<RankDev>& ranks, const RunConfig& cfg,
                            uint32_t rank, uint32_t world) {
  if (world < 2 || world > kMaxPeers)
    throw Error(kInvalid, "peer mode: world size must be in [2, " + std::to_string(kMaxPeers) + "]");
  if (rank >= world) throw Error(kInvalid, "peer mode: rank out of range");
  if (ranks.size() != 1 || cfg.mu != world || ranks[0].tau != rank)
    throw Error(kRuntime, "peer mode: prepare this context as partition rank of world first");
}

void Context::peer_export(void* out) {
  DFS_CUDA(cudaSetDevice(device_));
  if (ranks_.size() != 1) throw Error(kRuntime, "peer mode: prepare a single partition first");
  peer_close();
  PeerBox* box = peer_box();
  DFS_CUDA(cudaMemsetAsync(box, 0, sizeof(PeerBox), stream_));  // barrier epochs restart at 0
  sync();
  PeerHandle h{};
  DFS_CUDA(cudaIpcGetMemHandle(&h.box, box));
  DFS_CUDA(cudaIpcGetMemHandle(&h.scores, ranks_[0].scores));
  DFS_CUDA(cudaIpcGetMemHandle(&h.dirty, ranks_[0].dirty));
  device_uuid(device_, h.uuid);
  h.pid = int64_t(getpid());
  std::memset(out, 0, kPeerHandleBytes);
  std::memcpy(out, &h, sizeof h);
}

void Context::peer_open(uint32_t rank, uint32_t world, const void* handles) {
  NvtxRange nv("dfs.peer_open");
  DFS_CUDA(cudaSetDevice(device_));
  check_partition(ranks_, cfg_, rank, world);
  for (void* p : peer_.opened) cudaIpcCloseMemHandle(p);
  peer_.opened.clear();
  PeerState ps;
  ps.world = world;
  ps.rank = rank;
  ps.box = peer_box();
  ps.view.world = world;
  ps.view.rank = rank;
  ps.view.timeout_ns = peer_timeout_ns();
  unsigned char me[16];
  device_uuid(device_, me);
  const auto* hs = static_cast<const unsigned char*>(handles);
  ps.grid_share = 0;
  for (uint32_t t = 0; t < world; ++t) {
    PeerHandle h;
    std::memcpy(&h, hs + size_t(t) * kPeerHandleBytes, sizeof h);
    if (std::memcmp(h.uuid, me, 16) == 0) ++ps.grid_share;
    if (t == rank) {
      ps.view.box[t] = ps.box;
      ps.view.scores[t] = ranks_[0].scores;
      ps.view.dirty[t] = ranks_[0].dirty;
      continue;
    }
    if (h.pid == int64_t(getpid()))
      throw Error(kInvalid, "peer mode: same-process peers must be linked with peer_link");
    void* pb = nullptr;
    void* psc = nullptr;
    DFS_CUDA(cudaIpcOpenMemHandle(&pb, h.box, cudaIpcMemLazyEnablePeerAccess));
    ps.opened.push_back(pb);
    DFS_CUDA(cudaIpcOpenMemHandle(&psc, h.scores, cudaIpcMemLazyEnablePeerAccess));
    ps.opened.push_back(psc);
    void* pd = nullptr;
    DFS_CUDA(cudaIpcOpenMemHandle(&pd, h.dirty, cudaIpcMemLazyEnablePeerAccess));
    ps.opened.push_back(pd);
    ps.view.box[t] = static_cast<PeerBox*>(pb);
    ps.view.scores[t] = static_cast<const double*>(psc);
    ps.view.dirty[t] = static_cast<const uint32_t*>(pd);
  }
  if (ps.grid_share < 1) ps.grid_share = 1;
  peer_ = std::move(ps);
}

void Context::peer_link(const std::vector<Context*>& ctxs) {
  const uint32_t world = uint32_t(ctxs.size());
  for (uint32_t i = 0; i < world; ++i) {
    Context* c = ctxs[i];
    check_partition(c->ranks_, c->cfg_, i, world);
    DFS_CUDA(cudaSetDevice(c->device_));
    c->peer_close();
    PeerBox* box = c->peer_box();
    DFS_CUDA(cudaMemset(box, 0, sizeof(PeerBox)));
  }
  for (uint32_t i = 0; i < world; ++i) {
    Context* c = ctxs[i];
    DFS_CUDA(cudaSetDevice(c->device_));
    PeerState ps;
    ps.world = world;
    ps.rank = i;
    ps.box = c->peer_box();
    ps.view.world = world;
    ps.view.rank = i;
    ps.view.timeout_ns = peer_timeout_ns();
    ps.grid_share = 0;
    for (uint32_t t = 0; t < world; ++t) {
      Context* o = ctxs[t];
      if (o->device_ == c->device_) {
        // Two persistent grids of one process on one device cannot be relied
        // on to run concurrently (device-synchronising runtime calls and
        // cooperative-launch serialisation): use one process per rank there.
        if (o != c)
          throw Error(kInvalid, "peer mode: same-process peers must be on distinct devices "
                                "(use one process per rank, dfs_peer_export/open)");
        ++ps.grid_share;
      } else {
        int can = 0;
        DFS_CUDA(cudaDeviceCanAccessPeer(&can, c->device_, o->device_));
        if (!can) throw Error(kRuntime, "peer mode: no P2P access between the peer devices");
        const cudaError_t e = cudaDeviceEnablePeerAccess(o->device_, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) DFS_CUDA(e);
        cudaGetLastError();
      }
      ps.view.box[t] = o->peer_box();
      ps.view.scores[t] = o->ranks_[0].scores;
      ps.view.dirty[t] = o->ranks_[0].dirty;
    }
    c->peer_ = std::move(ps);
  }
}

// ---------------------------------------------------------------- stage API
static void check_tau(uint32_t tau, size_t n) {
  if (tau >= n) throw Error(kIndex, "rank index out of range (prepare first)");
}

void Context::stage_fill(uint32_t tau) {
  check_tau(tau, ranks_.size());
  launch_fill(ranks_[tau], nullptr, 0, stream_);
  sync();
}

int Context::stage_simulate(uint32_t tau, int cap, int jacobi, int count) {
  check_tau(tau, ranks_.size());
  RankDev& r = ranks_[tau];
  if (jacobi && !r.snap) {
    r.snap = as<int8_t>(arena_.get("r" + std::to_string(tau) + ".snap",
                                   std::max<size_t>(r.n, 1) * r.Jp));
  }
  if (count && !r.tbits)
    r.tbits = as<uint32_t>(arena_.get("r" + std::to_string(tau) + ".tbits",
                                      (std::max<size_t>(r.n, 1) * r.W32 + 31) / 32 * 4 + 4));
  launch_simulate(r, jacobi, jacobi ? count : 0, cap, nullptr, 0, stream_);
  RankCtl c{};
  DFS_CUDA(cudaMemcpyAsync(&c, r.ctl, sizeof c, cudaMemcpyDeviceToHost, stream_));
  sync();
  if (c.error) {
    int zero = 0;
    DFS_CUDA(cudaMemcpy(&r.ctl->error, &zero, sizeof zero, cudaMemcpyHostToDevice));
    return -1;
  }
  return int(c.sweeps);
}

void Context::stage_scores(uint32_t tau, double* out) {
  check_tau(tau, ranks_.size());
  launch_score(ranks_[tau], 1, nullptr, 0, stream_);
  DFS_CUDA(cudaMemcpyAsync(out, ranks_[tau].scores, size_t(g_.n) * 8, cudaMemcpyDeviceToHost,
                           stream_));
  sync();
}

uint64_t Context::stage_commit_cascade(uint32_t tau, uint32_t seed) {
  check_tau(tau, ranks_.size());
  if (seed >= g_.n) throw Error(kIndex, "seed id out of range");
  launch_cascade(ranks_[tau], nullptr, seed, stream_);
  sync();
  return stage_visited(tau);
}

uint64_t Context::stage_visited(uint32_t tau) {
  check_tau(tau, ranks_.size());
  RankCtl c{};
  DFS_CUDA(cudaMemcpy(&c, ranks_[tau].ctl, sizeof c, cudaMemcpyDeviceToHost));
  return c.visited;
}

void Context::stage_counters(uint32_t tau, uint64_t out[8]) {
  check_tau(tau, ranks_.size());
  RankCtl c{};
  DFS_CUDA(cudaMemcpy(&c, ranks_[tau].ctl, sizeof c, cudaMemcpyDeviceToHost));
  const uint64_t v[8] = {c.updates,     c.items_processed, c.cnt_edges,        c.cnt_batches,
                         c.cnt_touched, c.cnt_sweeps,      c.cnt_convergences, c.visited};
  for (int i = 0; i < 8; ++i) out[i] = v[i];
}

void Context::stage_scores_device(uint32_t tau, int full, double* dst) {
  check_tau(tau, ranks_.size());
  launch_score(ranks_[tau], full, nullptr, 0, stream_);
  if (dst)
    DFS_CUDA(cudaMemcpyAsync(dst, ranks_[tau].scores, size_t(g_.n) * 8, cudaMemcpyDeviceToDevice,
                             stream_));
  sync();
}

void Context::stage_rebuild(uint32_t tau) {
  check_tau(tau, ranks_.size());
  launch_fill(ranks_[tau], nullptr, 0, stream_);
  launch_simulate(ranks_[tau], cfg_.jacobi, 0, cfg_.sim_cap, nullptr, 0, stream_);
  launch_score(ranks_[tau], 1, nullptr, 0, stream_);
  RankCtl c{};
  DFS_CUDA(cudaMemcpyAsync(&c, ranks_[tau].ctl, sizeof c, cudaMemcpyDeviceToHost, stream_));
  sync();
  if (c.error)
    throw Error(kRuntime, "simulate did not converge within " + std::to_string(cfg_.sim_cap) +
                              " iterations; register monotonicity must be broken");
}

// Registers are stored on the device as value + 1 per byte (VISITED -1 -> 0,
// DESIGN.md §2); the stage API speaks the reference's int8 values.
void Context::stage_get_registers(uint32_t tau, int8_t* out) {
  check_tau(tau, ranks_.size());
  const RankDev& r = ranks_[tau];
  if (!r.n) return;
  DFS_CUDA(cudaMemcpy2DAsync(out, r.J, r.regs, r.Jp, r.J, r.n, cudaMemcpyDeviceToHost, stream_));
  sync();
  const size_t total = size_t(r.n) * r.J;
  for (size_t i = 0; i < total; ++i) out[i] = int8_t(uint8_t(out[i]) - 1u);
}

// VISITED bitset in the reference layout (sketch.hpp:35-87): per row ceil(J/64)
// u64 words; the device mirror holds W32 = Jp/32 u32 words per row (pads 0).
void Context::stage_get_visited(uint32_t tau, uint64_t* out) {
  check_tau(tau, ranks_.size());
  const RankDev& r = ranks_[tau];
  if (!r.n) return;
  std::vector<uint32_t> v(size_t(r.n) * r.W32);
  DFS_CUDA(cudaMemcpyAsync(v.data(), r.vis, v.size() * 4, cudaMemcpyDeviceToHost, stream_));
  sync();
  const uint32_t words = (r.J + 63) / 64;
  for (size_t u = 0; u < r.n; ++u)
    for (uint32_t w = 0; w < words; ++w) {
      const uint64_t lo = v[u * r.W32 + 2 * w];
      const uint64_t hi = 2 * w + 1 < r.W32 ? v[u * r.W32 + 2 * w + 1] : 0;
      out[u * words + w] = lo | (hi << 32);
    }
}

void Context::stage_set_registers(uint32_t tau, const int8_t* in) {
  check_tau(tau, ranks_.size());
  RankDev& r = ranks_[tau];
  if (!r.n) return;
  // registers + the VISITED bitset mirror + running count (sketch.hpp:35-87)
  std::vector<int8_t> full(size_t(r.n) * r.Jp, int8_t(0));  // stored value + 1: pads VISITED
  std::vector<uint32_t> vis(size_t(r.n) * r.W32, 0);
  uint64_t visited = 0;
  for (uint32_t u = 0; u < r.n; ++u)
    for (uint32_t j = 0; j < r.J; ++j) {
      const int8_t v = in[size_t(u) * r.J + j];
      full[size_t(u) * r.Jp + j] = int8_t(uint8_t(v) + 1u);
      if (v == -1) {
        vis[size_t(u) * r.W32 + j / 32] |= 1u << (j % 32);
        ++visited;
      }
    }
  DFS_CUDA(cudaMemcpy(r.regs, full.data(), full.size(), cudaMemcpyHostToDevice));
  DFS_CUDA(cudaMemcpy(r.vis, vis.data(), vis.size() * 4, cudaMemcpyHostToDevice));
  DFS_CUDA(cudaMemcpy(&r.ctl->visited, &visited, 8, cudaMemcpyHostToDevice));
}

// Reference layout of the device graph (engine.hpp:14-29): CSR of the edges
// live in >= 1 local simulation plus u64 liveness masks, rebuilt on the host
// from the forward items (edges appear as consecutive items of their row).
void Context::stage_device_graph(uint32_t tau, std::vector<uint64_t>& off,
                                 std::vector<uint32_t>& adj, std::vector<uint64_t>& mask,
                                 uint32_t* words_out) {
  check_tau(tau, ranks_.size());
  const RankDev& r = ranks_[tau];
  const Items& it = r.fwd;
  const uint32_t words = (r.J + 63) / 64;
  std::vector<uint64_t> roff(size_t(r.n) + 1);
  std::vector<uint32_t> other(it.count), mk(it.count);
  std::vector<uint8_t> b(it.count);
  DFS_CUDA(cudaMemcpy(roff.data(), it.row_off, roff.size() * 8, cudaMemcpyDeviceToHost));
  if (it.count) {
    DFS_CUDA(cudaMemcpy(other.data(), it.other, it.count * 4, cudaMemcpyDeviceToHost));
    DFS_CUDA(cudaMemcpy(mk.data(), it.mask, it.count * 4, cudaMemcpyDeviceToHost));
    DFS_CUDA(cudaMemcpy(b.data(), it.batch, it.count, cudaMemcpyDeviceToHost));
  }
  off.assign(size_t(r.n) + 1, 0);
  adj.clear();
  mask.clear();
  for (uint32_t u = 0; u < r.n; ++u) {
    off[u] = adj.size();
    for (uint64_t i = roff[u]; i < roff[u + 1]; ++i) {
      if (i == roff[u] || other[i] != other[i - 1]) {
        adj.push_back(other[i]);
        mask.resize(mask.size() + words, 0);
      }
      const uint32_t j0 = uint32_t(b[i]) * 32;
      uint64_t* mw = mask.data() + mask.size() - words;
      mw[j0 / 64] |= uint64_t(mk[i]) << (j0 % 64);
    }
  }
  off[r.n] = adj.size();
  *words_out = words;
}

}  // namespace dfs
