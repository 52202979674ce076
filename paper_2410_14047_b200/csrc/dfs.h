// dfs.h — internal declarations shared by the host runtime (runtime.cpp) and
// the sm_100a kernels (kernels.cu).  Not part of the public C-ABI
// (include/difuser_b200.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace dfs {

// Status codes of the C-ABI; mapped to the reference's exception classes by
// the Python mirror (std::invalid_argument -> ValueError, runtime_error ->
// RuntimeError, see proj/bindings/pymodule.cpp and SURVEY.md §8(b)).
enum Status : int {
  kOk = 0,
  kInvalid = 1,   // std::invalid_argument
  kRuntime = 2,   // std::runtime_error
  kCuda = 3,      // CUDA failure (RuntimeError)
  kNoMem = 4,     // allocation failure (MemoryError)
  kIndex = 5,     // out-of-range (IndexError)
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);
#define DFS_CUDA(x) ::dfs::cuda_check((x), #x)

// Simulations are grouped in 32-sim batches (one u32 of live/visited bits).
constexpr uint32_t kBatch = 32;
// Items per work chunk: a warp owns one chunk (4 passes of 32 lanes).
constexpr uint32_t kChunk = 128;
// Items::big entries carry this flag when the chunk is its row's only chunk
// (the processing warp owns the row: plain stores instead of CAS).
constexpr uint32_t kBigOwner = 0x80000000u;

// ---------------------------------------------------------------- device views
// Full weighted graph, resident for the context (CSR by source u, plus its
// transpose by target v).  ehash/in_degree are computed on the device.
struct DevGraph {
  uint32_t n = 0;
  uint64_t m = 0;
  uint64_t* off = nullptr;    // n+1
  uint32_t* adj = nullptr;    // m   (target v of edge e)
  uint32_t* src = nullptr;    // m   (source u of edge e)
  uint32_t* ehash = nullptr;  // m
  uint32_t* indeg = nullptr;  // n
  uint64_t* toff = nullptr;   // n+1 (transpose offsets by v)
  uint32_t* tedge = nullptr;  // m   (edge ids sorted by (v, e))
  uint32_t* tsrc = nullptr;   // m   transposed order: source u of position p
  uint32_t* thash = nullptr;  // m   transposed order: edge hash
  uint32_t* tdst = nullptr;   // m   transposed order: target v (row)
};

// One direction of the sampled ("device") graph as sparse 32-sim items:
// item i of row r = (other endpoint, live mask over batch b).  Rows are split
// into chunks of <= kChunk items; chunk c covers items [cbeg[c], cbeg[c+1]).
struct Items {
  uint64_t count = 0;
  uint64_t chunks = 0;
  uint64_t* row_off = nullptr;     // n+1 item offsets per row
  uint32_t* row = nullptr;         // count (row of each item: flat full-pass sweeps)
  uint32_t* other = nullptr;       // count
  uint32_t* mask = nullptr;        // count
  uint8_t* batch = nullptr;        // count
  uint32_t* chunk_row = nullptr;   // chunks
  uint64_t* chunk_beg = nullptr;   // chunks+1
  uint32_t* row_chunk = nullptr;   // n+1 first chunk of each row
  // chunk ids split by row size: rows with <= kSmallRow items (one chunk,
  // processed item-parallel) and larger rows (processed warp-per-chunk pull)
  uint32_t* small = nullptr;
  uint32_t* big = nullptr;    // chunk id | kBigOwner
  uint32_t nsmall = 0, nbig = 0;
  // flat list of the item indices of small rows (flat full passes)
  uint32_t* small_items = nullptr;
  uint64_t nsmall_items = 0;
  uint64_t live = 0;  // live (item, simulation) pairs (host copy; fwd only)
};
#ifndef DFS_SMALL_ROW
#define DFS_SMALL_ROW 32
#endif
constexpr uint32_t kSmallRow = DFS_SMALL_ROW;  // rows with <= kSmallRow items: item-parallel

// Device-resident control block of one rank (sample-space partition tau).
struct RankCtl {
  unsigned long long visited;   // running VISITED register count
  unsigned long long updates;   // live (item, sim) pairs merged (instrumentation)
  unsigned long long items_processed;
  unsigned int tick;            // strictly increasing stamp source
  unsigned int sweeps;          // sweeps of the last simulate
  unsigned int total_sweeps;
  unsigned int levels;          // cascade levels (last)
  int error;                    // 1 = simulate cap exceeded
  unsigned int dirty_count;     // rows to rescore
  unsigned int max_sweeps;      // most sweeps one convergence took (async sim_cap check)
  unsigned int pad[5];
  // reference-schedule work counters (count mode):
  // E edges processed, B live 32-sim batches, T touched (row, batch) pairs
  unsigned long long cnt_edges, cnt_batches, cnt_touched, cnt_sweeps, cnt_convergences;
  // solo-mode hand-back word: (launch tick << 32) | (resume sweep/level << 2) | code
  unsigned long long release;
  // cascade work units of the reference schedule (count mode): frontier rows
  // summed over levels, device-graph edges out of them, cascades started
  unsigned long long cnt_cas_rows, cnt_cas_edges, cnt_cascades;
  // rows this run actually rescored (full passes after fills + dirty rows):
  // the performed score work, next to the reference schedule's K full passes
  unsigned long long rescored_rows;
};

// Work queues used by the persistent simulate / cascade kernels.  Rotating
// generations (simulate: sweep % 3, cascade: level % 4) so that a generation
// can be reset while the next one is being filled without an extra barrier.
constexpr int kGens = 4;
struct Queues {
  uint32_t* chunks[kGens];      // chunk ids to process
  uint32_t* rows[kGens];        // rows (deduplicated) of that generation
  unsigned int* counts;         // [0..3] chunk counts, [4..7] row counts, [8..11] work counters
};

struct RankDev {
  uint32_t n = 0, J = 0, Jp = 0, W32 = 0, tau = 0;
  uint32_t j_offset = 0;
  uint64_t reg_key = 0;
  uint32_t* x = nullptr;          // Jp sorted slice values (pads 0xFFFFFFFF)
  uint32_t* xlut = nullptr;       // 4097: first slot with x >= k << 19 (FASST windows)
  uint64_t* jkey = nullptr;       // Jp register hash keys
  int8_t* regs = nullptr;         // n*Jp
  int8_t* snap = nullptr;         // n*Jp (Jacobi schedule only)
  int8_t* pristine = nullptr;     // n*Jp cached first fill (rebuilds copy it), optional
  uint32_t* vis = nullptr;        // n*W32 visited bitset
  uint32_t* fresh[3] = {nullptr, nullptr, nullptr};  // n*W32 cascade frontier bits
  uint32_t* lstamp = nullptr;     // n  queue-membership stamps
  uint32_t* dstamp = nullptr;     // n  dirty-row stamps
  unsigned long long* cstamp = nullptr;  // n  cascade: (round << 32) | level stamp
  uint32_t* dirty = nullptr;      // n  rows to rescore
  uint32_t* tbits = nullptr;      // n*W32 bits: touched (row, batch) of a sweep (count mode)
  double* scores = nullptr;       // n
  RankCtl* ctl = nullptr;
  Queues q{};
  Items fwd, rev;                 // cascade uses fwd (by u), simulate uses rev (by v)
};

// Run-level control block (single device copy, written by the round kernels).
struct RunCtl {
  unsigned int step;
  unsigned int choice;
  unsigned int saturated;
  unsigned int rebuild_now;
  unsigned int n_rebuilds;
  unsigned int argmax_done;       // last-block counter of the argmax
  unsigned int snap_dirty;        // dirty rows left by the last cascade (all partitions)
  unsigned int pad;
  double oldscore;
  // Parked-grid rounds (one partition, no peers): blocks other than block 0
  // wait on park_seq while block 0 runs rounds alone; block 0 wakes them with
  // (reason, round, stamp base) when a round needs the grid.
  unsigned int park_seq, park_reason, park_step, park_base;
};

struct RunArrays {
  RunCtl* ctl = nullptr;
  uint8_t* committed = nullptr;   // n
  uint32_t* seeds = nullptr;      // k
  double* traj = nullptr;         // k
  uint32_t* rebuild_rounds = nullptr;  // k
  double* reduced = nullptr;      // n (tree-summed scores, mu > 1)
  double* blk_score = nullptr;    // argmax partials
  uint32_t* blk_arg = nullptr;
  uint32_t* blk_min = nullptr;
  uint32_t nblk = 0;
  // Argmax cache (one local partition): best positive uncommitted (score,
  // id) and smallest uncommitted id of every kSeg-row segment; only segments
  // holding rescored rows are recomputed each round.
  double* seg_score = nullptr;
  uint32_t* seg_arg = nullptr;
  uint32_t* seg_min = nullptr;
  uint32_t* seg_stamp = nullptr;
  uint32_t nseg = 0;
};
constexpr uint32_t kSeg = 1024;

// ---------------------------------------------------------------- peer mode
// Multi-GPU: one FASST partition per GPU (one process, or one context, per
// GPU).  The per-round exchange of proj/src/runtime.cpp:88-130 (partial score
// reduce in binomial order, argmax, seed broadcast, covered-count allreduce)
// runs INSIDE the persistent k_run kernel over peer memory (NVLink P2P loads
// of mapped peer buffers, CUDA IPC across processes) with flag barriers; the
// host is not involved between rounds.
constexpr uint32_t kMaxPeers = 16;

// Mailbox of one rank in its own HBM; peers read it through a mapping.
struct alignas(128) PeerBox {
  unsigned long long arrive;   // last barrier epoch this rank reached (monotonic)
  unsigned long long visited;  // this rank's VISITED count after the round's cascade
  double best_s;               // best positive uncommitted reduced score of the slice
  unsigned int best_v;         // its id (0xFFFFFFFF: none)
  unsigned int minu;           // smallest uncommitted id of the slice (0xFFFFFFFF: none)
  unsigned long long timeouts; // barriers abandoned after the deadline (peer died)
  unsigned int ndirty;         // rows this rank rescored this round (kAllDirty: all)
  unsigned int pad0;
  unsigned long long pad[10];
};
constexpr unsigned int kAllDirty = 0xFFFFFFFFu;

struct PeerView {
  uint32_t world = 0, rank = 0;
  PeerBox* box[kMaxPeers] = {};          // box[t]: rank t's mailbox (own one for t == rank)
  const double* scores[kMaxPeers] = {};  // rank t's partial score vector (n doubles)
  const uint32_t* dirty[kMaxPeers] = {}; // rank t's rescored rows of the round
  unsigned long long timeout_ns = 120ull * 1000 * 1000 * 1000;  // a barrier's patience
};

// ---------------------------------------------------------------- launchers
// Graph preparation (once per upload): src, ehash, in-degree, transpose.
size_t graph_prepare_tmp_bytes(uint64_t m, uint32_t n);
void launch_graph_prepare(DevGraph& g, void* tmp, size_t tmp_bytes, cudaStream_t s);
// Weights: kind 0 = const (W), 1 = wc (from in-degree).  Other kinds are
// computed on the host (std::mt19937_64) and uploaded.
void launch_weights(const DevGraph& g, int kind, uint32_t W, uint32_t* w, cudaStream_t s);
// Exclusive scan u32 -> u64 (out has n+1 entries; out[n] = total).
size_t scan_tmp_bytes(uint64_t n);
void scan_u32_u64(const uint32_t* in, uint64_t* out, uint64_t n, void* tmp, size_t tmp_bytes,
                  cudaStream_t s);
// Sampled-item construction for one rank and direction (dir 0 = by source u
// over the CSR, dir 1 = by target v over the transpose).  write = 0 counts
// items per edge position into cnt; write = 1 emits them at pos_off.
// Reverse-direction item counts per transposed position, gathered from the
// forward item offsets (an edge has the same items in both directions).
void launch_rev_counts(const DevGraph& g, const uint64_t* pos_f, uint32_t* cnt, cudaStream_t s);
void launch_items_pass(const DevGraph& g, const uint32_t* w, const uint32_t* tw, const RankDev& r,
                       int dir, int fasst, int write, uint32_t* cnt, const uint64_t* pos_off,
                       Items& it, cudaStream_t s);
// Weights in transposed order (kind 0 const, 1 wc, 2 gather of w).
void launch_tweights(const DevGraph& g, int kind, uint32_t W, const uint32_t* w, uint32_t* tw,
                     cudaStream_t s);
// Slot LUT of a partition (first slot with x >= k << 19, FASST windows).
void launch_xlut(const RankDev& r, cudaStream_t s);
void launch_xlut_of(const uint32_t* x, uint32_t J, uint32_t* lut, cudaStream_t s);
// Monte-Carlo influence (oracle.cpp:30-79) of batches [batch0, batch0+nbatch)
// of 32 trials: live masks (nbatch*m), BFS scratch (vis nbatch*n, fresh and
// queue nbatch*2n), reached counts (nbatch*32).
void launch_mc_influence(const DevGraph& g, const uint32_t* w, uint64_t base, uint32_t trials,
                         uint64_t total, uint64_t batch0, uint32_t nbatch, const uint32_t* seeds,
                         uint32_t nseeds, uint32_t* live, uint32_t* vis, uint32_t* fresh,
                         uint32_t* queue, uint32_t* reached, cudaStream_t s);
// FASST analytics (fasst.cpp:101-168): out = [dup counts 0..mu | loads | live
// lanes | batches] (2 mu + 3 u64).
void launch_fasst_stats(const DevGraph& g, const uint32_t* w, const uint32_t* x,
                        const uint32_t* xlut, uint32_t R, uint32_t mu, int sorted, int fill,
                        unsigned long long* out, cudaStream_t s);
// One-pass sampled-item build of one direction (count + scan + write in one
// launch with a decoupled look-back; writes it.row_off too).  wconst != 0:
// every edge has that fixed-point weight (w/tw unused).  Items beyond `cap`
// are dropped (the host re-runs with the exact total, meta[0]); meta[1] +=
// live (item, simulation) pairs.  tile_state: items_tiles(m) zeroed words,
// tile_ctr zeroed.  row_cnt != nullptr (FASST multi-partition plans): positions
// whose window misses the partition's value range are skipped and per-row item
// counts accumulate in row_cnt (n+1 zeroed entries) instead of it.row_off
// (the caller scans them).
uint64_t items_tiles(uint64_t npos);
void launch_items_onepass(const DevGraph& g, const uint32_t* w, const uint32_t* tw,
                          uint32_t wconst, const RankDev& r, int dir, int fasst, Items& it,
                          uint64_t cap, unsigned long long* tile_state, unsigned int* tile_ctr,
                          unsigned long long* meta, uint32_t* row_cnt, cudaStream_t s);
// meta[0] += items of every stride-th forward position (capacity estimate).
void launch_items_sample(const DevGraph& g, const uint32_t* w, uint32_t wconst, const RankDev& r,
                         int fasst, uint64_t stride, unsigned long long* meta, cudaStream_t s);
// row_cnt[r] = chunks of row r (from it.row_off).
void launch_row_chunks(uint32_t n, const Items& it, uint32_t* row_cnt, cudaStream_t s);
// row_off[r] = pos_off[graph row start]; then per-row chunk counts.
void launch_row_offsets(const DevGraph& g, int dir, const uint64_t* pos_off, Items& it,
                        uint32_t* row_cnt, cudaStream_t s);
void launch_chunk_write(uint32_t n, Items& it, const uint64_t* row_chunk64, cudaStream_t s);
// Split chunk ids into it.small / it.big (counts written to cnt2[0..1]); the
// chunk count is read on the device (*chunks_dev), chunks_cap bounds it.
void launch_split_chunks(Items& it, const uint64_t* chunks_dev, uint64_t chunks_cap,
                         unsigned int* cnt2, cudaStream_t s);
// it.small_items <- item indices of the chunks in it.small (count *nsmall_dev
// on the device; total items written to *cnt).
void launch_small_items(Items& it, const unsigned int* nsmall_dev, uint64_t chunks_cap,
                        unsigned long long* cnt, cudaStream_t s);
// Fill registers (VISITED kept, pads VISITED).  gate: run only if *gate == want.
void launch_fill(const RankDev& r, const unsigned int* gate, unsigned int want, cudaStream_t s,
                 bool use_pristine = false);
// Persistent cooperative simulate to convergence.  jacobi != 0 reproduces the
// reference's snapshot schedule exactly (same sweep count); count != 0 (with
// jacobi) also tallies the reference-schedule work units E/B/T/L.
void launch_simulate(const RankDev& r, int jacobi, int count, int cap, const unsigned int* gate,
                     unsigned int want, cudaStream_t s);
// Number of kernels this library launched (all launchers), for gpu_launches.
unsigned long long launches();
void dump_trace();  // debug (DFS_DBG bit 2)
// Row scores: full = all rows, else the dirty list of the last cascade.
void launch_score(const RankDev& r, int full, const unsigned int* gate, unsigned int want,
                  cudaStream_t s);
void launch_treesum(const double* const* parts_dev, uint32_t mu, uint32_t n, double* out,
                    cudaStream_t s);
void launch_argmax(const double* scores, RunArrays& ra, uint32_t n, cudaStream_t s);
// Commit of *choice (or of `seed` when choice == nullptr) + full cascade.
void launch_cascade(const RankDev& r, const unsigned int* choice, uint32_t seed,
                    cudaStream_t s);
void launch_round_end(RunArrays& ra, RankCtl* const* ctls_dev, uint32_t mu, uint32_t k,
                      uint32_t r, double eps, cudaStream_t s);
int coop_grid(int which, int variant = 0);  // 0 simulate, 1 cascade, 2 whole run
// The whole greedy loop (after the build phase) as one persistent kernel.
void launch_run(const RankDev* ranks_dev, uint32_t mu, uint32_t k, uint32_t R, uint32_t n,
                double eps, int cap, int jacobi, int count, int K, RunArrays& ra,
                const double* const* parts, RankCtl* const* ctls, double* reduced,
                unsigned long long* phase_ns, const PeerView* peer, int grid_share,
                int sim_pull_f, int cas_pull_f, cudaStream_t s);
// *out += live (item, simulation) pairs of `count` masks.
void launch_popc_sum(const uint32_t* mask, uint64_t count, unsigned long long* out,
                     cudaStream_t s);

}  // namespace dfs
