// kernels.cu — sm_100a kernels of the sketch-IM hot path.
//
// Memory-bound integer work throughout (byte max-merge, xor/compare sampling,
// bitset BFS): no tensor cores.  The design points:
//  * sampling is never materialised as dense masks (the reference bakes
//    m_tau x ceil(J/64) words, proj/src/fasst.cpp:72-82); instead each edge is
//    expanded once per run into sparse 32-sim "items" (other endpoint, live
//    mask, batch) — only batches where the edge is live in >= 1 simulation.
//    With FASST-sorted x values the live simulations of an edge form one
//    contiguous window, found by two binary searches;
//  * simulate is a persistent cooperative kernel: push-style (source row v to
//    all u with a live edge u->v), in place, lock-free byte-max via 64-bit
//    CAS, frontier of changed rows between sweeps, one grid barrier per sweep;
//  * the cascade (coverage removal) is a persistent level-synchronous bitset
//    BFS over the forward items; the score is bit-exact via an integer sum.
#include <cooperative_groups.h>
#include <cooperative_groups/scan.h>
#include <cub/cub.cuh>
#include <cuda/std/functional>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "dfs.h"
#include "hash.cuh"

namespace cg = cooperative_groups;

namespace dfs {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(e == cudaErrorMemoryAllocation ? kNoMem : kCuda,
                std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + what);
}

// Debug trace (DFS_DBG bit 2): (kind, index, frontier, clock) records written
// by block 0 thread 0; dumped by dump_trace().  Not used on the timed path.
__device__ unsigned long long g_trace[8192][4];
__device__ unsigned int g_trace_n;

namespace {

__device__ __forceinline__ void trace(unsigned long long kind, unsigned long long idx,
                                      unsigned long long nc) {
  const unsigned k = atomicAdd(&g_trace_n, 1u);
  if (k < 8192) {
    g_trace[k][0] = kind;
    g_trace[k][1] = idx;
    g_trace[k][2] = nc;
    g_trace[k][3] = clock64();
  }
}

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    DFS_CUDA(cudaGetDevice(&dev));
    DFS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

int grid_for(uint64_t work, int per_block = kThreads) {
  uint64_t b = (work + per_block - 1) / per_block;
  uint64_t cap = uint64_t(num_sms()) * 16;
  if (b > cap) b = cap;
  return b ? int(b) : 1;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }

template <class T>
__device__ __forceinline__ T ld_volatile(const T* p) {
  return *reinterpret_cast<const volatile T*>(p);
}

// ---------------------------------------------------------------- graph prep
__global__ void k_src(uint32_t n, const uint64_t* __restrict__ off, uint32_t* __restrict__ src) {
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t u = warp; u < n; u += nw)
    for (uint64_t e = off[u] + lane_id(); e < off[u + 1]; e += 32) src[e] = uint32_t(u);
}

__global__ void k_ehash(uint64_t m, const uint32_t* __restrict__ src,
                        const uint32_t* __restrict__ adj, uint32_t* __restrict__ ehash,
                        uint32_t* __restrict__ iota) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x) {
    ehash[e] = edge_hash(src[e], adj[e]);  // graph.cpp:180, on dense ids
    iota[e] = uint32_t(e);
  }
}

// In-degrees from the sorted targets instead of one atomic per edge (R-MAT
// hubs serialise those): the last position of each target's run records the
// run end; an inclusive max-scan of the ends gives toff[1..n].
__global__ void k_run_ends(uint64_t m, const uint32_t* __restrict__ tdst,
                           uint32_t* __restrict__ ends) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t v = tdst[i];
    if (i + 1 == m || tdst[i + 1] != v) ends[v] = uint32_t(i + 1);
  }
}

__global__ void k_indeg(uint32_t n, const uint64_t* __restrict__ toff,
                        uint32_t* __restrict__ indeg) {
  for (uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x)
    indeg[v] = uint32_t(toff[v + 1] - toff[v]);
}

struct MaxU64 {
  __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const {
    return a > b ? a : b;
  }
};

// ---------------------------------------------------------------- weights
// graph.cpp:30-35 + :250-258: W = llround(w * 2^31), wc w = 1/indeg(v).
__global__ void k_weights(uint64_t m, int kind, uint32_t W, const uint32_t* __restrict__ adj,
                          const uint32_t* __restrict__ indeg, uint32_t* __restrict__ w) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x) {
    if (kind == 0) {
      w[e] = W;
    } else {
      const double p = __ddiv_rn(1.0, double(indeg[adj[e]]));
      w[e] = uint32_t(llround(__dmul_rn(p, 2147483648.0)));
    }
  }
}

// ---------------------------------------------------------------- items
// Live window of an edge in the sorted slice: (x ^ h) < W implies x agrees
// with h on all bits above floor(log2 W), i.e. x lies in one aligned block of
// size 2^(floor(log2 W)+1) around h; sorted order turns
// that block into the contiguous slot range [lo, hi).
constexpr int kLutBits = 12;                 // slot LUT over the top 12 bits of x
constexpr int kLutShift = 31 - kLutBits;     // 2^19-wide x buckets

__device__ __forceinline__ uint32_t lower_bound_x(const uint32_t* sx, uint32_t J, uint64_t key) {
  uint32_t a = 0, z = J;
  while (a < z) {
    const uint32_t mid = (a + z) >> 1;
    if (uint64_t(sx[mid]) < key) a = mid + 1; else z = mid;
  }
  return a;
}

__device__ __forceinline__ uint32_t lower_bound_in(const uint32_t* sx, uint32_t a, uint32_t z,
                                                   uint64_t key) {
  while (a < z) {
    const uint32_t mid = (a + z) >> 1;
    if (uint64_t(sx[mid]) < key) a = mid + 1; else z = mid;
  }
  return a;
}

// Window [lo, hi) plus its all-live half [alo, ahi): inside the block, bit b
// of x splits the sorted window in two; where it equals bit b of h, x ^ h <
// 2^b <= W, so every slot of that half samples the edge without a test (the
// other half still needs (x ^ h) < W).  Naive plans: the whole slice, tested.
__device__ __forceinline__ void edge_window(const uint32_t* sx, const uint32_t* lut, uint32_t J,
                                            uint32_t h, uint32_t W, int fasst, uint32_t& lo,
                                            uint32_t& hi, uint32_t& alo, uint32_t& ahi) {
  if (!fasst) {
    lo = 0;
    hi = J;
    alo = ahi = 0;
    return;
  }
  const int b = 31 - __clz(W);  // W >= 1
  const uint64_t half = uint64_t(1) << b;
  const uint64_t span = half << 1;
  const uint64_t lx = uint64_t(h) & ~(span - 1);
  const uint64_t hx = lx + span;  // exclusive
  const uint64_t mx = lx + half;  // first value with bit b set
  if (b + 1 >= kLutShift) {       // block boundaries are LUT bucket boundaries: exact
    lo = lut[lx >> kLutShift];
    hi = (hx >> kLutShift) > (1u << kLutBits) ? J : lut[hx >> kLutShift];
  } else {
    lo = lower_bound_x(sx, J, lx);
    hi = lower_bound_x(sx, J, hx);
  }
  const uint32_t mid = b >= kLutShift ? lut[mx >> kLutShift] : lower_bound_in(sx, lo, hi, mx);
  if ((h >> b) & 1u) {
    alo = mid;
    ahi = hi;
  } else {
    alo = lo;
    ahi = mid;
  }
}

// dir 0: positions = CSR edges (row = src u, other = adj v)
// dir 1: positions = transpose (edge = tedge[p], row = adj v, other = src u)
// Positions are edges in CSR order (dir 0: row = source u, other = target v)
// or in transposed order (dir 1: row = v, other = u); every input array is
// indexed by position, so both directions stream coalesced.
template <int WRITE>
__global__ void k_items(uint64_t npos, const uint32_t* __restrict__ p_hash,
                        const uint32_t* __restrict__ p_w, const uint32_t* __restrict__ p_other,
                        const uint32_t* __restrict__ p_row, const uint32_t* __restrict__ x,
                        uint32_t J, uint32_t Jp, int fasst, uint32_t* __restrict__ cnt,
                        const uint64_t* __restrict__ pos_off, uint32_t* __restrict__ it_other,
                        uint32_t* __restrict__ it_mask, uint8_t* __restrict__ it_batch,
                        uint32_t* __restrict__ it_row, const uint32_t* __restrict__ glut) {
  extern __shared__ __align__(16) uint32_t sx[];
  uint32_t* lut = sx + Jp;  // lut[k] = lower_bound(x, k << kLutShift), k in [0, 2^kLutBits]
  for (uint32_t i = threadIdx.x; i < Jp; i += blockDim.x) sx[i] = x[i];
  __syncthreads();
  if (fasst)
    for (uint32_t k = threadIdx.x; k <= (1u << kLutBits); k += blockDim.x) lut[k] = glut[k];
  __syncthreads();
  for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < npos;
       p += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t W = p_w[p];
    uint32_t c = 0;
    if (W != 0) {  // fasst.cpp:71 — W = 0 never samples
      const uint32_t h = p_hash[p];
      uint32_t lo, hi, alo, ahi;
      edge_window(sx, lut, J, h, W, fasst, lo, hi, alo, ahi);
      if (hi > lo) {
        uint64_t o = WRITE ? pos_off[p] : 0;
        const uint32_t other = WRITE ? p_other[p] : 0;
        const uint32_t rowv = WRITE ? p_row[p] : 0;
        for (uint32_t b = lo >> 5; b <= (hi - 1) >> 5; ++b) {
          const uint32_t bb = b * 32;
          const uint32_t i0 = max(lo, bb), i1 = min(hi, bb + 32);
          // all-live half: a contiguous run of bits, no test
          const uint32_t a0 = max(alo, i0), a1 = min(ahi, i1);
          uint32_t mk = 0;
          if (a1 > a0)
            mk = (a1 - a0 == 32 ? 0xFFFFFFFFu : ((1u << (a1 - a0)) - 1u)) << (a0 - bb);
          // the other half (one range, [alo, ahi) being a prefix or suffix of
          // the window) is tested with aligned 4-slot vector loads; a group's
          // slots outside the window fail on their own and slots of the live
          // half pass, so no masking is needed (sampling.hpp:37-39)
          const uint32_t t0 = alo == lo ? max(i0, ahi) : i0;
          const uint32_t t1 = alo == lo ? i1 : min(i1, alo);
          for (uint32_t g = t0 & ~3u; g < t1; g += 4) {
            const uint4 xv = *reinterpret_cast<const uint4*>(sx + g);
            const uint32_t m4 = uint32_t((xv.x ^ h) < W) | (uint32_t((xv.y ^ h) < W) << 1) |
                                (uint32_t((xv.z ^ h) < W) << 2) | (uint32_t((xv.w ^ h) < W) << 3);
            mk |= m4 << (g - bb);
          }
          if (mk) {
            if (WRITE) {
              it_other[o] = other;
              it_row[o] = rowv;
              it_mask[o] = mk;
              it_batch[o] = uint8_t(b);
              ++o;
            }
            ++c;
          }
        }
      }
    }
    if (!WRITE) cnt[p] = c;
  }
}

// ---- one-pass item build (count, scan and write in a single launch) --------
// Positions are processed in tiles of kTileThreads x kPosPerThread consecutive
// positions.  A thread evaluates the sampling windows of its 8 positions once
// and keeps the masks of the first two batches of each window in registers
// (IC windows rarely cover more); the block scans the per-thread item counts,
// obtains the tile's global item offset by a decoupled look-back over the
// tile status words, and writes the items in position order (= the order of
// the count/scan/write formulation, fasst.cpp:50-88 CSR order).  The first
// position of every row also writes that row's item offset (row_off), so no
// per-position count or offset array exists.  Windows spanning more than two
// batches are re-evaluated in the write phase.
constexpr int kTileThreads = 256;
constexpr int kPosPerThread = 8;
constexpr uint32_t kTilePos = kTileThreads * kPosPerThread;
constexpr unsigned long long kStAgg = 1ull << 62, kStInc = 2ull << 62,
                             kStVal = (1ull << 62) - 1;

// Mask of batch b of an edge's window (the live-half bit range plus tested
// slots; sampling.hpp:37-39).
__device__ __forceinline__ uint32_t window_batch_mask(const uint32_t* sx, uint32_t h, uint32_t W,
                                                      uint32_t lo, uint32_t hi, uint32_t alo,
                                                      uint32_t ahi, uint32_t b) {
  const uint32_t bb = b * 32;
  const uint32_t i0 = max(lo, bb), i1 = min(hi, bb + 32);
  const uint32_t a0 = max(alo, i0), a1 = min(ahi, i1);
  uint32_t mk = 0;
  if (a1 > a0) mk = (a1 - a0 == 32 ? 0xFFFFFFFFu : ((1u << (a1 - a0)) - 1u)) << (a0 - bb);
  const uint32_t t0 = alo == lo ? max(i0, ahi) : i0;
  const uint32_t t1 = alo == lo ? i1 : min(i1, alo);
  for (uint32_t g = t0 & ~3u; g < t1; g += 4) {
    const uint4 xv = *reinterpret_cast<const uint4*>(sx + g);
    const uint32_t m4 = uint32_t((xv.x ^ h) < W) | (uint32_t((xv.y ^ h) < W) << 1) |
                        (uint32_t((xv.z ^ h) < W) << 2) | (uint32_t((xv.w ^ h) < W) << 3);
    mk |= m4 << (g - bb);
  }
  return mk;
}

struct ItemsPass {
  uint64_t npos;
  uint32_t n;                // rows (row_off has n+1 entries)
  const uint32_t* p_hash;
  const uint32_t* p_w;       // nullptr: constant weight Wc
  uint32_t Wc;
  const uint32_t* p_other;
  const uint32_t* p_row;
  const uint32_t* x;
  const uint32_t* glut;
  uint32_t J, Jp;
  int fasst;
  uint64_t cap;              // item capacity (writes beyond it are dropped; host re-runs)
  uint32_t* it_other;
  uint32_t* it_mask;
  uint8_t* it_batch;
  uint32_t* it_row;
  uint64_t* row_off;
  uint32_t* row_cnt;               // FILTER: per-row item counts (row offsets scanned after)
  unsigned long long* tile_state;  // per tile: flag (2 bits) | value
  unsigned int* tile_ctr;          // dynamic tile ids (look-back forward progress)
  unsigned long long* meta;        // [0] total items, [1] live (item, sim) pairs
};

// Look-back of a tile whose aggregate is already published: sums the
// predecessors back to the nearest published inclusive prefix (block-wide,
// 256 predecessors per step), publishes this tile's inclusive prefix and
// leaves the exclusive prefix in s_prefix (valid after the final barrier).
__device__ __forceinline__ void lookback_resolve(unsigned long long* st, uint64_t tile,
                                                 uint32_t tile_total,
                                                 unsigned long long& s_prefix,
                                                 unsigned long long& s_lb_sum,
                                                 unsigned int& s_lb_first) {
  if (threadIdx.x == 0) s_lb_sum = 0;
  unsigned long long prefix = 0;
  for (int64_t base = int64_t(tile) - 1; base >= 0; base -= kTileThreads) {
    const int64_t t = base - int64_t(threadIdx.x);
    unsigned long long v = kStInc;
    if (t >= 0)
      do {
        v = ld_volatile(st + t);
      } while ((v >> 62) == 0);
    if (threadIdx.x == 0) s_lb_first = kTileThreads;
    __syncthreads();
    if ((v >> 62) == 2) atomicMin(&s_lb_first, unsigned(threadIdx.x));
    __syncthreads();
    const unsigned first = s_lb_first;
    unsigned long long val = threadIdx.x <= first ? (v & kStVal) : 0ull;
    for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
    if (lane_id() == 0 && val) atomicAdd(&s_lb_sum, val);
    __syncthreads();
    prefix = s_lb_sum;
    if (first < kTileThreads) break;
  }
  if (threadIdx.x == 0) {
    if (tile) __stcg(st + tile, kStInc | (prefix + tile_total));
    s_prefix = prefix;
  }
  __syncthreads();
}

// Partition-sparse variant of the one-pass build (FASST multi-partition
// plans): a tile's positions whose window block misses the partition's
// slot-value range (≈ 1 - 1/mu of them) are dropped right after their
// hash/weight load, the rest are compacted (in position order, warp ballots)
// into a shared-memory list, and the windows and the scan run over that dense
// list with every lane busy.  Row offsets come from per-row item counts
// (segmented warp sums, one atomic per row segment) scanned after the pass.
//
// Tiles are taken round-robin (tile = block + k * grid) and each tile's
// item writes are DEFERRED by one tile: after tile t's windows and scan the
// block publishes t's aggregate, then resolves the look-back of its previous
// tile (whose predecessors have long published theirs) and writes that
// tile's items, and keeps t's lists for the next round (a tile listing more
// than kPendCap positions is resolved and written at once).  Without the
// deferral, a tile's look-back waited for the slowest tile of its wave (39%
// of the stall samples).  The next tile's hashes/weights are loaded while the
// current one is processed.
constexpr int kSparseCap = kTilePos;  // list capacity = every position of a tile
constexpr int kPendCap = 512;         // deferred list capacity
constexpr int kTileWarps = kTileThreads / 32;

// Items and per-row counts of one tile's list (positions t0 + idx[j]).
__device__ __forceinline__ void sparse_write(const ItemsPass& a, const uint32_t* sx,
                                             const uint32_t* lut, uint64_t t0, uint32_t nrel,
                                             const uint16_t* idx, const uint32_t* info_l,
                                             const uint32_t* la, const uint32_t* lb,
                                             const uint32_t* loff, const uint32_t* lrow,
                                             unsigned long long prefix) {
  for (uint32_t j0 = (threadIdx.x & ~31u); j0 < nrel; j0 += kTileThreads) {
    const uint32_t j = j0 + lane_id();
    const bool in = j < nrel;
    const uint32_t info = in ? info_l[j] : 0u;
    const uint32_t c = info & 0xFFFFu;
    const uint64_t p = t0 + (in ? idx[j] : 0u);
    const uint32_t row = c ? lrow[j] : 0xFFFFFFFFu;
    const uint32_t other = c ? a.p_other[p] : 0u;  // in flight during the segmented sum
    // segmented inclusive sum of c over runs of equal rows (head-flag scan)
    const uint32_t rprev = __shfl_up_sync(0xffffffffu, row, 1);
    uint32_t sum = c, head = (lane_id() == 0 || rprev != row) ? 1u : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t up = __shfl_up_sync(0xffffffffu, sum, o);
      const uint32_t fup = __shfl_up_sync(0xffffffffu, head, o);
      if (lane_id() >= unsigned(o)) {
        if (!head) sum += up;
        head |= fup;
      }
    }
    const uint32_t rnext = __shfl_down_sync(0xffffffffu, row, 1);
    const bool seg_end = lane_id() == 31 || rnext != row;
    if (c && seg_end) atomicAdd(a.row_cnt + row, sum);
    if (!c) continue;
    uint64_t o = prefix + loff[j];
    const uint32_t b0 = info >> 24, nb = (info >> 16) & 0xFFu;
    auto emit = [&](uint32_t b, uint32_t mk) {
      if (!mk) return;
      if (o < a.cap) {
        a.it_other[o] = other;
        a.it_row[o] = row;
        a.it_mask[o] = mk;
        a.it_batch[o] = uint8_t(b);
      }
      ++o;
    };
    emit(b0, la[j]);
    if (nb >= 2) emit(b0 + 1, lb[j]);
    if (nb > 2) {
      const uint32_t W = a.p_w ? a.p_w[p] : a.Wc, h = a.p_hash[p];
      uint32_t lo, hi, alo, ahi;
      edge_window(sx, lut, a.J, h, W, 1, lo, hi, alo, ahi);
      for (uint32_t b = b0 + 2; b <= (hi - 1) >> 5; ++b)
        emit(b, window_batch_mask(sx, h, W, lo, hi, alo, ahi, b));
    }
  }
}

size_t sparse_extra_smem() {
  return size_t(kSparseCap + 5 * kPendCap) * sizeof(uint32_t) + size_t(kPendCap) * sizeof(uint16_t);
}

__global__ void __launch_bounds__(kTileThreads, 3) k_items_sparse(ItemsPass a) {
  extern __shared__ __align__(16) uint32_t sx[];
  uint32_t* lut = sx + a.Jp;
  uint32_t* l_row = lut + (1u << kLutBits) + 1;  // kSparseCap
  uint32_t* q_info = l_row + kSparseCap;          // deferred tile: kPendCap each
  uint32_t* q_a = q_info + kPendCap;
  uint32_t* q_b = q_a + kPendCap;
  uint32_t* q_off = q_b + kPendCap;
  uint32_t* q_row = q_off + kPendCap;
  uint16_t* q_idx = reinterpret_cast<uint16_t*>(q_row + kPendCap);
  using BlockScan = cub::BlockScan<uint32_t, kTileThreads>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  __shared__ uint16_t l_idx[kSparseCap];  // tile-relative position
  __shared__ uint32_t l_info[kSparseCap], l_a[kSparseCap], l_b[kSparseCap], l_off[kSparseCap];
  __shared__ uint32_t s_wcnt[kPosPerThread * kTileWarps];
  __shared__ unsigned long long s_prefix, s_lb_sum;
  __shared__ unsigned int s_lb_first, s_nrel;
  for (uint32_t i = threadIdx.x; i < a.Jp; i += blockDim.x) sx[i] = a.x[i];
  for (uint32_t k = threadIdx.x; k <= (1u << kLutBits); k += blockDim.x) lut[k] = a.glut[k];
  const uint64_t ntiles = (a.npos + kTilePos - 1) / kTilePos;
  __syncthreads();
  const uint64_t xmin = sx[0], xmax = sx[a.J - 1];
  const unsigned lane = lane_id(), wi = threadIdx.x >> 5;
  uint32_t ph[kPosPerThread], pw[kPosPerThread];
  auto prefetch = [&](uint64_t t) {
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i) {
      const uint64_t p = t * kTilePos + uint64_t(i) * kTileThreads + threadIdx.x;
      const bool ok = t < ntiles && p < a.npos;
      pw[i] = ok ? (a.p_w ? __ldcs(a.p_w + p) : a.Wc) : 0u;
      ph[i] = ok ? __ldcs(a.p_hash + p) : 0u;
    }
  };
  // resolve the look-back of tile t and write its items from the given lists
  auto finish_tile = [&](uint64_t t, uint32_t total, uint32_t n, const uint16_t* idx,
                         const uint32_t* info_l, const uint32_t* la, const uint32_t* lb,
                         const uint32_t* loff, const uint32_t* lrow) {
    lookback_resolve(a.tile_state, t, total, s_prefix, s_lb_sum, s_lb_first);
    const unsigned long long prefix = s_prefix;
    if (threadIdx.x == 0 && t + 1 == ntiles) a.meta[0] = prefix + total;
    sparse_write(a, sx, lut, t * kTilePos, n, idx, info_l, la, lb, loff, lrow, prefix);
    __syncthreads();  // lists / s_prefix reusable
  };
  constexpr uint64_t kNone = ~0ull;
  uint64_t pend = kNone;
  uint32_t pend_total = 0, pend_n = 0;
  prefetch(blockIdx.x);
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t t0 = tile * kTilePos;
    // ---- A: relevance of the tile's positions (striped, coalesced loads)
    uint32_t rel[kPosPerThread];
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i) {
      const uint32_t W = pw[i], h = ph[i];
      rel[i] = 0;
      if (W != 0) {  // fasst.cpp:71; the window block must meet [x_0, x_{J-1}]
        const uint64_t span = uint64_t(2) << (31 - __clz(W));
        const uint64_t lx = uint64_t(h) & ~(span - 1);
        rel[i] = (lx + span > xmin && lx <= xmax) ? 1u : 0u;
      }
    }
    prefetch(tile + gridDim.x);
    // compaction in position order: (step i, warp, lane) is position order
    unsigned bal[kPosPerThread];
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i) bal[i] = __ballot_sync(0xffffffffu, rel[i] != 0);
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < kPosPerThread; ++i) s_wcnt[i * kTileWarps + wi] = __popc(bal[i]);
    __syncthreads();
    if (wi == 0) {  // exclusive scan of the 64 (step, warp) counts, two per lane
      const uint32_t c0 = s_wcnt[2 * lane], c1 = s_wcnt[2 * lane + 1];
      uint32_t incl = c0 + c1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= unsigned(o)) incl += t;
      }
      const uint32_t ex = incl - c0 - c1;
      s_wcnt[2 * lane] = ex;
      s_wcnt[2 * lane + 1] = ex + c0;
      if (lane == 31) s_nrel = incl;
    }
    __syncthreads();
    const unsigned below = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i)
      if (rel[i])
        l_idx[s_wcnt[i * kTileWarps + wi] + __popc(bal[i] & below)] =
            uint16_t(i * kTileThreads + threadIdx.x);
    const uint32_t nrel = s_nrel;
    __syncthreads();
    // ---- B: windows of the listed positions (dense)
    uint32_t live = 0;
    for (uint32_t j = threadIdx.x; j < nrel; j += kTileThreads) {
      const uint64_t p = t0 + l_idx[j];
      const uint32_t W = a.p_w ? a.p_w[p] : a.Wc, h = a.p_hash[p];
      // row of the listed position: loaded here, in flight while the window
      // is evaluated (the write phase reads it from shared memory)
      const uint32_t prow = a.p_row[p];
      uint32_t lo, hi, alo, ahi, info = 0, mA = 0, mB = 0;
      edge_window(sx, lut, a.J, h, W, 1, lo, hi, alo, ahi);
      if (hi > lo) {
        const uint32_t b0 = lo >> 5, b1 = (hi - 1) >> 5, nb = b1 - b0 + 1;
        uint32_t c = 0;
        for (uint32_t b = b0; b <= b1; ++b) {
          const uint32_t mk = window_batch_mask(sx, h, W, lo, hi, alo, ahi, b);
          if (b == b0) mA = mk;
          else if (b == b0 + 1) mB = mk;
          c += mk != 0;
          live += __popc(mk);
        }
        info = (b0 << 24) | (min(nb, 255u) << 16) | c;
      }
      l_info[j] = info;
      l_a[j] = mA;
      l_b[j] = mB;
      l_row[j] = prow;
    }
    __syncthreads();
    // ---- C: item offsets in list (= position) order; publish the aggregate
    uint32_t c8[kPosPerThread];
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i) {
      const uint32_t j = threadIdx.x * kPosPerThread + i;  // blocked
      c8[i] = j < nrel ? (l_info[j] & 0xFFFFu) : 0u;
    }
    uint32_t tile_total;
    BlockScan(scan_tmp).ExclusiveSum(c8, c8, tile_total);
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i) {
      const uint32_t j = threadIdx.x * kPosPerThread + i;
      if (j < nrel) l_off[j] = c8[i];
    }
    if (threadIdx.x == 0) __stcg(a.tile_state + tile, (tile == 0 ? kStInc : kStAgg) | tile_total);
    for (int o = 16; o; o >>= 1) live += __shfl_xor_sync(0xffffffffu, live, o);
    if (lane == 0 && live) atomicAdd(&a.meta[1], (unsigned long long)live);
    __syncthreads();
    // ---- D: the previous tile's items, then defer this one
    if (pend != kNone)
      finish_tile(pend, pend_total, pend_n, q_idx, q_info, q_a, q_b, q_off, q_row);
    if (nrel <= uint32_t(kPendCap)) {
      for (uint32_t j = threadIdx.x; j < nrel; j += kTileThreads) {
        q_idx[j] = l_idx[j];
        q_info[j] = l_info[j];
        q_a[j] = l_a[j];
        q_b[j] = l_b[j];
        q_off[j] = l_off[j];
        q_row[j] = l_row[j];
      }
      pend = tile;
      pend_total = tile_total;
      pend_n = nrel;
      __syncthreads();
    } else {
      finish_tile(tile, tile_total, nrel, l_idx, l_info, l_a, l_b, l_off, l_row);
      pend = kNone;
    }
  }
  if (pend != kNone) finish_tile(pend, pend_total, pend_n, q_idx, q_info, q_a, q_b, q_off, q_row);
}

// One-pass build of one direction (one partition per context, or a naive
// plan): persistent blocks take 2048-position tiles round-robin (tile =
// block + k * grid); a thread evaluates the windows of its 8 striped
// positions once, the tile's counts are scanned in position order, and the
// tile's aggregate is published at once.  The item and row-offset writes are
// DEFERRED by one tile (per-position masks, counts, offsets and rows parked
// in shared memory): the block resolves the look-back of its previous tile
// -- whose predecessors published long ago -- and writes it while the next
// tile is in flight, instead of waiting for the slowest tile of the wave.
constexpr uint32_t kDeferWords = 5 * kTilePos;  // deferred tile: mA, mB, info, offset, row

// MINB blocks per SM: 3 for constant weights (one narrow window per edge:
// C2 build 1.24 -> 1.10 ms, north star 7.9 -> 7.15 ms), 2 for per-edge weights
// (wide weighted-cascade windows need the registers: C3 58 -> 62 ms at 3).
template <int MINB>
__global__ void __launch_bounds__(kTileThreads, MINB) k_items_onepass(ItemsPass a) {
  extern __shared__ __align__(16) uint32_t sx[];
  uint32_t* lut = sx + a.Jp;
  uint32_t* d_a = lut + (1u << kLutBits) + 1;  // striped position index i * 256 + tid
  uint32_t* d_b = d_a + kTilePos;
  uint32_t* d_info = d_b + kTilePos;  // b0 << 24 | nb << 16 | count
  uint32_t* d_off = d_info + kTilePos;
  uint32_t* d_row = d_off + kTilePos;
  using BlockScan = cub::BlockScan<uint32_t, kTileThreads>;
  using BlockExch = cub::BlockExchange<uint32_t, kTileThreads, kPosPerThread>;
  __shared__ union {
    typename BlockScan::TempStorage scan;
    typename BlockExch::TempStorage exch;
  } tmp;
  __shared__ unsigned long long s_prefix, s_lb_sum;
  __shared__ unsigned int s_lb_first;
  for (uint32_t i = threadIdx.x; i < a.Jp; i += blockDim.x) sx[i] = a.x[i];
  if (a.fasst)
    for (uint32_t k = threadIdx.x; k <= (1u << kLutBits); k += blockDim.x) lut[k] = a.glut[k];
  const uint64_t ntiles = (a.npos + kTilePos - 1) / kTilePos;
  __syncthreads();
  // look-back of tile t (aggregate already published), then its writes
  auto finish_tile = [&](uint64_t t, uint32_t total) {
    lookback_resolve(a.tile_state, t, total, s_prefix, s_lb_sum, s_lb_first);
    const unsigned long long prefix = s_prefix;
    if (threadIdx.x == 0 && t + 1 == ntiles) a.meta[0] = prefix + total;
    const uint64_t pbase = t * kTilePos + threadIdx.x;
    uint32_t othv[kPosPerThread];
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i) {  // every position's other endpoint in flight
      const uint32_t k = i * kTileThreads + threadIdx.x;
      const uint64_t p = pbase + uint64_t(i) * kTileThreads;
      othv[i] = (p < a.npos && (d_info[k] & 0xFFFFu)) ? __ldcs(a.p_other + p) : 0u;
    }
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i) {
      const uint32_t k = i * kTileThreads + threadIdx.x;
      const uint64_t p = pbase + uint64_t(i) * kTileThreads;
      if (p >= a.npos) continue;
      const uint32_t row = d_row[k], info = d_info[k], c = info & 0xFFFFu;
      uint64_t o = prefix + d_off[k];
      // rows (prev_row, row] start at this position (rows without edges share it)
      const uint32_t prev = k ? d_row[k - 1] : (p ? __ldcs(a.p_row + p - 1) : 0xFFFFFFFFu);
      for (uint32_t r = prev + 1; r <= row; ++r) a.row_off[r] = o;
      if (p + 1 == a.npos)  // rows after the last edge's row end at the total
        for (uint32_t r = row + 1; r <= a.n; ++r) a.row_off[r] = o + c;
      if (!c) continue;
      const uint32_t other = othv[i];
      const uint32_t b0 = info >> 24, nb = (info >> 16) & 0xFFu;
      auto emit = [&](uint32_t b, uint32_t mk) {
        if (!mk) return;
        if (o < a.cap) {
          a.it_other[o] = other;
          a.it_row[o] = row;
          a.it_mask[o] = mk;
          a.it_batch[o] = uint8_t(b);
        }
        ++o;
      };
      emit(b0, d_a[k]);
      if (nb >= 2) emit(b0 + 1, d_b[k]);
      if (nb > 2) {  // wide window: re-evaluate the remaining batches
        const uint32_t h = a.p_hash[p], W = a.p_w ? a.p_w[p] : a.Wc;
        uint32_t lo, hi, alo, ahi;
        edge_window(sx, lut, a.J, h, W, a.fasst, lo, hi, alo, ahi);
        for (uint32_t b = b0 + 2; b <= (hi - 1) >> 5; ++b)
          emit(b, window_batch_mask(sx, h, W, lo, hi, alo, ahi, b));
      }
    }
    __syncthreads();  // deferred buffers reusable
  };
  constexpr uint64_t kNone = ~0ull;
  uint64_t pend = kNone;
  uint32_t pend_total = 0;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // striped positions: step i covers kTileThreads consecutive positions
    // (coalesced loads, and consecutive lanes write consecutive items)
    const uint64_t pbase = tile * kTilePos + threadIdx.x;
    // ---- phase 1: windows, counts, masks of the first two batches
    uint32_t mA[kPosPerThread], mB[kPosPerThread], info[kPosPerThread];
    uint32_t cnt[kPosPerThread];
    uint32_t live = 0;
    // every position's hash and weight in flight together
    uint32_t hv[kPosPerThread], wv[kPosPerThread];
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i) {
      const uint64_t p = pbase + uint64_t(i) * kTileThreads;
      const bool ok = p < a.npos;
      wv[i] = ok ? (a.p_w ? __ldcs(a.p_w + p) : a.Wc) : 0u;
      hv[i] = ok ? __ldcs(a.p_hash + p) : 0u;
    }
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i) {
      mA[i] = mB[i] = 0;
      info[i] = 0;
      cnt[i] = 0;
      const uint32_t W = wv[i], h = hv[i];
      if (W == 0) continue;  // fasst.cpp:71 (and past the end)
      uint32_t lo, hi, alo, ahi;
      edge_window(sx, lut, a.J, h, W, a.fasst, lo, hi, alo, ahi);
      if (hi <= lo) continue;
      const uint32_t b0 = lo >> 5, b1 = (hi - 1) >> 5, nb = b1 - b0 + 1;
      uint32_t c = 0;
      for (uint32_t b = b0; b <= b1; ++b) {
        const uint32_t mk = window_batch_mask(sx, h, W, lo, hi, alo, ahi, b);
        if (b == b0) mA[i] = mk;
        else if (b == b0 + 1) mB[i] = mk;
        c += mk != 0;
        live += __popc(mk);
      }
      info[i] = (b0 << 24) | (min(nb, 255u) << 16) | c;
      cnt[i] = c;
    }
    // rows of all 8 positions in flight while the tile is scanned
    uint32_t rowv[kPosPerThread];
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i) {
      const uint64_t p = pbase + uint64_t(i) * kTileThreads;
      rowv[i] = p < a.npos ? __ldcs(a.p_row + p) : 0u;
    }
    // ---- tile scan in position order (striped -> blocked -> striped)
    BlockExch(tmp.exch).StripedToBlocked(cnt);
    __syncthreads();
    uint32_t tile_total;
    BlockScan(tmp.scan).ExclusiveSum(cnt, cnt, tile_total);
    __syncthreads();
    BlockExch(tmp.exch).BlockedToStriped(cnt);
    if (threadIdx.x == 0) __stcg(a.tile_state + tile, (tile == 0 ? kStInc : kStAgg) | tile_total);
    for (int o = 16; o; o >>= 1) live += __shfl_xor_sync(0xffffffffu, live, o);
    if (lane_id() == 0 && live) atomicAdd(&a.meta[1], (unsigned long long)live);
    __syncthreads();
    // ---- the previous tile's writes, then park this one
    if (pend != kNone) finish_tile(pend, pend_total);
#pragma unroll
    for (int i = 0; i < kPosPerThread; ++i) {
      const uint32_t k = i * kTileThreads + threadIdx.x;
      d_a[k] = mA[i];
      d_b[k] = mB[i];
      d_info[k] = info[i];
      d_off[k] = cnt[i];
      d_row[k] = rowv[i];
    }
    pend = tile;
    pend_total = tile_total;
    __syncthreads();
  }
  if (pend != kNone) finish_tile(pend, pend_total);
}

// Item count of every stride-th position (capacity estimate of a one-pass
// build: the exact total is known only when the pass ends).
__global__ void k_items_sample(ItemsPass a, uint64_t stride) {
  extern __shared__ __align__(16) uint32_t sx[];
  uint32_t* lut = sx + a.Jp;
  for (uint32_t i = threadIdx.x; i < a.Jp; i += blockDim.x) sx[i] = a.x[i];
  if (a.fasst)
    for (uint32_t k = threadIdx.x; k <= (1u << kLutBits); k += blockDim.x) lut[k] = a.glut[k];
  __syncthreads();
  unsigned long long c = 0;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k * stride < a.npos;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t p = k * stride;
    const uint32_t W = a.p_w ? a.p_w[p] : a.Wc, h = a.p_hash[p];
    if (W == 0) continue;
    uint32_t lo, hi, alo, ahi;
    edge_window(sx, lut, a.J, h, W, a.fasst, lo, hi, alo, ahi);
    if (hi <= lo) continue;
    for (uint32_t b = lo >> 5; b <= (hi - 1) >> 5; ++b)
      c += window_batch_mask(sx, h, W, lo, hi, alo, ahi, b) != 0;
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane_id() == 0 && c) atomicAdd(&a.meta[0], c);
}

// Per-row chunk counts from the row item offsets.
__global__ void k_row_chunks(uint32_t n, const uint64_t* __restrict__ row_off,
                             uint32_t* __restrict__ row_cnt) {
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x)
    row_cnt[r] = uint32_t((row_off[r + 1] - row_off[r] + kChunk - 1) / kChunk);
}

// Transposed position p holds edge tedge[p], whose item count is its forward
// count (the sampling test depends on (edge hash, weight, slot) only): one
// gather instead of re-evaluating the windows.  cnt[m] = 0 closes the scan.
__global__ void k_rev_counts(uint64_t m, const uint32_t* __restrict__ tedge,
                             const uint64_t* __restrict__ pos_f, uint32_t* __restrict__ cnt) {
  for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p <= m;
       p += uint64_t(gridDim.x) * blockDim.x) {
    if (p == m) {
      cnt[m] = 0;
      continue;
    }
    const uint32_t e = tedge[p];
    cnt[p] = uint32_t(pos_f[e + 1] - pos_f[e]);
  }
}

// Slot LUT: lut[k] = first slot with x >= k << kLutShift (sorted slices).
__global__ void k_xlut(const uint32_t* __restrict__ x, uint32_t J, uint32_t* __restrict__ lut) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k <= (1u << kLutBits);
       k += gridDim.x * blockDim.x)
    lut[k] = lower_bound_x(x, J, uint64_t(k) << kLutShift);
}

// Transposed position p holds edge tedge[p]; its target is the sort key
// (tdst, written by the sort), its source one gather, and its hash is
// recomputed (hash.hpp:91-93) instead of gathered.
__global__ void k_transpose_fields(uint64_t m, const uint32_t* __restrict__ tedge,
                                   const uint32_t* __restrict__ src,
                                   const uint32_t* __restrict__ tdst, uint32_t* __restrict__ tsrc,
                                   uint32_t* __restrict__ thash) {
  for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < m;
       p += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t u = src[tedge[p]];
    tsrc[p] = u;
    thash[p] = edge_hash(u, tdst[p]);
  }
}

// Weights in transposed order: const / wc from the target's in-degree, or a
// gather of host-assigned weights.
__global__ void k_tweights(uint64_t m, const uint32_t* __restrict__ tedge,
                           const uint32_t* __restrict__ tdst, int kind, uint32_t W,
                           const uint32_t* __restrict__ indeg, const uint32_t* __restrict__ w,
                           uint32_t* __restrict__ tw) {
  for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < m;
       p += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t wv = W;
    if (kind == 1)
      wv = uint32_t(llround(__dmul_rn(__ddiv_rn(1.0, double(indeg[tdst[p]])), 2147483648.0)));
    else if (kind == 2)
      wv = w[tedge[p]];
    tw[p] = wv;
  }
}

__global__ void k_row_offsets(uint32_t n, const uint64_t* __restrict__ graph_off,
                              const uint64_t* __restrict__ pos_off, uint64_t* __restrict__ row_off,
                              uint32_t* __restrict__ row_cnt) {
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r <= n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    row_off[r] = pos_off[graph_off[r]];
    if (r < n) {
      const uint64_t items = pos_off[graph_off[r + 1]] - pos_off[graph_off[r]];
      row_cnt[r] = uint32_t((items + kChunk - 1) / kChunk);
    }
  }
}

__global__ void k_chunk_write(uint32_t n, const uint64_t* __restrict__ row_chunk64,
                              const uint64_t* __restrict__ row_off, uint32_t* __restrict__ row_chunk,
                              uint32_t* __restrict__ chunk_row, uint64_t* __restrict__ chunk_beg) {
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r <= n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t c0 = row_chunk64[r];
    row_chunk[r] = uint32_t(c0);
    if (r == n) {
      chunk_beg[c0] = row_off[n];  // total items
      continue;
    }
    const uint64_t c1 = row_chunk64[r + 1];
    for (uint64_t c = c0; c < c1; ++c) {
      chunk_row[c] = uint32_t(r);
      chunk_beg[c] = row_off[r] + (c - c0) * kChunk;
    }
  }
}

// Chunk count read on the device (no host round trip during the build).
__global__ void k_split_chunks(const uint64_t* __restrict__ chunks_dev,
                               const uint32_t* __restrict__ chunk_row,
                               const uint64_t* __restrict__ row_off, uint32_t* __restrict__ small,
                               uint32_t* __restrict__ big, unsigned int* cnt2) {
  const uint64_t chunks = *chunks_dev;
  for (uint64_t c0 = uint64_t(blockIdx.x) * blockDim.x; c0 < chunks;
       c0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t c = c0 + threadIdx.x;
    bool isb = false, single = false, valid = c < chunks;
    if (valid) {
      const uint32_t r = chunk_row[c];
      const uint64_t items = row_off[r + 1] - row_off[r];
      isb = items > kSmallRow;
      single = items <= kChunk;  // the row is this one chunk: its warp owns the row
    }
    const unsigned mb = __ballot_sync(0xffffffffu, valid && isb);
    const unsigned ms = __ballot_sync(0xffffffffu, valid && !isb);
    unsigned bb = 0, bs = 0;
    if (lane_id() == 0) {
      if (mb) bb = atomicAdd(&cnt2[1], __popc(mb));
      if (ms) bs = atomicAdd(&cnt2[0], __popc(ms));
    }
    bb = __shfl_sync(0xffffffffu, bb, 0);
    bs = __shfl_sync(0xffffffffu, bs, 0);
    const unsigned below = (1u << lane_id()) - 1;
    if (valid && isb) big[bb + __popc(mb & below)] = uint32_t(c) | (single ? kBigOwner : 0u);
    if (valid && !isb) small[bs + __popc(ms & below)] = uint32_t(c);
  }
}

// Item indices of small chunks (each small row is one chunk of <= kSmallRow
// items): warp per 32 chunks, warp-aggregated append keeps rows contiguous.
__global__ void k_small_items(const unsigned int* __restrict__ nsmall_dev,
                              const uint32_t* __restrict__ small,
                              const uint64_t* __restrict__ chunk_beg, uint32_t* __restrict__ out,
                              unsigned long long* cnt) {
  const uint32_t nsmall = *nsmall_dev;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t k0 = ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32; k0 < nsmall;
       k0 += nw * 32) {
    const uint64_t k = k0 + lane_id();
    uint64_t beg = 0;
    uint32_t len = 0;
    if (k < nsmall) {
      const uint32_t c = small[k];
      beg = chunk_beg[c];
      len = uint32_t(chunk_beg[c + 1] - beg);
    }
    uint32_t incl = len;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane_id() >= unsigned(o)) incl += t;
    }
    unsigned long long base = 0;
    if (lane_id() == 31) base = atomicAdd(cnt, (unsigned long long)incl);
    base = __shfl_sync(0xffffffffu, base, 31);
    const uint64_t o = base + incl - len;
    for (uint32_t j = 0; j < len; ++j) out[o + j] = uint32_t(beg + j);
  }
}

// ---------------------------------------------------------------- FASST analytics
// duplication_stats / device_edge_loads / fill_rate of proj/src/fasst.cpp:
// 101-168 in one pass over the edges.  x: the plan's slot values (sorted for
// FASST, generation order for naive; chunk tau = slots [tau*J, (tau+1)*J)),
// which is also the order fill_rate batches X in.  Sorted slots use the live
// window of each edge; naive plans test every slot.  Counters are exact
// integers (block-shared, one global atomic per counter per block).
// out: [0, mu] duplication counts, [mu+1, 2mu] loads, [2mu+1] live lanes,
// [2mu+2] counted batches.
__global__ void k_fasst_stats(uint64_t m, const uint32_t* __restrict__ ehash,
                              const uint32_t* __restrict__ w, const uint32_t* __restrict__ x,
                              const uint32_t* __restrict__ glut, uint32_t R, uint32_t mu,
                              int sorted, int fill, unsigned long long* out) {
  extern __shared__ uint32_t sx[];
  uint32_t* lut = sx + R;
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(lut + (1u << kLutBits) + 2);
  const uint32_t ncnt = 2 * mu + 3;
  for (uint32_t i = threadIdx.x; i < R; i += blockDim.x) sx[i] = x[i];
  if (sorted)
    for (uint32_t k = threadIdx.x; k <= (1u << kLutBits); k += blockDim.x) lut[k] = glut[k];
  for (uint32_t i = threadIdx.x; i < ncnt; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const uint32_t J = R / mu;
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < m;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t W = w[e];
    if (W == 0) {  // fasst.cpp:107-109: never sampled, k = 0
      atomicAdd(&cnt[0], 1ull);
      continue;
    }
    const uint32_t h = ehash[e];
    uint32_t lo = 0, hi = R, alo, ahi;
    if (sorted) edge_window(sx, lut, R, h, W, 1, lo, hi, alo, ahi);
    unsigned long long hits = 0;  // chunks sampling e (mu <= 64)
    uint32_t bc = 0, cur_b = lo >> 5;
    unsigned long long lanes = 0, batches = 0;
    for (uint32_t i = lo; i < hi; ++i) {
      if ((i >> 5) != cur_b) {
        if (bc) {
          lanes += bc;
          ++batches;
        }
        bc = 0;
        cur_b = i >> 5;
      }
      if ((sx[i] ^ h) < W) {  // sampling.hpp:37-39
        hits |= 1ull << (i / J);
        ++bc;
      }
    }
    if (bc) {
      lanes += bc;
      ++batches;
    }
    atomicAdd(&cnt[__popcll(hits)], 1ull);
    for (unsigned long long t = hits; t; t &= t - 1) atomicAdd(&cnt[mu + 1 + __ffsll(t) - 1], 1ull);
    if (fill && batches) {
      atomicAdd(&cnt[2 * mu + 1], lanes);
      atomicAdd(&cnt[2 * mu + 2], batches);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < ncnt; i += blockDim.x)
    if (cnt[i]) atomicAdd(&out[i], cnt[i]);
}

// ---------------------------------------------------------------- MC influence
// Monte-Carlo oracle of proj/src/oracle.cpp:30-79 on the GPU, bit-identical:
// trial i = (run, t) draws the liveness of every edge in edge order from its
// own std::mt19937_64(trial_seed) — (rng() >> 33) < W[e] — then counts the
// vertices reachable from the seeds over live edges.  32 trials form a batch:
// phase 1 (k_mc_live) runs 32 generators side by side in one block (one warp
// per trial, the 312-word twist split over the warp's lanes) and writes one
// 32-trial live mask per edge (a ballot transpose of the per-trial bits);
// phase 2 (k_mc_bfs) is a bitset BFS of the 32 trials together, one block per
// batch.  The per-trial reached counts go to the host, which accumulates the
// mean / standard error in the reference's trial order (the double sums there
// are not all exact, so the order matters).
constexpr int kMtN = 312, kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull, kMtUpper = 0xFFFFFFFF80000000ull,
                   kMtLower = 0x7FFFFFFFull;

__device__ __forceinline__ uint64_t mt_mix(uint64_t hi_src, uint64_t lo_src) {
  const uint64_t y = (hi_src & kMtUpper) | (lo_src & kMtLower);
  return (y >> 1) ^ ((y & 1) ? kMtA : 0ull);
}
__device__ __forceinline__ uint64_t mt_temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}
// libstdc++ _M_gen_rand: the three segments in order; each lane reads its
// inputs before the warp writes (in-place update).
__device__ __forceinline__ void mt_twist(uint64_t* mt, unsigned lane) {
  for (int k0 = 0; k0 < kMtN - kMtM; k0 += 32) {
    const int k = k0 + lane;
    uint64_t v = 0;
    if (k < kMtN - kMtM) v = mt[k + kMtM] ^ mt_mix(mt[k], mt[k + 1]);
    __syncwarp();
    if (k < kMtN - kMtM) mt[k] = v;
    __syncwarp();
  }
  for (int k0 = kMtN - kMtM; k0 < kMtN - 1; k0 += 32) {
    const int k = k0 + lane;
    uint64_t v = 0;
    if (k < kMtN - 1) v = mt[k + kMtM - kMtN] ^ mt_mix(mt[k], mt[k + 1]);
    __syncwarp();
    if (k < kMtN - 1) mt[k] = v;
    __syncwarp();
  }
  if (lane == 0) mt[kMtN - 1] = mt[kMtM - 1] ^ mt_mix(mt[kMtN - 1], mt[0]);
  __syncwarp();
}

struct McArgs {
  uint64_t m;
  const uint32_t* w;
  uint64_t base;       // derive_seed(seed, kSeedTagOracle)
  uint32_t trials;     // per run
  uint64_t total;      // trials * runs
  uint64_t batch0;     // first batch of this launch
  uint32_t nbatch;     // batches in this launch
  uint32_t* live;      // nbatch * m masks
};

// One block (32 warps) per batch; warp t runs trial 32*batch + t.
constexpr size_t kMcLiveSmem = 32 * kMtN * 8 + 32 * (kMtN / 32 + 1) * 4;
__global__ void __launch_bounds__(1024, 1) k_mc_live(McArgs a) {
  extern __shared__ uint64_t mc_smem[];
  uint64_t (*mt)[kMtN] = reinterpret_cast<uint64_t (*)[kMtN]>(mc_smem);
  uint32_t (*bits)[kMtN / 32 + 1] =
      reinterpret_cast<uint32_t (*)[kMtN / 32 + 1]>(mc_smem + 32 * kMtN);
  const unsigned lane = threadIdx.x & 31, wt = threadIdx.x >> 5;
  for (uint32_t bb = blockIdx.x; bb < a.nbatch; bb += gridDim.x) {
    const uint64_t trial = (a.batch0 + bb) * 32 + wt;
    const bool real = trial < a.total;
    uint64_t* st = mt[wt];
    if (lane == 0) {  // std::mt19937_64(seed): sequential initialisation
      const uint64_t run = real ? trial / a.trials : 0, t = real ? trial % a.trials : 0;
      uint64_t x = splitmix64_at(splitmix64_at(a.base, run), t);  // oracle.cpp:23-25
      st[0] = x;
      for (int i = 1; i < kMtN; ++i) {
        x = 6364136223846793005ull * (x ^ (x >> 62)) + uint64_t(i);
        st[i] = x;
      }
    }
    __syncwarp();
    uint32_t* out = a.live + uint64_t(bb) * a.m;
    for (uint64_t e0 = 0; e0 < a.m; e0 += kMtN) {
      mt_twist(st, lane);  // every block of 312 draws starts with a twist
      const uint64_t rem = a.m - e0;
      const uint32_t cnt = rem < uint64_t(kMtN) ? uint32_t(rem) : uint32_t(kMtN);
      for (uint32_t c = 0; c * 32 < cnt; ++c) {
        const uint32_t i = c * 32 + lane;
        bool lv = false;
        if (i < cnt && real) lv = uint32_t(mt_temper(st[i]) >> 33) < __ldg(a.w + e0 + i);
        const unsigned word = __ballot_sync(0xffffffffu, lv);
        if (lane == 0) bits[wt][c] = word;
      }
      __syncthreads();
      // transpose: warp c turns the 32 trials' words of edges [32c, 32c+32)
      // into one 32-trial mask per edge
      if (wt * 32 < cnt) {
        const unsigned word = bits[lane][wt];
        unsigned mine = 0;
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
          const unsigned msk = __ballot_sync(0xffffffffu, (word >> j) & 1u);
          if (lane == j) mine = msk;
        }
        if (wt * 32 + lane < cnt) out[e0 + wt * 32 + lane] = mine;
      }
      __syncthreads();
    }
  }
}

struct McBfs {
  uint32_t n;
  const uint64_t* off;
  const uint32_t* adj;
  uint64_t m;
  const uint32_t* live;    // nbatch * m
  const uint32_t* seeds;
  uint32_t nseeds;
  uint32_t nbatch;
  uint32_t* vis;           // nbatch * n
  uint32_t* fresh;         // nbatch * 2n
  uint32_t* queue;         // nbatch * 2n
  uint32_t* reached;       // nbatch * 32
};

// One block per batch: level-synchronous BFS of 32 trials as bitsets.
__global__ void __launch_bounds__(1024, 1) k_mc_bfs(McBfs a) {
  __shared__ unsigned int qn[2];
  __shared__ unsigned int cnt[32];
  for (uint32_t bb = blockIdx.x; bb < a.nbatch; bb += gridDim.x) {
    const uint32_t* live = a.live + uint64_t(bb) * a.m;
    uint32_t* vis = a.vis + uint64_t(bb) * a.n;
    uint32_t* fr[2] = {a.fresh + uint64_t(bb) * 2 * a.n, a.fresh + uint64_t(bb) * 2 * a.n + a.n};
    uint32_t* q[2] = {a.queue + uint64_t(bb) * 2 * a.n, a.queue + uint64_t(bb) * 2 * a.n + a.n};
    for (uint32_t v = threadIdx.x; v < a.n; v += blockDim.x) {
      vis[v] = 0;
      fr[0][v] = 0;
      fr[1][v] = 0;
    }
    if (threadIdx.x < 32) cnt[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
      qn[0] = 0;
      qn[1] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (uint32_t i = 0; i < a.nseeds; ++i) {
        const uint32_t s = a.seeds[i];
        if (!vis[s]) {
          vis[s] = 0xFFFFFFFFu;
          fr[0][s] = 0xFFFFFFFFu;
          q[0][qn[0]++] = s;
        }
      }
    __syncthreads();
    int cur = 0;
    while (qn[cur]) {
      const int nx = cur ^ 1;
      const unsigned len = qn[cur];
      // warp per frontier vertex, lanes over its out-edges
      for (unsigned k = threadIdx.x >> 5; k < len; k += blockDim.x >> 5) {
        const uint32_t u = q[cur][k];
        const uint32_t fu = fr[cur][u];
        for (uint64_t e = a.off[u] + (threadIdx.x & 31); e < a.off[u + 1]; e += 32) {
          const uint32_t c = fu & live[e];
          if (!c) continue;
          const uint32_t v = a.adj[e];
          if (!(c & ~ld_volatile(vis + v))) continue;
          const uint32_t nb = c & ~atomicOr(vis + v, c);
          if (!nb) continue;
          if (atomicOr(fr[nx] + v, nb) == 0) q[nx][atomicAdd(&qn[nx], 1u)] = v;
        }
      }
      __syncthreads();
      for (unsigned k = threadIdx.x; k < len; k += blockDim.x) fr[cur][q[cur][k]] = 0;
      if (threadIdx.x == 0) qn[cur] = 0;
      __syncthreads();
      cur = nx;
    }
    // reached count per trial: ballot transpose of the visited words
    unsigned mine = 0;
    for (uint32_t v0 = (threadIdx.x >> 5) * 32; v0 < a.n; v0 += blockDim.x) {
      const uint32_t v = v0 + (threadIdx.x & 31);
      const uint32_t word = v < a.n ? vis[v] : 0;
#pragma unroll 8
      for (int t = 0; t < 32; ++t) {
        const unsigned c = __popc(__ballot_sync(0xffffffffu, (word >> t) & 1u));
        if ((threadIdx.x & 31) == unsigned(t)) mine += c;
      }
    }
    atomicAdd(&cnt[threadIdx.x & 31], mine);
    __syncthreads();
    if (threadIdx.x < 32) a.reached[uint64_t(bb) * 32 + threadIdx.x] = cnt[threadIdx.x];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- fill
// 4 mask bits -> 4 bytes of 0xFF / 0x00.
__device__ __forceinline__ uint32_t expand4(uint32_t m4) {
  return ((m4 * 0x00204081u) & 0x01010101u) * 0xFFu;
}
// clz64(fmix64(k)) (hash.hpp:9-16) on 32-bit halves with only the words the
// count needs: the final k ^= k >> 33 never moves the leading one (bits
// 31..63 are unchanged by it, and below 2^31 it is the identity), so the count
// is that of the second product, whose high word is hi*Clo + lo*Chi +
// umulhi(lo, Clo); its low word matters only when the high word is zero.
__device__ __forceinline__ uint32_t clz_fmix64(uint64_t k) {
  constexpr uint32_t c1lo = 0xed558ccdu, c1hi = 0xff51afd7u;
  constexpr uint32_t c2lo = 0x1a85ec53u, c2hi = 0xc4ceb9feu;
  uint32_t lo = uint32_t(k), hi = uint32_t(k >> 32);
  lo ^= hi >> 1;                                             // k ^= k >> 33
  const uint32_t lo2 = lo * c1lo;                            // k *= C1
  const uint32_t hi2 = hi * c1lo + lo * c1hi + __umulhi(lo, c1lo);
  const uint32_t lo3 = lo2 ^ (hi2 >> 1);                     // k ^= k >> 33
  const uint32_t hi4 = hi2 * c2lo + lo3 * c2hi + __umulhi(lo3, c2lo);  // (k *= C2) >> 32
  if (__builtin_expect(hi4 != 0, 1)) return uint32_t(__clz(hi4));
  return 32u + uint32_t(__clz(lo3 * c2lo));  // (probability 2^-32)
}

// 64-bit add on the integer ALU (add.cc / addc): written as a + b the
// compiler folds it into the multiply-add pipe (IMAD.WIDE), which the hash's
// multiplies already saturate.
__device__ __forceinline__ uint64_t add64_alu(uint64_t a, uint64_t b) {
  uint32_t lo, hi;
  asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;"
      : "=r"(lo), "=r"(hi)
      : "r"(uint32_t(a)), "r"(uint32_t(a >> 32)), "r"(uint32_t(b)), "r"(uint32_t(b >> 32)));
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// sketch.cpp:55-66: M[u][j] = clz64(fmix64(jkey[j] + u*golden)) unless VISITED.
// One thread per 4 registers (one u32 store, coalesced across the warp).
// use_pristine: registers are the cached first fill with VISITED re-applied
// (fill values depend only on (u, j), so a rebuild need not rehash); else the
// hashes are computed and, when a pristine buffer exists, cached.
__device__ __forceinline__ void fill_body(uint32_t n, uint32_t J, uint32_t Jp,
                                          const uint64_t* __restrict__ jkey,
                                          const uint32_t* __restrict__ vis,
                                          int8_t* __restrict__ regs, RankCtl* ctl,
                                          int8_t* __restrict__ pristine, bool use_pristine) {
  if (ctl && blockIdx.x == 0 && threadIdx.x == 0) ctl->dirty_count = 0;  // full rescore follows
  const uint32_t q = Jp >> 2;
  const uint32_t W32 = Jp >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  if (use_pristine && pristine) {
    // Streaming copy (16-byte vectors, G lanes per row — at most a quarter of
    // the row's words, so every lane has 4 loads in flight) with the VISITED
    // bits re-applied.
    const uint32_t q16 = Jp >> 4;
    uint32_t G = 32;
    while (G > 1 && 4 * G > q16) G >>= 1;
    const uint32_t R = 32 / G, lane = lane_id(), sub = lane / G, sl = lane % G;
    const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    for (uint64_t u0 = gw * R; u0 < n; u0 += nw * R) {
      const uint64_t u = u0 + sub;
      if (u >= n) continue;
      const uint4* src = reinterpret_cast<const uint4*>(pristine + u * Jp);
      uint4* dst = reinterpret_cast<uint4*>(regs + u * Jp);
      const uint32_t* vrow = vis + u * W32;
      for (uint32_t w0 = sl; w0 < q16; w0 += 4 * G) {
        uint4 v[4];
        uint32_t vb[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t w = w0 + t * G;
          if (w < q16) {
            v[t] = __ldcs(src + w);
            vb[t] = __ldcg(vrow + (w >> 1)) >> ((w & 1) * 16);
          }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t w = w0 + t * G;
          if (w < q16) {
            uint4 o = v[t];
            o.x &= ~expand4(vb[t] & 15u);
            o.y &= ~expand4((vb[t] >> 4) & 15u);
            o.z &= ~expand4((vb[t] >> 8) & 15u);
            o.w &= ~expand4((vb[t] >> 12) & 15u);
            dst[w] = o;
          }
        }
      }
    }
    return;
  }
  // warp per row, lanes over 4-register words (coalesced u32 stores).  The
  // four hashes of a word are independent (keys fetched as two 16-byte
  // loads, pads have key 0 and are masked after), no per-register branches.
  for (uint64_t u = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < n; u += nw) {
    const uint64_t ug = u * kGolden;
    uint32_t* row = reinterpret_cast<uint32_t*>(regs + u * Jp);
    uint32_t* prow = pristine ? reinterpret_cast<uint32_t*>(pristine + u * Jp) : nullptr;
    for (uint32_t w = lane_id(); w < q; w += 32) {
      const uint32_t j0 = w * 4;
      const ulonglong2 k01 = __ldg(reinterpret_cast<const ulonglong2*>(jkey + j0));
      const ulonglong2 k23 = __ldg(reinterpret_cast<const ulonglong2*>(jkey + j0 + 2));
      const uint32_t vb = (vis[u * W32 + (j0 >> 5)] >> (j0 & 31)) & 15u;
      // stored byte = register value + 1 (clz <= 64: no carry between bytes)
      // four counts packed by byte permutes (ALU) rather than shifts the
      // compiler would issue as IMAD.SHL on the busy multiply pipe
      const uint32_t c01 = __byte_perm(clz_fmix64(add64_alu(k01.x, ug)),
                                       clz_fmix64(add64_alu(k01.y, ug)), 0x1140);
      const uint32_t c23 = __byte_perm(clz_fmix64(add64_alu(k23.x, ug)),
                                       clz_fmix64(add64_alu(k23.y, ug)), 0x1140);
      uint32_t pw = __byte_perm(c01, c23, 0x5410) + 0x01010101u;
      if (j0 + 4 > J) {  // pad registers are VISITED (stored 0)
        const uint32_t live = J > j0 ? J - j0 : 0;  // < 4
        pw &= ~(0xFFFFFFFFu << (8 * live));
      }
      row[w] = pw & ~expand4(vb);
      if (prow) prow[w] = pw;
    }
  }
}

__global__ void k_fill(uint32_t n, uint32_t J, uint32_t Jp, const uint64_t* __restrict__ jkey,
                       const uint32_t* __restrict__ vis, int8_t* __restrict__ regs,
                       const unsigned int* gate, unsigned int want, RankCtl* ctl,
                       int8_t* pristine, bool use_pristine) {
  if (gate && ld_volatile(gate) != want) return;
  fill_body(n, J, Jp, jkey, vis, regs, ctl, pristine, use_pristine);
}

// ---------------------------------------------------------------- simulate
// Register bytes are stored as value + 1 (VISITED -1 -> 0, clz values 0..64
// -> 1..65), so every stored byte is < 128 and a byte-wise max
// is four SIMD-within-a-register instructions:
//   t = (x | 0x80) - y per byte (no borrow crosses a byte: 0x80 + x - y >= 1),
//   bit 7 of t <=> x >= y, replicated over the byte by a sign-extending PRMT.
// bit 7 of every byte replicated over the byte (PTX prmt sign mode; the
// __byte_perm intrinsic ignores the selector's sign bit)
__device__ __forceinline__ uint32_t sign_bytes(uint32_t t) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(r) : "r"(t));
  return r;
}
__device__ __forceinline__ uint32_t ge_mask7(uint32_t x, uint32_t y) {
  return sign_bytes((x | 0x80808080u) - y);
}
__device__ __forceinline__ uint32_t max7(uint32_t x, uint32_t y) {
  const uint32_t m = ge_mask7(x, y);
  return (x & m) | (y & ~m);
}
// 0xFF per non-zero (non-VISITED) byte: b + 0x7F has bit 7 set iff b >= 1
// (b < 128: no carry leaves the byte).
__device__ __forceinline__ uint32_t nz_bits7(uint32_t d) { return (d + 0x7F7F7F7Fu) & 0x80808080u; }
__device__ __forceinline__ uint32_t nz_mask7(uint32_t d) { return sign_bytes(d + 0x7F7F7F7Fu); }
// dst takes max(dst, src) on live simulations (engine.cpp:22-53): VISITED
// (0) in dst is absorbing, VISITED in src never wins, dead simulations (bm
// byte 0) contribute 0.  bm = 0xFF per live byte.
__device__ __forceinline__ uint32_t merge4(uint32_t d, uint32_t s, uint32_t bm) {
  return max7(d, s & bm & nz_mask7(d));
}
__device__ __forceinline__ unsigned long long merge8(unsigned long long d, unsigned long long s,
                                                     uint32_t m8) {
  const uint32_t lo = merge4(uint32_t(d), uint32_t(s), expand4(m8 & 15u));
  const uint32_t hi = merge4(uint32_t(d >> 32), uint32_t(s >> 32), expand4(m8 >> 4));
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}

// Warp-aggregated append: the lanes that reach this call together reserve
// their slots with one atomic (a same-address atomic per lane serialises at
// the L2 slice and was the top stall of the first profiles).
__device__ __forceinline__ unsigned agg_reserve(unsigned int* ctr, unsigned count) {
  cg::coalesced_group grp = cg::coalesced_threads();
  const unsigned excl = cg::exclusive_scan(grp, count);
  unsigned base = 0;
  const unsigned last = grp.size() - 1;
  if (grp.thread_rank() == last) base = atomicAdd(ctr, excl + count);
  return grp.shfl(base, last) + excl;
}
__device__ __forceinline__ unsigned long long agg_reserve64(unsigned long long* ctr,
                                                            unsigned long long count) {
  cg::coalesced_group grp = cg::coalesced_threads();
  const unsigned long long excl = cg::exclusive_scan(grp, count);
  unsigned long long base = 0;
  const unsigned last = grp.size() - 1;
  if (grp.thread_rank() == last) base = atomicAdd(ctr, excl + count);
  return grp.shfl(base, last) + excl;
}

// Queue generation counter: (rows << 32) | chunks, so one atomic reserves
// both the row slot and the chunk slots of a pushed row.
__device__ __forceinline__ uint32_t qchunks(const unsigned long long* qc, int g) {
  return uint32_t(ld_volatile(&qc[g]));
}
__device__ __forceinline__ uint32_t qrows(const unsigned long long* qc, int g) {
  return uint32_t(ld_volatile(&qc[g]) >> 32);
}

// Per-warp staging for the flattened item distribution, plus the warp's
// pending frontier marks (rows for the next generation; cascade: rows newly
// dirty).
constexpr unsigned kMarkCap = 160;   // >= kMarkFlush + 128 (four items per lane per step)
constexpr unsigned kMarkFlush = 32;  // flush at a convergent point once this many are pending
struct WarpStage {
  uint32_t incl[32];
  uint32_t row[32];
  unsigned long long beg[32];
  uint32_t mrows[kMarkCap];
  uint32_t mdirty[kMarkCap];
  unsigned nr, nd;
};

// Push of row u into the next generation, deduplicated by stamp: u is parked
// in the warp's buffer and published with its chunk ids by mark_flush
// (overflow falls back to a direct reservation).
__device__ __forceinline__ void push_row_buf(uint32_t u, uint32_t stamp, uint32_t* lstamp,
                                             const uint32_t* row_chunk, uint32_t* rows,
                                             uint32_t* chunks, unsigned long long* qcg,
                                             WarpStage& ws) {
  if (ld_volatile(&lstamp[u]) == stamp) return;
  if (atomicExch(&lstamp[u], stamp) == stamp) return;
  const unsigned i = atomicAdd(&ws.nr, 1u);
  if (i < kMarkCap) {
    ws.mrows[i] = u;
    return;
  }
  const uint32_t c0 = row_chunk[u], c1 = row_chunk[u + 1];
  const unsigned long long o = agg_reserve64(qcg, (1ull << 32) | (c1 - c0));
  rows[o >> 32] = u;
  const uint32_t ci = uint32_t(o);
  for (uint32_t c = c0; c < c1; ++c) chunks[ci + (c - c0)] = c;
}

// Cascade bookkeeping of a row that just received new VISITED bits: one
// 64-bit stamp (round base << 32 | level stamp) deduplicates both the dirty
// list (rows to rescore after this cascade) and the next-level frontier.
// The queue/dirty reservations are deferred into the warp's buffer (a level
// of a large cascade marks ~10^5 rows: one global counter atomic per row
// serialises at that address) and published by mark_flush.
__device__ __forceinline__ void cascade_mark(uint32_t v, uint32_t base, uint32_t stamp,
                                             unsigned long long* cstamp, uint32_t* dirty,
                                             unsigned int* dirty_count, const uint32_t* row_chunk,
                                             uint32_t* rows, uint32_t* chunks,
                                             unsigned long long* qcg, WarpStage& ws) {
  const unsigned long long want = (static_cast<unsigned long long>(base) << 32) | stamp;
  if (ld_volatile(&cstamp[v]) == want) return;
  const unsigned long long old = atomicExch(&cstamp[v], want);
  if (old == want) return;
  if (uint32_t(old >> 32) != base) {
    const unsigned i = atomicAdd(&ws.nd, 1u);
    if (i < kMarkCap) ws.mdirty[i] = v;
    else dirty[agg_reserve(dirty_count, 1u)] = v;
  }
  if (uint32_t(old) != stamp) {
    const unsigned i = atomicAdd(&ws.nr, 1u);
    if (i < kMarkCap) {
      ws.mrows[i] = v;
    } else {
      const uint32_t c0 = row_chunk[v], c1 = row_chunk[v + 1];
      const unsigned long long o = agg_reserve64(qcg, (1ull << 32) | (c1 - c0));
      rows[o >> 32] = v;
      const uint32_t ci = uint32_t(o);
      for (uint32_t c = c0; c < c1; ++c) chunks[ci + (c - c0)] = c;
    }
  }
}

// Publish the warp's pending marks (warp-converged): one counter atomic per
// list, rows with their chunk ids laid out by a warp prefix sum.
__device__ __forceinline__ void mark_flush(WarpStage& ws, uint32_t* dirty,
                                           unsigned int* dirty_count, const uint32_t* row_chunk,
                                           uint32_t* rows, uint32_t* chunks,
                                           unsigned long long* qcg) {
  __syncwarp();
  const unsigned lane = lane_id();
  const unsigned nd = min(ws.nd, kMarkCap), nr = min(ws.nr, kMarkCap);
  if (nd) {
    unsigned o = 0;
    if (lane == 0) o = atomicAdd(dirty_count, nd);
    o = __shfl_sync(0xffffffffu, o, 0);
    for (unsigned i = lane; i < nd; i += 32) dirty[o + i] = ws.mdirty[i];
  }
  if (nr) {
    uint32_t c0[kMarkCap / 32], cn[kMarkCap / 32], ex[kMarkCap / 32];
    uint32_t run = 0;
#pragma unroll
    for (unsigned k = 0; k < kMarkCap / 32; ++k) {
      const unsigned i = k * 32 + lane;
      c0[k] = cn[k] = 0;
      if (i < nr) {
        const uint32_t v = ws.mrows[i];
        c0[k] = row_chunk[v];
        cn[k] = row_chunk[v + 1] - c0[k];
      }
      uint32_t incl = cn[k];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= unsigned(o)) incl += t;
      }
      ex[k] = run + incl - cn[k];
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    unsigned long long o = 0;
    if (lane == 0) o = atomicAdd(qcg, (static_cast<unsigned long long>(nr) << 32) | run);
    o = __shfl_sync(0xffffffffu, o, 0);
    const uint32_t ro = uint32_t(o >> 32), co = uint32_t(o);
#pragma unroll
    for (unsigned k = 0; k < kMarkCap / 32; ++k) {
      const unsigned i = k * 32 + lane;
      if (i < nr) {
        rows[ro + i] = ws.mrows[i];
        for (uint32_t c = 0; c < cn[k]; ++c) chunks[co + ex[k] + c] = c0[k] + c;
      }
    }
  }
  __syncwarp();
  if (lane == 0) ws.nr = ws.nd = 0;
  __syncwarp();
}

// Per-step hook of for_frontier_items (warp-converged): none by default.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// Warp-cooperative work distribution over a frontier of chunks: one atomic
// claims 32 frontier slots, the items of those chunks are flattened (warp
// prefix sum of their sizes) and dealt to lanes 32 at a time, so lanes stay
// busy even when most rows have only a handful of items (R-MAT tails) and
// hub rows are spread over many warps.  f(row_a, item_a, ok_a, row_b, item_b,
// ok_b) per pair of items (two independent load chains in flight per lane);
// hook() after each pair step, all lanes converged.
template <class F, class H = NoHook>
__device__ __forceinline__ void for_frontier_items(const Items& it, const uint32_t* frontier,
                                                   uint32_t nc, unsigned int* work_ctr,
                                                   WarpStage& ws, uint64_t n_warps, F&& f,
                                                   H&& hook = H()) {
  const unsigned lane = lane_id();
  // Chunks claimed per warp: 32 when the frontier is large (tiny R-MAT rows
  // keep lanes busy), fewer when it is small so that a few full chunks
  // (<= 128 items each) are spread over many warps instead of serialised.
  const uint64_t per = n_warps ? nc / n_warps : nc;
  const uint32_t G = per >= 32 ? 32u : (per < 1 ? 1u : uint32_t(per));
  for (;;) {
    unsigned b0 = 0;
    if (lane == 0) b0 = atomicAdd(work_ctr, G);
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    if (b0 >= nc) break;
    const uint32_t idx = b0 + lane;
    uint32_t row = 0, cntc = 0;
    unsigned long long beg = 0;
    if (lane < G && idx < nc) {
      const uint32_t c = frontier ? __ldcg(frontier + idx) : idx;
      row = it.chunk_row[c];
      beg = it.chunk_beg[c];
      cntc = uint32_t(it.chunk_beg[c + 1] - beg);
    }
    uint32_t incl = cntc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= unsigned(o)) incl += t;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    ws.incl[lane] = incl;
    ws.row[lane] = row;
    ws.beg[lane] = beg;
    __syncwarp();
    // two items per lane per step (independent load chains in flight)
    for (uint32_t t0 = 0; t0 < total; t0 += 64) {
      const uint32_t ta = t0 + lane, tb = t0 + 32 + lane;
      uint32_t rowa = 0, rowb = 0;
      uint64_t ia = 0, ib = 0;
      const bool oka = ta < total, okb = tb < total;
      if (oka) {
        uint32_t lo = 0, hi = 31;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (ws.incl[mid] > ta) hi = mid; else lo = mid + 1;
        }
        rowa = ws.row[lo];
        ia = ws.beg[lo] + (ta - (lo ? ws.incl[lo - 1] : 0));
      }
      if (okb) {
        uint32_t lo = 0, hi = 31;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (ws.incl[mid] > tb) hi = mid; else lo = mid + 1;
        }
        rowb = ws.row[lo];
        ib = ws.beg[lo] + (tb - (lo ? ws.incl[lo - 1] : 0));
      }
      f(rowa, ia, oka, rowb, ib, okb);
      __syncwarp();
      hook();
    }
    __syncwarp();
  }
}

constexpr unsigned long long kNeg8 = 0;  // "no contribution" (stored bytes are value + 1)
#ifndef DFS_SOLO_CHUNKS
#define DFS_SOLO_CHUNKS 16
#endif
constexpr uint32_t kSoloChunks = DFS_SOLO_CHUNKS;  // frontier (chunks) a single block iterates alone
constexpr uint32_t kSoloDirty = 512;  // dirty rows block 0 rescores alone
constexpr uint32_t kPullMaxJp = 4096;  // pull accumulators live in shared memory

// Shared-memory running max of the live bytes of one source word.
__device__ __forceinline__ void acc_max(unsigned long long* a, unsigned long long sv, uint32_t m8) {
  const uint32_t slo = uint32_t(sv) & expand4(m8 & 15u);
  const uint32_t shi = uint32_t(sv >> 32) & expand4(m8 >> 4);
  unsigned long long old = *a;
  for (;;) {
    const unsigned long long nv =
        (static_cast<unsigned long long>(max7(uint32_t(old >> 32), shi)) << 32) |
        max7(uint32_t(old), slo);
    if (nv == old) return;
    const unsigned long long prev = atomicCAS(a, old, nv);
    if (prev == old) return;
    old = prev;
  }
}

// dst = max(dst, a) bytewise with VISITED (0) dst absorbing (a already masked).
__device__ __forceinline__ unsigned long long merge8_full(unsigned long long d,
                                                          unsigned long long a) {
  const uint32_t lo = max7(uint32_t(d), uint32_t(a) & nz_mask7(uint32_t(d)));
  const uint32_t hi = max7(uint32_t(d >> 32), uint32_t(a >> 32) & nz_mask7(uint32_t(d >> 32)));
  return (static_cast<unsigned long long>(hi) << 32) | lo;
}

// Fields of one reverse item (push sweeps).
struct SimItem {
  uint32_t u, mk, b;
};

__device__ __forceinline__ void sim_fields(SimItem& it, const Items& rev, uint64_t i) {
  it.u = __ldg(rev.other + i);
  it.mk = __ldg(rev.mask + i);
  it.b = __ldg(rev.batch + i);
}

// Byte-max CAS loop on one destination word (engine.cpp:22-53 semantics).
__device__ __forceinline__ bool cas_merge(unsigned long long* dp, unsigned long long d,
                                          unsigned long long sv, uint32_t m8) {
  unsigned long long nv = merge8(d, sv, m8);
  while (nv != d) {
    const unsigned long long old = atomicCAS(dp, d, nv);
    if (old == d) return true;
    d = old;
    nv = merge8(d, sv, m8);
  }
  return false;
}

// Two items: the first live 8-sim word of each is loaded together (thin IC
// windows rarely have more), remaining words follow one by one.
__device__ __forceinline__ void sim_pair(uint32_t ua, uint32_t mka, uint32_t bba, bool pa,
                                         const int8_t* sa, uint32_t ub, uint32_t mkb, uint32_t bbb,
                                         bool pb, const int8_t* sb, int8_t* regs, uint32_t Jp,
                                         bool& ca, bool& cb) {
  const int wa = pa ? (__ffs(mka) - 1) >> 3 : 0, wb = pb ? (__ffs(mkb) - 1) >> 3 : 0;
  const unsigned long long* spa = reinterpret_cast<const unsigned long long*>(sa + bba * 32);
  const unsigned long long* spb = reinterpret_cast<const unsigned long long*>(sb + bbb * 32);
  unsigned long long* dpa = reinterpret_cast<unsigned long long*>(regs + uint64_t(ua) * Jp + bba * 32);
  unsigned long long* dpb = reinterpret_cast<unsigned long long*>(regs + uint64_t(ub) * Jp + bbb * 32);
  unsigned long long s0 = 0, d0 = 0, s1 = 0, d1 = 0;
  if (pa) {
    s0 = __ldcg(spa + wa);
    d0 = __ldcg(dpa + wa);
  }
  if (pb) {
    s1 = __ldcg(spb + wb);
    d1 = __ldcg(dpb + wb);
  }
  ca = pa && cas_merge(dpa + wa, d0, s0, (mka >> (8 * wa)) & 0xFFu);
  cb = pb && cas_merge(dpb + wb, d1, s1, (mkb >> (8 * wb)) & 0xFFu);
  // further live words of each item: all its loads issued together
  auto rest = [](unsigned long long* dp, const unsigned long long* sp, uint32_t mk, int w0) {
    unsigned long long sx[3], dx[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int w = w0 + 1 + t;
      const bool live = w < 4 && ((mk >> (8 * w)) & 0xFFu);
      sx[t] = live ? __ldcg(sp + w) : 0;
      dx[t] = live ? __ldcg(dp + w) : 0;
    }
    bool ch = false;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int w = w0 + 1 + t;
      const uint32_t m8 = w < 4 ? (mk >> (8 * w)) & 0xFFu : 0u;
      if (m8) ch |= cas_merge(dp + w, dx[t], sx[t], m8);
    }
    return ch;
  };
  if (pa && (uint64_t(mka) >> (8 * (wa + 1)))) ca |= rest(dpa, spa, mka, wa);
  if (pb && (uint64_t(mkb) >> (8 * (wb + 1)))) cb |= rest(dpb, spb, mkb, wb);
}

struct SimArgs {
  RankDev r;
  int cap;
  const unsigned int* gate;
  unsigned int want;
  int dbg;  // experiments only (DFS_DBG): bit0 skip big-row pull, bit1 skip small rows
  int pull_f;  // pull when frontier chunks * pull_f > total chunks (DFS_SIM_PULL, default 4)
};

// Persistent simulate-to-convergence (engine.cpp:57-96 semantics).  Sweep s
// processes the reverse chunks of rows that changed in sweep s-1 (all chunks
// in sweep 1).  Async mode (JAC = 0) reads and writes the live matrix in place
// (the fixpoint is schedule-independent: DESIGN.md §simulate); Jacobi mode
// reads the snapshot and re-syncs changed rows after each sweep, which
// reproduces the reference's sweep count exactly.  CNT = 1 (Jacobi only)
// tallies the reference-schedule work units of SURVEY.md §8(d).
#ifndef DFS_SIM_MINB
#define DFS_SIM_MINB 3
#endif
#ifndef DFS_SIM_CLAIM
#define DFS_SIM_CLAIM 128
#endif
struct SimOpts {
  int cap;
  int dbg;
  int pull_f;
};

template <int JAC, int CNT>
// `base`: this partition's stamp base, identical in every block (callers pass
// a value no block can have advanced yet); returns the next base.  Reading
// r.ctl->tick here instead would race with block 0 finishing a solo-only
// phase (and advancing the tick) before a late block starts it.
__device__ __forceinline__ uint32_t simulate_body(const RankDev& r, const SimOpts& a,
                                              cg::grid_group& grid, WarpStage* stage,
                                              unsigned long long& s_release,
                                              unsigned long long* dyn_smem, uint32_t base) {
  unsigned int* cnt = r.q.counts;
  unsigned long long* qc = reinterpret_cast<unsigned long long*>(r.q.counts);
  const unsigned lane = lane_id();
  const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t gthreads = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t gwarp = gtid >> 5;
  const uint64_t nw = gthreads >> 5;
  WarpStage& ws = stage[threadIdx.x >> 5];
  if (lane == 0) ws.nr = ws.nd = 0;
  __syncwarp();
  // Pull accumulator: Jp bytes of running maxima + touched-batch bits per warp.
  const uint32_t W32 = r.W32;
  const bool pull_ok = r.Jp <= kPullMaxJp;
  unsigned long long* acc = dyn_smem + (threadIdx.x >> 5) * (kPullMaxJp / 8 + 8);
  uint32_t* touched = reinterpret_cast<uint32_t*>(acc + r.Jp / 8);
  if (pull_ok) {
    for (uint32_t w = lane; w < r.Jp / 8; w += 32) acc[w] = kNeg8;
    if (lane < 4) touched[lane] = 0;
    __syncwarp();
  }
  if (gwarp == 0 && lane < 16) cnt[lane] = 0;
  if (JAC) {  // SimulateBuffers::reset (engine.cpp:9-15): snapshot := registers
    const uint64_t n16 = uint64_t(r.n) * r.Jp / 16;
    const uint4* s4 = reinterpret_cast<const uint4*>(r.regs);
    uint4* d4 = reinterpret_cast<uint4*>(r.snap);
    for (uint64_t i = gtid; i < n16; i += gthreads) d4[i] = s4[i];
  }
  const uint64_t tb_words = CNT ? (uint64_t(r.n) * r.W32 + 31) / 32 : 0;
  if (CNT)
    for (uint64_t i = gtid; i < tb_words; i += gthreads) r.tbits[i] = 0;
  grid.sync();

  const int8_t* srcm = JAC ? r.snap : r.regs;
  const uint32_t Jp = r.Jp;
  unsigned long long upd = 0, nitems = 0, nedges = 0, ntouched = 0;

  // One sweep.  solo: only block 0 participates (small frontier), barriers
  // are block-level; otherwise the whole grid.
  auto sweep = [&](uint32_t s, bool solo) {
    const int g = s % 3, gn = (s + 1) % 3, gr = (s + 2) % 3;
    const uint64_t my_warp = solo ? (threadIdx.x >> 5) : gwarp;
    const uint64_t n_warps = solo ? kWarps : nw;
    const uint32_t nc = (s == 1) ? uint32_t(r.rev.chunks) : qchunks(qc, g);
    if (my_warp == 0 && lane == 0) {
      qc[gr] = 0;
      cnt[8 + gr] = 0;
      *reinterpret_cast<unsigned long long*>(&cnt[12 + 2 * ((s + 1) & 1)]) = 0;  // next sweep's
    }
    const uint32_t stamp = base + s;
    uint32_t* rows_n = r.q.rows[gn];
    uint32_t* chunks_n = r.q.chunks[gn];
    auto flush = [&] {
      mark_flush(ws, nullptr, nullptr, r.rev.row_chunk, rows_n, chunks_n, &qc[gn]);
    };
    auto hook = [&] {  // warp-converged, after a __syncwarp
      if (ws.nr >= kMarkFlush) flush();
    };
    if ((a.dbg & 4) && blockIdx.x == 0 && threadIdx.x == 0) trace(solo ? 1 : 0, s, nc);
    // Large frontiers (and sweep 1) run PULL-style over row-owned forward
    // chunks: a warp gathers the sources of one destination row chunk into a
    // shared-memory accumulator and writes each touched word once (plain store
    // when it owns the row, CAS otherwise), so out-hub rows see one update per
    // chunk instead of one contended CAS per item.  Small frontiers push.
    // Count mode keeps the exact push frontier of the reference schedule.
    const bool pull =
        !CNT && !solo && pull_ok && (s == 1 || uint64_t(nc) * a.pull_f > r.rev.chunks);
    if (pull) {
      const uint32_t need = base + s - 1;  // source changed in sweep s-1 (or later)
      const uint64_t nbig = (a.dbg & 1) ? 0 : r.fwd.nbig;
      {
      // chunk headers one iteration ahead (their two dependent loads overlap
      // the current chunk instead of heading its latency chain)
      uint32_t c_nx = my_warp < nbig ? r.fwd.big[my_warp] : 0;
      for (uint64_t k = my_warp; k < nbig; k += n_warps) {
        __syncwarp();
        hook();
        const uint32_t c = c_nx & ~kBigOwner;
        const bool owner = (c_nx & kBigOwner) != 0;
        const uint32_t u = r.fwd.chunk_row[c];
        const uint64_t beg = r.fwd.chunk_beg[c], end = r.fwd.chunk_beg[c + 1];
        if (k + n_warps < nbig) c_nx = r.fwd.big[k + n_warps];
        // A chunk has <= 4*32 items: each lane stages its (up to) 4 items'
        // fields, stamps and first live source word before any is consumed.
        uint32_t vq[4], mq[4], bq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint64_t i = beg + lane + 32 * q;
          const bool act = i < end;
          vq[q] = act ? __ldg(r.fwd.other + i) : 0;
          mq[q] = act ? __ldg(r.fwd.mask + i) : 0;
          bq[q] = act ? __ldg(r.fwd.batch + i) : 0;
        }
        // Source stamps and first live source words are loaded together
        // (speculatively: pull sweeps run when most sources changed), then
        // items whose source did not change since the previous sweep drop out.
        uint32_t st[4];
        unsigned long long s0[4];
        int w0[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          w0[q] = mq[q] ? (__ffs(mq[q]) - 1) >> 3 : 0;
          st[q] = (s > 1 && mq[q]) ? __ldcg(r.lstamp + vq[q]) : 0xFFFFFFFFu;
          s0[q] = mq[q] ? __ldcg(reinterpret_cast<const unsigned long long*>(
                              srcm + uint64_t(vq[q]) * Jp + bq[q] * 32) + w0[q])
                        : 0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (st[q] < need) mq[q] = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (!mq[q]) continue;
          const uint32_t b = bq[q];
          const unsigned long long* sp =
              reinterpret_cast<const unsigned long long*>(srcm + uint64_t(vq[q]) * Jp + b * 32);
          // the item's further live words are loaded together (one round trip)
          unsigned long long sx[3];
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const int wv = w0[q] + 1 + t;
            sx[t] = (wv < 4 && ((mq[q] >> (8 * wv)) & 0xFFu)) ? __ldcg(sp + wv) : 0;
          }
#ifdef DFS_EXPERIMENTS
          if (a.dbg & 32)  // timing experiment only: the first acc max twice (a smaller value: no effect)
            acc_max(&acc[b * 4 + w0[q]], s0[q] & 0xFEFEFEFEFEFEFEFEull, (mq[q] >> (8 * w0[q])) & 0xFFu);
#endif
          acc_max(&acc[b * 4 + w0[q]], s0[q], (mq[q] >> (8 * w0[q])) & 0xFFu);
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const int wv = w0[q] + 1 + t;
            const uint32_t m8 = wv < 4 ? (mq[q] >> (8 * wv)) & 0xFFu : 0u;
            if (m8) acc_max(&acc[b * 4 + wv], sx[t], m8);
          }
          atomicOr(&touched[b >> 5], 1u << (b & 31));
          upd += __popc(mq[q]);
          ++nitems;
        }
        __syncwarp();
        unsigned long long* drow = reinterpret_cast<unsigned long long*>(r.regs + uint64_t(u) * Jp);
        bool changed = false;
        // Write-back spread over the lanes by 8-byte word (word w = batch
        // w/4): every lane issues its (up to 4) destination loads together,
        // so a chunk costs one memory round trip instead of one per word.
        const uint32_t nwords = W32 * 4;
        for (uint32_t w0 = 0; w0 < nwords; w0 += 128) {
          unsigned long long av[4], dv[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint32_t w = w0 + 32 * t + lane;
            av[t] = kNeg8;
            if (w < nwords && ((touched[w >> 7] >> ((w >> 2) & 31)) & 1u)) {
              av[t] = acc[w];
              if (av[t] != kNeg8) acc[w] = kNeg8;
            }
            dv[t] = av[t] != kNeg8 ? __ldcg(drow + w) : 0;
          }
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            if (av[t] == kNeg8) continue;
            unsigned long long* dp = drow + w0 + 32 * t + lane;
            unsigned long long d = dv[t];
            unsigned long long nv = merge8_full(d, av[t]);
            if (nv == d) continue;
            if (owner) {
              *dp = nv;
              changed = true;
            } else {
              while (nv != d) {
                const unsigned long long old = atomicCAS(dp, d, nv);
                if (old == d) {
                  changed = true;
                  break;
                }
                d = old;
                nv = merge8_full(d, av[t]);
              }
            }
          }
        }
        __syncwarp();
        if (lane < 4) touched[lane] = 0;
        __syncwarp();
        if (__any_sync(0xffffffffu, changed) && lane == 0)
          push_row_buf(u, stamp, r.lstamp, r.rev.row_chunk, rows_n, chunks_n, &qc[gn], ws);
      }
      }
      // Small destination rows (<= kSmallRow items): item-parallel over the
      // flattened chunks, one CAS per item on a lightly contended row.
      {
        const uint64_t nsi = (a.dbg & 2) ? 0 : r.fwd.nsmall_items;
        // dynamic: a warp claims DFS_SIM_CLAIM items at a time (balances the
        // big-row tail), 128 per step; 0 = static grid-stride
        unsigned long long kc = 0, ke = 0;
        uint64_t kst = my_warp * 128;
        for (;;) {
          unsigned long long k0;
          if (DFS_SIM_CLAIM == 0) {
            k0 = kst;
            kst += n_warps * 128;
          } else {
            if (kc >= ke) {
              unsigned long long b = 0;
              if (lane == 0)
                b = atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[12 + 2 * (s & 1)]),
                              (unsigned long long)(DFS_SIM_CLAIM));
              kc = __shfl_sync(0xffffffffu, b, 0);
              ke = kc + DFS_SIM_CLAIM;
            }
            k0 = kc;
            kc += 128;
          }
          if (k0 >= nsi) break;
          // four items per lane, every load stage issued for all four first
          uint64_t iq[4];
          uint32_t uq[4], vq[4], mq[4], bq[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint64_t kk = k0 + lane + 32 * q;
            iq[q] = kk < nsi ? __ldg(r.fwd.small_items + kk) : 0;
            mq[q] = kk < nsi ? 1u : 0u;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uq[q] = mq[q] ? __ldg(r.fwd.row + iq[q]) : 0;
            vq[q] = mq[q] ? __ldg(r.fwd.other + iq[q]) : 0;
            bq[q] = mq[q] ? __ldg(r.fwd.batch + iq[q]) : 0;
            mq[q] = mq[q] ? __ldg(r.fwd.mask + iq[q]) : 0;
          }
          // stamps, first source and destination words in one round trip
          uint32_t st[4];
          unsigned long long s0[4], d0[4];
          int w0[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            w0[q] = mq[q] ? (__ffs(mq[q]) - 1) >> 3 : 0;
            st[q] = (s > 1 && mq[q]) ? __ldcg(r.lstamp + vq[q]) : 0xFFFFFFFFu;
            s0[q] = mq[q] ? __ldcg(reinterpret_cast<const unsigned long long*>(
                                srcm + uint64_t(vq[q]) * Jp + bq[q] * 32) + w0[q])
                          : 0;
            d0[q] = mq[q] ? __ldcg(reinterpret_cast<const unsigned long long*>(
                                r.regs + uint64_t(uq[q]) * Jp + bq[q] * 32) + w0[q])
                          : 0;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (st[q] < need) mq[q] = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (!mq[q]) continue;
            unsigned long long* dp =
                reinterpret_cast<unsigned long long*>(r.regs + uint64_t(uq[q]) * Jp + bq[q] * 32);
            const unsigned long long* sp = reinterpret_cast<const unsigned long long*>(
                srcm + uint64_t(vq[q]) * Jp + bq[q] * 32);
            bool ch = cas_merge(dp + w0[q], d0[q], s0[q], (mq[q] >> (8 * w0[q])) & 0xFFu);
            for (int wv = w0[q] + 1; wv < 4; ++wv) {
              const uint32_t m8 = (mq[q] >> (8 * wv)) & 0xFFu;
              if (m8) ch |= cas_merge(dp + wv, __ldcg(dp + wv), __ldcg(sp + wv), m8);
            }
            upd += __popc(mq[q]);
            ++nitems;
            if (ch)
              push_row_buf(uq[q], stamp, r.lstamp, r.rev.row_chunk, rows_n, chunks_n, &qc[gn], ws);
          }
          __syncwarp();
          hook();
        }
      }
    } else {
      for_frontier_items(
          r.rev, s == 1 ? nullptr : r.q.chunks[g], nc, &cnt[8 + g], ws, n_warps,
          [&](uint32_t va, uint64_t ia, bool pa, uint32_t vb, uint64_t ib, bool pb) {
            SimItem A, B;
            if (pa) sim_fields(A, r.rev, ia);
            if (pb) sim_fields(B, r.rev, ib);
            bool ca, cb;
            sim_pair(A.u, A.mk, A.b, pa, srcm + uint64_t(va) * Jp, B.u, B.mk, B.b, pb,
                     srcm + uint64_t(vb) * Jp, r.regs, Jp, ca, cb);
            if (pa) {
              upd += __popc(A.mk);
              ++nitems;
            }
            if (pb) {
              upd += __popc(B.mk);
              ++nitems;
            }
            if (CNT) {
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                const bool p = q ? pb : pa;
                if (!p) continue;
                const uint64_t i = q ? ib : ia;
                const uint32_t v = q ? vb : va;
                const SimItem& X = q ? B : A;
                // E: first item of its edge (items of one edge are consecutive, same u)
                if (i == r.rev.row_off[v] || r.rev.other[i - 1] != X.u) ++nedges;
                // T: distinct (u, b) touched in this sweep
                const uint64_t bit = uint64_t(X.u) * r.W32 + X.b;
                const uint32_t m1 = 1u << (bit & 31);
                if (!(atomicOr(&r.tbits[bit >> 5], m1) & m1)) ++ntouched;
              }
            }
            if (ca)
              push_row_buf(A.u, stamp, r.lstamp, r.rev.row_chunk, rows_n, chunks_n, &qc[gn], ws);
            if (cb)
              push_row_buf(B.u, stamp, r.lstamp, r.rev.row_chunk, rows_n, chunks_n, &qc[gn], ws);
          }, hook);
    }
    __syncwarp();
    if (ws.nr) flush();
  };
  // engine.cpp:81-82: re-sync snapshot rows that moved (Jacobi schedule).
  auto resync = [&](uint32_t s, bool solo) {
    const int gn = (s + 1) % 3;
    const unsigned nr = qrows(qc, gn);
    const uint64_t my_warp = solo ? (threadIdx.x >> 5) : gwarp;
    const uint64_t n_warps = solo ? kWarps : nw;
    for (uint64_t k = my_warp; k < nr; k += n_warps) {
      const uint64_t row = uint64_t(__ldcg(r.q.rows[gn] + k)) * Jp;
      const uint4* sp4 = reinterpret_cast<const uint4*>(r.regs + row);
      uint4* dp4 = reinterpret_cast<uint4*>(r.snap + row);
      for (uint32_t j = lane; j < Jp / 16; j += 32) dp4[j] = __ldcg(sp4 + j);
    }
    if (CNT) {
      const uint64_t t0 = solo ? threadIdx.x : gtid, ts = solo ? blockDim.x : gthreads;
      for (uint64_t i = t0; i < tb_words; i += ts) r.tbits[i] = 0;
    }
  };

  uint32_t s = 1;
  int err = 0;
  for (;;) {
    const int g = s % 3;
    if (s > 1 && qrows(qc, g) == 0) break;  // no row changed in sweep s-1
    if (s > uint32_t(a.cap)) {
      err = 1;
      break;
    }
    if (s > 1 && qchunks(qc, g) <= kSoloChunks) {
      // Small frontier: block 0 iterates alone with block barriers; the rest
      // of the grid parks until it hands back (grid barriers cost more than
      // the work of a tail sweep).
      if (blockIdx.x == 0) {
        uint32_t code = 0;  // 0 resume grid mode at s, 1 converged, 2 cap exceeded
        for (;;) {
          const int gg = s % 3;
          if (qrows(qc, gg) == 0) {
            code = 1;
            break;
          }
          if (s > uint32_t(a.cap)) {
            code = 2;
            break;
          }
          if (qchunks(qc, gg) > 4 * kSoloChunks) break;
          sweep(s, true);
          __syncthreads();
          if (JAC) {
            resync(s, true);
            __syncthreads();
          }
          ++s;
        }
        if (threadIdx.x == 0) {
          __threadfence();
          atomicExch(&r.ctl->release,
                     (static_cast<unsigned long long>(base) << 32) | (uint64_t(s) << 2) | code);
        }
        __syncthreads();
        if (code == 1) break;
        if (code == 2) {
          err = 1;
          break;
        }
      } else {
        if (threadIdx.x == 0) {
          unsigned long long rv;
          for (;;) {
            rv = ld_volatile(&r.ctl->release);
            if ((rv >> 32) == base && uint32_t((rv >> 2) & 0x3FFFFFFFu) > s) break;
            __nanosleep(256);
          }
          __threadfence();
          s_release = rv;
        }
        __syncthreads();
        const unsigned long long rv = s_release;
        s = uint32_t((rv >> 2) & 0x3FFFFFFFu);
        if ((rv & 3) == 1) break;
        if ((rv & 3) == 2) {
          err = 1;
          break;
        }
      }
      continue;
    }
    sweep(s, false);
    grid.sync();
    if (JAC) {
      resync(s, false);
      grid.sync();
    }
    ++s;
  }
  // Instrumentation: one atomic per warp.
  for (int o = 16; o; o >>= 1) {
    upd += __shfl_xor_sync(0xffffffffu, upd, o);
    nitems += __shfl_xor_sync(0xffffffffu, nitems, o);
    if (CNT) {
      nedges += __shfl_xor_sync(0xffffffffu, nedges, o);
      ntouched += __shfl_xor_sync(0xffffffffu, ntouched, o);
    }
  }
  if (lane == 0 && upd) {
    atomicAdd(&r.ctl->updates, upd);
    atomicAdd(&r.ctl->items_processed, nitems);
    if (CNT) {
      atomicAdd(&r.ctl->cnt_edges, nedges);
      atomicAdd(&r.ctl->cnt_batches, nitems);
      atomicAdd(&r.ctl->cnt_touched, ntouched);
    }
  }
  if (gwarp == 0 && lane == 0) {
    const uint32_t sw = err ? s : s - 1;
    r.ctl->sweeps = sw;
    r.ctl->max_sweeps = max(r.ctl->max_sweeps, sw);
    r.ctl->total_sweeps += sw;
    r.ctl->cnt_sweeps += sw;
    r.ctl->cnt_convergences += 1;
    r.ctl->tick = base + s + 2;
    if (err) r.ctl->error = 1;
  }
  return base + s + 2;
}

template <int JAC, int CNT>
__global__ void __launch_bounds__(kThreads, DFS_SIM_MINB) k_simulate(SimArgs a) {
  if (a.gate && ld_volatile(a.gate) != a.want) return;  // grid-uniform
  __shared__ WarpStage stage[kWarps];
  __shared__ unsigned long long s_release;
  __shared__ RankDev s_r;
  extern __shared__ unsigned long long dyn_smem[];
  if (threadIdx.x == 0) s_r = a.r;
  __syncthreads();
  cg::grid_group grid = cg::this_grid();
  const SimOpts o{a.cap, a.dbg, a.pull_f};
  // read before simulate_body's first grid barrier: no block can advance it yet
  const uint32_t base = ld_volatile(&a.r.ctl->tick);
  simulate_body<JAC, CNT>(s_r, o, grid, stage, s_release, dyn_smem, base);
}

// ---------------------------------------------------------------- score
// sketch.cpp:119-131: live = #non-VISITED, denom = sum 2^-M[j] (ascending j),
// score = live*live / (denom*phi).  With every live register <= K and
// J * 2^K <= 2^53, each sequential partial sum is an exact multiple of 2^-K
// below 2^53 * 2^-K, so the reference's double sum is exact and equals the
// integer sum sum 2^(K-M[j]) scaled by 2^-K.  Rows with a
// larger register fall back to the sequential double sum.
// Streaming 16-byte load that the compiler may not sink to its first use
// (keeps a lane's batch of loads in flight together).
__device__ __forceinline__ uint4 ld_stream_early(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Empty asm "rewriting" a loaded vector: compute on it cannot be hoisted
// above this point, so a batch of ld_stream_early loads issues back to back.
__device__ __forceinline__ void pin_after_loads(uint4& v) {
  asm volatile("" : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w));
}

// Score lookup table (shared memory): the high words of 256 doubles (the low
// words are 0), indexed by a stored register byte c = r + 1: live r <= K ->
// 2^-r; live r > K -> 2^60 (flags the exact sequential fallback: without it
// the sum is <= J < 2^50); c = 0 (VISITED) -> 0.0.  32-bit entries: one bank
// per value, so a warp's lookups are (nearly) conflict-free.
__device__ __forceinline__ void score_table(uint32_t* tbl, int K) {
  // high word of 2^-b is (1023 - b) << 20 (b <= 64 keeps it normal); 2^60 flags
  // stored byte c = register value + 1; c == 0: VISITED
  for (int c = threadIdx.x; c < 256; c += blockDim.x)
    tbl[c] = (c == 0 || c >= 128) ? 0u
                                  : (c - 1 <= K ? uint32_t(1023 - (c - 1)) << 20
                                                : uint32_t(1023 + 60) << 20);
  __syncthreads();
}

__device__ __forceinline__ double score_term(const uint32_t* tbl, uint32_t w, uint32_t sel) {
  return __hiloint2double(int(tbl[__byte_perm(w, 0, sel)]), 0);
}

// 16 registers: live count and the sum of table terms (pairwise tree: short
// dependency chains; the sum is exact in any order, see score_body).
__device__ __forceinline__ void score_acc(uint4 v, const uint32_t* tbl, uint32_t& live,
                                          double& den) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  double p[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    live += __popc(nz_bits7(w[i]));
    p[i] = (score_term(tbl, w[i], 0x4440) + score_term(tbl, w[i], 0x4441)) +
           (score_term(tbl, w[i], 0x4442) + score_term(tbl, w[i], 0x4443));
  }
  den += (p[0] + p[1]) + (p[2] + p[3]);
}

// Called by every thread of a block; tbl: 256 words of shared memory.
__device__ __forceinline__ void score_body(const int8_t* __restrict__ regs, uint32_t n, uint32_t J,
                                           uint32_t Jp, int K, int full,
                                           const uint32_t* __restrict__ rows, RankCtl* ctl,
                                           double* __restrict__ scores, uint32_t* tbl,
                                           bool block_only = false) {
  score_table(tbl, K);
  const uint32_t nrows = full ? n : ld_volatile(&ctl->dirty_count);
  if (threadIdx.x == 0 && (block_only || blockIdx.x == 0) && ctl)
    atomicAdd(&ctl->rescored_rows, (unsigned long long)nrows);
  const unsigned lane = lane_id();
  const uint64_t nw = block_only ? kWarps : (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t gw = block_only ? threadIdx.x >> 5
                                 : (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  // G lanes per row (power of two, at most a quarter of the row's 16-byte
  // words), R rows per warp, two row groups per step: every lane keeps 8
  // independent 16-byte loads in flight before reducing (the score is a
  // streaming pass; with G up to the row's word count, J = 1024 rows left half
  // and J = 256 rows three quarters of the slots empty).
  const uint32_t q16 = Jp >> 4;
  uint32_t G = 32;
  while (G > 1 && 4 * G > q16) G >>= 1;
  const uint32_t R = 32 / G, sub = lane / G, sl = lane % G;
  const uint4 kDead = make_uint4(0u, 0u, 0u, 0u);  // all VISITED
  for (uint64_t k0 = gw * 2 * R; k0 < nrows; k0 += nw * 2 * R) {
    uint32_t u[2], live[2] = {0, 0};
    bool ok[2];
    double den[2] = {0.0, 0.0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t kk = k0 + h * R + sub;
      ok[h] = kk < nrows;
      u[h] = ok[h] ? (full ? uint32_t(kk) : __ldcg(rows + kk)) : 0;
    }
    for (uint32_t w0 = sl; w0 < q16; w0 += 4 * G) {
      uint4 va[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4* rp = reinterpret_cast<const uint4*>(regs + uint64_t(u[h]) * Jp);
#pragma unroll
        for (int t = 0; t < 4; ++t) {  // all live loads in flight together
          // (idx < q16 is warp-uniform: q16 is a multiple of G)
          const uint32_t idx = w0 + t * G;
          va[h][t] = idx < q16 ? ld_stream_early(rp + idx) : kDead;
          if (!ok[h]) va[h][t] = kDead;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int t = 0; t < 4; ++t) pin_after_loads(va[h][t]);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (w0 - sl + t * G < q16) score_acc(va[h][t], tbl, live[h], den[h]);
    }
    for (uint32_t o = G >> 1; o; o >>= 1) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        live[h] += __shfl_xor_sync(0xffffffffu, live[h], o);
        den[h] += __shfl_xor_sync(0xffffffffu, den[h], o);
      }
    }
    if (sl == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!ok[h]) continue;
        double sc = 0.0;
        if (live[h]) {
          // Every live register <= K with J * 2^K <= 2^53: each partial sum of
          // 2^-r is an exact multiple of 2^-K, so any summation order equals
          // the reference's sequential sum (sketch.cpp:122-126) bit for bit.
          double denom = den[h];
          if (denom >= 1125899906842624.0) {  // a register > K (2^50): exact sequential replay
            denom = 0.0;
            const int8_t* rb = regs + uint64_t(u[h]) * Jp;
            for (uint32_t j = 0; j < J; ++j)
              if (rb[j] != 0) denom = __dadd_rn(denom, ldexp(1.0, -(int(uint8_t(rb[j])) - 1)));
          }
          const double lv = double(live[h]);
          sc = __ddiv_rn(__dmul_rn(lv, lv), __dmul_rn(denom, kPhi));
        }
        scores[u[h]] = sc;
      }
    }
  }
}

__global__ void k_score(const int8_t* __restrict__ regs, uint32_t n, uint32_t J, uint32_t Jp,
                        int K, int full, const uint32_t* __restrict__ rows, RankCtl* ctl,
                        double* __restrict__ scores, const unsigned int* gate, unsigned int want) {
  if (gate && ld_volatile(gate) != want) return;
  __shared__ uint32_t tbl[256];
  score_body(regs, n, J, Jp, K, full, rows, ctl, scores, tbl);
}

// ---------------------------------------------------------------- reduce/argmax
// collectives.cpp:44-64: level k folds rank+2^k into rank (fixed order).
__device__ __forceinline__ void treesum_body(const double* const* __restrict__ parts,
                                             uint32_t mu, uint32_t n, double* __restrict__ out) {
  for (uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += uint64_t(gridDim.x) * blockDim.x) {
    double acc[64];
    for (uint32_t t = 0; t < mu; ++t) acc[t] = parts[t][v];
    for (uint32_t st = 1; st < mu; st <<= 1)
      for (uint32_t t = 0; t + st < mu; t += 2 * st) acc[t] = __dadd_rn(acc[t], acc[t + st]);
    out[v] = acc[0];
  }
}

__global__ void k_treesum(const double* const* __restrict__ parts, uint32_t mu, uint32_t n,
                          double* __restrict__ out) {
  treesum_body(parts, mu, n, out);
}

struct Best {
  double s;
  uint32_t v;
  uint32_t minu;
};
__device__ __forceinline__ Best best_of(Best a, Best b) {
  Best r;
  // runtime.cpp:95-119: strict '>' from 0.0 in ascending v == max score, ties
  // to the smallest id, only positive scores qualify.
  if (b.s > a.s || (b.s == a.s && b.v < a.v)) {
    r.s = b.s;
    r.v = b.v;
  } else {
    r.s = a.s;
    r.v = a.v;
  }
  r.minu = min(a.minu, b.minu);
  return r;
}

// Block partial of the argmax (runtime.cpp:95-119) over ids [lo, hi): best
// positive uncommitted (score, id) and the smallest uncommitted id of this
// block.  val(v) yields the (reduced) score of v.
template <class V>
__device__ __forceinline__ void argmax_partial_range(uint32_t lo, uint32_t hi, V&& val,
                                                     const RunArrays& ra, Best* sb) {
  Best b{0.0, 0xFFFFFFFFu, 0xFFFFFFFFu};
  for (uint64_t v = lo + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < hi;
       v += uint64_t(gridDim.x) * blockDim.x) {
    if (ra.committed[v]) continue;
    const double s = val(uint32_t(v));
    if (b.minu == 0xFFFFFFFFu) b.minu = uint32_t(v);
    if (s > b.s) {  // ascending v within a thread: strict > keeps the first
      b.s = s;
      b.v = uint32_t(v);
    }
  }
  for (int o = 16; o; o >>= 1) {
    Best x{__shfl_xor_sync(0xffffffffu, b.s, o), __shfl_xor_sync(0xffffffffu, b.v, o),
           __shfl_xor_sync(0xffffffffu, b.minu, o)};
    b = best_of(b, x);
  }
  __syncthreads();
  if (lane_id() == 0) sb[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    Best t = sb[0];
    for (int w = 1; w < kWarps; ++w) t = best_of(t, sb[w]);
    ra.blk_score[blockIdx.x] = t.s;
    ra.blk_arg[blockIdx.x] = t.v;
    ra.blk_min[blockIdx.x] = t.minu;
  }
}

__device__ __forceinline__ void argmax_partial(const double* __restrict__ scores, uint32_t n,
                                               const RunArrays& ra, Best* sb) {
  argmax_partial_range(0, n, [&](uint32_t v) { return scores[v]; }, ra, sb);
}

// Combine nblk partials (one block); the result is valid in thread 0.
__device__ __forceinline__ Best argmax_combine(uint32_t nblk, const RunArrays& ra, Best* sb) {
  Best t{0.0, 0xFFFFFFFFu, 0xFFFFFFFFu};
  for (uint32_t k = threadIdx.x; k < nblk; k += blockDim.x)
    t = best_of(t, Best{__ldcg(ra.blk_score + k), __ldcg(ra.blk_arg + k), __ldcg(ra.blk_min + k)});
  for (int o = 16; o; o >>= 1) {
    Best x{__shfl_xor_sync(0xffffffffu, t.s, o), __shfl_xor_sync(0xffffffffu, t.v, o),
           __shfl_xor_sync(0xffffffffu, t.minu, o)};
    t = best_of(t, x);
  }
  __syncthreads();
  if (lane_id() == 0) sb[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    t = sb[0];
    for (int w = 1; w < kWarps; ++w) t = best_of(t, sb[w]);
  }
  return t;
}

// Commit the winner (thread 0): choice, committed mark, saturation fallback to
// the smallest uncommitted id (runtime.cpp:95-121).
__device__ __forceinline__ void commit_choice(Best t, const RunArrays& ra) {
  uint32_t choice = t.v;
  if (choice == 0xFFFFFFFFu) {  // saturated: smallest uncommitted id
    ra.ctl->saturated = 1;
    choice = t.minu;
  }
  ra.ctl->choice = choice;
  ra.committed[choice] = 1;
  ra.ctl->argmax_done = 0;
}

__device__ __forceinline__ void argmax_finish(uint32_t nblk, const RunArrays& ra, Best* sb) {
  const Best t = argmax_combine(nblk, ra, sb);
  if (threadIdx.x == 0) commit_choice(t, ra);
}

// Argmax cache: best of segment `seg` (one warp; ascending ids per lane, then
// best_of = strict > from 0.0 with ties to the smaller id, runtime.cpp:95-119).
// Rows [base + seg*kSeg, min(n, ...)) (base: the peer slice start, else 0).
__device__ __forceinline__ void seg_recompute(const double* __restrict__ scores, uint32_t n,
                                              uint32_t seg, const RunArrays& ra,
                                              uint32_t base = 0) {
  const unsigned lane = lane_id();
  Best b{0.0, 0xFFFFFFFFu, 0xFFFFFFFFu};
  const uint32_t lo = base + seg * kSeg, hi = min(n, lo + kSeg);
  for (uint32_t v0 = lo + lane; v0 < hi; v0 += 256) {
    double sc[8];
    uint32_t cm[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // 8 independent loads in flight per lane
      const uint32_t v = v0 + 32 * k;
      const bool ok = v < hi;
      sc[k] = ok ? __ldcg(scores + v) : 0.0;
      cm[k] = ok ? ld_volatile(ra.committed + v) : 1u;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (cm[k]) continue;
      const uint32_t v = v0 + 32 * k;
      if (b.minu == 0xFFFFFFFFu) b.minu = v;
      if (sc[k] > b.s) {
        b.s = sc[k];
        b.v = v;
      }
    }
  }
  for (int o = 16; o; o >>= 1) {
    Best x{__shfl_xor_sync(0xffffffffu, b.s, o), __shfl_xor_sync(0xffffffffu, b.v, o),
           __shfl_xor_sync(0xffffffffu, b.minu, o)};
    b = best_of(b, x);
  }
  if (lane == 0) {
    ra.seg_score[seg] = b.s;
    ra.seg_arg[seg] = b.v;
    ra.seg_min[seg] = b.minu;
  }
}

// Block-wide best over the segment cache; valid in thread 0.
__device__ __forceinline__ Best seg_combine(const RunArrays& ra, Best* sb, uint32_t nseg) {
  Best t{0.0, 0xFFFFFFFFu, 0xFFFFFFFFu};
  for (uint32_t k = threadIdx.x; k < nseg; k += blockDim.x)
    t = best_of(t, Best{__ldcg(ra.seg_score + k), __ldcg(ra.seg_arg + k), __ldcg(ra.seg_min + k)});
  for (int o = 16; o; o >>= 1) {
    Best x{__shfl_xor_sync(0xffffffffu, t.s, o), __shfl_xor_sync(0xffffffffu, t.v, o),
           __shfl_xor_sync(0xffffffffu, t.minu, o)};
    t = best_of(t, x);
  }
  __syncthreads();
  if (lane_id() == 0) sb[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    t = sb[0];
    for (int w = 1; w < kWarps; ++w) t = best_of(t, sb[w]);
  }
  return t;
}

__global__ void __launch_bounds__(kThreads) k_argmax(const double* __restrict__ scores,
                                                     uint32_t n, RunArrays ra) {
  __shared__ Best sb[kWarps];
  __shared__ bool last;
  argmax_partial(scores, n, ra, sb);
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&ra.ctl->argmax_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  argmax_finish(gridDim.x, ra, sb);
}

// ---------------------------------------------------------------- cascade
struct CasArgs {
  RankDev r;
  const unsigned int* choice;
  uint32_t seed;
  int dbg;  // experiments only (DFS_DBG bit 2): per-level trace
  int pull_f;  // bottom-up when frontier chunks * pull_f > total (DFS_CAS_PULL, default 8)
};

// Clear the fresh bits of the rows listed in one generation.  A warp takes 32
// listed rows at a time (one coalesced load of their ids, then 32 rows of
// independent stores): one row per warp iteration made every row a dependent
// id load -> store round trip, ~0.4 ms per million-row level.
__device__ __forceinline__ void clear_rows(uint32_t* f, const uint32_t* rows, unsigned nr,
                                           uint32_t W32, uint64_t gwarp, uint64_t nw,
                                           unsigned lane) {
  for (uint64_t k0 = gwarp * 32; k0 < nr; k0 += nw * 32) {
    const uint64_t k = k0 + lane;
    const uint32_t mine = k < nr ? __ldcg(rows + k) : 0u;
    const uint32_t cnt = nr - k0 < 32 ? uint32_t(nr - k0) : 32u;
    for (uint32_t j = 0; j < cnt; ++j) {
      const uint64_t row = uint64_t(__shfl_sync(0xffffffffu, mine, j)) * W32;
      for (uint32_t w = lane; w < W32; w += 32) f[row + w] = 0;
    }
  }
}

// commit_seed + cascade (engine.cpp:106-144): level-synchronous BFS of fresh
// VISITED bits along forward items; cand = fresh_u & live & ~vis_v.  Post:
// VISITED_j(v) <=> v reachable from a committed seed in sample j.  One grid
// barrier per level: level L reads fresh[L%3], writes fresh[(L+1)%3] and
// clears the rows of level L-1 in fresh[(L+2)%3]; queues rotate mod 4.
struct CasOpts {
  const unsigned int* choice;
  uint32_t seed;
  int dbg;
  int pull_f;
  int cnt;  // count mode: tally the reference-schedule cascade work units
  // parked-grid rounds (k_run, one partition): block 0 wakes the parked
  // blocks when the cascade first needs the grid (unless *awake), and defers
  // the final release to the caller (episode returned in *defer_e)
  RunCtl* park = nullptr;
  uint32_t step = 0;
  uint32_t* awake = nullptr;
  uint32_t* defer_e = nullptr;
};

constexpr unsigned int kWakeSelect = 1, kWakeCascade = 2, kWakeRebuild = 3, kWakeDone = 4;
// Block 0, thread 0: wake the parked blocks with (reason, round, stamp base).
__device__ __forceinline__ void park_wake(RunCtl* c, unsigned int reason, uint32_t step,
                                          uint32_t base) {
  c->park_reason = reason;
  c->park_step = step;
  c->park_base = base;
  __threadfence();
  atomicAdd(&c->park_seq, 1u);
}

// `base` as in simulate_body; returns the next stamp base.  CNT: count mode
// (a compile-time switch: its bookkeeping stays out of the timed variant's
// register allocation).
template <int CNT>
__device__ __forceinline__ uint32_t cascade_body(const RankDev& r, const CasOpts& a,
                                             cg::grid_group& grid, WarpStage* stage,
                                             unsigned long long& s_release, uint32_t* cas_smem,
                                                 uint32_t base) {
  unsigned int* cnt = r.q.counts;
  unsigned long long* qc = reinterpret_cast<unsigned long long*>(r.q.counts);
  const unsigned lane = lane_id();
  const uint64_t gwarp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t W32 = r.W32;
  WarpStage& ws = stage[threadIdx.x >> 5];
  if (lane == 0) ws.nr = ws.nd = 0;
  __syncwarp();
  unsigned long long marked = 0;
  const bool pull_ok = r.Jp <= kPullMaxJp;
  uint32_t* cacc = cas_smem + (threadIdx.x >> 5) * (kPullMaxJp / 32);
  if (pull_ok) {
    for (uint32_t w = lane; w < W32; w += 32) cacc[w] = 0;
    __syncwarp();
  }

  if (gwarp == 0) {
    if (lane < 16) cnt[lane] = 0;
    __syncwarp();
    const uint32_t s = a.choice ? ld_volatile(a.choice) : a.seed;
    if (lane == 0) {
      r.ctl->dirty_count = 1;
      r.dirty[0] = s;
    }
    // engine.cpp:106-118: every non-VISITED register of s becomes fresh.
    bool any = false;
    for (uint32_t w = lane; w < W32; w += 32) {
      const uint32_t rem = r.J - w * 32;
      const uint32_t tail = rem >= 32 ? 0xFFFFFFFFu : ((1u << rem) - 1u);
      const uint32_t bits = tail & ~r.vis[uint64_t(s) * W32 + w];
      if (bits) {
        r.vis[uint64_t(s) * W32 + w] |= bits;
        r.fresh[1][uint64_t(s) * W32 + w] = bits;
        int8_t* rb = r.regs + uint64_t(s) * r.Jp + w * 32;
        for (uint32_t t = bits; t; t &= t - 1) rb[__ffs(t) - 1] = 0;
        marked += __popc(bits);
        any = true;
      }
    }
    any = __any_sync(0xffffffffu, any);
    __syncwarp();
    if (lane == 0) {
      r.cstamp[s] = (static_cast<unsigned long long>(base) << 32) | (any ? base + 1 : 0u);
      if (any && CNT) r.ctl->cnt_cascades += 1;
      if (any) {
        const uint32_t c0 = r.fwd.row_chunk[s], c1 = r.fwd.row_chunk[s + 1];
        qc[1] = (1ull << 32) | (c1 - c0);
        r.q.rows[1][0] = s;
        for (uint32_t c = c0; c < c1; ++c) r.q.chunks[1][c - c0] = c;
      }
    }
  }

  // One BFS level.  solo: only block 0 (small frontier, block barriers).
  auto level = [&](uint32_t L, bool solo) {
    const int g = L % 4, gn = (L + 1) % 4, gr = (L + 2) % 4, gp = (L + 3) % 4;
    const uint64_t my_warp = solo ? (threadIdx.x >> 5) : gwarp;
    const uint64_t n_warps = solo ? kWarps : nw;
    const uint32_t* fcur = r.fresh[L % 3];
    uint32_t* fnxt = r.fresh[(L + 1) % 3];
    uint32_t* fprev = r.fresh[(L + 2) % 3];
    const uint32_t nc = qchunks(qc, g);
    if (my_warp == 0 && lane == 0) {
      qc[gr] = 0;
      cnt[8 + gr] = 0;
    }
    clear_rows(fprev, r.q.rows[gp], qrows(qc, gp), W32, my_warp, n_warps, lane);
    if ((a.dbg & 4) && blockIdx.x == 0 && threadIdx.x == 0) trace(2 + (solo ? 1 : 0), L, nc);
    if (CNT) {  // frontier rows and their device-graph out-edges
      const unsigned nr = qrows(qc, g);
      if (my_warp == 0 && lane == 0) atomicAdd(&r.ctl->cnt_cas_rows, (unsigned long long)nr);
      unsigned long long ne = 0;
      for (uint64_t kk = my_warp; kk < nr; kk += n_warps) {
        const uint32_t u = __ldcg(r.q.rows[g] + kk);
        const uint64_t b0 = r.fwd.row_off[u], b1 = r.fwd.row_off[u + 1];
        for (uint64_t i = b0 + lane; i < b1; i += 32)  // items of one edge are consecutive
          ne += (i == b0 || r.fwd.other[i] != r.fwd.other[i - 1]) ? 1 : 0;
      }
      for (int o = 16; o; o >>= 1) ne += __shfl_xor_sync(0xffffffffu, ne, o);
      if (lane == 0 && ne) atomicAdd(&r.ctl->cnt_cas_edges, ne);
    }
    const uint32_t stamp = base + L + 1;
    uint32_t* rows_n = r.q.rows[gn];
    uint32_t* chunks_n = r.q.chunks[gn];
    // Claim newly reached registers of target row v in batch b.
    auto claim = [&](uint32_t v, uint32_t b, uint32_t cand) {
      uint32_t* vw = r.vis + uint64_t(v) * W32 + b;
      const uint32_t nb = cand & ~atomicOr(vw, cand);
      if (!nb) return;
      int8_t* rb = r.regs + uint64_t(v) * r.Jp + b * 32;
      for (uint32_t t = nb; t; t &= t - 1) rb[__ffs(t) - 1] = 0;
      atomicOr(fnxt + uint64_t(v) * W32 + b, nb);
      marked += __popc(nb);
      cascade_mark(v, base, stamp, r.cstamp, r.dirty, &r.ctl->dirty_count, r.fwd.row_chunk, rows_n,
                   chunks_n, &qc[gn], ws);
    };
    auto flush = [&] {
      mark_flush(ws, r.dirty, &r.ctl->dirty_count, r.fwd.row_chunk, rows_n, chunks_n, &qc[gn]);
    };
    auto hook = [&] {  // warp-converged, after a __syncwarp
      if (ws.nr >= kMarkFlush || ws.nd >= kMarkFlush) flush();
    };
    // Top-down pair: frontier row u -> targets of two forward items.
    auto visit = [&](uint32_t ua, uint64_t ia, bool pa, uint32_t ub, uint64_t ib, bool pb) {
      const uint32_t ba = pa ? __ldg(r.fwd.batch + ia) : 0, bb = pb ? __ldg(r.fwd.batch + ib) : 0;
      const uint32_t ma = pa ? __ldg(r.fwd.mask + ia) : 0, mb = pb ? __ldg(r.fwd.mask + ib) : 0;
      const uint32_t va = pa ? __ldg(r.fwd.other + ia) : 0, vb = pb ? __ldg(r.fwd.other + ib) : 0;
      uint32_t ca = pa ? __ldcg(fcur + uint64_t(ua) * W32 + ba) & ma : 0;
      uint32_t cb = pb ? __ldcg(fcur + uint64_t(ub) * W32 + bb) & mb : 0;
      const uint32_t xa = ca ? __ldcg(r.vis + uint64_t(va) * W32 + ba) : 0;
      const uint32_t xb = cb ? __ldcg(r.vis + uint64_t(vb) * W32 + bb) : 0;
      ca &= ~xa;
      cb &= ~xb;
      if (ca) claim(va, ba, ca);
      if (cb) claim(vb, bb, cb);
    };
    if (!solo && pull_ok && uint64_t(nc) * a.pull_f > r.fwd.chunks) {
      // Large frontier: bottom-up (pull) level over row-owned reverse chunks.
      // A warp ORs the fresh bits of all in-neighbours of one target row into
      // a shared accumulator, then claims the unvisited ones with one update
      // per batch word (direction-optimising BFS, Beamer et al.).
      const uint64_t nbig = r.rev.nbig;
      // Parents' bits: the live VISITED bitset, read in place, instead of the
      // level's fresh bits (count mode keeps the reference's level structure).
      // VISITED is closed under live edges after every cascade, so a parent's
      // older bits add no candidate, and bits a parent gained earlier in THIS
      // level propagate at once (fewer bottom-up levels; same closure).
      const uint32_t* fpar = CNT ? fcur : r.vis;
      uint32_t c_nx = my_warp < nbig ? r.rev.big[my_warp] : 0;  // one iteration ahead (| owner flag)
      for (uint64_t k = my_warp; k < nbig; k += n_warps) {
        __syncwarp();
        hook();
        const uint32_t c = c_nx & ~kBigOwner;
        const uint32_t v = r.rev.chunk_row[c];
        const uint64_t beg = r.rev.chunk_beg[c], end = r.rev.chunk_beg[c + 1];
        if (k + n_warps < nbig) c_nx = r.rev.big[k + n_warps];
        bool any = false;
        uint32_t uq[4], mq[4], bq[4], fq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint64_t i = beg + lane + 32 * q;
          const bool act = i < end;
          uq[q] = act ? __ldg(r.rev.other + i) : 0;
          mq[q] = act ? __ldg(r.rev.mask + i) : 0;
          bq[q] = act ? __ldg(r.rev.batch + i) : 0;
        }
        // bottom-up: only simulations still unvisited at v look for a parent.
        // v's visited row is one coalesced load (lane b holds batch b) issued
        // with the item fields; items pick their batch word by shuffle, and
        // only items with unvisited live simulations load their parent's
        // fresh word.
        const uint32_t* vrow = r.vis + uint64_t(v) * W32;
        const bool narrow = W32 <= 32;
        const uint32_t vw = (narrow && lane < W32) ? __ldcg(vrow + lane) : 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t x;
          if (narrow) x = __shfl_sync(0xffffffffu, vw, bq[q] & 31);
          else x = mq[q] ? __ldcg(vrow + bq[q]) : 0;
          mq[q] &= ~x;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          fq[q] = mq[q] ? __ldcg(fpar + uint64_t(uq[q]) * W32 + bq[q]) & mq[q] : 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (fq[q]) {
            atomicOr(&cacc[bq[q]], fq[q]);
            any = true;
          }
        if (!__any_sync(0xffffffffu, any)) continue;
        __syncwarp();
        const bool owner = r.rev.row_chunk[v + 1] - r.rev.row_chunk[v] == 1;
        bool got = false;
        for (uint32_t b = lane; b < W32; b += 32) {
          uint32_t a = cacc[b];
          if (!a) continue;
          cacc[b] = 0;
          uint32_t* vw = r.vis + uint64_t(v) * W32 + b;
          a &= ~__ldcg(vw);
          if (!a) continue;
          uint32_t nb;
          if (owner) {
            nb = a;
            *vw = __ldcg(vw) | a;
          } else {
            nb = a & ~atomicOr(vw, a);
            if (!nb) continue;
          }
          int8_t* rb = r.regs + uint64_t(v) * r.Jp + b * 32;
          for (uint32_t t = nb; t; t &= t - 1) rb[__ffs(t) - 1] = 0;
          if (owner) fnxt[uint64_t(v) * W32 + b] |= nb;
          else atomicOr(fnxt + uint64_t(v) * W32 + b, nb);
          marked += __popc(nb);
          got = true;
        }
        __syncwarp();
        if (__any_sync(0xffffffffu, got) && lane == 0)
          cascade_mark(v, base, stamp, r.cstamp, r.dirty, &r.ctl->dirty_count, r.fwd.row_chunk,
                       rows_n, chunks_n, &qc[gn], ws);
      }
      // Small target rows: item-parallel straight over their flat item list
      // (no chunk indirection), four items per lane with every load stage
      // issued for all four first; one atomicOr per newly reached word.
      // Static grid-stride (dynamic claiming measured slower here: C2/C3 IC).
      const uint64_t nsi = r.rev.nsmall_items;
      for (uint64_t k0 = my_warp * 128; k0 < nsi; k0 += n_warps * 128) {
        uint64_t iq[4];
        uint32_t vq[4], uq[4], mq[4], bq[4], xq[4], fq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint64_t kk = k0 + lane + 32 * q;
          iq[q] = kk < nsi ? __ldg(r.rev.small_items + kk) : 0;
          mq[q] = kk < nsi ? 1u : 0u;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          vq[q] = mq[q] ? __ldg(r.rev.row + iq[q]) : 0;
          uq[q] = mq[q] ? __ldg(r.rev.other + iq[q]) : 0;
          bq[q] = mq[q] ? __ldg(r.rev.batch + iq[q]) : 0;
          mq[q] = mq[q] ? __ldg(r.rev.mask + iq[q]) : 0;
        }
        // the target's visited word and the parent's fresh word together
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          xq[q] = mq[q] ? __ldcg(r.vis + uint64_t(vq[q]) * W32 + bq[q]) : 0xFFFFFFFFu;
          fq[q] = mq[q] ? __ldcg(fpar + uint64_t(uq[q]) * W32 + bq[q]) : 0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t c = fq[q] & mq[q] & ~xq[q];
          if (c) claim(vq[q], bq[q], c);
        }
        __syncwarp();
        hook();
      }
    } else {
      for_frontier_items(r.fwd, r.q.chunks[g], nc, &cnt[8 + g], ws, n_warps, visit, hook);
    }
    __syncwarp();
    if (ws.nr || ws.nd) flush();
  };
  // Final clean-up: fresh bits left by the last two levels.
  auto finish = [&](uint32_t L, bool solo) {
    const int g = L % 4, gp = (L + 3) % 4;
    const uint64_t my_warp = solo ? (threadIdx.x >> 5) : gwarp;
    const uint64_t n_warps = solo ? kWarps : nw;
    clear_rows(r.fresh[L % 3], r.q.rows[g], qrows(qc, g), W32, my_warp, n_warps, lane);
    clear_rows(r.fresh[(L + 2) % 3], r.q.rows[gp], qrows(qc, gp), W32, my_warp,
               n_warps, lane);
  };

  // Episodes: block 0 iterates small-frontier levels alone (the rest of the
  // grid parks on a release word); large frontiers run grid-wide with one
  // grid barrier per level.  Episode 0 starts right after the commit, so a
  // tiny cascade never touches a grid barrier.
  uint32_t L = 1, e = 0;
  for (;;) {
    uint32_t code = 0;
    if (blockIdx.x == 0) {
      __syncthreads();
      for (;;) {
        const uint32_t nc = qchunks(qc, L % 4);
        if (nc == 0) {
          // a last frontier of rows without device-graph out-edges is still a
          // level of the reference's loop (engine.cpp:121-124): count its rows
          if (CNT && threadIdx.x == 0)
            r.ctl->cnt_cas_rows += qrows(qc, L % 4);
          finish(L, true);
          code = 1;
          break;
        }
        if (nc > kSoloChunks) break;
        level(L, true);
        __syncthreads();
        ++L;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (code == 0 && a.park && !*a.awake) {  // parked blocks join for the grid levels
          park_wake(a.park, kWakeCascade, a.step, base);
          *a.awake = 1;
        }
        if (code == 1 && a.defer_e) {
          *a.defer_e = e;  // the caller publishes the final release after its round end
        } else {
          __threadfence();
          atomicExch(&r.ctl->release, (static_cast<unsigned long long>(base) << 32) |
                                          (uint64_t(e & 0xFFFu) << 20) | (uint64_t(L) << 2) | code);
        }
      }
    } else {
      if (threadIdx.x == 0) {
        unsigned long long rv;
        for (;;) {
          rv = ld_volatile(&r.ctl->release);
          if ((rv >> 32) == base && ((rv >> 20) & 0xFFFu) == (e & 0xFFFu)) break;
          __nanosleep(256);
        }
        __threadfence();
        s_release = rv;
      }
      __syncthreads();
      L = uint32_t((s_release >> 2) & 0x3FFFFu);
      code = uint32_t(s_release & 3u);
    }
    ++e;
    if (code == 1) break;
    for (;;) {  // grid-wide levels while the frontier is large
      if (qchunks(qc, L % 4) <= kSoloChunks) break;
      level(L, false);
      // VISITED counts of the grid levels land before the barrier, so block 0
      // holds the complete count when the cascade ends in its solo episode
      for (int o = 16; o; o >>= 1) marked += __shfl_xor_sync(0xffffffffu, marked, o);
      if (lane == 0 && marked) atomicAdd(&r.ctl->visited, marked);
      marked = 0;
      grid.sync();
      ++L;
    }
  }
  for (int o = 16; o; o >>= 1) marked += __shfl_xor_sync(0xffffffffu, marked, o);
  if (lane == 0 && marked) atomicAdd(&r.ctl->visited, marked);
  if (gwarp == 0 && lane == 0) {
    r.ctl->levels = L;
    r.ctl->tick = base + L + 2;
  }
  return base + L + 2;
}

__global__ void __launch_bounds__(kThreads, DFS_SIM_MINB) k_cascade(CasArgs a) {
  __shared__ WarpStage stage[kWarps];
  __shared__ unsigned long long s_release;
  __shared__ RankDev s_r;
  extern __shared__ unsigned long long dyn_smem[];
  if (threadIdx.x == 0) s_r = a.r;
  __syncthreads();
  cg::grid_group grid = cg::this_grid();
  const CasOpts o{a.choice, a.seed, a.dbg, a.pull_f, 0};
  const uint32_t base = ld_volatile(&a.r.ctl->tick);
  grid.sync();  // every block holds `base` before block 0 can finish a solo cascade
  cascade_body<0>(s_r, o, grid, stage, s_release, reinterpret_cast<uint32_t*>(dyn_smem), base);
}

// ---------------------------------------------------------------- round end
__device__ __forceinline__ void round_end_covered(const RunArrays& ra,
                                                  unsigned long long covered, uint32_t k,
                                                  uint32_t R, double eps) {
  const double score = __ddiv_rn(double(covered), double(R));  // runtime.cpp:130
  RunCtl* c = ra.ctl;
  const uint32_t step = c->step;
  ra.seeds[step] = c->choice;
  ra.traj[step] = score;
  // runtime.cpp:139-140
  const bool rebuild =
      step + 1 < k && __dadd_rn(score, -c->oldscore) > __dmul_rn(eps, score);
  c->rebuild_now = rebuild ? 1u : 0u;
  if (rebuild) {
    ra.rebuild_rounds[c->n_rebuilds++] = step;
    c->oldscore = score;
  }
  c->step = step + 1;
}

__device__ __forceinline__ void round_end_body(const RunArrays& ra, RankCtl* const* ctls,
                                               uint32_t mu, uint32_t k, uint32_t R, double eps) {
  if (threadIdx.x || blockIdx.x) return;
  unsigned long long covered = 0;  // collectives.cpp:96-113 (exact u64 sum)
  for (uint32_t t = 0; t < mu; ++t) covered += ld_volatile(&ctls[t]->visited);
  round_end_covered(ra, covered, k, R, eps);
}

__global__ void k_round_end(RunArrays ra, RankCtl* const* ctls, uint32_t mu, uint32_t k,
                            uint32_t R, double eps) {
  round_end_body(ra, ctls, mu, k, R, eps);
}

}  // namespace

// ---------------------------------------------------------------- whole run
// The greedy loop of proj/src/runtime.cpp:87-154 as ONE persistent
// cooperative kernel: fill -> simulate -> score, then K rounds of rescore ->
// (binomial sum) -> argmax -> commit+cascade -> covered count / rebuild
// decision -> (fill -> simulate -> score).  Every decision is read by all
// blocks after a grid barrier, so the host launches once per run.  Phase
// times are accumulated by block 0 from the global nanosecond timer.
struct RunArgs {
  const RankDev* ranks;  // device array [mu]
  uint32_t mu, k, R, n;
  double eps;
  int cap, dbg, sim_pull_f, cas_pull_f, K;
  RunArrays ra;
  const double* const* parts;
  RankCtl* const* ctls;
  double* reduced;
  unsigned long long* phase_ns;  // fill, simulate, select, cascade
  int peer;                      // 1: one partition per GPU, exchange over peer memory
  PeerView pv;
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- peer exchange primitives (system-scope release/acquire over NVLink)
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Peer data read after a barrier's acquire: explicit system-scope relaxed
// loads (the barrier's acquire orders them; L1 is never consulted).
__device__ __forceinline__ unsigned int ld_relaxed_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
  return __longlong_as_double(
      static_cast<long long>(ld_relaxed_sys(reinterpret_cast<const unsigned long long*>(p))));
}

// Cross-GPU barrier of epoch `ep`, called by every thread of the grid: after
// it, every write any rank made before arriving is visible here.  Lane t of
// block 0's first warp waits for rank t; a peer that never arrives (dead
// process) releases the wait after pv.timeout_ns (DFS_PEER_TIMEOUT_S) and is
// reported by the host; once that happened, later barriers of the launch do
// not wait any more (the results are discarded anyway).
__device__ __noinline__ void peer_sync(const PeerView& pv, unsigned long long ep,
                                      unsigned long long timeouts0) {
  cg::grid_group grid = cg::this_grid();
  __threadfence_system();
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const unsigned lane = threadIdx.x;
    PeerBox* mine = pv.box[pv.rank];
    if (lane == 0) st_release_sys(&mine->arrive, ep);
    // a barrier of THIS launch already timed out (timeouts0: the count when
    // the launch started): stop waiting, the host discards the results
    const bool failed = ld_volatile(&mine->timeouts) != timeouts0;
    if (!failed && lane < pv.world && lane != pv.rank) {
      const unsigned long long t0 = global_ns();
      while (ld_acquire_sys(&pv.box[lane]->arrive) < ep) {
        if (global_ns() - t0 > pv.timeout_ns) {
          atomicAdd(&mine->timeouts, 1ull);
          break;
        }
        __nanosleep(64);
      }
    }
    __syncwarp();
    __threadfence_system();
  }
  grid.sync();
}

// Partial scores of every rank summed in the reference's binomial-tree order
// (collectives.cpp:51-59) straight from peer memory.
__device__ __forceinline__ double peer_reduced(const PeerView& pv, uint32_t v) {
  double acc[kMaxPeers];
#pragma unroll 4
  for (uint32_t t = 0; t < pv.world; ++t) acc[t] = ld_relaxed_sys(pv.scores[t] + v);
  for (uint32_t st = 1; st < pv.world; st <<= 1)
    for (uint32_t t = 0; t + st < pv.world; t += 2 * st) acc[t] = __dadd_rn(acc[t], acc[t + st]);
  return acc[0];
}

// Out-of-line phase bodies keep the register allocation of each phase local.
#ifndef DFS_PHASE_INLINE
#define DFS_PHASE_INLINE __noinline__
#endif
template <int JAC, int CNT>
__device__ DFS_PHASE_INLINE uint32_t run_simulate(const RankDev& r, const SimOpts& o, WarpStage* stage,
                                              unsigned long long& s_release,
                                              unsigned long long* dyn, uint32_t base) {
  cg::grid_group grid = cg::this_grid();
  return simulate_body<JAC, CNT>(r, o, grid, stage, s_release, dyn, base);
}
template <int CNT>
__device__ DFS_PHASE_INLINE uint32_t run_cascade(const RankDev& r, const CasOpts& o, WarpStage* stage,
                                             unsigned long long& s_release, uint32_t* dyn,
                                             uint32_t base) {
  cg::grid_group grid = cg::this_grid();
  return cascade_body<CNT>(r, o, grid, stage, s_release, dyn, base);
}

// PARKED: the parked-grid round loop (one partition, no peers); else the
// general loop (several partitions on this GPU, or peer mode).  Separate
// instantiations keep each loop's live state out of the other's register
// allocation (the phase bodies are out-of-line calls).
template <int JAC, int CNT, int PARKED>
__global__ void __launch_bounds__(kThreads, DFS_SIM_MINB) k_run(RunArgs a) {
  __shared__ WarpStage stage[kWarps];
  __shared__ unsigned long long s_release;
  __shared__ RankDev s_r;
  __shared__ Best sb[kWarps];
  // Per-partition stamp bases, tracked identically by every block (each phase
  // returns the next one) so that no block reads a tick another block may
  // already have advanced.  Read once here, before the first grid barrier.
  __shared__ uint32_t s_tick[64];
  extern __shared__ unsigned long long dyn_smem[];
  cg::grid_group grid = cg::this_grid();
  for (uint32_t t = threadIdx.x; t < a.mu; t += blockDim.x) s_tick[t] = ld_volatile(&a.ranks[t].ctl->tick);
  __syncthreads();
  const bool timer = blockIdx.x == 0 && threadIdx.x == 0;
  // Loop-carried per-block state lives in shared memory: the phase bodies
  // are out-of-line calls, and every register the caller keeps live across
  // them is one the (interprocedurally allocated) callee cannot use.
  __shared__ unsigned long long s_t0;
  __shared__ uint32_t s_cur_rank, s_first_fill;
  if (threadIdx.x == 0) {
    s_t0 = timer ? global_ns() : 0;
    s_cur_rank = 0xFFFFFFFFu;
    s_first_fill = 1;
  }
  __syncthreads();
  auto phase = [&](int which) {
    if (timer) {
      const unsigned long long t1 = global_ns();
      a.phase_ns[which] += t1 - s_t0;
      s_t0 = t1;
    }
  };
  auto load_rank = [&](uint32_t t) {  // s_r is never modified once loaded
    if (t == s_cur_rank) return;
    __syncthreads();
    if (threadIdx.x == 0) {
      s_r = a.ranks[t];
      s_cur_rank = t;
    }
    __syncthreads();
  };
  const SimOpts so{a.cap, a.dbg, a.sim_pull_f};
  // no peers: argmax through the segment cache (over the binomial-order sum
  // of the partitions' scores when mu > 1), and rounds with few dirty rows
  // run their select step in block 0 alone
  const bool segs = !a.peer;
  const double* segsrc = a.mu > 1 ? a.reduced : a.ranks[0].scores;
  // reduced score of v from the mu partial vectors (collectives.cpp:51-59)
  auto reduce_row = [&](uint32_t v) {
    double acc[64];
    for (uint32_t t = 0; t < a.mu; ++t) acc[t] = __ldcg(a.parts[t] + v);
    for (uint32_t st = 1; st < a.mu; st <<= 1)
      for (uint32_t t = 0; t + st < a.mu; t += 2 * st) acc[t] = __dadd_rn(acc[t], acc[t + st]);
    a.reduced[v] = acc[0];
  };
  // (s_first_fill: the first fill ran as a separate full-occupancy launch)
  auto rebuild = [&]() {  // fill -> simulate -> full rescore, every partition
    if (!s_first_fill)
      for (uint32_t t = 0; t < a.mu; ++t) {
        load_rank(t);
        fill_body(s_r.n, s_r.J, s_r.Jp, s_r.jkey, s_r.vis, s_r.regs, s_r.ctl, s_r.pristine, true);
      }
    __syncthreads();
    if (threadIdx.x == 0) s_first_fill = 0;
    grid.sync();
    phase(0);
    for (uint32_t t = 0; t < a.mu; ++t) {
      load_rank(t);
      const uint32_t nt = run_simulate<JAC, CNT>(s_r, so, stage, s_release, dyn_smem, s_tick[t]);
      grid.sync();
      if (threadIdx.x == 0) s_tick[t] = nt;
    }
    phase(1);
    for (uint32_t t = 0; t < a.mu; ++t) {
      load_rank(t);
      score_body(s_r.regs, s_r.n, s_r.J, s_r.Jp, a.K, 1, s_r.dirty, s_r.ctl, s_r.scores,
                 reinterpret_cast<uint32_t*>(dyn_smem));
    }
    grid.sync();
    if (segs) {  // full rescore: rebuild the whole argmax cache
      if (a.mu > 1) {
        treesum_body(a.parts, a.mu, a.n, a.reduced);
        grid.sync();
      }
      const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
      const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
      for (uint64_t sg = gw; sg < a.ra.nseg; sg += nw)
        seg_recompute(segsrc, a.n, uint32_t(sg), a.ra);
      grid.sync();
    }
  };
  bool rebuilt = true;
  // peer mode: this rank reduces and searches the id slice [plo, phi)
  unsigned long long ep = a.peer ? ld_volatile(&a.pv.box[a.pv.rank]->arrive) : 0;
  const unsigned long long to0 = a.peer ? ld_volatile(&a.pv.box[a.pv.rank]->timeouts) : 0;
  const uint32_t pslice = a.peer ? (a.n + a.pv.world - 1) / a.pv.world : 0;
  const uint32_t plo = a.peer ? min(a.n, a.pv.rank * pslice) : 0;
  const uint32_t phi = a.peer ? min(a.n, plo + pslice) : 0;
  const uint32_t pnseg = (phi - plo + kSeg - 1) / kSeg;  // slice segments (peer mode)
  const bool tr = (a.dbg & 4) && blockIdx.x == 0 && threadIdx.x == 0;  // DFS_DBG bit 2
  // select (runtime.cpp:88-121) through the argmax cache.  Small dirty sets:
  // block 0 rescores them, refreshes their segments and picks the winner with
  // block barriers only (select_solo, block 0 alone); larger ones run
  // grid-wide (select_grid, every block).
  auto select_solo = [&](uint32_t step, bool was_rebuilt) {
    if (tr) trace(6, step, 0);
    if (!was_rebuilt) {
      for (uint32_t t = 0; t < a.mu; ++t) {
        load_rank(t);
        score_body(s_r.regs, s_r.n, s_r.J, s_r.Jp, a.K, 0, s_r.dirty, s_r.ctl, s_r.scores,
                   reinterpret_cast<uint32_t*>(dyn_smem), true);
      }
      __syncthreads();
      if (a.mu > 1) {  // rows dirty in any partition: new binomial sums
        for (uint32_t t = 0; t < a.mu; ++t) {
          const RankDev& rt = a.ranks[t];
          const uint32_t c = ld_volatile(&rt.ctl->dirty_count);
          for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) reduce_row(__ldcg(rt.dirty + i));
        }
        __syncthreads();
      }
      if (tr) trace(5, step, 0);
      // duplicates of one segment compute identical values (benign)
      for (uint32_t t = 0; t < a.mu; ++t) {
        const RankDev& rt = a.ranks[t];
        const uint32_t c = ld_volatile(&rt.ctl->dirty_count);
        for (uint32_t i = threadIdx.x >> 5; i < c; i += kWarps)
          seg_recompute(segsrc, a.n, __ldcg(rt.dirty + i) / kSeg, a.ra);
      }
      __syncthreads();
      if (tr) trace(6, step, 1);
    }
    const Best t = seg_combine(a.ra, sb, a.ra.nseg);
    if (threadIdx.x == 0) commit_choice(t, a.ra);
    __syncthreads();
    if (tr) trace(7, step, ld_volatile(&a.ra.ctl->choice));
  };
  auto select_grid = [&](uint32_t step) {
    for (uint32_t t = 0; t < a.mu; ++t) {
      load_rank(t);
      score_body(s_r.regs, s_r.n, s_r.J, s_r.Jp, a.K, 0, s_r.dirty, s_r.ctl, s_r.scores,
                 reinterpret_cast<uint32_t*>(dyn_smem));
    }
    grid.sync();
    const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t gthreads = uint64_t(gridDim.x) * blockDim.x;
    if (a.mu > 1) {
      for (uint32_t t = 0; t < a.mu; ++t) {
        const RankDev& rt = a.ranks[t];
        const uint32_t c = ld_volatile(&rt.ctl->dirty_count);
        for (uint64_t i = gtid; i < c; i += gthreads) reduce_row(__ldcg(rt.dirty + i));
      }
      grid.sync();
    }
    const uint64_t gw = gtid >> 5, nw = gthreads >> 5;
    const uint32_t stampv = step + 1;
    for (uint32_t t = 0; t < a.mu; ++t) {
      const RankDev& rt = a.ranks[t];
      const uint32_t c = ld_volatile(&rt.ctl->dirty_count);
      for (uint64_t i = gw; i < c; i += nw) {
        const uint32_t sg = __ldcg(rt.dirty + i) / kSeg;
        unsigned prev = 0;
        if (lane_id() == 0) prev = atomicExch(&a.ra.seg_stamp[sg], stampv);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev != stampv) seg_recompute(segsrc, a.n, sg, a.ra);
      }
    }
    grid.sync();
    if (blockIdx.x == 0) {
      const Best t = seg_combine(a.ra, sb, a.ra.nseg);
      if (threadIdx.x == 0) commit_choice(t, a.ra);
      __syncthreads();
    }
  };
  // Parked-grid rounds (one partition, no peers): the other blocks park on
  // park_seq while block 0 runs whole rounds alone (solo select, solo cascade
  // levels, round end) without grid barriers; block 0 wakes them with the
  // round and stamp base when a round needs the grid (a large dirty set, a
  // large cascade level, a rebuild) and once at the end.  A round of C2's
  // tail (a few solo cascade levels) costs one block's work instead of two
  // grid barriers plus the release hand-offs.
  if (PARKED) {
    __shared__ uint32_t s_awake, s_defer_e, s_wake[4];
    // Every block executes rebuild() at ONE call site (the interprocedural
    // register allocation of the out-of-line simulate phase depends on its
    // call sites): the loop starts with the initial build for everyone, and
    // block 0 breaks out of its solo rounds when a rebuild is due.
    uint32_t seen = 0, step0 = 0;
    bool rebuilt = true;
    uint32_t reason = kWakeRebuild;  // the initial fill -> simulate -> score
    for (;;) {
      if (reason == kWakeRebuild) {
        rebuild();
        if (blockIdx.x == 0 && step0) phase(2);
        rebuilt = true;
      }
      if (blockIdx.x != 0) {
        if (threadIdx.x == 0) {
          uint32_t v;
          for (;;) {
            v = ld_volatile(&a.ra.ctl->park_seq);
            if (v != seen) break;
            __nanosleep(128);
          }
          __threadfence();
          s_wake[0] = ld_volatile(&a.ra.ctl->park_reason);
          s_wake[1] = ld_volatile(&a.ra.ctl->park_step);
          s_wake[3] = v;
          s_tick[0] = ld_volatile(&a.ra.ctl->park_base);
        }
        __syncthreads();
        reason = s_wake[0];
        const uint32_t step = s_wake[1];
        seen = s_wake[3];
        __syncthreads();
        if (reason == kWakeDone) break;
        if (reason == kWakeRebuild) continue;
        if (reason == kWakeSelect) select_grid(step);
        load_rank(0);
        const CasOpts co{&a.ra.ctl->choice, 0, a.dbg, a.cas_pull_f, CNT};
        const uint32_t nt =
            run_cascade<CNT>(s_r, co, stage, s_release, reinterpret_cast<uint32_t*>(dyn_smem), s_tick[0]);
        if (threadIdx.x == 0) s_tick[0] = nt;  // (the next wake sets it again)
        continue;
      }
      // block 0: rounds until a rebuild is due or the loop ends
      reason = kWakeDone;
      for (; step0 < a.k; ++step0) {
        const uint32_t step = step0;
        const uint32_t nd = rebuilt ? 0u : ld_volatile(&a.ra.ctl->snap_dirty);
        if (tr) trace(4, step, nd);
        bool awake = false;
        if (nd <= kSoloDirty) {
          select_solo(step, rebuilt);
        } else {
          if (threadIdx.x == 0) park_wake(a.ra.ctl, kWakeSelect, step, s_tick[0]);
          awake = true;
          select_grid(step);
        }
        rebuilt = false;
        phase(2);
        load_rank(0);
        if (threadIdx.x == 0) {
          s_awake = awake ? 1u : 0u;
          s_defer_e = 0;
        }
        __syncthreads();
        const uint32_t base = s_tick[0];
        CasOpts co{&a.ra.ctl->choice, 0, a.dbg, a.cas_pull_f, CNT};
        co.park = a.ra.ctl;
        co.step = step;
        co.awake = &s_awake;
        co.defer_e = &s_defer_e;
        const uint32_t nt =
            run_cascade<CNT>(s_r, co, stage, s_release, reinterpret_cast<uint32_t*>(dyn_smem), base);
        __syncthreads();  // block 0's VISITED counts are in (each warp adds at the cascade end)
        if (threadIdx.x == 0) {
          s_tick[0] = nt;
          a.ra.ctl->snap_dirty = ld_volatile(&a.ranks[0].ctl->dirty_count);
          round_end_covered(a.ra, ld_volatile(&a.ranks[0].ctl->visited), a.k, a.R, a.eps);
          // blocks that joined this round's cascade leave it now (deferred release)
          __threadfence();
          atomicExch(&a.ranks[0].ctl->release,
                     (static_cast<unsigned long long>(base) << 32) |
                         (uint64_t(s_defer_e & 0xFFFu) << 20) | (uint64_t(nt - base - 2) << 2) | 1ull);
        }
        __syncthreads();
        phase(3);
        if (step + 1 < a.k && ld_volatile(&a.ra.ctl->rebuild_now)) {
          if (threadIdx.x == 0) park_wake(a.ra.ctl, kWakeRebuild, step, s_tick[0]);
          reason = kWakeRebuild;
          ++step0;
          break;
        }
      }
      if (reason == kWakeDone) {
        if (threadIdx.x == 0) park_wake(a.ra.ctl, kWakeDone, a.k, 0);
        break;
      }
    }
    return;
  } else {
  rebuild();
  for (uint32_t step = 0; step < a.k; ++step) {
    if (tr) trace(4, step, 0);
    if (segs) {
      // select (runtime.cpp:88-121) through the argmax cache.  Small dirty
      // sets: block 0 rescores them, refreshes their segments and picks the
      // winner with block barriers only; the other blocks go straight to the
      // cascade, whose first (solo) levels block 0 runs as well.
      // dirty rows over all partitions (snapshot of the previous round end)
      const uint32_t nd = rebuilt ? 0u : ld_volatile(&a.ra.ctl->snap_dirty);
      if (nd <= kSoloDirty) {
        if (blockIdx.x == 0) select_solo(step, rebuilt);
      } else {
        select_grid(step);
      }
      rebuilt = false;
      // the cascade's commit (block 0, warp 0) reads the choice; the other
      // blocks wait on its release word, so no grid barrier is needed here
    } else if (!rebuilt) {  // peer mode: rows dirtied by the last cascade
      for (uint32_t t = 0; t < a.mu; ++t) {
        load_rank(t);
        score_body(s_r.regs, s_r.n, s_r.J, s_r.Jp, a.K, 0, s_r.dirty, s_r.ctl, s_r.scores,
                   reinterpret_cast<uint32_t*>(dyn_smem));
      }
      grid.sync();
      if (tr) trace(5, step, ld_volatile(&a.ranks[0].ctl->dirty_count));
    }
    if (a.peer) {
      // reduce_to_root + root argmax + broadcast (runtime.cpp:88-121) as: every
      // rank publishes which rows it rescored -> barrier -> each rank re-sums
      // (binomial order, straight from the peers' partial vectors) only the
      // rows of ITS id slice that some rank rescored, refreshes the slice's
      // segment cache and publishes its best -> barrier -> every rank picks
      // the same winner.  After a rebuild every row counts as rescored.
      if (blockIdx.x == 0 && threadIdx.x == 0)
        a.pv.box[a.pv.rank]->ndirty =
            rebuilt ? kAllDirty : ld_volatile(&a.ranks[0].ctl->dirty_count);
      peer_sync(a.pv, ++ep, to0);
      const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
      const uint64_t gthreads = uint64_t(gridDim.x) * blockDim.x;
      const uint64_t gw = gtid >> 5, nw = gthreads >> 5;
      if (rebuilt) {  // rebuilds are decided identically on every rank
        for (uint64_t v = plo + gtid; v < phi; v += gthreads) a.reduced[v] = peer_reduced(a.pv, uint32_t(v));
        grid.sync();
        for (uint64_t sg = gw; sg < pnseg; sg += nw) seg_recompute(a.reduced, phi, uint32_t(sg), a.ra, plo);
      } else {
        for (uint32_t q = 0; q < a.pv.world; ++q) {
          const uint32_t c = ld_relaxed_sys(&a.pv.box[q]->ndirty);
          const uint32_t* dq = a.pv.dirty[q];
          for (uint64_t i = gtid; i < c; i += gthreads) {
            const uint32_t v = ld_relaxed_sys(dq + i);
            if (v >= plo && v < phi) a.reduced[v] = peer_reduced(a.pv, v);
          }
        }
        grid.sync();
        const uint32_t stampv = step + 1;
        for (uint32_t q = 0; q < a.pv.world; ++q) {
          const uint32_t c = ld_relaxed_sys(&a.pv.box[q]->ndirty);
          const uint32_t* dq = a.pv.dirty[q];
          for (uint64_t i = gw; i < c; i += nw) {
            const uint32_t v = ld_relaxed_sys(dq + i);
            if (v < plo || v >= phi) continue;  // warp-uniform
            const uint32_t sg = (v - plo) / kSeg;
            unsigned prev = 0;
            if (lane_id() == 0) prev = atomicExch(&a.ra.seg_stamp[sg], stampv);
            prev = __shfl_sync(0xffffffffu, prev, 0);
            if (prev != stampv) seg_recompute(a.reduced, phi, sg, a.ra, plo);
          }
        }
      }
      grid.sync();
      if (blockIdx.x == 0) {
        const Best t = seg_combine(a.ra, sb, pnseg);
        if (threadIdx.x == 0) {
          PeerBox* mine = a.pv.box[a.pv.rank];
          mine->best_s = t.s;
          mine->best_v = t.v;
          mine->minu = t.minu;
        }
      }
      peer_sync(a.pv, ++ep, to0);
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        Best t{0.0, 0xFFFFFFFFu, 0xFFFFFFFFu};
        for (uint32_t q = 0; q < a.pv.world; ++q) {  // ascending id slices
          const PeerBox* b = a.pv.box[q];
          t = best_of(t, Best{ld_relaxed_sys(&b->best_s), ld_relaxed_sys(&b->best_v),
                              ld_relaxed_sys(&b->minu)});
        }
        commit_choice(t, a.ra);
      }
      grid.sync();
      rebuilt = false;
    }
    phase(2);
    for (uint32_t t = 0; t < a.mu; ++t) {
      load_rank(t);
      const CasOpts co{&a.ra.ctl->choice, 0, a.dbg, a.cas_pull_f, CNT};
      const uint32_t nt =
          run_cascade<CNT>(s_r, co, stage, s_release, reinterpret_cast<uint32_t*>(dyn_smem), s_tick[t]);
      grid.sync();
      if (threadIdx.x == 0) s_tick[t] = nt;
    }
    // dirty rows for the next select, snapshotted before the barrier below: the
    // next cascade (block 0 may start it early) overwrites the counts
    if (segs && blockIdx.x == 0 && threadIdx.x == 0) {
      uint32_t nd = 0;
      for (uint32_t t = 0; t < a.mu; ++t) nd += ld_volatile(&a.ranks[t].ctl->dirty_count);
      a.ra.ctl->snap_dirty = nd;
    }
    if (a.peer) {  // allreduce(count_visited) (runtime.cpp:129, collectives.cpp:96-113)
      if (blockIdx.x == 0 && threadIdx.x == 0)
        a.pv.box[a.pv.rank]->visited = ld_volatile(&a.ranks[0].ctl->visited);
      peer_sync(a.pv, ++ep, to0);
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long covered = 0;
        for (uint32_t q = 0; q < a.pv.world; ++q) covered += ld_relaxed_sys(&a.pv.box[q]->visited);
        round_end_covered(a.ra, covered, a.k, a.R, a.eps);
      }
    } else {
      round_end_body(a.ra, a.ctls, a.mu, a.k, a.R, a.eps);
    }
    grid.sync();
    phase(3);
    if (step + 1 < a.k && ld_volatile(&a.ra.ctl->rebuild_now)) {
      rebuild();
      phase(2);
      rebuilt = true;
    }
  }
  }  // !PARKED
}

// ================================================================= launchers
static unsigned long long g_launches = 0;
unsigned long long launches() { return g_launches; }

void dump_trace() {
  static unsigned long long h[8192][4];
  unsigned int n = 0;
  DFS_CUDA(cudaDeviceSynchronize());
  DFS_CUDA(cudaMemcpyFromSymbol(&n, g_trace_n, sizeof n));
  n = n > 8192 ? 8192 : n;
  DFS_CUDA(cudaMemcpyFromSymbol(h, g_trace, sizeof(unsigned long long) * 4 * n));
  static const char* names[] = {"sim",   "sim-solo", "cas",    "cas-solo",
                                "round", "rescored", "argmax", "chosen"};
  for (unsigned i = 0; i < n; ++i)
    fprintf(stderr, "trace %-8s idx=%-4llu nc=%-8llu dt=%.1f us\n", names[h[i][0] & 7], h[i][1],
            h[i][2], i ? (h[i][3] - h[i - 1][3]) / 1965.0 : 0.0);
  unsigned int z = 0;
  DFS_CUDA(cudaMemcpyToSymbol(g_trace_n, &z, sizeof z));
}
size_t graph_prepare_tmp_bytes(uint64_t m, uint32_t n) {
  size_t sort_bytes = 0, scan_bytes = 0, max_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, m ? m : 1);
  scan_bytes = scan_tmp_bytes(n + 1);
  cub::DeviceScan::InclusiveScan(nullptr, max_bytes, (const uint32_t*)nullptr, (uint64_t*)nullptr,
                                 MaxU64{}, n ? n : 1);
  // layout: iota(m) | cub temp
  return (m + 16) * sizeof(uint32_t) + std::max(sort_bytes, std::max(scan_bytes, max_bytes)) +
         1024;
}

size_t scan_tmp_bytes(uint64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, bytes, (const uint32_t*)nullptr, (uint64_t*)nullptr,
                                 cuda::std::plus<uint64_t>{}, uint64_t(0), n ? n : 1);
  return bytes + 256;
}

void scan_u32_u64(const uint32_t* in, uint64_t* out, uint64_t n, void* tmp, size_t tmp_bytes,
                  cudaStream_t s) {
  // exclusive scan of n values into out[0..n); out[n] = total via a scan of n+1
  // values whose last input is read as 0 (caller guarantees in[n] == 0).
  size_t bytes = tmp_bytes;
  DFS_CUDA(cub::DeviceScan::ExclusiveScan(tmp, bytes, in, out, cuda::std::plus<uint64_t>{},
                                          uint64_t(0), n + 1, s));
}

void launch_graph_prepare(DevGraph& g, void* tmp, size_t tmp_bytes, cudaStream_t s) {
  const uint64_t m = g.m;
  char* p = static_cast<char*>(tmp);
  uint32_t* iota = reinterpret_cast<uint32_t*>(p);
  p += (m + 16) * sizeof(uint32_t);
  void* cubtmp = p;
  size_t cub_bytes = tmp_bytes - size_t(p - static_cast<char*>(tmp));

  // indeg doubles as the run-end array until the in-degrees are written
  DFS_CUDA(cudaMemsetAsync(g.indeg, 0, (size_t(g.n) + 1) * sizeof(uint32_t), s));
  DFS_CUDA(cudaMemsetAsync(g.toff, 0, sizeof(uint64_t), s));
  if (!m) {
    DFS_CUDA(cudaMemsetAsync(g.toff, 0, (size_t(g.n) + 1) * sizeof(uint64_t), s));
    return;
  }
  k_src<<<grid_for(uint64_t(g.n) * 32), kThreads, 0, s>>>(g.n, g.off, g.src);
  k_ehash<<<grid_for(m), kThreads, 0, s>>>(m, g.src, g.adj, g.ehash, iota);
  int end_bit = 1;
  while (end_bit < 32 && (uint64_t(1) << end_bit) < g.n) ++end_bit;
  size_t bytes = cub_bytes;
  // keys out = the targets in transposed order (tdst), values out = edge ids
  // (stable: a target's in-edges stay in CSR order)
  DFS_CUDA(cub::DeviceRadixSort::SortPairs(cubtmp, bytes, g.adj, g.tdst, iota, g.tedge, m, 0,
                                           end_bit, s));
  k_run_ends<<<grid_for(m), kThreads, 0, s>>>(m, g.tdst, g.indeg);
  bytes = cub_bytes;
  DFS_CUDA(cub::DeviceScan::InclusiveScan(cubtmp, bytes, g.indeg, g.toff + 1, MaxU64{}, g.n, s));
  k_indeg<<<grid_for(g.n), kThreads, 0, s>>>(g.n, g.toff, g.indeg);
  k_transpose_fields<<<grid_for(m), kThreads, 0, s>>>(m, g.tedge, g.src, g.tdst, g.tsrc, g.thash);
  DFS_CUDA(cudaGetLastError());
  g_launches += 5;  // own kernels (the sort and scan are cub's)
}

void launch_tweights(const DevGraph& g, int kind, uint32_t W, const uint32_t* w, uint32_t* tw,
                     cudaStream_t s) {
  if (!g.m) return;
  k_tweights<<<grid_for(g.m), kThreads, 0, s>>>(g.m, g.tedge, g.tdst, kind, W, g.indeg, w, tw);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_weights(const DevGraph& g, int kind, uint32_t W, uint32_t* w, cudaStream_t s) {
  if (!g.m) return;
  k_weights<<<grid_for(g.m), kThreads, 0, s>>>(g.m, kind, W, g.adj, g.indeg, w);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_rev_counts(const DevGraph& g, const uint64_t* pos_f, uint32_t* cnt, cudaStream_t s) {
  k_rev_counts<<<grid_for(g.m + 1), kThreads, 0, s>>>(g.m, g.tedge, pos_f, cnt);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_items_pass(const DevGraph& g, const uint32_t* w, const uint32_t* tw, const RankDev& r,
                       int dir, int fasst, int write, uint32_t* cnt, const uint64_t* pos_off,
                       Items& it, cudaStream_t s) {
  if (!g.m) return;
  const size_t smem = (size_t(r.Jp) + (1u << kLutBits) + 1) * sizeof(uint32_t);
  static bool attr = false;
  if (!attr) {
    DFS_CUDA(cudaFuncSetAttribute(k_items<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10));
    DFS_CUDA(cudaFuncSetAttribute(k_items<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10));
    attr = true;
  }
  const uint32_t* ph = dir ? g.thash : g.ehash;
  const uint32_t* pw = dir ? tw : w;
  const uint32_t* po = dir ? g.tsrc : g.adj;
  const uint32_t* pr = dir ? g.tdst : g.src;
  const int grid = grid_for(g.m, kThreads * 4);  // fewer, longer-lived blocks (smem fill)
  if (write)
    k_items<1><<<grid, kThreads, smem, s>>>(g.m, ph, pw, po, pr, r.x, r.J, r.Jp, fasst, cnt, pos_off,
                                            it.other, it.mask, it.batch, it.row, r.xlut);
  else
    k_items<0><<<grid, kThreads, smem, s>>>(g.m, ph, pw, po, pr, r.x, r.J, r.Jp, fasst, cnt, pos_off,
                                            nullptr, nullptr, nullptr, nullptr, r.xlut);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

uint64_t items_tiles(uint64_t npos) { return (npos + kTilePos - 1) / kTilePos; }

static ItemsPass items_pass_args(const DevGraph& g, const uint32_t* w, const uint32_t* tw,
                                 uint32_t wconst, const RankDev& r, int dir, int fasst) {
  ItemsPass a{};
  a.npos = g.m;
  a.n = g.n;
  a.p_hash = dir ? g.thash : g.ehash;
  a.p_w = wconst ? nullptr : (dir ? tw : w);
  a.Wc = wconst;
  a.p_other = dir ? g.tsrc : g.adj;
  a.p_row = dir ? g.tdst : g.src;
  a.x = r.x;
  a.glut = r.xlut;
  a.J = r.J;
  a.Jp = r.Jp;
  a.fasst = fasst;
  return a;
}

static size_t items_smem(const RankDev& r) {
  static bool attr = false;
  if (!attr) {
    DFS_CUDA(cudaFuncSetAttribute(k_items_onepass<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 << 10));
    DFS_CUDA(cudaFuncSetAttribute(k_items_onepass<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 << 10));
    DFS_CUDA(cudaFuncSetAttribute(k_items_sparse, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 << 10));
    DFS_CUDA(cudaFuncSetAttribute(k_items_sample, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10));
    attr = true;
  }
  return (size_t(r.Jp) + (1u << kLutBits) + 1) * sizeof(uint32_t);
}

void launch_items_sample(const DevGraph& g, const uint32_t* w, uint32_t wconst, const RankDev& r,
                         int fasst, uint64_t stride, unsigned long long* meta, cudaStream_t s) {
  if (!g.m) return;
  ItemsPass a = items_pass_args(g, w, nullptr, wconst, r, 0, fasst);
  a.meta = meta;
  const size_t smem = items_smem(r);
  k_items_sample<<<grid_for((g.m + stride - 1) / stride, kThreads * 4), kThreads, smem, s>>>(a, stride);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_items_onepass(const DevGraph& g, const uint32_t* w, const uint32_t* tw,
                          uint32_t wconst, const RankDev& r, int dir, int fasst, Items& it,
                          uint64_t cap, unsigned long long* tile_state, unsigned int* tile_ctr,
                          unsigned long long* meta, uint32_t* row_cnt, cudaStream_t s) {
  if (!g.m) return;
  ItemsPass a = items_pass_args(g, w, tw, wconst, r, dir, fasst);
  a.cap = cap;
  a.it_other = it.other;
  a.it_mask = it.mask;
  a.it_batch = it.batch;
  a.it_row = it.row;
  a.row_off = it.row_off;
  a.row_cnt = row_cnt;
  a.tile_state = tile_state;
  a.tile_ctr = tile_ctr;
  a.meta = meta;
  const size_t smem = items_smem(r);
  const bool filter = row_cnt != nullptr;
  const uint64_t tiles = items_tiles(g.m);
  if (filter) {
    int ps = 0;
    const size_t ssm = smem + sparse_extra_smem();
    DFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, k_items_sparse, kTileThreads, ssm));
    const int gs = int(std::min<uint64_t>(tiles, uint64_t(std::max(ps, 1)) * num_sms()));
    k_items_sparse<<<gs, kTileThreads, ssm, s>>>(a);
  } else {
    int per = 0;
    const size_t dsm = smem + size_t(kDeferWords) * sizeof(uint32_t);
    const void* fn = wconst ? (const void*)k_items_onepass<3> : (const void*)k_items_onepass<2>;
    DFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kTileThreads, dsm));
    const int grid = int(std::min<uint64_t>(tiles, uint64_t(std::max(per, 1)) * num_sms()));
    if (wconst) k_items_onepass<3><<<grid, kTileThreads, dsm, s>>>(a);
    else k_items_onepass<2><<<grid, kTileThreads, dsm, s>>>(a);
  }
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_row_chunks(uint32_t n, const Items& it, uint32_t* row_cnt, cudaStream_t s) {
  if (!n) return;
  k_row_chunks<<<grid_for(n), kThreads, 0, s>>>(n, it.row_off, row_cnt);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_fasst_stats(const DevGraph& g, const uint32_t* w, const uint32_t* x,
                        const uint32_t* xlut, uint32_t R, uint32_t mu, int sorted, int fill,
                        unsigned long long* out, cudaStream_t s) {
  DFS_CUDA(cudaMemsetAsync(out, 0, (2 * size_t(mu) + 3) * 8, s));
  if (!g.m) return;
  const size_t smem = (size_t(R) + (1u << kLutBits) + 2) * 4 + (2 * size_t(mu) + 3) * 8 + 16;
  DFS_CUDA(cudaFuncSetAttribute(k_fasst_stats, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(std::max<size_t>(smem, 48 << 10))));
  k_fasst_stats<<<grid_for(g.m, kThreads * 4), kThreads, smem, s>>>(g.m, g.ehash, w, x, xlut, R, mu,
                                                                     sorted, fill, out);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_mc_influence(const DevGraph& g, const uint32_t* w, uint64_t base, uint32_t trials,
                         uint64_t total, uint64_t batch0, uint32_t nbatch, const uint32_t* seeds,
                         uint32_t nseeds, uint32_t* live, uint32_t* vis, uint32_t* fresh,
                         uint32_t* queue, uint32_t* reached, cudaStream_t s) {
  const int blocks = std::max(1, std::min<int>(int(nbatch), num_sms()));
  if (g.m) {
    McArgs a{g.m, w, base, trials, total, batch0, nbatch, live};
    DFS_CUDA(cudaFuncSetAttribute(k_mc_live, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kMcLiveSmem)));
    k_mc_live<<<blocks, 1024, kMcLiveSmem, s>>>(a);
    DFS_CUDA(cudaGetLastError());
    ++g_launches;
  }
  McBfs b{g.n, g.off, g.adj, g.m, live, seeds, nseeds, nbatch, vis, fresh, queue, reached};
  k_mc_bfs<<<blocks, 1024, 0, s>>>(b);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

// Live (item, simulation) pairs of a direction: the density that decides how
// early sweeps / cascade levels switch to pull.
__global__ void k_popc_sum(const uint32_t* __restrict__ mask, uint64_t count,
                           unsigned long long* out) {
  unsigned long long c = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x)
    c += __popc(mask[i]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane_id() == 0 && c) atomicAdd(out, c);
}

void launch_popc_sum(const uint32_t* mask, uint64_t count, unsigned long long* out,
                     cudaStream_t s) {
  if (!count) return;
  k_popc_sum<<<grid_for(count), kThreads, 0, s>>>(mask, count, out);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_xlut_of(const uint32_t* x, uint32_t J, uint32_t* lut, cudaStream_t s) {
  k_xlut<<<(((1u << kLutBits) + 1) + kThreads - 1) / kThreads, kThreads, 0, s>>>(x, J, lut);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_xlut(const RankDev& r, cudaStream_t s) {
  k_xlut<<<(((1u << kLutBits) + 1) + kThreads - 1) / kThreads, kThreads, 0, s>>>(r.x, r.J, r.xlut);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_row_offsets(const DevGraph& g, int dir, const uint64_t* pos_off, Items& it,
                        uint32_t* row_cnt, cudaStream_t s) {
  k_row_offsets<<<grid_for(uint64_t(g.n) + 1), kThreads, 0, s>>>(g.n, dir ? g.toff : g.off,
                                                                   pos_off, it.row_off, row_cnt);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_chunk_write(uint32_t n, Items& it, const uint64_t* row_chunk64, cudaStream_t s) {
  k_chunk_write<<<grid_for(uint64_t(n) + 1), kThreads, 0, s>>>(
      n, row_chunk64, it.row_off, it.row_chunk, it.chunk_row, it.chunk_beg);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_split_chunks(Items& it, const uint64_t* chunks_dev, uint64_t chunks_cap,
                         unsigned int* cnt2, cudaStream_t s) {
  if (!chunks_cap) return;
  k_split_chunks<<<grid_for(chunks_cap), kThreads, 0, s>>>(chunks_dev, it.chunk_row, it.row_off,
                                                           it.small, it.big, cnt2);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_small_items(Items& it, const unsigned int* nsmall_dev, uint64_t chunks_cap,
                        unsigned long long* cnt, cudaStream_t s) {
  if (!chunks_cap) return;
  k_small_items<<<grid_for(chunks_cap), kThreads, 0, s>>>(nsmall_dev, it.small, it.chunk_beg,
                                                          it.small_items, cnt);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_fill(const RankDev& r, const unsigned int* gate, unsigned int want, cudaStream_t s,
                 bool use_pristine) {
  const uint64_t total = uint64_t(r.n) * 32;
  if (!r.n) return;
  k_fill<<<grid_for(total), kThreads, 0, s>>>(r.n, r.J, r.Jp, r.jkey, r.vis, r.regs, gate, want,
                                              r.ctl, r.pristine, use_pristine);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

constexpr size_t kSimSmem = size_t(kWarps) * (kPullMaxJp / 8 + 8) * 8;
constexpr size_t kCasSmem = size_t(kWarps) * (kPullMaxJp / 32) * 4;

static const void* sim_kernel(int variant) {
  switch (variant) {
    case 0: return (const void*)k_simulate<0, 0>;
    case 1: return (const void*)k_simulate<1, 0>;
    default: return (const void*)k_simulate<1, 1>;
  }
}

// variants 0-2: general loop (async, Jacobi, Jacobi + count); 3-5: parked
static const void* run_kernel(int variant) {
  switch (variant) {
    case 0: return (const void*)k_run<0, 0, 0>;
    case 1: return (const void*)k_run<1, 0, 0>;
    case 2: return (const void*)k_run<1, 1, 0>;
    case 3: return (const void*)k_run<0, 0, 1>;
    case 4: return (const void*)k_run<1, 0, 1>;
    default: return (const void*)k_run<1, 1, 1>;
  }
}

int coop_grid(int which, int variant) {
  static int g[16] = {};
  const int slot = which == 0 ? variant : which == 1 ? 3 : 4 + variant;
  if (!g[slot]) {
    int per = 0;
    const void* fn = which == 0   ? sim_kernel(variant)
                     : which == 1 ? (const void*)k_cascade
                                  : run_kernel(variant);
    const size_t smem = which == 1 ? kCasSmem : kSimSmem;
    DFS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    DFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kThreads, smem));
    if (per < 1) per = 1;
    // Tunables (blocks per SM): a smaller cascade grid makes its per-level
    // grid barrier cheaper; frontiers there are usually small.
    const char* env = getenv(which == 1 ? "DFS_CAS_BPS" : "DFS_SIM_BPS");
    int want = env ? atoi(env) : per;
    if (want >= 1 && want < per) per = want;
    g[slot] = per * num_sms();
  }
  return g[slot];
}

void launch_simulate(const RankDev& r, int jacobi, int count, int cap, const unsigned int* gate,
                     unsigned int want, cudaStream_t s) {
  static const int dbg = getenv("DFS_DBG") ? atoi(getenv("DFS_DBG")) : 0;
  static const int pf = getenv("DFS_SIM_PULL") ? atoi(getenv("DFS_SIM_PULL")) : 4;
  SimArgs a{r, cap, gate, want, dbg, pf};
  void* args[] = {&a};
  const int variant = jacobi ? (count ? 2 : 1) : 0;
  DFS_CUDA(cudaLaunchCooperativeKernel(sim_kernel(variant), dim3(coop_grid(0, variant)),
                                       dim3(kThreads), args, kSimSmem, s));
  ++g_launches;
}

void launch_score(const RankDev& r, int full, const unsigned int* gate, unsigned int want,
                  cudaStream_t s) {
  int lj = 0;
  while ((1u << lj) < r.J) ++lj;
  const int K = 53 - lj;
  const uint64_t rows = full ? r.n : r.n;  // grid sized for the worst case
  k_score<<<grid_for(rows * 32), kThreads, 0, s>>>(r.regs, r.n, r.J, r.Jp, K, full, r.dirty, r.ctl,
                                                   r.scores, gate, want);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_treesum(const double* const* parts_dev, uint32_t mu, uint32_t n, double* out,
                    cudaStream_t s) {
  k_treesum<<<grid_for(n), kThreads, 0, s>>>(parts_dev, mu, n, out);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_argmax(const double* scores, RunArrays& ra, uint32_t n, cudaStream_t s) {
  k_argmax<<<ra.nblk, kThreads, 0, s>>>(scores, n, ra);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_cascade(const RankDev& r, const unsigned int* choice, uint32_t seed, cudaStream_t s) {
  static const int dbg = getenv("DFS_DBG") ? atoi(getenv("DFS_DBG")) : 0;
  static const int pf = getenv("DFS_CAS_PULL") ? atoi(getenv("DFS_CAS_PULL")) : 8;
  CasArgs a{r, choice, seed, dbg, pf};
  void* args[] = {&a};
  DFS_CUDA(cudaLaunchCooperativeKernel((void*)k_cascade, dim3(coop_grid(1)), dim3(kThreads), args,
                                       kCasSmem, s));
  ++g_launches;
}

void launch_round_end(RunArrays& ra, RankCtl* const* ctls_dev, uint32_t mu, uint32_t k, uint32_t r,
                      double eps, cudaStream_t s) {
  k_round_end<<<1, 32, 0, s>>>(ra, ctls_dev, mu, k, r, eps);
  DFS_CUDA(cudaGetLastError());
  ++g_launches;
}

void launch_run(const RankDev* ranks_dev, uint32_t mu, uint32_t k, uint32_t R, uint32_t n,
                double eps, int cap, int jacobi, int count, int K, RunArrays& ra,
                const double* const* parts, RankCtl* const* ctls, double* reduced,
                unsigned long long* phase_ns, const PeerView* peer, int grid_share,
                int sim_pull_f, int cas_pull_f, cudaStream_t s) {
  static const int dbg = getenv("DFS_DBG") ? atoi(getenv("DFS_DBG")) : 0;
  static const int spf_env = getenv("DFS_SIM_PULL") ? atoi(getenv("DFS_SIM_PULL")) : 0;
  static const int cpf_env = getenv("DFS_CAS_PULL") ? atoi(getenv("DFS_CAS_PULL")) : 0;
  const int spf = spf_env > 0 ? spf_env : sim_pull_f;
  const int cpf = cpf_env > 0 ? cpf_env : cas_pull_f;
  RunArgs a{ranks_dev, mu, k, R, n, eps, cap, dbg, spf, cpf, K, ra, parts, ctls, reduced, phase_ns,
            peer ? 1 : 0, peer ? *peer : PeerView{}};
  void* args[] = {&a};
  const int variant = (jacobi ? (count ? 2 : 1) : 0) + (mu == 1 && !peer ? 3 : 0);
  // Ranks sharing one device (single-GPU tests of the peer protocol) split
  // its SMs so that all their persistent grids are co-resident.
  const int share = grid_share > 1 ? grid_share : 1;
  const int grid = std::max(1, coop_grid(2, variant) / share);
  DFS_CUDA(cudaLaunchCooperativeKernel(run_kernel(variant), dim3(grid), dim3(kThreads), args,
                                       kSimSmem, s));
  ++g_launches;
}

}  // namespace dfs
