// graph.h — host graph substrate: the input format the kernels consume.
// Behaviour mirrors proj/include/difuser/graph.hpp (WeightedGraph :44-58,
// WeightSetting :65-80) so that graphs, weights and reports are bit-identical
// to the reference's for the same input.
#pragma once
#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

namespace dfs {

// proj/include/difuser/graph.hpp:44-58 (CSR by source, dense ids).
struct HostGraph {
  uint32_t n = 0;
  uint64_t m = 0;
  std::vector<uint64_t> offsets;    // n+1
  std::vector<uint32_t> adj;        // m, sorted per row
  std::vector<uint32_t> weights;    // m, fixed point (as loaded)
  // Derived on first host use (ensure_graph_fields): the GPU path never
  // reads them (k_ehash / k_indeg recompute both at upload), so loaders and
  // generators do not spend host time on them.
  mutable std::vector<uint32_t> ehash;      // m, edge_hash(u, v) on dense ids
  mutable std::vector<uint32_t> in_degree;  // n
  std::vector<uint64_t> orig_id;    // n, ascending
};

uint32_t to_fixed_point(double w);  // graph.cpp:30-35 semantics

enum class WeightKind { Constant, WeightedCascade, Normal, Uniform };
struct WeightSetting {  // graph.hpp:65-80
  WeightKind kind = WeightKind::Constant;
  double a = 0.1, b = 0.0;
  static WeightSetting parse(std::string_view spec);
  std::string to_string() const;
};

HostGraph graph_from_text(std::string_view text, bool directed);
HostGraph load_graph(const std::string& path, bool directed);
void save_graph_cache(const HostGraph& g, const std::string& path);
// Raw CSR (already dense, sorted, duplicate-free); ehash/in_degree derived.
HostGraph graph_from_csr(uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* adj,
                         const uint64_t* orig_ids);
// Deterministic synthetic generators (bench/test inputs; not in the reference
// library): exactly m unique directed edges without
// self-loops, then the reference's dense relabelling.
HostGraph generate_rmat(uint32_t scale, uint64_t m, uint64_t seed);
HostGraph generate_er(uint32_t n, uint64_t m, uint64_t seed);

// apply_weights on the host (runtime.cpp:15-17, graph.cpp:247-274).
void assign_weights(const HostGraph& g, const WeightSetting& s, uint64_t seed,
                    std::vector<uint32_t>& w);

// Monte-Carlo oracle semantics of proj/src/oracle.cpp:30-79 (host, not on the
// hot path): mean and standard error of reached vertices.
void influence_stats(const HostGraph& g, const std::vector<uint32_t>& w,
                     const std::vector<uint32_t>& seeds, uint32_t trials, uint64_t seed,
                     uint32_t runs, double* mean, double* std_error);

// Exact greedy under the same trial coupling (proj/src/oracle.cpp:152-250);
// reachability per trial by pruned BFS instead of SCC condensation — the gains
// are the same integers.  Small graphs only (verification, not the hot path).
std::vector<uint32_t> greedy_exact(const HostGraph& g, const std::vector<uint32_t>& w, uint32_t k,
                                   uint32_t trials, uint64_t seed);

void ensure_graph_fields(const HostGraph& g);  // ehash + in_degree (parallel), once

}  // namespace dfs
