// refprobe — TEST INFRASTRUCTURE ONLY (never shipped, never on the product path).
//
// A pybind11 harness compiled together with the *unmodified* reference sources
// (/root/reference/proj/src/*.cpp, see oracle/Makefile) so that the reference's
// own engine-level entry points can be driven stage by stage and their internal
// state dumped as golden vectors: device graph + baked masks
// (proj/src/fasst.cpp:50-88), registers after fill (proj/src/sketch.cpp:55-66),
// after simulate_to_convergence (proj/src/engine.cpp:88-96), row scores
// (proj/src/sketch.cpp:119-131) and registers/visited after commit_seed+cascade
// (proj/src/engine.cpp:106-144).  Nothing here re-implements the algorithm; it
// only calls the reference.
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstring>
#include <string>
#include <vector>

#include "difuser/engine.hpp"
#include "difuser/fasst.hpp"
#include "difuser/graph.hpp"
#include "difuser/hash.hpp"
#include "difuser/report.hpp"
#include "difuser/runtime.hpp"
#include "difuser/sampling.hpp"
#include "difuser/sketch.hpp"

namespace py = pybind11;
using namespace difuser;

namespace {

WeightedGraph make_graph(const std::vector<uint64_t>& offsets,
                         const std::vector<uint32_t>& adj,
                         const std::vector<uint32_t>& weights) {
  WeightedGraph g;
  g.n = static_cast<vertex_t>(offsets.size() - 1);
  g.m = adj.size();
  g.offsets = offsets;
  g.adj = adj;
  g.weights = weights;
  g.ehash.resize(g.m);
  g.in_degree.assign(g.n, 0);
  g.orig_id.resize(g.n);
  for (vertex_t u = 0; u < g.n; ++u) {
    g.orig_id[u] = u;
    for (uint64_t e = g.offsets[u]; e < g.offsets[u + 1]; ++e) {
      g.ehash[e] = edge_hash(u, g.adj[e]);
      g.in_degree[g.adj[e]]++;
    }
  }
  return g;
}

py::bytes regs_bytes(const SketchMatrix& m) {
  return py::bytes(reinterpret_cast<const char*>(m.row(0)),
                   size_t(m.n()) * m.j_local());
}

}  // namespace

PYBIND11_MODULE(_refprobe, mod) {
  mod.doc() = "stage-level dumps of the reference engine (test oracle only)";

  mod.def("plan", [](uint32_t r, uint32_t mu, const std::string& mode,
                     uint64_t seed) {
    PartitionPlan p = make_plan(
        gen_random_vector(r, derive_seed(seed, kSeedTagSamples)), mu,
        parse_partition_mode(mode));
    py::dict d;
    d["x"] = p.x.values;
    d["order"] = p.order;
    d["chunk"] = p.chunk;
    d["degraded"] = p.degraded;
    d["reg_key"] = derive_seed(seed, kSeedTagRegisters);
    return d;
  });

  // Weighted graph as the reference sees it after apply_weights.
  mod.def("weights", [](const std::vector<uint64_t>& offsets,
                        const std::vector<uint32_t>& adj,
                        const std::string& spec, uint64_t seed) {
    WeightedGraph g = make_graph(offsets, adj,
                                 std::vector<uint32_t>(adj.size(), 0));
    RunConfig cfg;
    cfg.weights = WeightSetting::parse(spec);
    cfg.seed = seed;
    apply_weights(g, cfg);
    return g.weights;
  });

  // Full stage trace of one device tau: device graph, fill, simulate, scores,
  // then commit+cascade of each seed in `seeds` (registers after each).
  mod.def(
      "device_trace",
      [](const std::vector<uint64_t>& offsets, const std::vector<uint32_t>& adj,
         const std::vector<uint32_t>& weights, uint32_t r, uint32_t mu,
         const std::string& mode, uint64_t seed, uint32_t tau,
         const std::vector<uint32_t>& seeds) {
        WeightedGraph g = make_graph(offsets, adj, weights);
        PartitionPlan plan = make_plan(
            gen_random_vector(r, derive_seed(seed, kSeedTagSamples)), mu,
            parse_partition_mode(mode));
        DeviceGraph dg = build_device_graph(g, plan, tau);
        SketchMatrix m(g.n, plan.chunk, tau * plan.chunk,
                       derive_seed(seed, kSeedTagRegisters));
        py::dict d;
        d["dg_offsets"] = dg.offsets;
        d["dg_adj"] = dg.adj;
        d["dg_mask"] = dg.mask;
        d["mask_words"] = dg.mask_words;
        fill_sketches(m);
        d["regs_fill"] = regs_bytes(m);
        SimulateBuffers buf;
        d["sweeps"] = simulate_to_convergence(dg, m, buf);
        d["regs_sim"] = regs_bytes(m);
        d["scores"] = sketchwise_score(m);
        CascadeState cs;
        cs.init(g.n, m.words());
        py::list after;
        py::list counts;
        for (uint32_t s : seeds) {
          commit_seed(m, cs, s);
          cascade(dg, m, cs);
          after.append(regs_bytes(m));
          counts.append(count_visited(m));
        }
        d["regs_cascade"] = after;
        d["visited"] = counts;
        return d;
      },
      py::arg("offsets"), py::arg("adj"), py::arg("weights"), py::arg("r"),
      py::arg("mu"), py::arg("mode"), py::arg("seed"), py::arg("tau"),
      py::arg("seeds") = std::vector<uint32_t>{});

  // FASST analytics (proj/src/fasst.cpp:101-168): duplication histogram,
  // per-device edge loads and the 32-lane batch fill rate, on the weighted
  // graph as apply_weights leaves it.
  mod.def(
      "fasst_stats",
      [](const std::vector<uint64_t>& offsets, const std::vector<uint32_t>& adj,
         const std::vector<uint32_t>& weights, uint32_t r, uint32_t mu,
         const std::string& mode, uint64_t seed) {
        WeightedGraph g = make_graph(offsets, adj, weights);
        RandomVector x = gen_random_vector(r, derive_seed(seed, kSeedTagSamples));
        PartitionPlan plan = make_plan(x, mu, parse_partition_mode(mode));
        DuplicationHistogram h = duplication_stats(g, plan);
        py::dict d;
        d["dup_count"] = h.count;
        d["dup_fraction"] = h.fraction;
        d["share_within_1"] = h.sampled_share_within(1);
        d["share_within_2"] = h.sampled_share_within(2);
        d["loads"] = device_edge_loads(g, plan);
        if (r % 32 == 0) {
          FillRateReport fr = fill_rate(g, x, parse_partition_mode(mode));
          d["fill_rate"] = fr.fill_rate;
          d["fill_batches"] = fr.batches;
        }
        return d;
      },
      py::arg("offsets"), py::arg("adj"), py::arg("weights"), py::arg("r"), py::arg("mu"),
      py::arg("mode"), py::arg("seed"));

  mod.def("fmix64", [](uint64_t k) { return fmix64(k); });
  mod.def("splitmix64_at", [](uint64_t s, uint64_t i) { return splitmix64_at(s, i); });
  mod.def("murmur3_pair", [](uint64_t a, uint64_t b) {
    Hash128 h = murmur3_pair(a, b);
    return py::make_tuple(h.lo, h.hi);
  });
  mod.def("register_hash", [](uint64_t k, uint64_t v) { return register_hash(k, v); });
  mod.def("to_fixed_point", [](double w) { return to_fixed_point(w); });
  mod.def("weight_string", [](const std::string& s) {
    return WeightSetting::parse(s).to_string();
  });

  mod.def("row_score", [](const std::vector<int8_t>& row) {
    return row_score(std::span<const int8_t>(row.data(), row.size()));
  });

  // The reference hot-path entry on raw CSR arrays (weights applied inside,
  // exactly like run_json).  Returns the report JSON (no timings unless asked).
  mod.def(
      "run_arrays",
      [](const std::vector<uint64_t>& offsets, const std::vector<uint32_t>& adj,
         const std::vector<uint64_t>& orig_ids, uint32_t k, uint32_t r,
         uint32_t devices, const std::string& mode, const std::string& weights,
         double rebuild_eps, uint64_t seed, bool timings) {
        WeightedGraph g = make_graph(offsets, adj,
                                     std::vector<uint32_t>(adj.size(), 0));
        if (!orig_ids.empty()) g.orig_id = orig_ids;
        RunConfig cfg;
        cfg.k = k;
        cfg.r = r;
        cfg.mu = devices;
        cfg.mode = parse_partition_mode(mode);
        cfg.weights = WeightSetting::parse(weights);
        cfg.rebuild_eps = rebuild_eps;
        cfg.seed = seed;
        apply_weights(g, cfg);
        return report_to_json(run(g, cfg), timings);
      },
      py::arg("offsets"), py::arg("adj"), py::arg("orig_ids"), py::arg("k"),
      py::arg("r"), py::arg("devices"), py::arg("mode"), py::arg("weights"),
      py::arg("rebuild_eps"), py::arg("seed"), py::arg("timings") = false);
}
