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

#include <algorithm>
#include <bit>
#include <cstring>
#include <stdexcept>
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

  // Reference-schedule work units of a whole devices=1 run,
  // the numerator of bench.py's roofline: the reference's own stages
  // (build_device_graph fasst.cpp:50-88, fill_sketches sketch.cpp:55-66,
  // simulate_iteration engine.cpp:57-86, commit_seed/cascade engine.cpp:106-144)
  // driven with the seeds and rebuild rounds of the reference's report; the
  // counters are read off the reference's own state between its calls:
  //   per sweep  E = edges whose source changed in the previous sweep
  //              (changed_prev, engine.cpp:70), B = their non-zero 32-sim
  //              mask halves, L = their live bits, T = distinct (row, batch)
  //              pairs among them;  S = sweeps (simulate_to_convergence's count)
  //   cascades   F = frontier rows summed over levels, Ec = their device-graph
  //              out-edges, C = cascades started (frontier non-empty after
  //              commit_seed).  The level loop below mirrors engine.cpp:120-144
  //              on copies and is checked against the reference's cascade().
  mod.def(
      "run_units",
      [](const std::vector<uint64_t>& offsets, const std::vector<uint32_t>& adj,
         const std::vector<uint32_t>& weights, uint32_t r, uint64_t seed,
         const std::vector<uint32_t>& seeds, const std::vector<uint32_t>& rebuild_rounds) {
        WeightedGraph g = make_graph(offsets, adj, weights);
        PartitionPlan plan = make_plan(
            gen_random_vector(r, derive_seed(seed, kSeedTagSamples)), 1, PartitionMode::Fasst);
        DeviceGraph dg = build_device_graph(g, plan, 0);
        SketchMatrix m(g.n, plan.chunk, 0, derive_seed(seed, kSeedTagRegisters));
        const uint32_t words = dg.mask_words, halves = (plan.chunk + 31) / 32;
        uint64_t E = 0, B = 0, L = 0, T = 0, S = 0, conv = 0, F = 0, Ec = 0, Cn = 0;
        std::vector<uint8_t> touched(size_t(g.n) * halves);
        auto simulate = [&]() {
          SimulateBuffers buf;
          buf.reset(m);
          for (int it = 1; it <= 256; ++it) {
            std::fill(touched.begin(), touched.end(), 0);
            for (vertex_t u = 0; u < dg.n; ++u)
              for (uint64_t e = dg.offsets[u]; e < dg.offsets[u + 1]; ++e) {
                if (!buf.changed_prev[dg.adj[e]]) continue;
                ++E;
                const uint64_t* em = dg.edge_mask(e);
                for (uint32_t h = 0; h < halves; ++h) {
                  const uint32_t bits = uint32_t(em[h / 2] >> (32 * (h & 1)));
                  if (!bits) continue;
                  ++B;
                  L += std::popcount(bits);
                  uint8_t& t = touched[size_t(u) * halves + h];
                  if (!t) {
                    t = 1;
                    ++T;
                  }
                }
              }
            ++S;
            if (!simulate_iteration(dg, m, buf)) break;
          }
          ++conv;
        };
        fill_sketches(m);
        simulate();
        CascadeState cs;
        cs.init(g.n, m.words());
        for (uint32_t step = 0; step < seeds.size(); ++step) {
          commit_seed(m, cs, seeds[step]);
          // counting replica of the level loop on copies of the state
          SketchMatrix m2 = m;
          CascadeState c2 = cs;
          if (!c2.q.empty()) ++Cn;
          while (!c2.q.empty()) {
            for (vertex_t u : c2.q.items) {
              ++F;
              Ec += dg.offsets[u + 1] - dg.offsets[u];
              const uint64_t* fu = c2.fresh_row(c2.fresh_cur, u);
              for (uint64_t e = dg.offsets[u]; e < dg.offsets[u + 1]; ++e) {
                const vertex_t v = dg.adj[e];
                const uint64_t* em = dg.edge_mask(e);
                for (uint32_t w = 0; w < c2.words; ++w) {
                  const uint64_t cand = fu[w] & em[w] & ~m2.vis_row(v)[w];
                  if (!cand) continue;
                  m2.mark_visited_word(v, w, cand);
                  c2.fresh_row(c2.fresh_next, v)[w] |= cand;
                  c2.q_next.push(v);
                }
              }
            }
            for (vertex_t u : c2.q.items) std::memset(c2.fresh_row(c2.fresh_cur, u), 0, c2.words * 8);
            c2.q.clear();
            std::swap(c2.q.items, c2.q_next.items);
            std::swap(c2.q.member, c2.q_next.member);
            std::swap(c2.fresh_cur, c2.fresh_next);
          }
          cascade(dg, m, cs);  // the reference's own cascade advances the real state
          if (count_visited(m) != count_visited(m2) ||
              std::memcmp(m.row(0), m2.row(0), size_t(g.n) * m.j_local()) != 0)
            throw std::runtime_error("run_units: counting replica diverged from cascade()");
          if (std::find(rebuild_rounds.begin(), rebuild_rounds.end(), step) != rebuild_rounds.end()) {
            fill_sketches(m);
            simulate();
          }
        }
        (void)words;
        py::dict d;
        d["E"] = E; d["B"] = B; d["T"] = T; d["L"] = L; d["S"] = S; d["convergences"] = conv;
        d["cascade_rows"] = F; d["cascade_edges"] = Ec; d["cascades"] = Cn;
        return d;
      },
      py::arg("offsets"), py::arg("adj"), py::arg("weights"), py::arg("r"), py::arg("seed"),
      py::arg("seeds"), py::arg("rebuild_rounds"));

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
