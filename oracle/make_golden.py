"""Generate tests/golden/* from the UNMODIFIED reference (TEST INFRASTRUCTURE).

Run in the build container (needs /root/reference and ``make -C oracle ref``):

    python oracle/make_golden.py

Every value written here is produced by the compiled reference (oracle/_ref:
its own pybind module ``_difuser`` and the stage harness ``_refprobe``), never
by the oracle restatement or the product.  The fixtures are small; the GPU box
reads them (it has no /root/reference).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
REF_CSV = "/root/reference/proj/tests/data/hash_vectors.csv"


def graph_dict(g: O.CSR):
    return {"offsets": g.offsets.tolist(), "adj": g.adj.tolist(), "orig_ids": g.orig_ids.tolist()}


def small_graphs():
    """Named small graphs (edge lists are test inputs; CSR via build_csr, checked
    against the reference's own graph_from_text n/m/orig_ids below)."""
    gs = {}
    for name, (n, m, s) in {"er40": (40, 200, 3), "er120": (120, 700, 5), "er200": (200, 1600, 7),
                            "er300": (300, 1500, 4)}.items():
        gs[name] = O.build_csr(*O.er_edges(n, m, s))
    path = np.arange(11, dtype=np.uint64)
    gs["path12"] = O.build_csr(path, path + 1)
    gs["star30"] = O.build_csr(np.full(29, 1000, np.uint64), np.arange(1001, 1030, dtype=np.uint64))
    cyc = np.arange(16, dtype=np.uint64)
    gs["cycle16"] = O.build_csr(cyc, (cyc + 1) % 16)
    two = [(0, i) for i in range(1, 41)] + [(41, i) for i in range(42, 62)]
    gs["twostars"] = O.build_csr([a for a, _ in two], [b for _, b in two])
    # self-loops are kept by the reference (graph.cpp:60-62 comment): include one
    gs["selfloop"] = O.build_csr([0, 0, 1, 2, 2], [0, 1, 2, 0, 3])
    return gs


def main():
    ref, probe = O.load_reference()
    if ref is None:
        sys.exit("reference build missing: run `make -C oracle ref` first")
    os.makedirs(OUT, exist_ok=True)

    # ---- hashes ------------------------------------------------------------
    pairs = []
    with open(REF_CSV) as f:
        next(f)
        for line in f:
            if line.strip():
                u, v = line.split(",")[:2]
                pairs.append((int(u), int(v)))
    rng = np.random.default_rng(2024)
    pairs += [(int(a), int(b)) for a, b in rng.integers(0, 2**40, size=(200, 2))]
    pairs += [(int(a), int(b)) for a, b in rng.integers(0, 2**20, size=(200, 2))]
    hashes = {
        "pairs": [[u, v, probe.murmur3_pair(u, v)[0], probe.murmur3_pair(u, v)[1], ref.edge_hash(u, v)]
                  for u, v in pairs],
        "fmix64": [[k, probe.fmix64(k)] for k in [0, 1, 2, 0xdeadbeef, 0x9e3779b97f4a7c15, 2**64 - 1]
                   + [int(x) for x in rng.integers(0, 2**63, 50)]],
        "splitmix64_at": [[s, i, probe.splitmix64_at(s, i)] for s in [0, 42, 0x123456789abcdef, 7]
                          for i in [0, 1, 2, 3, 1000, 2**33]],
        "register_hash": [[k, v, probe.register_hash(k, v)]
                          for k in [probe.splitmix64_at(42, 3), probe.splitmix64_at(7, 0), 0, 2**64 - 1]
                          for v in [0, 1, 17, 12345, 2**31, 2**32 + 5]],
        "random_value_at": [[s, r, ref.random_value_at(s, r)] for s in [0, 7, 17, 2**63 + 5]
                            for r in [0, 1, 2, 63, 1023, 4095]],
        "to_fixed_point": [[w, probe.to_fixed_point(w)] for w in
                           [0.0, 1.0, 0.5, 0.1, 0.01, 0.005, 0.3, 1 / 3, 1 / 7, 1e-9, 0.99999999]],
        "weight_string": [[s, probe.weight_string(s)] for s in
                          ["const:0.1", "const:1", "const:0.01", "const:0.005", "wc", "const:0.25",
                           "normal:0.1,0.05", "uniform:0,0.9"]],
    }
    with open(os.path.join(OUT, "hashes.json"), "w") as f:
        json.dump(hashes, f)

    # ---- graphs checked against the reference's own build_graph -------------
    gs = small_graphs()
    for name, g in gs.items():
        rg = ref.graph_from_text(g.edges_text())
        assert (rg.n, rg.m, list(rg.orig_ids)) == (g.n, g.m, g.orig_ids.tolist()), name
        assert [rg.out_degree(u) for u in range(g.n)] == np.diff(g.offsets).tolist(), name

    # ---- end-to-end reports (run_json, timings=False) ------------------------
    cases = []
    grid = [
        ("path12", dict(k=3, r=32, devices=1, weights="const:1", seed=0)),
        ("star30", dict(k=1, r=64, devices=1, weights="const:1", seed=0)),
        ("star30", dict(k=1, r=64, devices=2, weights="const:1", seed=0)),
        ("twostars", dict(k=2, r=128, devices=1, weights="const:0.9", seed=5)),
        ("twostars", dict(k=2, r=128, devices=4, weights="const:0.9", seed=5)),
        ("cycle16", dict(k=4, r=64, devices=1, weights="const:0.5", seed=1)),
        ("selfloop", dict(k=4, r=64, devices=2, weights="const:0.7", seed=2)),
        ("er40", dict(k=2, r=64, devices=4, weights="const:0.5", seed=0)),
        ("er40", dict(k=2, r=64, devices=4, mode="naive", weights="const:0.5", seed=0)),
        ("er120", dict(k=8, r=128, devices=2, weights="const:0.2", seed=3)),
        ("er120", dict(k=8, r=256, devices=1, weights="const:0.1", seed=11)),
        ("er120", dict(k=8, r=256, devices=8, weights="const:0.1", seed=11)),
        ("er200", dict(k=5, r=256, devices=1, weights="const:0.1", seed=4)),
        ("er200", dict(k=10, r=96, devices=3, weights="const:0.3", seed=9)),
        ("er200", dict(k=6, r=100, devices=1, weights="wc", seed=2)),
        ("er200", dict(k=6, r=64, devices=1, weights="const:0.15", seed=2, rebuild_eps=0.0)),
        ("er200", dict(k=6, r=64, devices=1, weights="const:0.15", seed=2, rebuild_eps=1.0)),
        ("er300", dict(k=12, r=1024, devices=8, weights="const:0.1", seed=33)),
        ("er300", dict(k=12, r=512, devices=2, weights="wc", seed=5)),
        ("er300", dict(k=12, r=64, devices=8, weights="const:0.2", seed=5)),
        ("er300", dict(k=300, r=32, devices=1, weights="const:0.5", seed=1)),
    ]
    for name, cfg in grid:
        g = gs[name]
        rg = ref.graph_from_text(g.edges_text())
        text = ref.run_json(rg, timings=False, **cfg)
        cases.append({"graph": name, "config": cfg, "json": text})
    with open(os.path.join(OUT, "runs.json"), "w") as f:
        json.dump({"graphs": {k: graph_dict(v) for k, v in gs.items()}, "cases": cases}, f)

    # ---- stage traces (device graph, registers, scores, cascade) -------------
    traces = []
    for name, r, mu, mode, wspec, seed, seeds in [
        ("er40", 64, 1, "fasst", "const:0.5", 0, [3, 17]),
        ("er120", 128, 2, "fasst", "const:0.2", 3, [5, 60, 7]),
        ("er120", 96, 3, "naive", "const:0.3", 1, [1]),
        ("er200", 100, 1, "fasst", "wc", 2, [10, 20]),
        ("path12", 64, 1, "fasst", "const:1", 5, [0]),
        ("er300", 256, 8, "fasst", "const:0.1", 33, [100, 7]),
    ]:
        g = gs[name]
        w = probe.weights(g.offsets.tolist(), g.adj.tolist(), wspec, seed)
        for tau in range(mu):
            d = probe.device_trace(g.offsets.tolist(), g.adj.tolist(), w, r, mu, mode, seed, tau, seeds)
            traces.append({
                "graph": name, "r": r, "mu": mu, "mode": mode, "weights": wspec, "seed": seed,
                "tau": tau, "seeds": seeds, "w": list(w),
                "dg_offsets": list(d["dg_offsets"]), "dg_adj": list(d["dg_adj"]),
                "dg_mask": [int(x) for x in d["dg_mask"]], "mask_words": d["mask_words"],
                "regs_fill": d["regs_fill"].hex(), "regs_sim": d["regs_sim"].hex(),
                "sweeps": d["sweeps"], "scores": [float(s).hex() for s in d["scores"]],
                "regs_cascade": [b.hex() for b in d["regs_cascade"]], "visited": list(d["visited"]),
            })
    with open(os.path.join(OUT, "traces.json"), "w") as f:
        json.dump(traces, f)

    # ---- FASST analytics (fasst.cpp:101-168) ----------------------------------
    fs_graphs = {"er200": gs["er200"], "er300": gs["er300"],
                 "er3000": O.build_csr(*O.er_edges(3000, 24000, 21))}
    fstats = []
    for name, r, mu, mode, wspec, seed in [
        ("er200", 256, 4, "fasst", "const:0.1", 2), ("er200", 256, 4, "naive", "const:0.1", 2),
        ("er300", 1024, 8, "fasst", "const:0.01", 7), ("er300", 1024, 8, "naive", "const:0.01", 7),
        ("er300", 96, 3, "fasst", "wc", 5), ("er3000", 512, 8, "fasst", "const:0.05", 3),
        ("er3000", 512, 8, "naive", "const:0.05", 3), ("er3000", 256, 2, "fasst", "wc", 1),
        ("er3000", 4096, 8, "fasst", "const:0.005", 9), ("er3000", 128, 1, "naive", "const:1", 4),
    ]:
        g = fs_graphs[name]
        w = probe.weights(g.offsets.tolist(), g.adj.tolist(), wspec, seed)
        d = probe.fasst_stats(g.offsets.tolist(), g.adj.tolist(), w, r, mu, mode, seed)
        fstats.append({"graph": name, "r": r, "mu": mu, "mode": mode, "weights": wspec,
                       "seed": seed, **{k: (list(v) if isinstance(v, (list, tuple)) else v)
                                        for k, v in d.items()}})
    with open(os.path.join(OUT, "fasst_stats.json"), "w") as f:
        json.dump({"graphs": {k: graph_dict(v) for k, v in fs_graphs.items()}, "cases": fstats}, f)
    # ---- Monte-Carlo influence (oracle.cpp:30-79, the binding's influence()) ---
    infl = []
    for name, seeds, trials, seed, runs, wspec in [
        ("er200", [0, 5, 17], 300, 4, 1, "const:0.1"), ("er300", [1, 2], 257, 7, 2, "const:0.2"),
        ("er3000", [10, 200, 3000 - 1], 100, 3, 1, "const:0.05"), ("er3000", [5], 64, 1, 3, "wc"),
        ("er120", [], 40, 0, 1, "const:0.5"), ("cycle16", [3], 33, 9, 1, "const:0.5"),
        ("er3000", [7, 8], 96, 11, 1, "uniform:0,0.2"),
    ]:
        g = fs_graphs.get(name) or gs[name]
        rg = ref.graph_from_text(g.edges_text())
        mean, se = ref.influence(rg, seeds, trials=trials, seed=seed, runs=runs, weights=wspec)
        infl.append({"graph": name, "seeds": seeds, "trials": trials, "seed": seed, "runs": runs,
                     "weights": wspec, "mean": float(mean).hex(), "std_error": float(se).hex()})
    with open(os.path.join(OUT, "influence.json"), "w") as f:
        json.dump({"graphs": {k: graph_dict(v) for k, v in list(fs_graphs.items()) +
                              [(k, gs[k]) for k in ("er120", "cycle16")]}, "cases": infl}, f)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
