"""CPU tests of the product library's host side: the C-ABI library loads and
exports every symbol of include/difuser_b200.h, and the host graph substrate
(loader, weights, hashes, generators, verification oracles) matches the
reference (golden fixtures; the live compiled reference when present).
No compute calls need a GPU here."""
import json
import os
import re

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = pytest.importorskip("paper_2410_14047_b200")
REF, PROBE = O.load_reference()


def test_library_exports_header_symbols():
    import ctypes
    header = open(os.path.join(ROOT, "include", "difuser_b200.h")).read()
    declared = set(re.findall(r"\b(dfs_[a-z0-9_]+)\s*\(", header))
    lib = ctypes.CDLL(D._capi.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(D._capi.SYMBOLS)


def test_edge_hash_and_sampling_helpers(golden):
    for u, v, lo, hi, eh in golden["hashes"]["pairs"]:
        assert D.edge_hash(u, v) == eh
    for s, r, v in golden["hashes"]["random_value_at"]:
        assert D.random_value_at(s, r) == v
    x = D.random_value_at(0, 0)
    assert D.is_sampled(x, D.edge_hash(0, 1), 1.0)
    assert not D.is_sampled(x, D.edge_hash(0, 1), 0.0)
    with pytest.raises(ValueError):
        D.is_sampled(1, 2, 1.5)


def test_graph_builder_matches_reference(golden):
    for name, gd in golden["runs"]["graphs"].items():
        g = O.CSR(gd["offsets"], gd["adj"], gd["orig_ids"])
        mine = D.graph_from_text(g.edges_text())
        assert mine.n == g.n and mine.m == g.m, name
        assert mine.orig_ids == gd["orig_ids"], name
        assert mine.offsets.tolist() == gd["offsets"], name
        assert mine.adj.tolist() == gd["adj"], name
        assert mine.ehash.tolist() == g.ehash().tolist(), name
        for spec in ("const:0.1", "wc", "const:1", "const:0"):
            assert mine.weights(spec).tolist() == g.weights(spec).tolist(), (name, spec)


def test_weight_strings(golden):
    import ctypes
    for spec, want in golden["hashes"]["weight_string"]:
        out = ctypes.c_char_p()
        D._capi.check(D.lib().dfs_weight_string(spec.encode(), ctypes.byref(out)))
        assert out.value.decode() == want


def test_text_parser_semantics():
    # proj/tests/test_graph.cpp:25-110
    g = D.graph_from_text("100 5\n5 7\n7 100\n7 5\n", True)
    assert (g.n, g.m) == (3, 4) and g.orig_ids == [5, 7, 100]
    assert g.out_degree(0) == 1 and g.out_degree(1) == 2
    assert g.in_degree.tolist() == [2, 1, 1]
    u = D.graph_from_text("0 1\n1 2\n", False)
    assert (u.n, u.m) == (3, 4)
    assert D.graph_from_text("0 0\n0 1\n", False).m == 3
    w = D.graph_from_text("0 1 0.5\n0 1 0.5\n# c\n\n2 0 0.25\n", True)
    assert w.m == 2
    for text, line in [("0 1\n7\n", 2), ("0 1\n1 2\nx y\n", 3), ("0 1 1.5\n", 1), ("0 1 0.5 9\n", 1)]:
        with pytest.raises(RuntimeError, match=f"line {line}"):
            D.graph_from_text(text)
    with pytest.raises(RuntimeError):
        D.graph_from_text("")
    with pytest.raises(RuntimeError):
        D.graph_from_text("# only comments\n")
    with pytest.raises(RuntimeError):
        D.graph_from_text("0 1 0.5\n0 1\n")
    with pytest.raises(IndexError):
        g.out_degree(3)
    assert "difuser.Graph" in repr(g)


def test_cache_roundtrip(tmp_path):
    g = D.generate("rmat", 10, 3000, 5)
    p = str(tmp_path / "g.bin")
    D.save_cache(g, p)
    h = D.load_graph(p)
    assert (h.n, h.m) == (g.n, g.m)
    assert h.orig_ids == g.orig_ids
    assert np.array_equal(h.offsets, g.offsets) and np.array_equal(h.adj, g.adj)
    assert np.array_equal(h.ehash, g.ehash)
    t = tmp_path / "g.txt"
    t.write_text("0 1\n1 2\n2 3\n")
    assert (D.load_graph(str(t)).n, D.load_graph(str(t)).m) == (4, 3)


@pytest.mark.skipif(REF is None, reason="compiled reference (oracle/_ref) not present")
def test_cache_interop_with_reference(tmp_path):
    g = D.generate("rmat", 11, 8000, 9)
    p = str(tmp_path / "g.bin")
    D.save_cache(g, p)
    rg = REF.load_graph(p)
    assert (rg.n, rg.m) == (g.n, g.m) and list(rg.orig_ids) == g.orig_ids
    p2 = str(tmp_path / "r.bin")
    REF.save_cache(rg, p2)
    assert open(p, "rb").read() == open(p2, "rb").read()


@pytest.mark.skipif(REF is None, reason="compiled reference (oracle/_ref) not present")
def test_random_weights_match_reference():
    g = D.generate("er", 300, 2000, 3)
    for spec in ("normal:0.1,0.05", "uniform:0,0.9", "uniform:0.2,0.2", "normal:0.5,2"):
        for seed in (0, 7):
            want = PROBE.weights(g.offsets.tolist(), g.adj.tolist(), spec, seed)
            assert g.weights(spec, seed).tolist() == list(want), spec


def test_generator_is_deterministic_and_exact():
    a = D.generate("rmat", 12, 20000, 7)
    b = D.generate("rmat", 12, 20000, 7)
    assert a.m == 20000 and np.array_equal(a.adj, b.adj) and a.orig_ids == b.orig_ids
    off = a.offsets
    for u in range(0, a.n, 97):  # sorted rows, no duplicates, no self-loops
        row = a.adj[off[u]:off[u + 1]]
        assert np.all(np.diff(row.astype(np.int64)) > 0)
        assert not np.any(row == u)
    e = D.generate("er", 10000, 80000, 7)
    assert (e.n, e.m) == (10000, 80000)


def test_influence_and_greedy_exact_chain():
    chain = D.graph_from_text("0 1\n1 2\n2 3\n")
    mean, se = D.influence(chain, [0], trials=200, weights="const:1")
    assert mean == pytest.approx(4.0) and se == pytest.approx(0.0)
    assert D.greedy_exact(chain, k=1, trials=64, weights="const:1") == [0]
    with pytest.raises(ValueError):
        D.influence(chain, [9], trials=10)
    with pytest.raises(ValueError):
        D.greedy_exact(chain, k=0)


@pytest.mark.skipif(REF is None, reason="compiled reference (oracle/_ref) not present")
def test_oracles_match_reference():
    g = D.generate("er", 120, 700, 5)
    rg = REF.graph_from_text(O.CSR(g.offsets, g.adj, np.array(g.orig_ids)).edges_text())
    for seeds in ([0], [3, 50, 77], []):
        assert D.influence(g, seeds, trials=300, seed=4, runs=2, weights="const:0.2") == \
            REF.influence(rg, seeds, trials=300, seed=4, runs=2, weights="const:0.2")
    assert D.greedy_exact(g, 3, trials=40, seed=2, weights="const:0.15") == \
        REF.greedy_exact(rg, 3, trials=40, seed=2, weights="const:0.15")


def test_no_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(RuntimeError, match="CUDA"):
        D.Context(0)
    with pytest.raises(RuntimeError):
        D.run(D.graph_from_text("0 1\n"), k=1, r=64)


@pytest.mark.parametrize("kind,a,m", [("rmat", 12, 40000), ("rmat", 16, 400000), ("er", 5000, 20000)])
def test_oracle_synthesizer_matches_product_generator(tmp_path, kind, a, m):
    """bench.py's reference arm builds its graph with the oracle-side
    synthesizer (oracle/synth.c) so that it never loads the product library:
    the cache must be byte-identical to save_cache(generate(...))."""
    po, pp = str(tmp_path / "o.bin"), str(tmp_path / "p.bin")
    n = O.generate_cache(kind, a, m, 7, po)
    g = D.generate(kind, a, m, 7)
    D.save_cache(g, pp)
    assert n == g.n
    assert open(po, "rb").read() == open(pp, "rb").read()


def test_bench_reference_reports_recorded():
    """The reference reports bench.py checks its own report against exist for
    the headline workload at every GPU count of the scaling run."""
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "bench_reports.json")))
    assert set(gold["c2"]["reports"]) >= {"1", "2", "4", "8"}
    for d, rep in gold["c2"]["reports"].items():
        r = json.loads(rep)
        assert r["config"]["devices"] == int(d) and len(r["seeds"]) == 50
