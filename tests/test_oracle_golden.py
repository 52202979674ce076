"""Pin the oracle restatement (oracle/difuser_oracle.c) to the reference:
golden vectors of the reference's own tests (tests/data/hash_vectors.csv and
the test_hash.cpp KATs) and fixtures produced by the compiled reference
(tests/golden, oracle/make_golden.py).  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle as O


def _csr(gd):
    return O.CSR(gd["offsets"], gd["adj"], gd["orig_ids"])


def test_hash_kats():
    # proj/tests/test_hash.cpp:14-32, 60-90
    assert O.fmix64(0) == 0
    assert O.fmix64(1) == 0xb456bcfc34c2cb2c
    assert O.fmix64(0xdeadbeef) == 0xd24bd59f862a1dac
    assert O.splitmix64_at(0, 0) == 0xe220a8397b1dcdaf
    assert O.splitmix64_at(0x123456789abcdef, 2) == 0x2f90b72e996dccbe
    assert O.edge_hash(3, 5) == 266300377
    assert O.edge_hash(5, 3) == 389432881
    assert O.murmur3_pair(0, 0)[0] == 0x4bbd1bf27da918d6
    key = O.splitmix64_at(42, 3)
    assert key == 0x581ce1ff0e4ae394
    assert O.register_hash(key, 17) == 0xff9d70add4d5b390


def test_hash_golden(golden):
    h = golden["hashes"]
    for u, v, lo, hi, eh in h["pairs"]:
        assert O.murmur3_pair(u, v) == (lo, hi)
        assert O.edge_hash(u, v) == eh
    us = np.array([p[0] for p in h["pairs"] if p[0] < 2**63 and p[1] < 2**63], np.uint64)
    vs = np.array([p[1] for p in h["pairs"] if p[0] < 2**63 and p[1] < 2**63], np.uint64)
    want = [p[4] for p in h["pairs"] if p[0] < 2**63 and p[1] < 2**63]
    assert O.edge_hash_np(us, vs).tolist() == want
    for k, v in h["fmix64"]:
        assert O.fmix64(k) == v
    for s, i, v in h["splitmix64_at"]:
        assert O.splitmix64_at(s, i) == v
    for k, x, v in h["register_hash"]:
        assert O.register_hash(k, x) == v
    for s, r, v in h["random_value_at"]:
        assert O.random_value_at(s, r) == v
    for w, v in h["to_fixed_point"]:
        assert O.to_fixed_point(w) == v


def test_sampling_exact_rate():
    # proj/tests/test_sampling.cpp:30-41: #{x < 2^16 : (x ^ h) < W} == W
    x = np.arange(1 << 16, dtype=np.uint32)
    for h in (0, 1, 0x5A5A, 0xFFFF):
        for w in (0, 1, 100, 32768, 65536):
            assert int(((x ^ np.uint32(h)) < np.uint32(w)).sum()) == w


def test_traces_match_reference(golden):
    graphs = golden["runs"]["graphs"]
    for tr in golden["traces"]:
        g = _csr(graphs[tr["graph"]])
        w = np.array(tr["w"], np.uint32)
        assert g.weights(tr["weights"]).tolist() == tr["w"]
        x, order, _ = O.make_plan(tr["r"], tr["mu"], tr["mode"], tr["seed"])
        J = tr["r"] // tr["mu"]
        tau = tr["tau"]
        off, adj, mask = O.device_graph(g, w, x[tau * J:(tau + 1) * J])
        assert off.tolist() == tr["dg_offsets"]
        assert adj.tolist() == tr["dg_adj"]
        assert mask.tolist() == tr["dg_mask"]
        regs = O.fill(g.n, J, tau * J, O.splitmix64_at(tr["seed"], 2))
        assert regs.tobytes().hex() == tr["regs_fill"]
        assert O.simulate(g.n, off, adj, mask, J, regs) == tr["sweeps"]
        assert regs.tobytes().hex() == tr["regs_sim"]
        assert [float(O.row_score(regs[u * J:(u + 1) * J])).hex() for u in range(g.n)] == \
            tr["scores"]
        vis = np.zeros(g.n * ((J + 63) // 64) + 1, np.uint64)
        total = 0
        for s, want_regs, want_vis in zip(tr["seeds"], tr["regs_cascade"], tr["visited"]):
            total += O.commit_cascade(g.n, off, adj, mask, J, regs, vis, s)
            assert total == want_vis
            assert regs.tobytes().hex() == want_regs


def test_runs_match_reference(golden):
    runs = golden["runs"]
    for case in runs["cases"]:
        g = _csr(runs["graphs"][case["graph"]])
        want = json.loads(case["json"])
        got = O.run(g, **case["config"])
        for key, val in got.items():
            assert want[key] == val, (case["config"], key)


def test_row_score_kats():
    # proj/tests/test_sketch.cpp:157-202
    assert O.row_score(np.zeros(1024, np.int8)) == pytest.approx(1024 / 0.77351, rel=1e-12)
    assert O.row_score(np.array([4, -1, 4, -1], np.int8)) == O.row_score(np.array([4, 4], np.int8))
    assert O.row_score(np.full(4, -1, np.int8)) == 0.0
    broad = np.full(64, 3, np.int8)
    narrow = np.full(64, -1, np.int8)
    narrow[:8] = 6
    assert O.row_score(broad) == pytest.approx(O.row_score(narrow))


def test_plan_semantics():
    # proj/tests/test_fasst.cpp:15-57
    with pytest.raises(ValueError):
        O.make_plan(65, 2, "fasst", 1)
    x, order, deg = O.make_plan(128, 4, "fasst", 3)
    assert list(x) == sorted(x) and not deg
    assert sorted(order.tolist()) == list(range(128))
    s = O.splitmix64_at(3, 1)
    assert all(x[i] == O.random_value_at(s, int(order[i])) for i in range(128))
    xn, on, degn = O.make_plan(128, 4, "naive", 3)
    assert on.tolist() == list(range(128)) and not degn
    assert O.make_plan(64, 4, "fasst", 3)[2] and not O.make_plan(64, 4, "naive", 3)[2]


REF, PROBE = O.load_reference()


@pytest.mark.skipif(REF is None, reason="compiled reference (oracle/_ref) not present")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_vs_live_reference(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 400))
    g = O.build_csr(*O.er_edges(n, int(n * rng.integers(2, 9)), seed))
    rg = REF.graph_from_text(g.edges_text())
    for cfg in [dict(k=min(6, g.n), r=64, devices=1, weights="const:0.2"),
                dict(k=min(5, g.n), r=256, devices=4, weights="wc"),
                dict(k=min(7, g.n), r=96, devices=3, weights="const:0.05", mode="naive")]:
        want = json.loads(REF.run_json(rg, timings=False, seed=seed, **cfg))
        got = O.run(g, seed=seed, **cfg)
        for key, val in got.items():
            assert want[key] == val, (cfg, key)


def test_golden_fixture_generator_present():
    assert os.path.exists(os.path.join(os.path.dirname(O.HERE), "oracle", "make_golden.py"))


def test_fasst_stats_match_reference(golden_fasst):
    """duplication_stats / device_edge_loads / fill_rate (fasst.cpp:101-168)
    of the restatement vs the compiled reference's own values."""
    gs = golden_fasst["graphs"]
    for c in golden_fasst["cases"]:
        gd = gs[c["graph"]]
        g = O.CSR(gd["offsets"], gd["adj"], gd["orig_ids"])
        got = O.fasst_stats(g, c["r"], c["mu"], c["mode"], c["weights"], c["seed"])
        for key in ("dup_count", "dup_fraction", "loads", "share_within_1", "share_within_2",
                    "fill_rate", "fill_batches"):
            if key in c:
                assert got[key] == c[key], (key, c["graph"], c["r"], c["mu"], c["mode"])
