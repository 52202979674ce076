"""GPU parity: the sm_100a path through the C-ABI vs the reference's golden
fixtures (tests/golden, produced by the compiled reference) and vs the oracle
restatement (oracle/, checked against the same fixtures in
test_oracle_golden.py).  Integer/byte state is compared bit-exactly; scores
are compared as IEEE bit patterns; reports byte-identically (minus timings).
"""
import json

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _graph(D, gd):
    return D.graph_from_csr(np.array(gd["offsets"], np.uint64), np.array(gd["adj"], np.uint32),
                            np.array(gd["orig_ids"], np.uint64))


@pytest.fixture(scope="module")
def D():
    import paper_2410_14047_b200 as D
    return D


def test_run_json_byte_identical(D, ctx, golden):
    runs = golden["runs"]
    for case in runs["cases"]:
        g = _graph(D, runs["graphs"][case["graph"]])
        got = ctx.run_json(g, timings=False, **case["config"])
        assert got == case["json"], (case["graph"], case["config"])


def test_run_json_jacobi_schedule_same_report(D, ctx, golden):
    runs = golden["runs"]
    for case in runs["cases"][:12]:
        g = _graph(D, runs["graphs"][case["graph"]])
        got = ctx.run_json(g, timings=False, jacobi=1, **case["config"])
        assert got == case["json"], (case["graph"], case["config"])


def test_stage_traces(D, ctx, golden):
    graphs = golden["runs"]["graphs"]
    for tr in golden["traces"]:
        g = _graph(D, graphs[tr["graph"]])
        ctx.prepare(g, r=tr["r"], devices=tr["mu"], mode=tr["mode"], weights=tr["weights"],
                    seed=tr["seed"])
        tau, J = tr["tau"], tr["r"] // tr["mu"]
        # sampled-edge set: device graph + baked masks (fasst.cpp:50-88)
        off, adj, mask, words = ctx.device_graph(tau)
        assert words == tr["mask_words"]
        assert off.tolist() == tr["dg_offsets"]
        assert adj.tolist() == tr["dg_adj"]
        assert mask.tolist() == tr["dg_mask"]
        # fill (sketch.cpp:55-66)
        ctx.fill(tau)
        assert ctx.registers(tau).tobytes().hex() == tr["regs_fill"]
        # simulate: async schedule -> same registers; Jacobi -> same sweep count too
        sweeps = ctx.simulate(tau)
        assert 1 <= sweeps <= tr["sweeps"]
        assert ctx.registers(tau).tobytes().hex() == tr["regs_sim"]
        ctx.fill(tau)
        assert ctx.simulate(tau, jacobi=1) == tr["sweeps"]
        assert ctx.registers(tau).tobytes().hex() == tr["regs_sim"]
        # row scores, bit-exact doubles (sketch.cpp:119-131)
        assert [float(s).hex() for s in ctx.scores(tau)] == tr["scores"]
        # commit + cascade (engine.cpp:106-144)
        for s, regs, vis in zip(tr["seeds"], tr["regs_cascade"], tr["visited"]):
            assert ctx.commit_cascade(tau, s) == vis
            assert ctx.registers(tau).tobytes().hex() == regs
        assert J == len(tr["regs_fill"]) // 2 // g.n


def _oracle_csr(g):
    return O.CSR(g.offsets, g.adj, np.array(g.orig_ids, np.uint64))


@pytest.mark.parametrize("devices", [1, 8])
def test_c1_config_matches_oracle(D, ctx, devices):
    """BASELINE configs[0]: ER n=10k avg-deg 8, IC p=0.1, R=64, K=10."""
    g = D.generate("er", 10000, 80000, 7)
    got = json.loads(ctx.run_json(g, k=10, r=64, devices=devices, weights="const:0.1", seed=7,
                                  timings=False))
    ref = O.run(_oracle_csr(g), k=10, r=64, devices=devices, weights="const:0.1", seed=7)
    for key, val in ref.items():
        assert got[key] == val, key


@pytest.mark.parametrize("spec", [
    dict(n=3000, m=24000, k=12, r=256, devices=1, weights="const:0.05"),
    dict(n=3000, m=24000, k=12, r=256, devices=2, weights="wc"),
    dict(n=2000, m=30000, k=8, r=96, devices=3, weights="const:0.2", mode="naive"),
    dict(n=5000, m=20000, k=15, r=1024, devices=4, weights="const:0.01"),
    dict(n=1500, m=9000, k=10, r=100, devices=1, weights="const:0.3", rebuild_eps=0.0),
])
def test_random_configs_match_oracle(D, ctx, spec):
    spec = dict(spec)
    n, m = spec.pop("n"), spec.pop("m")
    g = D.generate("er", n, m, 11)
    got = json.loads(ctx.run_json(g, seed=5, timings=False, **spec))
    ref = O.run(_oracle_csr(g), seed=5, **spec)
    for key, val in ref.items():
        assert got[key] == val, key


def test_rmat_registers_match_oracle(D, ctx):
    g = D.generate("rmat", 12, 40000, 3)
    cg = _oracle_csr(g)
    for r, mu, w in [(256, 1, "const:0.01"), (512, 2, "wc"), (64, 1, "const:0.2")]:
        ctx.prepare(g, r=r, devices=mu, weights=w, seed=9)
        wf = cg.weights(w)
        x, _, _ = O.make_plan(r, mu, "fasst", 9)
        J = r // mu
        for tau in range(mu):
            off, adj, mask = O.device_graph(cg, wf, x[tau * J:(tau + 1) * J])
            goff, gadj, gmask, _ = ctx.device_graph(tau)
            assert np.array_equal(off, goff) and np.array_equal(adj, gadj)
            assert np.array_equal(mask, gmask)
            regs = O.fill(g.n, J, tau * J, O.splitmix64_at(9, 2))
            ctx.fill(tau)
            assert np.array_equal(ctx.registers(tau), regs)
            sweeps = O.simulate(g.n, off, adj, mask, J, regs)
            assert ctx.simulate(tau) <= sweeps
            assert np.array_equal(ctx.registers(tau), regs)
            ctx.fill(tau)
            assert ctx.simulate(tau, jacobi=1) == sweeps
            sc = ctx.scores(tau)
            want = [O.row_score(regs[u * J:(u + 1) * J]) for u in range(g.n)]
            assert sc.tolist() == want


def test_pre_visited_registers_respected(D, ctx):
    """engine test 'simulate respects pre-VISITED registers'."""
    g = D.generate("er", 20, 60, 3)
    ctx.prepare(g, r=64, weights="const:0.8", seed=9)
    rng = np.random.default_rng(4)
    regs = np.zeros(g.n * 64, np.int8)
    for _ in range(200):
        regs[rng.integers(g.n) * 64 + rng.integers(64)] = -1
    before = int((regs == -1).sum())
    ctx.set_registers(0, regs)
    ctx.fill(0)
    cg = _oracle_csr(g)
    x, _, _ = O.make_plan(64, 1, "fasst", 9)
    off, adj, mask = O.device_graph(cg, cg.weights("const:0.8"), x)
    ref = regs.copy()
    O.fill(g.n, 64, 0, O.splitmix64_at(9, 2), ref)
    O.simulate(g.n, off, adj, mask, 64, ref)
    ctx.simulate(0)
    got = ctx.registers(0)
    assert np.array_equal(got, ref)
    assert int((got == -1).sum()) == before == ctx.visited_count(0)


def test_simulate_cap_and_depth():
    """Chain of 12, max planted at the tail: Jacobi needs depth+1 = 12 sweeps,
    cap 3 raises (tests/test_engine.cpp:114-134)."""
    import paper_2410_14047_b200 as D
    ctx = D.Context(0)
    g = D.graph_from_csr(np.array(list(range(12)) + [11], np.uint64),
                         np.arange(1, 12, dtype=np.uint32), list(range(12)))
    ctx.prepare(g, r=64, weights="const:1", seed=5)
    regs = np.zeros(12 * 64, np.int8)
    regs[11 * 64] = 50
    ctx.set_registers(0, regs)
    with pytest.raises(RuntimeError):
        ctx.simulate(0, cap=3, jacobi=1)
    ctx.set_registers(0, regs)
    assert ctx.simulate(0, cap=64, jacobi=1) == 12
    assert all(ctx.registers(0)[u * 64] == 50 for u in range(12))


def test_recommit_covered_seed_is_noop(D, ctx):
    g = D.graph_from_csr(np.array([0, 1, 2, 3, 4, 5, 5], np.uint64),
                         np.arange(1, 6, dtype=np.uint32), list(range(6)))
    ctx.prepare(g, r=32, weights="const:1", seed=2)
    ctx.fill(0)
    assert ctx.commit_cascade(0, 0) == 6 * 32
    assert ctx.commit_cascade(0, 3) == 6 * 32


def test_validation_errors(D, ctx):
    g = D.graph_from_text("0 1\n1 2\n2 3\n")
    with pytest.raises(ValueError):
        ctx.run_json(g, k=0, r=64)
    with pytest.raises(ValueError):
        ctx.run_json(g, k=5, r=64)
    with pytest.raises(ValueError):
        ctx.run_json(g, k=1, r=64, devices=0)
    with pytest.raises(ValueError):
        ctx.run_json(g, k=1, r=63, devices=2)
    with pytest.raises(ValueError):
        ctx.run_json(g, k=1, r=64, rebuild_eps=-0.5)
    with pytest.raises(ValueError):
        ctx.run_json(g, k=1, r=0)
    with pytest.raises(RuntimeError):
        ctx.run_json(g, k=1, r=64, mode="bogus")
    with pytest.raises(RuntimeError):
        ctx.run_json(g, k=1, r=64, weights="const:2")


def test_python_smoke_mirror(D):
    """tests/py/test_smoke.py:40-51 through the package-level API."""
    chain = D.graph_from_text("0 1\n1 2\n2 3\n", directed=True)
    rep = D.run(chain, k=2, r=64, weights="const:1", seed=3)
    assert rep["seeds"][0] == 0
    assert rep["config"]["k"] == 2
    assert len(rep["score_trajectory"]) == 2
    assert rep["score_trajectory"][0] == pytest.approx(4.0)
    assert rep["saturated"]
    quiet = json.loads(D.run_json(chain, k=2, r=64, weights="const:1", seed=3, timings=False))
    assert "timings" not in quiet
    assert quiet["seeds"] == rep["seeds"]
    assert set(rep["timings"]) == {"build", "fill", "simulate", "select", "cascade", "total"}


def test_partition_contexts_match_reference(D, golden):
    """The multi-process path's per-partition C-ABI (dfs_prepare_partition,
    dfs_scores_device, dfs_rebuild, commit/cascade) driven for mu partitions on
    one GPU, with the exchange done locally in the binomial order."""
    import ctypes as C
    import torch
    from paper_2410_14047_b200 import _capi, _config
    from paper_2410_14047_b200.dist import binomial_sum, select_seed
    runs = golden["runs"]
    for case in [c for c in runs["cases"] if c["config"]["devices"] in (2, 3, 4)]:
        cfg = dict(case["config"])
        g = _graph(D, runs["graphs"][case["graph"]])
        mu, k, r = cfg["devices"], cfg["k"], cfg["r"]
        ctxs = [D.Context(0) for _ in range(mu)]
        bufs = []
        for t, cx in enumerate(ctxs):
            c = _config(k, r, mu, cfg.get("mode", "fasst"), cfg["weights"],
                        cfg.get("rebuild_eps", 0.01), cfg.get("seed", 0))
            _capi.check(_capi.lib().dfs_prepare_partition(cx._h, g._h, C.byref(c), t, mu))
            _capi.check(_capi.lib().dfs_rebuild(cx._h, 0))
            b = torch.empty(g.n, dtype=torch.float64, device="cuda")
            _capi.check(_capi.lib().dfs_scores_device(cx._h, 0, 1, C.c_void_p(b.data_ptr())))
            bufs.append(b)
        committed = torch.zeros(g.n, dtype=torch.bool, device="cuda")
        want = json.loads(case["json"])
        old, seeds, traj, rb = 0.0, [], [], []
        rebuilt = True
        for step in range(k):
            if not rebuilt:
                for cx, b in zip(ctxs, bufs):
                    _capi.check(_capi.lib().dfs_scores_device(cx._h, 0, 0, C.c_void_p(b.data_ptr())))
            rebuilt = False
            s, _ = select_seed(binomial_sum(torch.stack(bufs)), committed, 0, 1)
            committed[s] = True
            covered = sum(cx.commit_cascade(0, s) for cx in ctxs)
            score = covered / r
            seeds.append(s)
            traj.append(score)
            if step + 1 < k and (score - old) > cfg.get("rebuild_eps", 0.01) * score:
                for cx, b in zip(ctxs, bufs):
                    _capi.check(_capi.lib().dfs_rebuild(cx._h, 0))
                    _capi.check(_capi.lib().dfs_scores_device(cx._h, 0, 1, C.c_void_p(b.data_ptr())))
                rebuilt = True
                old = score
                rb.append(step)
        assert seeds == want["seeds_dense"], cfg
        assert traj == want["score_trajectory"], cfg
        assert rb == want["rebuild_rounds"], cfg


def test_dist_runner_single_rank_report(D, ctx, golden):
    """DistRunner (the multi-process driver) at world=1 produces the reference
    report byte-for-byte."""
    from paper_2410_14047_b200.dist import DistRunner
    runs = golden["runs"]
    for case in [c for c in runs["cases"] if c["config"]["devices"] == 1][:6]:
        cfg = dict(case["config"])
        cfg.pop("devices")
        g = _graph(D, runs["graphs"][case["graph"]])
        got = DistRunner(ctx, g, 0, 1).run(**cfg)
        assert got == case["json"], case["config"]


def test_fasst_stats_match_reference(D, ctx, golden_fasst):
    """FASST analytics on the GPU (duplication histogram, per-device edge loads,
    fill rate; proj/src/fasst.cpp:101-168) vs the compiled reference."""
    gs = golden_fasst["graphs"]
    for c in golden_fasst["cases"]:
        g = _graph(D, gs[c["graph"]])
        got = ctx.fasst_stats(g, r=c["r"], devices=c["mu"], mode=c["mode"], weights=c["weights"],
                              seed=c["seed"])
        for key in ("dup_count", "dup_fraction", "loads", "share_within_1", "share_within_2",
                    "fill_rate", "fill_batches"):
            if key in c:
                assert got[key] == c[key], (key, c["graph"], c["r"], c["mu"], c["mode"])


@pytest.mark.parametrize("mode", ["fasst", "naive"])
def test_fasst_stats_match_oracle_rmat(D, ctx, mode):
    g = D.generate("rmat", 14, 200000, 3)
    got = ctx.fasst_stats(g, r=1024, devices=8, mode=mode, weights="wc", seed=5)
    want = O.fasst_stats(_oracle_csr(g), 1024, 8, mode, "wc", 5)
    assert got == want


def test_mc_influence_matches_reference(D, ctx, golden_influence):
    """Monte-Carlo influence on the GPU (32 mt19937_64 streams per block, bitset
    BFS) == the reference's influence() bit for bit (oracle.cpp:30-79)."""
    gs = golden_influence["graphs"]
    for c in golden_influence["cases"]:
        g = _graph(D, gs[c["graph"]])
        mean, se = ctx.influence(g, c["seeds"], trials=c["trials"], seed=c["seed"], runs=c["runs"],
                                 weights=c["weights"])
        assert (mean.hex(), se.hex()) == (c["mean"], c["std_error"]), c


def test_mc_influence_gpu_equals_host_rmat(D, ctx):
    g = D.generate("rmat", 12, 40000, 5)
    seeds = [0, 3, 77, 1000]
    for w in ("const:0.05", "wc"):
        got = ctx.influence(g, seeds, trials=200, seed=2, runs=2, weights=w)
        assert got == D.influence(g, seeds, trials=200, seed=2, runs=2, weights=w)
    with pytest.raises(ValueError):
        ctx.influence(g, [g.n], trials=10)
    with pytest.raises(ValueError):
        ctx.influence(g, [0], trials=0)


def test_widest_partition_matches_oracle(D, ctx):
    """J = 8192 simulations in one partition (byte batch index at its limit;
    pull paths disabled above 4096, push only) and a 4096-wide one."""
    g = D.generate("er", 1500, 9000, 13)
    cg = _oracle_csr(g)
    for r in (8192, 4096):
        got = json.loads(ctx.run_json(g, k=3, r=r, weights="const:0.05", seed=2, timings=False))
        want = O.run(cg, k=3, r=r, devices=1, weights="const:0.05", seed=2)
        for key, val in want.items():
            assert got[key] == val, (r, key)
