"""N>1 host path on CPU: the product's multi-rank exchange protocol
(paper_2410_14047_b200.dist: all_to_all score slices, binomial-order sum,
slice argmax + all_gather, int64 covered all_reduce) run by world_size-2 gloo
processes.  Each rank's partition state (registers, cascade) comes from the
oracle restatement, so the selected seeds / trajectory / rebuild rounds must
equal the reference's own run with devices=2 (golden fixtures)."""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, cases, graphs, outq):
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    from paper_2410_14047_b200.dist import allreduce_count, select_seed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    results = []
    for case in cases:
        cfg = case["config"]
        gd = graphs[case["graph"]]
        g = O.CSR(gd["offsets"], gd["adj"], gd["orig_ids"])
        k, r, mu = cfg["k"], cfg["r"], cfg["devices"]
        w = g.weights(cfg.get("weights", "const:0.1"), cfg.get("seed", 0))
        seed = cfg.get("seed", 0)
        x, _, _ = O.make_plan(r, mu, cfg.get("mode", "fasst"), seed)
        J = r // mu
        off, adj, mask = O.device_graph(g, w, x[rank * J:(rank + 1) * J])
        key = O.splitmix64_at(seed, 2)
        regs = O.fill(g.n, J, rank * J, key)
        O.simulate(g.n, off, adj, mask, J, regs)
        vis = np.zeros(g.n * ((J + 63) // 64) + 1, np.uint64)
        committed = torch.zeros(g.n, dtype=torch.bool)
        visited, old, eps = 0, 0.0, cfg.get("rebuild_eps", 0.01)
        seeds, traj, rb, sat_any = [], [], [], False
        for step in range(k):
            sc = torch.tensor([O.row_score(regs[u * J:(u + 1) * J]) for u in range(g.n)],
                              dtype=torch.float64)
            s, sat = select_seed(sc, committed, rank, world)
            sat_any |= sat
            committed[s] = True
            visited += O.commit_cascade(g.n, off, adj, mask, J, regs, vis, s)
            score = allreduce_count(visited, torch.device("cpu")) / r
            seeds.append(s)
            traj.append(score)
            if step + 1 < k and (score - old) > eps * score:
                O.fill(g.n, J, rank * J, key, regs)
                O.simulate(g.n, off, adj, mask, J, regs)
                old = score
                rb.append(step)
        results.append({"seeds_dense": seeds, "score_trajectory": traj, "rebuild_rounds": rb,
                        "saturated": sat_any})
    outq.put((rank, results))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_protocol_matches_reference(golden, world):
    runs = golden["runs"]
    cases = [c for c in runs["cases"] if c["config"]["devices"] == world]
    assert cases
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, cases, runs["graphs"], q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for case, *ranks in zip(cases, *[got[r] for r in range(world)]):
        want = json.loads(case["json"])
        for res in ranks:  # every rank reaches the same decisions
            for key in ("seeds_dense", "score_trajectory", "rebuild_rounds", "saturated"):
                assert res[key] == want[key], (case["config"], key)


def test_binomial_sum_is_the_reference_tree_order():
    from paper_2410_14047_b200.dist import binomial_sum
    vals = [1e16, 1.0, -1e16, 3.1415926535897932, 2.718281828459045e-8, 7.0, -3.5, 1e-300]
    for mu in (1, 2, 3, 5, 8):
        parts = torch.tensor([[vals[t % len(vals)]] * 4 for t in range(mu)], dtype=torch.float64)
        acc = [vals[t % len(vals)] for t in range(mu)]
        step = 1
        while step < mu:  # proj/src/collectives.cpp:51-59
            for t in range(0, mu, 2 * step):
                if t + step < mu:
                    acc[t] = acc[t] + acc[t + step]
            step *= 2
        assert binomial_sum(parts).tolist() == [acc[0]] * 4
