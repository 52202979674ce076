"""Peer (multi-GPU) mode: one process per rank, one FASST partition each.
The per-round exchange (binomial-order partial-score reduce, argmax, seed
broadcast, visited-count allreduce; proj/src/runtime.cpp:88-130,
collectives.cpp:44-113) happens INSIDE every rank's persistent kernel over
peer memory (CUDA IPC mappings; NVLink loads on a multi-GPU box); gloo only
swaps the IPC handles.  On the one-GPU test box all ranks share cuda:0 and
their kernels are time-sliced, which exercises the same protocol.  Every rank
must return the reference's report for devices = world byte-for-byte (golden
fixtures from the compiled reference; the oracle on generated graphs).
"""
import json
import os
import sys

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _spawn(world, cases):
    import torch.multiprocessing as mp
    if HERE not in sys.path:
        sys.path.insert(0, HERE)
    import peer_worker
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 23000 + (os.getpid() * 7 + world) % 20000
    ps = [ctx.Process(target=peer_worker.worker, args=(r, world, port, cases, q))
          for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, out, err = q.get(timeout=900)
            assert err is None, (r, err)
            res[r] = out
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    return res


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_peer_processes_match_reference_reports(golden, world):
    runs = golden["runs"]
    sel = [c for c in runs["cases"] if c["config"]["devices"] == world]
    if not sel:
        pytest.skip(f"no golden case with devices={world}")
    cases = []
    for c in sel:
        gd = runs["graphs"][c["graph"]]
        cases.append((("csr", gd["offsets"], gd["adj"], gd["orig_ids"]), c["config"], 1, True))
    res = _spawn(world, cases)
    for r in range(world):
        for c, reps in zip(sel, res[r]):
            assert reps[0] == c["json"], (r, c["graph"], c["config"])


def test_peer_processes_match_oracle():
    """Generated graphs at world 2, two runs per setup (barrier epochs carry
    over between runs), the host-upload (e2e) path and the resident path."""
    world = 2
    specs = [(("er", 3000, 24000, 11), dict(k=12, r=128, weights="const:0.1", seed=5)),
             (("rmat", 12, 30000, 11), dict(k=10, r=256, weights="wc", seed=5))]
    cases = [(sp, cfg, 2, res) for (sp, cfg), res in zip(specs, (True, False))]
    out = _spawn(world, cases)
    import paper_2410_14047_b200 as D
    import peer_worker
    for i, (sp, cfg) in enumerate(specs):
        g = peer_worker.make_graph(D, sp)
        want = O.run(O.CSR(g.offsets, g.adj, np.array(g.orig_ids, np.uint64)), devices=world,
                     **cfg)
        for r in range(world):
            reps = out[r][i]
            assert reps[0] == reps[1]
            rep = json.loads(reps[0])
            for key, val in want.items():
                assert rep[key] == val, (key, sp, r)


def test_peer_setup_errors():
    import paper_2410_14047_b200 as D
    g = D.generate("er", 500, 3000, 2)
    cx = D.Context(0)
    cx.upload(g)
    with pytest.raises(RuntimeError):  # no peer setup
        cx.run_peer_json(None, k=2, r=64, devices=2, resident=True)
    cx.prepare_partition(g, 0, 2, k=2, r=64)
    with pytest.raises(ValueError):  # a world of one is not a peer session
        D.peer_link([cx])
    cy = D.Context(0)
    cy.upload(g)
    cy.prepare_partition(g, 1, 2, k=2, r=64)
    with pytest.raises(ValueError):  # same process + same device: one process per rank
        D.peer_link([cx, cy])


def test_peer_processes_many_segments_and_rounds():
    """Slices spanning many argmax-cache segments, rebuilds and 30 rounds at
    world 3 (uneven slices)."""
    world = 3
    sp, cfg = ("rmat", 14, 150000, 4), dict(k=30, r=96, weights="const:0.05", seed=9)
    out = _spawn(world, [(sp, cfg, 1, True)])
    import paper_2410_14047_b200 as D
    import peer_worker
    g = peer_worker.make_graph(D, sp)
    want = O.run(O.CSR(g.offsets, g.adj, np.array(g.orig_ids, np.uint64)), devices=world, **cfg)
    for r in range(world):
        rep = json.loads(out[r][0][0])
        for key, val in want.items():
            assert rep[key] == val, (key, r)


def test_peer_dead_rank_fails_instead_of_hanging():
    """A rank that never reaches the round barriers (failed process): the
    survivors' kernels give up after DFS_PEER_TIMEOUT_S and the call raises
    RuntimeError (SURVEY §5 failure detection) instead of hanging the GPU."""
    os.environ["DFS_PEER_TIMEOUT_S"] = "3"
    try:
        out = _spawn(2, [(("er", 2000, 16000, 5), dict(k=4, r=64, weights="const:0.1", seed=1),
                          1, True, 1)])
    finally:
        del os.environ["DFS_PEER_TIMEOUT_S"]
    assert out[1][0] == ["dead"]
    msg = out[0][0][0]
    assert msg.startswith("ERR:") and "peer" in msg, msg


def _torchrun(args, timeout=900):
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(os.path.dirname(HERE), "bench.py")] + args
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout,
                         cwd=os.path.dirname(HERE))
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


def test_scale_command_path_two_ranks():
    """The driver's scaling command (torchrun -> bench.py --gpus 2 -> PeerRunner)
    end to end, both ranks sharing this GPU: one JSON line, the reference's
    devices=2 report reproduced byte-for-byte."""
    line = _torchrun(["--gpus", "2", "--share-gpu", "--steps", "2", "--warmup", "1",
                      "--no-north-star", "--no-cpu-baseline"])
    assert line["n_gpus"] == 2 and line["config"]["devices"] == 2
    assert line["metric"] and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["report_parity"] == "identical"


def test_scale_command_path_reference_arm():
    """--impl reference under torchrun: rank 0 alone runs the unmodified
    reference at devices = world and reports the same config."""
    line = _torchrun(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0"])
    assert line["impl"] == "reference" and line["config"]["devices"] == 2
    assert line["report_parity"] == "identical"
