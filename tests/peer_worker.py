"""Rank process of the multi-process peer-mode tests (test_gpu_peer.py).
Not a test module: spawned by torch.multiprocessing with the tests dir on
sys.path.  Every rank uses cuda:0 of the test box (the ranks' persistent
kernels are time-sliced there), swaps CUDA IPC handles over gloo and runs
each case through PeerRunner (the multi-GPU driver of bench.py)."""
import os

import numpy as np


def make_graph(D, spec):
    if spec[0] == "csr":
        _, off, adj, oid = spec
        return D.graph_from_csr(np.array(off, np.uint64), np.array(adj, np.uint32),
                                np.array(oid, np.uint64))
    kind, a, m, seed = spec
    return D.generate(kind, a, m, seed)


def worker(rank, world, port, cases, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2410_14047_b200 as D
        from paper_2410_14047_b200.dist import PeerRunner
        ctx = D.Context(0)
        out = []
        for case in cases:
            spec, cfg, repeat, resident = case[:4]
            dead = case[4] if len(case) > 4 else None  # rank that sets up but never runs
            g = make_graph(D, spec)
            ctx.upload(g)
            pr = PeerRunner(ctx, g, rank, world)
            kw = {k: v for k, v in cfg.items() if k != "devices"}
            if dead is not None:
                pr.setup(**kw)
                if rank == dead:
                    out.append(["dead"])
                    continue
                try:
                    out.append([pr.run_json(resident=resident, timings=False, **kw)])
                except RuntimeError as ex:
                    out.append(["ERR:" + str(ex)])
                continue
            reps = [pr.run_json(resident=resident, timings=False, **kw) for _ in range(repeat)]
            out.append(reps)
        q.put((rank, out, None))
    except Exception as ex:  # reported to the parent
        q.put((rank, None, repr(ex)))
    finally:
        dist.destroy_process_group()
