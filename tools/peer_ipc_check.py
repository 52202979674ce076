"""Peer mode across PROCESSES (CUDA IPC mappings, torch.distributed gloo only
for the handle swap): `world` processes, every one on cuda:0 of this box (or
cuda:rank with --spread), run one greedy IM run in peer mode and compare the
report with the oracle at devices = world.  On one GPU the processes' kernels
are time-sliced (no MPS), so this checks the protocol, not speed.
Usage: python tools/peer_ipc_check.py [world] [--spread]"""
import json
import os
import sys

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, spread, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2410_14047_b200 as D
    from paper_2410_14047_b200.dist import PeerRunner
    g = D.generate("er", 3000, 24000, 11)
    ctx = D.Context(rank if spread else 0)
    ctx.upload(g)
    pr = PeerRunner(ctx, g, rank, world)
    reps = [pr.run_json(k=8, r=128, weights="const:0.1", seed=5) for _ in range(2)]
    q.put((rank, reps))
    dist.barrier()
    dist.destroy_process_group()


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    spread = "--spread" in sys.argv
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    ps = [ctx.Process(target=worker, args=(r, world, spread, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join()
    import oracle as O
    import paper_2410_14047_b200 as D
    g = D.generate("er", 3000, 24000, 11)
    want = O.run(O.CSR(g.offsets, g.adj, np.array(g.orig_ids, np.uint64)), k=8, r=128,
                 devices=world, weights="const:0.1", seed=5)
    ok = True
    for r, reps in sorted(res.items()):
        for rep in reps:
            got = json.loads(rep)
            bad = [k for k, v in want.items() if got[k] != v]
            ok &= not bad
            print(f"rank {r}: seeds {got['seeds'][:5]}... mismatched keys: {bad}")
    print("PEER IPC", "OK" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
