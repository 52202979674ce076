"""Multi-GPU greedy loop: one process per GPU, one FASST partition per rank.

Sample-space partitioning (proj/src/fasst.cpp:21-88) gives rank tau the
sorted simulation slots [tau*J, (tau+1)*J), its own sampled items, registers
and visited bits: fill, simulate and cascade need no communication.  The only
exchange is once per greedy round (proj/src/runtime.cpp:88-130):

  1. every rank rescores the rows its last cascade touched (device buffer);
  2. ``all_to_all`` of score slices: rank k receives the mu partial scores of
     vertex range k and sums them in the reference's binomial-tree order
     (proj/src/collectives.cpp:44-64) — bit-identical to reduce_to_root;
  3. slice argmax (strict > from 0.0, committed skipped, ties to the smallest
     id; saturation falls back to the smallest uncommitted id,
     runtime.cpp:95-119), ``all_gather`` of (score, id, min-uncommitted) so
     every rank picks the same seed — this replaces the seed broadcast;
  4. commit + cascade locally, ``all_reduce`` (int64 sum) of the visited
     counts (collectives.cpp:96-113) -> score = covered / R;
  5. the eps-gated rebuild decision is identical on every rank.

No floating-point all-reduce is used: NCCL's summation order is not the
reference's tree order.  The protocol functions are backend-agnostic (NCCL on
GPUs, gloo on CPU for tests).
"""
from __future__ import annotations

import ctypes as C
import math
import time

import numpy as np
import torch
import torch.distributed as dist

from . import _capi
from ._capi import ReportFields, check, lib


def binomial_sum(parts: torch.Tensor) -> torch.Tensor:
    """Sum parts[0..mu) in binomial-tree order: level k folds rank+2^k into
    rank for ranks aligned to 2^(k+1) (collectives.cpp:51-59)."""
    acc = [parts[t].clone() for t in range(parts.shape[0])]
    mu = len(acc)
    step = 1
    while step < mu:
        for t in range(0, mu, 2 * step):
            if t + step < mu:
                acc[t] += acc[t + step]
        step *= 2
    return acc[0]


def select_seed(local_scores: torch.Tensor, committed: torch.Tensor, rank: int, world: int,
                group=None):
    """Steps 2-3 above.  local_scores: this rank's partial score of every row
    (n doubles); committed: bool[n], identical on all ranks.  Returns
    (seed, saturated) — identical on every rank."""
    n = local_scores.shape[0]
    S = max(1, math.ceil(n / world))
    dev = local_scores.device
    send = torch.zeros(world * S, dtype=torch.float64, device=dev)
    send[:n] = local_scores
    recv = torch.empty_like(send)
    if world > 1:
        dist.all_to_all_single(recv, send, group=group)
    else:
        recv.copy_(send)
    red = binomial_sum(recv.view(world, S))
    lo = rank * S
    com = torch.ones(S, dtype=torch.bool, device=dev)
    hi = min(n, lo + S)
    if hi > lo:
        com[:hi - lo] = committed[lo:hi]
    masked = torch.where(com | ~(red > 0), torch.full_like(red, -1.0), red)
    idx = int(torch.argmax(masked).item())  # first maximal element
    val = float(masked[idx].item())
    free = (~com).nonzero()
    minu = lo + int(free[0].item()) if free.numel() else 1 << 62
    mine = torch.tensor([val, float(lo + idx), float(minu)], dtype=torch.float64, device=dev)
    if world > 1:
        allv = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allv, mine, group=group)
    else:
        allv = [mine]
    rows = [(float(t[0].item()), int(t[1].item()), int(t[2].item())) for t in allv]
    best_v, best_i = -1.0, None
    for v, i, _ in rows:  # ranks hold ascending id ranges: first max wins ties
        if v > 0 and v > best_v:
            best_v, best_i = v, i
    if best_i is not None:
        return best_i, False
    return min(m for _, _, m in rows), True


def allreduce_count(value: int, device, group=None) -> int:
    t = torch.tensor([value], dtype=torch.int64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def _ceil_log2(mu):
    l, s = 0, 1
    while s < mu:
        l, s = l + 1, s * 2
    return l


class DistRunner:
    """Drives one rank (one GPU) of a multi-process IM run through the C-ABI."""

    def __init__(self, ctx, graph, rank: int, world: int, group=None):
        self.ctx, self.g, self.rank, self.world, self.group = ctx, graph, rank, world, group
        self.dev = torch.device("cuda", ctx.device)

    def run(self, k=10, r=256, mode="fasst", weights="const:0.1", rebuild_eps=0.01, seed=0,
            resident=False, timings=False):
        from . import _config
        t0 = time.perf_counter()
        ctx, g = self.ctx, self.g
        cfg = _config(k, r, self.world, mode, weights, rebuild_eps, seed)
        check(lib().dfs_prepare_partition(ctx._h, None if resident else g._h, C.byref(cfg),
                                          self.rank, self.world))
        n = g.n
        J = r // self.world
        scores = torch.empty(max(n, 1), dtype=torch.float64, device=self.dev)
        committed = torch.zeros(n, dtype=torch.bool, device=self.dev)
        check(lib().dfs_rebuild(ctx._h, 0))  # fill + simulate + full score
        check(lib().dfs_scores_device(ctx._h, 0, 1, C.c_void_p(scores.data_ptr())))
        seeds_dense, traj, rebuild_rounds = [], [], []
        saturated = False
        oldscore = 0.0
        rebuilt = True
        for step in range(k):
            if not rebuilt:  # rows dirtied by the last cascade only
                check(lib().dfs_scores_device(ctx._h, 0, 0, C.c_void_p(scores.data_ptr())))
            rebuilt = False
            s, sat = select_seed(scores[:n], committed, self.rank, self.world, self.group)
            saturated |= sat
            committed[s] = True
            local = ctx.commit_cascade(0, s)
            covered = allreduce_count(local, self.dev, self.group)
            score = covered / r
            seeds_dense.append(s)
            traj.append(score)
            if step + 1 < k and (score - oldscore) > rebuild_eps * score:
                check(lib().dfs_rebuild(ctx._h, 0))
                check(lib().dfs_scores_device(ctx._h, 0, 1, C.c_void_p(scores.data_ptr())))
                rebuilt = True
                oldscore = score
                rebuild_rounds.append(step)
        total = time.perf_counter() - t0
        mu = self.world
        orig = g.orig_ids
        f = ReportFields()
        f.k, f.r, f.devices = k, r, mu
        f.mode, f.weights, f.rebuild_eps, f.seed = mode.encode(), weights.encode(), rebuild_eps, seed
        f.n, f.m, f.steps = n, g.m, k
        a_seeds = np.array([orig[s] for s in seeds_dense], np.uint64)
        a_dense = np.array(seeds_dense, np.uint32)
        a_traj = np.array(traj, np.float64)
        a_rb = np.array(rebuild_rounds if rebuild_rounds else [0], np.uint32)
        f.seeds, f.seeds_dense, f.traj = a_seeds.ctypes.data, a_dense.ctypes.data, a_traj.ctypes.data
        f.rebuilds, f.rebuild_rounds = len(rebuild_rounds), a_rb.ctypes.data
        f.saturated = int(saturated)
        f.degraded = int(mode == "fasst" and J < 32)
        f.reduced_elements = k * (n + 1) * (mu - 1)
        f.broadcast_elements = k * 2 * (mu - 1)
        f.barriers = k * (8 + _ceil_log2(mu))
        f.with_timings = int(timings)
        f.t_total = total
        out = C.c_void_p()
        check(lib().dfs_format_report(C.byref(f), C.byref(out)))
        return ctx._take_json(out)

    def run_json(self, **kw):
        return self.run(**kw)


class PeerRunner:
    """One rank (one GPU, one process) of a multi-GPU run in PEER mode: the
    whole greedy loop is one persistent kernel per GPU and the per-round
    exchange (binomial-order partial-score reduce, argmax, seed broadcast,
    visited-count allreduce; runtime.cpp:88-130) happens inside it over
    NVLink peer memory (CUDA IPC mappings of every rank's mailbox and partial
    score vector).  torch.distributed is used only to swap the IPC handles.
    """

    def __init__(self, ctx, graph, rank: int, world: int, group=None):
        self.ctx, self.g, self.rank, self.world, self.group = ctx, graph, rank, world, group
        self._key = None

    def setup(self, k=10, r=256, mode="fasst", weights="const:0.1", rebuild_eps=0.01, seed=0,
              resident=True):
        if dist.is_initialized():
            dist.barrier(group=self.group)  # no peer kernel of a previous run is still reading
        self.ctx.prepare_partition(None if resident else self.g, self.rank, self.world, k=k, r=r,
                                   mode=mode, weights=weights, rebuild_eps=rebuild_eps, seed=seed,
                                   resident=resident)
        mine = self.ctx.peer_export()
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=self.group)
        self.ctx.peer_open(self.rank, self.world, handles)
        self._key = (self.g.n, self.g.m, r, mode)

    def run_json(self, k=10, r=256, mode="fasst", weights="const:0.1", rebuild_eps=0.01, seed=0,
                 resident=True, timings=False):
        if self._key != (self.g.n, self.g.m, r, mode):
            self.setup(k=k, r=r, mode=mode, weights=weights, rebuild_eps=rebuild_eps, seed=seed,
                       resident=True)
        try:
            return self.ctx.run_peer_json(None if resident else self.g, k=k, r=r,
                                          devices=self.world, mode=mode, weights=weights,
                                          rebuild_eps=rebuild_eps, seed=seed, timings=timings,
                                          resident=resident)
        except RuntimeError:
            self._key = None  # a failed peer run invalidates the mapping: set up again next time
            raise


__all__ = ["binomial_sum", "select_seed", "allreduce_count", "DistRunner", "PeerRunner", "_capi"]
