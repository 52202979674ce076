"""B200-native sketch-based influence maximization (DiFuseR, arxiv 2410.14047).

Drop-in mirror of the reference's Python surface (``difuser`` package,
proj/python/difuser/__init__.py and proj/bindings/pymodule.cpp): the same
names, keyword defaults and exception classes, backed by hand-written sm_100a
kernels behind the C-ABI in ``include/difuser_b200.h``.  There is no CPU
fallback: without the built library or a GPU the hot-path calls raise.
"""
from __future__ import annotations

import ctypes as C
import json as _json
import threading

import numpy as np

from . import _capi
from ._capi import Config, Stats, check, lib

__all__ = ["_config", 
    "Graph", "edge_hash", "graph_from_text", "greedy_exact", "influence", "is_sampled",
    "load_graph", "random_value_at", "run", "run_json", "save_cache", "generate", "Context",
    "peer_link", "fasst_stats",
]


class Graph:
    """Immutable dense CSR graph (proj/include/difuser/graph.hpp:44-58)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        capi = globals().get("_capi")  # None while the interpreter tears modules down
        if h is not None and h.value and capi is not None and capi._lib is not None:
            capi._lib.dfs_graph_free(h)
            self._h = None

    @property
    def n(self) -> int:
        return int(lib().dfs_graph_n(self._h))

    @property
    def m(self) -> int:
        return int(lib().dfs_graph_m(self._h))

    def _arrays(self):
        ps = [C.c_void_p() for _ in range(5)]
        check(lib().dfs_graph_arrays(self._h, *[C.byref(p) for p in ps]))
        return ps

    def _view(self, idx, dtype, count):
        if count == 0:
            return np.zeros(0, dtype)
        p = self._arrays()[idx].value
        buf = (C.c_char * (count * np.dtype(dtype).itemsize)).from_address(p)
        return np.frombuffer(buf, dtype=dtype, count=count).copy()

    @property
    def offsets(self) -> np.ndarray:
        return self._view(0, np.uint64, self.n + 1)

    @property
    def adj(self) -> np.ndarray:
        return self._view(1, np.uint32, self.m)

    @property
    def ehash(self) -> np.ndarray:
        return self._view(3, np.uint32, self.m)

    @property
    def in_degree(self) -> np.ndarray:
        return self._view(4, np.uint32, self.n)

    @property
    def orig_ids(self):
        return self._view(2, np.uint64, self.n).tolist()

    def out_degree(self, u: int) -> int:
        if not (0 <= u < self.n):
            raise IndexError()
        off = self._arrays()[0].value
        a = C.c_uint64.from_address(off + 8 * u).value
        b = C.c_uint64.from_address(off + 8 * (u + 1)).value
        return b - a

    def pin(self) -> None:
        """Page-lock the CSR arrays (uploads become DMA from pinned memory)."""
        check(lib().dfs_graph_pin(self._h))

    def weights(self, spec: str = "const:0.1", seed: int = 0) -> np.ndarray:
        """apply_weights on the host (runtime.cpp:15-17), fixed point."""
        out = np.zeros(max(self.m, 1), np.uint32)
        check(lib().dfs_graph_weights(self._h, spec.encode(), seed, out.ctypes.data))
        return out[: self.m]

    def __repr__(self):
        return f"<difuser.Graph n={self.n} m={self.m}>"


def _new_graph(fn, *args) -> Graph:
    h = C.c_void_p()
    check(fn(*args, C.byref(h)))
    return Graph(h.value)


def load_graph(path: str, directed: bool = True) -> Graph:
    """Load an edge-list text file or a binary graph cache."""
    return _new_graph(lib().dfs_graph_load, str(path).encode(), int(directed))


def graph_from_text(text: str, directed: bool = True) -> Graph:
    """Build a graph from edge-list text ("u v [p]" lines)."""
    b = text.encode()
    return _new_graph(lib().dfs_graph_from_text, b, len(b), int(directed))


def graph_from_csr(offsets, adj, orig_ids=None) -> Graph:
    offsets = np.ascontiguousarray(offsets, np.uint64)
    adj = np.ascontiguousarray(adj, np.uint32)
    oid = None if orig_ids is None else np.ascontiguousarray(orig_ids, np.uint64)
    return _new_graph(lib().dfs_graph_from_csr, len(offsets) - 1, len(adj), offsets.ctypes.data,
                      adj.ctypes.data if len(adj) else None,
                      None if oid is None else oid.ctypes.data)


def generate(kind: str, a: int, m: int, seed: int = 0) -> Graph:
    """Deterministic synthetic graph: kind "rmat" (a = scale) or "er" (a = n)."""
    return _new_graph(lib().dfs_graph_generate, kind.encode(), a, m, seed)


def save_cache(graph: Graph, path: str) -> None:
    check(lib().dfs_graph_save_cache(graph._h, str(path).encode()))


def edge_hash(u: int, v: int) -> int:
    """31-bit hash of the ordered endpoint pair."""
    return int(lib().dfs_edge_hash(u, v))


def random_value_at(seed: int, r: int) -> int:
    """Per-simulation 31-bit value at index r."""
    return int(lib().dfs_random_value_at(seed, r))


def is_sampled(x: int, h: int, w: float) -> bool:
    """Does the simulation owning value x sample an edge with hash h?"""
    out = C.c_int()
    check(lib().dfs_is_sampled(x, h, float(w), C.byref(out)))
    return bool(out.value)


def _config(k, r, devices, mode, weights, rebuild_eps, seed, sim_cap=256, jacobi=0, count=0):
    return Config(k, r, devices, mode.encode(), weights.encode(), float(rebuild_eps), seed,
                  sim_cap, jacobi, count)


def _serialized(cls):
    """Every public method of a Context holds the context's lock: the library
    is loaded with ctypes.CDLL, which releases the GIL, and a context (its
    arena, partitions, stream, last report) is not re-entrant
    (include/difuser_b200.h).  The reference's run_json is a pure function
    under the GIL, so concurrent callers must not race here either."""
    import functools
    for name, fn in list(vars(cls).items()):
        if name.startswith("_") or not callable(fn):
            continue

        def wrap(f):
            @functools.wraps(f)
            def locked(self, *a, **kw):
                with self._lock:
                    return f(self, *a, **kw)
            return locked
        setattr(cls, name, wrap(fn))
    return cls


@_serialized
class Context:
    """One CUDA device: resident graph, prepared partitions, stage entry points."""

    def __init__(self, device: int = 0):
        self._lock = threading.RLock()
        h = C.c_void_p()
        check(lib().dfs_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device
        self._graph = None

    def __del__(self):
        h = getattr(self, "_h", None)
        capi = globals().get("_capi")  # None while the interpreter tears modules down
        if h is not None and h.value and capi is not None and capi._lib is not None:
            capi._lib.dfs_ctx_destroy(h)
            self._h = None

    # ---- hot path
    def upload(self, graph: Graph):
        check(lib().dfs_upload(self._h, graph._h))
        self._graph = graph

    def _take_json(self, p):
        s = C.cast(p, C.c_char_p).value.decode()
        lib().dfs_free(p)
        return s

    def run_json(self, graph, k=10, r=256, devices=1, mode="fasst", weights="const:0.1",
                 rebuild_eps=0.01, seed=0, timings=True, jacobi=0, resident=False, count=0):
        cfg = _config(k, r, devices, mode, weights, rebuild_eps, seed, jacobi=jacobi,
                      count=count)
        out = C.c_void_p()
        if resident:
            check(lib().dfs_run_resident_json(self._h, graph._h if graph is not None else None,
                                              C.byref(cfg), int(timings), C.byref(out)))
        else:
            check(lib().dfs_run_json(self._h, graph._h, C.byref(cfg), int(timings), C.byref(out)))
        return self._take_json(out)

    @property
    def stream(self) -> int:
        p = C.c_void_p()
        check(lib().dfs_ctx_stream(self._h, C.byref(p)))
        return p.value or 0

    def counters(self, tau: int) -> dict:
        out = np.zeros(8, np.uint64)
        check(lib().dfs_rank_counters(self._h, tau, out.ctypes.data))
        keys = ("updates", "items", "edges", "batches", "touched", "sweeps", "convergences",
                "visited")
        return dict(zip(keys, (int(v) for v in out)))

    def stats(self) -> dict:
        st = Stats()
        check(lib().dfs_last_stats(self._h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in Stats._fields_}

    # ---- stage API (parity harness)
    def prepare(self, graph, k=1, r=256, devices=1, mode="fasst", weights="const:0.1",
                rebuild_eps=0.01, seed=0, jacobi=0):
        self._cfg = dict(k=k, r=r, devices=devices)
        cfg = _config(k, r, devices, mode, weights, rebuild_eps, seed, jacobi=jacobi)
        check(lib().dfs_prepare(self._h, graph._h, C.byref(cfg)))
        self._graph = graph
        self._J = r // devices

    def plan(self):
        r = self._cfg["r"]
        x = np.zeros(r, np.uint32)
        o = np.zeros(r, np.uint32)
        d = C.c_int()
        check(lib().dfs_plan(self._h, x.ctypes.data, o.ctypes.data, C.byref(d)))
        return x, o, bool(d.value)

    def device_graph(self, tau: int):
        m = C.c_uint64()
        w = C.c_uint32()
        check(lib().dfs_device_graph_size(self._h, tau, C.byref(m), C.byref(w)))
        n = self._graph.n
        off = np.zeros(n + 1, np.uint64)
        adj = np.zeros(max(m.value, 1), np.uint32)
        mask = np.zeros(max(m.value * w.value, 1), np.uint64)
        check(lib().dfs_device_graph(self._h, tau, off.ctypes.data, adj.ctypes.data,
                                     mask.ctypes.data))
        return off, adj[: m.value], mask[: m.value * w.value], w.value

    def fill(self, tau: int):
        check(lib().dfs_fill(self._h, tau))

    def simulate(self, tau: int, cap: int = 256, jacobi: int = 0, count: int = 0) -> int:
        s = C.c_int()
        check(lib().dfs_simulate(self._h, tau, cap, jacobi | (count << 1), C.byref(s)))
        return s.value

    def scores(self, tau: int) -> np.ndarray:
        out = np.zeros(max(self._graph.n, 1), np.float64)
        check(lib().dfs_scores(self._h, tau, out.ctypes.data))
        return out[: self._graph.n]

    def commit_cascade(self, tau: int, seed: int) -> int:
        v = C.c_uint64()
        check(lib().dfs_commit_cascade(self._h, tau, seed, C.byref(v)))
        return v.value

    def visited_count(self, tau: int) -> int:
        v = C.c_uint64()
        check(lib().dfs_visited_count(self._h, tau, C.byref(v)))
        return v.value

    def registers(self, tau: int) -> np.ndarray:
        out = np.zeros(max(self._graph.n * self._J, 1), np.int8)
        check(lib().dfs_get_registers(self._h, tau, out.ctypes.data))
        return out[: self._graph.n * self._J]

    def visited(self, tau: int) -> np.ndarray:
        """VISITED bitset, reference layout: n rows of ceil(J/64) u64 words."""
        words = (self._J + 63) // 64
        out = np.zeros(max(self._graph.n * words, 1), np.uint64)
        check(lib().dfs_get_visited(self._h, tau, out.ctypes.data))
        return out[: self._graph.n * words]

    def set_registers(self, tau: int, regs) -> None:
        regs = np.ascontiguousarray(regs, np.int8)
        check(lib().dfs_set_registers(self._h, tau, regs.ctypes.data))

    # ---- Monte-Carlo influence on the GPU (proj/src/oracle.cpp:30-79)
    def influence(self, graph, seeds, trials=10000, seed=0, runs=1, weights="const:0.1",
                  resident=False, per_trial=False):
        """(mean, std_error) of the reached set of a dense-id seed set, equal
        bit for bit to the reference's influence(); per_trial=True also
        returns the per-trial reached counts (run-major)."""
        s = np.ascontiguousarray(list(seeds), np.uint32)
        mean, se = C.c_double(), C.c_double()
        reached = np.zeros(max(trials * runs, 1), np.uint32)
        check(lib().dfs_mc_influence(self._h, graph._h if graph is not None else None,
                                     int(resident), s.ctypes.data if len(s) else None, len(s),
                                     trials, seed, runs, weights.encode(), C.byref(mean),
                                     C.byref(se), reached.ctypes.data))
        if not resident and graph is not None:
            self._graph = graph
        if per_trial:
            return mean.value, se.value, reached[: trials * runs]
        return mean.value, se.value

    # ---- FASST analytics (proj/src/fasst.cpp:101-168)
    def fasst_stats(self, graph, r=256, devices=1, mode="fasst", weights="const:0.1", seed=0,
                    resident=False) -> dict:
        """duplication_stats + device_edge_loads + fill_rate of the plan of
        (r, devices, mode, seed) under `weights`, on the GPU.  Same fields as
        the reference's DuplicationHistogram / loads / FillRateReport."""
        if not resident:
            self.upload(graph)
        cfg = _config(1, r, devices, mode, weights, 0.01, seed)
        dup = np.zeros(devices + 1, np.uint64)
        loads = np.zeros(devices, np.uint64)
        fill = np.zeros(2, np.uint64)
        check(lib().dfs_fasst_stats(self._h, graph._h if graph is not None else None,
                                    C.byref(cfg), dup.ctypes.data, loads.ctypes.data,
                                    fill.ctypes.data))
        m = int(self._graph.m) if self._graph is not None else graph.m
        counts = [int(x) for x in dup]
        sampled = sum(counts[1:])
        out = {"dup_count": counts, "dup_fraction": [c / m if m else 0.0 for c in counts],
               "loads": [int(x) for x in loads]}
        for lim in (1, 2):  # DuplicationHistogram::sampled_share_within (fasst.cpp:119-126)
            out[f"share_within_{lim}"] = (sum(counts[1:lim + 1]) / sampled) if sampled else 0.0
        if r % 32 == 0:  # FillRateReport (fasst.cpp:140-168)
            lanes, batches = int(fill[0]), int(fill[1])
            out["fill_rate"] = lanes / (32.0 * batches) if batches else 0.0
            out["fill_batches"] = batches
        return out

    # ---- peer (multi-GPU) mode: one FASST partition per GPU, exchange in-kernel
    def prepare_partition(self, graph, rank, world, k=1, r=256, mode="fasst",
                          weights="const:0.1", rebuild_eps=0.01, seed=0, resident=False):
        """Build only partition `rank` of `world` (= devices) on this context."""
        cfg = _config(k, r, world, mode, weights, rebuild_eps, seed)
        check(lib().dfs_prepare_partition(self._h, None if resident else graph._h, C.byref(cfg),
                                          rank, world))
        if graph is not None:
            self._graph = graph
        self._cfg = dict(k=k, r=r, devices=world)
        self._J = r // world

    def peer_export(self) -> bytes:
        buf = C.create_string_buffer(_capi.PEER_HANDLE_BYTES)
        check(lib().dfs_peer_export(self._h, buf))
        return buf.raw

    def peer_open(self, rank: int, world: int, handles) -> None:
        blob = b"".join(handles)
        assert len(blob) == world * _capi.PEER_HANDLE_BYTES
        buf = C.create_string_buffer(blob, len(blob))
        check(lib().dfs_peer_open(self._h, rank, world, buf))

    def run_peer_json(self, graph, k=10, r=256, devices=2, mode="fasst", weights="const:0.1",
                      rebuild_eps=0.01, seed=0, timings=True, resident=False):
        """This rank's share of a multi-GPU run; every rank returns the same report."""
        cfg = _config(k, r, devices, mode, weights, rebuild_eps, seed)
        out = C.c_void_p()
        check(lib().dfs_peer_run_json(self._h, graph._h if graph is not None else None,
                                      C.byref(cfg), int(timings), int(resident), C.byref(out)))
        return self._take_json(out)


def fasst_stats(graph, r=256, devices=1, mode="fasst", weights="const:0.1", seed=0) -> dict:
    """FASST analytics (duplication histogram, device edge loads, fill rate)."""
    return default_context().fasst_stats(graph, r=r, devices=devices, mode=mode, weights=weights,
                                         seed=seed)


def peer_link(ctxs) -> None:
    """Link same-process contexts (partition i on ctxs[i]) for peer-mode runs."""
    arr = (C.c_void_p * len(ctxs))(*[c._h.value for c in ctxs])
    check(lib().dfs_peer_link(arr, len(ctxs)))


_ctx_lock = threading.Lock()
_default = {}


def default_context(device: int = 0) -> Context:
    with _ctx_lock:
        if device not in _default:
            _default[device] = Context(device)
        return _default[device]


def run_json(graph, k=10, r=256, devices=1, mode="fasst", weights="const:0.1", rebuild_eps=0.01,
             seed=0, timings=True):
    """Select seeds; returns the report as a JSON string (pymodule.cpp:75-90)."""
    return default_context().run_json(graph, k=k, r=r, devices=devices, mode=mode,
                                      weights=weights, rebuild_eps=rebuild_eps, seed=seed,
                                      timings=timings)


def run(graph, **kwargs):
    """Select seeds and return the report as a dict (see run_json)."""
    return _json.loads(run_json(graph, **kwargs))


def influence(graph, seeds, trials=10000, seed=0, runs=1, weights="const:0.1"):
    """Monte Carlo influence of a dense-id seed set: (mean, std_error)."""
    s = np.ascontiguousarray(list(seeds), np.uint32)
    mean, se = C.c_double(), C.c_double()
    check(lib().dfs_influence(graph._h, s.ctypes.data if len(s) else None, len(s), trials, seed,
                              runs, weights.encode(), C.byref(mean), C.byref(se)))
    return mean.value, se.value


def greedy_exact(graph, k, trials=1000, seed=0, weights="const:0.1"):
    """Reference greedy selection (dense ids)."""
    out = np.zeros(max(k, 1), np.uint32)
    check(lib().dfs_greedy_exact(graph._h, k, trials, seed, weights.encode(), out.ctypes.data))
    return out[:k].tolist()
