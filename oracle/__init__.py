"""oracle — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).

ctypes view of the plain-C restatement in ``difuser_oracle.c`` plus a numpy
restatement of the reference's graph assembly (``proj/src/graph.cpp:128-183``)
used to turn edge lists into the CSR arrays every side consumes.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this package; the product package
``paper_2410_14047_b200`` never does.

``load_reference()`` returns the UNMODIFIED reference (compiled in place from
/root/reference/proj into ``oracle/_ref`` by ``make -C oracle ref``) when that
build exists, else None.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")

_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_lib = None


def build() -> str:
    """Compile the C restatement (cheap, seconds)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.dor_fmix64.restype = C.c_uint64
        L.dor_fmix64.argtypes = [C.c_uint64]
        L.dor_splitmix64_at.restype = C.c_uint64
        L.dor_splitmix64_at.argtypes = [C.c_uint64, C.c_uint64]
        L.dor_murmur3_pair.restype = None
        L.dor_murmur3_pair.argtypes = [C.c_uint64, C.c_uint64, _u64p]
        L.dor_edge_hash.restype = C.c_uint32
        L.dor_edge_hash.argtypes = [C.c_uint64, C.c_uint64]
        L.dor_register_hash.restype = C.c_uint64
        L.dor_register_hash.argtypes = [C.c_uint64, C.c_uint64]
        L.dor_random_value_at.restype = C.c_uint32
        L.dor_random_value_at.argtypes = [C.c_uint64, C.c_uint32]
        L.dor_to_fixed_point.restype = C.c_uint32
        L.dor_to_fixed_point.argtypes = [C.c_double]
        L.dor_weights_const.restype = None
        L.dor_weights_const.argtypes = [C.c_double, C.c_uint64, _u32p]
        L.dor_weights_wc.restype = None
        L.dor_weights_wc.argtypes = [C.c_uint32, C.c_uint64, _u64p, _u32p, _u32p]
        L.dor_make_plan.restype = C.c_int
        L.dor_make_plan.argtypes = [C.c_uint32, C.c_uint32, C.c_int, C.c_uint64,
                                    _u32p, _u32p, C.POINTER(C.c_int)]
        L.dor_device_graph.restype = C.c_uint64
        L.dor_device_graph.argtypes = [C.c_uint32, _u64p, _u32p, _u32p, _u32p, _u32p,
                                       C.c_uint32, _u64p, _u32p, _u64p]
        L.dor_fill.restype = None
        L.dor_fill.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, _i8p]
        L.dor_row_score.restype = C.c_double
        L.dor_row_score.argtypes = [_i8p, C.c_uint32]
        L.dor_simulate.restype = C.c_int
        L.dor_simulate.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, C.c_uint32, _i8p, C.c_int]
        L.dor_commit_cascade.restype = C.c_uint64
        L.dor_commit_cascade.argtypes = [C.c_uint32, _u64p, _u32p, _u64p, C.c_uint32,
                                         _i8p, _u64p, C.c_uint32]
        L.dor_generate_cache.restype = C.c_int
        L.dor_generate_cache.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_char_p,
                                         C.POINTER(C.c_uint32)]
        L.dor_fasst_stats.restype = None
        L.dor_fasst_stats.argtypes = [C.c_uint64, _u32p, _u32p, _u32p, _u32p, C.c_uint32,
                                      C.c_uint32, _u64p, _u64p, C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64)]
        L.dor_run.restype = C.c_int
        L.dor_run.argtypes = [C.c_uint32, C.c_uint64, _u64p, _u32p, _u32p, C.c_uint32,
                              C.c_uint32, C.c_uint32, C.c_int, C.c_double, C.c_uint64,
                              C.c_int, _u32p, _f64p, _u32p, C.POINTER(C.c_uint32),
                              C.POINTER(C.c_int), C.POINTER(C.c_int), _u64p]
        _lib = L
    return _lib


# ---------------------------------------------------------------- primitives
def fmix64(k):
    return lib().dor_fmix64(k)


def splitmix64_at(s, i):
    return lib().dor_splitmix64_at(s, i)


def murmur3_pair(a, b):
    out = np.zeros(2, np.uint64)
    lib().dor_murmur3_pair(a, b, out)
    return int(out[0]), int(out[1])


def edge_hash(u, v):
    return lib().dor_edge_hash(u, v)


def register_hash(k, v):
    return lib().dor_register_hash(k, v)


def random_value_at(seed, r):
    return lib().dor_random_value_at(seed, r)


def to_fixed_point(w):
    if not (0.0 <= w <= 1.0):
        raise ValueError(f"probability out of [0, 1]: {w}")
    return lib().dor_to_fixed_point(w)


# ---------------------------------------------------------------- graphs
class CSR:
    """Dense CSR graph as the reference builds it (graph.cpp:128-183)."""

    def __init__(self, offsets, adj, orig_ids):
        self.offsets = np.ascontiguousarray(offsets, np.uint64)
        self.adj = np.ascontiguousarray(adj, np.uint32)
        self.orig_ids = np.ascontiguousarray(orig_ids, np.uint64)
        self.n = len(self.offsets) - 1
        self.m = len(self.adj)

    def ehash(self):
        u = np.repeat(np.arange(self.n, dtype=np.uint64), np.diff(self.offsets).astype(np.int64))
        return edge_hash_np(u, self.adj.astype(np.uint64))

    def weights(self, spec: str, seed: int = 0):
        """apply_weights for const:/wc (runtime.cpp:15-17, graph.cpp:247-258)."""
        w = np.zeros(self.m, np.uint32)
        if spec == "wc":
            lib().dor_weights_wc(self.n, self.m, self.offsets, self.adj, w)
        elif spec.startswith("const:"):
            p = float(spec.split(":", 1)[1])
            lib().dor_weights_const(p, self.m, w)
        else:
            raise ValueError("oracle restates const:/wc weights only")
        return w

    def edges_text(self):
        u = np.repeat(self.orig_ids[:self.n], np.diff(self.offsets).astype(np.int64))
        v = self.orig_ids[self.adj]
        return "".join(f"{a} {b}\n" for a, b in zip(u.tolist(), v.tolist()))


def build_csr(us, vs) -> CSR:
    """build_graph restated for unweighted edge lists: dense relabel by sorted
    unique ids (graph.cpp:131-142), (u, v) sort and dedup (:144-160)."""
    us = np.asarray(us, np.uint64)
    vs = np.asarray(vs, np.uint64)
    ids = np.unique(np.concatenate([us, vs]))
    du = np.searchsorted(ids, us).astype(np.uint64)
    dv = np.searchsorted(ids, vs).astype(np.uint64)
    key = np.unique((du << np.uint64(32)) | dv)
    su = (key >> np.uint64(32)).astype(np.int64)
    sv = (key & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    n = len(ids)
    offsets = np.zeros(n + 1, np.uint64)
    np.add.at(offsets, su + 1, 1)
    offsets = np.cumsum(offsets).astype(np.uint64)
    return CSR(offsets, sv, ids)


_M64 = (1 << 64) - 1


def _np_fmix64(k):
    k = k ^ (k >> np.uint64(33))
    k = k * np.uint64(0xff51afd7ed558ccd)
    k = k ^ (k >> np.uint64(33))
    k = k * np.uint64(0xc4ceb9fe1a85ec53)
    return k ^ (k >> np.uint64(33))


def _np_rotl(x, r):
    return (x << np.uint64(r)) | (x >> np.uint64(64 - r))


def edge_hash_np(u, v):
    """Vectorised murmur3_pair(u, v).lo & (2^31-1) (hash.hpp:50-93)."""
    with np.errstate(over="ignore"):
        c1 = np.uint64(0x87c37b91114253d5)
        c2 = np.uint64(0x4cf5ad432745937f)
        k1 = _np_rotl(u * c1, 31) * c2
        h1 = _np_rotl(k1, 27)
        h1 = h1 * np.uint64(5) + np.uint64(0x52dce729)
        k2 = _np_rotl(v * c2, 33) * c1
        h2 = _np_rotl(k2, 31) + h1
        h2 = h2 * np.uint64(5) + np.uint64(0x38495ab5)
        h1 = h1 ^ np.uint64(16)
        h2 = h2 ^ np.uint64(16)
        h1 = h1 + h2
        h2 = h2 + h1
        h1 = _np_fmix64(h1)
        h2 = _np_fmix64(h2)
        h1 = h1 + h2
    return (h1 & np.uint64(0x7FFFFFFF)).astype(np.uint32)


def generate_cache(kind, a, m, seed, path):
    """Write the deterministic R-MAT ("rmat", a = scale) / ER ("er", a = n)
    graph as a DFSG0001 cache the reference's load_graph reads (synth.c);
    returns n.  Same graph as the product's generate(kind, a, m, seed)."""
    n = C.c_uint32(0)
    rc = lib().dor_generate_cache({"rmat": 0, "er": 1}[kind], a, m, seed, path.encode(),
                                  C.byref(n))
    if rc:
        raise RuntimeError(f"generate_cache failed ({rc})")
    return n.value


def er_edges(n, m, seed):
    """Small deterministic directed ER edge list (no self loops); test input only."""
    rng = np.random.default_rng(seed)
    u = rng.integers(0, n, size=m * 2, dtype=np.uint64)
    v = rng.integers(0, n, size=m * 2, dtype=np.uint64)
    keep = u != v
    return u[keep][:m], v[keep][:m]


# ---------------------------------------------------------------- engine
def make_plan(r, mu, mode, seed):
    x = np.zeros(r, np.uint32)
    order = np.zeros(r, np.uint32)
    deg = C.c_int(0)
    if lib().dor_make_plan(r, mu, 1 if mode == "fasst" else 0, seed, x, order, C.byref(deg)) != 0:
        raise ValueError("make_plan: mu must divide R")
    return x, order, bool(deg.value)


def fasst_stats(g: CSR, r, mu, mode, weights, seed):
    """duplication_stats / device_edge_loads / fill_rate (fasst.cpp:101-168),
    returned in the layout of oracle/refprobe.cpp's fasst_stats."""
    xs, order, _ = make_plan(r, mu, mode, seed)
    # fill_rate sorts X itself for FASST and keeps generation order otherwise
    xfill = np.sort(xs, kind="stable") if mode == "fasst" else xs
    w = np.ascontiguousarray(g.weights(weights, seed), np.uint32)
    dup = np.zeros(mu + 1, np.uint64)
    loads = np.zeros(mu, np.uint64)
    lanes, batches = C.c_uint64(), C.c_uint64()
    lib().dor_fasst_stats(g.m, np.ascontiguousarray(g.ehash(), np.uint32), w, xs,
                          np.ascontiguousarray(xfill, np.uint32), r, mu, dup, loads,
                          C.byref(lanes), C.byref(batches))
    out = {"dup_count": [int(x) for x in dup], "dup_fraction": [int(x) / g.m if g.m else 0.0
                                                                 for x in dup],
           "loads": [int(x) for x in loads]}
    sampled = sum(out["dup_count"][1:])
    for lim in (1, 2):
        out[f"share_within_{lim}"] = (sum(out["dup_count"][1:lim + 1]) / sampled) if sampled else 0.0
    if r % 32 == 0:
        out["fill_rate"] = lanes.value / (32.0 * batches.value) if batches.value else 0.0
        out["fill_batches"] = batches.value
    return out


def device_graph(g: CSR, w, xs):
    J = len(xs)
    words = (J + 63) // 64
    off = np.zeros(g.n + 1, np.uint64)
    adj = np.zeros(max(g.m, 1), np.uint32)
    mask = np.zeros(max(g.m, 1) * words, np.uint64)
    md = lib().dor_device_graph(g.n, g.offsets, g.adj, g.ehash(), np.ascontiguousarray(w, np.uint32),
                                np.ascontiguousarray(xs, np.uint32), J, off, adj, mask)
    return off, adj[:md].copy(), mask[:md * words].copy()


def fill(n, J, j_offset, key, regs=None):
    if regs is None:
        regs = np.zeros(n * J, np.int8)
    lib().dor_fill(n, J, j_offset, key, regs)
    return regs


def row_score(row):
    row = np.ascontiguousarray(row, np.int8)
    return lib().dor_row_score(row, len(row))


def simulate(n, off, adj, mask, J, regs, cap=256):
    return lib().dor_simulate(n, off, adj if len(adj) else np.zeros(1, np.uint32),
                              mask if len(mask) else np.zeros(1, np.uint64), J, regs, cap)


def commit_cascade(n, off, adj, mask, J, regs, vis, seed):
    return lib().dor_commit_cascade(n, off, adj if len(adj) else np.zeros(1, np.uint32),
                                    mask if len(mask) else np.zeros(1, np.uint64), J, regs, vis, seed)


def run(g: CSR, k=10, r=256, devices=1, mode="fasst", weights="const:0.1", rebuild_eps=0.01,
        seed=0, sim_cap=256):
    """Greedy run restated (runtime.cpp:37-179); returns the report fields."""
    w = g.weights(weights, seed)
    seeds = np.zeros(max(k, 1), np.uint32)
    traj = np.zeros(max(k, 1), np.float64)
    rb = np.zeros(max(k, 1), np.uint32)
    nrb = C.c_uint32(0)
    sat = C.c_int(0)
    deg = C.c_int(0)
    cnt = np.zeros(3, np.uint64)
    rc = lib().dor_run(g.n, g.m, g.offsets, g.adj if g.m else np.zeros(1, np.uint32),
                       w if g.m else np.zeros(1, np.uint32), k, r, devices,
                       1 if mode == "fasst" else 0, rebuild_eps, seed, sim_cap, seeds, traj, rb,
                       C.byref(nrb), C.byref(sat), C.byref(deg), cnt)
    if rc == -1:
        raise ValueError("invalid run configuration")
    if rc == -2:
        raise RuntimeError("simulate did not converge")
    if rc != 0:
        raise MemoryError("oracle out of memory")
    return {
        "seeds_dense": seeds[:k].tolist(),
        "seeds": [int(g.orig_ids[s]) for s in seeds[:k]],
        "score_trajectory": traj[:k].tolist(),
        "rebuilds": int(nrb.value),
        "rebuild_rounds": rb[:nrb.value].tolist(),
        "saturated": bool(sat.value),
        "degraded_plan": bool(deg.value),
        "comms": {"reduced_elements": int(cnt[0]), "broadcast_elements": int(cnt[1]),
                  "barriers": int(cnt[2])},
    }


# ---------------------------------------------------------------- reference
def load_reference():
    """(difuser_ref, _refprobe) from oracle/_ref, or (None, None)."""
    if not os.path.isdir(REF_DIR):
        return None, None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import difuser_ref  # noqa: F401
        import _refprobe  # noqa: F401
    except ImportError:
        return None, None
    return difuser_ref, _refprobe
