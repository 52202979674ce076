"""ctypes binding of the C-ABI in include/difuser_b200.h.

The shared library is built in-tree (``paper_2410_14047_b200/lib``) by
``__graft_entry__.build()``; importing this module without it fails loudly —
there is no CPU fallback for the hot path.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.environ.get("DFS_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                     "libdifuser_b200.so")

# Exported symbols (kept in sync with include/difuser_b200.h; checked by tests).
SYMBOLS = [
    "dfs_last_error", "dfs_version", "dfs_free", "dfs_edge_hash", "dfs_random_value_at",
    "dfs_to_fixed_point", "dfs_is_sampled", "dfs_graph_from_text", "dfs_graph_load",
    "dfs_graph_save_cache", "dfs_graph_from_csr", "dfs_graph_generate", "dfs_graph_free",
    "dfs_graph_n", "dfs_graph_m", "dfs_graph_arrays", "dfs_graph_weights", "dfs_weight_string",
    "dfs_ctx_create", "dfs_ctx_destroy", "dfs_upload", "dfs_run_json", "dfs_run_resident_json",
    "dfs_last_stats", "dfs_prepare", "dfs_plan", "dfs_device_graph_size", "dfs_device_graph",
    "dfs_fill", "dfs_simulate", "dfs_scores", "dfs_commit_cascade", "dfs_visited_count",
    "dfs_get_registers", "dfs_get_visited", "dfs_set_registers", "dfs_influence", "dfs_greedy_exact",
    "dfs_ctx_stream", "dfs_graph_pin", "dfs_rank_counters", "dfs_prepare_partition",
    "dfs_scores_device", "dfs_rebuild", "dfs_format_report", "dfs_peer_export", "dfs_peer_open",
    "dfs_peer_link", "dfs_peer_run_json", "dfs_fasst_stats", "dfs_mc_influence",
]

PEER_HANDLE_BYTES = 216  # DFS_PEER_HANDLE_BYTES


class Config(C.Structure):
    _fields_ = [("k", C.c_uint32), ("r", C.c_uint32), ("devices", C.c_uint32),
                ("mode", C.c_char_p), ("weights", C.c_char_p), ("rebuild_eps", C.c_double),
                ("seed", C.c_uint64), ("sim_cap", C.c_int32), ("jacobi", C.c_int32),
                ("count", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [(f, C.c_double) for f in ("build", "fill", "simulate", "select", "cascade",
                                          "total", "upload")] + \
               [(f, C.c_uint64) for f in ("sketch_edge_updates", "items_processed",
                                          "sweeps_total", "items_fwd", "items_rev", "cnt_edges",
                                          "cnt_batches", "cnt_touched", "cnt_sweeps",
                                          "cnt_convergences", "launches")] + \
               [("sim_active", C.c_double), ("sim_launches", C.c_uint32), ("n", C.c_uint32),
                ("m", C.c_uint64), ("cnt_cas_rows", C.c_uint64), ("cnt_cas_edges", C.c_uint64),
                ("cnt_cascades", C.c_uint64), ("run_kernel", C.c_double),
                ("item_density", C.c_double), ("max_sweeps", C.c_uint32),
                ("rerun_jacobi", C.c_uint32), ("rescored_rows", C.c_uint64)]


class ReportFields(C.Structure):
    _fields_ = [("k", C.c_uint32), ("r", C.c_uint32), ("devices", C.c_uint32),
                ("mode", C.c_char_p), ("weights", C.c_char_p), ("rebuild_eps", C.c_double),
                ("seed", C.c_uint64), ("n", C.c_uint64), ("m", C.c_uint64), ("steps", C.c_uint32),
                ("seeds", C.c_void_p), ("seeds_dense", C.c_void_p), ("traj", C.c_void_p),
                ("rebuilds", C.c_uint32), ("rebuild_rounds", C.c_void_p),
                ("saturated", C.c_int32), ("degraded", C.c_int32),
                ("reduced_elements", C.c_uint64), ("broadcast_elements", C.c_uint64),
                ("barriers", C.c_uint64), ("with_timings", C.c_int32)] + \
               [(f, C.c_double) for f in ("t_build", "t_fill", "t_simulate", "t_select",
                                          "t_cascade", "t_total")]


class DfsError(RuntimeError):
    pass


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    pp = C.POINTER(C.c_void_p)
    sig = {
        "dfs_last_error": (C.c_char_p, []),
        "dfs_version": (i32, []),
        "dfs_free": (None, [vp]),
        "dfs_edge_hash": (u32, [u64, u64]),
        "dfs_random_value_at": (u32, [u64, u32]),
        "dfs_to_fixed_point": (i32, [C.c_double, C.POINTER(u32)]),
        "dfs_is_sampled": (i32, [u32, u32, C.c_double, C.POINTER(i32)]),
        "dfs_graph_from_text": (i32, [C.c_char_p, C.c_size_t, i32, pp]),
        "dfs_graph_load": (i32, [C.c_char_p, i32, pp]),
        "dfs_graph_save_cache": (i32, [vp, C.c_char_p]),
        "dfs_graph_from_csr": (i32, [u32, u64, vp, vp, vp, pp]),
        "dfs_graph_generate": (i32, [C.c_char_p, u32, u64, u64, pp]),
        "dfs_graph_free": (None, [vp]),
        "dfs_graph_n": (u32, [vp]),
        "dfs_graph_m": (u64, [vp]),
        "dfs_graph_arrays": (i32, [vp, pp, pp, pp, pp, pp]),
        "dfs_graph_weights": (i32, [vp, C.c_char_p, u64, vp]),
        "dfs_weight_string": (i32, [C.c_char_p, C.POINTER(C.c_char_p)]),
        "dfs_ctx_create": (i32, [i32, pp]),
        "dfs_ctx_destroy": (None, [vp]),
        "dfs_upload": (i32, [vp, vp]),
        "dfs_run_json": (i32, [vp, vp, C.POINTER(Config), i32, C.POINTER(C.c_void_p)]),
        "dfs_run_resident_json": (i32, [vp, vp, C.POINTER(Config), i32, C.POINTER(C.c_void_p)]),
        "dfs_last_stats": (i32, [vp, C.POINTER(Stats)]),
        "dfs_prepare": (i32, [vp, vp, C.POINTER(Config)]),
        "dfs_plan": (i32, [vp, vp, vp, C.POINTER(i32)]),
        "dfs_device_graph_size": (i32, [vp, u32, C.POINTER(u64), C.POINTER(u32)]),
        "dfs_device_graph": (i32, [vp, u32, vp, vp, vp]),
        "dfs_fill": (i32, [vp, u32]),
        "dfs_simulate": (i32, [vp, u32, i32, i32, C.POINTER(i32)]),
        "dfs_scores": (i32, [vp, u32, vp]),
        "dfs_commit_cascade": (i32, [vp, u32, u32, C.POINTER(u64)]),
        "dfs_visited_count": (i32, [vp, u32, C.POINTER(u64)]),
        "dfs_get_registers": (i32, [vp, u32, vp]),
        "dfs_get_visited": (i32, [vp, u32, vp]),
        "dfs_set_registers": (i32, [vp, u32, vp]),
        "dfs_influence": (i32, [vp, vp, u32, u32, u64, u32, C.c_char_p, C.POINTER(C.c_double),
                                C.POINTER(C.c_double)]),
        "dfs_greedy_exact": (i32, [vp, u32, u32, u64, C.c_char_p, vp]),
        "dfs_ctx_stream": (i32, [vp, pp]),
        "dfs_graph_pin": (i32, [vp]),
        "dfs_rank_counters": (i32, [vp, u32, vp]),
        "dfs_prepare_partition": (i32, [vp, vp, C.POINTER(Config), u32, u32]),
        "dfs_scores_device": (i32, [vp, u32, i32, vp]),
        "dfs_rebuild": (i32, [vp, u32]),
        "dfs_format_report": (i32, [C.POINTER(ReportFields), C.POINTER(C.c_void_p)]),
        "dfs_fasst_stats": (i32, [vp, vp, C.POINTER(Config), vp, vp, vp]),
        "dfs_mc_influence": (i32, [vp, vp, i32, vp, u32, u32, u64, u32, C.c_char_p,
                                   C.POINTER(C.c_double), C.POINTER(C.c_double), vp]),
        "dfs_peer_export": (i32, [vp, vp]),
        "dfs_peer_open": (i32, [vp, u32, u32, vp]),
        "dfs_peer_link": (i32, [C.POINTER(C.c_void_p), u32]),
        "dfs_peer_run_json": (i32, [vp, vp, C.POINTER(Config), i32, i32, C.POINTER(C.c_void_p)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int):
    """Map C-ABI status codes to the reference's exception classes
    (std::invalid_argument -> ValueError, std::runtime_error -> RuntimeError)."""
    if status == 0:
        return
    msg = (lib().dfs_last_error() or b"").decode()
    if status == 1:
        raise ValueError(msg)
    if status == 4:
        raise MemoryError(msg)
    if status == 5:
        raise IndexError(msg)
    raise RuntimeError(msg)
