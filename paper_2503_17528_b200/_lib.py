"""ctypes binding of libserinv.so (include/serinv.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libserinv.so")

c_i64 = ctypes.c_int64
c_p = ctypes.c_void_p


class BTA(ctypes.Structure):
    _fields_ = [("n", c_i64), ("b", c_i64), ("a", c_i64),
                ("diag", c_p), ("lower", c_p), ("arrow", c_p), ("tip", c_p)]


class Part(ctypes.Structure):
    _fields_ = [("P", ctypes.c_int), ("rank", ctypes.c_int),
                ("n_global", c_i64), ("start", c_i64), ("count", c_i64)]


class GraphStats(ctypes.Structure):
    _fields_ = [("tasks", c_i64), ("counters", c_i64), ("flops", ctypes.c_double),
                ("grid", ctypes.c_int), ("tile", ctypes.c_int)]


_lib = None


def lib():
    """Load libserinv.so; raises (never falls back) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libserinv.so not found at {LIB_PATH}; build it with "
            "`python -m paper_2503_17528_b200.build` (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    sz = ctypes.POINTER(ctypes.c_size_t)
    L.serinv_version.restype = ctypes.c_char_p
    L.serinv_status_string.restype = ctypes.c_char_p
    L.serinv_status_string.argtypes = [ctypes.c_int]
    L.serinv_create.argtypes = [ctypes.POINTER(c_p), ctypes.c_int]
    L.serinv_destroy.argtypes = [c_p]
    for f in ("serinv_pobtaf_ws", "serinv_pobtasi_ws", "serinv_selinv_ws"):
        getattr(L, f).argtypes = [c_i64, c_i64, c_i64, sz]
    L.serinv_prepare.argtypes = [c_p, ctypes.c_int, c_i64, c_i64, c_i64]
    L.serinv_pobtaf.argtypes = [c_p, ctypes.POINTER(BTA), c_p, ctypes.c_size_t, c_p, c_p, c_p]
    L.serinv_pobtasi.argtypes = [c_p, ctypes.POINTER(BTA), c_p, ctypes.c_size_t, c_p, c_p]
    L.serinv_selinv.argtypes = [c_p, ctypes.POINTER(BTA), c_p, ctypes.c_size_t, c_p, c_p, c_p]
    L.serinv_plan.argtypes = [c_i64, ctypes.c_int, ctypes.c_double, ctypes.POINTER(c_i64)]
    L.serinv_plan_ends.argtypes = [c_i64, ctypes.c_int, ctypes.c_double, ctypes.POINTER(c_i64)]
    L.serinv_pselinv_ws.argtypes = [c_i64, c_i64, c_i64, ctypes.c_int, ctypes.c_double, sz]
    L.serinv_pselinv.argtypes = [c_p, ctypes.POINTER(BTA), ctypes.c_int, ctypes.c_double, c_p,
                                 ctypes.c_size_t, c_p, c_p, c_p]
    ip = ctypes.POINTER(ctypes.c_int)
    L.serinv_auto_partitions.argtypes = [c_i64, c_i64, ip, ctypes.c_int]
    L.serinv_pselinv_nested_ws.argtypes = [c_i64, c_i64, c_i64, ctypes.c_int, ip, ctypes.c_double, sz]
    L.serinv_pselinv_nested.argtypes = [c_p, ctypes.POINTER(BTA), ctypes.c_int, ip, ctypes.c_double, c_p,
                                        ctypes.c_size_t, c_p, c_p, c_p]
    L.serinv_graph_stats_nested.argtypes = [c_p, c_i64, c_i64, c_i64, ctypes.c_int, ip, ctypes.c_double,
                                            ctypes.POINTER(GraphStats)]
    L.serinv_exchange_bytes.argtypes = [c_i64, c_i64, sz]
    L.serinv_ppobtaf_ws.argtypes = [ctypes.POINTER(Part), ctypes.c_int, c_i64, c_i64, sz]
    L.serinv_ppobtaf.argtypes = [c_p, c_p, ctypes.POINTER(Part), ctypes.c_int, ctypes.POINTER(BTA), c_p,
                                 ctypes.c_size_t, c_p, c_p]
    L.serinv_ppobtasi.argtypes = [c_p, c_p, ctypes.POINTER(Part), ctypes.c_int, ctypes.POINTER(BTA), c_p,
                                  ctypes.c_size_t, c_p, c_p, c_p]
    L.serinv_nccl_unique_id.argtypes = [c_p]
    L.serinv_comm_init.argtypes = [ctypes.POINTER(c_p), c_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.serinv_comm_destroy.argtypes = [c_p]
    L.serinv_pselinv_plan.argtypes = [c_i64, ctypes.c_int, ctypes.c_double, ctypes.POINTER(c_i64)]
    L.serinv_ppobtaf_q_ws.argtypes = [ctypes.POINTER(Part), ctypes.c_int, c_i64, c_i64, sz]
    L.serinv_ppobtaf_q.argtypes = [c_p, ctypes.POINTER(Part), ctypes.c_int, ctypes.POINTER(BTA), c_p,
                                   ctypes.c_size_t, c_p, c_p, c_p]
    L.serinv_ppobtasi_q.argtypes = [c_p, ctypes.POINTER(Part), ctypes.c_int, ctypes.POINTER(BTA), c_p,
                                    ctypes.c_size_t, c_p, c_p, c_p, c_p]
    L.serinv_dist_auto_q.argtypes = [c_i64, c_i64]
    L.serinv_graph_stats.argtypes = [c_p, ctypes.c_int, c_i64, c_i64, c_i64, ctypes.c_int,
                                     ctypes.c_double, ctypes.POINTER(GraphStats)]
    L.serinv_selinv_host.argtypes = [c_p, ctypes.POINTER(BTA), ctypes.POINTER(BTA), ctypes.POINTER(BTA), c_p,
                                     ctypes.c_size_t, c_p, c_p, c_p]
    L.serinv_bench_gemm.argtypes = [c_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_p, ctypes.c_size_t, c_p]
    L.serinv_set_trace.argtypes = [c_p, c_p, ctypes.c_size_t]
    L.serinv_last_launches.argtypes = [c_p, ctypes.POINTER(ctypes.c_int)]
    L.serinv_sb_auto_plan.argtypes = [c_i64, c_i64, c_i64, ip, ctypes.c_int]
    L.serinv_sb_ws.argtypes = [c_i64, c_i64, c_i64, ctypes.c_int, ip, sz]
    L.serinv_sb_selinv.argtypes = [c_p, ctypes.POINTER(BTA), ctypes.c_int, ip, c_p, ctypes.c_size_t, c_p, c_p,
                                   c_p]
    _lib = L
    return L


EXPORTED = [
    "serinv_version", "serinv_status_string", "serinv_create", "serinv_destroy",
    "serinv_pobtaf_ws", "serinv_pobtasi_ws", "serinv_selinv_ws", "serinv_prepare",
    "serinv_pobtaf", "serinv_pobtasi", "serinv_selinv", "serinv_plan", "serinv_plan_ends",
    "serinv_pselinv_ws", "serinv_pselinv", "serinv_exchange_bytes", "serinv_ppobtaf_ws",
    "serinv_ppobtaf", "serinv_ppobtasi", "serinv_graph_stats", "serinv_last_launches", "serinv_set_trace", "serinv_selinv_host", "serinv_bench_gemm",
    "serinv_auto_partitions", "serinv_pselinv_nested_ws", "serinv_pselinv_nested", "serinv_graph_stats_nested",
    "serinv_ppobtaf_q_ws", "serinv_ppobtaf_q", "serinv_ppobtasi_q", "serinv_dist_auto_q",
    "serinv_nccl_unique_id", "serinv_comm_init", "serinv_comm_destroy", "serinv_pselinv_plan",
    "serinv_sb_auto_plan", "serinv_sb_ws", "serinv_sb_selinv",
]
