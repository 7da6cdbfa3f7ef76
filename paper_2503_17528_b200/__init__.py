"""serinv-b200: FP64 POBTAF / POBTASI (Serinv, arXiv 2503.17528) on NVIDIA B200.

Thin Python binding over libserinv.so (include/serinv.h): argument marshalling
only -- every step of the factorisation / selected inversion runs in the
library's sm_100a kernels.  Inputs are torch float64 CUDA tensors in the
C-ABI layout (row-major blocks):

    diag  [n, b, b]    A_{i,i}      lower [n-1, b, b]  A_{i+1,i}
    arrow [n, a, b]    A_{n,i}      tip   [a, a]       A_{n,n}

All routines work IN PLACE (like the C-ABI) on the caller's current CUDA
stream.  There is no CPU fallback: importing works without a GPU, but every
compute call requires the CUDA library and a device.
"""
from __future__ import annotations

import ctypes
import threading

from . import _lib
from ._lib import BTA, GraphStats, Part

__all__ = ["Handle", "pobtaf", "pobtasi", "selinv", "selinv_host", "pselinv", "plan", "version",
           "NotPositiveDefinite", "SerinvError", "ppobtaf", "ppobtasi", "exchange_bytes",
           "graph_stats", "default_handle", "auto_partitions", "pselinv_plan", "plan_ends", "Comm",
           "selinv_sb", "sb_auto_plan"]


class SerinvError(RuntimeError):
    def __init__(self, status: int, where: str = ""):
        msg = _lib.lib().serinv_status_string(status).decode()
        super().__init__(f"{where}: serinv status {status} ({msg})")
        self.status = status


class NotPositiveDefinite(ArithmeticError):
    """dpotrf-style failure: `row` is the 1-based global row of the first bad pivot."""

    def __init__(self, row: int, b: int, n: int):
        blk = (row - 1) // b
        where = "the tip" if blk >= n else f"block {blk}"
        super().__init__(f"matrix is not positive definite (first non-positive pivot at global row {row}, {where})")
        self.row = row


def version() -> str:
    return _lib.lib().serinv_version().decode()


def _check(rc: int, where: str):
    if rc != 0:
        raise SerinvError(rc, where)


class Handle:
    """Library handle bound to one CUDA device (caches task graphs per shape)."""

    def __init__(self, device: int | None = None):
        import torch
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self._h = ctypes.c_void_p()
        _check(_lib.lib().serinv_create(ctypes.byref(self._h), self.device), "serinv_create")
        self._ws = {}

    def close(self):
        if self._h:
            _lib.lib().serinv_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def workspace(self, nbytes: int):
        """Device workspace of at least nbytes (cached, grown on demand)."""
        import torch
        ws = self._ws.get("ws")
        if ws is None or ws.numel() < nbytes:
            self._ws["ws"] = ws = torch.empty(max(nbytes, 256), dtype=torch.uint8,
                                              device=f"cuda:{self.device}")
        return ws

    def scalars(self):
        import torch
        s = self._ws.get("scal")
        if s is None:
            s = (torch.zeros(1, dtype=torch.int32, device=f"cuda:{self.device}"),
                 torch.zeros(1, dtype=torch.float64, device=f"cuda:{self.device}"))
            self._ws["scal"] = s
        return s

    def last_launches(self) -> int:
        v = ctypes.c_int(0)
        _lib.lib().serinv_last_launches(self._h, ctypes.byref(v))
        return v.value


_default = threading.local()


def default_handle(device: int | None = None) -> Handle:
    """The calling thread's handle for `device` (one per thread and device: its
    workspace, info and log det buffers are not shared between threads)."""
    import torch
    d = torch.cuda.current_device() if device is None else int(device)
    hs = getattr(_default, "handles", None)
    if hs is None:
        hs = _default.handles = {}
    h = hs.get(d)
    if h is None:
        h = hs[d] = Handle(d)
    return h


def _bta(diag, lower, arrow, tip) -> BTA:
    import torch
    if diag.dtype != torch.float64 or not diag.is_cuda:
        raise TypeError("diag must be a float64 CUDA tensor")
    n, b = diag.shape[0], diag.shape[1]
    a = tip.shape[0] if tip is not None else 0
    for name, t, shp in (("diag", diag, (n, b, b)), ("lower", lower, (n - 1, b, b)),
                         ("arrow", arrow, (n, a, b)), ("tip", tip, (a, a))):
        if t is None:
            if name in ("diag",) or (name == "lower" and n > 1) or (name in ("arrow", "tip") and a > 0):
                raise ValueError(f"{name} is required")
            continue
        if tuple(t.shape) != shp:
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {shp}")
        if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
            raise TypeError(f"{name} must be a contiguous float64 CUDA tensor")
        if t.device != diag.device:
            raise ValueError(f"{name} is on {t.device}, diag on {diag.device}")

    def ptr(t):
        return t.data_ptr() if (t is not None and t.numel() > 0) else None
    return BTA(n, b, a, ptr(diag), ptr(lower), ptr(arrow), ptr(tip))


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _finish(h: Handle, info_t, logdet_t, check: bool, b: int, n: int):
    if not check:
        return None
    info = int(info_t.item())
    if info < 0:
        raise RuntimeError("serinv: internal watchdog fired (a task dependency never completed)")
    if info:
        raise NotPositiveDefinite(info, b, n)
    return float(logdet_t.item()) if logdet_t is not None else None


def _run(kind: str, diag, lower, arrow, tip, handle, check, info=None, logdet=None):
    L = _lib.lib()
    h = handle or default_handle(diag.device.index)
    A = _bta(diag, lower, arrow, tip)
    n, b, a = A.n, A.b, A.a
    wsq = {"pobtaf": L.serinv_pobtaf_ws, "pobtasi": L.serinv_pobtasi_ws, "selinv": L.serinv_selinv_ws}[kind]
    nb = ctypes.c_size_t(0)
    _check(wsq(n, b, a, ctypes.byref(nb)), kind + "_ws")
    ws = h.workspace(nb.value)
    si, sl = h.scalars()
    info = si if info is None else info
    logdet = sl if logdet is None else logdet
    if kind == "pobtasi":
        rc = L.serinv_pobtasi(h._h, ctypes.byref(A), ws.data_ptr(), ws.numel(), info.data_ptr(), _stream())
        _check(rc, kind)
        return _finish(h, info, None, check, b, n)
    fn = L.serinv_pobtaf if kind == "pobtaf" else L.serinv_selinv
    rc = fn(h._h, ctypes.byref(A), ws.data_ptr(), ws.numel(), info.data_ptr(), logdet.data_ptr(), _stream())
    _check(rc, kind)
    return _finish(h, info, logdet, check, b, n)


def pobtaf(diag, lower, arrow, tip, *, handle: Handle | None = None, check: bool = True, info=None, logdet=None):
    """In-place POBTAF (Alg. 1): A -> L.  Returns log det A (check=True)."""
    return _run("pobtaf", diag, lower, arrow, tip, handle, check, info, logdet)


def pobtasi(diag, lower, arrow, tip, *, handle: Handle | None = None, check: bool = True, info=None):
    """In-place POBTASI (Alg. 2): L -> X (selected inverse on the BTA pattern)."""
    return _run("pobtasi", diag, lower, arrow, tip, handle, check, info, None)


def selinv(diag, lower, arrow, tip, *, handle: Handle | None = None, check: bool = True, info=None, logdet=None):
    """In-place POBTAF + POBTASI as one task graph: A -> X.  Returns log det A."""
    return _run("selinv", diag, lower, arrow, tip, handle, check, info, logdet)


def _bta_host(T, n, b, a):
    import torch
    for k in ("diag", "lower", "arrow", "tip"):
        t = T.get(k)
        if t is None:
            continue
        if not isinstance(t, torch.Tensor) or t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
            raise TypeError(f"host {k} must be a contiguous float64 CPU tensor (pinned for overlap)")

    def ptr(t):
        return t.data_ptr() if (t is not None and t.numel() > 0) else None
    return BTA(n, b, a, ptr(T.get("diag")), ptr(T.get("lower")), ptr(T.get("arrow")), ptr(T.get("tip")))


def selinv_host(A_host, D, X_host=None, *, handle: Handle | None = None, check: bool = True, info=None,
                logdet=None):
    """POBTAF + POBTASI from HOST buffers with streaming IO (serinv_selinv_host): the
    H2D copy of A_host (pinned CPU tensors) into the device work buffers D overlaps
    the factorisation, and X is copied back into X_host (default: A_host) node by
    node while the inversion runs.  Returns log det A (check=True syncs)."""
    L = _lib.lib()
    h = handle or default_handle(D["diag"].device.index)
    Ad = _bta(D["diag"], D.get("lower"), D.get("arrow"), D.get("tip"))
    n, b, a = Ad.n, Ad.b, Ad.a
    Ah = _bta_host(A_host, n, b, a)
    Xh = _bta_host(X_host if X_host is not None else A_host, n, b, a)
    nb = ctypes.c_size_t(0)
    _check(L.serinv_selinv_ws(n, b, a, ctypes.byref(nb)), "selinv_ws")
    ws = h.workspace(nb.value)
    si, sl = h.scalars()
    info = si if info is None else info
    logdet = sl if logdet is None else logdet
    rc = L.serinv_selinv_host(h._h, ctypes.byref(Ah), ctypes.byref(Xh), ctypes.byref(Ad), ws.data_ptr(), ws.numel(),
                              info.data_ptr(), logdet.data_ptr(), _stream())
    _check(rc, "selinv_host")
    return _finish(h, info, logdet, check, b, n)


def plan(n: int, P: int, r: float = 1.0):
    """The paper's partition plan (reading R6, Fig. 2): [(start, end)] for ranks 0..P-1.
    The partitioned solvers use pselinv_plan (the twisted scheme by default)."""
    starts = (ctypes.c_int64 * (P + 1))()
    _check(_lib.lib().serinv_plan(n, P, float(r), starts), "serinv_plan")
    return [(starts[p], starts[p + 1]) for p in range(P)]


def pselinv_plan(n: int, P: int, r: float = 1.0):
    """The partition plan pselinv / pselinv_nested actually use (serinv_pselinv_plan):
    plan_ends with the twisted last partition (default), plan with
    SERINV_OPT=twist_last=0.  [(start, end)]."""
    starts = (ctypes.c_int64 * (P + 1))()
    _check(_lib.lib().serinv_pselinv_plan(n, P, float(r), starts), "serinv_pselinv_plan")
    return [(starts[p], starts[p + 1]) for p in range(P)]


def plan_ends(n: int, P: int, r: float = 1.0):
    """Twisted-scheme partition plan (reading R14, serinv_plan_ends): the first and
    the last partition get r times a middle partition's blocks.  [(start, end)]."""
    starts = (ctypes.c_int64 * (P + 1))()
    _check(_lib.lib().serinv_plan_ends(n, P, float(r), starts), "serinv_plan_ends")
    return [(starts[p], starts[p + 1]) for p in range(P)]


def auto_partitions(n: int, b: int) -> list[int]:
    """The library's default one-device nesting plan (serinv_auto_partitions)."""
    out = (ctypes.c_int * 8)()
    k = _lib.lib().serinv_auto_partitions(n, b, out, 8)
    if k < 1:
        raise SerinvError(k, "auto_partitions")
    return list(out[:k])


def pselinv(diag, lower, arrow, tip, P, r: float = 1.0, *, handle: Handle | None = None,
            check: bool = True, info=None, logdet=None):
    """In-process partitioned selected inversion on one device (PPOBTAF -> POBTARSSI ->
    PPOBTASI, Sec. 3) with P partitions.  P may be a sequence [P0, P1, ...]:
    nested solving (Sec. 4.2), the reduced system of level k solved with P_{k+1}
    partitions.  A -> X in place.  Returns log det."""
    L = _lib.lib()
    h = handle or default_handle(diag.device.index)
    A = _bta(diag, lower, arrow, tip)
    Ps = [int(P)] if isinstance(P, int) else [int(x) for x in P]
    arr = (ctypes.c_int * len(Ps))(*Ps)
    nb = ctypes.c_size_t(0)
    _check(L.serinv_pselinv_nested_ws(A.n, A.b, A.a, len(Ps), arr, float(r), ctypes.byref(nb)), "pselinv_ws")
    ws = h.workspace(nb.value)
    si, sl = h.scalars()
    info = si if info is None else info
    logdet = sl if logdet is None else logdet
    rc = L.serinv_pselinv_nested(h._h, ctypes.byref(A), len(Ps), arr, float(r), ws.data_ptr(), ws.numel(),
                                 info.data_ptr(), logdet.data_ptr(), _stream())
    _check(rc, "pselinv")
    return _finish(h, info, logdet, check, A.b, A.n)


def sb_auto_plan(n: int, b: int, a: int) -> list[int]:
    """The small-block engine's default nesting plan (serinv_sb_auto_plan)."""
    out = (ctypes.c_int * 32)()
    k = _lib.lib().serinv_sb_auto_plan(n, b, a, out, 32)
    if k < 0:
        raise SerinvError(-k, "sb_auto_plan")
    return list(out[:k])


def selinv_sb(diag, lower, arrow, tip, Ps=None, *, handle: Handle | None = None, check: bool = True, info=None,
              logdet=None):
    """POBTAF + POBTASI by the small-block engine (b <= 64, a <= 16; serinv_sb_selinv):
    the partitioned method with nested solving, Ps = partitions per level (None: the
    library's plan; [] = one chain).  A -> X in place.  Returns log det."""
    L = _lib.lib()
    h = handle or default_handle(diag.device.index)
    A = _bta(diag, lower, arrow, tip)
    nlev = -1 if Ps is None else len(Ps)
    arr = (ctypes.c_int * max(1, nlev))(*([] if Ps is None else [int(x) for x in Ps]))
    nb = ctypes.c_size_t(0)
    _check(L.serinv_sb_ws(A.n, A.b, A.a, nlev, arr, ctypes.byref(nb)), "sb_ws")
    ws = h.workspace(nb.value)
    si, sl = h.scalars()
    info = si if info is None else info
    logdet = sl if logdet is None else logdet
    rc = L.serinv_sb_selinv(h._h, ctypes.byref(A), nlev, arr, ws.data_ptr(), ws.numel(), info.data_ptr(),
                            logdet.data_ptr(), _stream())
    _check(rc, "sb_selinv")
    return _finish(h, info, logdet, check, A.b, A.n)


def exchange_bytes(b: int, a: int) -> int:
    nb = ctypes.c_size_t(0)
    _check(_lib.lib().serinv_exchange_bytes(b, a, ctypes.byref(nb)), "exchange_bytes")
    return nb.value


def graph_stats(kind: int, n: int, b: int, a: int, P=1, r: float = 1.0, handle: Handle | None = None):
    h = handle or default_handle()
    st = GraphStats()
    if kind == 3 and not isinstance(P, int):
        Ps = [int(x) for x in P]
        arr = (ctypes.c_int * len(Ps))(*Ps)
        _check(_lib.lib().serinv_graph_stats_nested(h._h, n, b, a, len(Ps), arr, float(r), ctypes.byref(st)),
               "graph_stats")
    else:
        _check(_lib.lib().serinv_graph_stats(h._h, kind, n, b, a, P, float(r), ctypes.byref(st)), "graph_stats")
    return dict(tasks=st.tasks, counters=st.counters, flops=st.flops, grid=st.grid, tile=st.tile)


from .distributed import Comm, ppobtaf, ppobtasi  # noqa: E402,F401
from . import distributed  # noqa: E402,F401
