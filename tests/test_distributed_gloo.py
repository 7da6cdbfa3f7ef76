"""Multi-process (world_size 2 and 3, gloo, CPU) test of the distributed path's
host logic: partition plan, per-rank graphs, the exchange record layout and the
all-gather (`paper_2503_17528_b200.distributed.exchange`, the same function the
NCCL path uses), reduced-system assembly in rank order and the backward pass.
The per-rank graphs are executed by the host interpreter test tool (no GPU)."""
import ctypes
import os
import socket

import numpy as np
import pytest

P_ = ctypes.c_void_p


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, b, a, out_q, Q=1):
    import sys
    import torch
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import btagen
    from paper_2503_17528_b200 import distributed as sd
    from paper_2503_17528_b200.build import build_daginterp
    from oracle import parallel as par
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = ctypes.CDLL(build_daginterp())
    lib.dag_dist_ws_doubles_q.restype = ctypes.c_int64
    lib.dag_exchange_doubles.restype = ctypes.c_int64
    A = btagen.g2(5, n, b, a)
    parts = par.plan(n, world, 1.0)
    s, e = parts[rank]
    D = sd.local_blocks(A, s, e, last=(rank == world - 1))
    D = {k: np.ascontiguousarray(v) for k, v in D.items()}
    if a == 0:
        D["arrow"] = np.zeros((1, 1, b))
        D["tip"] = np.zeros((1, 1))
    i64 = ctypes.c_int64
    wsd = lib.dag_dist_ws_doubles_q(world, Q, rank, i64(n), i64(s), i64(e - s), i64(b), i64(a))
    rec = lib.dag_exchange_doubles(i64(b), i64(a))
    ws = np.zeros(wsd + 64)
    send = torch.zeros(Q * rec, dtype=torch.float64)         # Q records per rank (sub-partitions)
    recv = torch.zeros(world * Q * rec, dtype=torch.float64)
    info = ctypes.c_int(0)
    ld = ctypes.c_double(0)
    ptrs = [D[k].ctypes.data_as(P_) for k in ("diag", "lower", "arrow", "tip")]
    rc = lib.dag_run_dist_phase_q(0, world, Q, rank, i64(n), i64(s), i64(e - s), i64(b), i64(a), *ptrs,
                                ws.ctypes.data_as(P_), P_(send.data_ptr()), None, None, ctypes.byref(info))
    assert rc == 0 and info.value == 0
    sd.exchange(send, recv)                      # the real all-gather (gloo here, NCCL on GPUs)
    rc = lib.dag_run_dist_phase_q(1, world, Q, rank, i64(n), i64(s), i64(e - s), i64(b), i64(a), *ptrs,
                                ws.ctypes.data_as(P_), None, P_(recv.data_ptr()), ctypes.byref(ld),
                                ctypes.byref(info))
    assert rc == 0 and info.value == 0
    out_q.put((rank, s, e, {k: v for k, v in D.items()}, ld.value))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,b,a,Q", [(2, 9, 5, 2, 1), (3, 11, 4, 0, 1), (3, 13, 66, 3, 1),
                                           (2, 20, 5, 2, 3), (3, 26, 4, 1, 4)])
def test_distributed_gloo(world, n, b, a, Q):
    import multiprocessing as mp
    import btagen
    from oracle import invariants as inv, sequential as seq
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, b, a, q, Q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = btagen.g2(5, n, b, a)
    L, X, ld = seq.selinv(A)
    lds = set()
    for rank, s, e, D, ldr in res:
        lds.add(ldr)
        for i in range(s, e):
            assert inv.rel_err(D["diag"][i - s], X["diag"][i]) < 1e-11
            if a:
                assert inv.rel_err(D["arrow"][i - s], X["arrow"][i]) < 1e-11
            if i < n - 1:
                assert inv.rel_err(D["lower"][i - s], X["lower"][i]) < 1e-11
        if a:
            assert inv.rel_err(D["tip"], X["tip"]) < 1e-11
        assert abs(ldr - ld) <= 1e-12 * abs(ld)
    assert len(lds) == 1   # every rank computes the same log det (redundant reduced solve)
