"""GPU tests of the distributed path's plumbing (Sec. 3, Alg. 3-6).

* real per-rank processes: world size 2 and 3 on ONE B200 (each process its own
  CUDA context), serinv_ppobtaf_q -> gloo all-gather of host-staged records ->
  serinv_ppobtasi_q, compared with the oracle.  NCCL cannot put two ranks of one
  communicator on the same GPU, so the multi-rank NCCL path itself runs only on
  a multi-GPU box (bench.py --gpus N);
* the library's communicator (serinv_comm_t) at P = 1: with a real NCCL
  unique id (ncclCommInitRank + ncclAllGather of one rank) and without NCCL;
* the status of a non-SPD matrix: the same global row on every rank, NaN log det;
* the paper's exact partition scheme (SERINV_OPT=twist_last=0, 2P-1 reduced blocks);
* one handle used from two streams without host synchronisation;
* compute-sanitizer memcheck / racecheck / synccheck on small launches.
"""
import ctypes
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import btagen
from oracle import invariants as inv, parallel as par, sequential as seq
from tests.gpu_util import args, to_dev, to_host

pytestmark = pytest.mark.gpu
TOL = 1e-10
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sb():
    import paper_2503_17528_b200 as sb
    return sb


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_worker(rank, world, port, n, b, a, Q, out_q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import btagen as bg
    import paper_2503_17528_b200 as sb
    from paper_2503_17528_b200 import distributed as sd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    A = bg.g2(31, n, b, a)
    s, e = sb.plan_ends(n, world, 1.0)[rank]
    loc = sd.local_blocks(A, s, e, last=(rank == world - 1))
    D = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in loc.items()}
    ctx = sd.DistContext(sb.default_handle(0), world, rank, n, s, e - s, b, a, device=0, Q=Q)
    sd.ppobtaf(ctx, D)
    send_h = ctx.send.cpu()                       # host-staged records, gloo all-gather
    recv_h = torch.empty(world * send_h.numel(), dtype=torch.float64)
    sd.exchange(send_h, recv_h)
    ctx.recv.copy_(recv_h)
    sd.ppobtasi(ctx, D)
    torch.cuda.synchronize()
    out_q.put((rank, s, e, {k: v.cpu().numpy() for k, v in D.items()}, int(ctx.info.item()),
               float(ctx.logdet.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,b,a,Q", [(2, 40, 64, 4, 1), (3, 45, 70, 3, 1), (3, 90, 64, 2, 4)])
def test_real_rank_processes_on_one_gpu(world, n, b, a, Q):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, n, b, a, Q, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    A = btagen.g2(31, n, b, a)
    L, X, ld = seq.selinv(A)
    lds = set()
    for rank, s, e, D, info, ldr in res:
        assert info == 0
        lds.add(ldr)
        for i in range(s, e):
            assert inv.rel_err(D["diag"][i - s], X["diag"][i]) <= TOL
            if a:
                assert inv.rel_err(D["arrow"][i - s], X["arrow"][i]) <= TOL
            if i < n - 1:
                assert inv.rel_err(D["lower"][i - s], X["lower"][i]) <= TOL
        if a:
            assert inv.rel_err(D["tip"], X["tip"]) <= TOL
        assert abs(ldr - ld) <= 1e-12 * abs(ld)
    assert len(lds) == 1


@pytest.mark.parametrize("use_nccl", [True, False])
@pytest.mark.parametrize("Q", [1, 3])
def test_comm_entry_points_single_rank(use_nccl, Q):
    # serinv_ppobtaf (factor + pack + the library's all-gather) / serinv_ppobtasi through
    # a serinv_comm_t of one rank: NCCL (real unique id) or none (device copy)
    import torch
    sb = _sb()
    from paper_2503_17528_b200 import _lib
    from paper_2503_17528_b200 import distributed as sd
    L_ = _lib.lib()
    n, b, a = 30, 64, 3
    A = btagen.g1(9, n, b, a)
    Lf, X, ld = seq.selinv(A)
    c = ctypes.c_void_p()
    if use_nccl:
        uid = (ctypes.c_ubyte * 128)()
        assert L_.serinv_nccl_unique_id(uid) == 0
        assert L_.serinv_comm_init(ctypes.byref(c), uid, 1, 0, 0) == 0
    else:
        assert L_.serinv_comm_init(ctypes.byref(c), None, 1, 0, 0) == 0
    comm = sd.Comm.__new__(sd.Comm)
    comm.P, comm.rank, comm.device, comm._c = 1, 0, 0, c
    D = to_dev(A)
    ctx = sd.DistContext(sb.default_handle(), 1, 0, n, 0, n, b, a, Q=Q, comm=comm)
    ldg = sd.pselinv_step(ctx, D)
    e, where = inv.max_block_err(to_host(D), X)
    assert e <= TOL, (e, where)
    assert abs(ldg - ld) <= 1e-12 * abs(ld)
    comm.close()
    del D
    torch.cuda.empty_cache()


def _simulated_ranks(A, P, Q):
    import torch
    sb = _sb()
    from paper_2503_17528_b200 import distributed as sd
    n, b = A["diag"].shape[0], A["diag"].shape[1]
    a = A["tip"].shape[0]
    parts = sb.plan(n, P, 1.0)
    h = sb.default_handle()
    ranks = []
    for p, (s, e) in enumerate(parts):
        loc = sd.local_blocks(A, s, e, last=(p == P - 1))
        D = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in loc.items()}
        ranks.append((s, e, D, sd.DistContext(h, P, p, n, s, e - s, b, a, Q=Q)))
    for s, e, D, ctx in ranks:
        sd.ppobtaf(ctx, D)
    recv = torch.cat([ctx.send for _, _, _, ctx in ranks])
    for s, e, D, ctx in ranks:
        ctx.recv.copy_(recv)
        sd.ppobtasi(ctx, D)
    torch.cuda.synchronize()
    return ranks


@pytest.mark.parametrize("P,Q", [(3, 1), (3, 2), (2, 4)])
@pytest.mark.parametrize("where", ["interior", "boundary", "tip"])
def test_distributed_status_is_global_and_agreed(P, Q, where):
    # after serinv_ppobtasi every rank holds the same info (the genuine
    # failure's global row, dpotrf semantics) and a NaN log det
    n, b, a = 36, 64, 2
    A = btagen.g1(5, n, b, a)
    s1, e1 = par.plan(n, P, 1.0)[1]
    c1 = (e1 - s1) // Q + ((e1 - s1) % Q > 0)
    if where == "interior":
        blk = s1 + 1 if P > 2 else s1 + c1 - 2
        A["diag"][blk][1, 1] = -1e6
        expect = blk * b + 2
    elif where == "boundary":
        blk = s1
        A["diag"][blk][3, 3] = -1e6
        expect = blk * b + 4
    else:
        A["tip"][1, 1] = -1e6
        expect = n * b + 2
    ranks = _simulated_ranks(A, P, Q)
    for s, e, D, ctx in ranks:
        assert int(ctx.info.item()) == expect, (s, int(ctx.info.item()), expect)
        assert np.isnan(float(ctx.logdet.item()))


@pytest.mark.parametrize("P", [2, 3, 4])
def test_paper_partition_scheme_twist_last_0(P, monkeypatch):
    # the paper's scheme (2P-1 reduced blocks, every non-top partition PERMUTED_POBTAF)
    # on the GPU: in-process pselinv and simulated ranks; a fresh handle (graphs are
    # cached per handle and option string)
    monkeypatch.setenv("SERINV_OPT", "twist_last=0")
    sb = _sb()
    n, b, a = 23, 64, 3
    A = btagen.g2(17, n, b, a)
    L, X, ld = seq.selinv(A)
    h = sb.Handle(0)
    assert sb.pselinv_plan(n, P, 1.0) == sb.plan(n, P, 1.0)
    D = to_dev(A)
    ldg = sb.pselinv(*args(D), P, handle=h)
    e, where = inv.max_block_err(to_host(D), X)
    assert e <= TOL, (e, where)
    assert abs(ldg - ld) <= 1e-12 * abs(ld)
    ranks = _simulated_ranks(A, P, 1)
    for s, e_, D, ctx in ranks:
        G = {k: v.cpu().numpy() for k, v in D.items()}
        for i in range(s, e_):
            assert inv.rel_err(G["diag"][i - s], X["diag"][i]) <= TOL
        assert abs(float(ctx.logdet.item()) - ld) <= 1e-12 * abs(ld)
    h.close()


def test_one_handle_two_streams_without_sync():
    # serinv_ctx::call_mu + ev_last: calls through one handle run in call order on the
    # device even when enqueued on different streams (the cached graph's counters are
    # reset per call).  Two matrices of the same shape, separate workspaces/scalars.
    import torch
    sb = _sb()
    from paper_2503_17528_b200 import _lib
    n, b, a = 12, 128, 4
    As = [btagen.g1(s, n, b, a) for s in (1, 2)]
    refs = [seq.selinv(A) for A in As]
    h = sb.Handle(0)
    Ds = [to_dev(A) for A in As]
    nb = ctypes.c_size_t(0)
    _lib.lib().serinv_selinv_ws(n, b, a, ctypes.byref(nb))
    ws = [torch.empty(nb.value, dtype=torch.uint8, device="cuda") for _ in Ds]
    infos = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in Ds]
    lds = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in Ds]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for it in range(3):
        for k in range(2):
            with torch.cuda.stream(streams[k]):
                A = sb._bta(*args(Ds[k]))
                rc = _lib.lib().serinv_selinv(h._h, ctypes.byref(A), ws[k].data_ptr(), ws[k].numel(),
                                              infos[k].data_ptr(), lds[k].data_ptr(),
                                              ctypes.c_void_p(streams[k].cuda_stream))
                assert rc == 0
                if it < 2:   # restore the input for the next round, on the same stream
                    for key in Ds[k]:
                        Ds[k][key].copy_(torch.from_numpy(np.ascontiguousarray(As[k][key])).cuda(non_blocking=False))
    torch.cuda.synchronize()
    for k in range(2):
        assert int(infos[k].item()) == 0
        e, where = inv.max_block_err(to_host(Ds[k]), refs[k][1])
        assert e <= TOL, (k, e, where)
    h.close()


_SANITIZE = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch, btagen
import paper_2503_17528_b200 as sb
from paper_2503_17528_b200 import distributed as sd
A = btagen.g2(3, 9, 40, 3)
D = {{k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in A.items() if k in ("diag", "lower", "arrow", "tip")}}
sb.selinv(D["diag"], D["lower"], D["arrow"], D["tip"])
D = {{k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in A.items() if k in ("diag", "lower", "arrow", "tip")}}
sb.pobtaf(D["diag"], D["lower"], D["arrow"], D["tip"]); sb.pobtasi(D["diag"], D["lower"], D["arrow"], D["tip"])
D = {{k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in A.items() if k in ("diag", "lower", "arrow", "tip")}}
sb.pselinv(D["diag"], D["lower"], D["arrow"], D["tip"], [3])
A = btagen.g2(4, 30, 16, 2)
D = {{k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in A.items() if k in ("diag", "lower", "arrow", "tip")}}
sb.pselinv(D["diag"], D["lower"], D["arrow"], D["tip"], [4, 2])
torch.cuda.synchronize()
print("SANITIZE_OK")
"""


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool, tmp_path):
    cs = "/usr/local/cuda/bin/compute-sanitizer"
    if os.environ.get("SERINV_SANITIZER") != "1":
        pytest.skip("opt-in (SERINV_SANITIZER=1): the GPU pool blocks compute-sanitizer runs")
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    script = tmp_path / "san.py"
    script.write_text(_SANITIZE.format(root=ROOT))
    cmd = [cs, "--tool", tool, "--error-exitcode", "86", "--target-processes", "all"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    out = subprocess.run(cmd + [sys.executable, str(script)], capture_output=True, text=True, timeout=900)
    log = out.stdout + out.stderr
    assert out.returncode == 0 and "SANITIZE_OK" in log, log[-4000:]
    assert "ERROR SUMMARY: 0 errors" in log or "RACECHECK SUMMARY: 0 hazards" in log, log[-4000:]
