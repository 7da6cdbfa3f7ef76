"""The C-ABI library loads without a GPU and exports every symbol include/*.h declares."""
import ctypes
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(serinv_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    from paper_2503_17528_b200.build import build
    lib = ctypes.CDLL(build(verbose=False))
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def test_host_only_entry_points():
    import paper_2503_17528_b200 as sb
    from paper_2503_17528_b200 import _lib
    L = _lib.lib()
    assert L.serinv_version().decode().startswith("serinv-b200")
    assert sb.plan(11, 3, 1.0) == [(0, 3), (3, 7), (7, 11)]   # Fig. 2
    n = ctypes.c_size_t(0)
    assert L.serinv_selinv_ws(128, 1024, 64, ctypes.byref(n)) == 0 and n.value > 0
    assert L.serinv_exchange_bytes(16, 4, ctypes.byref(n)) == 0 and n.value >= 8 * (4 * 256 + 2 * 64 + 16 + 1)
    starts = (ctypes.c_int64 * 4)()
    assert L.serinv_plan(4, 3, 1.0, starts) == 1007  # SERINV_ERR_PLAN: n < 2P-1
    assert L.serinv_pobtaf(None, None, None, 0, None, None, None) == 1004  # SERINV_ERR_HANDLE
    assert L.serinv_status_string(1002).decode().startswith("workspace")


def test_sb_plan_host_only():
    # small-block engine: plans and workspace queries need no GPU
    import paper_2503_17528_b200 as sb
    from paper_2503_17528_b200 import _lib
    L = _lib.lib()
    nb = ctypes.c_size_t(0)
    for n, b, a in ((16384, 64, 8), (3000, 64, 8), (100, 32, 0), (12, 64, 16), (1, 1, 0)):
        Ps = sb.sb_auto_plan(n, b, a)
        m = n
        for P in Ps:   # every level feasible: ends >= 1 block, middles >= 2 (twisted plan, R14)
            st = sb.plan_ends(m, P)
            assert st[0][0] == 0 and st[-1][1] == m
            assert all(e - s >= (1 if p in (0, P - 1) else 2) for p, (s, e) in enumerate(st))
            m = 2 * P - 2
        assert m <= 12
        arr = (ctypes.c_int * max(1, len(Ps)))(*Ps)
        assert L.serinv_sb_ws(n, b, a, len(Ps), arr, ctypes.byref(nb)) == 0 and nb.value > 0
        assert L.serinv_sb_ws(n, b, a, -1, None, ctypes.byref(nb)) == 0
    assert sb.sb_auto_plan(16384, 64, 8)[0] == 148        # one level-0 partition per SM
    assert L.serinv_sb_ws(10, 65, 4, 0, None, ctypes.byref(nb)) == 1005
    assert L.serinv_sb_ws(10, 64, 17, 0, None, ctypes.byref(nb)) == 1005
    bad = (ctypes.c_int * 1)(9)
    assert L.serinv_sb_ws(10, 64, 4, 1, bad, ctypes.byref(nb)) == 1007
    assert L.serinv_sb_selinv(None, None, 0, None, None, 0, None, None, None) == 1004
