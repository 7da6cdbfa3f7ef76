"""Per-task phase times of independent tile GEMMs through the executor (dev tool)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2503_17528_b200 as sb
from paper_2503_17528_b200 import _lib

h = sb.default_handle()
L = _lib.lib()
ws = torch.zeros((2 * 64 * 64 * 2048 * 64 + 64 ** 3 * 64) // 8, dtype=torch.float64, device="cuda")
for k, nt in [(64, 20000), (256, 20000), (1024, 8000)]:
    buf = torch.zeros(12 * nt, dtype=torch.int64, device="cuda")
    L.serinv_set_trace(h._h, buf.data_ptr(), buf.numel() * 8)
    for r in range(2):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        L.serinv_bench_gemm(h._h, nt, k, 1, ws.data_ptr(), ws.numel() * 8, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        e1.record(); torch.cuda.synchronize()
    L.serinv_set_trace(h._h, None, 0)
    tr = buf[:4 * nt].view(nt, 4).cpu().numpy().astype(np.int64)
    ph = buf[4 * nt:].view(nt, 8).cpu().numpy().astype(np.int64)
    claim, start, end = tr[:, 0], tr[:, 1], tr[:, 2]
    m5, m6, m7 = ph[:, 5], ph[:, 6], ph[:, 7]
    d = lambda a, b: np.median(a - b) / 1e3
    print(f"K={k}: launch {e0.elapsed_time(e1):.2f} ms; per task (median us): claim->start {d(start, claim):.2f}, "
          f"mainloop {d(m5, start):.2f}, epilogue(c0) {d(m6, m5):.2f}, store {d(m7, m6):.2f}, publish {d(end, m7):.2f}, "
          f"total {d(end, claim):.2f}; gap to next claim on same CTA n/a", flush=True)
    # gap between a CTA's consecutive tasks: sort by (sm, claim)
    sm = (tr[:, 3] >> 16) & 0xFFFF
    o = np.lexsort((claim, sm))
    g = []
    for i in range(1, len(o)):
        if sm[o[i]] == sm[o[i - 1]] and claim[o[i]] > end[o[i - 1]]:
            g.append(claim[o[i]] - end[o[i - 1]])
    if g:
        print(f"   end -> next claim on the same SM (median) {np.median(g) / 1e3:.2f} us")
