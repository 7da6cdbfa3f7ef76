"""Tile-engine throughput: independent 64x64xK tile GEMMs through the persistent executor."""
import ctypes, sys
import torch
sys.path.insert(0, "/root/repo")
import paper_2503_17528_b200 as sb
from paper_2503_17528_b200 import _lib

h = sb.default_handle()
L = _lib.lib()
ws = torch.zeros(8 * (2 * 64 * 64 * 2048 * 64 + 64 ** 3 * 64) // 8, dtype=torch.float64, device="cuda")
for k, nseg, nt in [(64, 1, 20000), (256, 1, 20000), (1024, 1, 8000), (1024, 4, 8000), (2048, 1, 4000)]:
    best = 1e9
    for r in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = L.serinv_bench_gemm(h._h, nt, k, nseg, ws.data_ptr(), ws.numel() * 8,
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        e1.record(); torch.cuda.synchronize()
        assert rc == 0, rc
        best = min(best, e0.elapsed_time(e1))
    fl = 2.0 * 64 * 64 * k * nt
    print(f"K={k:5d} nseg={nseg} tasks={nt}: {best:.2f} ms  {fl / best / 1e9:.2f} TFLOP/s  per-task {best*1e3/nt*296:.1f} us/CTA", flush=True)
