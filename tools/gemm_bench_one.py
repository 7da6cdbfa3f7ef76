import ctypes, sys
import torch
sys.path.insert(0, "/root/repo")
import paper_2503_17528_b200 as sb
from paper_2503_17528_b200 import _lib
h = sb.default_handle(); L = _lib.lib()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ws = torch.zeros((2 * 64 * 64 * k * 64 + 64 ** 3 * 64), dtype=torch.float64, device="cuda")
for r in range(2):
    rc = L.serinv_bench_gemm(h._h, 8000, k, 1, ws.data_ptr(), ws.numel() * 8, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("ok", rc)
