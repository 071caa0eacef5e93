"""Diagnostic (not collected): one GEMM shape, a few launches (for ncu)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_01869_b200 import _abi
M, N, K, epi = (int(x) for x in sys.argv[1:5])
a = torch.randn(M, K, device="cuda").half(); w = (torch.randn(N, K, device="cuda") * 0.02).half()
out = torch.empty(M, N, device="cuda", dtype=torch.float16); outf = torch.zeros(M, N, device="cuda")
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(4):
    _abi.check(_abi.lib.isim_debug_gemm(a.data_ptr(), w.data_ptr(), M, N, K, epi, None, out.data_ptr(), N,
                                        outf.data_ptr(), N, 0, st))
torch.cuda.synchronize()
