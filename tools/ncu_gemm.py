"""One GEMM shape through isim_debug_gemm, for ncu captures (not collected).
Usage: python tools/ncu_gemm.py M N K [epi=0] [flags=0] [reps=3]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2402_01869_b200 import _abi  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
epi = int(sys.argv[4]) if len(sys.argv) > 4 else 0
flags = int(sys.argv[5]) if len(sys.argv) > 5 else 0
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
a = (torch.randn(M, K, device="cuda") * 0.5).half()
w = (torch.randn(N, K, device="cuda") * 0.02).half()
wt = torch.empty(((N + 127) // 128 * 128) * K, dtype=torch.float16, device="cuda")
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
_abi.check(_abi.lib.isim_debug_tile_weights(w.data_ptr(), wt.data_ptr(), N, K, s))
out = torch.empty(M, N // 2 if epi == 3 else N, dtype=torch.float16, device="cuda")
outf = torch.zeros(M, N, device="cuda") if epi in (2, 4) else None
for _ in range(reps):
    _abi.check(_abi.lib.isim_debug_gemm(a.data_ptr(), wt.data_ptr(), M, N, K, epi, None,
                                        out.data_ptr() if outf is None else None, out.shape[1] if outf is None else 0,
                                        outf.data_ptr() if outf is not None else None, N if outf is not None else 0,
                                        2 | flags, s))
torch.cuda.synchronize()
print("ok", M, N, K)
