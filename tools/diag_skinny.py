"""Diagnostic (not collected): decode-sized projection GEMMs with the weights
rotated over 8 copies (800 MB+, beyond L2) so every launch streams from HBM."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_01869_b200 import _abi
M = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = 40
shapes = {"qkv": (12288, 4096, 0), "o": (4096, 4096, 2), "mlp_in": (16384, 4096, 1), "mlp_out": (4096, 16384, 2)}
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for name, (N, K, epi) in shapes.items():
    a = torch.randn(M, K, device="cuda").half()
    w0 = (torch.randn(N, K, device="cuda") * 0.02).half()
    ws = []
    for _ in range(8):
        w = torch.empty(((N + 127) // 128 * 128) * K, device="cuda", dtype=torch.float16)
        _abi.check(_abi.lib.isim_debug_tile_weights(w0.data_ptr(), w.data_ptr(), N, K, st))
        ws.append(w)
    out = torch.empty(M, N, device="cuda", dtype=torch.float16)
    outf = torch.zeros(M, N, device="cuda")
    def go(i):
        _abi.check(_abi.lib.isim_debug_gemm(a.data_ptr(), ws[i % 8].data_ptr(), M, N, K, epi, None, out.data_ptr(), N,
                                            outf.data_ptr(), N, 2, st))
    for i in range(8): go(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps): go(i)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    print(f"{name:8s} M={M} N={N} K={K}: {us:7.1f} us  {N*K*2/us/1e3:7.0f} GB/s", flush=True)
