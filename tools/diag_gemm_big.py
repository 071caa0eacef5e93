"""Diagnostic (not collected): chunk-sized (M = 300..2048) GPT-J projection
GEMMs, weights rotated over 4 copies; TFLOP/s per shape."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_01869_b200 import _abi
shapes = {"qkv": (12288, 4096, 0), "o": (4096, 4096, 2), "mlp_in": (16384, 4096, 1), "mlp_out": (4096, 16384, 2)}
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for M in [int(x) for x in (sys.argv[1:] or ["300", "980", "2048"])]:
    for name, (N, K, epi) in shapes.items():
        a = torch.randn(M, K, device="cuda").half()
        w0 = (torch.randn(N, K, device="cuda") * 0.02).half()
        ws = []
        for _ in range(4):
            w = torch.empty(((N + 127) // 128 * 128) * K, device="cuda", dtype=torch.float16)
            _abi.check(_abi.lib.isim_debug_tile_weights(w0.data_ptr(), w.data_ptr(), N, K, st))
            ws.append(w)
        out = torch.empty(M, N, device="cuda", dtype=torch.float16)
        outf = torch.zeros(M, N, device="cuda")
        def go(i):
            _abi.check(_abi.lib.isim_debug_gemm(a.data_ptr(), ws[i % 4].data_ptr(), M, N, K, epi, None, out.data_ptr(), N,
                                                outf.data_ptr(), N, 2, st))
        for i in range(4): go(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(20): go(i)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        print(f"{name:8s} M={M:5d} N={N} K={K}: {us:8.1f} us  {2*M*N*K/us/1e6:7.0f} TFLOP/s", flush=True)
