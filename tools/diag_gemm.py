"""Diagnostic (not collected): time the GPT-J decode-step projection GEMMs
(M tokens, fp16 weights) back to back with CUDA events."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_01869_b200 import _abi
M = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
shapes = {"qkv": (12288, 4096, 0), "o": (4096, 4096, 2), "mlp_in": (16384, 4096, 1), "mlp_out": (4096, 16384, 2),
          "lm": (50400, 4096, 4)}
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for name, (N, K, epi) in shapes.items():
    a = torch.randn(M, K, device="cuda").half()
    w0 = (torch.randn(N, K, device="cuda") * 0.02).half()
    w = torch.empty(((N + 127) // 128 * 128) * K, device="cuda", dtype=torch.float16)
    _abi.check(_abi.lib.isim_debug_tile_weights(w0.data_ptr(), w.data_ptr(), N, K, st))
    out = torch.empty(M, N, device="cuda", dtype=torch.float16)
    outf = torch.zeros(M, N, device="cuda")
    def go():
        _abi.check(_abi.lib.isim_debug_gemm(a.data_ptr(), w.data_ptr(), M, N, K, epi, None, out.data_ptr(), N,
                                            outf.data_ptr(), N, 2, st))
    for _ in range(3): go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): go()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    print(f"{name:8s} M={M} N={N} K={K}: {us:7.1f} us  {N*K*2/us/1e3:7.0f} GB/s")
