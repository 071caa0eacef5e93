"""Pair GEMM tile width (256x256 vs 256x128) timed per 13B projection shape.
Usage (GPU box): python tools/gemm_bn_bench.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2402_01869_b200 import _abi  # noqa: E402

STORE, GELU, RESID, SWIGLU, STOREF32 = range(5)
L = _abi.lib


def time_gemm(M, N, K, epi, flags, reps=20):
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    w = (torch.randn(N, K, device="cuda") * 0.02).half()
    wt = torch.empty(((N + 127) // 128 * 128) * K, dtype=torch.float16, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _abi.check(L.isim_debug_tile_weights(w.data_ptr(), wt.data_ptr(), N, K, s))
    out = torch.empty(M, N // 2 if epi == SWIGLU else N, dtype=torch.float16, device="cuda")
    outf = torch.zeros(M, N, device="cuda") if epi in (RESID, STOREF32) else None

    def run():
        _abi.check(L.isim_debug_gemm(a.data_ptr(), wt.data_ptr(), M, N, K, epi, None,
                                     out.data_ptr() if outf is None else None, out.shape[1] if outf is None else 0,
                                     outf.data_ptr() if outf is not None else None, N if outf is not None else 0,
                                     2 | flags, s))
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


MODE = sys.argv[1] if len(sys.argv) > 1 else "bn"
if MODE == "plain":  # one timing per shape at the current settings (env-driven A/B)
    for M in [int(x) for x in sys.argv[2].split(",")]:
        for (N, K, epi, name) in ((15360, 5120, STORE, "qkv13"), (27648, 5120, SWIGLU, "gu13"), (12288, 4096, STORE, "qkv6"),
                                  (16384, 4096, GELU, "fcin6"), (4096, 4096, RESID, "o6"), (4096, 16384, RESID, "fcout6"),
                                  (50400, 4096, STOREF32, "lm6")):
            t = time_gemm(M, N, K, epi, 0)
            print(f"M={M:4d} {name:7s} {t:8.1f} us  {N * K * 2 / t / 1e3:7.0f} GB/s")
    sys.exit(0)
if MODE == "bn":
    for M in (600, 1218, 2048):
        for (N, K, epi, name) in ((15360, 5120, STORE, "qkv"), (5120, 5120, RESID, "o"), (27648, 5120, SWIGLU, "gate_up"),
                                  (5120, 13824, RESID, "down")):
            t256 = time_gemm(M, N, K, epi, 8)
            t128 = time_gemm(M, N, K, epi, 4)
            tf = 2 * M * N * K / 1e12
            print(f"M={M:5d} {name:8s} N={N:6d} K={K:6d}: 256x256 {t256:8.1f} us ({tf / t256 * 1e6:6.0f} TF/s)  "
                  f"256x128 {t128:8.1f} us ({tf / t128 * 1e6:6.0f} TF/s)  best {'128' if t128 < t256 else '256'}")
else:  # stream-K / split tail on (flags 0) vs off (flag 16), 13B and GPT-J projections
    for M in (32, 108, 600, 1218, 2048) if len(sys.argv) < 3 else [int(x) for x in sys.argv[2].split(",")]:
        for (N, K, epi, name) in ((15360, 5120, STORE, "qkv13"), (5120, 5120, RESID, "o13"), (27648, 5120, SWIGLU, "gu13"),
                                  (5120, 13824, RESID, "down13"), (12288, 4096, STORE, "qkv6"), (16384, 4096, GELU, "fcin6"),
                                  (32000, 5120, STOREF32, "lm13")):
            ton = time_gemm(M, N, K, epi, 32)
            toff = time_gemm(M, N, K, epi, 16)
            print(f"M={M:5d} {name:7s} N={N:6d} K={K:6d}: split on {ton:8.1f} us  off {toff:8.1f} us  "
                  f"({100 * (toff - ton) / toff:+5.1f} %)")
