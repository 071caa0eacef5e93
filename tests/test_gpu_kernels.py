"""K3 projection GEMM (tcgen05 / TMEM / TMA) vs a plain PyTorch fp32 reference.

Each fused epilogue is checked on ragged shapes (M not a multiple of the 128-row
tile, tiny decode-sized M, K tails handled by TMA zero fill), and the tcgen05
kernel is cross-checked against the CUDA-core SIMT kernel.
"""
import ctypes

import pytest

from conftest import have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]

STORE, GELU, RESID, SWIGLU, STOREF32 = range(5)


def run_gemm(a, w, epi, bias=None, resid=None, force_simt=False, flags=0):
    import torch
    from paper_2402_01869_b200 import _abi
    M, K = a.shape
    N = w.shape[0]
    out = outf = None
    if epi in (STORE, GELU):
        out = torch.empty(M, N, dtype=torch.float16, device="cuda")
    elif epi == SWIGLU:
        out = torch.empty(M, N // 2, dtype=torch.float16, device="cuda")
    elif epi == RESID:
        outf = resid.clone()
    else:
        outf = torch.empty(M, N, dtype=torch.float32, device="cuda")
    st = _abi.lib.isim_debug_gemm(
        a.data_ptr(), w.data_ptr(), M, N, K, epi, bias.data_ptr() if bias is not None else None,
        out.data_ptr() if out is not None else None, out.shape[1] if out is not None else 0,
        outf.data_ptr() if outf is not None else None, outf.shape[1] if outf is not None else 0,
        (1 if force_simt else 0) | flags, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _abi.check(st)
    return out if out is not None else outf


def reference(a, w, epi, bias=None, resid=None):
    import torch
    acc = a.float() @ w.float().t()
    if bias is not None and epi != SWIGLU:
        acc = acc + bias.float()
    if epi == STORE:
        return acc.half()
    if epi == GELU:
        return torch.nn.functional.gelu(acc, approximate="tanh").half()
    if epi == RESID:
        return resid + acc
    if epi == SWIGLU:
        g, u = acc[:, 0::2], acc[:, 1::2]
        return (torch.nn.functional.silu(g) * u).half()
    return acc


# M <= 256 exercises the swap-AB split-K path, larger M the 128-row-tile path;
# N = 50400 (GPT-J vocabulary) and 1000 exercise masked N tails.
SHAPES = [(1, 256, 256), (16, 4096, 4096), (37, 768, 256), (128, 1024, 256), (200, 3072, 1024), (256, 4096, 16384),
          (29, 50400, 4096), (300, 512, 4096), (1000, 12288, 4096), (2048, 256, 1024), (513, 16384, 4096),
          (700, 1000, 512), (61, 1000, 512), (1500, 4096, 16384), (333, 5632, 1024), (200, 4096, 4096), (150, 4096, 16384)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("epi", [STORE, GELU, RESID, SWIGLU, STOREF32])
def test_gemm_epilogues(M, N, K, epi):
    import torch
    torch.manual_seed(M * 7 + N + K + epi)
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    w = (torch.randn(N, K, device="cuda") * 0.02).half()
    bias = (torch.randn(N, device="cuda") * 0.02).half() if epi != SWIGLU else None
    resid = torch.randn(M, N, device="cuda") if epi == RESID else None
    got = run_gemm(a, w, epi, bias, resid).float()
    ref = reference(a, w, epi, bias, resid).float()
    scale = ref.abs().max().item() + 1e-6
    err = (got - ref).abs().max().item() / scale
    tol = 2e-3 if epi in (STORE, GELU, SWIGLU) else 1e-4  # fp16 output rounding vs fp32 outputs
    assert err <= tol, (M, N, K, epi, err)


# Vicuna-13B projections (QKV, O, gate+up SwiGLU, down, LM head) at decode
# (32), decode-heavy (200) and recompute-chunk (2048) batch sizes: the split-K
# planner at 80 / 216 k-blocks and the CTA-pair kernel at both tile widths.
SHAPES_13B = [(M, N, K, epi) for M in (32, 200, 2048)
              for (N, K, epi) in ((15360, 5120, STORE), (5120, 5120, RESID), (27648, 5120, SWIGLU),
                                  (5120, 13824, RESID), (32000, 5120, STOREF32))]


def _check(M, N, K, epi, flags=0):
    import torch
    torch.manual_seed(M * 7 + N + K + epi)
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    w = (torch.randn(N, K, device="cuda") * 0.02).half()
    bias = (torch.randn(N, device="cuda") * 0.02).half() if epi != SWIGLU else None
    resid = torch.randn(M, N, device="cuda") if epi == RESID else None
    got = run_gemm(a, w, epi, bias, resid, flags=flags).float()
    ref = reference(a, w, epi, bias, resid).float()
    scale = ref.abs().max().item() + 1e-6
    err = (got - ref).abs().max().item() / scale
    tol = 2e-3 if epi in (STORE, GELU, SWIGLU) else 1e-4
    assert err <= tol, (M, N, K, epi, flags, err)


@pytest.mark.parametrize("M,N,K,epi", SHAPES_13B)
def test_gemm_13b_shapes(M, N, K, epi):
    _check(M, N, K, epi)


@pytest.mark.parametrize("flags", [4, 8])
@pytest.mark.parametrize("M,N,K,epi", [(1218, 5120, 5120, RESID), (1218, 15360, 5120, STORE),
                                       (513, 27648, 5120, SWIGLU), (300, 1000, 512, GELU), (2048, 32000, 5120, STOREF32)])
def test_pair_gemm_tile_widths(M, N, K, epi, flags):
    _check(M, N, K, epi, flags)


@pytest.mark.parametrize("M,N,K,epi", [(32, 12288, 4096, STORE), (29, 50400, 4096, STOREF32), (45, 16384, 4096, GELU),
                                       (200, 16384, 4096, SWIGLU), (16, 4096, 16384, RESID), (1, 256, 256, STORE),
                                       (250, 4096, 4096, RESID)])
def test_decode_gemm_stream_k(M, N, K, epi):
    """Stream-K (whole-tile decode GEMMs over every SM) against the fp32
    reference, the classic tile split (flag 16) and itself (deterministic)."""
    import torch
    _check(M, N, K, epi, flags=32)
    _check(M, N, K, epi, flags=16)
    torch.manual_seed(1)
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    w = (torch.randn(N, K, device="cuda") * 0.02).half()
    resid = torch.randn(M, N, device="cuda") if epi == RESID else None
    x = run_gemm(a, w, epi, None, resid, flags=32).clone()
    y = run_gemm(a, w, epi, None, resid, flags=32).clone()
    assert torch.equal(x, y), "stream-K result not deterministic"


@pytest.mark.parametrize("M,N,K,epi", [(1218, 5120, 5120, RESID), (300, 1000, 512, GELU), (2065, 15360, 5120, STORE),
                                       (513, 27648, 5120, SWIGLU), (1218, 5120, 13824, RESID), (257, 4096, 4096, STOREF32)])
def test_pair_gemm_stream_k_tail(M, N, K, epi):
    """CTA-pair GEMM with the stream-K tail (tiles not a multiple of the 74
    pairs) against the fp32 reference, without the tail (flag 16), and itself
    (deterministic)."""
    import torch
    _check(M, N, K, epi, flags=32)
    _check(M, N, K, epi, flags=16)
    torch.manual_seed(2)
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    w = (torch.randn(N, K, device="cuda") * 0.02).half()
    resid = torch.randn(M, N, device="cuda") if epi == RESID else None
    x = run_gemm(a, w, epi, None, resid, flags=32).clone()
    y = run_gemm(a, w, epi, None, resid, flags=32).clone()
    assert torch.equal(x, y), "stream-K tail result not deterministic"


@pytest.mark.parametrize("M,N,K", [(77, 1024, 1024), (640, 4096, 4096)])
def test_tcgen05_matches_simt(M, N, K):
    import torch
    torch.manual_seed(3)
    a = (torch.randn(M, K, device="cuda") * 0.5).half()
    w = (torch.randn(N, K, device="cuda") * 0.02).half()
    x = run_gemm(a, w, STOREF32)
    y = run_gemm(a, w, STOREF32, force_simt=True)
    assert (x - y).abs().max().item() <= 1e-4 * (y.abs().max().item() + 1e-6)


def test_gemm_bandwidth_smoke():
    # GPT-J QKV at decode batch: weight-bandwidth bound.  Reported, not gated.
    import torch
    M, N, K = 32, 12288, 4096
    a = (torch.randn(M, K, device="cuda")).half()
    w = (torch.randn(N, K, device="cuda") * 0.02).half()
    for _ in range(3):
        run_gemm(a, w, STORE)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        run_gemm(a, w, STORE)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"QKV GEMM M=32: {ms * 1e3:.1f} us, {N * K * 2 / ms / 1e6:.0f} GB/s weights")
