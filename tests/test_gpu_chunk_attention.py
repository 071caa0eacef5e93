"""K2 (tcgen05 chunk attention) on hand-made plans vs the CPU oracle.

The scheduler-driven parity tests mostly see short chunks; these plans pin the
cases the kernel's tiling has to get right: multi-tile prompts (128-row query
tiles, causal diagonal inside a key tile), an API-returned chunk over a long
resident prefix (split-KV items + the combine pass), a ragged recompute chunk
after a discard, and decode rows in the same batch -- for head dims 64, 128
and 256 (tiny GPT, LLaMA and GPT-J block structures).
"""
import pytest

from conftest import have_gpu
from test_gpu_model import replay

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]

GROW, SWAP_OUT, SWAP_IN, DISCARD, RECOMPUTE, RELEASE = range(6)
DECODE, FRESH, RECOMP = range(3)

MODELS = {
    "hd64": {"preset": "tiny", "max_pos": 2304},
    "hd128": {"preset": "vicuna-13b", "layers": 2, "d_model": 1024, "heads": 8, "ffn": 2816, "vocab": 8192,
              "max_pos": 2304},
    "hd256": {"preset": "gptj-6b", "layers": 2, "d_model": 1024, "heads": 4, "ffn": 4096, "vocab": 8192,
              "max_pos": 2304},
}


def plans():
    P = []

    def it(ops, spans):
        P.append({"it": len(P) + 1, "ops": ops, "spans": spans, "t": 0.0, "B": 0})

    # 1: a 1400-token prompt (11 query tiles, the last one ragged) + a short one.
    it([[0, GROW, 0, 0, 1400], [1, GROW, 0, 0, 100]], [[0, 0, 1400, FRESH, 1], [1, 0, 100, FRESH, 1]])
    # 2: decode rows.
    it([[0, GROW, 0, 1400, 1401], [1, GROW, 0, 100, 101]], [[0, 1400, 1, DECODE, 1], [1, 100, 1, DECODE, 1]])
    # 3: 200 API-returned tokens over a 1401-token prefix (split-KV), a decode
    #    row, then request 1 is discarded after the forward.
    it([[0, GROW, 0, 1401, 1601], [1, GROW, 0, 101, 102], [1, DISCARD, 1, 0, 102]],
       [[0, 1401, 200, FRESH, 1], [1, 101, 1, DECODE, 1]])
    # 4: recompute of request 1 (ragged 102 rows) + decode of request 0.
    it([[1, RECOMPUTE, 0, 0, 102], [0, GROW, 0, 1601, 1602]], [[1, 0, 102, RECOMP, 1], [0, 1601, 1, DECODE, 1]])
    # 5: a second long chunk at an unaligned position (keys not a multiple of
    #    the key tile), 37 rows over 1602 keys.
    it([[0, GROW, 0, 1602, 1639], [1, GROW, 0, 102, 103]], [[0, 1602, 37, FRESH, 1], [1, 102, 1, DECODE, 1]])
    # 6: release both.
    it([[0, RELEASE, 1, 0, 0], [1, RELEASE, 1, 0, 0]], [[0, 1639, 1, DECODE, 1], [1, 103, 1, DECODE, 0]])
    return P


@pytest.mark.parametrize("name", sorted(MODELS))
def test_chunk_attention_tiles_and_split_kv(name):
    pools = dict(gpu_blocks=512, host_bytes=64 << 20, max_requests=8, max_rows=2048, record=True, max_ctx=2304)
    r = replay(plans(), MODELS[name], pools, 6, kv_check=False)
    assert r["sampled"] >= 11
    assert r["worst"] <= 1e-3
    print(name, {k: v for k, v in r.items() if k != "stats"})
