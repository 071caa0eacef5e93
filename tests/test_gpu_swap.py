"""K7 swap path on hand-made plans vs the CPU oracle.

Covers both ways a swap-in gets its bytes back: forwarded from the swap-out
staging slot that still holds them (a short API call: swapped out and back in
two iterations later), and the PCIe round trip through the pinned host pool
(the staging slot was refilled by later swap-outs in between).  Checked: logits
of every sampled row within 1e-3, the swapped KV bytes identical before the
swap-out, on the host, and after the swap-in, device block tables equal the
CPU restatement, and the executor's forwarded-token counter.
"""
import pytest

from conftest import have_gpu
from test_gpu_model import replay

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]

GROW, SWAP_OUT, SWAP_IN, DISCARD, RECOMPUTE, RELEASE = range(6)
DECODE, FRESH, RECOMP = range(3)


def plans(gap_swapouts):
    """Request 0 is swapped out and back in; `gap_swapouts` other requests are
    swapped out (and later back in) in between."""
    P = []

    def it(ops, spans):
        P.append({"it": len(P) + 1, "ops": ops, "spans": spans, "t": 0.0, "B": 0})

    n_req = 2 + gap_swapouts
    it([[r, GROW, 0, 0, 40 + 7 * r] for r in range(n_req)], [[r, 0, 40 + 7 * r, FRESH, 1] for r in range(n_req)])
    ctx = {r: 40 + 7 * r for r in range(n_req)}

    def decode(rs, extra_ops=()):
        ops = [[r, GROW, 0, ctx[r], ctx[r] + 1] for r in rs] + list(extra_ops)
        spans = [[r, ctx[r], 1, DECODE, 1] for r in rs]
        for r in rs:
            ctx[r] += 1
        it(ops, spans)

    decode(range(n_req))
    # request 0 intercepted: its whole context leaves the GPU after this forward
    decode([r for r in range(1, n_req)], [[0, SWAP_OUT, 1, 0, ctx[0]]])
    for g in range(gap_swapouts):  # other requests swap out, refilling the staging slots
        r = 2 + g
        decode([1], [[r, SWAP_OUT, 1, 0, ctx[r]]])
    decode([1])
    # request 0 returns: swap-in before this forward, decoded next iteration
    decode([1], [[0, SWAP_IN, 0, 0, ctx[0]]])
    decode([0, 1])
    for g in range(gap_swapouts):
        r = 2 + g
        decode([0, 1], [[r, SWAP_IN, 0, 0, ctx[r]]])
        decode([0, 1, r])
    decode([0, 1])
    return P


@pytest.mark.parametrize("gap", [0, 3])
def test_swap_round_trip_forwarded_and_pcie(gap):
    pools = dict(gpu_blocks=256, host_bytes=64 << 20, max_requests=16, max_rows=512, record=True, stage_tokens=64,
                 swap_slots=2)
    P = plans(gap)
    r = replay(P, {"preset": "tiny"}, pools, len(P))
    assert r["sampled"] >= 8
    assert r["kv_checked"] > 0
    fwd = r["stats"]["swap_in_forwarded_tokens"]
    if gap == 0:
        assert fwd > 0, "a swap-in right after its swap-out should be served from the staging slot"
    else:
        assert fwd < r["stats"]["swap_in_tokens"], "refilled staging slots must fall back to the PCIe path"
    print(gap, {k: v for k, v in r.items() if k != "stats"}, "forwarded", fwd)
