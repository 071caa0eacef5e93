"""Profiling harness (not collected) at C3 shapes: the Vicuna-13B block
(d 5120, 40 heads of 128, SwiGLU ffn 13824) cut to 4 layers with a small KV
pool so `ncu --set full` replays stay fast, running what a Discard-heavy C3
iteration runs: recompute chunks of ~2k rows over 3k-token contexts (K2 with
split-KV + CTA-pair GEMMs at M ~ 2k) beside ~17 decode rows (K1).

  it 1..R  : request r recomputes [0, 2048) (RECOMPUTE rows, one request per iteration)
  it R+1.. : request r recomputes [2048, 3000) over its 2048-token prefix, with decode rows
Usage: python tools/prof_harness_c3.py [R=4] [DEC=17]
"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import paper_2402_01869_b200 as ib  # noqa: E402

GROW, RECOMPUTE_OP = 0, 4
DECODE, FRESH, RECOMP = 0, 1, 2
R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
DEC = int(sys.argv[2]) if len(sys.argv) > 2 else 17
CTX, FIRST, DCTX = 3000, 2048, 2500
blocks = (R + DEC) * (CTX // 16 + 8) + 64
ex = ib.Executor({"preset": "vicuna-13b", "layers": 4}, 0,
                 dict(gpu_blocks=blocks, host_bytes=64 << 20, max_requests=64, max_rows=4096, timing=True))
it = 0


def step(ops, spans):
    global it
    it += 1
    ex.step(ib.Plan.from_json({"it": it, "ops": ops, "spans": spans, "t": 0.0, "B": 0}))


# decode requests with 2.5k-token contexts (prefilled in 2 chunks each, untimed)
dec = list(range(100, 100 + DEC))
for d in dec:
    step([[d, GROW, 0, 0, 2048]], [[d, 0, 2048, FRESH, 0]])
    step([[d, GROW, 0, 2048, DCTX]], [[d, 2048, DCTX - 2048, FRESH, 1]])
ctx = {d: DCTX for d in dec}
ex.sync()
t0 = time.perf_counter()
ex.mark(0)
for r in range(R):
    ops = [[r, GROW, 0, 0, FIRST]] + [[d, GROW, 0, ctx[d], ctx[d] + 1] for d in dec]
    spans = [[r, 0, FIRST, RECOMP, 0]] + [[d, ctx[d], 1, DECODE, 1] for d in dec]
    step(ops, spans)
    for d in dec:
        ctx[d] += 1
for r in range(R):
    ops = [[r, GROW, 0, FIRST, CTX]] + [[d, GROW, 0, ctx[d], ctx[d] + 1] for d in dec]
    spans = [[r, FIRST, CTX - FIRST, RECOMP, 1]] + [[d, ctx[d], 1, DECODE, 1] for d in dec]
    step(ops, spans)
    for d in dec:
        ctx[d] += 1
ex.mark(1)
ex.sync()
ms = ex.elapsed_ms()
print(json.dumps({"layers": 4, "recompute_rows": [FIRST, CTX - FIRST], "decode_rows": DEC,
                  "ms_per_iteration": ms / (2 * R), "ms_per_layer_iteration": ms / (2 * R) / 4}))
