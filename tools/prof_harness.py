"""Profiling harness (not collected): the GPT-J-shaped executor on hand-made
plans that reproduce the C1 window's kernel shapes with a small KV pool, so
`ncu --set full` replays (which save and restore all device memory) stay fast.

  phase 1  prefill: R requests of CTX tokens, P requests per iteration
           (chunk rows -> K2 + CTA-pair GEMMs), chunked like the scheduler;
  phase 2  D decode iterations over all R requests (K1 + split-K GEMMs).

Usage: python tools/prof_harness.py [R=30] [CTX=1100] [D=6] [preset=gptj-6b] [layers]
Prints the algorithmic K1 bytes of one decode layer (for the ncu traffic
comparison) and the device time of the decode iterations.
"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import paper_2402_01869_b200 as ib  # noqa: E402

GROW, DECODE, FRESH = 0, 0, 1
R = int(sys.argv[1]) if len(sys.argv) > 1 else 30
CTX = int(sys.argv[2]) if len(sys.argv) > 2 else 1100
ND = int(sys.argv[3]) if len(sys.argv) > 3 else 6
PRESET = sys.argv[4] if len(sys.argv) > 4 else "gptj-6b"
LAYERS = int(sys.argv[5]) if len(sys.argv) > 5 else {"gptj-6b": 28, "vicuna-13b": 40}[PRESET]
PER = max(1, 3300 // CTX)
D_MODEL = {"gptj-6b": 4096, "vicuna-13b": 5120}[PRESET]

blocks = R * ((CTX + ND + 16) // 16 + 1) + 64
ex = ib.Executor({"preset": PRESET, "layers": LAYERS}, 0,
                 dict(gpu_blocks=blocks, host_bytes=64 << 20, max_requests=max(64, R), max_rows=4096, timing=True))
it = 0


def step(ops, spans):
    global it
    it += 1
    ex.step(ib.Plan.from_json({"it": it, "ops": ops, "spans": spans, "t": 0.0, "B": 0}))


ctx = {}
for r0 in range(0, R, PER):
    rs = range(r0, min(R, r0 + PER))
    step([[r, GROW, 0, 0, CTX] for r in rs], [[r, 0, CTX, FRESH, 1] for r in rs])
    for r in rs:
        ctx[r] = CTX
ex.sync()
k1_bytes = sum(c + 1 for c in ctx.values()) * 2 * D_MODEL * 2 + R * 2 * D_MODEL * 2
t0 = time.perf_counter()
ex.mark(0)
for _ in range(ND):
    step([[r, GROW, 0, ctx[r], ctx[r] + 1] for r in range(R)], [[r, ctx[r], 1, DECODE, 1] for r in range(R)])
    for r in range(R):
        ctx[r] += 1
ex.mark(1)
ex.sync()
ms = ex.elapsed_ms()
st = ex.stats()
print(json.dumps({"preset": PRESET, "layers": LAYERS, "requests": R, "ctx": CTX, "decode_iterations": ND,
                  "decode_ms_per_iteration": ms / ND,
                  "k1_algorithmic_bytes_first_decode_layer": k1_bytes,
                  "k1_gbs_timed_layer": st["k1_bytes"] / (st["k1_ms"] / 1e3) / 1e9 if st["k1_ms"] else None}))
