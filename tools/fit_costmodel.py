"""B200 offline profiler -> fitted CostModel.

Measures the device time of the executor's model step on one B200 as a
function of the batch's query rows B (decode rows at a fixed context, plus a
prefill chunk for the large-B points), writes the profile in the reference's
`batch_tokens,seconds` CSV format (proj/src/cost_model.cpp load_profile_csv)
and fits it with the same piecewise-linear fit the reference uses
(`isim_model_fit_csv`, cost_model.cpp fit_profile), so the scheduler's virtual
clock, saturation point S and swap budget N_i can describe this GPU instead of
the reference defaults.

Usage (on the GPU box):
  python tools/fit_costmodel.py [out_dir=profiles/costmodel] [preset=gptj-6b]
Writes <out_dir>/<preset>_profile.csv and <preset>_fitted.json.
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2402_01869_b200 as ib  # noqa: E402

GROW, DECODE, FRESH = 0, 0, 1
out_dir = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "costmodel")
preset = sys.argv[2] if len(sys.argv) > 2 else "gptj-6b"
CTX, REPS = 512, 3
R = 256 if preset != "vicuna-13b" else 128  # KV pool within ~60 GB
DECODE_B = [b for b in (1, 2, 4, 8, 16, 32, 64, 128, 256) if b <= R]
CHUNK_B = [512, 1024, 2048, 3072, 4000]
os.makedirs(out_dir, exist_ok=True)

extra_tokens = REPS * (len(DECODE_B) + len(CHUNK_B)) + 64
blocks = R * ((CTX + extra_tokens) // 16 + 2) + (4096 // 16 + 2) * 2
ex = ib.Executor({"preset": preset}, 0, dict(gpu_blocks=blocks, host_bytes=64 << 20, max_requests=R + 64,
                                               max_rows=4096))
it = 0
ctx = {}


def step(ops, spans, timed=False):
    global it
    it += 1
    plan = ib.Plan.from_json({"it": it, "ops": ops, "spans": spans, "t": 0.0, "B": 0})
    if not timed:
        ex.step(plan)
        return None
    ex.sync()
    ex.mark(0)
    ex.step(plan)
    ex.mark(1)
    return ex.elapsed_ms() / 1e3


# prefill R requests to CTX tokens (chunks of <= 4096 rows)
per = 4096 // CTX
for r0 in range(0, R, per):
    rs = range(r0, min(R, r0 + per))
    step([[r, GROW, 0, 0, CTX] for r in rs], [[r, 0, CTX, FRESH, 1] for r in rs])
    for r in rs:
        ctx[r] = CTX
step([[0, GROW, 0, ctx[0], ctx[0] + 1]], [[0, ctx[0], 1, DECODE, 1]])  # warm-up
ctx[0] += 1

points = []
for B in DECODE_B:
    ts = []
    for _ in range(REPS):
        rs = range(B)
        ts.append(step([[r, GROW, 0, ctx[r], ctx[r] + 1] for r in rs], [[r, ctx[r], 1, DECODE, 1] for r in rs],
                       timed=True))
        for r in rs:
            ctx[r] += 1
    points.append((B, statistics.median(ts)))
next_id = R
for B in CHUNK_B:
    ts = []
    for _ in range(REPS):
        rs = range(32)
        q = next_id
        next_id += 1
        c = B - 32
        ops = [[r, GROW, 0, ctx[r], ctx[r] + 1] for r in rs] + [[q, GROW, 0, 0, c]]
        spans = [[r, ctx[r], 1, DECODE, 1] for r in rs] + [[q, 0, c, FRESH, 1]]
        ts.append(step(ops, spans, timed=True))
        for r in rs:
            ctx[r] += 1
        step([[q, 5, 1, 0, 0]], [])  # release the chunk's request
    points.append((B, statistics.median(ts)))

csv_path = os.path.join(out_dir, f"{preset}_profile.csv")
with open(csv_path, "w") as f:
    f.write("batch_tokens,seconds\n")
    for b, t in points:
        f.write(f"{b},{t:.9f}\n")
mem = ex.stats()["kv_bytes_per_token"]
fitted = ib.CostModel.fit_csv(csv_path, {"mem_per_token": mem, "swap_per_token": mem / 50e9})
out = fitted.to_json()
json.dump(out, open(os.path.join(out_dir, f"{preset}_fitted.json"), "w"), indent=1)
print(json.dumps({"points": points, "fitted": {k: out[k] for k in ("t0", "slope_below", "slope_above",
                                                                    "saturation_point") if k in out}}))
