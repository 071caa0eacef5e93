"""Full-width numeric parity on the real configurations' schedules.

The bench configs' models at their real width -- GPT-J-6B (d 4096, 16 heads
of 256, ffn 16384, vocab 50400) and Vicuna-13B (d 5120, 40 heads of 128,
SwiGLU ffn 13824, vocab 32000) -- cut to 2 layers, replaying what the
scheduler actually emitted for C1 / C2 / C3.  A request's rows
attend only over its own context, so the plan log restricted to a few
requests (their spans and KV ops, every iteration they appear in) is itself a
valid plan sequence: the executor runs exactly the batches those requests saw
in the full schedule -- prompt chunks, decode rows over 1-3k contexts,
swap-outs and swap-ins under the budget, discards and ~2k-row recompute
chunks -- and oracle/forward.py replays the same plans.  Checked as in
test_gpu_model.replay: logits of every sampled row within the stated
relative tolerance (see CASES),
greedy ids equal except flagged near-ties, block tables / free-list size bit
exact, swapped KV bytes bit exact after the round trip.
"""
import json

import numpy as np
import pytest

from conftest import have_gpu
from test_gpu_model import pools_for, replay

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]

# Requests picked from each schedule for what they exercise (scheduler-only
# survey of the plan logs).
#
# Tolerance.  The fp16 rounding points (GEMM inputs, q/k/v, P, attention
# output, KV) set a floor on how closely ANY two fp32-accumulating
# implementations agree: a different summation order moves a value across an
# fp16 rounding boundary.  The floor depends on the block structure: the
# oracle's own float32 variant vs its float64 reference differs by a median
# 2.8e-4 (max 3.8e-4) at the GPT-J shape but 7.6e-4 (max 9.8e-4) at the
# Vicuna-13B shape (tests/test_oracle_floor.py pins the latter).  The device
# meets 1e-3 at the GPT-J shape; at the 13B shape it is held to 1.5e-3 per row
# and 1.1e-3 median -- within 1.5x of the CPU floor.
CASES = {
    # C1: swap-out + swap-in, a discard and a 463-row recompute (662); a
    # 1001-row recompute chunk (707)
    "C1": dict(model={"preset": "gptj-6b", "layers": 2}, rids=[662, 707], rtol=1e-3, median=1e-3),
    # C2: swaps + 914-row recompute (571); 2,531-token context, 2,043-row recompute (992)
    "C2": dict(model={"preset": "vicuna-13b", "layers": 2}, rids=[571, 992], rtol=1.5e-3, median=1.1e-3),
    # C3: ~3k-token context, swaps, 2,031-row recompute chunk (300)
    "C3": dict(model={"preset": "vicuna-13b", "layers": 2}, rids=[300], rtol=1.5e-3, median=1.1e-3),
}


def filtered_plans(name, rids, tmp_path):
    import bench
    import paper_2402_01869_b200 as ib
    cfg = bench.CONFIGS[name]
    path = str(tmp_path / f"{name}.jsonl")
    ib.run(ib.Trace.generate(cfg["workload"]), ib.CostModel.from_json(cfg["cost"]), dict(bench.RUN, plan_log=path))
    keep = set(rids)
    out = []
    with open(path) as f:
        for line in f:
            p = json.loads(line)
            spans = [s for s in p["spans"] if s[0] in keep]
            ops = [o for o in p["ops"] if o[0] in keep]
            if spans or ops:
                out.append(dict(p, spans=spans, ops=ops, B=sum(s[2] for s in spans)))
    return out, cfg


@pytest.mark.parametrize("name", sorted(CASES))
def test_fullwidth_parity_on_config_schedule(tmp_path, name):
    import paper_2402_01869_b200 as ib
    case = CASES[name]
    plans, cfg = filtered_plans(name, case["rids"], tmp_path)
    kinds = {o[1] for p in plans for o in p["ops"]}
    assert {ib.KV_SWAP_OUT, ib.KV_SWAP_IN, ib.KV_RELEASE} <= kinds
    rec = max((s[2] for p in plans for s in p["spans"] if s[3] == ib.SPAN_RECOMPUTE), default=0)
    ctx = max(s[1] + s[2] for p in plans for s in p["spans"])
    preset = case["model"]["preset"]
    d = {"gptj-6b": 4096, "vicuna-13b": 5120}[preset]
    model_m = 2 * 2 * d * 2  # KV bytes per token of the 2-layer model
    pools = pools_for(dict(cfg["cost"], gpu_kv_capacity=8 * 4160 * cfg["M"], cpu_kv_capacity=8 * 4160 * cfg["M"]),
                      model_m, max_requests=16, max_rows=4096)
    errs = []
    r = replay(plans, case["model"], pools, len(plans), check_tables_every=1, errors=errs, rtol=case["rtol"])
    med = float(np.median([e[5] for e in errs]))
    assert med <= case["median"], med
    assert r["sampled"] > 50
    # near-ties flip more often when the rounding floor is higher (13B shape)
    assert r["ties"] <= max(2, int(r["sampled"] * case["rtol"] * 10))
    assert r["kv_checked"] > 0, "no swapped bytes were round-tripped"
    print(name, preset, f"{len(plans)} iterations, max recompute chunk {rec}, max context {ctx}, median err {med:.2e}",
          {k: v for k, v in r.items() if k != "stats"})
