"""GPU parity on the scheduler paths the C0 replay rarely reaches.

* Eviction inside the API-return loop (reference proj/src/engine.cpp:357-386,
  evict 179-188): the victim's already-batched FRESH rows are dropped from the
  device batch and later recomputed -- as FRESH rows (synthetic ids), since
  their ids never reached the device history (tests/test_plan_history.py).
* The Dynamic estimator (engine.cpp:111-129): paused requests flip from
  Preserve to Discard at the start of an iteration (phase-0 discards), and a
  request's GPU positions may form two runs.
Both replay the scheduler's plans on the tiny model against the CPU oracle
(logits <= 1e-3 relative, block tables + free list bit-exact, swapped bytes
bit-exact).
"""
import json

import pytest

from conftest import C0_COST, C0_WORKLOAD, have_gpu
from test_gpu_model import pools_for, replay
from test_plan_history import EVICT_AT, EVICT_COST, EVICT_WORKLOAD, RECOMPUTE_AT, unread_positions

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]


def _plans(workload, cost, cfg, tmp_path):
    import paper_2402_01869_b200 as ib
    path = str(tmp_path / "plans.jsonl")
    ib.run(ib.Trace.generate(workload), ib.CostModel.from_json(cost), dict(cfg, plan_log=path))
    return [json.loads(l) for l in open(path)]


def test_eviction_in_api_return_loop(tmp_path):
    plans = _plans(EVICT_WORKLOAD, EVICT_COST, dict(policy="preserve"), tmp_path)
    assert unread_positions(plans) == []
    n = RECOMPUTE_AT + 40
    evictions = sum(1 for p in plans[:n] for o in p["ops"] if o[1] == 3)
    r = replay(plans, {"preset": "tiny"}, pools_for(EVICT_COST, 2048, max_rows=4096), n,
               check_tables_every=5)
    assert evictions > 0 and r["sampled"] > 300
    print("eviction replay", evictions, "discards", {k: v for k, v in r.items() if k != "stats"})


def test_dynamic_estimator_flips(tmp_path):
    plans = _plans(C0_WORKLOAD, C0_COST, dict(policy="infercept", estimator="dynamic"), tmp_path)
    flips = [p["it"] for p in plans[:1000] for o in p["ops"] if o[1] == 3 and o[2] == 0]
    assert len(flips) >= 3, flips
    r = replay(plans, {"preset": "tiny"}, pools_for(C0_COST, 2048), 1000, check_tables_every=5)
    assert r["sampled"] > 700 and r["kv_checked"] > 0
    print("dynamic replay flips", flips, {k: v for k, v in r.items() if k != "stats"})
