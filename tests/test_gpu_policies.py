"""f4 pinned on the device: the baseline policies' plan sequences (reference
proj/src/policy.cpp:10-31 named policies; NaiveSwap's synchronous per-block
swaps engine.cpp:226-241, Vanilla / Improved Discard engine.cpp:303-322)
replayed on the tiny model against the CPU oracle: logits <= 1e-3 relative,
block tables + free list bit exact, swapped bytes bit exact.  NaiveSwap runs
with overlap_swaps=false (the executor waits for every swap batch, as the
scheduler's stall charge assumes), the mode tools/policy_sweep.py measures.
"""
import json

import pytest

from conftest import C0_COST, C0_WORKLOAD, have_gpu
from test_gpu_model import pools_for, replay

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]


def _plans(policy, tmp_path):
    import paper_2402_01869_b200 as ib
    path = str(tmp_path / "plans.jsonl")
    ib.run(ib.Trace.generate(C0_WORKLOAD), ib.CostModel.from_json(C0_COST), dict(policy=policy, plan_log=path))
    return [json.loads(l) for l in open(path)]


@pytest.mark.parametrize("policy,overlap", [("swap", False), ("vanilla-discard", True), ("improved-discard", True),
                                            ("preserve", True)])
def test_baseline_policy_replay(tmp_path, policy, overlap):
    import paper_2402_01869_b200 as ib
    plans = _plans(policy, tmp_path)
    n = min(len(plans), 2500)
    kinds = {o[1] for p in plans[:n] for o in p["ops"]}
    if policy == "swap":
        assert ib.KV_SWAP_OUT in kinds and ib.KV_SWAP_IN in kinds and ib.KV_DISCARD not in kinds
    if "discard" in policy:
        assert ib.KV_DISCARD in kinds and ib.KV_RECOMPUTE in kinds and ib.KV_SWAP_OUT not in kinds
    r = replay(plans, {"preset": "tiny"}, pools_for(C0_COST, 2048, overlap_swaps=overlap, max_rows=4096), n,
               check_tables_every=5)
    assert r["sampled"] > 500
    if policy == "swap":
        assert r["kv_checked"] > 0
    print(policy, {k: v for k, v in r.items() if k != "stats"})
