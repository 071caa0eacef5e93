"""Plan-level invariant: every token id a row reads was produced before it is read.

A FRESH span writes its synthetic ids into the request's history; a sampling
row at position p writes the greedy id of position p+1; DECODE and RECOMPUTE
rows read the history.  An eviction inside the API-return loop
(reference proj/src/engine.cpp:357-386, evict 179-188) drops the victim's
already-batched FRESH rows from the device batch; their positions must come
back as FRESH (not RECOMPUTE) when the victim is recomputed, or the device
would embed ids that were never written.
"""
import json

from conftest import C0_COST, C0_WORKLOAD

# Preserve policy on a 4,096-token pool: request 0's API-return chunk
# [1258, 1294) is grown and then evicted in iteration 635, and recomputed in
# iteration 701 (found by sweeping seeds / pools).
EVICT_WORKLOAD = dict(C0_WORKLOAD, request_count=16, arrival_rate=4.0, seed=12, max_seq_len=2048)
EVICT_COST = dict(C0_COST, gpu_kv_capacity=4096 * 4096)
EVICT_AT, RECOMPUTE_AT = 635, 701


def unread_positions(plans):
    known, bad = {}, []
    for pj in plans:
        for (rid, pos, count, kind, sample) in pj["spans"]:
            k = known.setdefault(rid, set())
            if kind == 1:
                k.update(range(pos, pos + count))
            else:
                miss = [p for p in range(pos, pos + count) if p not in k]
                if miss:
                    bad.append((pj["it"], rid, kind, miss[:4], len(miss)))
            if sample:
                k.add(pos + count)
        for (rid, kind, phase, lo, hi) in pj["ops"]:
            if kind == 5:
                known.pop(rid, None)
    return bad


def plans_of(workload, cost, cfg, tmp_path):
    import paper_2402_01869_b200 as ib
    path = str(tmp_path / "plans.jsonl")
    ib.run(ib.Trace.generate(workload), ib.CostModel.from_json(cost), dict(cfg, plan_log=path, check_invariants=True))
    return [json.loads(l) for l in open(path)]


def test_c0_history_provenance(c0_plans):
    plans, _ = c0_plans
    assert unread_positions(plans) == []


def test_evicted_fresh_rows_are_reemitted_as_fresh(tmp_path):
    plans = plans_of(EVICT_WORKLOAD, EVICT_COST, dict(policy="preserve"), tmp_path)
    assert unread_positions(plans) == []
    by_it = {p["it"]: p for p in plans}
    # iteration 635: request 0 grows [1258, 1294) and is discarded; no rows run
    assert [o for o in by_it[EVICT_AT]["ops"] if o[0] == 0] == [[0, 0, 0, 1258, 1294], [0, 3, 0, 0, 1294]]
    assert [s for s in by_it[EVICT_AT]["spans"] if s[0] == 0] == []
    # iteration 701: one recompute op, rows split into history ids + synthetic ids
    assert [s for s in by_it[RECOMPUTE_AT]["spans"] if s[0] == 0] == [[0, 0, 1258, 2, 0], [0, 1258, 36, 1, 1]]


def test_dynamic_and_policies_history_provenance(tmp_path):
    for policy, est in [("infercept", "dynamic"), ("vanilla-discard", "oracle"), ("swap", "oracle")]:
        plans = plans_of(dict(C0_WORKLOAD, request_count=24), C0_COST, dict(policy=policy, estimator=est), tmp_path)
        assert unread_positions(plans) == [], (policy, est)


def test_fast_forward_keeps_the_schedule(tmp_path):
    """isim_session_fast_forward runs the same iterations as isim_session_step
    (the sink never influences decisions): identical counters and summary."""
    import paper_2402_01869_b200 as ib
    t = ib.Trace.generate(C0_WORKLOAD)
    m = ib.CostModel.from_json(C0_COST)
    a = ib.Session(t, m, dict(policy="infercept"))
    b = ib.Session(t, m, dict(policy="infercept"))
    for n in (500, 1200, 3000):
        assert a.step(n) == b.fast_forward(n)
        assert a.counters() == b.counters()
    a.step(10 ** 9)
    b.step(10 ** 9)
    assert a.finish().summary() == b.finish().summary()
