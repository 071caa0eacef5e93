"""The asynchronous (benchmarked) executor path against the synchronous one.

bench.py and session.step run the executor with record=False: plans are
enqueued up to 16 iterations ahead (plan ring), swap-outs are gathered into
recycled staging slots and copied D2H on a copy stream while later
iterations run, swap-ins are forwarded from a staging slot when its bytes are
still there (else H2D into a slot on the second copy stream), and sampled ids
go straight into mapped pinned memory.  Every numeric test uses record=True,
which synchronises all streams after every step.  Here the same plan sequence
runs through both executors side by side; at checkpoints (after sync()) the
device state of every live request must be identical bit for bit:
  * block table and free-list size;
  * token history (synthetic prompt / API-returned ids + sampled ids);
  * the KV bytes of every computed position, wherever they live (paged GPU
    pool or pinned host extent).
Plan sequences: the whole C0 trace (swaps, forwarding, discards, recompute),
an eviction inside the API-return loop (ghost rows, engine.cpp:359-386) and
the Dynamic estimator's Preserve->Discard flips (engine.cpp:111-129).
"""
import json

import numpy as np
import pytest

from conftest import C0_COST, C0_WORKLOAD, have_gpu
from test_gpu_model import pools_for
from test_plan_history import EVICT_COST, EVICT_WORKLOAD

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]


def _plans(workload, cost, cfg, tmp_path):
    import paper_2402_01869_b200 as ib
    path = str(tmp_path / "plans.jsonl")
    ib.run(ib.Trace.generate(workload), ib.CostModel.from_json(cost), dict(cfg, plan_log=path))
    return [json.loads(l) for l in open(path)]


class Positions:
    """Per request: positions whose KV has been computed and not discarded
    (readable on the GPU or the host), from the plans' ops."""

    def __init__(self):
        self.computed = {}

    def apply(self, plan_j):
        import paper_2402_01869_b200 as ib
        for phase in (0, 1):
            for (rid, kind, ph, lo, hi) in plan_j["ops"]:
                if ph != phase:
                    continue
                s = self.computed.setdefault(rid, set())
                if kind in (ib.KV_GROW, ib.KV_RECOMPUTE):
                    s.update(range(lo, hi))
                elif kind == ib.KV_DISCARD:
                    s.difference_update(range(lo, hi))
                elif kind == ib.KV_RELEASE:
                    self.computed.pop(rid, None)

    @staticmethod
    def runs(s):
        out, pos = [], sorted(s)
        i = 0
        while i < len(pos):
            j = i
            while j + 1 < len(pos) and pos[j + 1] == pos[j] + 1:
                j += 1
            out.append((pos[i], pos[j] + 1))
            i = j + 1
        return out


def compare(a, b, pos, L, D):
    assert a.free_blocks() == b.free_blocks()
    for rid, s in pos.computed.items():
        ta, tb = a.block_table(rid), b.block_table(rid)
        assert ta == tb, f"block table of {rid}"
        if not s:
            continue
        hi = max(s) + 2
        assert np.array_equal(a.read_history(rid, 0, hi), b.read_history(rid, 0, hi)), f"history of {rid}"
        for lo, h in Positions.runs(s):
            assert np.array_equal(a.read_kv(rid, lo, h, L, D), b.read_kv(rid, lo, h, L, D)), f"KV of {rid} [{lo},{h})"


def run_both(plans, n, check_every, **async_pools):
    import paper_2402_01869_b200 as ib
    model = {"preset": "tiny"}
    sync_ex = ib.Executor(model, 0, pools_for(C0_COST, 2048, max_rows=4096))
    async_ex = ib.Executor(model, 0, pools_for(C0_COST, 2048, max_rows=4096, record=False, **async_pools))
    pos = Positions()
    checks = 0
    for i, pj in enumerate(plans[:n]):
        p = ib.Plan.from_json(pj)
        sync_ex.step(p)
        async_ex.step(p)
        pos.apply(pj)
        if (i + 1) % check_every == 0 or i + 1 == min(n, len(plans)):
            async_ex.sync()
            compare(sync_ex, async_ex, pos, 2, 256)
            checks += 1
    async_ex.sync()
    return checks, async_ex.stats()


def test_async_path_matches_sync_whole_c0(tmp_path):
    plans = _plans(C0_WORKLOAD, C0_COST, dict(policy="infercept"), tmp_path)
    checks, st = run_both(plans, len(plans), 250, stage_tokens=256, swap_slots=4)
    assert checks >= 70
    assert st["swap_out_tokens"] > 0 and st["swap_in_tokens"] > 0
    assert st["swap_in_forwarded_tokens"] > 0, "no swap-in was forwarded from a staging slot"
    assert st["swap_in_forwarded_tokens"] < st["swap_in_tokens"], "no swap-in crossed the link"
    print("async == sync over", len(plans), "iterations;", checks, "checkpoints;",
          {k: st[k] for k in ("swap_in_tokens", "swap_out_tokens", "swap_in_forwarded_tokens")})


def test_async_path_matches_sync_eviction(tmp_path):
    plans = _plans(EVICT_WORKLOAD, EVICT_COST, dict(policy="preserve"), tmp_path)
    evictions = sum(1 for p in plans for o in p["ops"] if o[1] == 3)
    assert evictions > 0
    run_both(plans, 8000, 100, stage_tokens=256, swap_slots=4)


def test_async_path_matches_sync_dynamic(tmp_path):
    plans = _plans(C0_WORKLOAD, C0_COST, dict(policy="infercept", estimator="dynamic"), tmp_path)
    run_both(plans, 6000, 100, stage_tokens=256, swap_slots=4)
