"""Measured clocks: the scheduler advanced by the B200's
measured step time ("device") or by the wall clock with timed API calls
("wall") instead of the reference's analytic t_fwd.

With a measured clock the executor receives each iteration as two plans (the
phase-0 ops and rows, synchronised and timed, then the post-phase ops), so
these tests also check that the split execution keeps the device state right:
the plan log of a device-clock run replays through the single-plan executor
path against the CPU oracle (logits, block tables, swapped KV bytes).
"""
import json
import time

import pytest

from conftest import C0_COST, have_gpu
from test_gpu_model import pools_for, replay

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]

SHORT_API = dict(classes=[{"name": "Math"}, {"name": "VE"}], request_count=12, arrival_rate=20.0, seed=3,
                 max_seq_len=4096)


def _exec_cfg(record=False):
    return {"model": {"preset": "tiny"}, "pools": pools_for(C0_COST, 2048, record=record)}


def test_device_clock_runs_the_trace_on_measured_step_time(tmp_path):
    import paper_2402_01869_b200 as ib
    t = ib.Trace.generate(SHORT_API)
    m = ib.CostModel.from_json(C0_COST)
    virt = ib.run(t, m, dict(policy="infercept")).summary()
    path = str(tmp_path / "plans.jsonl")
    dev = ib.run(t, m, dict(policy="infercept", executor="b200", exec=_exec_cfg(), clock="device",
                            check_invariants=True, plan_log=path)).summary()
    assert dev["completed"] == dev["requests"] == 12 and dev["incomplete"] == 0
    # The tiny model steps in well under the cost model's 2 ms t0 on a B200.
    per_iter = dev["forwarding_time"] / dev["iterations"]
    assert 5e-6 < per_iter < 2e-3, per_iter
    assert dev["forwarding_time"] < virt["forwarding_time"]
    with open(path) as f:
        plans = [json.loads(l) for l in f]
    assert len(plans) == dev["iterations"]
    # The clock in the plan log is monotone and starts from the first arrival.
    ts = [p["t"] for p in plans]
    assert all(b >= a for a, b in zip(ts, ts[1:]))


def test_device_clock_split_plans_keep_device_state_exact(tmp_path):
    # Session with an external executor in device-clock mode: the executor
    # saw every iteration as forward + post-phase plans.  The plan log replays
    # through a fresh executor (one plan per iteration) under the oracle.
    import paper_2402_01869_b200 as ib
    t = ib.Trace.generate(SHORT_API)
    m = ib.CostModel.from_json(C0_COST)
    pools = pools_for(C0_COST, 2048, record=True)
    ex = ib.Executor({"preset": "tiny"}, 0, pools)
    path = str(tmp_path / "plans.jsonl")
    s = ib.Session(t, m, dict(policy="infercept", clock="device", plan_log=path, check_invariants=True), ex)
    done = False
    while not done:
        _, done = s.step(500)
    res = s.finish().summary()
    ex.sync()
    st = ex.stats()
    assert st["iterations"] == res["iterations"]
    assert ex.free_blocks() == pools["gpu_blocks"]  # every request released every block
    with open(path) as f:
        plans = [json.loads(l) for l in f]
    r = replay(plans, {"preset": "tiny"}, pools, n_iters=400)
    assert r["sampled"] > 0
    print("device-clock replay", {k: v for k, v in r.items() if k != "stats"})


def test_wall_clock_serves_in_real_time():
    import paper_2402_01869_b200 as ib
    t = ib.Trace.generate(SHORT_API)
    m = ib.CostModel.from_json(C0_COST)
    ex = ib.Executor({"preset": "tiny"}, 0, pools_for(C0_COST, 2048, record=False))
    s = ib.Session(t, m, dict(policy="infercept", clock="wall"), ex)
    t0 = time.perf_counter()
    done = False
    while not done:
        _, done = s.step(1000)
    elapsed = time.perf_counter() - t0
    res = s.finish().summary()
    assert res["completed"] == 12
    # The clock is real time: it cannot run ahead of the host's own clock
    # (idle periods sleep until the next arrival / API return) ...
    assert res["sim_wall"] <= elapsed + 0.05, (res["sim_wall"], elapsed)
    # ... and covers at least the arrivals and the timed API calls.
    last_arrival = 11 / SHORT_API["arrival_rate"] * 0.2  # loose: arrivals are Poisson
    assert res["sim_wall"] > last_arrival
    assert res["sim_wall"] > 0.5 * elapsed, (res["sim_wall"], elapsed)
