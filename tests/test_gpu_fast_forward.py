"""Executor hand-over after a scheduler-only fast-forward (isim_session_fast_forward).

The bench positions its timing windows with it: the executor releases every
request it held, the scheduler runs alone, then the executor is handed the
ledger's KV layout (GPU runs grown in place; host runs grown and swapped out)
and keeps executing.  Checked on the asynchronous (bench) executor path over
the whole C0 trace with three fast-forwards: no residency / host-extent
errors, the schedule is the scheduler-only one, and every device block and
host extent is returned at the end.
"""
import pytest

from conftest import C0_COST, C0_WORKLOAD, have_gpu
from test_gpu_model import pools_for

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]


def test_fast_forward_handover_c0():
    import paper_2402_01869_b200 as ib
    t = ib.Trace.generate(C0_WORKLOAD)
    m = ib.CostModel.from_json(C0_COST)
    pools = pools_for(C0_COST, 2048, record=False, stage_tokens=256, swap_slots=4)
    ex = ib.Executor({"preset": "tiny"}, 0, pools)
    s = ib.Session(t, m, dict(policy="infercept"), ex)
    ref = ib.Session(t, m, dict(policy="infercept"))
    for ff, run in ((300, 200), (2500, 300), (6000, 500)):
        assert s.fast_forward(ff) == ref.step(ff)
        assert s.step(run) == ref.step(run)
        ex.sync()
        st = ex.stats()
        assert st["swap_out_tokens"] > 0
    s.step(10 ** 9)
    ref.step(10 ** 9)
    assert s.finish().summary() == ref.finish().summary()
    ex.sync()
    assert ex.free_blocks() == pools["gpu_blocks"]
    assert ex.stats()["host_pool_used"] == 0
