"""Full-size parity through size-independent properties (BASELINE configs C1/C2).

The CPU oracle's forward is far too slow at 6B/13B width, so at the models'
real shapes the checks are the exact, integer ones: for the first iterations
of the real traces (GPT-J-6B shape on C1, Vicuna-13B shape on the C2 chat/VE
swap-stress trace), every K8 block table and the free-list size equal the CPU
restatement (oracle/blocktable.py) bit for bit, every swapped-out KV byte comes
back bit-identical after the D2H / H2D (or staging-forwarded) round trip, and
the sampled ids are valid vocabulary ids with finite logits.  The sizes stay
exact for the 13B's head_dim 128 (K1 / K2 / SwiGLU / RMSNorm) and the GPT-J's
head_dim 256 paths.
"""
import json

import numpy as np
import pytest

from conftest import have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]

CASES = {
    "C1-gptj6b": dict(
        model={"preset": "gptj-6b"}, M=458752,
        workload=dict(classes=[{"name": "Math"}, {"name": "QA"}, {"name": "Chatbot"}], request_count=2000,
                      arrival_rate=3.0, seed=11),
        cost=dict(mem_per_token=458752, gpu_kv_capacity=150e9, cpu_kv_capacity=128e9, swap_per_token=458752 / 50e9),
        iters=700),
    "C2-vicuna13b": dict(
        model={"preset": "vicuna-13b"}, M=819200,
        workload=dict(classes=[{"name": "Chatbot"}, {"name": "VE"}], request_count=1000, arrival_rate=2.0, seed=13),
        cost=dict(mem_per_token=819200, gpu_kv_capacity=120e9, cpu_kv_capacity=96e9, swap_per_token=819200 / 50e9),
        iters=700),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_full_size_tables_and_swapped_bytes(name, tmp_path):
    import paper_2402_01869_b200 as ib
    from oracle.blocktable import BlockTableOracle

    c = CASES[name]
    path = str(tmp_path / "plans.jsonl")
    sess = ib.Session(ib.Trace.generate(c["workload"]), ib.CostModel.from_json(c["cost"]),
                      {"policy": "infercept", "estimator": "oracle", "plan_log": path})
    sess.step(c["iters"])
    del sess
    plans = [json.loads(line) for line in open(path)]
    gpu_blocks = int(c["cost"]["gpu_kv_capacity"] // (16 * c["M"])) + 512
    pools = dict(gpu_blocks=gpu_blocks, host_bytes=24 << 30, max_requests=1024, max_rows=4096, record=True,
                 stage_tokens=1024, swap_slots=4)
    ex = ib.Executor(c["model"], 0, pools)
    vocab = ex.stats()["model"]["vocab"]
    L, D = ex.stats()["model"]["layers"], ex.stats()["model"]["d_model"]
    bt = BlockTableOracle(gpu_blocks)
    swapped = {}
    checked_bytes = checked_tables = sampled = 0
    for pj in plans:
        # Bytes about to leave the GPU that are resident before this forward
        # (a position decoded in this iteration is written by it).
        before = {}
        for o in pj["ops"]:
            if o[1] != ib.KV_SWAP_OUT:
                continue
            rid, lo, hi = o[0], o[3], o[4]
            hi = min(hi, min([s[1] for s in pj["spans"] if s[0] == rid], default=hi))
            if hi > lo:
                before[rid] = (lo, hi, ex.read_kv(rid, lo, hi, L, D))
        ex.step(ib.Plan.from_json(pj))
        bt.apply(pj)
        toks = [t for t, s in zip(ex.last_tokens(), pj["spans"]) if s[4]]
        if toks:
            logits = ex.last_logits()
            assert np.isfinite(logits).all(), f"non-finite logits at iteration {pj['it']}"
            assert all(0 <= t < vocab for t in toks)
            sampled += len(toks)
        for rid, (lo, hi, b) in before.items():
            assert np.array_equal(ex.read_kv(rid, lo, hi, L, D), b), f"swap-out bytes of {rid} at {pj['it']}"
            swapped[rid] = (lo, hi, b)
        for o in pj["ops"]:
            if o[1] == ib.KV_SWAP_IN and o[0] in swapped:
                lo, hi, b = swapped.pop(o[0])
                a, e = max(lo, o[3]), min(hi, o[4])
                if a < e:
                    assert np.array_equal(ex.read_kv(o[0], a, e, L, D), b[:, a - lo:e - lo]), f"swap-in of {o[0]}"
                    checked_bytes += (e - a) * L * 2 * D * 2
        if pj["it"] % 25 == 0:
            assert ex.free_blocks() == bt.free_blocks()
            live = {s[0] for s in pj["spans"]}
            for rid in sorted(live):
                if any(o[0] == rid and o[1] == ib.KV_RELEASE for o in pj["ops"]):
                    continue
                dev = ex.block_table(rid)
                assert dev == bt.table_of(rid, len(dev)), f"block table of {rid} at {pj['it']}"
                checked_tables += 1
    ex.sync()
    assert sampled > 100 and checked_tables > 50
    print(name, dict(iterations=len(plans), sampled=sampled, tables=checked_tables, swap_bytes_checked=checked_bytes,
                     forwarded=ex.stats()["swap_in_forwarded_tokens"]))
