"""GPU parity: the B200 executor vs the CPU oracle on the scheduler's own plans.

For each iteration of a scheduler-emitted plan log the executor (record mode)
and oracle/forward.py run the same BatchPlan; the oracle is teacher-forced with
the device's sampled ids.  Checked every iteration:
  * logits of every sampling row within 1e-3 relative (max |dlogit| / max
    |logit|, fp32 accumulation; north_star tolerance);
  * greedy ids equal except genuine near-ties (top-2 margin below 2e-3 of the
    row's max |logit|), which are counted and must stay rare;
  * the device block tables and free-list size equal the CPU restatement
    (oracle/blocktable.py) bit for bit;
  * swapped KV bytes survive the D2H / H2D round trip bit for bit.
"""
import json

import numpy as np
import pytest

from conftest import C0_COST, C0_WORKLOAD, have_gpu

pytestmark = pytest.mark.gpu

LOGIT_RTOL = 1e-3
TIE_FRAC = 2e-3


def pools_for(cost, model_m, **kw):
    gpu_blocks = int(cost["gpu_kv_capacity"] // (16 * cost["mem_per_token"])) + 2 * 256
    host = int(cost["cpu_kv_capacity"] / cost["mem_per_token"] * model_m * 1.25) + (64 << 20)
    d = dict(gpu_blocks=gpu_blocks, host_bytes=host, max_requests=256, max_rows=1024, record=True)
    d.update(kw)
    return d


def replay(plans, model, pools, n_iters, check_tables_every=1, kv_check=True, errors=None, rtol=LOGIT_RTOL):
    """errors: optional list collecting (iteration, span, kind, count, pos,
    rel err) of every sampled row."""
    import paper_2402_01869_b200 as ib
    from oracle.blocktable import BlockTableOracle
    from oracle.forward import ForwardOracle

    ex = ib.Executor(model, 0, pools)
    fo = ForwardOracle(model)
    bt = BlockTableOracle(pools["gpu_blocks"])
    L, D = fo.m.L, fo.m.D
    worst, ties, sampled, kv_checked = 0.0, 0, 0, 0
    pending_swaps = {}  # rid -> (lo, hi, bytes captured at swap-out)
    for plan_j in plans[:n_iters]:
        plan = ib.Plan.from_json(plan_j)
        # Bytes of positions that are about to leave the GPU (already resident).
        outs = [(o[0], o[3], o[4]) for o in plan_j["ops"] if o[1] == ib.KV_SWAP_OUT]
        pre = {}
        if kv_check:
            for rid, lo, hi in outs:
                grown = [s for s in plan_j["spans"] if s[0] == rid]
                resident_hi = min(hi, min([s[1] for s in grown], default=hi))
                if resident_hi > lo:
                    pre[rid] = (lo, resident_hi, ex.read_kv(rid, lo, resident_hi, L, D))
        ex.step(plan)
        bt.apply(plan_j)
        toks = ex.last_tokens()
        dev_tok = [t for t, s in zip(toks, plan_j["spans"]) if s[4]]
        ref = fo.step(plan_j, teacher_tokens=dev_tok)
        if dev_tok:
            glog = ex.last_logits().reshape(len(dev_tok), -1)
            sampled_spans = [s for s in plan_j["spans"] if s[4]]
            for i, t in enumerate(dev_tok):
                scale = float(np.max(np.abs(ref["logits"][i])))
                err = float(np.max(np.abs(glog[i] - ref["logits"][i]))) / scale
                worst = max(worst, err)
                if errors is not None:
                    sp = sampled_spans[i]
                    errors.append((plan_j["it"], sp[0], sp[3], sp[2], sp[1], err))
                assert err <= rtol, f"iteration {plan_j['it']} row {i}: logits rel err {err:.2e}"
                if t != ref["tokens"][i]:
                    # a flip needs a top-2 margin within the two logits' combined error
                    assert ref["margin"][i] <= TIE_FRAC * (rtol / LOGIT_RTOL) * scale, \
                        (plan_j["it"], i, t, ref["tokens"][i], ref["margin"][i])
                    ties += 1
                sampled += 1
        if kv_check:
            for rid, (lo, hi, before) in pre.items():
                after = ex.read_kv(rid, lo, hi, L, D)  # now read from the pinned host extent
                assert np.array_equal(before, after), f"swap-out bytes of request {rid} changed"
                pending_swaps[rid] = (lo, hi, after)
            for o in plan_j["ops"]:
                if o[1] == ib.KV_SWAP_IN and o[0] in pending_swaps:
                    lo, hi, host_bytes = pending_swaps[o[0]]
                    a, b = max(lo, o[3]), min(hi, o[4])
                    if a < b:
                        back = ex.read_kv(o[0], a, b, L, D)
                        assert np.array_equal(back, host_bytes[:, a - lo:b - lo]), f"swap-in bytes of {o[0]}"
                        kv_checked += b - a
        if plan_j["it"] % check_tables_every == 0:
            assert ex.free_blocks() == bt.free_blocks()
            live = {s[0] for s in plan_j["spans"]} | {o[0] for o in plan_j["ops"] if o[1] != ib.KV_RELEASE}
            for rid in sorted(live):
                if any(o[0] == rid and o[1] == ib.KV_RELEASE for o in plan_j["ops"]):
                    continue
                dev = ex.block_table(rid)
                assert dev == bt.table_of(rid, len(dev)), f"block table of request {rid} at it {plan_j['it']}"
    ex.sync()
    return dict(worst=worst, ties=ties, sampled=sampled, kv_checked=kv_checked, stats=ex.stats())


@pytest.mark.skipif(not have_gpu(), reason="needs a B200")
def test_c0_tiny_parity_with_swap_and_recompute(c0_plans):
    plans, _ = c0_plans
    # The whole C0 trace (18,182 iterations, all 64 requests to completion):
    # swap-outs (first at it 328), discards, swap-ins (450), recomputation
    # (451), completions (1171 on).  Block tables every 10 iterations.
    assert len(plans) == 18182
    r = replay(plans, {"preset": "tiny"}, pools_for(C0_COST, 2048), len(plans), check_tables_every=10)
    assert r["sampled"] > 15000
    assert r["ties"] <= max(2, r["sampled"] // 500)
    assert r["kv_checked"] > 0, "no swapped bytes were round-tripped"
    assert r["stats"]["swap_in_tokens"] > 0 and r["stats"]["swap_out_tokens"] > 0
    print("tiny parity", {k: v for k, v in r.items() if k != "stats"})


def _small_family_plans(tmp_path, n=24):
    import paper_2402_01869_b200 as ib
    wl = dict(C0_WORKLOAD, request_count=n, arrival_rate=4.0, max_seq_len=1024, seed=5)
    cost = dict(C0_COST, gpu_kv_capacity=24576 * 4096)
    path = str(tmp_path / "p.jsonl")
    ib.run(ib.Trace.generate(wl), ib.CostModel.from_json(cost), dict(policy="infercept", plan_log=path))
    return [json.loads(l) for l in open(path)], cost


@pytest.mark.skipif(not have_gpu(), reason="needs a B200")
@pytest.mark.parametrize("fused_qkv,overlap_mlp", [(False, True), (True, True), (False, False)])
def test_gptj_family_small_parity(tmp_path, fused_qkv, overlap_mlp):
    # GPT-J block structure at reduced width: head_dim 256, interleaved rotary
    # 64, parallel residual, LM-head bias; optionally RoPE + KV write fused
    # into the QKV GEMM epilogue; the MLP branch on the second stream or inline.
    plans, cost = _small_family_plans(tmp_path)
    model = {"preset": "gptj-6b", "layers": 2, "d_model": 1024, "heads": 4, "ffn": 4096, "vocab": 8192,
             "max_pos": 1088}
    r = replay(plans, model, pools_for(cost, 2 * 2 * 1024 * 2, max_ctx=1088, fused_qkv=fused_qkv,
                                                overlap_mlp=overlap_mlp), 250,
               check_tables_every=10)
    assert r["sampled"] > 100
    print("gptj-small parity", {k: v for k, v in r.items() if k != "stats"})


@pytest.mark.skipif(not have_gpu(), reason="needs a B200")
def test_llama_family_small_parity(tmp_path):
    # LLaMA block structure at reduced width: head_dim 128, rotate-half RoPE,
    # RMSNorm, SwiGLU.
    plans, cost = _small_family_plans(tmp_path)
    model = {"preset": "vicuna-13b", "layers": 2, "d_model": 1024, "heads": 8, "ffn": 2816, "vocab": 8192,
             "max_pos": 1088}
    r = replay(plans, model, pools_for(cost, 2 * 2 * 1024 * 2, max_ctx=1088), 250, check_tables_every=10)
    assert r["sampled"] > 100
    print("llama-small parity", {k: v for k, v in r.items() if k != "stats"})


@pytest.mark.skipif(not have_gpu(), reason="needs a B200")
def test_end_to_end_run_with_executor_matches_scheduler_only_run():
    # isim_run with the executor attached makes identical scheduling decisions.
    import paper_2402_01869_b200 as ib
    t = ib.Trace.generate(dict(C0_WORKLOAD, request_count=16))
    m = ib.CostModel.from_json(C0_COST)
    a = ib.run(t, m, dict(policy="infercept")).summary()
    b = ib.run(t, m, dict(policy="infercept", executor="b200",
                          exec={"model": {"preset": "tiny"}, "pools": pools_for(C0_COST, 2048, record=False)})).summary()
    assert a == b


@pytest.mark.skipif(not have_gpu(), reason="needs a B200")
def test_split_batch_option_parity(c0_plans):
    # The opt-in split_batch executor (decode rows and chunk rows as two
    # micro-batches on two streams; measured slower, kept for experiments)
    # against the oracle on the first 1,500 C0 iterations.
    plans, _ = c0_plans
    r = replay(plans, {"preset": "tiny"}, pools_for(C0_COST, 2048, split_batch=True), 1500, check_tables_every=10)
    assert r["sampled"] > 1000 and r["kv_checked"] > 0
