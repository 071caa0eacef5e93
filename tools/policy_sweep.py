"""Baseline policies on the B200: the paper's comparison of
InferCept's min-waste policy against Vanilla/Improved Discard, Preserve and
naive Swap, with every iteration's BatchPlan executed on the GPU.

For each policy the whole trace (GPT-J-6B shape, Math/QA/Chatbot mix, the C1
class mix, 400 requests at 6/s against a 40 GB KV ledger) is scheduled by the bit-exact scheduler
and run by the executor; reported per policy: requests completed per second of
device time, decode tokens per second, the recompute / swap work the policy
caused, iterations, and the scheduler's own (virtual-clock) makespan.

Usage (GPU box): python tools/policy_sweep.py [requests=400] [out=profiles/policy_sweep.json]
"""
import gc
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2402_01869_b200 as ib  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 400
OUT = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "policy_sweep.json")
# Memory pressure, where the policies differ: 40 GB of KV for the ledger and
# twice the C1 arrival rate (the C1 mix at 150 GB never fills).
C1 = bench.CONFIGS["C1"]
WL = dict(C1["workload"], request_count=N, arrival_rate=6.0)
COST = dict(C1["cost"], gpu_kv_capacity=40e9, cpu_kv_capacity=64e9)
POLICIES = ["infercept", "improved-discard", "vanilla-discard", "preserve", "swap"]

rows = []
ex = None
for pol in POLICIES:
    # Naive Swap is the synchronous baseline (the scheduler charges its swap
    # time as a stall, reference engine.cpp:226-241): its executor waits for
    # each swap batch on the compute stream instead of overlapping it.
    if ex is not None:
        del sess, ex
        gc.collect()  # the previous executor's pools must be released first
    blocks = int(COST["gpu_kv_capacity"] // (16 * bench.GPTJ_M)) + 512
    pools = dict(bench.pools_for(C1, 96, blocks), overlap_swaps=(pol != "swap"))  # pinned pool > the 64 GB CPU ledger
    ex = ib.Executor({"preset": "gptj-6b"}, 0, pools)
    s0 = ex.stats()
    sess = ib.Session(ib.Trace.generate(WL), ib.CostModel.from_json(COST), {"policy": pol, "estimator": "oracle"},
                      ex)
    c0 = sess.counters()
    t0 = time.perf_counter()
    ex.mark(0)
    done, finished = sess.step(10 ** 9)
    ex.mark(1)
    ex.sync()
    wall = time.perf_counter() - t0
    dev_s = ex.elapsed_ms() / 1e3
    c1, s1 = sess.counters(), ex.stats()
    summary = sess.finish().summary()
    row = dict(policy=pol, swaps_overlapped=pol != "swap", iterations=done, completed=c1["completed"] - c0["completed"], device_s=dev_s, wall_s=wall,
               req_per_s=(c1["completed"] - c0["completed"]) / dev_s,
               decode_tok_per_s=(c1["decode_rows"] - c0["decode_rows"]) / dev_s,
               normalized_latency=summary.get("normalized_latency"), waste_gb_min=summary["waste"]["total_gb_min"],
               swap_in_tokens=s1["swap_in_tokens"] - s0["swap_in_tokens"],
               swap_out_tokens=s1["swap_out_tokens"] - s0["swap_out_tokens"],
               forwarded_tokens=s1["swap_in_forwarded_tokens"] - s0["swap_in_forwarded_tokens"],
               virtual_throughput=summary.get("throughput"))
    rows.append(row)
    print(json.dumps(row), flush=True)
json.dump({"workload": WL, "model": "gptj-6b (random init, fp16)", "cost_model": COST, "rows": rows},
          open(OUT, "w"), indent=1)
