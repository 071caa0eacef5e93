#!/usr/bin/env python3
"""Measured lines for the BASELINE.json configs beside the C1 headline
(SURVEY §8d C2, C3, C4 and C1 itself), one B200, reference schedules.

Each config: the scheduler (virtual clock, bit-exact with the reference) is
fast-forwarded untimed, then K iterations are timed on the executor's compute
stream.  Reported per config: req/s and decode tok/s over device time, the
iteration mix (decode rows, chunk rows = prefill / API-return / recompute
rows, swapped tokens), K1 HBM GB/s against the measured copy peak, and the
swap link GB/s against the measured pinned-copy peak.

  C2  Vicuna-13B shape, Chatbot + VE (1000 req @2/s, seed 13), 120 GB GPU /
      96 GB CPU ledger: chunked swap under the swap budget.
  C3  Vicuna-13B shape, QA-shaped calls over 3000-token contexts (1000 req
      @2/s, seed 17), 40 GB GPU ledger: Discard-heavy, chunked
      recompute-prefill on the tensor cores.
  C4  Vicuna-13B shape, all six Table-1 classes, 4000 requests arriving at
      1000/s (seed 23, saturating), 140 GB / 64 GB: one replica of the sharded
      run.

Usage (GPU box): python tools/bench_configs.py [--configs C2,C3,C4] [--steps K]
Writes one JSON line per config to stdout.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (ClockSampler, measure_link, peaks)

# The configs live in bench.py (one definition for both); this tool times one
# contiguous window after a fast-forward instead of bench.py's stratified windows.
FAST_FORWARD = {"C1": 3000, "C2": 3000, "C3": 3000, "C4": 2000}
CONFIGS = {k: dict(v, fast_forward=FAST_FORWARD[k]) for k, v in bench.CONFIGS.items()}


def run_config(name, c, steps, host_gb, link, torch):
    import paper_2402_01869_b200 as ib
    trace = ib.Trace.generate(c["workload"])
    cost = ib.CostModel.from_json(c["cost"])
    # Ledger capacity in blocks + slack (the Oracle estimator keeps every
    # request's GPU positions a prefix, so the ledger's blocks suffice).
    blocks = int(c["cost"]["gpu_kv_capacity"] // (16 * c["M"])) + c.get("slack_blocks", 512)
    pools = dict(gpu_blocks=blocks, host_bytes=int(host_gb * 1e9), max_requests=1024, max_rows=4096, timing=True,
                 stage_tokens=1024, swap_slots=10)
    ex = ib.Executor(c["model"], 0, pools)
    sess = ib.Session(trace, cost, {"policy": "infercept", "estimator": "oracle"}, ex)
    ff, _ = sess.step(c["fast_forward"])
    sess.step(5)
    ex.sync()
    torch.cuda.synchronize()
    c0, s0 = sess.counters(), ex.stats()
    clocks = bench.ClockSampler(0)
    clocks.start()
    ex.mark(0)
    done, finished = sess.step(steps)
    ex.mark(1)
    ex.sync()
    dev_s = ex.elapsed_ms() / 1e3
    clk = clocks.stop()
    c1, s1 = sess.counters(), ex.stats()
    d = {k: s1[k] - s0[k] for k in ("k1_ms", "k1_bytes", "swap_ms", "swap_bytes_timed", "chunk_rows", "decode_rows",
                                    "swap_in_tokens", "swap_out_tokens", "swap_in_forwarded_tokens",
                                    "kernel_launches", "iterations")}
    pk = bench.peaks()
    k1 = d["k1_bytes"] / (d["k1_ms"] / 1e3) / 1e9 if d["k1_ms"] else None
    sw = d["swap_bytes_timed"] / (d["swap_ms"] / 1e3) / 1e9 if d["swap_ms"] else None
    link_peak = (link["h2d"] + link["d2h"]) / 2
    out = {
        "config": name, "model": c["model"]["preset"], "workload": c["workload"], "cost": c["cost"],
        "window_iterations": [ff + 6, ff + 5 + done], "trace_finished_in_window": finished,
        "steps": done, "ms_per_step": dev_s * 1e3 / max(done, 1),
        "req_s": (c1["completed"] - c0["completed"]) / dev_s,
        "decode_tok_s": (c1["decode_rows"] - c0["decode_rows"]) / dev_s,
        "completed_in_window": c1["completed"] - c0["completed"],
        "rows_per_iteration": {"decode": d["decode_rows"] / max(done, 1), "chunk": d["chunk_rows"] / max(done, 1)},
        "swap_tokens": {"in": d["swap_in_tokens"], "out": d["swap_out_tokens"],
                        "in_forwarded": d["swap_in_forwarded_tokens"]},
        "k1": {"achieved_gbs": k1, "peak_gbs": pk.get("hbm_gbs"),
               "frac": k1 / pk["hbm_gbs"] if k1 and pk.get("hbm_gbs") else None},
        "swap": {"achieved_gbs": sw, "peak_gbs": link_peak, "frac": sw / link_peak if sw else None},
        "gpu_launches": d["kernel_launches"], "clocks": clk,
    }
    del sess
    ex.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3,C4")
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--host-gb", type=float, default=64.0)
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    link = bench.measure_link(torch)
    for name in args.configs.split(","):
        t0 = time.time()
        line = run_config(name, CONFIGS[name], args.steps, args.host_gb, link, torch)
        line["host_seconds"] = time.time() - t0
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
