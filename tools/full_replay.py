"""Whole-trace replay on one B200 (validates bench.py's stratified estimator):
every iteration of the config's schedule through the executor, device time on
the compute stream and host wall time, req/s = requests / device seconds.
Usage: python tools/full_replay.py [C4]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2402_01869_b200 as ib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = bench.CONFIGS[name]
torch.cuda.set_device(0)
trace = ib.Trace.generate(cfg["workload"])
iters, done = bench.schedule_totals(ib, trace, cfg)
ex = ib.Executor(cfg["model"], 0, bench.pools_for(cfg, bench.host_pool_gb(cfg, 1, 0)))
sess = ib.Session(trace, ib.CostModel.from_json(cfg["cost"]), bench.RUN, ex)
segs = []
w0 = time.perf_counter()
total_dev = 0.0
n = 0
while True:
    ex.mark(0)
    k, fin = sess.step(1000)
    ex.mark(1)
    ex.sync()
    ms = ex.elapsed_ms()
    total_dev += ms / 1e3
    segs.append([n, k, round(ms / max(k, 1), 3)])
    n += k
    if fin or k == 0:
        break
wall = time.perf_counter() - w0
c = sess.counters()
print(json.dumps({"config": name, "iterations": n, "schedule_iterations": iters, "completed": c["completed"],
                  "device_s": total_dev, "wall_s": wall, "req_s_device": c["completed"] / total_dev,
                  "req_s_wall": c["completed"] / wall, "ms_per_iteration": 1e3 * total_dev / n,
                  "segments_ms_per_iteration": segs}))
