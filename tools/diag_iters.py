"""Diagnostic (not collected): per-iteration device time of the C1 window by
iteration type, split into preamble (swap-in scatters it waits for, block
tables, swap-in issue), forward, and post phase (swap-out gather, frees) --
plus how long the host spent inside consume() and blocked on events."""
import os
import sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2402_01869_b200 as ib
ff, n = int(sys.argv[1]), int(sys.argv[2])
C1 = bench.CONFIGS["C1"]
pools = bench.pools_for(C1, 48)
pools["trace_iterations"] = True
ex = ib.Executor({"preset": "gptj-6b"}, 0, pools)
sess = ib.Session(ib.Trace.generate(C1["workload"]), ib.CostModel.from_json(C1["cost"]), {"policy": "infercept"}, ex)
sess.step(ff)
ex.sync()
st0 = ex.stats()
k0 = len(st0["iter_ms"])
w0 = time.perf_counter()
sess.step(n)
w1 = time.perf_counter()
ex.sync()
w2 = time.perf_counter()
st = ex.stats()
print(f"host: step() returned after {1e3*(w1-w0):.0f} ms, sync waited {1e3*(w2-w1):.0f} ms; consume() host total "
      f"{1e3*(st['host_consume_s']-st0['host_consume_s']):.0f} ms; blocked (plan ring, tok ring, swap slot, host pool) ms:",
      [round(1e3*(a-b)) for a, b in zip(st['host_block_s'], st0['host_block_s'])])
ph = np.array(st["iter_ms"][k0:])            # iteration k0.. : [pre, fwd, post]
info = np.array(st["iter_info"][k0:k0 + len(ph)])
ms = ph.sum(axis=1)
rows, drows, crows, sin, sout = info.T
def show(name, mask):
    if mask.sum():
        p = ph[mask].mean(axis=0)
        print(f"{name:24s} n={mask.sum():4d} mean={ms[mask].mean():6.2f} p50={np.median(ms[mask]):6.2f} ms "
              f"[pre {p[0]:5.2f} fwd {p[1]:5.2f} post {p[2]:5.2f}] rows~{rows[mask].mean():.0f} "
              f"in~{sin[mask].mean():.0f} out~{sout[mask].mean():.0f}")
print("total", ms.sum(), "ms over", len(ms), "iterations")
show("decode-only, no swap", (crows == 0) & (sin + sout == 0))
show("decode-only, swap", (crows == 0) & (sin + sout > 0))
show("chunk<=256, no swap", (crows > 0) & (crows <= 256) & (sin + sout == 0))
show("chunk<=256, swap", (crows > 0) & (crows <= 256) & (sin + sout > 0))
show("chunk>256", crows > 256)
show("swap-in only", (sin > 0) & (sout == 0))
show("swap-out only", (sout > 0) & (sin == 0))
show("both directions", (sin > 0) & (sout > 0))
show("all", ms > -1)
if len(sys.argv) > 3:
    import json
    json.dump({"phases": ph.tolist(), "info": info.tolist(), "lead": st["iter_lead_ms"][k0:k0 + len(ph)],
               "host": st["iter_host_ms"][k0:k0 + len(ph)], "swaps": st["swap_trace"], "k0": k0},
              open(sys.argv[3], "w"))
