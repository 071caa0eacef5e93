"""Diagnostic (not collected): per-iteration device time of the C1 window by
iteration type (decode-only / chunk / with swaps)."""
import sys, json
sys.path.insert(0, "/root/repo")
import numpy as np
import bench
import paper_2402_01869_b200 as ib
ff, n = int(sys.argv[1]), int(sys.argv[2])
pools = bench.gpu_pools(48)
pools["trace_iterations"] = True
ex = ib.Executor({"preset": "gptj-6b"}, 0, pools)
sess = ib.Session(ib.Trace.generate(bench.WORKLOAD), ib.CostModel.from_json(bench.COST), {"policy": "infercept"}, ex)
sess.step(ff)
ex.sync()
st0 = ex.stats()
k0 = len(st0["iter_ms"])
sess.step(n)
ex.sync()
st = ex.stats()
ms = np.array(st["iter_ms"][k0:])
info = np.array(st["iter_info"][k0 + 1:k0 + 1 + len(ms)])  # iter_ms[i] = start(i) -> start(i+1)
ms = ms[:len(info)]
rows, drows, crows, sin, sout = info.T
def show(name, mask):
    if mask.sum():
        print(f"{name:28s} n={mask.sum():5d} mean={ms[mask].mean():7.2f} ms  p50={np.median(ms[mask]):7.2f}  total={ms[mask].sum():8.1f} ms  rows~{rows[mask].mean():.0f} swap~{(sin+sout)[mask].mean():.0f}")
print("total", ms.sum(), "ms over", len(ms), "iterations")
show("decode-only, no swap", (crows == 0) & (sin + sout == 0))
show("decode-only, swap", (crows == 0) & (sin + sout > 0))
show("chunk<=256, no swap", (crows > 0) & (crows <= 256) & (sin + sout == 0))
show("chunk<=256, swap", (crows > 0) & (crows <= 256) & (sin + sout > 0))
show("chunk>256", crows > 256)
show("swap-in only", (sin > 0) & (sout == 0))
show("swap-out only", (sout > 0) & (sin == 0))
show("both directions", (sin > 0) & (sout > 0))
