"""Diagnostic (not collected by pytest): per-iteration logits error, with and
without routing chunk rows through K1."""
import json, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2402_01869_b200 as ib
from oracle.forward import ForwardOracle
from conftest import C0_WORKLOAD, C0_COST
path = "/tmp/diag_plans.jsonl"
ib.run(ib.Trace.generate(C0_WORKLOAD), ib.CostModel.from_json(C0_COST), dict(policy="infercept", plan_log=path))
plans = [json.loads(l) for l in open(path)][:int(sys.argv[1]) if len(sys.argv) > 1 else 60]
for row_attn in (False, True):
    ex = ib.Executor({"preset": "tiny"}, 0, dict(gpu_blocks=1536, host_bytes=256 << 20, max_requests=128, max_rows=1024,
                                                 record=True, row_attention=row_attn))
    fo = ForwardOracle({"preset": "tiny"})
    errs = []
    for pj in plans:
        ex.step(ib.Plan.from_json(pj))
        toks = [t for t, s in zip(ex.last_tokens(), pj["spans"]) if s[4]]
        ref = fo.step(pj, teacher_tokens=toks)
        if toks:
            g = ex.last_logits().reshape(len(toks), -1)
            e = max(float(np.abs(g[i] - ref["logits"][i]).max() / np.abs(ref["logits"][i]).max()) for i in range(len(toks)))
            errs.append((pj["it"], round(e, 6), sum(s[2] for s in pj["spans"]), len(toks)))
    print("row_attention", row_attn, "worst", max(e[1] for e in errs))
    print(errs[:12])
