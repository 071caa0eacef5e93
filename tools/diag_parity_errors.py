"""Per-row logits error distribution of a full-width replay (GPU box).
Usage: python tools/diag_parity_errors.py C2"""
import os
import sys
import tempfile
from pathlib import Path

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
from test_gpu_fullwidth import CASES, filtered_plans  # noqa: E402
from test_gpu_model import pools_for, replay  # noqa: E402

name = sys.argv[1]
case = CASES[name]
plans, cfg = filtered_plans(name, case["rids"], Path(tempfile.mkdtemp()))
d = {"gptj-6b": 4096, "vicuna-13b": 5120}[case["model"]["preset"]]
pools = pools_for(dict(cfg["cost"], gpu_kv_capacity=8 * 4160 * cfg["M"], cpu_kv_capacity=8 * 4160 * cfg["M"]),
                  2 * 2 * d * 2, max_requests=16, max_rows=4096)
errs = []
r = replay(plans, case["model"], pools, len(plans), check_tables_every=1, errors=errs, rtol=1.0)
e = np.array([x[5] for x in errs])
print(name, "rows", len(e), "quantiles 50/90/99/max", np.quantile(e, [0.5, 0.9, 0.99]), e.max())
for kind in (0, 1, 2):
    k = np.array([x[5] for x in errs if x[2] == kind])
    if len(k):
        print(" kind", kind, "rows", len(k), "median", np.median(k), "max", k.max())
for x in sorted(errs, key=lambda x: -x[5])[:10]:
    print(" worst", x)
