"""The fp16 rounding-point floor of the logits comparison (CPU, oracle only).

Two implementations that round at the same fp16 points but accumulate in a
different order disagree wherever an intermediate value lands on the other
side of an fp16 rounding boundary.  Measured here with the oracle itself:
its float32 variant against its float64 reference on the first iterations of
a real C2 request (Vicuna-13B shape at full width, 2 layers).  This floor is
what the device's 13B-shape tolerance in tests/test_gpu_fullwidth.py is
derived from (device within 1.5x of it).
"""
import tempfile
from pathlib import Path

import numpy as np

from test_gpu_fullwidth import CASES, filtered_plans


def test_fp16_rounding_floor_at_13b_width():
    from oracle.forward import ForwardOracle
    case = CASES["C2"]
    plans, _ = filtered_plans("C2", case["rids"][:1], Path(tempfile.mkdtemp()))
    ref = ForwardOracle(case["model"])
    f32 = ForwardOracle(case["model"], precision="f32")
    errs = []
    for pj in plans[:24]:
        a = ref.step(pj)
        b = f32.step(pj, teacher_tokens=a["tokens"])
        for i in range(len(a["tokens"])):
            errs.append(float(np.abs(a["logits"][i] - b["logits"][i]).max() / np.abs(a["logits"][i]).max()))
    med = float(np.median(errs))
    # two CPU implementations already sit at ~7-8e-4 (median) of each other
    assert 5e-4 < med < 1e-3, med
    assert max(errs) < 1.5e-3
    print("oracle f32 vs f64 at the 13B shape:", len(errs), "rows, median", med, "max", max(errs))
