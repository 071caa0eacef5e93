"""Shared fixtures.  `-m "not gpu"` runs here (no GPU); `-m gpu` on a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/proj"
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libinterceptsim.so")
PRODUCT_LIB = os.path.join(ROOT, "paper_2402_01869_b200", "libinfercept_b200.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    # Build the product library and the reference oracle if they are missing
    # (the GPU box receives both prebuilt with the snapshot).
    if not os.path.exists(PRODUCT_LIB):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2402_01869_b200", "csrc"), "-j8"], check=True,
                       stdout=subprocess.DEVNULL)
    if not os.path.exists(REF_LIB) and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8"], check=True, stdout=subprocess.DEVNULL)


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# The C0 configuration of SURVEY §8d: tiny GPT, 64 requests, all three
# dispositions exercised (swap-out at it 328, swap-in 450, recompute 451).
C0_WORKLOAD = dict(classes=[{"name": c} for c in ["Math", "QA", "VE", "Chatbot", "Image", "TTS"]],
                   request_count=64, arrival_rate=1.0, seed=1, max_seq_len=4096)
C0_COST = dict(t0=2e-3, slope_below=1e-6, slope_above=1e-5, saturation_point=512, mem_per_token=4096,
               gpu_kv_capacity=16384 * 4096, cpu_kv_capacity=4 * 16384 * 4096, swap_per_token=8.192e-6,
               block_size=16)


@pytest.fixture(scope="session")
def c0_plans(tmp_path_factory):
    import paper_2402_01869_b200 as ib
    d = tmp_path_factory.mktemp("c0")
    path = str(d / "plans.jsonl")
    t = ib.Trace.generate(C0_WORKLOAD)
    m = ib.CostModel.from_json(C0_COST)
    res = ib.run(t, m, dict(policy="infercept", estimator="oracle", plan_log=path, check_invariants=True))
    with open(path) as f:
        plans = [json.loads(l) for l in f]
    return plans, res
