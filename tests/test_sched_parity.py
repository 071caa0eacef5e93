"""Scheduling parity: the product scheduler vs the reference simulator itself.

Both libraries are driven through the same C ABI on the same generated traces;
the per-iteration event logs (batch size, duration, swap in/out, recompute,
stall, fire/done/evict/swapin events, and per-request ledger snapshots) must be
byte-identical (ledger key order aside), and so must the summaries and the
per-request CSVs.  Reference: proj/src/engine.cpp:282-581.
"""
import json
import os

import pytest

from conftest import C0_COST, C0_WORKLOAD, REF_LIB
from refrun import assert_same_events, both

pytestmark = pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built (needs /root/reference)")

POLICIES = ["infercept", "vanilla-discard", "improved-discard", "preserve", "swap"]
ESTIMATORS = ["oracle", "profiled", "dynamic"]


def check(trace, cost, cfg, tmp_path):
    ref, ours = both(trace, cost, cfg, str(tmp_path))
    assert ref["status"] == ours["status"], (ref.get("error"), ours.get("error"))
    if ref["status"] != 0:
        assert ref["error"] == ours["error"]
    else:
        assert ref["summary"] == ours["summary"]
        assert ref["csv"] == ours["csv"]
    assert_same_events(ref["events"], ours["events"])
    return ref


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("estimator", ESTIMATORS)
def test_c0_tiny_all_policies(policy, estimator, tmp_path):
    ledger = 1 if policy == "infercept" else 0
    check(C0_WORKLOAD, C0_COST, dict(policy=policy, estimator=estimator, dump_ledger_every=ledger), tmp_path)


GPTJ_M = 458752
LINK = 50e9


def test_c1_gptj_mix(tmp_path):
    wl = dict(classes=[{"name": "Math"}, {"name": "QA"}, {"name": "Chatbot"}], request_count=2000, arrival_rate=3.0,
              seed=11)
    cost = dict(mem_per_token=GPTJ_M, gpu_kv_capacity=150e9, cpu_kv_capacity=128e9, swap_per_token=GPTJ_M / LINK)
    ref = check(wl, cost, dict(policy="infercept", estimator="oracle", dump_ledger_every=97), tmp_path)
    assert len(ref["events"].splitlines()) == 35589


def test_c2_vicuna_chat_ve(tmp_path):
    M = 819200
    wl = dict(classes=[{"name": "Chatbot", "weight": 0.5}, {"name": "VE", "weight": 0.5}], request_count=1000,
              arrival_rate=2.0, seed=13)
    cost = dict(mem_per_token=M, gpu_kv_capacity=120e9, cpu_kv_capacity=96e9, swap_per_token=M / LINK)
    ref = check(wl, cost, dict(policy="infercept", estimator="oracle", dump_ledger_every=101), tmp_path)
    assert len(ref["events"].splitlines()) == 29111


def test_c3_discard_heavy(tmp_path):
    M = 819200
    wl = dict(classes=[{"name": "QA", "context_mean": 3000, "context_var": 40000}], request_count=300,
              arrival_rate=2.0, seed=17)
    cost = dict(mem_per_token=M, gpu_kv_capacity=40e9, cpu_kv_capacity=128e9, swap_per_token=M / LINK)
    check(wl, cost, dict(policy="infercept", estimator="oracle", dump_ledger_every=50), tmp_path)


def test_deadlock_reproduced_identically(tmp_path):
    # a tiny pool deadlocks; both sides raise the same SimError.
    cost = dict(C0_COST, gpu_kv_capacity=8192 * 4096)
    wl = dict(C0_WORKLOAD, arrival_rate=4.0)
    ref = check(wl, cost, dict(policy="infercept"), tmp_path)
    assert ref["status"] == 7 and "cannot fit in GPU KV capacity" in ref["error"]


def test_fractional_memory_and_fit(tmp_path):
    # Non-integral mem_per_token exercises the double byte totals (memory.cpp:17).
    cost = dict(C0_COST, mem_per_token=3000.7, gpu_kv_capacity=16384 * 3000.7 * 1.01)
    check(dict(C0_WORKLOAD, request_count=32), cost, dict(policy="infercept", dump_ledger_every=1), tmp_path)


@pytest.mark.parametrize("workload", [
    "C0", dict(classes=[{"name": "Math"}, {"name": "QA"}, {"name": "Chatbot"}], request_count=300, arrival_rate=3.0, seed=11),
    dict(classes=[{"name": c} for c in ["Math", "QA", "VE", "Chatbot", "Image", "TTS"]], request_count=500,
         arrival_rate=1000.0, seed=23),
])
def test_saved_trace_jsonl_byte_identical(tmp_path, workload):
    """f3: a trace generated and saved by the product library is byte-identical
    to the reference's (proj/src/workload.cpp generation, trace_io.cpp format)."""
    import ctypes
    from conftest import C0_WORKLOAD, PRODUCT_LIB, REF_LIB
    wl = C0_WORKLOAD if workload == "C0" else workload
    outs = []
    for lib_path, tag in ((REF_LIB, "ref"), (PRODUCT_LIB, "ours")):
        L = ctypes.CDLL(lib_path)
        L.isim_trace_generate.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.isim_trace_save.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.isim_trace_free.argtypes = [ctypes.c_void_p]
        t = ctypes.c_void_p()
        assert L.isim_trace_generate(json.dumps(wl).encode(), ctypes.byref(t)) == 0
        path = str(tmp_path / f"{tag}.jsonl")
        assert L.isim_trace_save(t, path.encode()) == 0
        L.isim_trace_free(t)
        outs.append(open(path, "rb").read())
    assert outs[0] == outs[1] and len(outs[0]) > 1000
