"""Run a scheduler configuration through the reference (oracle/_ref) and the
product library through the SAME C ABI, collecting event logs (test helper)."""
import ctypes
import json
import os

from conftest import PRODUCT_LIB, REF_LIB

_libs = {}


def lib(path):
    if path not in _libs:
        L = ctypes.CDLL(path)
        L.isim_trace_generate.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.isim_trace_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.isim_model_from_json.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.isim_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.isim_last_error.restype = ctypes.c_char_p
        L.isim_result_summary_json.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
        L.isim_result_write_requests_csv.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.isim_string_free.argtypes = [ctypes.c_void_p]
        L.isim_trace_free.argtypes = [ctypes.c_void_p]
        L.isim_model_free.argtypes = [ctypes.c_void_p]
        L.isim_result_free.argtypes = [ctypes.c_void_p]
        _libs[path] = L
    return _libs[path]


def run_one(path, trace, cost, cfg, workdir, tag):
    """trace: workload dict (generated) or a path to a JSONL trace."""
    L = lib(path)
    t, m, r = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    if isinstance(trace, str):
        assert L.isim_trace_load(trace.encode(), ctypes.byref(t)) == 0, L.isim_last_error()
    else:
        assert L.isim_trace_generate(json.dumps(trace).encode(), ctypes.byref(t)) == 0, L.isim_last_error()
    assert L.isim_model_from_json(json.dumps(cost).encode(), ctypes.byref(m)) == 0, L.isim_last_error()
    log = os.path.join(workdir, f"{tag}.events.jsonl")
    csv = os.path.join(workdir, f"{tag}.requests.csv")
    c = dict(cfg, event_log=log)
    st = L.isim_run(t, m, json.dumps(c).encode(), ctypes.byref(r))
    out = {"status": st, "events": open(log).read() if os.path.exists(log) else ""}
    if st != 0:
        out["error"] = L.isim_last_error().decode()
    else:
        s = ctypes.c_void_p()
        L.isim_result_summary_json(r, ctypes.byref(s))
        out["summary"] = ctypes.cast(s, ctypes.c_char_p).value.decode()
        L.isim_string_free(s)
        L.isim_result_write_requests_csv(r, csv.encode())
        out["csv"] = open(csv).read()
        L.isim_result_free(r)
    L.isim_trace_free(t)
    L.isim_model_free(m)
    return out


def both(trace, cost, cfg, workdir):
    return run_one(REF_LIB, trace, cost, cfg, workdir, "ref"), run_one(PRODUCT_LIB, trace, cost, cfg, workdir, "ours")


def split_ledger(line):
    j = json.loads(line)
    led = j.pop("ledger", None)
    return json.dumps(j, sort_keys=True), led


def assert_same_events(a: str, b: str):
    la, lb = a.splitlines(), b.splitlines()
    assert len(la) == len(lb), (len(la), len(lb))
    for i, (x, y) in enumerate(zip(la, lb)):
        if x == y:
            continue
        # Only the ledger object's key order may differ (unordered_map).
        jx, lx = split_ledger(x)
        jy, ly = split_ledger(y)
        assert jx == jy and lx == ly, f"iteration {i + 1}:\nref  {x[:400]}\nours {y[:400]}"
