"""Per-iteration batch composition recovered from the REFERENCE's own outputs
(TEST INFRASTRUCTURE ONLY: the bench's --impl reference arm and tests use it;
the product never imports it).

The reference engine (interceptsim, compiled by oracle/Makefile into
oracle/_ref/libinterceptsim.so) emits no batch plan: its model step is the
analytic CostModel::t_fwd(B) at proj/src/engine.cpp:460.  What it does emit,
with run options {"event_log": path, "dump_ledger_every": 1}, is one JSON
record per iteration (engine.cpp:567-581 write_event_record) holding B (the
batch's query rows), the fire/done/swapin events and the KvLedger snapshot
after the iteration (memory.cpp:96-110 snapshot_json: gpu / cpu / discarded
token counts per live request).  This module derives each iteration's row
spans from consecutive snapshots alone, so the CPU path timed by the bench's
reference arm never touches the product scheduler:

  * fresh rows of request r   = delta of (gpu + cpu + discarded): prompt /
    API-returned / decode tokens are the only way a request's total token
    count grows (swaps and discards move tokens between the three counters,
    memory.cpp:13-94), phase-1 dispositions included;
  * recompute rows            = decrease of `discarded` (engine.cpp:388-424:
    recompute restores discarded tokens onto the GPU) when positive;
  * a request first seen this iteration grew from zero;
  * a request whose `done:` event fires this iteration left the ledger
    (engine.cpp:204-216 complete_request releases it), and an `evict:`-ed one
    had all its GPU tokens discarded (engine.cpp:179-188), which hides its
    rows; these take the iteration's remaining B (one row each beyond the
    first).  Ghost decode rows (a request evicted after it was batched,
    SURVEY H3) are counted in B, so they appear here although the product
    drops them from the device batch;
  * the span's first position = the request's context before the new rows
    (gpu + cpu before the iteration, plus restored tokens), i.e. the rows
    attend over everything before them, as the executor's rows do.

Exact for the row COUNTS the forward's cost depends on (sum of rows == B is
checked per iteration; tests/test_ref_plans.py compares the spans with the
product's plan log); positions of recompute spans after partial discards are
approximated (timing only).
"""
from __future__ import annotations

import ctypes
import json
import os
import re
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libinterceptsim.so")

DECODE, FRESH, RECOMPUTE = 0, 1, 2
_IT = re.compile(r'"it":(\d+)')


def _lib(path=REF_LIB):
    L = ctypes.CDLL(path)
    L.isim_trace_generate.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    L.isim_model_from_json.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    L.isim_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    L.isim_result_metric.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_double)]
    L.isim_last_error.restype = ctypes.c_char_p
    L.isim_trace_free.argtypes = [ctypes.c_void_p]
    L.isim_model_free.argtypes = [ctypes.c_void_p]
    L.isim_result_free.argtypes = [ctypes.c_void_p]
    return L


def run_reference(workload: dict, cost: dict, run_cfg: dict, event_log: str | None, ledger_every: int = 1,
                  lib_path: str = REF_LIB) -> dict:
    """isim_run of the reference library with an event log; returns the
    summary metrics the bench needs and the wall time of the run
    (event_log None: no log, the scheduler's own speed)."""
    import time
    L = _lib(lib_path)
    t, m, r = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    if L.isim_trace_generate(json.dumps(workload).encode(), ctypes.byref(t)):
        raise RuntimeError(L.isim_last_error().decode())
    if L.isim_model_from_json(json.dumps(cost).encode(), ctypes.byref(m)):
        raise RuntimeError(L.isim_last_error().decode())
    cfg = dict(run_cfg)
    if event_log:
        cfg["event_log"] = event_log
    if event_log and ledger_every:
        cfg["dump_ledger_every"] = ledger_every
    t0 = time.perf_counter()
    st = L.isim_run(t, m, json.dumps(cfg).encode(), ctypes.byref(r))
    wall = time.perf_counter() - t0
    if st:
        raise RuntimeError(L.isim_last_error().decode())
    out = {"wall_s": wall}
    for name in ("iterations", "completed", "throughput"):
        v = ctypes.c_double()
        if L.isim_result_metric(r, name.encode(), ctypes.byref(v)) == 0:
            out[name] = v.value
    L.isim_result_free(r)
    L.isim_trace_free(t)
    L.isim_model_free(m)
    return out


def _spans_of(rec, prev):
    led = rec["ledger"]["requests"]
    done = [int(e.split(":")[1]) for e in rec["events"] if e.startswith("done:")]
    evicted = {int(e.split(":")[1]) for e in rec["events"] if e.startswith("evict:")}
    spans = []
    total = 0
    for key, e in led.items():
        rid = int(key)
        if rid in evicted:
            continue  # its rows are confounded with the discard-all (below)
        g0, c0, d0 = prev.get(rid, (0, 0, 0))
        g1, c1, d1 = e["gpu"], e["cpu"], e["discarded"]
        fresh = (g1 + c1 + d1) - (g0 + c0 + d0)
        rec_rows = max(0, d0 - d1)
        if fresh <= 0 and rec_rows == 0:
            continue
        fresh = max(fresh, 0)
        # restored tokens (swap-in: cpu -> gpu) are resident before the rows run
        swapped_in = max(0, c0 - c1) if g1 > g0 else 0
        ctx_before = g0 + swapped_in
        if rec_rows:
            spans.append([rid, ctx_before, rec_rows, RECOMPUTE, 0 if fresh else 1])
            ctx_before += rec_rows
            total += rec_rows
        if fresh:
            spans.append([rid, ctx_before, fresh, FRESH, 1])
            total += fresh
    # Requests that finished (released) or were evicted (engine.cpp:179-188,
    # discard-all) this iteration: the rest of B, one row each beyond the first.
    rest = rec["B"] - total
    tail = done + sorted(r for r in evicted if r not in done)
    for i, rid in enumerate(tail):
        g0, c0, d0 = prev.get(rid, (0, 0, 0))
        n = rest - (len(tail) - 1) if i == 0 else 1
        if n <= 0:
            continue
        if rid in evicted and d0 > 0 and n > 1:
            k = min(n, d0)
            spans.append([rid, g0 if g0 else 0, k, RECOMPUTE, 1 if k == n else 0])
            if n > k:
                spans.append([rid, g0 + k, n - k, FRESH, 1])
        else:
            spans.append([rid, g0 + c0, n, FRESH, 1])
        total += n
    return spans, total


def plans_from_events(lines, keep=None):
    """Yield {"it", "B", "rows", "spans": [[rid, pos, count, kind, sample]]}
    per event-log record (every record must carry a ledger snapshot).
    keep: optional set of iteration numbers to emit (all are tracked).

    Kinds and sample flags need one record of look-ahead: a one-row fresh
    span of a request that gets at most one row in the next iteration, or
    whose interception fires now, is a decode row; a chunk samples unless the request's
    next iteration continues it with another multi-row chunk."""
    prev = {}
    pending = None  # (record, spans, total) awaiting the next record
    def emit(item, nxt_rows):
        rec, spans, total = item
        if keep is not None and rec["it"] not in keep:
            return None
        fired = {int(e.split(":")[1]) for e in rec["events"] if e.startswith("fire:")}
        for s in spans:
            if s[3] == FRESH:
                nxt = nxt_rows.get(s[0], 0)
                if s[2] == 1 and (nxt <= 1 or s[0] in fired):
                    s[3] = DECODE
                elif s[2] > 1 and nxt > 1:
                    s[4] = 0
            elif s[3] == RECOMPUTE and s[4] and nxt_rows.get(s[0], 0) > 1:
                s[4] = 0
        return {"it": rec["it"], "B": rec["B"], "rows": total, "spans": spans, "ops": [],
                "evicted": sorted(int(e.split(":")[1]) for e in rec["events"] if e.startswith("evict:"))}
    need = None if keep is None else {k + d for k in keep for d in (-1, 0, 1)}
    for line in lines:
        if need is not None and isinstance(line, str):
            m = _IT.search(line)
            if m and int(m.group(1)) not in need:
                pending = None  # records outside the kept neighbourhoods are skipped unparsed
                prev = {}
                continue
        rec = json.loads(line) if isinstance(line, str) else line
        spans, total = _spans_of(rec, prev)
        prev = {int(k): (e["gpu"], e["cpu"], e["discarded"]) for k, e in rec["ledger"]["requests"].items()}
        if pending is not None:
            rows = {}
            for s in spans:
                rows[s[0]] = rows.get(s[0], 0) + s[2]
            out = emit(pending, rows)
            if out:
                yield out
        pending = (rec, spans, total)
    if pending is not None:
        out = emit(pending, {})
        if out:
            yield out


def reference_schedule(workload: dict, cost: dict, run_cfg: dict, keep=None, workdir: str | None = None):
    """Run the reference once; return (summary, [plans of the kept iterations])."""
    d = workdir or tempfile.mkdtemp()
    log = os.path.join(d, "ref_events.jsonl")
    summ = run_reference(workload, cost, run_cfg, log)
    with open(log) as f:
        plans = list(plans_from_events(f, keep))
    done = 0
    with open(log) as f:
        for line in f:
            if '"done:' in line:
                done += line.count('"done:')
    summ["done_events"] = done
    if not workdir:
        os.remove(log)
    return summ, plans
