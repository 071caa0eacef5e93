"""B200-native InferCept serving hot path.

Python mirror of the reference simulator's interface (proj/include/interceptsim.h)
over this framework's C ABI (include/infercept_b200.h):

    Trace.generate / load / save / request_count / stats      (interceptsim.h:56-62)
    CostModel.default / from_json / load / fit_csv / ...        (interceptsim.h:66-79)
    run(trace, model, run_cfg) -> Result                         (interceptsim.h:98)
    Result.summary / metric / write_requests_csv                 (interceptsim.h:101-111)

plus the B200 additions: BatchPlan (the per-iteration plan the scheduler emits
at the model-step hook, reference engine.cpp:460), Executor (runs a plan on
one GPU) and Session (step the scheduler K iterations at a time).
Errors raise IsimError carrying the reference's status code.
"""
from __future__ import annotations

import ctypes
import json
from typing import Iterable, Optional

from . import _abi
from ._abi import (BatchPlan, IsimError, KvOp, RowSpan, KV_GROW, KV_SWAP_OUT, KV_SWAP_IN, KV_DISCARD,
                   KV_RECOMPUTE, KV_RELEASE, SPAN_DECODE, SPAN_FRESH, SPAN_RECOMPUTE)

__all__ = ["Trace", "CostModel", "Result", "run", "Executor", "Session", "Plan", "read_plan_log", "IsimError",
           "abi_version", "KV_GROW", "KV_SWAP_OUT", "KV_SWAP_IN", "KV_DISCARD", "KV_RECOMPUTE", "KV_RELEASE",
           "SPAN_DECODE", "SPAN_FRESH", "SPAN_RECOMPUTE", "MODEL_PRESETS"]

_L = _abi.lib

MODEL_PRESETS = {
    "tiny": dict(family="gpt2", layers=2, d_model=256, heads=4, ffn=1024, vocab=4096, rotary_dim=0),
    "gptj-6b": dict(family="gptj", layers=28, d_model=4096, heads=16, ffn=16384, vocab=50400, rotary_dim=64),
    "vicuna-13b": dict(family="llama", layers=40, d_model=5120, heads=40, ffn=13824, vocab=32000, rotary_dim=128),
}


def abi_version() -> int:
    return int(_L.isim_abi_version())


def _enc(d) -> bytes:
    return (d if isinstance(d, str) else json.dumps(d)).encode()


class _Handle:
    _free = None

    def __init__(self, ptr: ctypes.c_void_p):
        self._ptr = ptr

    @property
    def ptr(self):
        return self._ptr

    def close(self):
        if self._ptr and self._ptr.value:
            type(self)._free(self._ptr)
            self._ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Trace(_Handle):
    _free = _L.isim_trace_free

    @classmethod
    def generate(cls, workload: dict | str) -> "Trace":
        p = ctypes.c_void_p()
        _abi.check(_L.isim_trace_generate(_enc(workload), ctypes.byref(p)))
        return cls(p)

    @classmethod
    def load(cls, path: str) -> "Trace":
        p = ctypes.c_void_p()
        _abi.check(_L.isim_trace_load(path.encode(), ctypes.byref(p)))
        return cls(p)

    def save(self, path: str) -> None:
        _abi.check(_L.isim_trace_save(self._ptr, path.encode()))

    def request_count(self) -> int:
        return int(_L.isim_trace_request_count(self._ptr))

    def stats(self) -> dict:
        s = ctypes.c_void_p()
        _abi.check(_L.isim_trace_stats_json(self._ptr, ctypes.byref(s)))
        return json.loads(_abi.take_string(s))


class CostModel(_Handle):
    _free = _L.isim_model_free

    @classmethod
    def default(cls) -> "CostModel":
        p = ctypes.c_void_p()
        _abi.check(_L.isim_model_default(ctypes.byref(p)))
        return cls(p)

    @classmethod
    def from_json(cls, spec: dict | str) -> "CostModel":
        p = ctypes.c_void_p()
        _abi.check(_L.isim_model_from_json(_enc(spec), ctypes.byref(p)))
        return cls(p)

    @classmethod
    def load(cls, path: str) -> "CostModel":
        p = ctypes.c_void_p()
        _abi.check(_L.isim_model_load(path.encode(), ctypes.byref(p)))
        return cls(p)

    @classmethod
    def fit_csv(cls, csv_path: str, base: Optional[dict | str] = None) -> "CostModel":
        p = ctypes.c_void_p()
        _abi.check(_L.isim_model_fit_csv(csv_path.encode(), _enc(base) if base is not None else None, ctypes.byref(p)))
        return cls(p)

    def to_json(self) -> dict:
        s = ctypes.c_void_p()
        _abi.check(_L.isim_model_to_json(self._ptr, ctypes.byref(s)))
        return json.loads(_abi.take_string(s))

    def save(self, path: str) -> None:
        _abi.check(_L.isim_model_save(self._ptr, path.encode()))

    def t_fwd(self, batch_tokens: float) -> float:
        return float(_L.isim_model_t_fwd(self._ptr, float(batch_tokens)))

    def t_swap(self, tokens: float) -> float:
        return float(_L.isim_model_t_swap(self._ptr, float(tokens)))


class Result(_Handle):
    _free = _L.isim_result_free

    def summary(self) -> dict:
        s = ctypes.c_void_p()
        _abi.check(_L.isim_result_summary_json(self._ptr, ctypes.byref(s)))
        return json.loads(_abi.take_string(s))

    def metric(self, name: str) -> float:
        v = ctypes.c_double()
        _abi.check(_L.isim_result_metric(self._ptr, name.encode(), ctypes.byref(v)))
        return v.value

    def write_requests_csv(self, path: str) -> None:
        _abi.check(_L.isim_result_write_requests_csv(self._ptr, path.encode()))


def run(trace: Trace, model: CostModel, run_cfg: Optional[dict | str] = None) -> Result:
    """isim_run: the whole scheduler loop; with {"executor": "b200"} every
    iteration's plan also runs on the GPU."""
    p = ctypes.c_void_p()
    _abi.check(_L.isim_run(trace.ptr, model.ptr, _enc(run_cfg) if run_cfg is not None else None, ctypes.byref(p)))
    return Result(p)


class Plan:
    """One BatchPlan held in ctypes memory (from a plan log or built by hand)."""

    def __init__(self, it: int, ops: Iterable, spans: Iterable, t_end: float = 0.0, batch_tokens: int = 0):
        ops = list(ops)
        spans = list(spans)
        self.iteration = it
        self.ops = ops
        self.spans = spans
        self._ops = (KvOp * max(1, len(ops)))(*[KvOp(*o) for o in ops])
        self._spans = (RowSpan * max(1, len(spans)))(*[RowSpan(*s) for s in spans])
        self.c = BatchPlan(it, t_end, batch_tokens, 0, 0, 0, len(ops), len(spans), self._ops, self._spans)

    @classmethod
    def from_json(cls, j: dict) -> "Plan":
        return cls(j["it"], j["ops"], j["spans"], j.get("t", 0.0), j.get("B", 0))


def read_plan_log(path: str) -> list:
    with open(path) as f:
        return [Plan.from_json(json.loads(line)) for line in f if line.strip()]


class Executor(_Handle):
    """isim_exec_*: one B200 executor (weights, paged KV pool, swap pool)."""
    _free = _L.isim_exec_free

    def __init__(self, model: dict | str = None, device: int = 0, pools: Optional[dict] = None):
        p = ctypes.c_void_p()
        _abi.check(_L.isim_exec_create(_enc(model if model is not None else {"preset": "tiny"}), device,
                                       _enc(pools or {}), ctypes.byref(p)))
        super().__init__(p)

    def step(self, plan: Plan) -> None:
        _abi.check(_L.isim_exec_step(self._ptr, ctypes.byref(plan.c)))

    def sync(self) -> None:
        _abi.check(_L.isim_exec_sync(self._ptr))

    def mark(self, which: int) -> None:
        """Record the start (0) / stop (1) timing mark on the compute stream."""
        _abi.check(_L.isim_exec_timer(self._ptr, which, None))

    def elapsed_ms(self) -> float:
        v = ctypes.c_double()
        _abi.check(_L.isim_exec_timer(self._ptr, 2, ctypes.byref(v)))
        return v.value

    def stats(self) -> dict:
        s = ctypes.c_void_p()
        _abi.check(_L.isim_exec_stats_json(self._ptr, ctypes.byref(s)))
        return json.loads(_abi.take_string(s))

    def last_tokens(self) -> list:
        n = ctypes.c_int32()
        _abi.check(_L.isim_exec_last_tokens(self._ptr, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_int32 * max(1, n.value))()
        _abi.check(_L.isim_exec_last_tokens(self._ptr, buf, n.value, ctypes.byref(n)))
        return list(buf)[: n.value]

    def last_logits(self):
        import numpy as np
        n = ctypes.c_int64()
        _abi.check(_L.isim_exec_last_logits(self._ptr, None, 0, ctypes.byref(n)))
        out = np.empty(n.value, dtype=np.float32)
        _abi.check(_L.isim_exec_last_logits(self._ptr, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), n.value,
                                            ctypes.byref(n)))
        return out

    def block_table(self, request_id: int) -> list:
        n = ctypes.c_int32()
        buf = (ctypes.c_int32 * 4096)()
        _abi.check(_L.isim_exec_block_table(self._ptr, request_id, buf, 4096, ctypes.byref(n)))
        return list(buf)[: n.value]

    def free_blocks(self) -> int:
        v = ctypes.c_int64()
        _abi.check(_L.isim_exec_free_blocks(self._ptr, ctypes.byref(v)))
        return v.value

    def read_kv(self, request_id: int, lo: int, hi: int, layers: int, d_model: int):
        import numpy as np
        out = np.empty((layers, hi - lo, 2, d_model), dtype=np.uint16)
        _abi.check(_L.isim_exec_read_kv(self._ptr, request_id, lo, hi, out.ctypes.data, out.nbytes))
        return out

    def read_history(self, request_id: int, lo: int, hi: int):
        import numpy as np
        out = np.empty(hi - lo, dtype=np.int32)
        _abi.check(_L.isim_exec_read_history(self._ptr, request_id, lo, hi, out.ctypes.data, out.size))
        return out


class Session(_Handle):
    """isim_session_*: the scheduler stepped K iterations at a time."""
    _free = _L.isim_session_free

    def __init__(self, trace: Trace, model: CostModel, run_cfg: Optional[dict] = None,
                 executor: Optional[Executor] = None):
        p = ctypes.c_void_p()
        _abi.check(_L.isim_session_open(trace.ptr, model.ptr, _enc(run_cfg or {}),
                                        executor.ptr if executor is not None else None, ctypes.byref(p)))
        super().__init__(p)
        self._trace, self._model, self._exec = trace, model, executor  # keep alive

    def step(self, max_iters: int) -> tuple:
        done = ctypes.c_int64()
        fin = ctypes.c_int32()
        _abi.check(_L.isim_session_step(self._ptr, max_iters, ctypes.byref(done), ctypes.byref(fin)))
        return done.value, bool(fin.value)

    def fast_forward(self, max_iters: int) -> tuple:
        """Scheduler-only iterations, then the executor is handed the ledger's
        KV layout (isim_session_fast_forward): positions timing windows."""
        done = ctypes.c_int64()
        fin = ctypes.c_int32()
        _abi.check(_L.isim_session_fast_forward(self._ptr, max_iters, ctypes.byref(done), ctypes.byref(fin)))
        return done.value, bool(fin.value)

    def counters(self) -> dict:
        v = [ctypes.c_int64() for _ in range(4)]
        _abi.check(_L.isim_session_counters(self._ptr, *[ctypes.byref(x) for x in v]))
        return dict(completed=v[0].value, decode_rows=v[1].value, batch_tokens=v[2].value, swapped_tokens=v[3].value)

    def finish(self) -> Result:
        p = ctypes.c_void_p()
        _abi.check(_L.isim_session_finish(self._ptr, ctypes.byref(p)))
        return Result(p)
