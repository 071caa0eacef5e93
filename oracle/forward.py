"""CPU numerical oracle of the B200 model step (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module, and only as the checker.  The product path never calls it.

Parity status: *unpinned* for model arithmetic.  The reference (interceptsim)
has no model -- its model step is the analytic CostModel::t_fwd
(proj/include/interceptsim/cost_model.hpp:33-37, called at
proj/src/engine.cpp:460) -- so there are no logits or token ids to pin against.
This module restates the forward the executor runs with the same fp16
rounding points (GEMM inputs, q/k/v, attention output, KV cache, fp32
residual stream), and consumes the very BatchPlans the scheduler emits.
Between rounding points it accumulates in float64 by default (the parity
reference: the exact value each fp16 rounding point rounds; two fp32
implementations with different summation orders land on different sides of
an fp16 rounding boundary about twice as often as either does against the
exact value), or in float32 (precision="f32": the bench's CPU timing sample,
a plain fp32 CPU implementation).  The *scheduling* that
produces those plans is pinned bit-exactly against the reference itself
(oracle/_ref, see tests/test_sched_parity.py).

Semantics restated:
  * token ids: synthetic ids for prompt / API-returned positions are
    mix64(mix64(token_seed + C*(rid+1)) + pos) % V (same hash as the device);
    a sampling row at position p writes the greedy id for position p+1;
  * a row at position p attends over keys [0, p] of its request (causal);
  * KV of a position is written once per (re)computation; swaps move bytes.
"""
from __future__ import annotations

import math

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * np.uint64(0xBF58476D1CE4E5B9)
        z = z ^ (z >> np.uint64(27))
        z = z * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def synth_weight(seed: int, tensor_id: int, count: int) -> np.ndarray:
    """Device init kernel restated: exec/common.cuh synth_weight (element-wise,
    so large tensors are hashed in pieces on the thread pool)."""
    with np.errstate(over="ignore"):
        base = mix64(np.uint64((seed + 0x9E3779B97F4A7C15 * (tensor_id + 1)) & 0xFFFFFFFFFFFFFFFF))
    out = np.empty(count, np.float32)

    def piece(lo, hi=None):
        hi = min(count, lo + _PIECE)
        with np.errstate(over="ignore"):
            h = mix64(base + np.arange(lo, hi, dtype=np.uint64))
        u24 = (h >> np.uint64(40)).astype(np.float32)
        out[lo:hi] = (u24 * np.float32(1.1920928955078125e-07) - np.float32(1.0)) * np.float32(0.034641016)

    starts = range(0, count, _PIECE)
    if count > _PIECE:
        list(_pool().map(piece, starts))
    else:
        for lo in starts:
            piece(lo)
    return out


_PIECE = 1 << 22


def synth_token(seed: int, rid: int, pos, vocab: int):
    with np.errstate(over="ignore"):
        base = mix64(np.uint64((seed + 0xD1B54A32D192ED03 * (rid + 1)) & 0xFFFFFFFFFFFFFFFF))
        return (mix64(base + np.asarray(pos, dtype=np.uint64)) % np.uint64(vocab)).astype(np.int64)


def r16(x: np.ndarray) -> np.ndarray:
    """Round to IEEE fp16 (nearest-even; float64 inputs round directly, no
    double rounding), returned as float32: the executor's storage type for
    weights, activations and the KV cache."""
    return np.asarray(x).astype(np.float16).astype(np.float32)


PRESETS = {
    "tiny": dict(family="gpt2", layers=2, d_model=256, heads=4, ffn=1024, vocab=4096, rotary_dim=0),
    "gptj-6b": dict(family="gptj", layers=28, d_model=4096, heads=16, ffn=16384, vocab=50400, rotary_dim=64),
    "vicuna-13b": dict(family="llama", layers=40, d_model=5120, heads=40, ffn=13824, vocab=32000, rotary_dim=128),
}


class ModelOracle:
    """Weights + forward of one model (exec/model.cpp layout_weights order)."""

    def __init__(self, spec: dict, fast_random: bool = False, precision: str = "f64"):
        # fast_random: plain numpy normals instead of the device hash, for the
        # bench's CPU timing sample only (values then differ from the device).
        # precision: accumulation type between the fp16 rounding points.
        self.fast_random = fast_random
        self.A = {"f64": np.float64, "f32": np.float32}[precision]
        s = dict(PRESETS[spec.get("preset", "tiny")])
        s.update({k: v for k, v in spec.items() if k != "preset"})
        s.setdefault("max_pos", 4160)
        s.setdefault("weight_seed", 1234)
        s.setdefault("token_seed", 99)
        s.setdefault("norm_eps", 1e-6 if s["family"] == "llama" else 1e-5)
        self.s = s
        self.fam = s["family"]
        self.L, self.D, self.H, self.F, self.V = s["layers"], s["d_model"], s["heads"], s["ffn"], s["vocab"]
        self.hd = self.D // self.H
        self.rot = s["rotary_dim"]
        self._next_id = 0
        D, F, V = self.D, self.F, self.V
        bias = self.fam != "llama"
        self.tok_emb = self._put(V * D, 0).reshape(V, D)
        self.pos_emb = self._put(s["max_pos"] * D, 0).reshape(s["max_pos"], D) if self.fam == "gpt2" else None
        self.layers = []
        for _ in range(self.L):
            lw = {}
            lw["ln1_g"] = self._put(D, 1)
            lw["ln1_b"] = self._put(D, 2) if bias else None
            if self.fam != "gptj":
                lw["ln2_g"] = self._put(D, 1)
                lw["ln2_b"] = self._put(D, 2) if bias else None
            lw["w_qkv"] = self._put(3 * D * D, 0).reshape(3 * D, D)
            lw["b_qkv"] = self._put(3 * D, 0) if self.fam == "gpt2" else None
            lw["w_o"] = self._put(D * D, 0).reshape(D, D)
            lw["b_o"] = self._put(D, 0) if self.fam == "gpt2" else None
            fin = 2 * F if self.fam == "llama" else F
            lw["w_in"] = self._put(fin * D, 0).reshape(fin, D)
            lw["b_in"] = self._put(F, 0) if bias else None
            lw["w_out"] = self._put(D * F, 0).reshape(D, F)
            lw["b_out"] = self._put(D, 0) if bias else None
            self.layers.append(lw)
        self.lnf_g = self._put(D, 1)
        self.lnf_b = self._put(D, 2) if bias else None
        self.lm_w = self._put(V * D, 0).reshape(V, D)
        self.lm_b = self._put(V, 0) if self.fam == "gptj" else None
        if self.rot:
            half = self.rot // 2
            pos = np.arange(s["max_pos"], dtype=np.float64)[:, None]
            inv = np.array([math.pow(10000.0, -2.0 * i / self.rot) for i in range(half)])
            ang = pos * inv[None, :]
            self.cos = np.cos(ang).astype(np.float32)
            self.sin = np.sin(ang).astype(np.float32)

    def _put(self, count: int, kind: int) -> np.ndarray:
        tid = self._next_id
        self._next_id += 1
        if kind == 1:
            return np.ones(count, self.A)
        if kind == 2:
            return np.zeros(count, self.A)
        if self.fast_random:
            w = np.random.default_rng(tid).standard_normal(count, dtype=np.float32) * np.float32(0.02)
        else:
            w = r16(synth_weight(self.s["weight_seed"], tid, count))
        return w if self.A is np.float32 else w.astype(self.A)

    # ---- pieces ---------------------------------------------------------------
    def norm(self, x, g, b):
        A = self.A
        x = np.asarray(x, A)
        eps = A(np.float32(self.s["norm_eps"]))
        if self.fam == "llama":
            var = np.mean(x * x, axis=-1, keepdims=True, dtype=A)
            y = x * (A(1.0) / np.sqrt(var + eps)) * g
        else:
            mu = np.mean(x, axis=-1, keepdims=True, dtype=A)
            d = x - mu
            var = np.mean(d * d, axis=-1, keepdims=True, dtype=A)
            y = d * (A(1.0) / np.sqrt(var + eps)) * g
            if b is not None:
                y = y + b
        return r16(y)

    def lin(self, x, w, b=None):
        y = np.asarray(x, self.A) @ w.T
        return y + b if b is not None else y

    def rope(self, t, pos):
        """t: [n, H, hd] fp16-valued float32; rotated in float32, re-rounded."""
        if not self.rot:
            return t
        half = self.rot // 2
        c = self.cos[pos][:, None, :].astype(self.A)
        s = self.sin[pos][:, None, :].astype(self.A)
        t = t.astype(self.A)
        if self.fam == "gptj":
            a, b = t[..., 0:self.rot:2].copy(), t[..., 1:self.rot:2].copy()
            t[..., 0:self.rot:2] = a * c - b * s
            t[..., 1:self.rot:2] = b * c + a * s
        else:
            a, b = t[..., :half].copy(), t[..., half:self.rot].copy()
            t[..., :half] = a * c - b * s
            t[..., half:self.rot] = b * c + a * s
        return r16(t)


class ForwardOracle:
    """Replays BatchPlans (dicts from the scheduler's plan log) on the CPU."""

    def __init__(self, model_spec: dict, fast_random: bool = False, precision: str = "f64"):
        self.m = ModelOracle(model_spec, fast_random, precision)
        self.hist = {}     # rid -> int64[ctx]
        self.kv = {}       # rid -> float32[L, 2, H, cap, hd] (fp16 values; head-major for batched matmuls)

    def _ensure(self, rid, upto):
        L, H, hd = self.m.L, self.m.H, self.m.hd
        if rid not in self.hist:
            self.hist[rid] = np.zeros(max(64, upto + 1), np.int64)
            self.kv[rid] = np.zeros((L, 2, H, max(64, upto), hd), self.m.A)
        if self.hist[rid].shape[0] < upto + 1:
            h = np.zeros(max(upto + 1, 2 * self.hist[rid].shape[0]), np.int64)
            h[: self.hist[rid].shape[0]] = self.hist[rid]
            self.hist[rid] = h
        cap = self.kv[rid].shape[3]
        if cap < upto:
            k = np.zeros((L, 2, H, max(upto, 2 * cap), hd), self.m.A)
            k[:, :, :, :cap] = self.kv[rid]
            self.kv[rid] = k

    def step(self, plan: dict, teacher_tokens=None) -> dict:
        """Run one plan; returns {"logits": [S, V], "tokens": [S], "margin": [S]}.

        teacher_tokens: tokens the device sampled (one per sampling span, in
        span order); they overwrite the oracle's own ids in the history so
        both sides continue from identical inputs (ties stay harmless)."""
        m = self.m
        D, H, hd, V = m.D, m.H, m.hd, m.V
        rows_rid, rows_pos, sample_rows, spans = [], [], [], []
        for (rid, pos, count, kind, sample) in plan["spans"]:
            self._ensure(rid, pos + count + 1)
            r0 = len(rows_rid)
            for k in range(count):
                rows_rid.append(rid)
                rows_pos.append(pos + k)
            if kind == 1:  # fresh: synthetic ids
                self.hist[rid][pos:pos + count] = synth_token(m.s["token_seed"], rid, np.arange(pos, pos + count), V)
            spans.append((rid, pos, count, r0))
            if sample:
                sample_rows.append(r0 + count - 1)
        out = self._forward(plan, rows_rid, rows_pos, sample_rows, spans, teacher_tokens)
        for (rid, kind, phase, lo, hi) in plan["ops"]:
            if kind == 5:  # release (phase 1: after this iteration's forward)
                self.hist.pop(rid, None)
                self.kv.pop(rid, None)
        return out

    def _forward_only(self, plan: dict) -> dict:
        """Timing entry for the bench's CPU baseline (no teacher forcing)."""
        return self.step(plan)

    def _forward(self, plan, rows_rid, rows_pos, sample_rows, spans, teacher_tokens):
        m = self.m
        D, H, hd, V = m.D, m.H, m.hd, m.V
        n = len(rows_rid)
        if n == 0:
            return {"logits": np.zeros((0, V), np.float32), "tokens": [], "margin": []}
        pos_arr = np.array(rows_pos)
        toks = np.array([self.hist[r][p] for r, p in zip(rows_rid, rows_pos)])
        x = m.tok_emb[toks].astype(np.float32)
        if m.pos_emb is not None:
            x = (x + m.pos_emb[pos_arr]).astype(np.float32)
        A = m.A
        scale = A(np.float32(1.0 / math.sqrt(hd)))
        for li, lw in enumerate(m.layers):
            xn = m.norm(x, lw["ln1_g"], lw["ln1_b"])
            qkv = r16(m.lin(xn, lw["w_qkv"], lw["b_qkv"]))
            q = m.rope(qkv[:, :D].reshape(n, H, hd), pos_arr)
            k = m.rope(qkv[:, D:2 * D].reshape(n, H, hd), pos_arr)
            v = qkv[:, 2 * D:].reshape(n, H, hd)
            for (rid, pos, count, r0) in spans:
                self.kv[rid][li, 0, :, pos:pos + count] = k[r0:r0 + count].transpose(1, 0, 2)
                self.kv[rid][li, 1, :, pos:pos + count] = v[r0:r0 + count].transpose(1, 0, 2)
            attn = np.zeros((n, D), np.float32)

            def attend(span, li=li, q=q, attn=attn):
                rid, pos, count, r0 = span
                K = self.kv[rid][li, 0, :, : pos + count]      # [H, k, hd]
                Vv = self.kv[rid][li, 1, :, : pos + count]
                qq = q[r0:r0 + count].transpose(1, 0, 2)        # [H, c, hd]
                s = np.matmul(qq, K.transpose(0, 2, 1)) * scale  # [H, c, k]
                if count > 1:
                    kpos = np.arange(pos + count)
                    qpos = pos + np.arange(count)
                    s = np.where(kpos[None, None, :] <= qpos[None, :, None], s, -np.inf)
                s = s - s.max(axis=-1, keepdims=True)
                p = np.exp(s)
                p = p / p.sum(axis=-1, keepdims=True)
                o = np.matmul(p, Vv)                             # [H, c, hd]
                attn[r0:r0 + count] = o.transpose(1, 0, 2).reshape(count, D)

            # Spans are independent (each writes its own rows): numpy releases
            # the GIL, so many small (decode) spans use all host cores.
            if len(spans) > 4:
                list(_pool().map(attend, spans))
            else:
                for sp in spans:
                    attend(sp)
            attn = r16(attn)
            # x is the executor's fp32 residual stream: rounded to fp32 after every add.
            if m.fam == "gptj":
                x = (x + m.lin(attn, lw["w_o"], lw["b_o"])).astype(np.float32)
                u = m.lin(xn, lw["w_in"], lw["b_in"])
                u = r16(_gelu(u))
                x = (x + m.lin(u, lw["w_out"], lw["b_out"])).astype(np.float32)
            else:
                x = (x + m.lin(attn, lw["w_o"], lw["b_o"])).astype(np.float32)
                xn2 = m.norm(x, lw["ln2_g"], lw["ln2_b"])
                if m.fam == "llama":
                    gu = m.lin(xn2, lw["w_in"])
                    g, u = gu[:, 0::2], gu[:, 1::2]
                    h = r16((g / (A(1) + np.exp(-g))) * u)
                else:
                    h = r16(_gelu(m.lin(xn2, lw["w_in"], lw["b_in"])))
                x = (x + m.lin(h, lw["w_out"], lw["b_out"])).astype(np.float32)
        if not sample_rows:
            return {"logits": np.zeros((0, V), np.float32), "tokens": [], "margin": []}
        xs = m.norm(x[sample_rows], m.lnf_g, m.lnf_b)
        logits = m.lin(xs, m.lm_w, m.lm_b).astype(np.float32)
        top2 = np.sort(logits, axis=-1)[:, -2:]
        toks_out = np.argmax(logits, axis=-1)
        margin = top2[:, 1] - top2[:, 0]
        chosen = teacher_tokens if teacher_tokens is not None else toks_out
        for i, r in enumerate(sample_rows):
            self.hist[rows_rid[r]][rows_pos[r] + 1] = int(chosen[i])
        return {"logits": logits, "tokens": toks_out.tolist(), "margin": margin.tolist()}


_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        import os
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=os.cpu_count() or 1)
    return _POOL


def _gelu(v: np.ndarray) -> np.ndarray:
    A = v.dtype.type
    c0, c1 = A(np.float32(0.7978845608028654)), A(np.float32(0.044715))
    return A(0.5) * v * (A(1.0) + np.tanh(c0 * (v + c1 * v * v * v)))
