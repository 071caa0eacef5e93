#!/usr/bin/env python3
"""Benchmark of the B200 InferCept serving hot path (driver contract).

Workload (BASELINE.json configs[1]): a GPT-J-6B-shaped
random-init model serving the Math/QA/Chatbot API-augmented trace (2000
requests @3/s, seed 11) under InferCept's min-waste policy (reference cost
model defaults, M = 458,752 B/token, 150 GB GPU KV pool, 50 GB/s link).  A
"step" is one scheduler iteration: the C++ scheduler forms the batch (decode
rows + API-return / prefill / recompute chunks + budgeted swaps) and the
executor runs the model step on the paged KV cache.

The trace is first fast-forwarded (untimed) to steady state, then W warm-up
iterations, then exactly K timed iterations.  `value` = requests completed in
the timed window / device seconds (CUDA events on the executor's stream);
`e2e` = the same through the public C ABI session with host wall clock,
including each step's plan H2D upload from pinned memory and the D2H read of
the sampled token ids.  N > 1 (torchrun): request-sharded replicas (id mod N),
one per GPU, no collective on the data path; value = sum over ranks / max time.

--impl reference: the reference's CPU path of this step on the host cores:
the reference scheduler (oracle/_ref, compiled from /root/reference) plus the
CPU oracle port of the model step (numpy; bounded sample, extrapolated).
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
GPTJ_M = 458752
LINK = 50e9
WORKLOAD = dict(classes=[{"name": "Math"}, {"name": "QA"}, {"name": "Chatbot"}], request_count=2000,
                arrival_rate=3.0, seed=11)
COST = dict(mem_per_token=GPTJ_M, gpu_kv_capacity=150e9, cpu_kv_capacity=128e9, swap_per_token=GPTJ_M / LINK)
WORKLOAD_NAME = ("C1: GPT-J-6B-shaped random-init fp16 model, Math/QA/Chatbot API trace (2000 req @3/s, seed 11), "
                 "InferCept min-waste policy, reference cost-model defaults, 150 GB KV pool")


def k1_traffic():
    """ncu-measured DRAM bytes of one K1 launch vs its algorithmic bytes
    (profiles/k1_traffic.json, written by tools/ncu_traffic.py)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "k1_traffic.json")))
    except Exception:
        return None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def loop():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        sm = sorted(float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples if len(s) >= 7 for i in range(4) if s[3 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def workload_for(world):
    """The trace the N replicas serve: 2000*N requests at 3*N/s (same class mix
    and seed), so each replica's id-mod-N shard is statistically the C1 trace:
    per-GPU work is fixed as N grows (weak scaling)."""
    if world == 1:
        return WORKLOAD
    return dict(WORKLOAD, request_count=WORKLOAD["request_count"] * world,
                arrival_rate=WORKLOAD["arrival_rate"] * world)


def shard_trace(ib, world, rank, tmpdir):
    trace = ib.Trace.generate(workload_for(world))
    if world == 1:
        return trace
    full = os.path.join(tmpdir, "full.jsonl")
    trace.save(full)
    lines = open(full).read().splitlines()
    out = os.path.join(tmpdir, f"shard{rank}.jsonl")
    with open(out, "w") as f:
        f.write(lines[0] + "\n")
        for line in lines[1:]:
            if json.loads(line)["id"] % world == rank:
                f.write(line + "\n")
    return ib.Trace.load(out)


def gpu_pools(host_gb, gpu_blocks=0):
    blocks = gpu_blocks or int(COST["gpu_kv_capacity"] // (16 * GPTJ_M)) + 512
    return dict(gpu_blocks=blocks, host_bytes=int(host_gb * 1e9), max_requests=1024, max_rows=4096, timing=True,
                stage_tokens=1024, swap_slots=10)


def cpu_forward_sample(plans, n_plans=3):
    """Time the CPU oracle port of the GPT-J-shaped model step on plans taken
    from the timed window: 1- and 2-layer variants give the per-layer cost,
    extrapolated to 28 layers.  KV contents are synthetic (timing only)."""
    import numpy as np
    from oracle.forward import ForwardOracle

    def timed(layers):
        fo = ForwardOracle({"preset": "gptj-6b", "layers": layers, "max_pos": 4160}, fast_random=True)
        for pj in plans[:n_plans]:  # materialize contexts
            for (rid, pos, count, kind, sample) in pj["spans"]:
                fo._ensure(rid, pos + count + 1)
        fo._forward_only(plans[0])  # untimed warm-up (first-touch of weights, BLAS threads)
        t = time.perf_counter()
        for pj in plans[:n_plans]:
            fo._forward_only(pj)
        return (time.perf_counter() - t) / n_plans

    t1 = timed(1)
    t2 = timed(2)
    per_iter = t1 + 27 * max(t2 - t1, 0.0)
    return per_iter, dict(t1=t1, t2=t2)


def measure_link(torch, mb=512, reps=3):
    """Pinned host <-> device copy bandwidth on this box (the swap roofline)."""
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        with torch.cuda.stream(s):
            fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                fn()
            e1.record(s)
        torch.cuda.synchronize()
        out[name] = reps * n / (e0.elapsed_time(e1) / 1e3) / 1e9
    del h, d
    return out


def run_b200(args):
    import torch
    import paper_2402_01869_b200 as ib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    link = measure_link(torch)
    tmp = tempfile.mkdtemp()
    trace = shard_trace(ib, world, rank, tmp)
    cost = ib.CostModel.from_json(COST)
    ex = ib.Executor({"preset": "gptj-6b"}, local, gpu_pools(args.host_gb, args.gpu_blocks))
    sess = ib.Session(trace, cost, {"policy": "infercept", "estimator": "oracle"}, ex)

    # Fast-forward to steady state, then warm up.
    sess.step(args.fast_forward)
    sess.step(args.warmup)
    ex.sync()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    c0, s0 = sess.counters(), ex.stats()
    clocks = ClockSampler(local)
    clocks.start()
    profiling = os.environ.get("BENCH_PROFILE") == "1"
    if profiling:  # ncu --profile-from-start off: capture only the timed window
        torch.cuda.profiler.start()
    wall0 = time.perf_counter()
    ex.mark(0)
    done, finished = sess.step(args.steps)
    ex.mark(1)
    ex.sync()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if profiling:
        torch.cuda.profiler.stop()
    dev_ms = ex.elapsed_ms()
    clk = clocks.stop()
    c1, s1 = sess.counters(), ex.stats()
    if done != args.steps:
        raise SystemExit(f"trace ended after {done} of {args.steps} timed iterations; lower --fast-forward")

    completed = c1["completed"] - c0["completed"]
    decode = c1["decode_rows"] - c0["decode_rows"]
    swapped = c1["swapped_tokens"] - c0["swapped_tokens"]
    local_stats = dict(dev_s=dev_ms / 1e3, wall_s=wall, completed=completed, decode=decode, swapped=swapped,
                       k1_ms=s1["k1_ms"] - s0["k1_ms"], k1_bytes=s1["k1_bytes"] - s0["k1_bytes"],
                       k1_launches=s1["k1_timed_launches"] - s0["k1_timed_launches"],
                       swap_ms=s1["swap_ms"] - s0["swap_ms"], swap_bytes=s1["swap_bytes_timed"] - s0["swap_bytes_timed"],
                       fwd_tok=s1["swap_in_forwarded_tokens"] - s0["swap_in_forwarded_tokens"],
                       launches=s1["kernel_launches"] - s0["kernel_launches"],
                       h2d=s1["h2d_bytes"] - s0["h2d_bytes"], d2h=s1["d2h_bytes"] - s0["d2h_bytes"])
    if dist:
        gathered = [None] * world
        dist.all_gather_object(gathered, local_stats)
    else:
        gathered = [local_stats]
    if rank != 0:
        dist.destroy_process_group()
        return
    dev_s = max(g["dev_s"] for g in gathered)
    wall_s = max(g["wall_s"] for g in gathered)
    tot = {k: sum(g[k] for g in gathered) for k in ("completed", "decode", "swapped", "launches", "h2d", "d2h",
                                                    "fwd_tok")}
    pk = peaks()
    k1_gbs = local_stats["k1_bytes"] / (local_stats["k1_ms"] / 1e3) / 1e9 if local_stats["k1_ms"] else None
    swap_gbs = local_stats["swap_bytes"] / (local_stats["swap_ms"] / 1e3) / 1e9 if local_stats["swap_ms"] else None
    line = {
        "metric": METRIC,
        "value": tot["completed"] / dev_s,
        "unit": "req/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_s * 1e3 / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f16 (fp32 accumulate)",
        "data": "synthetic (generated API trace, random-init weights, synthetic token ids)",
        "config": {"workload": WORKLOAD_NAME, "window_iterations": [args.fast_forward + args.warmup + 1,
                                                                    args.fast_forward + args.warmup + args.steps],
                   "fast_forward_untimed": args.fast_forward,
                   "parallelism": f"replicas{world}: one engine + KV pool per GPU serving request ids = rank mod N of a "
                                  f"{workload_for(world)['request_count']}-request trace at "
                                  f"{workload_for(world)['arrival_rate']:g}/s (per-GPU load = C1)",
                   "l2": "inputs larger than L2 (KV pool ~154 GB; ~15 GB of KV read per iteration)"},
        "decode_tok_s": tot["decode"] / dev_s,
        "completed_in_window": tot["completed"],
        "swap_gbs_achieved": swap_gbs,
        "swap_tokens_in_window": tot["swapped"],
        "swap_in_forwarded_tokens": tot["fwd_tok"],
        "host_pool_peak_gb": s1["host_pool_peak"] / 1e9,
        "swap_roofline": {"bound": "host link", "achieved": swap_gbs, "unit": "GB/s",
                          "peak": (link["h2d"] + link["d2h"]) / 2, "peak_h2d": link["h2d"], "peak_d2h": link["d2h"],
                          "frac": swap_gbs / ((link["h2d"] + link["d2h"]) / 2) if swap_gbs else None,
                          "peak_source": "pinned 512 MiB copies measured by bench.py on this box",
                          "note": "achieved = swapped bytes / time of each PCIe batch on the copy streams; "
                                  "swap-ins forwarded from swap-out staging do not cross the link"},
        "roofline": {"bound": "hbm", "kernel": "K1 paged decode attention (middle layer, every timed iteration)",
                     "achieved": k1_gbs, "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                     "frac": (k1_gbs / pk["hbm_gbs"]) if k1_gbs and pk.get("hbm_gbs") else None,
                     "traffic": (k1_traffic() or {}).get("dram_bytes_per_launch"),
                     "traffic_algorithmic_bytes": (k1_traffic() or {}).get("algorithmic_bytes_per_launch"),
                     "traffic_source": (k1_traffic() or {}).get("source"),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"},
        "e2e": {"value": tot["completed"] / wall_s, "unit": "req/s",
                "h2d_bytes_per_step": tot["h2d"] / args.steps / world,
                "d2h_bytes_per_step": tot["d2h"] / args.steps / world},
        "gpu_launches": tot["launches"],
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(ib, args, per_iter_completed=tot["completed"] / args.steps)
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def window_plans(ib, args, n):
    """Plans of the first n timed iterations (scheduler only, CPU)."""
    tmp = tempfile.mkdtemp()
    path = os.path.join(tmp, "plans.jsonl")
    sess2 = ib.Session(ib.Trace.generate(WORKLOAD), ib.CostModel.from_json(COST),
                       {"policy": "infercept", "estimator": "oracle", "plan_log": path})
    sess2.step(args.fast_forward + args.warmup + n)
    del sess2
    lines = open(path).read().splitlines()
    return [json.loads(l) for l in lines[-n:]]


def cpu_baseline(ib, args, per_iter_completed):
    plans = window_plans(ib, args, 3)
    per_iter, detail = cpu_forward_sample(plans, 3)
    return {"value": per_iter_completed / per_iter, "unit": "req/s", "cores": os.cpu_count(), "kind": "port",
            "sample": (f"numpy fp32 oracle forward of 3 timed-window iterations of the GPT-J-shaped step "
                       f"(1- and 2-layer runs {detail['t1']:.2f}s/{detail['t2']:.2f}s, extrapolated to 28 layers: "
                       f"{per_iter:.2f} s/iteration); KV contents synthetic"),
            "s_per_iteration": per_iter}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import ctypes
    import paper_2402_01869_b200 as ib
    ref = os.path.join(ROOT, "oracle", "_ref", "libinterceptsim.so")
    sched_us = None
    if os.path.exists(ref):
        L = ctypes.CDLL(ref)
        L.isim_trace_generate.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.isim_model_from_json.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.isim_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.isim_result_metric.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_double)]
        t, m, r = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        L.isim_trace_generate(json.dumps(WORKLOAD).encode(), ctypes.byref(t))
        L.isim_model_from_json(json.dumps(COST).encode(), ctypes.byref(m))
        t0 = time.perf_counter()
        L.isim_run(t, m, b'{"policy":"infercept","estimator":"oracle"}', ctypes.byref(r))
        el = time.perf_counter() - t0
        it = ctypes.c_double()
        L.isim_result_metric(r, b"iterations", ctypes.byref(it))
        sched_us = el / it.value * 1e6
    plans = window_plans(ib, args, 3)
    # completions per iteration in the window, from the scheduler
    sess = ib.Session(ib.Trace.generate(WORKLOAD), ib.CostModel.from_json(COST), {"policy": "infercept"})
    sess.step(args.fast_forward + args.warmup)
    c0 = sess.counters()
    # Completions per iteration of the schedule (cheap: scheduler only), over
    # at least 1000 iterations so a short --steps still sees completions.
    n_sched = max(args.steps, 1000)
    sess.step(n_sched)
    c1 = sess.counters()
    per_iter_completed = (c1["completed"] - c0["completed"]) / n_sched
    per_iter, detail = cpu_forward_sample(plans, 3)
    per_iter += (sched_us or 0.0) / 1e6
    value = per_iter_completed / per_iter
    line = {
        "metric": METRIC, "value": value, "unit": "req/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_iter * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "fp32 (numpy)", "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD_NAME, "host": "rank 0 only, host cores (no GPU used)"},
        "cpu_baseline": {"value": value, "unit": "req/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": (f"reference scheduler (oracle/_ref, {sched_us:.2f} us/iteration, whole trace) + "
                                    f"numpy oracle forward of 3 window iterations (1/2-layer runs "
                                    f"{detail['t1']:.2f}/{detail['t2']:.2f} s, extrapolated to 28 layers)")
                         if sched_us else "numpy oracle forward sample"},
        "e2e": {"value": value, "unit": "req/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--fast-forward", type=int, default=3000)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--host-gb", type=float, default=48.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gpu-blocks", type=int, default=0,
                    help="override the KV pool size (profiling runs only; the scheduler's capacity is unchanged)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
