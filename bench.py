#!/usr/bin/env python3
"""Benchmark of the B200 InferCept serving hot path (driver contract).

Workload (BASELINE.json configs[4], SURVEY §8d C4 -- the largest single-GPU
configuration and the one the scaling run shards): a Vicuna-13B-shaped
random-init model serving a fixed 4000-request API-augmented trace (all six
Table-1 classes, seed 23, arrivals at 1000/s: saturating) under InferCept's
min-waste policy (reference cost model defaults, M = 819,200 B/token, 140 GB
GPU / 64 GB CPU KV ledger per replica, 50 GB/s link).  With N GPUs, rank r
serves the requests with id mod N == r at their original arrival times (its
own engine, KV pool and pinned host pool; no collective on the data path):
strong scaling of one fixed trace (reference concurrency
contract proj/include/interceptsim.h:10-11).

A "step" is one scheduler iteration: the C++ scheduler (bit-exact with the
reference engine, proj/src/engine.cpp:282-548) forms the batch and the
executor runs the model step at the engine.cpp:460 hook on the paged KV
cache.

Estimator (identical in both arms).  The reference's throughput is
completed / makespan (proj/src/metrics.cpp:41-50).  A replica's schedule is
deterministic, so its completions C and iteration count I are known from a
scheduler-only run (cheap, CPU); what is measured is the time per iteration.
The K timed iterations are spread over n windows centred on evenly spaced
points of the replica's schedule (a stratified sample of the whole replay;
each window is reached by a scheduler-only fast-forward, then W untimed
warm-up iterations on the GPU, then its timed iterations between a barrier
and device syncs).  value = sum_r C_r / max_r (I_r * mean device s/iteration
of rank r); e2e the same with host wall seconds through the public C ABI
session (plan upload from pinned memory and sampled-id read-back included).

--impl reference: the reference's CPU path of the same schedule on this host:
the reference engine (oracle/_ref, compiled from /root/reference) runs the
whole trace; its event log with ledger snapshots gives each iteration's batch
(oracle/ref_plans.py, no product code loaded); the numpy fp32 oracle forward
(oracle/forward.py) of the same timed iterations as the B200 arm, each timed
with all host threads (1- and 2-layer runs, extrapolated to the model's
depth), plus the reference scheduler's own seconds per iteration, is its time
per iteration.  --full-trace (C0) times every iteration at full depth instead.
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
LINK = 50e9
ALL6 = [{"name": c} for c in ["Math", "QA", "VE", "Chatbot", "Image", "TTS"]]
GPTJ_M, M13 = 458752, 819200
RUN = {"policy": "infercept", "estimator": "oracle"}

# SURVEY §8d configurations.
CONFIGS = {
    "C0": dict(l2="inputs fit in L2 (64 MiB KV pool): the tiny CPU-runnable case, not a headline", model={"preset": "tiny"}, layers=2, M=4096,
               workload=dict(classes=[{"name": c} for c in ["Math", "QA", "VE", "Chatbot", "Image", "TTS"]],
                             request_count=64, arrival_rate=1.0, seed=1, max_seq_len=4096),
               cost=dict(t0=2e-3, slope_below=1e-6, slope_above=1e-5, saturation_point=512, mem_per_token=4096,
                         gpu_kv_capacity=16384 * 4096, cpu_kv_capacity=4 * 16384 * 4096, swap_per_token=8.192e-6,
                         block_size=16),
               slack_blocks=512,
               name="C0: tiny GPT (2 layers, d=256, 4 heads, fp32 cost model M=4096), 64-request trace of all six "
                    "API classes (seed 1), InferCept min-waste policy, 64 MiB GPU / 256 MiB CPU KV ledger"),
    "C1": dict(l2="inputs larger than L2 (150 GB KV pool, ~15 GB of KV read per iteration)", model={"preset": "gptj-6b"}, layers=28, M=GPTJ_M,
               workload=dict(classes=[{"name": "Math"}, {"name": "QA"}, {"name": "Chatbot"}], request_count=2000,
                             arrival_rate=3.0, seed=11),
               cost=dict(mem_per_token=GPTJ_M, gpu_kv_capacity=150e9, cpu_kv_capacity=128e9,
                         swap_per_token=GPTJ_M / LINK),
               slack_blocks=512,
               name="C1: GPT-J-6B-shaped random-init fp16 model, Math/QA/Chatbot API trace (2000 req @3/s, seed 11), "
                    "InferCept min-waste policy, reference cost-model defaults, 150 GB GPU / 128 GB CPU KV ledger"),
    "C2": dict(l2="inputs larger than L2 (120 GB KV pool)", model={"preset": "vicuna-13b"}, layers=40, M=M13,
               workload=dict(classes=[{"name": "Chatbot"}, {"name": "VE"}], request_count=1000, arrival_rate=2.0,
                             seed=13),
               cost=dict(mem_per_token=M13, gpu_kv_capacity=120e9, cpu_kv_capacity=96e9, swap_per_token=M13 / LINK),
               slack_blocks=512,
               name="C2: Vicuna-13B-shaped model, Chatbot + VE trace (1000 req @2/s, seed 13), 120 GB / 96 GB ledger: "
                    "chunked swap under the swap budget"),
    "C3": dict(l2="inputs larger than L2 (40 GB KV pool, 3k-token contexts)", model={"preset": "vicuna-13b"}, layers=40, M=M13,
               workload=dict(classes=[{"name": "QA", "context_mean": 3000.0, "context_var": 200.0 ** 2}],
                             request_count=1000, arrival_rate=2.0, seed=17),
               cost=dict(mem_per_token=M13, gpu_kv_capacity=40e9, cpu_kv_capacity=128e9, swap_per_token=M13 / LINK),
               slack_blocks=512,
               name="C3: Vicuna-13B-shaped model, QA-shaped calls over 3000-token contexts (1000 req @2/s, seed 17), "
                    "40 GB GPU ledger: Discard-heavy chunked recompute"),
    "C4": dict(l2="inputs larger than L2 (140 GB KV pool, tens of GB of KV read per iteration)", model={"preset": "vicuna-13b"}, layers=40, M=M13,
               workload=dict(classes=ALL6, request_count=4000, arrival_rate=1000.0, seed=23),
               cost=dict(mem_per_token=M13, gpu_kv_capacity=140e9, cpu_kv_capacity=64e9, swap_per_token=M13 / LINK),
               slack_blocks=64,  # 140 GB pool + 26 GB of weights: little room for slack
               name="C4: Vicuna-13B-shaped random-init fp16 model, fixed 4000-request trace of all six API classes "
                    "(seed 23, arrivals 1000/s), InferCept min-waste policy, reference cost-model defaults, "
                    "140 GB GPU / 64 GB CPU KV ledger per replica, requests sharded id mod N"),
}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}


def k1_traffic():
    """ncu-measured DRAM bytes of one K1 launch vs its algorithmic bytes
    (profiles/k1_traffic.json, written by tools/ncu_traffic.py)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "k1_traffic.json")))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled only while `active`
    (the timed windows)."""

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.active = False
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def loop():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                if self.active:
                    try:
                        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                             timeout=5).stdout.strip()
                        if self.active:
                            self.samples.append([x.strip() for x in out.split(",")])
                    except Exception:
                        pass
                self._stop.wait(0.1)
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


def shard_trace(ib, cfg, world, rank, tmpdir):
    """Requests with id mod world == rank, original arrival times."""
    trace = ib.Trace.generate(cfg["workload"])
    if world == 1:
        return trace
    full = os.path.join(tmpdir, "full.jsonl")
    trace.save(full)
    with open(full) as f:
        lines = f.read().splitlines()
    out = os.path.join(tmpdir, f"shard{rank}.jsonl")
    with open(out, "w") as f:
        f.write(lines[0] + "\n")
        for line in lines[1:]:
            if json.loads(line)["id"] % world == rank:
                f.write(line + "\n")
    return ib.Trace.load(out)


def windows(total_iters, steps, warmup, n_win):
    """[(first timed iteration index, timed count)]: n_win windows centred on
    evenly spaced points of the schedule, each preceded by `warmup`
    iterations, never overlapping (iteration indices are 0-based counts of
    iterations already run)."""
    n_win = max(1, min(n_win, steps))
    per = [steps // n_win + (1 if j < steps % n_win else 0) for j in range(n_win)]
    out, pos = [], 0
    for j in range(n_win):
        start = max(int((j + 0.5) * total_iters / n_win) - per[j] // 2, pos + warmup)
        out.append((start, per[j]))
        pos = start + per[j]
    if pos > total_iters:
        raise SystemExit(f"schedule has {total_iters} iterations: too short for {steps} timed + warm-up")
    return out


def default_windows(steps):
    return max(1, min(4, steps // 5))


def schedule_totals(ib, trace, cfg):
    """(iterations, completed) of the replica's whole schedule (scheduler only)."""
    s = ib.Session(trace, ib.CostModel.from_json(cfg["cost"]), RUN)
    it, fin = s.step(10 ** 9)
    assert fin
    return it, s.counters()["completed"]


def combine(gathered, steps):
    """Whole-job figures from the ranks' stats: (requests served by all
    ranks, [estimated device seconds of each rank's replay], [same, wall])."""
    done_all = sum(g["total_done"] for g in gathered)
    replay = [g["iters"] * g["dev_s"] / steps for g in gathered]
    replay_wall = [g["iters"] * g["wall_s"] / steps for g in gathered]
    return done_all, replay, replay_wall


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


def pools_for(cfg, host_gb, gpu_blocks=0):
    """Executor pools: the ledger's GPU capacity in 16-token blocks + slack
    (the Oracle estimator keeps every request's GPU positions a prefix, so the
    ledger's blocks suffice; the executor enforces it), the pinned host pool,
    the bench's staging ring, and the step-roofline peaks."""
    pk = peaks()
    blocks = gpu_blocks or int(cfg["cost"]["gpu_kv_capacity"] // (16 * cfg["M"])) + cfg["slack_blocks"]
    return dict(gpu_blocks=blocks, host_bytes=int(host_gb * 1e9), max_requests=1024, max_rows=4096, timing=True,
                stage_tokens=1024, swap_slots=10, roof_hbm_gbs=pk.get("hbm_gbs", 6526.0),
                roof_tflops=pk.get("bf16_tflops", 1662.0))


def host_pool_gb(cfg, world, override):
    """Pinned host pool per rank: the CPU ledger x 1.25 (extent rounding and
    staging) + 4 GB, capped at 3/4 of the host's available memory shared by
    the ranks on this node."""
    if override:
        return override
    want = cfg["cost"]["cpu_kv_capacity"] / 1e9 * 1.25 + 4.0
    try:
        with open("/proc/meminfo") as f:
            avail = next(int(l.split()[1]) for l in f if l.startswith("MemAvailable")) * 1024 / 1e9
        local = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        return min(want, 0.75 * avail / max(1, local))
    except Exception:
        return want


def run_b200(args):
    import torch
    import paper_2402_01869_b200 as ib

    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # BENCH_DEVICE pins every rank to one device (tests of the N > 1 plumbing
    # on a single GPU with a small config); normally rank = local GPU.
    local = int(os.environ.get("BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if "BENCH_DEVICE" in os.environ:  # ranks share one GPU: NCCL refuses duplicate devices
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    link = measure_link(torch)
    pk = peaks()
    tmp = tempfile.mkdtemp()
    trace = shard_trace(ib, cfg, world, rank, tmp)
    total_iters, total_done = schedule_totals(ib, trace, cfg)
    n_win = args.windows or default_windows(args.steps)
    wins = windows(total_iters, args.steps, args.warmup, n_win)

    ex = ib.Executor(cfg["model"], local, pools_for(cfg, host_pool_gb(cfg, world, args.host_gb), args.gpu_blocks))
    sess = ib.Session(trace, ib.CostModel.from_json(cfg["cost"]), RUN, ex)

    clocks = ClockSampler(local)
    clocks.start()
    keys = ("k1_ms", "k1_bytes", "k1_timed_launches", "swap_ms", "swap_bytes_timed", "swap_in_forwarded_tokens",
            "kernel_launches", "h2d_bytes", "d2h_bytes", "roof_s", "roof_bytes", "roof_flops", "chunk_rows",
            "swap_in_tokens", "swap_out_tokens")
    acc = {k: 0.0 for k in keys}
    acc.update(dev_s=0.0, wall_s=0.0, completed=0, decode=0, swapped=0)
    pos = 0
    win_ms = []  # device ms per iteration of each window
    profiling = os.environ.get("BENCH_PROFILE") == "1"
    for (start, count) in wins:
        if start - args.warmup > pos:
            done, _ = sess.fast_forward(start - args.warmup - pos)
            pos += done
        done, _ = sess.step(start - pos)  # warm-up on the GPU
        pos += done
        ex.sync()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        c0, s0 = sess.counters(), ex.stats()
        clocks.active = True
        if profiling:  # ncu --profile-from-start off: capture only the timed windows
            torch.cuda.profiler.start()
        wall0 = time.perf_counter()
        ex.mark(0)
        done, _ = sess.step(count)
        ex.mark(1)
        ex.sync()
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
        if profiling:
            torch.cuda.profiler.stop()
        clocks.active = False
        if done != count:
            raise SystemExit(f"schedule ended inside a timed window ({done} of {count})")
        pos += done
        c1, s1 = sess.counters(), ex.stats()
        win_ms.append(round(ex.elapsed_ms() / count, 3))
        acc["dev_s"] += ex.elapsed_ms() / 1e3
        acc["wall_s"] += wall
        acc["completed"] += c1["completed"] - c0["completed"]
        acc["decode"] += c1["decode_rows"] - c0["decode_rows"]
        acc["swapped"] += c1["swapped_tokens"] - c0["swapped_tokens"]
        for k in keys:
            acc[k] += s1[k] - s0[k]
    clk = clocks.stop()
    host_peak = ex.stats()["host_pool_peak"]
    local_stats = dict(acc, iters=total_iters, total_done=total_done, host_peak=host_peak, win_ms=win_ms)
    if dist:
        gathered = [None] * world
        dist.all_gather_object(gathered, local_stats)
    else:
        gathered = [local_stats]
    if rank != 0:
        dist.destroy_process_group()
        return
    K = args.steps
    done_all, replay, replay_wall = combine(gathered, K)
    dev_s_max = max(g["dev_s"] for g in gathered)
    tot = {k: sum(g[k] for g in gathered) for k in ("decode", "swapped", "kernel_launches", "h2d_bytes", "d2h_bytes",
                                                    "swap_in_forwarded_tokens", "completed")}
    me = gathered[0]
    k1_gbs = me["k1_bytes"] / (me["k1_ms"] / 1e3) / 1e9 if me["k1_ms"] else None
    swap_gbs = me["swap_bytes_timed"] / (me["swap_ms"] / 1e3) / 1e9 if me["swap_ms"] else None
    link_peak = (link["h2d"] + link["d2h"]) / 2
    line = {
        "metric": METRIC,
        "value": done_all / max(replay),
        "unit": "req/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": dev_s_max * 1e3 / K,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f16 (fp32 accumulate)",
        "data": "synthetic (generated API trace, random-init weights, synthetic token ids)",
        "config": {"workload": cfg["name"], "config": args.config,
                   "parallelism": f"replicas{world}: one engine + KV pool + pinned host pool per GPU, requests id mod "
                                  f"{world}, no collective on the data path",
                   "estimator": "value = requests of the trace / max over ranks of (iterations of the rank's "
                                "bit-exact schedule x measured device seconds per iteration); the timed iterations "
                                "are a stratified sample of each schedule",
                   "windows": [[s, c] for s, c in wins], "warmup_per_window": args.warmup,
                   "window_ms_per_iteration": [g["win_ms"] for g in gathered],
                   "schedule_iterations": [g["iters"] for g in gathered],
                   "l2": cfg["l2"]},
        "decode_tok_s": tot["decode"] / dev_s_max,
        "completed_in_windows": tot["completed"],
        "replay_seconds_estimated": max(replay),
        "step_roofline": {"bound": "max(weights + KV bytes / HBM, FLOPs / tensor peak) per iteration",
                          "bound_s": me["roof_s"], "measured_s": me["dev_s"],
                          "frac": me["roof_s"] / me["dev_s"] if me["dev_s"] else None,
                          "algorithmic_bytes": me["roof_bytes"], "algorithmic_flops": me["roof_flops"],
                          "peaks": {"hbm_gbs": pk.get("hbm_gbs"), "tflops": pk.get("bf16_tflops")}},
        "swap_gbs_achieved": swap_gbs,
        "swap_tokens_in_windows": tot["swapped"],
        "swap_in_forwarded_tokens": tot["swap_in_forwarded_tokens"],
        "host_pool_peak_gb": me["host_peak"] / 1e9,
        "swap_roofline": {"bound": "host link", "achieved": swap_gbs, "unit": "GB/s",
                          "peak": link_peak, "peak_h2d": link["h2d"], "peak_d2h": link["d2h"],
                          "frac": swap_gbs / link_peak if swap_gbs else None,
                          "peak_source": "pinned 512 MiB copies measured by bench.py on this box",
                          "note": "achieved = swapped bytes / time of each PCIe batch on the copy streams "
                                  "(DMA efficiency while a batch runs); swap-ins forwarded from swap-out staging do "
                                  "not cross the link; swaps overlap later iterations (cross-iteration pipelining, "
                                  "not per layer)",
                          "window_gbs": me["swap_bytes_timed"] / me["dev_s"] / 1e9 if me["dev_s"] else None,
                          "window_frac": (me["swap_bytes_timed"] / me["dev_s"] / 1e9 / link_peak) if me["dev_s"] else None,
                          "window_note": "PCIe swap bytes / device time of the timed windows: how much of the link "
                                         "the workload used under the model step"},
        "roofline": {"bound": "hbm", "kernel": "K1 paged decode attention (middle layer, every timed iteration)",
                     "achieved": k1_gbs, "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                     "frac": (k1_gbs / pk["hbm_gbs"]) if k1_gbs and pk.get("hbm_gbs") else None,
                     "traffic": (k1_traffic() or {}).get("dram_bytes_per_launch"),
                     "traffic_algorithmic_bytes": (k1_traffic() or {}).get("algorithmic_bytes_per_launch"),
                     "traffic_source": (k1_traffic() or {}).get("source"),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"},
        "e2e": {"value": done_all / max(replay_wall), "unit": "req/s",
                "h2d_bytes_per_step": tot["h2d_bytes"] / K / world,
                "d2h_bytes_per_step": tot["d2h_bytes"] / K / world},
        "gpu_launches": int(tot["kernel_launches"]),
        "clocks": clk,
    }
    ref_lib = os.path.join(ROOT, "oracle", "_ref", "libinterceptsim.so")  # the cpu_baseline leg's checker
    if world == 1 and not args.no_cpu_baseline and not os.path.exists(ref_lib):
        line["cpu_baseline"] = {"value": None, "unit": "req/s", "cores": os.cpu_count(), "kind": "reference",
                                "sample": f"unavailable: {ref_lib} not built"}
    elif world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference(cfg, args, wins)
        line["cpu_baseline"] = {"value": cpu["value"], "unit": "req/s", "cores": cpu["cores"], "kind": "port",
                                "sample": cpu["sample"], "s_per_iteration": cpu["s_per_iteration"]}
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def cpu_forward_seconds(preset, layers_total, plans):
    """Seconds per iteration of the numpy fp32 oracle forward over `plans`
    with all host threads: each plan timed with a 1- and a 2-layer model
    (after one untimed warm-up), extrapolated to `layers_total` layers, then
    averaged.  KV rows are materialised with non-zero contents (real memory
    traffic)."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle.forward import ForwardOracle

    cores = os.cpu_count()
    per_layers = {}
    with threadpool_limits(limits=cores):
        for layers in (1, 2):
            fo = ForwardOracle({"preset": preset, "layers": layers, "max_pos": 4160}, fast_random=True,
                               precision="f32")
            for pj in plans:
                for (rid, pos, count, kind, sample) in pj["spans"]:
                    fo._ensure(rid, pos + count + 1)
            for kv in fo.kv.values():
                kv.fill(np.float32(1e-3))
            fo._forward_only(plans[0])
            times = []
            for pj in plans:
                t = time.perf_counter()
                fo._forward_only(pj)
                times.append(time.perf_counter() - t)
            per_layers[layers] = times
            del fo
    if layers_total <= 2:  # the model itself was timed
        per_plan = list(per_layers[layers_total])
    else:
        per_plan = [a + (layers_total - 1) * max(b - a, 0.0) for a, b in zip(per_layers[1], per_layers[2])]
    per_iter = sum(per_plan) / len(per_plan)
    t1 = sum(per_layers[1]) / len(plans)
    t2 = sum(per_layers[2]) / len(plans)
    return per_iter, dict(t1=t1, t2=t2, cores=cores, per_iteration_s=[round(x, 3) for x in per_plan],
                          runs={str(k): [round(x, 4) for x in v] for k, v in per_layers.items()})


def cpu_full_trace_seconds(preset, plans):
    """Whole-trace CPU time of the numpy fp32 oracle forward at full depth
    (every iteration of the schedule, all host threads): measured, not
    extrapolated.  Only sensible for the tiny C0 model."""
    from threadpoolctl import threadpool_limits
    from oracle.forward import ForwardOracle
    with threadpool_limits(limits=os.cpu_count()):
        fo = ForwardOracle({"preset": preset}, precision="f32")
        t = time.perf_counter()
        for pj in plans:
            fo._forward_only(pj)
        return (time.perf_counter() - t) / len(plans)


def validate_depth(preset, layers_total, plans):
    """Check the layer extrapolation on the sampled plan with the least KV:
    its 1- and 2-layer forwards extrapolated to `layers_total` vs the same
    plan run at full depth (memory: the oracle keeps fp32 KV of every layer)."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle.forward import ForwardOracle

    def kv_of(pj):
        return sum(pos + count for (rid, pos, count, kind, sample) in pj["spans"])
    pj = min(plans, key=kv_of)
    out = {"iteration": pj["it"], "rows": sum(sp[2] for sp in pj["spans"]), "keys": kv_of(pj)}
    with threadpool_limits(limits=os.cpu_count()):
        for layers in (1, 2, layers_total):
            fo = ForwardOracle({"preset": preset, "layers": layers, "max_pos": 4160}, fast_random=True,
                               precision="f32")
            for (rid, pos, count, kind, sample) in pj["spans"]:
                fo._ensure(rid, pos + count + 1)
            for kv in fo.kv.values():
                kv.fill(np.float32(1e-3))
            fo._forward_only(pj)
            t = time.perf_counter()
            fo._forward_only(pj)
            out[f"t{layers}"] = time.perf_counter() - t
            del fo
    out["extrapolated"] = out["t1"] + (layers_total - 1) * (out["t2"] - out["t1"])
    out["measured"] = out[f"t{layers_total}"]
    out["measured_over_extrapolated"] = out["measured"] / out["extrapolated"]
    return out


def cpu_reference(cfg, args, wins):
    """The reference's CPU path on this host (see module docstring)."""
    from oracle.ref_plans import reference_schedule, run_reference as ref_run
    full = getattr(args, "full_trace", False)
    # every timed iteration of every window (event-log iteration numbers are 1-based)
    keep = None if full else {s + 1 + j for s, c in wins for j in range(c)}
    with tempfile.TemporaryDirectory() as d:
        summ, plans = reference_schedule(cfg["workload"], cfg["cost"], RUN, keep=keep, workdir=d)
    t_sched = ref_run(cfg["workload"], cfg["cost"], RUN, None)["wall_s"] / summ["iterations"]
    if full:
        fwd = cpu_full_trace_seconds(cfg["model"]["preset"], plans)
        per_iter = fwd + t_sched
        value = summ["done_events"] / (summ["iterations"] * per_iter)
        return {"value": value, "s_per_iteration": per_iter, "cores": os.cpu_count(), "iterations": summ["iterations"],
                "completed": summ["done_events"], "sched_us_per_iteration": t_sched * 1e6,
                "forward": {"runs": {str(cfg["layers"]): [fwd]}},
                "sample": (f"reference engine (oracle/_ref, {t_sched * 1e6:.1f} us/iteration) + numpy fp32 oracle "
                           f"forward of EVERY one of the {len(plans)} iterations at full depth (batches recovered "
                           f"from the reference's event log): {per_iter * 1e3:.2f} ms/iteration, measured over the "
                           f"whole trace")}
    per_iter, det = cpu_forward_seconds(cfg["model"]["preset"], cfg["layers"], plans)
    if getattr(args, "validate_depth", False):
        det["depth_check"] = validate_depth(cfg["model"]["preset"], cfg["layers"], plans)
    per_iter += t_sched
    value = summ["done_events"] / (summ["iterations"] * per_iter)
    return {"value": value, "s_per_iteration": per_iter, "cores": det["cores"], "iterations": summ["iterations"],
            "completed": summ["done_events"], "sched_us_per_iteration": t_sched * 1e6, "forward": det,
            "sample": (f"reference engine (oracle/_ref, whole trace: {int(summ['iterations'])} iterations, "
                       f"{t_sched * 1e6:.1f} us/iteration) + numpy fp32 oracle forward of the "
                       f"{len(plans)} timed iterations of the B200 arm's windows (batches recovered from the "
                       f"reference's event log), each timed with 1 and 2 layers (mean {det['t1']:.2f} / "
                       f"{det['t2']:.2f} s) and extrapolated to {cfg['layers']} layers: {per_iter:.2f} s/iteration "
                       f"(per iteration {min(det['per_iteration_s']):.1f}-{max(det['per_iteration_s']):.1f} s); "
                       f"EXTRAPOLATED, not a full-depth timed run")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    from oracle.ref_plans import REF_LIB
    if not os.path.exists(REF_LIB):
        print(json.dumps({"impl": "reference", "unavailable": f"{REF_LIB} not built (make -C oracle needs "
                                                              f"/root/reference)"}))
        return
    # Same window positions as the B200 arm at N = 1 (the whole trace, one host).
    from oracle.ref_plans import run_reference as ref_run
    summ = ref_run(cfg["workload"], cfg["cost"], RUN, None)
    wins = windows(int(summ["iterations"]), args.steps, args.warmup, args.windows or default_windows(args.steps))
    cpu = cpu_reference(cfg, args, wins)
    v = cpu["value"]
    line = {
        "metric": METRIC, "value": v, "unit": "req/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": cpu["s_per_iteration"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp32 (numpy)", "data": "synthetic", "impl": "reference",
        "extrapolated": not args.full_trace and cfg["layers"] > 2,
        "config": {"workload": cfg["name"], "config": args.config,
                   "host": "rank 0 only, all host threads, the whole (unsharded) trace; no GPU used",
                   "estimator": "value = requests / (iterations of the reference schedule x CPU seconds per "
                                "iteration), the per-iteration time " +
                                ("measured over every iteration of the trace" if args.full_trace else
                                 "sampled at the B200 arm's window positions"),
                   "windows": [[s, c] for s, c in wins]},
        "cpu_baseline": {"value": v, "unit": "req/s", "cores": cpu["cores"], "kind": "port",
                         "sample": cpu["sample"]},
        "forward_runs_s": cpu["forward"]["runs"],
        "depth_check": cpu["forward"].get("depth_check"),
        "e2e": {"value": v, "unit": "req/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--windows", type=int, default=0, help="timed windows (default: min(4, steps // 5))")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--host-gb", type=float, default=0.0, help="pinned host pool per rank (default: ledger x 1.25)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--validate-depth", action="store_true",
                    help="CPU path: also run the smallest sampled iteration at full depth to check the extrapolation")
    ap.add_argument("--full-trace", action="store_true",
                    help="CPU path: time the oracle forward over every iteration (C0 only: minutes)")
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
