"""Request-sharded replicas with world_size 2 over gloo on CPU.

The bench's C4 configuration (BASELINE configs[4]: a fixed 4000-request
trace, requests id mod N, original arrival times; strong scaling): each rank
takes its shard of the same generated trace, runs its own scheduler with a
plan log, and the ranks meet only in the reduction -- the plumbing bench.py
uses with NCCL on GPUs.  Checks: the shards partition the trace; each rank's
plan log (every batch the executor would run) and summary equal its shard
run alone; the window positions and the whole-job reduction
(bench.combine: requests / slowest rank's estimated replay).
"""
import hashlib
import json
import os
import socket
import tempfile

import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2402_01869_b200 as ib
    cfg = bench.CONFIGS["C4"]
    trace = bench.shard_trace(ib, cfg, world, rank, tempfile.mkdtemp())
    iters, done = bench.schedule_totals(ib, trace, cfg)
    plan_log = os.path.join(outdir, f"plans{rank}.jsonl")
    sess = ib.Session(trace, ib.CostModel.from_json(cfg["cost"]), dict(bench.RUN, plan_log=plan_log))
    _, finished = sess.step(10 ** 9)
    res = sess.finish().summary()
    del sess
    path = os.path.join(outdir, f"t{rank}.jsonl")
    trace.save(path)
    with open(path) as f:
        ids = [json.loads(l)["id"] for l in f.read().splitlines()[1:]]
    # stand-in device / wall seconds: rank 1 is the slower one
    local = dict(rank=rank, ids=ids, summary=res, iters=iters, total_done=done, finished=finished,
                 plan_sha=_sha(plan_log), wins=bench.windows(iters, 20, 5, 4),
                 dev_s=0.5 + rank, wall_s=0.6 + rank)
    out = [None] * world
    dist.all_gather_object(out, local)
    if rank == 0:
        json.dump(out, open(os.path.join(outdir, "gathered.json"), "w"))
    dist.destroy_process_group()


def test_two_rank_c4_sharding():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    import paper_2402_01869_b200 as ib
    outdir = tempfile.mkdtemp()
    mp.spawn(_worker, args=(2, _free_port(), outdir), nprocs=2, join=True)
    got = json.load(open(os.path.join(outdir, "gathered.json")))
    cfg = bench.CONFIGS["C4"]
    n = cfg["workload"]["request_count"]
    ids0, ids1 = set(got[0]["ids"]), set(got[1]["ids"])
    assert ids0.isdisjoint(ids1) and ids0 | ids1 == set(range(n))
    assert all(i % 2 == 0 for i in ids0) and all(i % 2 == 1 for i in ids1)
    assert all(g["finished"] for g in got)
    assert sum(g["total_done"] for g in got) == n == sum(g["summary"]["completed"] for g in got)
    # Each rank's schedule (plan log, summary) equals running its shard alone.
    for g in got:
        t = ib.Trace.load(os.path.join(outdir, f"t{g['rank']}.jsonl"))
        log = os.path.join(outdir, f"alone{g['rank']}.jsonl")
        alone = ib.run(t, ib.CostModel.from_json(cfg["cost"]), dict(bench.RUN, plan_log=log)).summary()
        assert alone == g["summary"]
        assert _sha(log) == g["plan_sha"]
        assert alone["iterations"] == g["iters"]
        # windows: 4 x 5 timed iterations, inside the schedule, in order, warm-up room before each
        w = g["wins"]
        assert sum(c for _, c in w) == 20 and len(w) == 4
        assert w[0][0] >= 5 and all(w[i][0] >= w[i - 1][0] + w[i - 1][1] + 5 for i in range(1, 4))
        assert w[-1][0] + w[-1][1] <= g["iters"]
    # the reduction: all requests / the slowest rank's estimated replay time
    done_all, replay, replay_wall = bench.combine(got, 20)
    assert done_all == n
    assert replay == [g["iters"] * g["dev_s"] / 20 for g in got]
    assert max(replay) == replay[1] and max(replay_wall) == replay_wall[1]
