"""Request-sharded replicas with world_size 2 over gloo on CPU.

Each rank takes the requests with id mod N == rank from the same generated
trace (original arrival times), runs its own scheduler, and the ranks meet only
in the timing / counter reduction -- the exact plumbing bench.py uses with
NCCL on GPUs.  Checks: the shards partition the trace, each rank's schedule is
identical to running its shard alone, and the max-over-ranks / sum reductions.
"""
import json
import os
import socket
import tempfile

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

WL = dict(classes=[{"name": "Math"}, {"name": "QA"}, {"name": "Chatbot"}], request_count=120, arrival_rate=3.0,
          seed=11)
COST = dict(mem_per_token=458752, gpu_kv_capacity=150e9, cpu_kv_capacity=128e9, swap_per_token=458752 / 50e9)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2402_01869_b200 as ib
    bench.WORKLOAD = WL
    trace = bench.shard_trace(ib, world, rank, tempfile.mkdtemp())
    sess = ib.Session(trace, ib.CostModel.from_json(COST), {"policy": "infercept"})
    _, finished = sess.step(10 ** 9)
    res = sess.finish().summary()
    ids = []
    path = os.path.join(outdir, f"t{rank}.jsonl")
    trace.save(path)
    with open(path) as f:
        ids = [json.loads(l)["id"] for l in f.read().splitlines()[1:]]
    local = dict(rank=rank, ids=ids, summary=res, iterations=res["iterations"], completed=res["completed"])
    out = [None] * world
    dist.all_gather_object(out, local)
    if rank == 0:
        json.dump(out, open(os.path.join(outdir, "gathered.json"), "w"))
    dist.destroy_process_group()


def test_two_rank_request_sharding():
    outdir = tempfile.mkdtemp()
    mp.spawn(_worker, args=(2, _free_port(), outdir), nprocs=2, join=True)
    got = json.load(open(os.path.join(outdir, "gathered.json")))
    ids0, ids1 = set(got[0]["ids"]), set(got[1]["ids"])
    # bench.workload_for: the 2-replica trace has 2x the requests at 2x the rate,
    # so each shard carries the single-GPU load (weak scaling).
    n = 2 * WL["request_count"]
    assert ids0.isdisjoint(ids1) and ids0 | ids1 == set(range(n))
    assert all(i % 2 == 0 for i in ids0) and all(i % 2 == 1 for i in ids1)
    assert sum(g["completed"] for g in got) == n
    assert abs(len(ids0) - WL["request_count"]) <= 1
    # Each rank's schedule equals running its shard alone in this process.
    import paper_2402_01869_b200 as ib
    for g in got:
        t = ib.Trace.load(os.path.join(outdir, f"t{g['rank']}.jsonl"))
        alone = ib.run(t, ib.CostModel.from_json(COST), {"policy": "infercept"}).summary()
        assert alone == g["summary"]
