"""bench.py under torchrun with two ranks (the N > 1 plumbing the scaling run
uses: rendezvous, per-rank shard schedules, barriers, gather of per-rank
stats, max-over-ranks replay time), both ranks on cuda:0 (BENCH_DEVICE) with
the tiny C0 configuration: one B200 is all this environment has.  The ranks
meet over gloo here (NCCL refuses two ranks on one device); with one GPU per
rank the bench uses NCCL."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT, have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a B200")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_c0():
    env = dict(os.environ, BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "C0",
           "--steps", "8", "--warmup", "3"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 8 and d["scaling"] == "strong"
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert len(d["config"]["schedule_iterations"]) == 2
