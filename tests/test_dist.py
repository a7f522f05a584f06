"""N > 1 host logic of bench.py on CPU with gloo, world_size 2: replica
instances per rank (distinct seeds, no data-path collective), max-over-ranks
timing and summed throughput, and the reference arm running on rank 0 only."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update({"WORLD_SIZE": str(world), "RANK": str(rank), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    sys.path.insert(0, ROOT)
    import bench
    from paper_2601_20174_b200 import problems
    d = bench.Dist()
    assert d.pg is not None and d.backend == "gloo"
    cfg = bench.replica_seeds(problems.C1, d.rank)
    pb = problems.generate(cfg)
    t_local = 1.0 + d.rank          # pretend timings
    out[rank] = (cfg.seed, cfg.s0_seed, float(pb.rhs[0]), d.max(t_local), d.sum(10.0 * (d.rank + 1)))
    d.barrier()
    d.close()


def test_replicas_and_reductions_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert r0[0] != r1[0] and r0[1] != r1[1]   # independent instances
    assert r0[2] != r1[2]
    assert r0[3] == r1[3] == 2.0               # max over ranks
    assert r0[4] == r1[4] == 30.0              # whole-job sum


def test_reference_arm_rank0_only_under_torchrun():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--config", "C1", "--steps", "1", "--warmup", "0",
           "--ref-step-seconds", "0.2", "--ref-threads", "2"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 2
    assert d["cpu_baseline"]["cores"] == 2 and d["e2e"]["h2d_bytes_per_step"] == 0
