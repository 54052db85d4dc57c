"""Host-side logic of the N>1 path on CPU with gloo (world_size 2).

The solve path shards as replicas (cases batched across GPUs):
the only cross-rank operations are the barrier and the max-over-ranks of the
step time that bench.py reports; the reference arm runs on rank 0 only."""
import os
import socket
import subprocess
import sys

import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench
    step = [2.0, 3.5][rank]
    kern = [1.0, 1.25][rank]
    got = bench.max_over_ranks([step, kern])
    out[rank] = (got, bench.whole_job_gbps(world, 1e9, got[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_and_whole_job_value():
    world = 2
    mgr = mp.get_context("spawn").Manager()  # no fork of a process that holds OpenMP threads
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for rank in range(world):
        got, val = out[rank]
        assert got == [3.5, 1.25]           # slowest rank's step time on every rank
        assert abs(val - 2 * 1e9 / 3.5e-3 / 1e9) < 1e-9  # bytes of ALL ranks / max time


def test_reference_arm_under_torchrun_prints_once():
    port = _free_port()
    env = dict(os.environ, PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"), "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "1", "--cells", "2", "2", "2", "--cases", "4"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and (d.get("value") or d.get("unavailable"))
