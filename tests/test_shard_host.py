"""Host side of the sharded path, world_size 2 over gloo on CPU (no GPU needed).

Covers what bench.py --gpus N does before any kernel runs: the process group, the
max-over-ranks timing reduction, the broadcast of the library's NCCL unique id, and the
slab split every rank computes independently (it must tile the last mode in rank order,
balanced to within one row). The device side is tests/test_gpu_shard.py.
"""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch.distributed as td
import bench
import paper_1703_09074_b200 as rcp

world, rank, local = bench.dist_env()
d = bench.Dist(world, rank, local)
assert d.dev == "cpu"
# max over ranks (the bench's timing rule)
assert d.max(10.0 + rank) == 10.0 + world - 1
# rank 0's NCCL unique id reaches every rank unchanged
uid = rcp.comm_unique_id() if rank == 0 else bytes(128)
got = d.broadcast_bytes(uid)
ref = [None] * world
td.all_gather_object(ref, got)
assert all(r == ref[0] for r in ref) and len(ref[0]) == 128 and ref[0] != bytes(128)
# slabs computed independently on every rank tile [0, E) in rank order
for E in (1, 7, 20, 500, 1024, 10000):
    mine = rcp.slab_range(E, world, rank)
    allr = [None] * world
    td.all_gather_object(allr, mine)
    assert allr[0][0] == 0 and allr[-1][1] == E
    for a, b in zip(allr, allr[1:]):
        assert a[1] == b[0]
    sizes = [h - l for l, h in allr]
    assert max(sizes) - min(sizes) <= 1
d.barrier()
d.close()
print("RANK_OK", rank)
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(300)
def test_gloo_world2_host_logic(rcp):
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, ROOT=ROOT, WORLD_SIZE="2", RANK=str(r), LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=240)[0] for p in procs]
    for r, (p, o) in enumerate(zip(procs, outs)):
        assert p.returncode == 0, o[-2000:]
        assert f"RANK_OK {r}" in o


@pytest.mark.timeout(300)
def test_bench_spawns_one_rank_per_gpu():
    """`bench.py --gpus 2` outside torchrun re-launches itself under torch.distributed.run with
    two ranks (gloo here, no GPU), asserts WORLD_SIZE == --gpus, and rank 0 alone prints one
    JSON line carrying the max over ranks."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--host-check"],
                         env=env, capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    import json
    rec = json.loads(lines[0])
    assert rec == {"host_check": True, "world": 2, "max_rank": 1.0}


def test_bench_rejects_world_mismatch():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--host-check"],
                         env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr
