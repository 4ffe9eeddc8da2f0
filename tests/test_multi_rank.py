"""The N > 1 path on CPU (gloo, world size 2): rod sharding and the result
gather.  Each rank builds only its slice of the hair batch (workloads.shard /
workloads.hair(first=...)), steps it independently -- no per-step
collective -- and the gathered result must equal stepping the whole batch in
one process, bit for bit.  On the GPU box bench.py runs the same flow with
NCCL (all_gather_into_tensor on the device state)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_2509_04277_b200 import workloads as wl

RODS, STEPS = 8, 20


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.oracle import OracleStepper
    from paper_2509_04277_b200 import workloads
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                            rank=rank, world_size=world)
    first, per = workloads.shard(RODS, world, rank)
    w = workloads.hair(per, 32, first=first)
    OracleStepper(w).run(STEPS)
    mine = torch.from_numpy(np.ascontiguousarray(w.positions).reshape(-1))
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    if rank == 0:
        out.put(torch.cat(parts).numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shards_tile_the_batch():
    firsts = [wl.shard(65536, 8, r) for r in range(8)]
    assert [f for f, _ in firsts] == [r * 8192 for r in range(8)]
    with pytest.raises(ValueError):
        wl.shard(10, 3, 0)
    full = wl.hair(6, 16)
    a, b = wl.hair(3, 16, first=0), wl.hair(3, 16, first=3)
    assert np.array_equal(np.concatenate([a.positions, b.positions]), full.positions)
    assert np.array_equal(np.concatenate([a.frames, b.frames]), full.frames)


def test_two_rank_gloo_gather_equals_single_process():
    from oracle.oracle import OracleStepper
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = wl.hair(RODS, 32)
    OracleStepper(ref).run(STEPS)
    assert np.array_equal(gathered.reshape(-1, 3), ref.positions)
