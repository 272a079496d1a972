"""Multi-process (gloo, world_size 2, CPU) coverage of the N>1 path: weak-scaling shot sharding.

bench.py gives every rank its own shot range (shot0 = rank * shots, no data-path
collective); the outputs must be exactly the shots of one big run, because
every draw is keyed by (seed, shot | shot word, instruction).
"""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, shots, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from goldens import load

    P = load("config2")["prog"]
    st, out, _ = oracle.sample(P, shots, seed=21, shot0=rank * shots, flags=0)
    mine = torch.from_numpy(np.concatenate([out.meas.ravel(), out.det.ravel(), out.obs.ravel(),
                                            out.accepted]).astype(np.int64))
    gathered = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # the bench's max-over-ranks timing reduction
    if rank == 0:
        q.put(([g.numpy() for g in gathered], float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_equal_single_run():
    import oracle
    from goldens import load

    world, shots = 2, 4096
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shots, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert tmax == 2.0
    P = load("config2")["prog"]
    _, full, _ = oracle.sample(P, world * shots, seed=21, shot0=0, flags=0)
    W = shots // 32
    for r in range(world):
        a = parts[r]
        U, D, O = P.num_user_records, P.num_detectors, P.num_observables
        meas = a[: U * W].reshape(U, W)
        det = a[U * W:(U + D) * W].reshape(D, W)
        np.testing.assert_array_equal(meas, full.meas[:U, r * W:(r + 1) * W])
        np.testing.assert_array_equal(det, full.det[:D, r * W:(r + 1) * W])
