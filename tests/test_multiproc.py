"""CPU, world_size 2 over gloo: the sharded bench path's host logic --
max-over-ranks timing and the all_gather of output ciphertext words (the only
collective; NCCL on the GPU box)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    rng = np.random.default_rng(rank)
    words = torch.from_numpy(rng.integers(0, 2 ** 40, size=4 * 2 * 3 * 16, dtype=np.int64))
    t = bench.max_over_ranks(0.5 + rank, "cpu")
    got = bench.gather_outputs(words)
    if rank == 0:
        q.put((t, [g.numpy().copy() for g in got]))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_and_max_over_ranks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    t, gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == pytest.approx(1.5)
    for r in range(world):
        want = np.random.default_rng(r).integers(0, 2 ** 40, size=4 * 2 * 3 * 16, dtype=np.int64)
        assert np.array_equal(gathered[r], want)
