"""Pose sharding across ranks (world_size 2, gloo, CPU): balanced contiguous
shards, the CT broadcast, the collecting buffer's collective fallback
(PeerRows in "collective" mode: each rank's rows gathered into rank 0's
buffer in global order, uneven shards included), the shared-loss all-reduce,
max-over-ranks timing and the rank rendezvous.  The CUDA path proper (the
kernels storing into rank 0's HBM, bitwise vs one process) is
tests/test_gpu_distributed.py."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["DRR_PEER_MODE"] = "collective"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2208_12737_b200.distributed import (PeerRows, allreduce_sum, broadcast_volume,
                                                   gather_rows, max_over_ranks, rank_sync,
                                                   shard_range)
    vol = torch.arange(24, dtype=torch.float32).reshape(2, 3, 4) if rank == 0 else None
    got = broadcast_volume(vol, (2, 3, 4), "cpu")
    n = 7
    start, stop = shard_range(n, rank, world)
    # each rank's "kernel" writes rows that depend only on the global pose index
    local = torch.stack([torch.full((2, 2), float(i)) for i in range(start, stop)])
    rows = gather_rows(local, n)
    pr = PeerRows(n, (2, 2), torch.float32, "cpu")
    assert pr.mode == "collective" and (pr.lo, pr.hi) == (start, stop)
    pr.shard_view().copy_(local + 100.0)
    pr.collect()
    rank_sync("cpu")
    collected = pr.rows()[:, 0, 0].tolist() if rank == 0 else None
    loss = allreduce_sum(torch.tensor([float(stop - start)]))
    slow = max_over_ranks(10.0 * (rank + 1), "cpu")
    results[rank] = (got.sum().item(), rows[:, 0, 0].tolist(), loss.item(), slow, collected)
    dist.destroy_process_group()


def test_shard_range_partition():
    from paper_2208_12737_b200.distributed import shard_range
    for n in (0, 1, 7, 64, 1023):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_gloo_sharding():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    results = manager.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    for r in range(world):
        vol_sum, rows, loss, slow, collected = results[r]
        assert vol_sum == sum(range(24))
        assert rows == [float(i) for i in range(7)]
        assert loss == 7.0
        assert slow == 20.0
    assert results[0][4] == [100.0 + i for i in range(7)]
    assert results[1][4] is None
