"""CPU, world_size 2 over gloo: sharding and the flow-window broadcast (the only
collective of the multi-GPU path)."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_09664_b200.pipeline import broadcast_window, shard_pairs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        window = torch.zeros((2, 8, 8, 2))
        if rank == 0:
            window = torch.arange(2 * 8 * 8 * 2, dtype=torch.float32).reshape(2, 8, 8, 2)
        broadcast_window(window, src=0)
        r = shard_pairs(10, rank, world)
        # every rank derives the same per-pair Philox words for a global pair index
        from oracle import philox

        words = np.stack(philox.draw(7, r.start, 3, np.arange(4, dtype=np.uint64), philox.TAG_PARTICLE_A))
        out[rank] = (float(window.sum()), (r.start, r.stop), words.tolist())
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_and_broadcast():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    full = float(np.arange(2 * 8 * 8 * 2).sum())
    assert out[0][0] == out[1][0] == full
    assert out[0][1] == (0, 5) and out[1][1] == (5, 10)
    from oracle import philox

    for rank in range(world):
        start = out[rank][1][0]
        want = np.stack(philox.draw(7, start, 3, np.arange(4, dtype=np.uint64), philox.TAG_PARTICLE_A))
        assert out[rank][2] == want.tolist()


def test_shards_partition_every_batch_size():
    for B in (1, 2, 7, 256, 8192):
        for n in (1, 2, 3, 4, 8):
            ranges = [shard_pairs(B, r, n) for r in range(n)]
            assert ranges[0].start == 0 and ranges[-1].stop == B
            assert all(a.stop == b.start for a, b in zip(ranges, ranges[1:]))
