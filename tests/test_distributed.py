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


def test_bench_spawns_one_rank_per_gpu_dry_run():
    """`python bench.py --gpus 2` outside torchrun re-launches itself under
    torch.distributed.run with two ranks (the driver's BENCH invocation);
    --dry-run exercises the launcher and rank plumbing on CPU (gloo)."""
    import json
    import subprocess
    import sys

    from _helpers import ROOT

    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    for cfg, want_batch in (("c2", 512), ("c5", 8192)):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                              "--config", cfg], capture_output=True, text=True, timeout=300, env=env)
        assert out.returncode == 0, out.stderr[-2000:]
        line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
        assert line["n_gpus"] == 2 and line["global_batch"] == want_batch
        assert sum(line["pairs_per_rank"]) == want_batch and len(line["pairs_per_rank"]) == 2


def test_sharded_export_uses_global_indices_and_merges(tmp_path):
    """Two shards of one batch (as two ranks write them) land under global pair
    indices; the per-shard sidecar parts merge into one params file in pair
    order (export.merge_sidecars)."""
    import json
    from types import SimpleNamespace

    from paper_2512_09664_b200 import GeneratorConfig, export

    from paper_2512_09664_b200 import OutputConfig

    cfg = GeneratorConfig(image_height=6, image_width=8, batch_size=4, output=OutputConfig(format="raw_f32"))
    rng = np.random.default_rng(0)

    def params(m):
        return SimpleNamespace(active_count=m, seeding_density=0.05, diameters=rng.uniform(0.8, 1.2, 5),
                               peak_intensities=np.ones(5), rhos=np.zeros(5))

    with export.DatasetWriter(cfg, str(tmp_path)) as w:
        for pr in (range(2, 4), range(0, 2)):          # rank 1's shard may finish first
            imgs = torch.from_numpy(rng.uniform(0, 1, (len(pr), 6, 8)).astype(np.float32))
            w.submit(SimpleNamespace(images1=imgs, images2=imgs, flow_fields=[], batch_index=3,
                                     pair_range=pr, params=[params(3) for _ in pr]))
    names = sorted(os.listdir(tmp_path))
    assert [n for n in names if n.endswith("_a.raw")] == [f"pair_000003_{i:04d}_a.raw" for i in range(4)]
    assert export.merge_sidecars(str(tmp_path)) == 1
    assert not [n for n in os.listdir(tmp_path) if ".part" in n]
    meta = json.load(open(tmp_path / "params_000003.json"))
    assert [p["pair_index"] for p in meta["pairs"]] == [0, 1, 2, 3]
