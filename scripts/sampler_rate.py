"""Sampler throughput (batches back to back, device-side images) for the
default Philox generator and the reference-RNG mode, C2 shape."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_09664_b200 as pg  # noqa: E402

H, W, B = 256, 256, 256
for rng, R, dev in (("philox", 1, False), ("philox", 1, True), ("philox", 1, "graph"), ("splitmix64", 1, True),
                    ("philox", 8, False), ("splitmix64", 8, False)):
    pg.register_flow_function("bench_vortex", bench.vortex(H, W), device=bool(dev), graph=dev == "graph")
    cfg = pg.with_updates(bench.make_cfg(pg, "c2", B), rng=rng, batches_per_flow_field=R)
    with pg.make_sampler(cfg, max_batches=25) as s:
        for _ in range(5):
            next(s)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            b = next(s)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 20
    where = "device (CUDA graph)" if dev == "graph" else "device" if dev else "host"
    print(f"{rng} R={R} flow on {where}: {B / dt / 1e6:.3f} M pairs/s ({dt * 1e6:.0f} us/batch, Sampler wall clock)")
