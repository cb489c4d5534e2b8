import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_09664_b200 as pg  # noqa: E402

pg.register_flow_function("bench_vortex", bench.vortex(256, 256))
cfg = pg.with_updates(bench.make_cfg(pg, "c2", 256), batches_per_flow_field=8)
with pg.make_sampler(cfg, max_batches=40) as s:
    for _ in range(5):
        next(s)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(20):
        next(s)
    torch.cuda.synchronize()
    pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
