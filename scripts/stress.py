"""Stress: random configs, pair ranges and streams; every result must equal a
cold single-stream run of the same batch (bit-identical). Exits non-zero on
any mismatch. Usage: python scripts/stress.py [seconds]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2512_09664_b200 as pg  # noqa: E402
from paper_2512_09664_b200 import _lib  # noqa: E402
from paper_2512_09664_b200.particles import native_config  # noqa: E402
from _helpers import vortex_fn  # noqa: E402



def run_stress(limit: float, seed: int = 0) -> int:
    """Random configs for `limit` seconds; returns the number checked, raises on a mismatch."""
    rng = np.random.default_rng(seed)
    streams = [torch.cuda.Stream() for _ in range(3)]
    t0 = time.time()
    n = 0
    while time.time() - t0 < limit:
        n += _one(rng, streams)
    return n


def _one(rng, streams) -> int:
    H = int(rng.choice([64, 96, 128, 200, 256]))
    W = int(rng.choice([64, 128, 160, 256]))
    B = int(rng.integers(1, 40))
    kw = dict(image_height=H, image_width=W, batch_size=B, seed=int(rng.integers(1 << 30)),
              seeding_density_range=(0.02, float(rng.uniform(0.03, 0.1))),
              diameter_range=(0.6, float(rng.uniform(0.8, 4.0))),
              flow_sources=(pg.FlowSource(function="s"),))
    if rng.random() < 0.5:
        kw["rho_range"] = (-0.3, 0.3)
    if rng.random() < 0.3:
        kw["frame2_sigma_std"] = 0.05
    cfg = pg.GeneratorConfig(**kw)
    flows = pg.from_function(vortex_fn(H, W), H, W).to_device().unsqueeze(0)
    ncfg = native_config(cfg)
    batch = int(rng.integers(0, 1000))

    def run(base, count, stream):
        img = [torch.empty((count, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
        _lib.call("pgb_generate_batch_dev", ncfg, batch, base, count, flows.data_ptr(), 1, B, _lib.OUT_F32,
                  img[0].data_ptr(), img[1].data_ptr(), None, None, stream.cuda_stream)
        return img

    torch.cuda.synchronize()
    want = run(0, B, torch.cuda.current_stream())
    torch.cuda.synchronize()
    parts, base = [], 0
    while base < B:
        c = int(rng.integers(1, B - base + 1))
        s = streams[int(rng.integers(0, len(streams)))]
        parts.append((base, run(base, c, s)))
        base += c
    torch.cuda.synchronize()
    for b0, img in parts:
        for f in range(2):
            if not torch.equal(img[f], want[f][b0:b0 + img[f].shape[0]]):
                raise AssertionError(f"MISMATCH {kw} batch {batch} base {b0} frame {f}")
    return 1
if __name__ == "__main__":
    limit = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    t0 = time.time()
    n = run_stress(limit)
    print(f"stress ok: {n} configs in {time.time() - t0:.0f} s")
