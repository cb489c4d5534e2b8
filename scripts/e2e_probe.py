"""e2e (host-buffer) path vs the PCIe D2H ceiling at the same transfer size.
Usage (GPU box): python scripts/e2e_probe.py [config]"""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
H, W, B = bench.CONFIGS[name][:3]
nbytes = B * H * W * 4
d = torch.empty(2 * nbytes // 4, dtype=torch.float32, device="cuda")
h = torch.empty_like(d, device="cpu").pin_memory()
for one in (True, False):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if one:
            h.copy_(d, non_blocking=True)
        else:
            h[: nbytes // 4].copy_(d[: nbytes // 4], non_blocking=True)
            h[nbytes // 4:].copy_(d[nbytes // 4:], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"D2H {'1 copy ' if one else '2 copies'} {2 * nbytes / 1e6:.1f} MB: {best * 1e3:.3f} ms = "
          f"{2 * nbytes / best / 1e9:.2f} GB/s -> {B / best / 1e3:.1f} k pairs/s ceiling")
for ch in ("1", "2", "4", "8", "16"):
    env = dict(os.environ, PGB_E2E_CHUNKS=ch)
    out = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--config", name,
                          "--no-cpu-baseline"], capture_output=True, text=True, env=env).stdout
    import json
    line = json.loads([l for l in out.splitlines() if l.startswith("{")][-1])
    print(f"chunks {ch:>2s}: e2e {line['e2e']['value'] / 1e3:.1f} k pairs/s")
