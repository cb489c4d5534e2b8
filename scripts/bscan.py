"""Band-kernel time vs batch size (fixed cost + marginal cost per pair).

Usage (GPU box): python scripts/bscan.py [config] [B ...]
Prints us/launch for back-to-back launches and with an L2 flush between them.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_09664_b200 as pg  # noqa: E402
from paper_2512_09664_b200 import _lib  # noqa: E402
from paper_2512_09664_b200.particles import native_config  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    Bs = [int(b) for b in sys.argv[2:]] or [1, 8, 32, 64, 128, 256, 512, 1024]
    H, W, _, _, _, flow, _ = bench.CONFIGS[name]
    pg.register_flow_function("bench_vortex", bench.vortex(H, W))
    pg.register_flow_function("bench_uniform", bench.uniform)
    field = pg.from_function(bench.vortex(H, W) if flow == "vortex" else bench.uniform, H, W)
    flows = field.to_device().unsqueeze(0).contiguous()
    lib = _lib.load()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    for B in Bs:
        cfg = bench.make_cfg(pg, name, B)
        ncfg = native_config(cfg)
        img1 = torch.empty((B, H, W), dtype=torch.float32, device="cuda")
        img2 = torch.empty_like(img1)

        def step(k):
            _lib.check(lib.pgb_generate_batch_dev(ncfg, k, 0, B, flows.data_ptr(), 1, B, _lib.OUT_F32,
                                                  img1.data_ptr(), img2.data_ptr(), None, None,
                                                  stream.cuda_stream))
        for k in range(5):
            step(k)
        torch.cuda.synchronize()
        n = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(n):
            step(100 + k)
        e1.record()
        torch.cuda.synchronize()
        b2b = e0.elapsed_time(e1) / n * 1e3
        ts = []
        for k in range(n):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step(200 + k)
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        fl = sum(a.elapsed_time(b) for a, b in ts) / n * 1e3
        import time
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(n):
            step(300 + k)
        host = (time.perf_counter() - t0) / n * 1e6
        torch.cuda.synchronize()
        print(f"{name} B={B:5d}  back-to-back {b2b:8.1f} us  flushed {fl:8.1f} us  "
              f"({fl / B:.3f} us/pair)  host enqueue {host:6.1f} us/call", flush=True)
        del img1, img2


if __name__ == "__main__":
    main()
