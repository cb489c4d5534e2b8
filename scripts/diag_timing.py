"""Diagnostic: per-step event timing (bench style, L2 flush between steps) vs
back-to-back launches vs host enqueue time, for the c2 workload."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_09664_b200 as pg  # noqa: E402
from paper_2512_09664_b200 import _lib  # noqa: E402
from paper_2512_09664_b200.particles import native_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
H, W, B = bench.CONFIGS[name][:3]
if len(sys.argv) > 2:
    B = int(sys.argv[2])
pg.register_flow_function("bench_vortex", bench.vortex(H, W))
pg.register_flow_function("bench_uniform", bench.uniform)
cfg = bench.make_cfg(pg, name, B)
print('B =', B, 'ablate', os.environ.get('PGB_ABLATE', '0'))
lib = _lib.load()
ncfg = native_config(cfg)
field = pg.from_function(bench.vortex(H, W), H, W)
flows = field.to_device("cuda").unsqueeze(0).contiguous()
img = [torch.empty((B, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
s = torch.cuda.current_stream()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def step(b):
    _lib.check(lib.pgb_generate_batch_dev(ncfg, b, 0, B, flows.data_ptr(), 1, B, _lib.OUT_F32,
                                          img[0].data_ptr(), img[1].data_ptr(), None, None, s.cuda_stream))


for b in range(5):
    step(b)
torch.cuda.synchronize()
K = 50
# host enqueue cost
t0 = time.perf_counter()
for k in range(K):
    step(100 + k)
t_host = (time.perf_counter() - t0) / K
torch.cuda.synchronize()
# back-to-back on the GPU (host enqueues ahead)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(s)
for k in range(K):
    step(200 + k)
e1.record(s)
torch.cuda.synchronize()
t_b2b = e0.elapsed_time(e1) / K
# bench style: flush + per-step events
st = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
en = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
for k in range(K):
    flush.zero_()
    st[k].record(s)
    step(300 + k)
    en[k].record(s)
torch.cuda.synchronize()
t_bench = sum(a.elapsed_time(b) for a, b in zip(st, en)) / K
# flush + per-step events, but the step is pre-enqueued behind a host-side gate:
# enqueue flush, start event, step, end event with the GPU held busy by a long
# kernel first so host latency is hidden
for k in range(K):
    flush.zero_()
    flush.zero_()
    st[k].record(s)
    step(400 + k)
    en[k].record(s)
torch.cuda.synchronize()
t_bench2 = sum(a.elapsed_time(b) for a, b in zip(st, en)) / K
print(f"host enqueue {t_host * 1e6:.1f} us/step; back-to-back {t_b2b * 1e3:.1f} us/step; "
      f"bench-style {t_bench * 1e3:.1f} us/step; bench-style with 2 flushes {t_bench2 * 1e3:.1f} us/step")
# raw write bandwidth of the same output bytes (torch fill), back-to-back
e0.record(s)
for k in range(K):
    img[0].fill_(0.5)
    img[1].fill_(0.5)
e1.record(s)
torch.cuda.synchronize()
t_fill = e0.elapsed_time(e1) / K
print(f"torch fill of both frames: {t_fill * 1e3:.1f} us/step = {2 * img[0].numel() * 4 / (t_fill * 1e-3) / 1e9:.0f} GB/s")
