"""Debug: per-phase cycle split of the band kernel (needs a PGB_PHASE_TIMING build).
Usage: PGB_PHASE_TIMING=1 python -m paper_2512_09664_b200.build --force && python scripts/phase_timing.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_09664_b200 as pg  # noqa: E402
from paper_2512_09664_b200 import _lib  # noqa: E402
from paper_2512_09664_b200.particles import native_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
H, W, B = bench.CONFIGS[name][:3]
pg.register_flow_function("bench_vortex", bench.vortex(H, W))
pg.register_flow_function("bench_uniform", bench.uniform)
cfg = bench.make_cfg(pg, name, B)
lib = _lib.load()
field = pg.from_function(bench.vortex(H, W), H, W)
flows = field.to_device("cuda").unsqueeze(0).contiguous()
img = [torch.empty((B, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
for it in range(3):
    _lib.check(lib.pgb_generate_batch_dev(native_config(cfg), it, 0, B, flows.data_ptr(), 1, B, _lib.OUT_F32,
                                          img[0].data_ptr(), img[1].data_ptr(), None, None,
                                          torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
fn = lib.pgb_debug_phase_timing
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(148 * 8 * 8 * 5, np.uint64)
n = fn(buf.ctypes.data, buf.size)
t = buf[:148 * 8 * 8 * 5 // 2].reshape(-1, 5).astype(np.float64)
t = t[t[:, 4] > 0]
tot = t[:, :4].sum(axis=1)
names = ["particles", "barrier(after particles)", "store", "barrier(after store)"]
print(f"warps with items: {len(t)}, items/warp mean {t[:, 4].mean():.2f}")
for k, nm in enumerate(names):
    print(f"{nm:28s} {100 * t[:, k].sum() / tot.sum():5.1f}%   mean cycles/item {t[:, k].sum() / t[:, 4].sum():9.0f}")
print(f"per-warp total cycles: min {tot.min():.0f} max {tot.max():.0f} mean {tot.mean():.0f}")
base = 148 * 8 * 8 * 5 // 2
ct = buf[base:base + 4 * 2048].reshape(-1, 4)
pt = buf[base + 4 * 2048:base + 4 * 2048 + 8 * 296].reshape(-1, 8).astype(np.float64)
ct = ct[ct[:, 0] > 0].astype(np.float64)
t0 = ct[:, 0].min()
ct -= t0
print(f"CTAs {len(ct)}: start max {ct[:,0].max()/1e3:.1f} us; prologue end mean {ct[:,1].mean()/1e3:.1f} max {ct[:,1].max()/1e3:.1f} us; "
      f"loop start mean {ct[:,2].mean()/1e3:.1f} max {ct[:,2].max()/1e3:.1f} us; end mean {ct[:,3].mean()/1e3:.1f} max {ct[:,3].max()/1e3:.1f} us")
pt = pt[pt[:, 0] > 0]
pt = (pt - t0) / 1e3
for k, nm in enumerate(["ppp/M done", "fp64 chain done", "histogram done", "scan done", "cof done", "prefix stored", "cof staged"]):
    print(f"prologue {nm:18s} mean {pt[:, k].mean():6.2f} us  max {pt[:, k].max():6.2f} us")
cyc = buf[base + 4 * 2048:base + 4 * 2048 + 8 * 296].reshape(-1, 8)[:, 7].astype(np.float64)
ok = (pt_raw := buf[base + 4 * 2048:base + 4 * 2048 + 8 * 296].reshape(-1, 8).astype(np.float64))[:, 0] > 0
ns = pt_raw[ok, 4] - pt_raw[ok, 0]
print(f"prologue stage0->4: {cyc[ok].mean():.0f} cycles over {ns.mean():.0f} ns -> {cyc[ok].mean() / ns.mean():.3f} GHz")
st = buf[base + 4 * 2048 + 8 * 296:base + 4 * 2048 + 8 * 296 + 2 * 296].reshape(-1, 2).astype(np.float64)
st = st[st[:, 1] > 0]
print(f"stager item_stage: mean {st[:, 0].sum() / st[:, 1].sum():.0f} cycles per item over {st[:, 1].sum():.0f} items")
