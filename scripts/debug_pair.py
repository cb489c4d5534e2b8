"""Debug: pair kernel with the default inbox capacity vs a tiny one (spill path)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_09664_b200 as pg
from paper_2512_09664_b200 import _lib
from paper_2512_09664_b200.particles import native_config
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from _helpers import vortex_fn

H = W = 128
B = 12
cfg = pg.GeneratorConfig(image_height=H, image_width=W, batch_size=B, seeding_density_range=(0.05, 0.1),
                         diameter_range=(0.5, 4.0), rho_range=(-0.5, 0.5), frame2_sigma_std=0.05,
                         frame2_intensity_std=0.05, frame2_rho_std=0.05, hide_probability=0.1, seed=9,
                         flow_sources=(pg.FlowSource(function="vortex"),))
flows = pg.from_function(vortex_fn(H, W), H, W).to_device().unsqueeze(0)
stats = {"seeding_density": torch.empty(B, dtype=torch.float64, device="cuda"),
         "active_count": torch.empty(B, dtype=torch.int32, device="cuda"),
         "side": torch.empty(B, dtype=torch.int32, device="cuda"),
         "d_max": torch.empty(B, dtype=torch.float32, device="cuda")}
st = _lib.PgbPairStats(**{k: v.data_ptr() for k, v in stats.items()})

def run(batch, cap=None):
    if cap:
        os.environ["PGB_PAIR_CAP"] = str(cap)
    else:
        os.environ.pop("PGB_PAIR_CAP", None)
    img = [torch.zeros((B, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
    _lib.call("pgb_generate_batch_dev", native_config(cfg), batch, 0, B, flows.data_ptr(), 1, B, _lib.OUT_RAW,
              img[0].data_ptr(), img[1].data_ptr(), st, None, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return [i.cpu().numpy() for i in img], {k: v.cpu().numpy().copy() for k, v in stats.items()}

a, sa = run(1)
a2, _ = run(1)
print("default repeat equal:", all(np.array_equal(x, y) for x, y in zip(a, a2)))
for cap in (64, 16, 3, 1):
    b, sb = run(1, cap)
    for f in range(2):
        d = np.abs(a[f] - b[f])
        bad = [p for p in range(B) if d[p].max() > 0]
        print(f"cap {cap} frame {f+1}: max diff {d.max():.3e}, pairs differing {bad}, "
              f"sum a {a[f].sum():.6f} sum b {b[f].sum():.6f}")
        if bad:
            p = bad[0]
            rows = np.where(d[p].max(axis=1) > 0)[0]
            print("   rows differing (pair %d):" % p, rows[:40], "count", rows.size)
print("stats equal:", {k: np.array_equal(sa[k], sb[k]) for k in sa})
