"""Small-config smoke of every generator entry (debug aid): prints after each call."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_09664_b200 as pg  # noqa: E402
from paper_2512_09664_b200 import _lib  # noqa: E402
from paper_2512_09664_b200.particles import native_config  # noqa: E402

H, W = int(sys.argv[1]) if len(sys.argv) > 1 else 40, int(sys.argv[2]) if len(sys.argv) > 2 else 48
B = 3
pg.register_flow_function("dbg", lambda x, y: (1.0 + 0.0 * x, 0.5 + 0.0 * y))
cfg = pg.GeneratorConfig(image_height=H, image_width=W, batch_size=B, seed=8,
                         flow_sources=(pg.FlowSource(function="dbg"),))
fld = pg.from_function(lambda x, y: (1.0 + 0.0 * x, 0.5 + 0.0 * y), H, W)
flows = fld.to_device().unsqueeze(0)
imgs = [torch.empty((B, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
print("generate_batch_dev ...", flush=True)
_lib.call("pgb_generate_batch_dev", native_config(cfg), 7, 0, B, flows.data_ptr(), 1, B,
          _lib.OUT_RAW, imgs[0].data_ptr(), imgs[1].data_ptr(), None, None,
          torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("  ok", float(imgs[0].sum()), flush=True)
print("sample_particles ...", flush=True)
arr = pg.particles.generate_particle_arrays(cfg, 1, range(0, B), flows=flows, pairs_per_field=B)
torch.cuda.synchronize()
print("  ok", {k: tuple(v.shape) for k, v in list(arr.items())[:3]}, flush=True)
print("sampler ...", flush=True)
with pg.make_sampler(cfg, start_batch=5, max_batches=2) as s:
    for b in s:
        print("  batch", b.batch_index, float(b.images1.sum()), flush=True)
        p = b.params
        print("  params ok", flush=True)
print("done", flush=True)
