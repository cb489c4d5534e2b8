"""Test helpers shared by the suites (importable as `_helpers`)."""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def constant_field(height, width, u, v):
    from paper_2512_09664_b200 import FlowField

    return FlowField(np.full((height, width), u, np.float32), np.full((height, width), v, np.float32))


def write_constant_flo(path, height, width, u, v):
    from paper_2512_09664_b200 import write_flo_file

    write_flo_file(path, constant_field(height, width, u, v))
    return path


def small_config(source_paths, height=64, width=64, **overrides):
    from paper_2512_09664_b200 import FlowSource, GeneratorConfig

    defaults = dict(image_height=height, image_width=width, batch_size=2, flow_fields_per_batch=1,
                    seeding_density_range=(0.02, 0.02), diameter_range=(0.8, 1.2),
                    peak_intensity_range=(0.6, 1.0),
                    flow_sources=tuple(FlowSource(path=p) for p in source_paths),
                    seed=11, threads=1)
    defaults.update(overrides)
    return GeneratorConfig(**defaults)


def assert_trees_identical(dir_a, dir_b):
    names_a = sorted(os.listdir(dir_a))
    assert names_a == sorted(os.listdir(dir_b))
    for name in names_a:
        with open(os.path.join(dir_a, name), "rb") as fa, open(os.path.join(dir_b, name), "rb") as fb:
            assert fa.read() == fb.read(), f"{name} differs"


def vortex_fn(h, w, scale=2.0):
    """Lamb-Oseen vortex: r_c = 0.1 W, v = 1.398 U (rc/r)(1 - e^{-(r/rc)^2})."""
    def fn(x, y):
        cx, cy = (w - 1) / 2.0, (h - 1) / 2.0
        rc = 0.1 * w
        dx, dy = x - cx, y - cy
        r = np.sqrt(dx * dx + dy * dy) + 1e-12
        vt = 1.398 * scale * (rc / r) * (1.0 - np.exp(-(r / rc) ** 2))
        return -vt * dy / r, vt * dx / r
    return fn
