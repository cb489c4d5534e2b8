"""Export writers against the reference's own writers
(export.py, via oracle/_ref): identical bytes for png16 / raw_f32 / .flo."""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import reference
from _helpers import vortex_fn

needs_ref = pytest.mark.skipif(not reference.available(), reason="oracle/_ref not built")


def _images():
    rng = np.random.default_rng(3)
    return [rng.uniform(-0.05, 1.05, (37, 53)).astype(np.float32),
            np.linspace(0, 1, 64 * 48, dtype=np.float32).reshape(48, 64),
            np.full((8, 9), 0.5, np.float32)]


@needs_ref
def test_png16_and_raw_bytes_match_reference(tmp_path):
    reference.load()
    from pivgen import export as rexp

    from paper_2512_09664_b200 import export as ex

    for k, img in enumerate(_images()):
        for name, ours, theirs in (("png", ex.write_png16, rexp.write_png16),
                                   ("raw", ex.write_raw_f32, rexp.write_raw_f32)):
            a, b = tmp_path / f"o{k}.{name}", tmp_path / f"r{k}.{name}"
            ours(str(a), img)
            theirs(str(b), img)
            assert a.read_bytes() == b.read_bytes(), f"{name} image {k}"
        # uint16 levels quantised elsewhere (the GPU path) give the same file
        q = ex.quantize_u16_host(img)
        np.testing.assert_array_equal(q, rexp.quantize_u16(img))
        c = tmp_path / f"q{k}.png"
        ex.write_png16(str(c), q)
        assert c.read_bytes() == (tmp_path / f"r{k}.png").read_bytes()
        np.testing.assert_array_equal(ex.read_png16(str(c)), rexp.read_png16(str(c)))
        np.testing.assert_array_equal(ex.read_raw_f32(str(tmp_path / f"o{k}.raw")), img)


def test_raw_reader_rejects_corrupt(tmp_path):
    from paper_2512_09664_b200 import export as ex

    p = tmp_path / "bad.raw"
    p.write_bytes(b"\x01\x00")
    with pytest.raises(ValueError):
        ex.read_raw_f32(str(p))
    p.write_bytes(np.array([2, 2], "<i4").tobytes() + b"\x00" * 12)
    with pytest.raises(ValueError):
        ex.read_raw_f32(str(p))


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["png16", "raw_f32"])
def test_generate_dataset_layout_and_contents(tmp_path, fmt):
    """generate_dataset writes the reference layout; every file decodes to the
    Sampler's own images, flows and parameters."""
    import json

    import paper_2512_09664_b200 as pg
    from paper_2512_09664_b200 import export as ex
    from paper_2512_09664_b200.config import OutputConfig
    from paper_2512_09664_b200.flowfield import load_flo_file, write_flo

    pg.register_flow_function("vortex40", vortex_fn(40, 48))
    cfg = pg.GeneratorConfig(image_height=40, image_width=48, batch_size=3, seed=8,
                             flow_sources=(pg.FlowSource(function="vortex40"),),
                             output=OutputConfig(format=fmt, directory=str(tmp_path)))
    info = ex.generate_dataset(cfg, 2, str(tmp_path), start_batch=5)
    assert info["pairs"] == 6
    ext = "png" if fmt == "png16" else "raw"
    names = sorted(os.listdir(tmp_path))
    want = sorted([os.path.basename(p) for b in (5, 6) for i in range(3) for p in ex.pair_paths("", ext, b, i)]
                  + ["params_000005.json", "params_000006.json"])
    assert names == want
    with pg.make_sampler(cfg, start_batch=5, max_batches=2) as s:
        for batch in s:
            for i in range(3):
                pa, pb, pf = ex.pair_paths(str(tmp_path), ext, batch.batch_index, i)
                for path, img in ((pa, batch.images1[i]), (pb, batch.images2[i])):
                    host = img.cpu().numpy()
                    if fmt == "png16":
                        np.testing.assert_array_equal(ex.read_png16(path),
                                                      ex.quantize_u16_host(host).astype(np.float32) / 65535.0)
                    else:
                        np.testing.assert_array_equal(ex.read_raw_f32(path), host)
                assert open(pf, "rb").read() == write_flo(batch.flow_fields[i])
                load_flo_file(pf)
            meta = json.load(open(os.path.join(tmp_path, f"params_{batch.batch_index:06d}.json")))
            assert meta == json.loads(json.dumps(ex.sidecar(cfg, batch)))
            assert meta["schema_version"] == 1 and len(meta["pairs"]) == 3
