"""GPU: the drop-in Sampler API (reference pipeline.py:147-367, SPEC acceptance)."""

from __future__ import annotations

import threading

import numpy as np
import pytest

from _helpers import vortex_fn
from oracle import render as orr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    import paper_2512_09664_b200 as pg

    pg.register_flow_function("vortex64", vortex_fn(64, 64))
    return pg


def _cfg(pg, make_config, **kw):
    return make_config(**kw)


def test_batch_shapes_and_ranges(pg, make_config):
    cfg = make_config(batch_size=4, seeding_density_range=(0.05, 0.1), hide_probability=0.1)
    with pg.make_sampler(cfg) as s:
        b = next(s)
        assert b.images1.shape == (4, 64, 64) and b.images1.dtype.__str__() == "torch.float32"
        assert b.images1.is_cuda and b.images2.is_cuda
        x = b.images1.cpu().numpy()
        assert x.min() >= 0.0 and x.max() <= 1.0 and x.max() > 0.1
        assert len(b.flow_fields) == 4 and b.batch_index == 0
        p = b.params[0]
        assert p.diameters.shape == (cfg.particle_capacity(),)
        assert 0.05 <= p.seeding_density <= 0.1
        assert p.active_count == round(p.seeding_density * 64 * 64)
        assert (p.peak_intensities[p.active_count:] == 0).all()
        s.check_overflow()


def test_determinism_and_seek(pg, make_config):
    cfg = make_config(batch_size=3, frame2_sigma_std=0.05, hide_probability=0.1)
    with pg.make_sampler(cfg) as a, pg.make_sampler(cfg) as b:
        ba = [next(a) for _ in range(3)]
        bb = [next(b) for _ in range(3)]
    for x, y in zip(ba, bb):
        assert np.array_equal(x.images1.cpu().numpy(), y.images1.cpu().numpy())
        assert np.array_equal(x.images2.cpu().numpy(), y.images2.cpu().numpy())
    with pg.make_sampler(cfg, start_batch=2) as c:
        bc = next(c)
    assert bc.batch_index == 2
    assert np.array_equal(bc.images1.cpu().numpy(), ba[2].images1.cpu().numpy())
    assert not np.array_equal(ba[0].images1.cpu().numpy(), ba[1].images1.cpu().numpy())


def test_zero_flow_frames_identical(pg, make_config):
    # zero flow, no jitter/hide/noise -> frames bit-identical
    cfg = make_config(flows=((0.0, 0.0),), batch_size=2)
    with pg.make_sampler(cfg) as s:
        b = next(s)
    assert np.array_equal(b.images1.cpu().numpy(), b.images2.cpu().numpy())


def test_constant_flow_translation(pg, make_config):
    # constant (2, -1) -> image2 = image1 shifted, <= 1e-5 on the overlap
    cfg = make_config(flows=((2.0, -1.0),), batch_size=2, peak_intensity_range=(1.0, 1.0))
    with pg.make_sampler(cfg) as s:
        b = next(s)
    a1 = b.images1.cpu().numpy()
    a2 = b.images2.cpu().numpy()
    # pixel (r, c) of frame 2 == pixel (r + 1, c - 2) of frame 1, away from borders
    # (particles entering from outside the frame only affect a margin of the patch size)
    m = 6
    diff = np.abs(a2[:, m:-m, m:-m] - a1[:, m + 1:64 - m + 1, m - 2:64 - m - 2])
    assert diff.max() <= 1e-5


def test_uint16_output_is_quantised_float32(pg, make_config):
    cfg = make_config(batch_size=2, noise=pg.NoiseConfig(0.05, 0.01))
    cfg16 = pg.with_updates(cfg, output_dtype="uint16")
    with pg.make_sampler(cfg) as a, pg.make_sampler(cfg16) as b:
        fa, fb = next(a), next(b)
    assert str(fb.images1.dtype) == "torch.uint16"
    np.testing.assert_array_equal(fb.images1.cpu().numpy(), orr.quantize_u16(fa.images1.cpu().numpy()))


def test_flow_rotation(pg, flo_dir):
    # B = 8, F = 2 -> pairs 0-3 share a field; with R = 2 the window
    # advances only on even batch indices
    from _helpers import small_config

    paths = flo_dir(64, 64, flows=[(float(i), 0.0) for i in range(5)])
    cfg = small_config(paths, batch_size=8, flow_fields_per_batch=2, batches_per_flow_field=2)
    with pg.make_sampler(cfg) as s:
        b0, b1, b2 = next(s), next(s), next(s)
    f0 = b0.flow_fields
    assert all(f is f0[0] for f in f0[:4]) and all(f is f0[4] for f in f0[4:])
    assert f0[0] is not f0[4]
    assert b1.flow_fields[0] is f0[0]
    assert b2.flow_fields[0] is not f0[0]
    assert float(b2.flow_fields[0].u[0, 0]) == 2.0
    fl = b0.flows.cpu().numpy()
    assert fl.shape == (8, 64, 64, 2) and fl[5, 0, 0, 0] == 1.0


def test_single_consumer_and_max_batches(pg, make_config):
    cfg = make_config(batch_size=2)
    with pg.make_sampler(cfg, max_batches=2) as s:
        assert len(list(s)) == 2
    with pg.make_sampler(cfg) as s:
        s._consumer_lock.acquire()
        try:
            with pytest.raises(RuntimeError):
                s.next_batch()
        finally:
            s._consumer_lock.release()


def test_prefetch_liveness_with_corrupt_source(pg, flo_dir, tmp_path):
    # capacity 2, 5 sources with 1 corrupt -> skipped with a warning
    from _helpers import small_config

    paths = flo_dir(64, 64, flows=[(1.0, 0.0)] * 4)
    bad = tmp_path / "bad.flo"
    bad.write_bytes(b"garbage")
    paths.insert(2, str(bad))
    cfg = small_config(paths, batch_size=2)
    done = []

    def run():
        with pg.make_sampler(cfg, prefetch_capacity=2) as s:
            for _ in range(20):
                next(s)
            done.append(s.skipped_sources)

    t = threading.Thread(target=run)
    t.start()
    t.join(60)
    assert done and any("bad.flo" in m for m in done[0])


def test_sources_exhausted(pg, tmp_path):
    from _helpers import small_config

    bad = tmp_path / "bad.flo"
    bad.write_bytes(b"garbage")
    good = tmp_path / "good.flo"
    from _helpers import write_constant_flo

    write_constant_flo(str(good), 64, 64, 1.0, 0.0)
    cfg = small_config([str(good), str(bad)], batch_size=2)
    with pg.make_sampler(cfg) as s:
        next(s)  # first source loads
    cfg2 = small_config([str(bad)], batch_size=2)
    with pytest.raises(Exception):
        pg.make_sampler(cfg2)


def test_shards_concatenate_to_full_batch(pg, make_config):
    cfg = make_config(batch_size=6, hide_probability=0.2, frame2_sigma_std=0.05)
    with pg.make_sampler(cfg) as full:
        bf = next(full)
    parts = []
    for r in range(3):
        with pg.make_sampler(cfg, rank=r, world_size=3) as s:
            parts.append(next(s))
    got = np.concatenate([p.images1.cpu().numpy() for p in parts])
    assert np.array_equal(got, bf.images1.cpu().numpy())
    assert [p.pair_range for p in parts] == [range(0, 2), range(2, 4), range(4, 6)]


def test_laser_sheet_and_erf_modes_run(pg, make_config):
    cfg = make_config(batch_size=2, psf="erf",
                      laser_sheet=pg.LaserSheetConfig(thickness=1.0, shape=2.0, out_of_plane=0.1))
    with pg.make_sampler(cfg) as s:
        b = next(s)
    x = b.images1.cpu().numpy()
    assert np.isfinite(x).all() and x.max() > 0


def test_functional_layer_roundtrip(pg):
    cfg = pg.GeneratorConfig(image_height=64, image_width=64, seeding_density_range=(0.05, 0.05),
                             frame2_sigma_std=0.05, hide_probability=0.2, seed=4,
                             flow_sources=(pg.FlowSource(function="vortex64"),))
    key = pg.pair_key(4, 0, 1)
    ps, params = pg.sample_particles(key, cfg)
    fld = pg.from_function(vortex_fn(64, 64), 64, 64)
    pg.advect(ps, fld)
    ps.app2 = pg.perturb_frame2(key, ps.app1, cfg)
    pg.apply_hiding(key, ps, cfg.hide_probability)
    side = pg.patch_side(float(params.diameters[:params.active_count].max()))
    r1, r2 = pg.render_pair(ps, 64, 64, side, cfg.noise, None, key)
    # the Sampler renders the same pair (same particles; the band kernel picks
    # its own fixed-point scale, and functional advect is the reference's
    # float64 arithmetic while the generator advects in fixed point + float32)
    with pg.make_sampler(pg.with_updates(cfg, batch_size=2)) as s:
        b = next(s)
    np.testing.assert_allclose(b.images1[1].cpu().numpy(), r1, atol=1e-5)
    np.testing.assert_allclose(b.images2[1].cpu().numpy(), r2, atol=1e-5)


def test_device_evaluated_flow_function(pg):
    """register_flow_function(..., device=True): the function runs on CUDA
    tensors every window (nothing crosses PCIe); the field equals the host
    evaluation to float32 rounding and the batches match the host path."""
    import torch

    from _helpers import vortex_fn

    H, W, B = 96, 128, 4
    host_fn = vortex_fn(H, W)

    def dev_fn(x, y):
        cx, cy = (W - 1) / 2.0, (H - 1) / 2.0
        rc = 0.1 * W
        dx, dy = x - cx, y - cy
        r = torch.sqrt(dx * dx + dy * dy) + 1e-12
        vt = 1.398 * 2.0 * (rc / r) * (1.0 - torch.exp(-(r / rc) ** 2))
        return -vt * dy / r, vt * dx / r

    fd = pg.from_function_device(dev_fn, H, W)
    fh = pg.from_function(host_fn, H, W)
    assert fd.on_device(torch.device("cuda", torch.cuda.current_device()))
    np.testing.assert_allclose(fd.u, fh.u, rtol=0, atol=1e-6)
    np.testing.assert_allclose(fd.v, fh.v, rtol=0, atol=1e-6)
    out = {}
    for name, fn, dev in (("h", host_fn, False), ("d", dev_fn, True)):
        pg.register_flow_function("devflow_" + name, fn, device=dev)
        cfg = pg.GeneratorConfig(image_height=H, image_width=W, batch_size=B, seed=5,
                                 flow_sources=(pg.FlowSource(function="devflow_" + name),))
        with pg.make_sampler(cfg, max_batches=3) as s:
            out[name] = [(b.images1.cpu().numpy(), b.images2.cpu().numpy()) for b in s]
        pg.unregister_flow_function("devflow_" + name)
    for (h1, h2), (d1, d2) in zip(out["h"], out["d"]):
        np.testing.assert_array_equal(h1, d1)            # frame 1 does not depend on the flow
        assert float(np.abs(h2 - d2).max()) <= 1e-5      # float32-rounding differences of the field


def test_graph_captured_flow_function(pg):
    """register_flow_function(..., device=True, graph=True): the evaluation is
    captured once as a CUDA graph and replayed; every replay gives the eager
    field bit for bit, a Sampler over it gives the eager Sampler's images, and
    a function that cannot be captured (a host sync inside) falls back to
    eager evaluation."""
    import torch

    H, W, B = 96, 128, 4

    def dev_fn(x, y):
        return 0.5 + 0.01 * torch.sin(0.05 * x) * y, -0.25 + 0.002 * x

    eager = pg.from_function_device(dev_fn, H, W)
    for _ in range(3):
        g = pg.from_function_device(dev_fn, H, W, graph=True)
        np.testing.assert_array_equal(g.u, eager.u)
        np.testing.assert_array_equal(g.v, eager.v)

    def syncing_fn(x, y):
        s = float(x.max().item())          # a host sync: not capturable
        return 0.0 * x + 1.0 / s, 0.0 * y

    a = pg.from_function_device(syncing_fn, H, W, graph=True)
    np.testing.assert_allclose(a.u, 1.0 / (W - 1), rtol=1e-6)
    out = {}
    for name, graph in (("e", False), ("g", True)):
        pg.register_flow_function("gflow_" + name, dev_fn, device=True, graph=graph)
        cfg = pg.GeneratorConfig(image_height=H, image_width=W, batch_size=B, seed=6,
                                 flow_sources=(pg.FlowSource(function="gflow_" + name),))
        with pg.make_sampler(cfg, max_batches=3) as s:
            out[name] = [(b.images1.cpu().numpy(), b.images2.cpu().numpy()) for b in s]
        pg.unregister_flow_function("gflow_" + name)
    for (e1, e2), (g1, g2) in zip(out["e"], out["g"]):
        np.testing.assert_array_equal(e1, g1)
        np.testing.assert_array_equal(e2, g2)
