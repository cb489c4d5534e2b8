"""Reference-RNG mode (rng='splitmix64'): the reference's own
random streams on the GPU. Particle arrays are compared with the REAL
reference (oracle/_ref) bit for bit; Sampler images within 1e-5."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import reference
from _helpers import vortex_fn

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not reference.available(), reason="oracle/_ref not built")]

CASES = [
    dict(image_height=64, image_width=64, seeding_density_range=(0.05, 0.1), diameter_range=(0.8, 2.5)),
    dict(image_height=48, image_width=80, seeding_density_range=(0.08, 0.08), diameter_range=(0.5, 4.0),
         rho_range=(-0.5, 0.5), hide_probability=0.2),
    dict(image_height=40, image_width=56, seeding_density_range=(0.03, 0.06), diameter_range=(0.8, 1.2),
         frame2_sigma_std=0.05, frame2_intensity_std=0.05, frame2_rho_std=0.02, rho_range=(-0.3, 0.3)),
]


def _cfgs(kw, batch_size=3, **extra):
    import paper_2512_09664_b200 as pg

    pv = reference.load()
    H, W = kw["image_height"], kw["image_width"]
    name = f"refrng_{H}x{W}"
    pg.register_flow_function(name, vortex_fn(H, W))
    pv.pipeline.register_flow_function(name, vortex_fn(H, W))
    ours = pg.GeneratorConfig(batch_size=batch_size, seed=31, rng="splitmix64",
                              flow_sources=(pg.FlowSource(function=name),), **kw, **extra)
    from pivgen import config as rc

    theirs = rc.GeneratorConfig(batch_size=batch_size, seed=31, threads=1,
                                flow_sources=(rc.FlowSource(function=name),), **kw, **extra)
    return pg, pv, ours, theirs


@pytest.mark.parametrize("kw", CASES)
def test_particle_arrays_match_reference(kw):
    from paper_2512_09664_b200.particles import generate_particle_arrays_splitmix

    pg, pv, ours, theirs = _cfgs(kw)
    from pivgen import particles as rp
    from pivgen import raster as rr
    from pivgen.rng import pair_key

    H, W = kw["image_height"], kw["image_width"]
    field = pg.from_function(vortex_fn(H, W), H, W)
    rfield = pv.flowfield.from_function(vortex_fn(H, W), H, W)
    flows = field.to_device().unsqueeze(0)
    batch = 7
    arr = generate_particle_arrays_splitmix(ours, batch, range(0, 3), flows, pairs_per_field=3)
    h = {k: v.cpu().numpy() for k, v in arr.items()}
    exact_f2 = not (kw.get("frame2_sigma_std") or kw.get("frame2_intensity_std") or kw.get("frame2_rho_std"))
    for p in range(3):
        key = pair_key(31, batch, p)
        ps, params = rp.sample_particles(key, theirs)
        rp.advect(ps, rfield)
        ps.app2 = rp.perturb_frame2(key, ps.app1, theirs)
        rp.apply_hiding(key, ps, theirs.hide_probability)
        m = params.active_count
        side = rr.patch_side(float(params.diameters[:m].max()) if m else theirs.diameter_range[1])
        assert int(h["active_count"][p]) == m and int(h["side"][p]) == side
        assert float(h["seeding_density"][p]) == params.seeding_density
        np.testing.assert_array_equal(h["pos1"][p], ps.pos1)
        np.testing.assert_array_equal(h["pos2"][p], ps.pos2)
        np.testing.assert_array_equal(h["diameter"][p], params.diameters)
        for ours_k, theirs_a in (("i0_1", ps.app1.i0), ("sx_1", ps.app1.sigma_x), ("sy_1", ps.app1.sigma_y),
                                 ("rho_1", ps.app1.rho)):
            np.testing.assert_array_equal(h[ours_k][p], theirs_a, err_msg=ours_k)
        np.testing.assert_array_equal(h["active"][p].astype(bool), ps.active)
        np.testing.assert_array_equal(h["visible1"][p].astype(bool), ps.visible1)
        np.testing.assert_array_equal(h["visible2"][p].astype(bool), ps.visible2)
        for ours_k, theirs_a in (("i0_2", ps.app2.i0), ("sx_2", ps.app2.sigma_x), ("sy_2", ps.app2.sigma_y),
                                 ("rho_2", ps.app2.rho)):
            if exact_f2:
                np.testing.assert_array_equal(h[ours_k][p], theirs_a, err_msg=ours_k)
            else:   # normcdfinv vs scipy ndtri: float64 agreement to a few ulp
                np.testing.assert_allclose(h[ours_k][p], theirs_a, rtol=2e-7, atol=1e-9, err_msg=ours_k)


@pytest.mark.parametrize("kw,noise", [(CASES[0], (0.0, 0.0)), (CASES[1], (0.05, 0.02)), (CASES[2], (0.0, 0.01))])
def test_sampler_images_match_reference_sampler(kw, noise):
    """End to end with the reference's RNG: our Sampler(rng='splitmix64') vs
    the reference's Sampler on the same config (no particle injection)."""
    extra = {}
    pg, pv, ours, theirs = _cfgs(kw, batch_size=3)
    from paper_2512_09664_b200.config import NoiseConfig as N1
    from pivgen.config import NoiseConfig as N2

    ours = pg.with_updates(ours, noise=N1(*noise))
    theirs = pv.config.with_updates(theirs, noise=N2(*noise)) if hasattr(pv.config, "with_updates") else \
        type(theirs)(**{**theirs.__dict__, "noise": N2(*noise)})
    with pg.make_sampler(ours, start_batch=2, max_batches=1) as s:
        a = next(s)
    with pv.pipeline.make_sampler(theirs, start_batch=2, max_batches=1) as s:
        b = next(s)
    for x, y in ((a.images1, b.images1), (a.images2, b.images2)):
        got = x.cpu().numpy()
        err = float(np.abs(got.astype(np.float64) - y.astype(np.float64)).max())
        assert err <= 1e-5, err
    for p in range(3):
        assert a.params[p].active_count == b.params[p].active_count
        np.testing.assert_array_equal(a.params[p].diameters, b.params[p].diameters)
