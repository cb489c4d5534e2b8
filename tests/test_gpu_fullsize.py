"""GPU parity at the BASELINE sizes (SURVEY 8(d) C3 1024^2 / C4 512^2), the
untruncated render_oracle, and oracle mode with patch sides beyond the tiled
kernel's plan (wide path).

* Oracle mode: the reference's own particle sets (live oracle/_ref, checked
  against the committed checksums in tests/golden/ref_full.npz) rendered by
  the CUDA path vs the reference splat (_native.pyx:14-66) on the full image
  and vs the committed reference crops: max-abs <= 1e-5, PSNR >= 100 dB; the
  inject kernel's per-tile counts bit-exact vs the oracle's counting rule.
* Generate mode: the band kernel at full C3 / C4 size vs the oracle
  restatement (oracle/generate.py particles, reference splat, finalize with
  the Philox noise), laser sheet and noise on for C4; erf PSF vs
  oracle/render.py render_erf.
"""

from __future__ import annotations

import ctypes
import math
import os
import sys
import threading

import numpy as np
import pytest

from oracle import generate as og
from oracle import reference
from oracle import render as orr
from _helpers import GOLDEN, vortex_fn

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not reference.available(), reason="oracle/_ref not built")

TOL = 1e-5


def _psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return math.inf if mse == 0 else 10 * math.log10(1.0 / mse)


def _assert_close(got, want, tol=TOL, psnr=100.0, what=""):
    err = float(np.abs(got.astype(np.float64) - want.astype(np.float64)).max()) if got.size else 0.0
    assert err <= tol, f"{what}: max-abs {err:.3e} > {tol:.1e}"
    assert _psnr(got, want) >= psnr, f"{what}: PSNR {_psnr(got, want):.1f} dB"


@pytest.fixture(scope="module")
def pg():
    import paper_2512_09664_b200 as pg
    from paper_2512_09664_b200 import _lib

    _lib.load()
    return pg


@pytest.fixture(scope="module")
def full():
    data = np.load(os.path.join(GOLDEN, "ref_full.npz"))
    cases = {}
    for name in data["names"]:
        prefix = f"{name}/"
        cases[str(name)] = {k[len(prefix):]: data[k] for k in data.files if k.startswith(prefix)}
    return cases


def _mg():
    if GOLDEN not in sys.path:
        sys.path.insert(0, GOLDEN)
    import make_golden

    return make_golden


def _ref_particles(name, c):
    """Live reference particles of a ref_full case, pinned by the committed checksum."""
    mg = _mg()
    pv = reference.load()
    H, W, seed, side, _, _ = (int(v) for v in c["args"])
    r = c["ranges"]
    cfg, key, ps, side2 = mg.full_case_particles(pv, name, H, W, (r[0], r[1]), (r[2], r[3]), (r[4], r[5]),
                                                 r[6], r[7], r[8], seed)
    assert side2 == side
    np.testing.assert_array_equal(mg.particle_checksum(ps), c["checksum"])
    return cfg, ps, side


def _frame_arrays(ps, f):
    pos, app = (ps.pos1, ps.app1) if f == 1 else (ps.pos2, ps.app2)
    from pivgen import raster

    mask = raster.contribution_mask(ps, f).astype(np.uint8)
    return (np.ascontiguousarray(pos), np.ascontiguousarray(app.i0), np.ascontiguousarray(app.sigma_x),
            np.ascontiguousarray(app.sigma_y), np.ascontiguousarray(app.rho), mask)


def _render_pairs(frames, side, H, W, out_mode, bg=0.0, psf=0):
    """pgb_render_pairs_dev on one pair; returns images and per-tile counts."""
    import torch

    from paper_2512_09664_b200 import _lib

    dev = torch.device("cuda")
    keep, structs = [], []
    for fr in frames:
        t = [torch.from_numpy(a).to(dev) for a in fr]
        keep.append(t)
        structs.append(_lib.PgbParticles(*[x.data_ptr() for x in t]))
    n = frames[0][0].shape[0]
    dt = torch.uint16 if out_mode == _lib.OUT_U16 else torch.float32
    out = [torch.zeros((1, H, W), dtype=dt, device=dev) for _ in range(2)]
    tiles = ctypes.c_int(0)
    bins = torch.full((2 * 65536,), -1, dtype=torch.int32, device=dev)
    sides = (ctypes.c_int * 1)(int(side))
    _lib.call("pgb_render_pairs_dev", ctypes.byref(structs[0]), ctypes.byref(structs[1]), n, 1, sides,
              H, W, psf, out_mode, bg, 0.0, 0, 0, 0, out[0].data_ptr(), out[1].data_ptr(),
              bins.data_ptr(), ctypes.byref(tiles), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    nt = tiles.value
    return [o[0].cpu().numpy() for o in out], (bins[:2 * nt].reshape(2, nt).cpu().numpy() if nt else None), nt


def _ref_splat(args, H, W):
    """The reference splat (native backend when oracle/_ref is built, else the
    bit-equal oracle restatement)."""
    if reference.available():
        reference.load()
        from pivgen import backend

        out = np.zeros((H, W), np.float32)
        backend.splat_accumulate(*args, out, 0, H)
        return out
    return orr.splat(*args, H, W)


@needs_ref
@pytest.mark.parametrize("name", ["c3_1024", "c4_512", "wide_96x128"])
def test_inject_full_size_vs_reference(pg, full, name):
    from paper_2512_09664_b200 import _lib

    reference.load()
    from pivgen import config, raster
    from pivgen.rng import STREAM_NOISE, pair_key

    c = full[name]
    H, W, seed, side, r0, c0 = (int(v) for v in c["args"])
    cfg, ps, side = _ref_particles(name, c)
    frames = [_frame_arrays(ps, f) for f in (1, 2)]
    raw, bins, nt = _render_pairs(frames, side, H, W, _lib.OUT_RAW)
    fin, _, _ = _render_pairs(frames, side, H, W, _lib.OUT_F32, bg=0.05)
    key = pair_key(seed, 0, 0)
    for f in (1, 2):
        want = raster.splat(ps, f, H, W, side)
        _assert_close(raw[f - 1], want, what=f"{name} raw{f}")
        crop = (slice(r0, r0 + 128), slice(c0, c0 + 128))
        _assert_close(raw[f - 1][crop], c[f"raw{f}_crop"], what=f"{name} raw{f} vs committed crop")
        assert abs(raw[f - 1].astype(np.float64).sum() - c[f"raw{f}_stats"][0]) <= 1e-5 * H * W
        want_fin = raster.finalize(want, config.NoiseConfig(background_offset=0.05),
                                   key.with_stream(STREAM_NOISE, lane=f))
        _assert_close(fin[f - 1], want_fin, what=f"{name} fin{f}")
        _assert_close(fin[f - 1][crop], c[f"fin{f}_crop"], what=f"{name} fin{f} vs committed crop")
        if nt:
            # per-tile counts of the inject kernel's counting sort, bit-exact
            info = _lib.PgbPlanInfo()
            _lib.call("pgb_plan", H, W, frames[0][0].shape[0], 0.0, side // 2, 2, ctypes.byref(info))
            fr = frames[f - 1]
            want_bins = orr.tile_counts(fr[0], fr[5], fr[2], fr[3], info.halo, info.tile_h, info.tile_w, H, W)
            np.testing.assert_array_equal(bins[f - 1], want_bins, err_msg=f"{name} tile counts f{f}")
        else:
            assert side > 64 or name.startswith("wide"), "only very large sides skip the tile plan"
    if name.startswith("wide"):
        assert side >= 65, "the wide case must exceed the tiled kernel's plan"
        # same images through the host seam and the splat entry point
        for f in (1, 2):
            got = np.zeros((H, W), np.float32)
            pg.splat_accumulate(*frames[f - 1], side, got, 0, H)
            _assert_close(got, c[f"raw{f}"], what=f"wide seam f{f}")


@pytest.mark.parametrize("name", ["wide_96x128"])
def test_render_oracle_untruncated_vs_reference(pg, full, name):
    """render_oracle (raster.py:129-151) on the GPU vs the reference's own
    render_oracle output (committed), float64 sums rounded once."""
    c = full[name]
    H, W = int(c["args"][0]), int(c["args"][1])
    if not reference.available():
        pytest.skip("particles come from the live reference")
    cfg, ps, side = _ref_particles(name, c)
    for f in (1, 2):
        got = pg.render_oracle(_pset(pg, ps), f, H, W)
        _assert_close(got, c[f"oracle{f}"], tol=2e-6, psnr=120, what=f"render_oracle f{f}")


def test_render_oracle_bounds_splat_truncation(pg, golden):
    """At 256^2 / C1 density the untruncated render and the truncated reference
    splat (golden) agree to the truncation error (~1.2e-7)."""
    c = golden["c1_uniform_256_p0"]
    H, W = (int(x) for x in c["hw"])
    for f in (1, 2):
        pset = pg.ParticleSet(count=c["pos1"].shape[0], pos1=c["pos1"], app1=pg.Appearance(c["i0_1"], c["sx_1"], c["sy_1"], c["rho_1"]),
                              active=c["mask1"].astype(bool) | c["mask2"].astype(bool),
                              pos2=c["pos2"], app2=pg.Appearance(c["i0_2"], c["sx_2"], c["sy_2"], c["rho_2"]),
                              visible1=c["mask1"].astype(bool), visible2=c["mask2"].astype(bool))
        got = pg.render_oracle(pset, f, H, W)
        _assert_close(got, c[f"raw{f}"], tol=1e-6, psnr=120, what=f"oracle vs splat f{f}")


def _pset(pg, ps):
    return pg.ParticleSet(count=ps.pos1.shape[0], pos1=ps.pos1, app1=pg.Appearance(ps.app1.i0, ps.app1.sigma_x, ps.app1.sigma_y, ps.app1.rho),
                          active=ps.active, pos2=ps.pos2,
                          app2=pg.Appearance(ps.app2.i0, ps.app2.sigma_x, ps.app2.sigma_y, ps.app2.rho),
                          visible1=ps.visible1, visible2=ps.visible2)


def _gen(pg, cfg, batch, pairs, mode):
    import torch

    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    H, W = cfg.image_height, cfg.image_width
    flow = pg.from_function(vortex_fn(H, W), H, W)
    flows = flow.to_device().unsqueeze(0)
    dt = torch.uint16 if mode == _lib.OUT_U16 else torch.float32
    img = [torch.empty((pairs, H, W), dtype=dt, device="cuda") for _ in range(2)]
    _lib.call("pgb_generate_batch_dev", native_config(cfg), batch, 0, pairs, flows.data_ptr(), 1, pairs, mode,
              img[0].data_ptr(), img[1].data_ptr(), None, None, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return flow, [i.cpu().numpy() for i in img]


def _oracle_cfg(cfg):
    ls = cfg.laser_sheet
    laser = None
    if ls is not None:
        zlo, zhi = ls.resolved_z_range()
        laser = dict(dz0=ls.thickness, shape=ls.shape, q=ls.efficiency, z_lo=zlo, z_hi=zhi, w=ls.out_of_plane)
    return og.GenConfig(height=cfg.image_height, width=cfg.image_width, seed=cfg.seed,
                        ppp_range=cfg.seeding_density_range, d_range=cfg.diameter_range,
                        i0_range=cfg.peak_intensity_range, rho_range=cfg.rho_range,
                        sigma_ratio=cfg.diameter_sigma_ratio, patch_multiplier=cfg.patch_multiplier,
                        f2_sigma_std=cfg.frame2_sigma_std, f2_rho_std=cfg.frame2_rho_std,
                        f2_i0_std=cfg.frame2_intensity_std, hide_probability=cfg.hide_probability,
                        laser=laser)


FULL_GEN = {
    # C3: 1024^2, ppp 0.1, d in [1, 4] (side 13) with correlated, jittered particles
    "c3": dict(image_height=1024, image_width=1024, seeding_density_range=(0.1, 0.1), diameter_range=(1.0, 4.0),
               rho_range=(-0.5, 0.5), frame2_sigma_std=0.05, frame2_intensity_std=0.05, hide_probability=0.05,
               seed=31),
    # C3 as benchmarked (uncorrelated: separable windows up to 12 px)
    "c3_bench": dict(image_height=1024, image_width=1024, seeding_density_range=(0.1, 0.1),
                     diameter_range=(1.0, 4.0), seed=0),
    # C4: 512^2, laser sheet, hiding, sensor noise
    "c4": dict(image_height=512, image_width=512, seeding_density_range=(0.06, 0.06), diameter_range=(0.8, 1.2),
               hide_probability=0.05, seed=0,
               laser_sheet={"thickness": 1.0, "shape": 2.0, "efficiency": 1.0, "out_of_plane": 0.1}),
}


@pytest.mark.parametrize("name", ["c3", "c3_bench", "c4"])
def test_generate_full_size_vs_oracle(pg, name):
    from paper_2512_09664_b200 import _lib

    kw = dict(FULL_GEN[name])
    noise = name == "c4"
    if noise:
        kw["noise"] = pg.NoiseConfig(background_offset=0.05, gaussian_std=0.02)
    cfg = pg.GeneratorConfig(batch_size=1, flow_sources=(pg.FlowSource(function="vortex"),), **kw)
    H, W = cfg.image_height, cfg.image_width
    flow, raw = _gen(pg, cfg, 3, 1, _lib.OUT_RAW)
    assert _lib.load().pgb_overflow_count() == 0
    o = og.sample_pair(_oracle_cfg(cfg), 3, 0, flow.interleaved())
    tol = 2e-5 if cfg.frame2_sigma_std else TOL
    for f in (1, 2):
        args = (o[f"pos{f}"], o[f"i0_{f}"], o[f"sx_{f}"], o[f"sy_{f}"], o[f"rho_{f}"],
                o[f"on{f}"].astype(np.uint8), o["side"])
        want = _ref_splat(args, H, W)
        _assert_close(raw[f - 1][0], want, tol=tol, what=f"{name} raw f{f}")
    if noise:
        _, fin = _gen(pg, cfg, 3, 1, _lib.OUT_F32)
        _, u16 = _gen(pg, cfg, 3, 1, _lib.OUT_U16)
        for f in (1, 2):
            want = orr.finalize(raw[f - 1][0], 0.05, 0.02, seed=cfg.seed, batch=3, gpair=0, frame=f)
            _assert_close(fin[f - 1][0], want, tol=2e-6, what=f"{name} fin f{f}")
            np.testing.assert_array_equal(u16[f - 1][0], orr.quantize_u16(fin[f - 1][0]))


@pytest.mark.parametrize("hw,kw", [
    ((96, 160), dict(seeding_density_range=(0.1, 0.1), diameter_range=(1.0, 4.0), rho_range=(-0.4, 0.4))),
    ((96, 160), dict(seeding_density_range=(0.08, 0.08), diameter_range=(0.8, 2.5))),
    ((512, 512), dict(seeding_density_range=(0.06, 0.06), diameter_range=(0.8, 1.2), hide_probability=0.05)),
])
def test_generate_erf_psf_vs_oracle(pg, hw, kw):
    """Band kernel with psf='erf' (pixel-area integration) vs the
    float64 restatement oracle/render.py render_erf on the oracle particles."""
    from paper_2512_09664_b200 import _lib

    H, W = hw
    cfg = pg.GeneratorConfig(image_height=H, image_width=W, batch_size=2, psf="erf", seed=17,
                             flow_sources=(pg.FlowSource(function="vortex"),), **kw)
    flow, raw = _gen(pg, cfg, 1, 2, _lib.OUT_RAW)
    oc = _oracle_cfg(cfg)
    for p in range(2):
        o = og.sample_pair(oc, 1, p, flow.interleaved())
        for f in (1, 2):
            want = orr.render_erf(o[f"pos{f}"], o[f"i0_{f}"], o[f"sx_{f}"], o[f"sy_{f}"], o[f"rho_{f}"],
                                  o[f"on{f}"], o["side"], H, W)
            _assert_close(raw[f - 1][p], want, tol=2e-5, psnr=95, what=f"erf {hw} p{p} f{f}")


def test_concurrent_band_calls_on_one_image(pg, golden):
    """The reference fans splat_band jobs out to a thread pool on disjoint row
    bands of one image (raster.py:116-124); concurrent host-buffer calls here
    must not lose each other's rows."""
    c = golden["small_64_dense_p1"]
    H, W = (int(x) for x in c["hw"])
    args = (c["pos1"], c["i0_1"], c["sx_1"], c["sy_1"], c["rho_1"], c["mask1"], int(c["side"]))
    whole = np.zeros((H, W), np.float32)
    pg.splat_accumulate(*args, whole, 0, H)
    for _ in range(3):
        out = np.zeros((H, W), np.float32)
        bands = [(0, 9), (9, 23), (23, 40), (40, 51), (51, H)]
        ths = [threading.Thread(target=pg.splat_accumulate, args=(*args, out, lo, hi)) for lo, hi in bands]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        np.testing.assert_array_equal(out, whole)


def test_progress_beside_a_long_kernel(pg):
    """The band kernel completes while a long kernel occupies SMs on another
    stream (its CTAs start as resources free up; no co-residency assumed)."""
    import torch

    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    H, W, B = 256, 256, 64
    cfg = pg.GeneratorConfig(image_height=H, image_width=W, batch_size=B, seed=3,
                             flow_sources=(pg.FlowSource(function="vortex"),))
    flows = pg.from_function(vortex_fn(H, W), H, W).to_device().unsqueeze(0)
    ncfg = native_config(cfg)

    def run(stream):
        img = [torch.empty((B, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
        _lib.call("pgb_generate_batch_dev", ncfg, 4, 0, B, flows.data_ptr(), 1, B, _lib.OUT_F32,
                  img[0].data_ptr(), img[1].data_ptr(), None, None, stream.cuda_stream)
        return img

    want = run(torch.cuda.current_stream())
    torch.cuda.synchronize()
    busy, work = torch.cuda.Stream(), torch.cuda.Stream()
    sink = torch.zeros(256, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    _lib.call("pgb_probe_ex2_dev", sms * 6, 20000, sink.data_ptr(), busy.cuda_stream)   # ~tens of ms
    got = run(work)
    torch.cuda.synchronize()
    for f in range(2):
        assert torch.equal(got[f], want[f])
