"""GPU parity: the CUDA path (through the C ABI) against the reference and the oracle.

Tolerances (north_star): rendered images max-abs <= 1e-5 and
PSNR >= 100 dB vs the reference; bin counts, positions (advection), masks,
M, side and uint16 quantisation bit-exact.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import pytest

from oracle import generate as og
from oracle import reference
from oracle import render as orr
from _helpers import vortex_fn

pytestmark = pytest.mark.gpu

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


def test_splat_seam_host_buffers_vs_reference(pg, golden):
    """pgb_splat_accumulate (host buffers) == _native.splat_accumulate contract."""
    from paper_2512_09664_b200 import _lib

    for name, c in golden.items():
        H, W = (int(x) for x in c["hw"])
        for f in (1, 2):
            out = np.zeros((H, W), np.float32)
            args = [np.ascontiguousarray(c[k]) for k in (f"pos{f}", f"i0_{f}", f"sx_{f}", f"sy_{f}",
                                                         f"rho_{f}", f"mask{f}")]
            n = args[0].shape[0]
            _lib.call("pgb_splat_accumulate", *[a.ctypes.data for a in args], n, int(c["side"]),
                      out.ctypes.data, H, W, 0, H)
            _assert_close(out, c[f"raw{f}"], what=f"{name} frame {f}")


def test_splat_seam_accumulates_in_place_and_bands(pg, golden):
    c = golden["small_64_rho_p0"]
    H, W = (int(x) for x in c["hw"])
    args = (c["pos1"], c["i0_1"], c["sx_1"], c["sy_1"], c["rho_1"], c["mask1"], int(c["side"]))
    whole = np.zeros((H, W), np.float32)
    pg.splat_accumulate(*args, whole, 0, H)
    banded = np.zeros((H, W), np.float32)
    for lo, hi in ((0, 17), (17, 40), (40, H)):
        pg.splat_accumulate(*args, banded, lo, hi)
    np.testing.assert_array_equal(banded, whole)          # band-independent, bit-exact
    twice = whole.copy()
    pg.splat_accumulate(*args, twice, 0, H)
    np.testing.assert_allclose(twice, 2 * whole, atol=2e-6)  # in-place +=


def _render_golden(pg, c, out_mode, bg=0.0):
    import torch

    from paper_2512_09664_b200 import _lib

    H, W = (int(x) for x in c["hw"])
    dev = torch.device("cuda")
    frames, keep = [], []
    for f in (1, 2):
        t = dict(pos=torch.from_numpy(c[f"pos{f}"]).to(dev),
                 i0=torch.from_numpy(c[f"i0_{f}"]).to(dev), sx=torch.from_numpy(c[f"sx_{f}"]).to(dev),
                 sy=torch.from_numpy(c[f"sy_{f}"]).to(dev), rho=torch.from_numpy(c[f"rho_{f}"]).to(dev),
                 mask=torch.from_numpy(c[f"mask{f}"]).to(dev))
        keep.append(t)
        frames.append(_lib.PgbParticles(t["pos"].data_ptr(), t["i0"].data_ptr(), t["sx"].data_ptr(),
                                        t["sy"].data_ptr(), t["rho"].data_ptr(), t["mask"].data_ptr()))
    n = c["pos1"].shape[0]
    out = [torch.zeros((1, H, W), dtype=torch.float32, device=dev) for _ in range(2)]
    tiles = ctypes.c_int(0)
    bins = torch.full((2 * 4096,), -1, dtype=torch.int32, device=dev)
    sides = (ctypes.c_int * 1)(int(c["side"]))
    _lib.call("pgb_render_pairs_dev", ctypes.byref(frames[0]), ctypes.byref(frames[1]), n, 1, sides,
              H, W, 0, out_mode, bg, 0.0, 0, 0, 0, out[0].data_ptr(), out[1].data_ptr(),
              bins.data_ptr(), ctypes.byref(tiles), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    nt = tiles.value
    return [o[0].cpu().numpy() for o in out], bins[:2 * nt].reshape(1, 2, nt).cpu().numpy(), nt


def test_render_pairs_raw_vs_reference(pg, golden):
    from paper_2512_09664_b200 import _lib

    for name, c in golden.items():
        imgs, _, _ = _render_golden(pg, c, _lib.OUT_RAW)
        for f in (1, 2):
            _assert_close(imgs[f - 1], c[f"raw{f}"], what=f"{name} raw{f}")


def test_render_pairs_finalized_vs_reference(pg, golden):
    from paper_2512_09664_b200 import _lib

    for name, c in golden.items():
        imgs, _, _ = _render_golden(pg, c, _lib.OUT_F32, bg=0.05)
        for f in (1, 2):
            _assert_close(imgs[f - 1], c[f"fin{f}"], what=f"{name} fin{f}")


def test_bin_counts_bit_exact(pg, golden):
    from paper_2512_09664_b200 import _lib

    for name, c in golden.items():
        H, W = (int(x) for x in c["hw"])
        _, bins, tiles = _render_golden(pg, c, _lib.OUT_RAW)
        info = _lib.PgbPlanInfo()
        _lib.call("pgb_plan", H, W, c["pos1"].shape[0], 0.0, int(c["side"]) // 2, 2, ctypes.byref(info))
        assert tiles == info.tiles_y * info.tiles_x
        for f in (1, 2):
            want = orr.tile_counts(c[f"pos{f}"], c[f"mask{f}"], c[f"sx_{f}"], c[f"sy_{f}"], info.halo,
                                   info.tile_h, info.tile_w, H, W)
            np.testing.assert_array_equal(bins[0, f - 1, :tiles], want, err_msg=f"{name} f{f}")


def test_advect_and_sample_flow_bit_exact(pg, golden):
    for name, c in golden.items():
        fld = pg.FlowField(c["flow"][..., 0], c["flow"][..., 1])
        ps = pg.ParticleSet(count=c["pos1"].shape[0], pos1=c["pos1"],
                            app1=pg.Appearance(c["i0_1"], c["sx_1"], c["sy_1"], c["rho_1"]),
                            active=np.ones(c["pos1"].shape[0], bool))
        pg.advect(ps, fld)
        np.testing.assert_array_equal(ps.pos2, c["pos2"], err_msg=name)
        uv = pg.sample_flow(fld, c["pos1"])
        np.testing.assert_array_equal(uv, og.sample_flow(c["flow"], c["pos1"]), err_msg=name)


def test_sample_flow_spec_examples(pg):
    fld = pg.FlowField(np.array([[0.0, 1.0], [0.0, 1.0]], np.float32), np.zeros((2, 2), np.float32))
    assert pg.sample_flow(fld, [(0.5, 0.5)])[0, 0] == 0.5
    const = pg.FlowField(np.full((4, 4), 2.0, np.float32), np.full((4, 4), -1.0, np.float32))
    np.testing.assert_array_equal(pg.sample_flow(const, [(-5, -5), (1.3, 2.7)]), [[2, -1], [2, -1]])


def test_quantize_bit_exact(pg):
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.uniform(-0.2, 1.2, 100000).astype(np.float32),
                        (np.arange(65536, dtype=np.float32) + 0.5) / np.float32(65535),
                        np.array([0.5, 0.0, 1.0, np.nextafter(np.float32(0.5), np.float32(1))], np.float32)])
    np.testing.assert_array_equal(pg.quantize_u16(x), orr.quantize_u16(x))


def test_spec_known_answers(pg):
    one = dict(pos=np.array([[5.0, 5.0]]), i0=np.array([1.0], np.float32), sx=np.array([1.0], np.float32),
               sy=np.array([1.0], np.float32), rho=np.array([0.0], np.float32))
    ps = pg.ParticleSet(count=1, pos1=one["pos"], app1=pg.Appearance(one["i0"], one["sx"], one["sy"], one["rho"]),
                        active=np.array([True]))
    img = pg.splat(ps, 1, 11, 11, 7)
    assert img[5, 5] == pytest.approx(1.0, abs=1e-6)
    assert img[5, 6] == pytest.approx(math.exp(-0.5), abs=1e-6)
    two = pg.ParticleSet(count=2, pos1=np.repeat(one["pos"], 2, 0),
                         app1=pg.Appearance(*(np.repeat(one[k], 2) for k in ("i0", "sx", "sy", "rho"))),
                         active=np.array([True, True]))
    np.testing.assert_allclose(pg.splat(two, 1, 11, 11, 7), 2 * img, atol=1e-6)
    empty = pg.ParticleSet(count=1, pos1=one["pos"],
                           app1=pg.Appearance(one["i0"], one["sx"], one["sy"], one["rho"]),
                           active=np.array([False]))
    assert not pg.splat(empty, 1, 11, 11, 7).any()
    assert pg.eval_particle(1, 1, 1, 0.5, (0, 0), (1, 1)) == pytest.approx(math.exp(-2 / 3), rel=1e-9)


def _gen_cfg(pg, **kw):
    base = dict(image_height=64, image_width=64, batch_size=4, seeding_density_range=(0.05, 0.1),
                diameter_range=(0.5, 4.0), rho_range=(-0.5, 0.5), frame2_sigma_std=0.05,
                frame2_intensity_std=0.05, frame2_rho_std=0.05, hide_probability=0.1, seed=9,
                flow_sources=(pg.FlowSource(function="vortex"),))
    base.update(kw)
    return pg.GeneratorConfig(**base)


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


@pytest.mark.parametrize("kw", [
    dict(),
    dict(image_height=256, image_width=256, seeding_density_range=(0.06, 0.06), diameter_range=(0.8, 1.2),
         rho_range=(0.0, 0.0), frame2_sigma_std=0.0, frame2_intensity_std=0.0, frame2_rho_std=0.0,
         hide_probability=0.0),
    dict(image_height=48, image_width=80, laser_sheet={"thickness": 1.0, "shape": 2.0, "out_of_plane": 0.1}),
])
def test_generated_particles_match_oracle(pg, kw):
    import torch

    cfg = _gen_cfg(pg, **kw)
    H, W = cfg.image_height, cfg.image_width
    flow = pg.from_function(vortex_fn(H, W), H, W)
    flows = flow.to_device().unsqueeze(0)
    arr = pg.particles.generate_particle_arrays(cfg, 3, range(0, cfg.batch_size), flows=flows,
                                                pairs_per_field=cfg.batch_size)
    oc = _oracle_cfg(cfg)
    for p in range(cfg.batch_size):
        o = og.sample_pair(oc, 3, p, flow.interleaved())
        g = {k: v[p].cpu().numpy() for k, v in arr.items() if v.ndim >= 2}
        assert int(arr["active_count"][p]) == o["M"]
        assert int(arr["side"][p]) == o["side"]
        assert float(arr["seeding_density"][p]) == o["ppp"]
        for k in ("pos1", "pos2", "sx_1", "sy_1", "rho_1", "diameter"):
            np.testing.assert_array_equal(g[k], o[k], err_msg=k)
        np.testing.assert_array_equal(g["active"].astype(bool), o["active"])
        np.testing.assert_array_equal(g["visible1"].astype(bool), o["visible1"])
        np.testing.assert_array_equal(g["visible2"].astype(bool), o["visible2"])
        if cfg.laser_sheet is None:
            np.testing.assert_array_equal(g["i0_1"], o["i0_1"])
        for k in ("i0_1", "i0_2", "sx_2", "sy_2", "rho_2"):
            np.testing.assert_allclose(g[k], o[k], rtol=2e-5, atol=2e-6, err_msg=k)
    torch.cuda.synchronize()


@pytest.mark.parametrize("kw", [
    dict(),
    dict(image_height=256, image_width=256, batch_size=3, seeding_density_range=(0.06, 0.06),
         diameter_range=(0.8, 1.2), rho_range=(0.0, 0.0), frame2_sigma_std=0.0,
         frame2_intensity_std=0.0, frame2_rho_std=0.0, hide_probability=0.0),
    dict(image_height=96, image_width=160, batch_size=2, seeding_density_range=(0.1, 0.1),
         diameter_range=(1.0, 4.0), rho_range=(0.0, 0.0)),
])
def test_fused_generate_raw_matches_oracle_render(pg, kw):
    import torch

    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    cfg = _gen_cfg(pg, **kw)
    H, W, B = cfg.image_height, cfg.image_width, cfg.batch_size
    flow = pg.from_function(vortex_fn(H, W), H, W)
    flows = flow.to_device().unsqueeze(0)
    img = [torch.empty((B, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
    _lib.call("pgb_generate_batch_dev", native_config(cfg), 5, 0, B, flows.data_ptr(), 1, B,
              _lib.OUT_RAW, img[0].data_ptr(), img[1].data_ptr(), None, None,
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert _lib.load().pgb_overflow_count() == 0
    oc = _oracle_cfg(cfg)
    for p in range(B):
        o = og.sample_pair(oc, 5, p, flow.interleaved())
        for f in (1, 2):
            want = orr.splat(o[f"pos{f}"], o[f"i0_{f}"], o[f"sx_{f}"], o[f"sy_{f}"], o[f"rho_{f}"],
                             o[f"on{f}"], o["side"], H, W)
            _assert_close(img[f - 1][p].cpu().numpy(), want, tol=2e-5 if cfg.frame2_sigma_std else TOL,
                          what=f"pair {p} frame {f}")


def test_fused_generate_final_with_noise_matches_oracle(pg):
    import torch

    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    cfg = _gen_cfg(pg, image_height=64, image_width=96, batch_size=2, rho_range=(0.0, 0.0),
                   frame2_sigma_std=0.0, frame2_intensity_std=0.0, frame2_rho_std=0.0,
                   noise=pg.NoiseConfig(background_offset=0.05, gaussian_std=0.02))
    H, W, B = cfg.image_height, cfg.image_width, cfg.batch_size
    flows = pg.from_function(vortex_fn(H, W), H, W).to_device().unsqueeze(0)
    out = {}
    for mode in (_lib.OUT_RAW, _lib.OUT_F32, _lib.OUT_U16):
        dt = torch.uint16 if mode == _lib.OUT_U16 else torch.float32
        img = [torch.empty((B, H, W), dtype=dt, device="cuda") for _ in range(2)]
        _lib.call("pgb_generate_batch_dev", native_config(cfg), 2, 0, B, flows.data_ptr(), 1, B, mode,
                  img[0].data_ptr(), img[1].data_ptr(), None, None, torch.cuda.current_stream().cuda_stream)
        out[mode] = [i.cpu().numpy() for i in img]
    for p in range(B):
        for f in (1, 2):
            raw = out[_lib.OUT_RAW][f - 1][p]
            want = orr.finalize(raw, 0.05, 0.02, seed=cfg.seed, batch=2, gpair=p, frame=f)
            _assert_close(out[_lib.OUT_F32][f - 1][p], want, tol=2e-6, what=f"fin p{p} f{f}")
            # fused uint16 == quantize_u16(fused float32), bit-exact
            np.testing.assert_array_equal(out[_lib.OUT_U16][f - 1][p],
                                          orr.quantize_u16(out[_lib.OUT_F32][f - 1][p]))
    # standalone finalize kernel uses the same noise stream as the fused epilogue
    raw_t = torch.from_numpy(np.stack(out[_lib.OUT_RAW][0])).cuda()
    fin = pg.finalize(raw_t, cfg.noise, pg.RngKey(cfg.seed, 2, 0), frame=1)
    np.testing.assert_array_equal(fin.cpu().numpy(), np.stack(out[_lib.OUT_F32][0]))


def test_sharding_and_determinism_bit_identical(pg):
    import torch

    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    cfg = _gen_cfg(pg, image_height=128, image_width=128, batch_size=8)
    H, W, B = 128, 128, 8
    flows = pg.from_function(vortex_fn(H, W), H, W).to_device().unsqueeze(0)

    def run(base, count):
        img = [torch.empty((count, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
        _lib.call("pgb_generate_batch_dev", native_config(cfg), 1, base, count, flows.data_ptr(), 1, B,
                  _lib.OUT_F32, img[0].data_ptr(), img[1].data_ptr(), None, None,
                  torch.cuda.current_stream().cuda_stream)
        return [i.cpu().numpy() for i in img]

    full = run(0, 8)
    again = run(0, 8)
    halves = [run(0, 3), run(3, 5)]
    for f in range(2):
        np.testing.assert_array_equal(full[f], again[f])
        np.testing.assert_array_equal(full[f], np.concatenate([halves[0][f], halves[1][f]]))


def test_erf_psf_matches_oracle(pg, golden):
    for name in ("small_64_rho_p0", "small_64_dense_p1", "rect_48x80_p1"):
        c = golden[name]
        H, W = (int(x) for x in c["hw"])
        for f in (1, 2):
            args = (c[f"pos{f}"], c[f"i0_{f}"], c[f"sx_{f}"], c[f"sy_{f}"], c[f"rho_{f}"], c[f"mask{f}"],
                    int(c["side"]))
            got = np.zeros((H, W), np.float32)
            pg.splat_accumulate(*args, got, 0, H, psf="erf")
            want = orr.render_erf(*args, H, W)
            _assert_close(got, want, tol=2e-5, psnr=90, what=f"{name} erf f{f}")


@pytest.mark.parametrize("seed", range(10))
def test_spec_oracle_equivalence_random_configs(pg, seed):
    """SPEC.md:600 (100 random 64^2 configs; 10 per test x 10 seeds): GPU splat vs the
    REAL reference's splat (oracle/_ref) or, if absent, the bit-equal restatement."""
    rng = np.random.default_rng(1000 + seed)
    use_ref = reference.available()
    if use_ref:
        reference.load()
        from pivgen import config as rc
        from pivgen import particles as rp
        from pivgen import raster as rr
        from pivgen.rng import pair_key as rkey
    for k in range(10):
        ppp = float(rng.uniform(0.01, 0.1))
        dmax = float(rng.uniform(0.6, 4.0))
        dmin = float(rng.uniform(0.3, dmax))
        rho = float(rng.uniform(0.0, 0.5))
        if use_ref:
            cfg = rc.GeneratorConfig(image_height=64, image_width=64, seeding_density_range=(ppp / 2, ppp),
                                     diameter_range=(dmin, dmax), rho_range=(-rho, rho),
                                     seed=int(rng.integers(1 << 30)))
            ps, params = rp.sample_particles(rkey(cfg.seed, 0, k), cfg)
            side = rr.patch_side(float(params.diameters[:params.active_count].max())
                                 if params.active_count else dmax)
            want = rr.splat(ps, 1, 64, 64, side)
            mask = rr.contribution_mask(ps, 1)
            pos, app = ps.pos1, ps.app1
            got = np.zeros((64, 64), np.float32)
            pg.splat_accumulate(pos, app.i0, app.sigma_x, app.sigma_y, app.rho, mask, side, got, 0, 64)
        else:
            oc = og.GenConfig(height=64, width=64, seed=k, ppp_range=(ppp / 2, ppp), d_range=(dmin, dmax),
                              rho_range=(-rho, rho))
            o = og.sample_pair(oc, 0, k, np.zeros((64, 64, 2), np.float32))
            side = o["side"]
            args = (o["pos1"], o["i0_1"], o["sx_1"], o["sy_1"], o["rho_1"], o["on1"], side)
            want = orr.splat(*args, 64, 64)
            got = np.zeros((64, 64), np.float32)
            pg.splat_accumulate(*args, got, 0, 64)
        _assert_close(got, want, what=f"config {seed}/{k}")


@pytest.mark.parametrize("env", [
    {},                                   # defaults: dynamic schedule, split last round, two control heads
    {"PGB_NO_SPLIT": "1"},               # whole tiles only
    {"PGB_TILE": "16,128"},              # other tilings: the integer accumulation and the
    {"PGB_TILE": "32,64"},               # Q17 positions make every pixel tiling-independent
    {"PGB_GRID": "1"},                   # one CTA runs every prologue and band ticket in order
    {"PGB_GRID": "7"},                   # far fewer CTAs than SMs (MPS / green-context limits)
])
@pytest.mark.parametrize("sep", [False, True])
@pytest.mark.parametrize("hw", [(128, 128), (64, 1040)])
def test_schedule_and_store_paths_bit_identical(pg, env, sep, hw, monkeypatch):
    """Every schedule / tiling / grid size yields the same bits as a cold
    default launch of the same batch, over consecutive batches on one stream
    (the two alternating control heads). PGB_GRID caps the grid: prologue and
    band items come from one ordered ticket sequence, so a single CTA
    completes the batch (forward progress needs no co-resident CTAs)."""
    import torch

    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    H, W = hw
    B = 12
    extra = dict(diameter_range=(0.8, 1.2), rho_range=(0.0, 0.0), frame2_sigma_std=0.0,
                 frame2_intensity_std=0.0, frame2_rho_std=0.0, hide_probability=0.0) if sep else {}
    cfg = _gen_cfg(pg, image_height=H, image_width=W, batch_size=B, **extra)
    flows = pg.from_function(vortex_fn(H, W), H, W).to_device().unsqueeze(0)
    stream = torch.cuda.current_stream()

    def run(batch, mode=_lib.OUT_F32):
        img = [torch.empty((B, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
        _lib.call("pgb_generate_batch_dev", native_config(cfg), batch, 0, B, flows.data_ptr(), 1, B, mode,
                  img[0].data_ptr(), img[1].data_ptr(), None, None, stream.cuda_stream)
        return [i.cpu().numpy() for i in img]

    ref = {}
    for b in range(4):
        run(99)                     # break any cached prologue
        ref[b] = run(b)             # cold launch of batch b
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    run(0)
    for b in range(1, 4):           # consecutive batches: warm pipeline
        got = run(b)
        for f in range(2):
            np.testing.assert_array_equal(got[f], ref[b][f], err_msg=f"{env} batch {b} frame {f + 1}")


@pytest.mark.parametrize("env", [{}, {"PGB_GRID": "1"}, {"PGB_GRID": "5"}, {"PGB_TILE": "64,128"}])
def test_split_prologue_dense_pairs(pg, env, monkeypatch):
    """Dense pairs split their prologue over CTAs (histogram parts and
    particle -> cell windows as their own tickets; 512^2 at ppp <= 0.25: four
    parts, three windows). Pair 0 matches the oracle render of the oracle
    particles (whose positions follow the cell histogram and counting-sort
    order exactly), and every grid / tiling gives the same bits: each ticket
    waits only on earlier tickets."""
    import torch

    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    H, W, B = 512, 512, 3
    cfg = _gen_cfg(pg, image_height=H, image_width=W, batch_size=B, seeding_density_range=(0.2, 0.25),
                   diameter_range=(1.0, 4.0), rho_range=(0.0, 0.0), frame2_sigma_std=0.0,
                   frame2_intensity_std=0.0, frame2_rho_std=0.0, hide_probability=0.0)
    flow = pg.from_function(vortex_fn(H, W), H, W)
    flows = flow.to_device().unsqueeze(0)
    stream = torch.cuda.current_stream()

    def run():
        img = [torch.empty((B, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
        _lib.call("pgb_generate_batch_dev", native_config(cfg), 5, 0, B, flows.data_ptr(), 1, B, _lib.OUT_RAW,
                  img[0].data_ptr(), img[1].data_ptr(), None, None, stream.cuda_stream)
        return [i.cpu().numpy() for i in img]

    want = run()
    o = og.sample_pair(_oracle_cfg(cfg), 5, 0, flow.interleaved())
    for f in (1, 2):
        ref = orr.splat(o[f"pos{f}"], o[f"i0_{f}"], o[f"sx_{f}"], o[f"sy_{f}"], o[f"rho_{f}"], o[f"on{f}"],
                        o["side"], H, W)
        _assert_close(want[f - 1][0], ref, what=f"split prologue frame {f}")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    got = run()
    for f in range(2):
        np.testing.assert_array_equal(got[f], want[f], err_msg=f"{env} frame {f + 1}")


def test_match_histogram_kernel_bit_exact(pg):
    """CUDA histogram specification (csrc/histmatch.cuh) vs the reference's own
    outputs (golden) and the oracle: single images, one batched launch over a
    stack, and in place."""
    import os

    import torch

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "histmatch_cases.npz"))
    inames = sorted({k.split("/")[1] for k in g.files if k.startswith("img/")})
    tnames = sorted({k.split("/")[1] for k in g.files if k.startswith("tgt/")})
    for t in tnames:
        tgt = g[f"tgt/{t}"]
        for i in inames:
            got = pg.match_histogram(g[f"img/{i}"], tgt)
            np.testing.assert_array_equal(got, g[f"out/{i}/{t}"], err_msg=f"{i}/{t}")
        stack = torch.from_numpy(np.stack([g[f"img/{i}"] for i in inames])).cuda()
        pg.match_histogram(stack, tgt, out=stack)
        for n, i in enumerate(inames):
            np.testing.assert_array_equal(stack[n].cpu().numpy(), g[f"out/{i}/{t}"], err_msg=f"stack {i}/{t}")
    rng = np.random.default_rng(5)
    for shape in ((37, 53), (3, 256, 256), (2, 17, 31)):
        img = rng.uniform(-0.1, 1.1, shape).astype(np.float32)
        tgt = rng.uniform(0, 1, 256)
        got = pg.match_histogram(img, tgt)
        want = np.stack([orr.match_histogram(x, tgt) for x in img.reshape(-1, *shape[-2:])]).reshape(shape)
        np.testing.assert_array_equal(got, want)


def test_sampler_target_histogram_float_and_u16(pg):
    """Sampler with target_histogram: every frame equals match_histogram of the
    plain frame (float32), and the uint16 output is its quantisation."""
    tgt = tuple(float(x) for x in np.exp(-np.arange(256) / 40.0))
    pg.register_flow_function("vortex64", vortex_fn(64, 64))
    base = pg.GeneratorConfig(image_height=64, image_width=64, batch_size=3, seed=21,
                              flow_sources=(pg.FlowSource(function="vortex64"),))
    with pg.make_sampler(base) as s:
        plain = next(s)
    with pg.make_sampler(pg.with_updates(base, target_histogram=tgt)) as s:
        matched = next(s)
    with pg.make_sampler(pg.with_updates(base, target_histogram=tgt, output_dtype="uint16")) as s:
        q = next(s)
    for a, b, c in ((plain.images1, matched.images1, q.images1), (plain.images2, matched.images2, q.images2)):
        for p in range(3):
            want = orr.match_histogram(a[p].cpu().numpy(), tgt)
            np.testing.assert_array_equal(b[p].cpu().numpy(), want)
            np.testing.assert_array_equal(c[p].cpu().numpy(), orr.quantize_u16(want))


def _bench_cfg(pg, name, batch=None):
    import bench

    H, W, B = bench.CONFIGS[name][:3]
    pg.register_flow_function("bench_vortex", bench.vortex(H, W))
    pg.register_flow_function("bench_uniform", bench.uniform)
    return bench.make_cfg(pg, name, batch or B), H, W, batch or B, bench.vortex(H, W)


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_full_size_configs_properties(pg, name):
    """BASELINE configs at full size (size-independent properties):
    repeatable, the union of two shards equals the whole batch, finalized
    intensities in [0, 1], and frame statistics consistent with the seeding."""
    import torch

    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    cfg, H, W, B, fn = _bench_cfg(pg, name)
    flows = pg.from_function(fn, H, W).to_device().unsqueeze(0)
    ncfg = native_config(cfg)

    def run(base, count, batch=3):
        img = [torch.empty((count, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
        _lib.call("pgb_generate_batch_dev", ncfg, batch, base, count, flows.data_ptr(), 1, B, _lib.OUT_F32,
                  img[0].data_ptr(), img[1].data_ptr(), None, None, torch.cuda.current_stream().cuda_stream)
        return img

    a = run(0, B)
    b = run(0, B)
    h = B // 2 + 1
    s1, s2 = run(0, h), run(h, B - h)
    for f in range(2):
        assert torch.equal(a[f], b[f]), f"{name}: not repeatable"
        assert torch.equal(a[f][:h], s1[f]) and torch.equal(a[f][h:], s2[f]), f"{name}: shards differ"
        assert float(a[f].min()) >= 0.0 and float(a[f].max()) <= 1.0
    c = run(0, B, batch=4)
    assert not torch.equal(a[0], c[0]), "batches must differ"
    if name == "c2":
        # mean raw intensity per pixel ~ ppp * E[2 pi sigma^2] (I0 = 1, images clipped at 1)
        sig2 = np.mean((np.linspace(0.8, 1.2, 10001) / 4.0) ** 2)
        expect = 0.06 * 2 * np.pi * sig2
        mean = float(a[0].mean())
        assert 0.8 * expect < mean < 1.05 * expect, (mean, expect)


def test_generate_edge_cases(pg):
    """Empty seeding (M = 0), a single pair, tiny and odd image sizes, very
    large particles (dynamic windows): the fused generator matches the oracle
    render of the oracle particles."""
    import torch

    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    cases = [
        dict(image_height=16, image_width=16, batch_size=2, seeding_density_range=(0.001, 0.001)),   # M = 0
        dict(image_height=2, image_width=2, batch_size=1, seeding_density_range=(0.5, 0.5)),
        dict(image_height=7, image_width=13, batch_size=1, seeding_density_range=(0.1, 0.1)),
        dict(image_height=40, image_width=36, batch_size=2, seeding_density_range=(0.01, 0.01),
             diameter_range=(6.0, 9.0)),
        dict(image_height=33, image_width=65, batch_size=3, seeding_density_range=(0.05, 0.08),
             diameter_range=(0.5, 3.0), rho_range=(-0.4, 0.4)),
        dict(image_height=20, image_width=1030, batch_size=2, seeding_density_range=(0.05, 0.05)),
    ]
    for kw in cases:
        kw = dict(kw, seed=77, flow_sources=(pg.FlowSource(function="edge"),))
        cfg = pg.GeneratorConfig(**kw)
        H, W, B = cfg.image_height, cfg.image_width, cfg.batch_size
        fld = pg.from_function(lambda x, y: (0.3 + 0.01 * y, -0.2 + 0.02 * x), H, W)
        flows = fld.to_device().unsqueeze(0)
        img = [torch.empty((B, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
        _lib.call("pgb_generate_batch_dev", native_config(cfg), 2, 0, B, flows.data_ptr(), 1, B, _lib.OUT_RAW,
                  img[0].data_ptr(), img[1].data_ptr(), None, None, torch.cuda.current_stream().cuda_stream)
        oc = _oracle_cfg(cfg)
        for p in range(B):
            o = og.sample_pair(oc, 2, p, fld.interleaved())
            for f in (1, 2):
                want = orr.splat(o[f"pos{f}"], o[f"i0_{f}"], o[f"sx_{f}"], o[f"sy_{f}"], o[f"rho_{f}"],
                                 o[f"on{f}"], o["side"], H, W)
                _assert_close(img[f - 1][p].cpu().numpy(), want, what=f"{kw} p{p} f{f}")
        if kw["seeding_density_range"] == (0.001, 0.001):
            assert float(img[0].abs().max()) == 0.0 and float(img[1].abs().max()) == 0.0


def test_concurrent_streams_have_private_workspaces(pg):
    """Launches on two streams may overlap on the device: each (device, stream)
    has its own tables and control heads, so both results equal serial runs."""
    import torch

    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    H, W, B = 128, 128, 40
    cfg = _gen_cfg(pg, image_height=H, image_width=W, batch_size=B)
    flows = pg.from_function(vortex_fn(H, W), H, W).to_device().unsqueeze(0)
    ncfg = native_config(cfg)

    def launch(batch, base, count, stream):
        img = [torch.empty((count, H, W), dtype=torch.float32, device="cuda") for _ in range(2)]
        _lib.call("pgb_generate_batch_dev", ncfg, batch, base, count, flows.data_ptr(), 1, B, _lib.OUT_F32,
                  img[0].data_ptr(), img[1].data_ptr(), None, None, stream.cuda_stream)
        return img

    main = torch.cuda.current_stream()
    want = [launch(b, 0, B, main) for b in (5, 6, 7)]
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    got = []
    for b, s in ((5, s1), (6, s2), (7, s1)):
        got.append(launch(b, 0, B, s))
    part = launch(6, 10, 17, s2)   # different pair count on the same stream
    torch.cuda.synchronize()
    for w, g in zip(want, got):
        for f in range(2):
            assert torch.equal(w[f], g[f])
    for f in range(2):
        assert torch.equal(part[f], want[1][f][10:27])


@pytest.mark.parametrize("mode,pinned,B", [("f32", True, 100), ("u16", False, 70), ("f32", False, 7)])
def test_host_buffer_pipeline_equals_device_path(pg, mode, pinned, B):
    """pgb_generate_batch (HOST buffers, chunked kernel + D2H pipeline on two
    streams) returns exactly the device path's images and pair statistics,
    for ragged chunkings, pinned and pageable buffers."""
    import torch

    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    H, W = 96, 128
    cfg = _gen_cfg(pg, image_height=H, image_width=W, batch_size=B,
                   noise=pg.NoiseConfig(background_offset=0.05, gaussian_std=0.02))
    field = pg.from_function(vortex_fn(H, W), H, W)
    flows = field.to_device().unsqueeze(0)
    ncfg = native_config(cfg)
    om, dt, ndt = ((_lib.OUT_F32, torch.float32, np.float32) if mode == "f32"
                   else (_lib.OUT_U16, torch.uint16, np.uint16))
    base = 3
    dev = [torch.empty((B, H, W), dtype=dt, device="cuda") for _ in range(2)]
    dst = {"seeding_density": torch.empty(B, dtype=torch.float64, device="cuda"),
           "active_count": torch.empty(B, dtype=torch.int32, device="cuda"),
           "side": torch.empty(B, dtype=torch.int32, device="cuda"),
           "d_max": torch.empty(B, dtype=torch.float32, device="cuda")}
    st = _lib.PgbPairStats(**{k: v.data_ptr() for k, v in dst.items()})
    _lib.call("pgb_generate_batch_dev", ncfg, 9, base, B, flows.data_ptr(), 1, B + base, om,
              dev[0].data_ptr(), dev[1].data_ptr(), st, None, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    if pinned:
        host = [torch.empty((B, H, W), dtype=dt).pin_memory() for _ in range(2)]
        hptr = [h.data_ptr() for h in host]
        harr = [h.numpy() for h in host]
    else:
        harr = [np.empty((B, H, W), dtype=ndt) for _ in range(2)]
        hptr = [a.ctypes.data for a in harr]
    hst = {"seeding_density": np.empty(B, np.float64), "active_count": np.empty(B, np.int32),
           "side": np.empty(B, np.int32), "d_max": np.empty(B, np.float32)}
    hs = _lib.PgbPairStats(**{k: v.ctypes.data for k, v in hst.items()})
    hflow = np.ascontiguousarray(field.interleaved())
    _lib.call("pgb_generate_batch", ncfg, 9, base, B, hflow.ctypes.data, 1, B + base, om, hptr[0], hptr[1], hs)
    for f in range(2):
        np.testing.assert_array_equal(harr[f], dev[f].cpu().numpy())
    for k, v in dst.items():
        np.testing.assert_array_equal(hst[k], v.cpu().numpy())
