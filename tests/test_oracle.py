"""CPU: pin the oracle restatement against the reference's golden vectors.

Runs without a GPU. The golden fixtures were produced by the real reference
(tests/golden/make_golden.py, oracle/_ref build of /root/reference/pkg).
"""

from __future__ import annotations

import math
import os

import numpy as np
import pytest

from oracle import generate as og
from oracle import philox as px
from oracle import reference
from oracle import render as orr
from _helpers import GOLDEN


def test_philox_random123_kat():
    for ctr, key, want in px.KAT:
        got = px.philox4x32_10(*ctr, *key)
        assert [int(x) for x in got] == list(want)


def test_philox_matches_nvidia_curand():
    with open(os.path.join(GOLDEN, "philox_curand.txt")) as fh:
        rows = [[int(x, 16) for x in line.split()] for line in fh if line.strip()]
    assert len(rows) == 64
    c = np.array(rows, dtype=np.uint64)
    got = px.philox4x32_10(c[:, 0], c[:, 1], c[:, 2], c[:, 3], 0, 0)  # keys differ per row
    for i, r in enumerate(rows):
        one = px.philox4x32_10(r[0], r[1], r[2], r[3], r[4], r[5])
        assert [int(x) for x in one] == r[6:], f"row {i}"
    assert got[0].shape == (64,)


def test_uniform_helpers_open_interval():
    w = np.array([0, 1, 2 ** 32 - 1], dtype=np.uint64)
    u = px.u32_to_unit(w)
    assert u[0] > 0 and u[-1] < 1
    # (2^53 - 1 + 0.5) rounds to 2^53 in float64: the top word maps to 1.0 exactly,
    # as in the reference (rng.py:93-95)
    assert px.u53_to_unit(0, 0) > 0 and px.u53_to_unit(2 ** 32 - 1, 2 ** 32 - 1) <= 1
    uf = px.u32_to_unitf(np.array([0, 2 ** 32 - 1], dtype=np.uint32))
    assert uf.dtype == np.float32 and 0 < uf[0] and uf[1] < 1


@pytest.mark.parametrize("name", ["c1_uniform_256_p0", "small_64_rho_p0", "small_64_rho_p1",
                                  "small_64_dense_p1", "rect_48x80_p0", "odd_37x53_p1"])
def test_oracle_splat_bit_equal_to_reference(golden, name):
    c = golden[name]
    H, W = (int(x) for x in c["hw"])
    for f in (1, 2):
        img = orr.splat(c[f"pos{f}"], c[f"i0_{f}"], c[f"sx_{f}"], c[f"sy_{f}"], c[f"rho_{f}"],
                        c[f"mask{f}"], int(c["side"]), H, W)
        np.testing.assert_array_equal(img, c[f"raw{f}"])


def test_oracle_finalize_matches_reference_noise_off(golden):
    for name, c in golden.items():
        for f in (1, 2):
            fin = orr.finalize(c[f"raw{f}"], 0.05, 0.0)
            np.testing.assert_array_equal(fin, c[f"fin{f}"], err_msg=name)


def test_oracle_advect_bit_equal_to_reference(golden):
    for name, c in golden.items():
        if name.startswith("c1"):
            continue
        pos2 = c["pos1"] + og.sample_flow(c["flow"], c["pos1"])
        np.testing.assert_array_equal(pos2, c["pos2"], err_msg=name)


def test_oracle_patch_side_matches_reference_rule():
    # SPEC-derived values plus staircase boundaries (raster.py:30-38)
    assert og.patch_side(1.2) == 5
    assert og.patch_side(1.0) == 5          # 3*1+1 = 4 -> odd 5
    assert og.patch_side(4.0) == 13
    assert og.patch_side(0.1) == 3
    assert og.patch_side(2.0) == 7
    assert og.patch_side(1.0 / 3.0 * 2.0) == 3


def test_oracle_particle_capacity_spec_example():
    assert og.particle_capacity(0.06, 512, 512) == 15729
    assert og.particle_capacity(0.06, 256, 256) == 3933
    assert og.particle_capacity(0.1, 1024, 1024) == 104858
    assert og.particle_capacity(0.1, 10, 10) == 10           # 9-digit guard


def test_oracle_quantize_u16_examples():
    q = orr.quantize_u16(np.array([0.0, 0.5, 1.0, 1.5, -0.2, 0.25], np.float32))
    assert q.tolist() == [0, 32768, 65535, 65535, 0, 16384]   # 0.5 -> 32768


def test_oracle_eval_known_answers():
    # SPEC.md:290-292 examples through the splat restatement
    out = orr.splat(np.array([[5.0, 5.0]]), np.array([1.0], np.float32), np.array([1.0], np.float32),
                    np.array([1.0], np.float32), np.array([0.0], np.float32), np.array([1], np.uint8),
                    7, 11, 11)
    assert out[5, 5] == pytest.approx(1.0, abs=1e-7)
    assert out[5, 6] == pytest.approx(math.exp(-0.5), abs=1e-7)
    two = orr.splat(np.array([[5.0, 5.0]] * 2), np.ones(2, np.float32), np.ones(2, np.float32),
                    np.ones(2, np.float32), np.zeros(2, np.float32), np.ones(2, np.uint8), 7, 11, 11)
    np.testing.assert_allclose(two, 2 * out, atol=1e-7)


def test_oracle_erf_converges_to_point_for_wide_psf():
    pos = np.array([[20.3, 19.6]])
    args = (np.array([1.0], np.float32), np.array([3.0], np.float32), np.array([3.0], np.float32),
            np.array([0.0], np.float32), np.array([1], np.uint8), 31, 40, 40)
    pt = orr.splat(pos, *args)
    ef = orr.render_erf(pos, *args)
    assert np.abs(pt - ef).max() < 0.01       # pixel-mean -> point value as sigma grows
    # rho != 0 quadrature path vs a dense numerical integral of one pixel
    r = 0.4
    e2 = orr.render_erf(pos, np.array([1.0], np.float32), np.array([1.0], np.float32),
                        np.array([0.8], np.float32), np.array([r], np.float32), np.array([1], np.uint8),
                        9, 40, 40)
    mid = 19.5 + (np.arange(1000) + 0.5) / 1000.0          # midpoint rule on the pixel
    yy, xx = np.meshgrid(mid, mid, indexing="ij")
    dx, dy = xx - pos[0, 0], yy - pos[0, 1]
    q = 1 - r * r
    g = np.exp(-(dx * dx / 1.0 - 2 * r * dx * dy / 0.8 + dy * dy / 0.64) / (2 * q))
    assert e2[20, 20] == pytest.approx(g.mean(), abs=2e-5)


def test_oracle_tile_counts_cover_every_window():
    rng = np.random.default_rng(0)
    pos = rng.uniform(4, 60, size=(500, 2))
    on = rng.random(500) < 0.9
    sig = np.full(500, 0.25, np.float32)
    counts = orr.tile_counts(pos, on, sig, sig, 2, 16, 32, 64, 64)
    assert counts.shape == (8,)
    # every interior particle lands in >= 1 tile, at most 4
    assert on.sum() <= counts.sum() <= 4 * on.sum()


def test_oracle_tight_window_is_exact():
    # every pixel outside the tight window contributes < 1/2 unit at shift 22
    rng = np.random.default_rng(5)
    for _ in range(200):
        fx, fy = rng.uniform(-0.5, 0.5, 2)
        s = np.float32(rng.uniform(0.1, 1.2))
        jlo, jhi, ilo, ihi = orr.tight_window(np.float32(fx), np.float32(fy), s, s, 20)
        for j in range(-20, 21):
            for i in (0,):
                v = 2.0 ** 22 * math.exp(-((j - float(np.float32(fx))) ** 2) / (2 * float(s) ** 2))
                if j < jlo or j > jhi:
                    assert v < 0.5


@pytest.mark.skipif(not reference.available(), reason="oracle/_ref not built")
def test_oracle_generation_restatement_is_self_consistent():
    cfg = og.GenConfig(height=64, width=64, seed=3, ppp_range=(0.05, 0.1), d_range=(0.5, 4.0),
                       rho_range=(-0.5, 0.5), hide_probability=0.2, f2_sigma_std=0.1)
    flow = np.zeros((64, 64, 2), np.float32)
    a = og.sample_pair(cfg, 0, 1, flow)
    b = og.sample_pair(cfg, 0, 1, flow)
    for k in ("pos1", "i0_1", "diameter", "visible1"):
        np.testing.assert_array_equal(a[k], b[k])
    assert 0 <= a["M"] <= cfg.n
    assert a["side"] == og.patch_side(a["d_max"])
    # restated oracle render of restated particles == the real reference's splat
    pv = reference.load()
    from pivgen import particles as rp

    ps = rp.ParticleSet(count=cfg.n, pos1=a["pos1"],
                        app1=rp.Appearance(a["i0_1"], a["sx_1"], a["sy_1"], a["rho_1"]),
                        active=a["active"], visible1=a["visible1"])
    from pivgen import raster as rr

    ref_img = rr.splat(ps, 1, 64, 64, a["side"])
    mine = orr.splat(a["pos1"], a["i0_1"], a["sx_1"], a["sy_1"], a["rho_1"], a["on1"], a["side"], 64, 64)
    np.testing.assert_array_equal(ref_img, mine)
    assert pv.active_backend() == "native"


def test_reproducible_log_exp():
    rng = np.random.default_rng(3)
    for v in np.concatenate([rng.uniform(0, 1, 2000), [2.0 ** -53, 0.5, 1.0 - 2.0 ** -53, 0.7071067811865476]]):
        assert abs(og.rlog(float(v)) - math.log(v)) <= 1e-14 * max(1.0, abs(math.log(v)))
    for y in np.concatenate([rng.uniform(-40, 0, 2000), [0.0, -1e-12]]):
        assert abs(og.rexp(float(y)) - math.exp(y)) <= 1e-14 * math.exp(y)


def test_stratified_seeding_law():
    # cell histogram sums to M; positions are uniform (chi-square on 8x8 bins);
    # the maximum diameter sits on particle J and bounds every other particle
    cfg = og.GenConfig(height=96, width=128, seed=11, ppp_range=(0.2, 0.2), d_range=(0.5, 3.0))
    flow = np.zeros((96, 128, 2), np.float32)
    xs, ys = [], []
    for p in range(4):
        o = og.sample_pair(cfg, 0, p, flow)
        m = o["M"]
        assert o["prefix"][-1] == m
        d = o["diameter"][:m]
        assert d.max() == np.float32(o["d_max"]) and (d <= o["d_max"]).all()
        xs.append(o["pos1"][:m, 0])
        ys.append(o["pos1"][:m, 1])
    x, y = np.concatenate(xs), np.concatenate(ys)
    assert x.min() > 0 and x.max() < 128 and y.min() > 0 and y.max() < 96
    hist, _, _ = np.histogram2d(y, x, bins=8, range=((0, 96), (0, 128)))
    e = x.size / 64
    chi2 = ((hist - e) ** 2 / e).sum()
    assert chi2 < 120          # 63 dof: p ~ 1e-5
    # diameters below the maximum are uniform on [d_lo, d_max]
    dd = np.concatenate([og.sample_pair(cfg, 1, p, flow)["diameter"][:100] for p in range(20)])
    assert 0.4 < (dd < 1.75).mean() < 0.6


def test_match_histogram_oracle_bit_exact_vs_reference_golden():
    """oracle.render.match_histogram == reference raster.match_histogram
    (raster.py:164-187) on the committed golden cases, bit for bit."""
    import os

    from oracle import render as orr

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "histmatch_cases.npz"))
    keys = [k for k in g.files if k.startswith("out/")]
    assert len(keys) == 25
    for k in keys:
        _, iname, tname = k.split("/")
        got = orr.match_histogram(g[f"img/{iname}"], g[f"tgt/{tname}"])
        assert got.dtype == np.float32
        np.testing.assert_array_equal(got, g[k], err_msg=k)
