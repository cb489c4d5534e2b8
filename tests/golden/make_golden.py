"""Generate golden fixtures from the REAL reference (oracle/_ref pivgen).

Run in the build container (needs oracle/_ref, built by oracle/build_ref.sh):
    python tests/golden/make_golden.py
Writes tests/golden/ref_cases.npz: reference particle sets (sample_particles ->
advect -> perturb_frame2 -> apply_hiding, pipeline.py:285-295), their patch
sides, the reference splat images of both frames (raster.splat -> native
_native.splat_accumulate) and reference finalize outputs (noise off), for
SPEC-style random configs. Also tests/golden/philox_curand.txt from NVIDIA's
curand_Philox4x32_10 (oracle/_ref/philox_curand_check).
"""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import reference  # noqa: E402

CASES = [
    # name, H, W, ppp, d_range, rho_range, sigma_std, i0_std, hide, flow, seed
    ("c1_uniform_256", 256, 256, (0.06, 0.06), (0.8, 1.2), (0.0, 0.0), 0.0, 0.0, 0.0, "uniform", 0),
    ("small_64_rho", 64, 64, (0.1, 0.1), (0.5, 4.0), (-0.5, 0.5), 0.1, 0.05, 0.1, "vortex", 11),
    ("small_64_dense", 64, 64, (0.05, 0.1), (1.0, 4.0), (0.0, 0.0), 0.0, 0.0, 0.0, "vortex", 5),
    ("rect_48x80", 48, 80, (0.08, 0.08), (0.8, 2.5), (-0.3, 0.3), 0.0, 0.0, 0.2, "uniform", 7),
    ("odd_37x53", 37, 53, (0.04, 0.07), (0.8, 1.2), (0.0, 0.0), 0.0, 0.1, 0.0, "vortex", 3),
]


def vortex(h, w):
    """Lamb-Oseen vortex centred in the image, r_c = 0.1 W, peak ~2.7 px."""
    def fn(x, y):
        cx, cy = (w - 1) / 2.0, (h - 1) / 2.0
        rc = 0.1 * w
        dx, dy = x - cx, y - cy
        r = np.sqrt(dx * dx + dy * dy) + 1e-12
        vt = 1.398 * 2.0 * (rc / r) * (1.0 - np.exp(-(r / rc) ** 2))
        return -vt * dy / r, vt * dx / r
    return fn


def main() -> None:
    pv = reference.load()
    from pivgen import config, flowfield, particles, raster
    from pivgen.rng import STREAM_NOISE, pair_key

    out = {}
    names = []
    for name, H, W, ppp, dr, rr, ss, si, hide, flow, seed in CASES:
        if flow == "uniform":
            field = flowfield.FlowField(np.full((H, W), 2.0, np.float32), np.full((H, W), -1.0, np.float32))
        else:
            field = flowfield.from_function(vortex(H, W), H, W)
        cfg = config.GeneratorConfig(image_height=H, image_width=W, seeding_density_range=ppp,
                                     diameter_range=dr, rho_range=rr, frame2_sigma_std=ss,
                                     frame2_intensity_std=si, hide_probability=hide, seed=seed)
        for pair in range(2):
            key = pair_key(seed, 0, pair)
            ps, params = particles.sample_particles(key, cfg)
            particles.advect(ps, field)
            ps.app2 = particles.perturb_frame2(key, ps.app1, cfg)
            particles.apply_hiding(key, ps, cfg.hide_probability)
            m = params.active_count
            dmax = float(params.diameters[:m].max()) if m else cfg.diameter_range[1]
            side = raster.patch_side(dmax, cfg.patch_multiplier)
            tag = f"{name}_p{pair}"
            names.append(tag)
            out[f"{tag}/hw"] = np.array([H, W])
            out[f"{tag}/side"] = np.array(side)
            out[f"{tag}/flow"] = np.stack([field.u, field.v], axis=-1)
            for f, (pos, app) in enumerate(((ps.pos1, ps.app1), (ps.pos2, ps.app2)), start=1):
                mask = raster.contribution_mask(ps, f)
                out[f"{tag}/pos{f}"] = pos
                out[f"{tag}/i0_{f}"] = app.i0
                out[f"{tag}/sx_{f}"] = app.sigma_x
                out[f"{tag}/sy_{f}"] = app.sigma_y
                out[f"{tag}/rho_{f}"] = app.rho
                out[f"{tag}/mask{f}"] = mask
                raw = raster.splat(ps, f, H, W, side)
                out[f"{tag}/raw{f}"] = raw
                fin = raster.finalize(raw, config.NoiseConfig(background_offset=0.05),
                                      key.with_stream(STREAM_NOISE, lane=f))
                out[f"{tag}/fin{f}"] = fin
    out["names"] = np.array(names)
    path = os.path.join(HERE, "ref_cases.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(names), "cases")

    make_histmatch(raster)
    make_full()

    exe = os.path.join(ROOT, "oracle", "_ref", "philox_curand_check")
    txt = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    with open(os.path.join(HERE, "philox_curand.txt"), "w") as fh:
        fh.write(txt)
    print("wrote philox_curand.txt")


# BASELINE-size cases and the wide-window / untruncated
# oracle cases. Full particle sets and images are too large to commit: the
# fixture holds each case's config, particle checksums, image statistics and
# 128 x 128 crops of the reference images; the GPU tests regenerate the
# particles with the live reference (oracle/_ref) and check them against the
# checksums, so the fixture pins the live run.
FULL_CASES = [
    # name, H, W, ppp, d_range, rho_range, sigma_std, i0_std, hide, seed, crop (r0, c0)
    ("c3_1024", 1024, 1024, (0.1, 0.1), (1.0, 4.0), (-0.5, 0.5), 0.05, 0.05, 0.05, 2, (448, 512)),
    ("c4_512", 512, 512, (0.06, 0.06), (0.8, 1.2), (0.0, 0.0), 0.0, 0.05, 0.05, 4, (192, 320)),
    ("wide_96x128", 96, 128, (0.004, 0.004), (10.0, 25.0), (-0.3, 0.3), 0.0, 0.0, 0.0, 6, (0, 0)),
]
CROP = 128


def full_case_particles(pv, name, H, W, ppp, dr, rr, ss, si, hide, seed):
    """Reference particles of pair 0, batch 0 (pipeline.py:285-295) in the vortex flow."""
    from pivgen import config, flowfield, particles, raster
    from pivgen.rng import pair_key

    field = flowfield.from_function(vortex(H, W), H, W)
    cfg = config.GeneratorConfig(image_height=H, image_width=W, seeding_density_range=ppp,
                                 diameter_range=dr, rho_range=rr, frame2_sigma_std=ss,
                                 frame2_intensity_std=si, hide_probability=hide, seed=seed)
    key = pair_key(seed, 0, 0)
    ps, params = particles.sample_particles(key, cfg)
    particles.advect(ps, field)
    ps.app2 = particles.perturb_frame2(key, ps.app1, cfg)
    particles.apply_hiding(key, ps, cfg.hide_probability)
    m = params.active_count
    dmax = float(params.diameters[:m].max()) if m else cfg.diameter_range[1]
    side = raster.patch_side(dmax, cfg.patch_multiplier)
    return cfg, key, ps, side


def particle_checksum(ps) -> np.ndarray:
    """float64 sums that change with any particle bit that matters."""
    vals = []
    for pos, app in ((ps.pos1, ps.app1), (ps.pos2, ps.app2)):
        vals += [float(np.sum(pos[:, 0])), float(np.sum(pos[:, 1])), float(np.sum(app.i0, dtype=np.float64)),
                 float(np.sum(app.sigma_x, dtype=np.float64)), float(np.sum(app.rho, dtype=np.float64))]
    vals += [float(np.sum(ps.visible1)), float(np.sum(ps.visible2)), float(np.sum(ps.active))]
    return np.array(vals)


def make_full() -> None:
    pv = reference.load()
    from pivgen import config, raster
    from pivgen.rng import STREAM_NOISE

    out = {}
    for name, H, W, ppp, dr, rr, ss, si, hide, seed, (r0, c0) in FULL_CASES:
        cfg, key, ps, side = full_case_particles(pv, name, H, W, ppp, dr, rr, ss, si, hide, seed)
        out[f"{name}/args"] = np.array([H, W, seed, side, r0, c0])
        out[f"{name}/ranges"] = np.array([*ppp, *dr, *rr, ss, si, hide])
        out[f"{name}/checksum"] = particle_checksum(ps)
        for f in (1, 2):
            raw = raster.splat(ps, f, H, W, side)
            fin = raster.finalize(raw, config.NoiseConfig(background_offset=0.05),
                                  key.with_stream(STREAM_NOISE, lane=f))
            for kind, img in (("raw", raw), ("fin", fin)):
                out[f"{name}/{kind}{f}_crop"] = img[r0:r0 + CROP, c0:c0 + CROP]
                out[f"{name}/{kind}{f}_stats"] = np.array([img.astype(np.float64).sum(),
                                                          (img.astype(np.float64) ** 2).sum(), img.max()])
            if name.startswith("wide"):
                # small image: keep the reference's untruncated render_oracle too
                out[f"{name}/oracle{f}"] = raster.render_oracle(ps, f, H, W)
                out[f"{name}/raw{f}"] = raw
    out["names"] = np.array([c[0] for c in FULL_CASES])
    path = os.path.join(HERE, "ref_full.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


def make_histmatch(raster) -> None:
    """tests/golden/histmatch_cases.npz: reference raster.match_histogram (raster.py:164-187)
    on rendered-looking and edge-case images against several target histograms."""
    rng = np.random.default_rng(2512)
    H, W = 48, 64
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    blobs = np.zeros((H, W))
    for _ in range(60):
        cy, cx, s = rng.uniform(0, H), rng.uniform(0, W), rng.uniform(0.3, 1.5)
        blobs += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * s * s))
    images = {
        "blobs": np.clip(blobs, 0, 1).astype(np.float32),
        "uniform": rng.uniform(0, 1, (H, W)).astype(np.float32),
        "constant": np.full((H, W), 0.37, np.float32),
        "out_of_range": rng.normal(0.5, 0.6, (H, W)).astype(np.float32),
        "half_levels": ((rng.integers(0, 256, (H, W)) + 0.5) / 255.0).astype(np.float32),
    }
    lev = np.arange(256, dtype=np.float64)
    targets = {
        "flat": np.ones(256),
        "dark": np.exp(-lev / 20.0),
        "gauss": np.exp(-0.5 * ((lev - 128.0) / 30.0) ** 2),
        "sparse": np.where(lev % 17 == 0, 3.0, 0.0),
        "random": rng.uniform(0, 1, 256),
    }
    out = {}
    for iname, img in images.items():
        out[f"img/{iname}"] = img
        for tname, tgt in targets.items():
            out[f"out/{iname}/{tname}"] = raster.match_histogram(img, tgt)
    for tname, tgt in targets.items():
        out[f"tgt/{tname}"] = tgt
    path = os.path.join(HERE, "histmatch_cases.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "full":
        make_full()
    else:
        main()
