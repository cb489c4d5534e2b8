"""CPU: the configuration schema is a drop-in superset of the reference's (config.py)."""

from __future__ import annotations

import pytest

import paper_2512_09664_b200 as pg
from oracle import reference


def test_defaults_match_reference_baseline():
    c = pg.GeneratorConfig()
    assert (c.image_height, c.image_width, c.batch_size) == (512, 512, 64)
    assert c.seeding_density_range == (0.06, 0.06) and c.diameter_range == (0.8, 1.2)
    assert c.particle_capacity() == 15729
    assert c.psf == "point" and c.output_dtype == "float32" and c.laser_sheet is None


def test_round_trip_with_extensions():
    c = pg.GeneratorConfig(image_height=96, batch_size=8, flow_fields_per_batch=2, psf="erf",
                           output_dtype="uint16", noise=pg.NoiseConfig(0.1, 0.02),
                           flow_sources=(pg.FlowSource(function="f", scale=2.0),
                                         pg.FlowSource(path="a.flo")),
                           laser_sheet=pg.LaserSheetConfig(thickness=0.5, z_range=(-1.0, 1.0)),
                           target_histogram=tuple([1.0] * 256), device="cuda:1")
    assert pg.parse_config(pg.render_config(c)) == c
    assert c.device_index == 1


@pytest.mark.parametrize("doc,field", [
    ("image_height: 0", "image_height"),
    ("batch_size: 6\nflow_fields_per_batch: 4", "flow_fields_per_batch"),
    ("seeding_density_range: [0.2, 0.1]", "seeding_density_range"),
    ("rho_range: [-1.0, 0.0]", "rho_range"),
    ("hide_probability: 1.0", "hide_probability"),
    ("noise: {background_offset: 1.5}", "noise.background_offset"),
    ("device: tpu", "device"),
    ("psf: gaussian", "psf"),
    ("output_dtype: int8", "output_dtype"),
    ("laser_sheet: {thickness: -1}", "laser_sheet.thickness"),
    ("flow_sources: [{path: a.xyz}]", "flow_sources"),
    ("bogus: 1", "unknown key"),
    ("image_width: 1.5", "image_width"),
])
def test_errors_name_the_field(doc, field):
    with pytest.raises(pg.ConfigError, match=field.replace(".", r"\.")):
        pg.parse_config(doc)


def test_legacy_cpu_device_accepted():
    assert pg.parse_config("device: cpu").device == "cpu"


@pytest.mark.skipif(not reference.available(), reason="oracle/_ref not built")
def test_reference_documents_parse_identically():
    pv = reference.load()
    ref_cfg = pv.GeneratorConfig(image_height=128, image_width=96, batch_size=4,
                                 seeding_density_range=(0.02, 0.05), frame2_sigma_std=0.1,
                                 hide_probability=0.2, noise=pv.NoiseConfig(0.1, 0.01),
                                 flow_sources=(pv.FlowSource(path="x.flo", scale=0.5),), seed=99)
    text = pv.render_config(ref_cfg)
    ours = pg.parse_config(text)
    for name in ("image_height", "image_width", "batch_size", "seeding_density_range",
                 "frame2_sigma_std", "hide_probability", "seed", "diameter_sigma_ratio"):
        assert getattr(ours, name) == getattr(ref_cfg, name), name
    assert ours.particle_capacity() == ref_cfg.particle_capacity()
    assert ours.noise.gaussian_std == 0.01 and ours.flow_sources[0].scale == 0.5
