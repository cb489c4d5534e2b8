"""Shared fixtures. Mirrors the reference's test fixtures (pkg/tests/conftest.py:1-66):
constant_field, flo_dir, small_config, make_config, assert_trees_identical (in _helpers)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from _helpers import GOLDEN, has_gpu, small_config, write_constant_flo


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpivgen_b200.so")


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture
def flo_dir(tmp_path):
    def build(height, width, flows=((2.0, -1.0),)):
        d = tmp_path / f"flows_{height}x{width}"
        d.mkdir(exist_ok=True)
        return [write_constant_flo(str(d / f"src_{i:02d}.flo"), height, width, u, v)
                for i, (u, v) in enumerate(flows)]
    return build


@pytest.fixture
def make_config(flo_dir):
    def build(height=64, width=64, flows=((2.0, -1.0),), **overrides):
        return small_config(flo_dir(height, width, flows), height, width, **overrides)
    return build


@pytest.fixture(scope="session")
def golden():
    data = np.load(os.path.join(GOLDEN, "ref_cases.npz"))
    cases = {}
    for name in data["names"]:
        prefix = f"{name}/"
        cases[str(name)] = {k[len(prefix):]: data[k] for k in data.files if k.startswith(prefix)}
    return cases
