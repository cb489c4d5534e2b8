"""CPU: the C-ABI library loads and exports every symbol include/pivgen_b200.h declares."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from _helpers import ROOT

HEADER = os.path.join(ROOT, "include", "pivgen_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pgb_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.build import build

    build()
    return _lib.load()


def test_every_declared_symbol_is_exported_and_bound(lib):
    from paper_2512_09664_b200 import _lib

    names = declared_symbols()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), f"{name} missing from libpivgen_b200.so"
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_host_only_entry_points(lib):
    assert lib.pgb_abi_version() == 1
    from oracle.generate import patch_side

    for d in (0.1, 0.5, 0.8, 1.0, 1.2, 4.0 / 3.0, 2.0, 3.999999999, 4.0, 7.25):
        assert lib.pgb_patch_side(d, 3.0) == patch_side(d, 3.0), d
    # staircase boundaries: 3d + 1 within 1e-10 of an integer rounds like Python
    for k in range(2, 40):
        for eps in (-3e-10, -1e-12, 0.0, 1e-12, 3e-10, 7e-10):
            d = (k - 1 + eps) / 3.0
            assert lib.pgb_patch_side(d, 3.0) == patch_side(d, 3.0), (k, eps)


def test_plan_fits_shared_memory(lib):
    from paper_2512_09664_b200 import _lib

    for H, W, n, halo in ((256, 256, 3933, 2), (512, 512, 15729, 2), (1024, 1024, 104858, 6),
                          (64, 64, 82, 2), (37, 53, 137, 6), (8, 4096, 2000, 3)):
        info = _lib.PgbPlanInfo()
        _lib.call("pgb_plan", H, W, n, 0.0, halo, 2, ctypes.byref(info))
        assert info.smem_bytes <= 220 * 1024
        assert info.tiles_y * info.tile_h >= H and info.tiles_x * info.tile_w >= W
        assert info.chunks * info.chunk >= n and info.tile_h >= min(H, 2 * halo + 1)
        assert info.capacity >= 8


def test_errors_are_reported_not_thrown(lib):
    from paper_2512_09664_b200 import _lib

    with pytest.raises(_lib.BackendError, match="info is NULL"):
        _lib.call("pgb_plan", 64, 64, 10, 0.0, 1, 2, None)
    with pytest.raises(_lib.BackendError, match="config is NULL"):
        _lib.call("pgb_generate_batch_dev", None, 0, 0, 1, None, 1, 1, 1, None, None, None, None, None)
