"""ctypes binding of libpivgen_b200.so (C ABI declared in include/pivgen_b200.h).

The shared library is the only compute path: there is no CPU fallback. If the
library is missing or a CUDA device is unavailable, calls raise
``BackendUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .build import LIB_PATH

PSF_POINT, PSF_ERF = 0, 1
OUT_RAW, OUT_F32, OUT_U16, OUT_ACCUM = 0, 1, 2, 3

PSF_CODES = {"point": PSF_POINT, "erf": PSF_ERF}


class BackendUnavailable(RuntimeError):
    """libpivgen_b200.so could not be loaded (not built, or no CUDA driver)."""


class BackendError(RuntimeError):
    """A libpivgen_b200 call returned an error status."""


class PgbConfig(C.Structure):
    _fields_ = [
        ("height", C.c_int32), ("width", C.c_int32),
        ("n_capacity", C.c_int32), ("psf", C.c_int32),
        ("seed", C.c_uint64),
        ("ppp_lo", C.c_double), ("ppp_hi", C.c_double),
        ("d_lo", C.c_double), ("d_hi", C.c_double),
        ("i0_lo", C.c_double), ("i0_hi", C.c_double),
        ("rho_lo", C.c_double), ("rho_hi", C.c_double),
        ("sigma_ratio", C.c_double), ("patch_multiplier", C.c_double),
        ("f2_sigma_std", C.c_double), ("f2_rho_std", C.c_double), ("f2_i0_std", C.c_double),
        ("hide_probability", C.c_double),
        ("bg_offset", C.c_double), ("noise_std", C.c_double),
        ("laser_enabled", C.c_int32), ("reserved0", C.c_int32),
        ("laser_dz0", C.c_double), ("laser_shape", C.c_double), ("laser_q", C.c_double),
        ("laser_z_lo", C.c_double), ("laser_z_hi", C.c_double), ("laser_w", C.c_double),
    ]


class PgbParticles(C.Structure):
    _fields_ = [("pos", C.c_void_p), ("i0", C.c_void_p), ("sigma_x", C.c_void_p),
                ("sigma_y", C.c_void_p), ("rho", C.c_void_p), ("mask", C.c_void_p)]


class PgbPairStats(C.Structure):
    _fields_ = [("seeding_density", C.c_void_p), ("active_count", C.c_void_p),
                ("side", C.c_void_p), ("d_max", C.c_void_p)]


class PgbParticleOut(C.Structure):
    _fields_ = [(name, C.c_void_p) for name in (
        "pos1", "pos2", "i0_1", "sx_1", "sy_1", "rho_1", "i0_2", "sx_2", "sy_2", "rho_2",
        "diameter", "z1", "active", "visible1", "visible2")]


class PgbPlanInfo(C.Structure):
    _fields_ = [(name, C.c_int) for name in (
        "tile_h", "tile_w", "tiles_y", "tiles_x", "chunks", "chunk", "capacity", "halo",
        "smem_bytes", "threads")]


# name -> (restype, argtypes)
_P, _I, _I64, _U64, _D = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
SIGNATURES = {
    "pgb_abi_version": (_I, []),
    "pgb_last_error": (C.c_char_p, []),
    "pgb_patch_side": (_I, [_D, _D]),
    "pgb_splat_accumulate": (_I, [_P, _P, _P, _P, _P, _P, _I64, _I, _P, _I, _I, _I, _I]),
    "pgb_splat_accumulate_dev": (_I, [_P, _P, _P, _P, _P, _P, _I64, _I, _P, _I, _I, _I, _I, _I, _P]),
    "pgb_render_pairs_dev": (_I, [C.POINTER(PgbParticles), C.POINTER(PgbParticles), _I64, _I,
                                  C.POINTER(C.c_int), _I, _I, _I, _I, _D, _D, _U64, _U64, _I64,
                                  _P, _P, _P, C.POINTER(C.c_int), _P]),
    "pgb_render_oracle_dev": (_I, [_P, _P, _P, _P, _P, _P, _I64, _I, _I, _P, _P]),
    "pgb_advect_dev": (_I, [_P, _I64, _P, _I, _I, _P, _P]),
    "pgb_sample_flow_dev": (_I, [_P, _I64, _P, _I, _I, _P, _P]),
    "pgb_finalize_dev": (_I, [_P, _I, _I, _I, _D, _D, _U64, _U64, _I64, _I, _I, _P, _P]),
    "pgb_quantize_u16_dev": (_I, [_P, _I64, _P, _P]),
    "pgb_match_histogram_dev": (_I, [_P, _P, _I64, _I64, _P, _P]),
    "pgb_sample_particles_splitmix_dev": (_I, [C.POINTER(PgbConfig), _U64, _I64, _I, _P, _I, _I,
                                               C.POINTER(PgbParticleOut), C.POINTER(PgbPairStats), _P]),
    "pgb_finalize_splitmix_dev": (_I, [_P, _P, _I64, _I, _D, _D, _U64, _U64, _I64, _I, _P]),
    "pgb_generate_batch_dev": (_I, [C.POINTER(PgbConfig), _U64, _I64, _I, _P, _I, _I, _I, _P, _P,
                                    C.POINTER(PgbPairStats), _P, _P]),
    "pgb_generate_batch": (_I, [C.POINTER(PgbConfig), _U64, _I64, _I, _P, _I, _I, _I, _P, _P,
                                C.POINTER(PgbPairStats)]),
    "pgb_sample_particles_dev": (_I, [C.POINTER(PgbConfig), _U64, _I64, _I, _P, _I, _I,
                                      C.POINTER(PgbParticleOut), C.POINTER(PgbPairStats), _P]),
    "pgb_perturb_frame2_dev": (_I, [_I64, _U64, _U64, _I64, _D, _D, _D, _P, _P, _P, _P, _P, _P,
                                    _P, _P, _P]),
    "pgb_apply_hiding_dev": (_I, [_I64, _U64, _U64, _I64, _D, _P, _P, _P, _P]),
    "pgb_plan": (_I, [_I, _I, _I64, _D, _I, _I, C.POINTER(PgbPlanInfo)]),
    "pgb_launch_count": (C.c_int64, []),
    "pgb_probe_ex2_dev": (_I, [_I, _I, _P, _P]),
    "pgb_overflow_count": (_I, []),
    "pgb_overflow_reset": (_I, []),
}

_lib = None
_lock = threading.Lock()


def lib_path() -> str:
    return os.environ.get("PGB_LIBRARY", LIB_PATH)


def load(require_symbols: bool = True):
    """Load (once) and return the ctypes handle. Raises BackendUnavailable."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not os.path.exists(path):
            raise BackendUnavailable(
                f"{path} is missing: build it with `python -m paper_2512_09664_b200.build` "
                "(nvcc, sm_100a). There is no CPU fallback.")
        try:
            handle = C.CDLL(path)
        except OSError as exc:  # pragma: no cover - depends on the driver
            raise BackendUnavailable(f"cannot load {path}: {exc}") from exc
        lenient = os.environ.get("PGB_LIB_LENIENT") == "1"   # A/B of older builds (debug)
        for name, (res, args) in SIGNATURES.items():
            if lenient and not hasattr(handle, name):
                continue
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
        return _lib


def check(status: int) -> None:
    if status != 0:
        msg = load().pgb_last_error().decode(errors="replace")
        raise BackendError(msg)


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and raise on error."""
    check(getattr(load(), name)(*args))
