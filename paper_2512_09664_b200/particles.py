"""Particle seeding, frame-2 perturbation, advection and hiding on the GPU.

Drop-in for the reference functional layer (particles.py:1-147). All draws
come from Philox4x32-10 keyed by (seed, batch, pair) (``RngKey``); the
kernels are the ones the band-kernel generator runs, so ``sample_particles`` +
``perturb_frame2`` + ``advect`` + ``apply_hiding`` reproduce exactly the
particle set rendered by ``Sampler`` for that pair.

Arrays are returned as numpy (the reference types); positions are float64,
appearances float32, masks bool.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from ._device import cuda_device, stream_ptr, to_dev
from .config import GeneratorConfig
from .flowfield import FlowField

SIGMA_FLOOR = 1e-3
RHO_CLAMP = 1.0 - 1e-3


@dataclass(frozen=True)
class RngKey:
    """Addresses the random streams of one image pair.

    The reference key (rng.py:54-106) folds (seed, stream, batch, pair, lane)
    with splitmix64; here the stream/lane selection lives inside the kernels
    (Philox counter word 3) and the key is just (seed, batch, pair). ``frame``
    selects the noise stream for ``finalize``.
    """

    seed: int
    batch: int = 0
    pair: int = 0
    frame: int = 1

    def with_frame(self, frame: int) -> "RngKey":
        return replace(self, frame=frame)


def pair_key(seed: int, batch: int, pair: int) -> RngKey:
    return RngKey(seed=seed, batch=batch, pair=pair)


@dataclass
class Appearance:
    i0: np.ndarray
    sigma_x: np.ndarray
    sigma_y: np.ndarray
    rho: np.ndarray

    def copy(self) -> "Appearance":
        return Appearance(self.i0.copy(), self.sigma_x.copy(), self.sigma_y.copy(), self.rho.copy())


@dataclass
class ParticleSet:
    count: int
    pos1: np.ndarray
    app1: Appearance
    active: np.ndarray
    pos2: np.ndarray | None = None
    app2: Appearance | None = None
    visible1: np.ndarray | None = None
    visible2: np.ndarray | None = None


@dataclass
class PairParams:
    """Realised parameters of one pair (particles.py:50-58)."""

    seeding_density: float
    diameters: np.ndarray
    peak_intensities: np.ndarray
    rhos: np.ndarray
    active_count: int


def native_config(cfg: GeneratorConfig) -> _lib.PgbConfig:
    """GeneratorConfig -> the C ABI struct."""
    c = _lib.PgbConfig()
    c.height, c.width = cfg.image_height, cfg.image_width
    c.n_capacity = cfg.particle_capacity()
    c.psf = _lib.PSF_CODES[cfg.psf]
    c.seed = cfg.seed
    c.ppp_lo, c.ppp_hi = cfg.seeding_density_range
    c.d_lo, c.d_hi = cfg.diameter_range
    c.i0_lo, c.i0_hi = cfg.peak_intensity_range
    c.rho_lo, c.rho_hi = cfg.rho_range
    c.sigma_ratio = cfg.diameter_sigma_ratio
    c.patch_multiplier = cfg.patch_multiplier
    c.f2_sigma_std = cfg.frame2_sigma_std
    c.f2_rho_std = cfg.frame2_rho_std
    c.f2_i0_std = cfg.frame2_intensity_std
    c.hide_probability = cfg.hide_probability
    c.bg_offset = cfg.noise.background_offset
    c.noise_std = cfg.noise.gaussian_std
    ls = cfg.laser_sheet
    if ls is not None:
        c.laser_enabled = 1
        c.laser_dz0, c.laser_shape, c.laser_q = ls.thickness, ls.shape, ls.efficiency
        c.laser_z_lo, c.laser_z_hi = ls.resolved_z_range()
        c.laser_w = ls.out_of_plane
    return c


_ZERO_FIELDS: dict = {}


def _zero_flow(height: int, width: int, device: torch.device) -> torch.Tensor:
    key = (height, width, device.index)
    t = _ZERO_FIELDS.get(key)
    if t is None:
        t = torch.zeros((height, width, 2), dtype=torch.float32, device=device)
        _ZERO_FIELDS[key] = t
    return t


def generate_particle_arrays(cfg: GeneratorConfig, batch: int, pairs: range,
                             flows: torch.Tensor | None = None, pairs_per_field: int | None = None,
                             device=None) -> dict:
    """All per-particle arrays the band kernel renders for global pairs
    ``pairs`` of ``batch`` (device tensors, shape (P, N[, 2]))."""
    dev = cuda_device(device)
    n = cfg.particle_capacity()
    P = len(pairs)
    base = pairs.start if P else 0
    if flows is None:
        flows = _zero_flow(cfg.image_height, cfg.image_width, dev).unsqueeze(0)
        ppf = max(base + P, 1)
    else:
        ppf = pairs_per_field or cfg.pairs_per_field
    f64 = dict(dtype=torch.float64, device=dev)
    f32 = dict(dtype=torch.float32, device=dev)
    u8 = dict(dtype=torch.uint8, device=dev)
    out = {
        "pos1": torch.empty((P, n, 2), **f64), "pos2": torch.empty((P, n, 2), **f64),
        "i0_1": torch.empty((P, n), **f32), "sx_1": torch.empty((P, n), **f32),
        "sy_1": torch.empty((P, n), **f32), "rho_1": torch.empty((P, n), **f32),
        "i0_2": torch.empty((P, n), **f32), "sx_2": torch.empty((P, n), **f32),
        "sy_2": torch.empty((P, n), **f32), "rho_2": torch.empty((P, n), **f32),
        "diameter": torch.empty((P, n), **f32), "z1": torch.empty((P, n), **f32),
        "active": torch.empty((P, n), **u8), "visible1": torch.empty((P, n), **u8),
        "visible2": torch.empty((P, n), **u8),
    }
    st = {"seeding_density": torch.empty(P, **f64),
          "active_count": torch.empty(P, dtype=torch.int32, device=dev),
          "side": torch.empty(P, dtype=torch.int32, device=dev),
          "d_max": torch.empty(P, **f32)}
    po = _lib.PgbParticleOut(**{k: v.data_ptr() for k, v in out.items()})
    ps = _lib.PgbPairStats(**{k: v.data_ptr() for k, v in st.items()})
    c = native_config(cfg)
    if P:
        _lib.call("pgb_sample_particles_dev", c, batch, base, P, flows.data_ptr(),
                  flows.shape[0], ppf, po, ps, stream_ptr(dev))
    out.update(st)
    return out


def generate_particle_arrays_splitmix(cfg: GeneratorConfig, batch: int, pairs: range,
                                      flows: torch.Tensor, pairs_per_field: int | None = None,
                                      device=None) -> dict:
    """Reference-RNG mode (rng.py:33-106 streams): the reference's
    sample_particles / perturb_frame2 / apply_hiding / advect arrays for
    global pairs ``pairs`` of ``batch`` (device tensors, shape (P, N[, 2])),
    plus per-pair ``seeding_density``, ``active_count``, ``side``, ``d_max``."""
    dev = cuda_device(device)
    n = cfg.particle_capacity()
    P = len(pairs)
    base = pairs.start if P else 0
    ppf = pairs_per_field or cfg.pairs_per_field
    f64 = dict(dtype=torch.float64, device=dev)
    f32 = dict(dtype=torch.float32, device=dev)
    u8 = dict(dtype=torch.uint8, device=dev)
    out = {
        "pos1": torch.empty((P, n, 2), **f64), "pos2": torch.empty((P, n, 2), **f64),
        "i0_1": torch.empty((P, n), **f32), "sx_1": torch.empty((P, n), **f32),
        "sy_1": torch.empty((P, n), **f32), "rho_1": torch.empty((P, n), **f32),
        "i0_2": torch.empty((P, n), **f32), "sx_2": torch.empty((P, n), **f32),
        "sy_2": torch.empty((P, n), **f32), "rho_2": torch.empty((P, n), **f32),
        "diameter": torch.empty((P, n), **f32), "z1": torch.empty((P, n), **f32),
        "active": torch.empty((P, n), **u8), "visible1": torch.empty((P, n), **u8),
        "visible2": torch.empty((P, n), **u8),
    }
    st = {"seeding_density": torch.empty(P, **f64),
          "active_count": torch.empty(P, dtype=torch.int32, device=dev),
          "side": torch.empty(P, dtype=torch.int32, device=dev),
          "d_max": torch.empty(P, **f32)}
    po = _lib.PgbParticleOut(**{k: v.data_ptr() for k, v in out.items()})
    ps = _lib.PgbPairStats(**{k: v.data_ptr() for k, v in st.items()})
    if P:
        _lib.call("pgb_sample_particles_splitmix_dev", native_config(cfg), batch, base, P, flows.data_ptr(),
                  flows.shape[0], ppf, po, ps, stream_ptr(dev))
    out.update(st)
    return out


def sample_particles(key: RngKey, cfg: GeneratorConfig) -> tuple[ParticleSet, PairParams]:
    """Frame-1 positions/appearances (particles.py:61-101) for one pair."""
    arr = generate_particle_arrays(cfg, key.batch, range(key.pair, key.pair + 1))
    h = {k: v[0].cpu().numpy() for k, v in arr.items()}
    active = h["active"].astype(bool)
    m = int(h["active_count"])
    app1 = Appearance(h["i0_1"], h["sx_1"], h["sy_1"], h["rho_1"])
    params = PairParams(seeding_density=float(h["seeding_density"]), diameters=h["diameter"],
                        peak_intensities=h["i0_1"].copy(), rhos=h["rho_1"].copy(), active_count=m)
    return ParticleSet(count=cfg.particle_capacity(), pos1=h["pos1"], app1=app1,
                       active=active), params


def perturb_frame2(key: RngKey, app1: Appearance, cfg: GeneratorConfig) -> Appearance:
    """Frame-2 appearances: zero-mean Gaussian jitter, floors/clamps (particles.py:104-126)."""
    dev = cuda_device(cfg.device)
    if not (cfg.frame2_sigma_std > 0 or cfg.frame2_intensity_std > 0 or cfg.frame2_rho_std > 0):
        return app1.copy()
    src = [to_dev(a, torch.float32, dev) for a in (app1.i0, app1.sigma_x, app1.sigma_y, app1.rho)]
    dst = [torch.empty_like(t) for t in src]
    n = src[0].numel()
    _lib.call("pgb_perturb_frame2_dev", n, key.seed, key.batch, key.pair, cfg.frame2_sigma_std,
              cfg.frame2_intensity_std, cfg.frame2_rho_std, *[t.data_ptr() for t in src],
              *[t.data_ptr() for t in dst], stream_ptr(dev))
    i0, sx, sy, rho = (t.cpu().numpy() for t in dst)
    return Appearance(i0, sx, sy, rho)


def advect(pset: ParticleSet, field: FlowField) -> ParticleSet:
    """pos2 = pos1 + bilinear flow at pos1 (particles.py:129-136), float64, bit-exact."""
    dev = cuda_device()
    pos = to_dev(pset.pos1, torch.float64, dev)
    out = torch.empty_like(pos)
    flow = field.to_device(dev)
    _lib.call("pgb_advect_dev", pos.data_ptr(), pos.shape[0], flow.data_ptr(), field.height,
              field.width, out.data_ptr(), stream_ptr(dev))
    pset.pos2 = out.cpu().numpy()
    return pset


def apply_hiding(key: RngKey, pset: ParticleSet, hide_probability: float,
                 seed: int | None = None) -> ParticleSet:
    """Per-frame visibility masks; inactive slots stay hidden (particles.py:139-147)."""
    dev = cuda_device()
    active = to_dev(pset.active, torch.uint8, dev)
    v1 = torch.empty_like(active)
    v2 = torch.empty_like(active)
    _lib.call("pgb_apply_hiding_dev", active.numel(), key.seed if seed is None else seed,
              key.batch, key.pair, float(hide_probability), active.data_ptr(), v1.data_ptr(),
              v2.data_ptr(), stream_ptr(dev))
    pset.visible1 = v1.cpu().numpy().astype(bool)
    pset.visible2 = v2.cpu().numpy().astype(bool)
    return pset
