"""CPU restatement of the seeding + advection path -- TEST INFRASTRUCTURE.

Mirrors paper_2512_09664_b200/csrc/fused.cuh make_particle() with the Philox
draw layout of the B200 kernels, and the reference semantics it implements:

  particle_capacity   config.py:139-146   N = ceil(round(ppp_max * H * W, 9))
  sample_particles    particles.py:61-101 positions U[0,W)xU[0,H), ppp, M,
                                          I0/d/rho ranges, sigma = d / ratio
  perturb_frame2      particles.py:104-126
  advect/sample_flow  particles.py:129-136, flowfield.py:207-232
  apply_hiding        particles.py:139-147
  patch_side          raster.py:30-38 (+ pipeline.py:291-294 for d_max)

Every float64 step is a separately rounded numpy op (no FMA), so positions,
diameters, sigma, i0, rho, masks, M and side are bit-identical to the GPU;
Box-Muller normals (frame-2 jitter) and the laser-sheet profile use float32
fast intrinsics on the GPU and agree to ~1e-6.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import philox as px

SIGMA_FLOOR = 1e-3          # particles.py:20
RHO_CLAMP = 1.0 - 1e-3      # particles.py:21


def particle_capacity(ppp_max: float, height: int, width: int) -> int:
    """config.py:139-146."""
    return math.ceil(round(ppp_max * height * width, 9))


def patch_side(max_diameter: float, multiplier: float = 3.0) -> int:
    """raster.py:30-38 (restated)."""
    side = math.ceil(round(multiplier * max_diameter + 1.0, 9))
    if side % 2 == 0:
        side += 1
    return max(side, 1)


def sample_flow(flow_uv: np.ndarray, pos: np.ndarray) -> np.ndarray:
    """flowfield.py:207-232 restated on an interleaved (H, W, 2) float32 grid."""
    height, width = flow_uv.shape[:2]
    x = np.clip(pos[:, 0], 0.0, width - 1.0)
    y = np.clip(pos[:, 1], 0.0, height - 1.0)
    x0 = np.clip(np.floor(x), 0, max(width - 2, 0)).astype(np.intp)
    y0 = np.clip(np.floor(y), 0, max(height - 2, 0)).astype(np.intp)
    x1 = np.minimum(x0 + 1, width - 1)
    y1 = np.minimum(y0 + 1, height - 1)
    fx = x - x0
    fy = y - y0
    out = np.empty((pos.shape[0], 2), dtype=np.float64)
    for col in range(2):
        g = flow_uv[:, :, col].astype(np.float64)
        top = (1.0 - fx) * g[y0, x0] + fx * g[y0, x1]
        bottom = (1.0 - fx) * g[y1, x0] + fx * g[y1, x1]
        out[:, col] = (1.0 - fy) * top + fy * bottom
    return out


@dataclass
class GenConfig:
    height: int
    width: int
    seed: int = 0
    ppp_range: tuple = (0.06, 0.06)
    d_range: tuple = (0.8, 1.2)
    i0_range: tuple = (1.0, 1.0)
    rho_range: tuple = (0.0, 0.0)
    sigma_ratio: float = 4.0
    patch_multiplier: float = 3.0
    f2_sigma_std: float = 0.0
    f2_rho_std: float = 0.0
    f2_i0_std: float = 0.0
    hide_probability: float = 0.0
    laser: dict | None = None   # {dz0, shape, q, z_lo, z_hi, w}

    @property
    def n(self) -> int:
        return particle_capacity(self.ppp_range[1], self.height, self.width)


def laser_profile(z: np.ndarray, dz0: float, shape: float, q: float) -> np.ndarray:
    """I0(z) = q exp(-(1/sqrt(2 pi)) |2 z^2 / dZ0^2|^s)."""
    t = 2.0 * np.asarray(z, np.float64) ** 2 / (dz0 * dz0)
    return q * np.exp(-(1.0 / math.sqrt(2.0 * math.pi)) * np.abs(t) ** shape)


def sample_pair(cfg: GenConfig, batch: int, gpair: int, flow_uv: np.ndarray) -> dict:
    """All per-particle arrays of one pair, as the B200 kernel generates them."""
    n = cfg.n
    H, W = cfg.height, cfg.width
    idx = np.arange(n, dtype=np.uint64)
    w = px.draw(cfg.seed, gpair, batch, np.uint64(0), px.TAG_PAIR)
    ppp = float(cfg.ppp_range[0] + (cfg.ppp_range[1] - cfg.ppp_range[0]) * px.u53_to_unit(w[0], w[1]))
    m = int(np.rint(ppp * H * W))
    m = min(max(m, 0), n)

    a = px.draw(cfg.seed, gpair, batch, idx, px.TAG_PARTICLE_A)
    x1 = px.u32_to_unit(a[0]) * W
    y1 = px.u32_to_unit(a[1]) * H
    d = cfg.d_range[0] + (cfg.d_range[1] - cfg.d_range[0]) * px.u32_to_unit(a[2])
    i0 = cfg.i0_range[0] + (cfg.i0_range[1] - cfg.i0_range[0]) * px.u32_to_unit(a[3])
    active = np.arange(n) < m

    need_b = (cfg.rho_range[0] != cfg.rho_range[1]) or cfg.hide_probability > 0 or cfg.laser is not None
    if need_b:
        b = px.draw(cfg.seed, gpair, batch, idx, px.TAG_PARTICLE_B)
        rho = cfg.rho_range[0] + (cfg.rho_range[1] - cfg.rho_range[0]) * px.u32_to_unit(b[0])
        vis1 = px.u32_to_unit(b[1]) >= cfg.hide_probability
        vis2 = px.u32_to_unit(b[2]) >= cfg.hide_probability
        z_lo, z_hi = (cfg.laser["z_lo"], cfg.laser["z_hi"]) if cfg.laser else (0.0, 0.0)
        z1 = z_lo + (z_hi - z_lo) * px.u32_to_unit(b[3])
    else:
        rho = np.full(n, cfg.rho_range[0])
        vis1 = vis2 = np.ones(n, dtype=bool)
        z1 = np.zeros(n)

    i0f = np.where(active, i0, 0.0).astype(np.float32)
    sig = (d / cfg.sigma_ratio).astype(np.float32)
    rhof = rho.astype(np.float32)
    sx2, sy2, i02, rho2 = sig.copy(), sig.copy(), i0f.copy(), rhof.copy()
    if cfg.f2_sigma_std > 0 or cfg.f2_rho_std > 0 or cfg.f2_i0_std > 0:
        c = px.draw(cfg.seed, gpair, batch, idx, px.TAG_PERTURB)
        n0, n1 = px.box_muller64(c[0], c[1])
        n2, n3 = px.box_muller64(c[2], c[3])
        sd = np.float64(np.float32(cfg.f2_sigma_std))
        if cfg.f2_sigma_std > 0:
            sx2 = np.maximum(sig.astype(np.float64) + sd * n0, SIGMA_FLOOR).astype(np.float32)
            sy2 = np.maximum(sig.astype(np.float64) + sd * n1, SIGMA_FLOOR).astype(np.float32)
        if cfg.f2_i0_std > 0:
            t = np.clip(i0f.astype(np.float64) + np.float64(np.float32(cfg.f2_i0_std)) * n2, 0.0, 1.0)
            i02 = np.where(i0f == 0.0, 0.0, t).astype(np.float32)
        if cfg.f2_rho_std > 0:
            t = np.clip(rhof.astype(np.float64) + np.float64(np.float32(cfg.f2_rho_std)) * n3,
                        -RHO_CLAMP, RHO_CLAMP)
            rho2 = t.astype(np.float32)
    amp1, amp2 = i0f.astype(np.float64), i02.astype(np.float64)
    if cfg.laser is not None:
        L = cfg.laser
        amp1 = amp1 * laser_profile(z1.astype(np.float32), L["dz0"], L["shape"], L["q"])
        amp2 = amp2 * laser_profile(z1.astype(np.float32) + np.float32(L["w"]), L["dz0"], L["shape"], L["q"])
    amp1 = amp1.astype(np.float32)
    amp2 = amp2.astype(np.float32)

    pos1 = np.stack([x1, y1], axis=1)
    pos2 = pos1 + sample_flow(flow_uv, pos1)
    on1 = active & vis1 & (amp1 > 0)
    on2 = active & vis2 & (amp2 > 0)
    diam = d.astype(np.float32)
    dmax = float(diam[:m].max()) if m else float(np.float32(cfg.d_range[1]))
    side = patch_side(dmax, cfg.patch_multiplier)
    return dict(ppp=ppp, M=m, pos1=pos1, pos2=pos2, i0_1=amp1, sx_1=sig, sy_1=sig.copy(),
                rho_1=rhof, i0_2=amp2, sx_2=sx2, sy_2=sy2, rho_2=rho2, diameter=diam,
                z1=z1.astype(np.float32), active=active, visible1=vis1 & active,
                visible2=vis2 & active, on1=on1, on2=on2, side=side, d_max=dmax)
