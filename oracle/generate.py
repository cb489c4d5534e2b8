"""CPU restatement of the seeding + advection path -- TEST INFRASTRUCTURE.

Mirrors paper_2512_09664_b200/csrc/band.cuh (prologue_kernel + seed_particle)
with the Philox draw layout of the B200 kernels, and the reference semantics
it implements:

  particle_capacity   config.py:139-146   N = ceil(round(ppp_max * H * W, 9))
  sample_particles    particles.py:61-101 positions U[0,W)xU[0,H), ppp, M,
                                          I0/d/rho ranges, sigma = d / ratio
  perturb_frame2      particles.py:104-126
  advect/sample_flow  particles.py:129-136, flowfield.py:207-232
  apply_hiding        particles.py:139-147
  patch_side          raster.py:30-38 (+ pipeline.py:291-294 for d_max)

Stratified seeding (same law as iid uniform positions): the image is split
into 2^sy x 2^sx equal-area cells; the cell counts are the histogram of M iid
uniform labels, particle g sits in the cell whose prefix range holds g, at a
uniform position inside it. The maximum diameter uniform is drawn first
(m = V^(1/M) with reproducible log/exp, on a uniform particle J); the others
are uniform on [0, qmax]. Positions are Q17 fixed point (X / 2^17, X odd: the
centre of a 2^-16 px bin; anchor + exact float32 fraction), advected in
Q20 relative to the anchor (displacement rounded to 2^-20 px);
every float32 step is a separately rounded numpy float32 op (no FMA), so
positions, diameters, sigma, i0, rho, masks, M and side are bit-identical to
the GPU; Box-Muller normals (frame-2 jitter) and the laser-sheet profile use
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


def laser_profile(z, dz0: float, shape: float, q: float):
    """I0(z) = q exp(-(1/sqrt(2 pi)) |2 z^2 / dZ0^2|^s), float64."""
    t = 2.0 * np.asarray(z, np.float64) ** 2 / (dz0 * dz0)
    return q * np.exp(-(1.0 / math.sqrt(2.0 * math.pi)) * np.abs(t) ** shape)


F32 = np.float32


def unit23(w) -> np.ndarray:
    """((w >> 9) + 0.5) * 2^-23 in float32: exact, strictly inside (0, 1)."""
    w = np.asarray(w, dtype=np.uint32)
    return ((w >> np.uint32(9)).astype(F32) + F32(0.5)) * F32(2.0 ** -23)


def lerp32(lo: float, hi: float, u: np.ndarray) -> np.ndarray:
    """f32(lo) + (f32(hi) - f32(lo)) * u, each op rounded to float32."""
    lo32, hi32 = F32(lo), F32(hi)
    span = F32(hi32 - lo32)
    return (lo32 + span * u).astype(F32)


def fixed_anchor(X: np.ndarray):
    """Q17 coordinate X / 2^17 -> (anchor floor(v + 1/2), float32 fraction) (fused.cuh fixed_anchor)."""
    X = np.asarray(X).astype(np.int64)
    an = (X + (1 << 16)) >> 17
    return an, ((X - (an << 17)).astype(np.float64) * 2.0 ** -17).astype(F32)


def fixed_cell(X: np.ndarray, n: int):
    """Clamped bilinear cell of a Q17 coordinate (fused.cuh fixed_cell)."""
    xc = np.minimum(np.asarray(X).astype(np.int64), (n - 1) << 17)
    c = np.minimum(xc >> 17, max(n - 2, 0))
    return c, ((xc - (c << 17)).astype(np.float64) * 2.0 ** -17).astype(F32)


def bilerp32(g00, g01, g10, g11, tx, ty):
    one = F32(1.0)
    sx, sy = (one - tx).astype(F32), (one - ty).astype(F32)
    top = (sx * g00).astype(F32) + (tx * g01).astype(F32)
    bot = (sx * g10).astype(F32) + (tx * g11).astype(F32)
    return ((sy * top).astype(F32) + (ty * bot).astype(F32)).astype(F32)


def advect_anchor(X, a, d):
    """fused.cuh advect_anchor: t = (X - a 2^17) 2^3 + rint(d 2^20) in Q20 (round half
    even), anchor a + floor(t / 2^20 + 1/2), exact float32 fraction."""
    X = np.asarray(X).astype(np.int64)
    a = np.asarray(a).astype(np.int64)
    t = ((X - (a << 17)) << 3) + np.rint(np.asarray(d, np.float32).astype(np.float64) * 1048576.0).astype(np.int64)
    k = (t + (1 << 19)) >> 20
    return a + k, ((t - (k << 20)).astype(np.float64) * 2.0 ** -20).astype(F32)


def hide_threshold(p: float) -> int:
    """visible iff (w + 1/2) 2^-32 >= p  <=>  w >= ceil(p 2^32 - 1/2)."""
    t = math.ceil(p * 4294967296.0 - 0.5)
    return int(min(max(t, 0), 4294967296))


MAX_CELL_BITS = 14
LN2 = 0.6931471805599453


FULL_WIDTH_MAX = 256


def cell_bits(height: int, width: int):
    """csrc/pivgen_b200.cu cell_bits: ~2-row x 4-column cells, at most 2^14
    cells; images up to FULL_WIDTH_MAX wide are rendered in full-width tiles
    and seeded in full-width cell rows (sx = 0)."""
    def bits(n, px):
        s = 0
        while (px << (s + 1)) <= n:
            s += 1
        return s
    sy, sx = bits(height, 2), (0 if width <= FULL_WIDTH_MAX else bits(width, 4))
    while sy + sx > MAX_CELL_BITS:
        if sx >= sy:
            sx -= 1
        else:
            sy -= 1
    return sy, sx


INV_ODD = [1.0 / float(2 * k + 1) for k in range(13)]
INV_INT = [0.0] + [1.0 / float(i) for i in range(1, 17)]


def rlog(x: float) -> float:
    """common.cuh rlog: only correctly rounded +,-,*,/ (bit-identical to the GPU)."""
    f, e = math.frexp(x)
    if f < 0.70710678118654752:
        f = f * 2.0
        e -= 1
    s = (f - 1.0) / (f + 1.0)
    z = s * s
    p = INV_ODD[12]
    for k in range(11, -1, -1):
        p = p * z + INV_ODD[k]
    return float(e) * LN2 + 2.0 * (s * p)


def rexp(y: float) -> float:
    """common.cuh rexp."""
    k = float(round(y * 1.4426950408889634))   # round-half-even == rint
    r = y - k * LN2
    p = 1.0
    for i in range(16, 0, -1):
        p = 1.0 + (r * p) * INV_INT[i]
    return math.ldexp(p, int(k))


def pair_header(cfg: "GenConfig", batch: int, gpair: int) -> dict:
    """prologue_kernel thread 0: density, M, maximum-diameter draw, patch side."""
    n = cfg.n
    H, W = cfg.height, cfg.width
    w = px.draw(cfg.seed, gpair, batch, np.uint64(0), px.TAG_PAIR)
    ppp = float(cfg.ppp_range[0] + (cfg.ppp_range[1] - cfg.ppp_range[0]) * px.u53_to_unit(w[0], w[1]))
    m = int(np.rint(ppp * H * W))
    m = min(max(m, 0), n)
    hd = dict(ppp=ppp, M=m, m=0.0, J=0, qmax=0, dmax=float(np.float32(cfg.d_range[1])))
    if m > 0:
        v = px.draw(cfg.seed, gpair, batch, np.uint64(1), px.TAG_PAIR)
        V = float(px.u53_to_unit(v[0], v[1]))
        mu = rexp(rlog(V) / float(m))
        w64 = (int(v[3]) << 32) | int(v[2])
        hd["m"] = mu
        hd["J"] = (w64 * m) >> 64
        hd["qmax"] = min(int(math.floor(mu * 8388608.0)), 0x7FFFFF)
        hd["dmax"] = float(lerp32(cfg.d_range[0], cfg.d_range[1], q_unit(np.array([hd["qmax"]])))[0])
    hd["side"] = patch_side(hd["dmax"] if m > 0 else cfg.d_range[1], cfg.patch_multiplier)
    return hd


def q_unit(q) -> np.ndarray:
    return (np.asarray(q).astype(F32) + F32(0.5)) * F32(2.0 ** -23)


def cell_prefix(cfg: "GenConfig", batch: int, gpair: int, M: int) -> np.ndarray:
    """prologue_kernel: histogram of M iid cell labels (word >> (32 - L)), exclusive prefix."""
    sy, sx = cell_bits(cfg.height, cfg.width)
    L = sy + sx
    q = np.arange((M + 3) // 4, dtype=np.uint64)
    words = np.stack(px.draw(cfg.seed, gpair, batch, q, px.TAG_CELL), axis=1).reshape(-1)[:M]
    labels = (words >> np.uint32(32 - L)).astype(np.int64) if L else np.zeros(M, np.int64)
    counts = np.bincount(labels, minlength=1 << L)
    return np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)


def cell_coord(cell, w, size: int, bits: int) -> np.ndarray:
    """fused.cuh cell_coord: Q17 X = 2 (cell CW + floor(w CW / 2^32)) + 1, CW = size << (16 - bits)."""
    cw = np.int64(size << (16 - bits))
    c = np.asarray(cell).astype(np.int64)
    w = np.asarray(w).astype(np.int64)
    return (((c * cw + ((w * cw) >> 32)) << 1) | 1).astype(np.int64)


def sample_pair(cfg: GenConfig, batch: int, gpair: int, flow_uv: np.ndarray) -> dict:
    """All per-particle arrays of one pair, exactly as csrc/band.cuh seed_particle()
    produces them: stratified fixed-point positions, float32 attributes and advection."""
    n = cfg.n
    H, W = cfg.height, cfg.width
    idx = np.arange(n, dtype=np.uint64)
    a = px.draw(cfg.seed, gpair, batch, idx, px.TAG_PARTICLE_A)
    hd = pair_header(cfg, batch, gpair)
    ppp, m = hd["ppp"], hd["M"]
    sy, sx = cell_bits(H, W)
    pre = cell_prefix(cfg, batch, gpair, m)
    active = np.arange(n) < m
    cell = np.searchsorted(pre, np.arange(n), side="right") - 1
    cell = np.where(active, np.minimum(cell, (1 << (sy + sx)) - 1), 0)
    cy, cx = cell >> sx, cell & ((1 << sx) - 1)
    X = np.where(active, cell_coord(cx, a[0], W, sx), cell_coord(0, a[0], W, 0))
    Y = np.where(active, cell_coord(cy, a[1], H, sy), cell_coord(0, a[1], H, 0))
    # diameters: particle J holds the maximum quantile qmax, the others are
    # uniform on [0, qmax]: floor(w (qmax + 1) / 2^32)
    q = (a[2].astype(np.int64) * (hd["qmax"] + 1)) >> 32
    if m > 0:
        q[hd["J"]] = hd["qmax"]
    d = np.where(active, lerp32(cfg.d_range[0], cfg.d_range[1], q_unit(q)),
                 lerp32(cfg.d_range[0], cfg.d_range[1], unit23(a[2]))).astype(F32)
    i0 = lerp32(cfg.i0_range[0], cfg.i0_range[1], unit23(a[3]))
    need_b = (cfg.rho_range[0] != cfg.rho_range[1]) or cfg.hide_probability > 0 or cfg.laser is not None
    if need_b:
        b = px.draw(cfg.seed, gpair, batch, idx, px.TAG_PARTICLE_B)
        rho = lerp32(cfg.rho_range[0], cfg.rho_range[1], unit23(b[0]))
        thr = hide_threshold(cfg.hide_probability)
        vis1 = b[1].astype(np.uint64) >= np.uint64(thr)
        vis2 = b[2].astype(np.uint64) >= np.uint64(thr)
        z_lo, z_hi = (cfg.laser["z_lo"], cfg.laser["z_hi"]) if cfg.laser else (0.0, 0.0)
        z1 = lerp32(z_lo, z_hi, unit23(b[3]))
    else:
        rho = np.full(n, F32(cfg.rho_range[0]), dtype=F32)
        vis1 = vis2 = np.ones(n, dtype=bool)
        z1 = np.zeros(n, dtype=F32)

    i0f = np.where(active, i0, F32(0.0)).astype(F32)
    sig = (d * F32(1.0 / cfg.sigma_ratio)).astype(F32)
    sx2, sy2, i02, rho2 = sig.copy(), sig.copy(), i0f.copy(), rho.copy()
    if cfg.f2_sigma_std > 0 or cfg.f2_rho_std > 0 or cfg.f2_i0_std > 0:
        c = px.draw(cfg.seed, gpair, batch, idx, px.TAG_PERTURB)
        n0, n1 = px.box_muller64(c[0], c[1])
        n2, n3 = px.box_muller64(c[2], c[3])
        if cfg.f2_sigma_std > 0:
            sd = F32(cfg.f2_sigma_std)
            sx2 = np.maximum(sig + (sd * n0.astype(F32)).astype(F32), F32(1e-3)).astype(F32)
            sy2 = np.maximum(sig + (sd * n1.astype(F32)).astype(F32), F32(1e-3)).astype(F32)
        if cfg.f2_i0_std > 0:
            t = np.clip(i0f + (F32(cfg.f2_i0_std) * n2.astype(F32)).astype(F32), F32(0), F32(1))
            i02 = np.where(i0f == 0.0, F32(0.0), t).astype(F32)
        if cfg.f2_rho_std > 0:
            rho2 = np.clip(rho + (F32(cfg.f2_rho_std) * n3.astype(F32)).astype(F32),
                           F32(-0.999), F32(0.999)).astype(F32)
    amp1, amp2 = i0f, i02
    if cfg.laser is not None:
        L = cfg.laser
        amp1 = (i0f * laser_profile(z1, L["dz0"], L["shape"], L["q"])).astype(F32)
        amp2 = (i02 * laser_profile((z1 + F32(L["w"])).astype(F32), L["dz0"], L["shape"],
                                     L["q"])).astype(F32)

    ax1, fx1 = fixed_anchor(X)
    ay1, fy1 = fixed_anchor(Y)
    cx, tx = fixed_cell(X, W)
    cy, ty = fixed_cell(Y, H)
    cx1 = np.minimum(cx + 1, W - 1)
    cy1 = np.minimum(cy + 1, H - 1)
    g = flow_uv.astype(F32)
    u = bilerp32(g[cy, cx, 0], g[cy, cx1, 0], g[cy1, cx, 0], g[cy1, cx1, 0], tx, ty)
    v = bilerp32(g[cy, cx, 1], g[cy, cx1, 1], g[cy1, cx, 1], g[cy1, cx1, 1], tx, ty)
    ax2, fx2 = advect_anchor(X, ax1, u)
    ay2, fy2 = advect_anchor(Y, ay1, v)

    pos1 = np.stack([ax1 + fx1.astype(np.float64), ay1 + fy1.astype(np.float64)], axis=1)
    pos2 = np.stack([ax2 + fx2.astype(np.float64), ay2 + fy2.astype(np.float64)], axis=1)
    on1 = active & vis1 & (amp1 > 0)
    on2 = active & vis2 & (amp2 > 0)
    dmax = float(d[:m].max()) if m else float(cfg.d_range[1])
    assert not m or dmax == hd["dmax"]
    side = hd["side"]
    return dict(ppp=ppp, M=m, pos1=pos1, pos2=pos2, i0_1=amp1, sx_1=sig, sy_1=sig.copy(),
                rho_1=rho, i0_2=amp2, sx_2=sx2, sy_2=sy2, rho_2=rho2, diameter=d,
                z1=z1, active=active, visible1=vis1 & active, visible2=vis2 & active,
                on1=on1, on2=on2, side=side, d_max=dmax,
                anchors=(ax1, ay1, ax2, ay2), fracs=(fx1, fy1, fx2, fy2), prefix=pre)
