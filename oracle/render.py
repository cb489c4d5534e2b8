"""CPU restatement of rendering and the epilogue -- TEST INFRASTRUCTURE.

  splat_accumulate  _native.pyx:14-66 (contract shared with _fallback.py:16-57):
                    per masked particle, anchor = floor(x + 0.5), window
                    [a - h, a + h] clipped to the row band and [0, W), value
                    I0 * exp(-(a dx^2 - b dx dy + c dy^2)) in float64 with
                    q = 1 - rho^2, a = 1/(2 q sx^2), b = rho/(q sx sy),
                    c = 1/(2 q sy^2), cast to float32 and added in particle
                    order.
  render_erf        extension: pixel-area mean of Eq. (1); the
                    same formula as fused.cuh splat_row<.., kPsfErf> in float64.
  finalize          raster.py:154-161 with the B200 Philox/Box-Muller noise.
  quantize_u16      export.py:19-20.
  tile_counts       per-tile particle counts of the fused kernel's distributed
                    counting sort (window of half-width `halo` vs tile).
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import erf

from . import philox as px

_GL_X, _GL_W = np.polynomial.legendre.leggauss(8)
GL_X = _GL_X / 2.0          # nodes on [-1/2, 1/2]
GL_W = _GL_W / 2.0          # weights summing to 1


def _patch_geometry(pos, side):
    half = side // 2
    ax = np.floor(pos[:, 0] + 0.5).astype(np.int64)
    ay = np.floor(pos[:, 1] + 0.5).astype(np.int64)
    off = np.arange(side, dtype=np.int64) - half
    cols = ax[:, None] + off[None, :]            # (m, side)
    rows = ay[:, None] + off[None, :]
    return ax, ay, rows, cols


def splat_accumulate(pos, i0, sigma_x, sigma_y, rho, mask, side, out, row_start, row_stop,
                     chunk: int = 8192) -> None:
    """In-place accumulate, particle order (reference contract)."""
    height, width = out.shape
    sel = np.flatnonzero(np.asarray(mask) != 0)
    flat = out.reshape(-1)
    for lo in range(0, sel.size, chunk):
        p = sel[lo:lo + chunk]
        x0 = pos[p, 0]
        y0 = pos[p, 1]
        _, _, rows, cols = _patch_geometry(pos[p], side)
        dx = cols - x0[:, None]                  # (m, side) float64
        dy = rows - y0[:, None]
        sx = sigma_x[p].astype(np.float64)[:, None, None]
        sy = sigma_y[p].astype(np.float64)[:, None, None]
        r = rho[p].astype(np.float64)[:, None, None]
        q = 1.0 - r * r
        ca = 1.0 / (2.0 * q * sx * sx)
        cb = r / (q * sx * sy)
        cc = 1.0 / (2.0 * q * sy * sy)
        ddx = dx[:, None, :]
        ddy = dy[:, :, None]
        e = ca * ddx * ddx - cb * ddx * ddy + cc * ddy * ddy     # (m, row, col)
        vals = (i0[p].astype(np.float64)[:, None, None] * np.exp(-e)).astype(np.float32)
        keep = (((rows >= row_start) & (rows < row_stop))[:, :, None]
                & ((cols >= 0) & (cols < width))[:, None, :])
        lin = rows[:, :, None] * width + cols[:, None, :]
        np.add.at(flat, lin[keep], vals[keep])


def splat(pos, i0, sigma_x, sigma_y, rho, mask, side, height, width) -> np.ndarray:
    out = np.zeros((height, width), dtype=np.float32)
    splat_accumulate(pos, i0, sigma_x, sigma_y, rho, mask, side, out, 0, height)
    return out


def render_erf(pos, i0, sigma_x, sigma_y, rho, mask, side, height, width) -> np.ndarray:
    """Pixel-area mean of Eq. (1) over the side x side window, float64 -> float32.

    rho == 0: amp * (pi/2) sx sy [erf]_x [erf]_y (exact);
    rho != 0: x | y is Gaussian (mean x0 + rho sx/sy (y - y0), std
    sx sqrt(1 - rho^2)); exact in x, 8-point Gauss-Legendre in y.
    """
    out = np.zeros((height, width), dtype=np.float64)
    sel = np.flatnonzero(np.asarray(mask) != 0)
    if sel.size == 0:
        return out.astype(np.float32)
    _, _, rows, cols = _patch_geometry(pos[sel], side)
    for k, p in enumerate(sel):
        x0, y0 = pos[p]
        sx, sy, r, amp = float(sigma_x[p]), float(sigma_y[p]), float(rho[p]), float(i0[p])
        dxc = cols[k] - x0           # column centres relative to x0
        dyc = rows[k] - y0
        if r == 0.0:
            ex = erf((dxc + 0.5) / (sx * math.sqrt(2))) - erf((dxc - 0.5) / (sx * math.sqrt(2)))
            ey = erf((dyc + 0.5) / (sy * math.sqrt(2))) - erf((dyc - 0.5) / (sy * math.sqrt(2)))
            patch = amp * (math.pi / 2) * sx * sy * ey[:, None] * ex[None, :]
        else:
            sc = sx * math.sqrt(max(1.0 - r * r, 0.0))
            slope = r * sx / sy
            yy = dyc[:, None] + GL_X[None, :]                    # (side, G)
            gy = np.exp(-yy * yy / (2.0 * sy * sy))
            mu = slope * yy
            hi = erf((dxc[None, None, :] + 0.5 - mu[:, :, None]) / (sc * math.sqrt(2)))
            lo = erf((dxc[None, None, :] - 0.5 - mu[:, :, None]) / (sc * math.sqrt(2)))
            patch = amp * sc * math.sqrt(math.pi / 2) * np.einsum("g,rg,rgc->rc", GL_W, gy, hi - lo)
        rr, cc = rows[k], cols[k]
        rm = (rr >= 0) & (rr < height)
        cm = (cc >= 0) & (cc < width)
        out[np.ix_(rr[rm], cc[cm])] += patch[np.ix_(rm, cm)]
    return out.astype(np.float32)


def noise_normals(seed: int, batch: int, gpair: int, frame: int, count: int) -> np.ndarray:
    """Per-pixel normals of the fused epilogue: quad q = p >> 2 of stream
    (TAG_NOISE + frame); Box-Muller on (w0, w1) and (w2, w3)."""
    quads = (count + 3) // 4
    w = px.draw(seed, gpair, batch, np.arange(quads, dtype=np.uint64), px.TAG_NOISE + frame)
    a0, a1 = px.box_muller64(w[0], w[1])
    b0, b1 = px.box_muller64(w[2], w[3])
    return np.stack([a0, a1, b0, b1], axis=1).reshape(-1)[:count]


def finalize(raw: np.ndarray, bg_offset: float, noise_std: float, seed: int = 0, batch: int = 0,
             gpair: int = 0, frame: int = 1) -> np.ndarray:
    """raster.py:154-161 restated (float64, clip to [0, 1], float32)."""
    img = raw.astype(np.float64)
    if bg_offset != 0.0:
        img = img + bg_offset
    if noise_std > 0.0:
        img = img + noise_std * noise_normals(seed, batch, gpair, frame, img.size).reshape(img.shape)
    return np.clip(img, 0.0, 1.0).astype(np.float32)


def quantize_u16(img: np.ndarray) -> np.ndarray:
    """export.py:19-20: rint(clip(x, 0, 1) * 65535) in float32, half-even."""
    x = np.clip(np.asarray(img, dtype=np.float32), np.float32(0.0), np.float32(1.0))
    return np.rint(x * np.float32(65535.0)).astype(np.uint16)


K_TIGHT_R = np.float32(5.6508017)   # sqrt(2 ln(2^22 / 0.49)) * 1.0001, as csrc/fused.cuh kTightR


def tight_window(fx, fy, sx, sy, halo, erf=False):
    """Per-record tight window of the B200 kernel (anchor offsets jlo..jhi,
    ilo..ihi): pixels outside it contribute an integer 0 at the maximum
    fixed-point shift (amp <= 1). Float32 ops mirror csrc/fused.cuh exactly."""
    fx = np.asarray(fx, np.float32)
    fy = np.asarray(fy, np.float32)
    R = (np.maximum(np.asarray(sx, np.float32), np.asarray(sy, np.float32)) * K_TIGHT_R).astype(np.float32)
    if erf:
        R = (R + np.float32(0.5)).astype(np.float32)
    jlo = np.maximum(-halo, np.ceil((fx - R).astype(np.float32)).astype(np.int64))
    jhi = np.minimum(halo, np.floor((fx + R).astype(np.float32)).astype(np.int64))
    ilo = np.maximum(-halo, np.ceil((fy - R).astype(np.float32)).astype(np.int64))
    ihi = np.minimum(halo, np.floor((fy + R).astype(np.float32)).astype(np.int64))
    return jlo, jhi, ilo, ihi


def anchors_f64(pos):
    """Anchor floor(x + 1/2) and float32 fraction of float64 positions (oracle mode)."""
    ax = np.floor(pos[:, 0] + 0.5)
    ay = np.floor(pos[:, 1] + 0.5)
    return ax.astype(np.int64), ay.astype(np.int64), (pos[:, 0] - ax).astype(np.float32), \
        (pos[:, 1] - ay).astype(np.float32)


def tile_counts(pos, on, sx, sy, halo, tile_h, tile_w, height, width, row_lo=0, row_hi=None,
                erf=False) -> np.ndarray:
    """Records per tile of the fused kernel's counting sort: each contributing
    particle goes to every tile its tight window (clipped to the image) touches."""
    row_hi = height if row_hi is None else row_hi
    rows = row_hi - row_lo
    tiles_y = -(-rows // tile_h)
    tiles_x = -(-width // tile_w)
    counts = np.zeros(tiles_y * tiles_x, dtype=np.int64)
    sel = np.flatnonzero(np.asarray(on) != 0)
    if sel.size == 0:
        return counts
    ax, ay, fx, fy = anchors_f64(pos[sel])
    jlo, jhi, ilo, ihi = tight_window(fx, fy, np.asarray(sx)[sel], np.asarray(sy)[sel], halo, erf)
    rlo = np.maximum(ay + ilo, row_lo)
    rhi = np.minimum(ay + ihi, row_hi - 1)
    clo = np.maximum(ax + jlo, 0)
    chi = np.minimum(ax + jhi, width - 1)
    ok = (jlo <= jhi) & (ilo <= ihi) & (rlo <= rhi) & (clo <= chi)
    for r_lo, r_hi, c_lo, c_hi in zip((rlo - row_lo)[ok] // tile_h, (rhi - row_lo)[ok] // tile_h,
                                      clo[ok] // tile_w, chi[ok] // tile_w):
        for ty in range(r_lo, r_hi + 1):
            counts[ty * tiles_x + c_lo: ty * tiles_x + c_hi + 1] += 1
    return counts


def match_histogram(img: np.ndarray, target) -> np.ndarray:
    """Histogram specification on 256 levels (restates reference raster.py:164-187):
    float32 levels rint(x * 255) clipped to [0, 255]; midpoint-CDF source
    quantile (cum - counts/2) / total in float64; first target-CDF entry >= it
    (searchsorted 'left', clipped to 255); output level / 255 as float32."""
    hist = np.asarray(target, dtype=np.float64)
    x = np.asarray(img, dtype=np.float32)
    lev = np.rint(x * np.float32(255.0)).astype(np.float32)
    lev = np.where(np.isnan(lev), np.float32(0.0), np.clip(lev, 0, 255)).astype(np.int64)
    counts = np.zeros(256, np.int64)
    np.add.at(counts, lev.reshape(-1), 1)
    cum = np.cumsum(counts).astype(np.float64)
    q = (cum - 0.5 * counts.astype(np.float64)) / float(x.size)
    cdf = np.cumsum(hist) / hist.sum()
    mapping = np.minimum(np.searchsorted(cdf, q, side="left"), 255)
    return (mapping[lev].astype(np.float64) / 255.0).astype(np.float32)
