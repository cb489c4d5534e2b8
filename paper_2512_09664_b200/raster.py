"""Rendering on the GPU: splat, finalize, quantisation (reference raster.py).

Oracle-mode images (caller-supplied particles) come from the inject kernel
(csrc/fused.cuh; csrc/wide.cuh for patch sides too large for its tile plan)
through the C ABI; the host functions here only move arrays and choose modes. Pixel
values accumulate as exact integers in 2^-22 units, so results do not depend
on tiling or banding (the reference guarantees band-independence by fixed
summation order, raster.py:108-126); they agree with the reference's float32
accumulation to ~1e-7.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from ._device import cuda_device, like_input, stream_ptr, to_dev
from .config import NoiseConfig
from .particles import Appearance, ParticleSet, RngKey


def patch_side(max_diameter: float, multiplier: float = 3.0) -> int:
    """Smallest odd side >= multiplier * max_diameter + 1 (raster.py:30-38).

    Same rule as the kernel's patch_side_exact (checked equal in tests)."""
    side = math.ceil(round(multiplier * max_diameter + 1.0, 9))
    if side % 2 == 0:
        side += 1
    return max(side, 1)


def eval_particle(i0: float, sigma_x: float, sigma_y: float, rho: float,
                  center: tuple[float, float], at: tuple[float, float]) -> float:
    """Eq. (1) of the paper at one point, float64 (raster.py:41-51)."""
    dx = at[0] - center[0]
    dy = at[1] - center[1]
    q = 1.0 - rho * rho
    quad = (dx * dx / (sigma_x * sigma_x) - 2.0 * rho * dx * dy / (sigma_x * sigma_y)
            + dy * dy / (sigma_y * sigma_y))
    return i0 * math.exp(-quad / (2.0 * q))


def kernel_patch(i0, sigma_x, sigma_y, rho, center, side):
    """side x side patch anchored at the nearest pixel (raster.py:54-69)."""
    ax = math.floor(center[0] + 0.5)
    ay = math.floor(center[1] + 0.5)
    half = side // 2
    out = np.empty((side, side), dtype=np.float64)
    for r in range(side):
        for c in range(side):
            out[r, c] = eval_particle(i0, sigma_x, sigma_y, rho, center,
                                      (ax - half + c, ay - half + r))
    return out, (ax, ay)


def _frame(pset: ParticleSet, frame: int):
    if frame == 1:
        pos, app, vis = pset.pos1, pset.app1, pset.visible1
    elif frame == 2:
        pos, app, vis = pset.pos2, pset.app2, pset.visible2
    else:
        raise ValueError(f"frame must be 1 or 2, got {frame}")
    if pos is None or app is None:
        raise ValueError(f"particle set is incomplete for frame {frame}")
    return pos, app, (pset.active if vis is None else vis)


def contribution_mask(pset: ParticleSet, frame: int) -> np.ndarray:
    """active & visible & i0 > 0 (raster.py:86-88)."""
    _, app, vis = _frame(pset, frame)
    return (np.asarray(pset.active) & np.asarray(vis) & (np.asarray(app.i0) > 0)).astype(np.uint8)


def splat_accumulate(pos, i0, sigma_x, sigma_y, rho, mask, side, out, row_start, row_stop,
                     psf: str = "point") -> None:
    """The reference's native seam (_native.pyx:14-17) on the GPU.

    Accumulates (+=) into ``out`` rows [row_start, row_stop). Accepts numpy
    (host round trip, like the reference) or CUDA tensors (in place)."""
    is_tensor = isinstance(out, torch.Tensor) and out.is_cuda
    dev = out.device if is_tensor else cuda_device()
    if not is_tensor:
        arr = np.asarray(out)
        if arr.dtype != np.float32 or not arr.flags.c_contiguous or not arr.flags.writeable:
            raise ValueError("out must be a writable C-contiguous float32 array")
    height, width = out.shape
    p = to_dev(pos, torch.float64, dev)
    if p.ndim != 2 or p.shape[-1] != 2:
        raise ValueError(f"pos must be (N, 2) float64, got {tuple(p.shape)}")
    n = p.shape[0]
    args = [to_dev(a, torch.float32, dev) for a in (i0, sigma_x, sigma_y, rho)]
    m = to_dev(mask, torch.uint8, dev)
    if any(a.numel() < n for a in args) or m.numel() < n:
        raise ValueError("per-particle arrays are shorter than pos")
    r0, r1 = max(0, int(row_start)), min(height, int(row_stop))
    if is_tensor:
        target = out
    else:
        # only the band's rows travel (in and back): concurrent calls on
        # disjoint bands of one image never overwrite each other's rows
        # (the reference's pool of splat_band jobs, raster.py:116-124)
        target = torch.zeros((height, width), dtype=torch.float32, device=dev)
        if r1 > r0:
            target[r0:r1].copy_(torch.from_numpy(np.asarray(out)[r0:r1]))
    _lib.call("pgb_splat_accumulate_dev", p.data_ptr(), args[0].data_ptr(), args[1].data_ptr(),
              args[2].data_ptr(), args[3].data_ptr(), m.data_ptr(), n, int(side),
              target.data_ptr(), height, width, r0, r1, _lib.PSF_CODES[psf], stream_ptr(dev))
    if not is_tensor and r1 > r0:
        np.copyto(out[r0:r1], target[r0:r1].cpu().numpy())


def splat_band(pset: ParticleSet, frame: int, out, side: int, row_start: int, row_stop: int) -> None:
    pos, app, _ = _frame(pset, frame)
    splat_accumulate(pos, app.i0, app.sigma_x, app.sigma_y, app.rho, contribution_mask(pset, frame),
                     side, out, row_start, row_stop)


def splat(pset: ParticleSet, frame: int, height: int, width: int, side: int,
          pool=None, bands: int = 1, psf: str = "point") -> np.ndarray:
    """Raw accumulation image, float32 >= 0, unclamped (raster.py:108-126).

    ``pool``/``bands`` are accepted for API compatibility; the GPU result does
    not depend on them."""
    out = np.zeros((height, width), dtype=np.float32)
    pos, app, _ = _frame(pset, frame)
    splat_accumulate(pos, app.i0, app.sigma_x, app.sigma_y, app.rho,
                     contribution_mask(pset, frame), side, out, 0, height, psf=psf)
    return out


def render_oracle(pset: ParticleSet, frame: int, height: int, width: int) -> np.ndarray:
    """Untruncated full-image render (raster.py:129-151): every masked particle
    at every pixel, float64, summed in particle-index order, rounded to float32
    once (pgb_render_oracle_dev). O(N H W): bounds the splat's truncation."""
    dev = cuda_device()
    pos, app, _ = _frame(pset, frame)
    p = to_dev(pos, torch.float64, dev)
    n = p.shape[0]
    args = [to_dev(a, torch.float32, dev) for a in (app.i0, app.sigma_x, app.sigma_y, app.rho)]
    m = to_dev(contribution_mask(pset, frame), torch.uint8, dev)
    out = torch.empty((height, width), dtype=torch.float32, device=dev)
    _lib.call("pgb_render_oracle_dev", p.data_ptr(), args[0].data_ptr(), args[1].data_ptr(),
              args[2].data_ptr(), args[3].data_ptr(), m.data_ptr(), n, height, width, out.data_ptr(),
              stream_ptr(dev))
    return out.cpu().numpy()


def _noise_args(noise: NoiseConfig):
    return float(noise.background_offset), float(noise.gaussian_std)


def finalize(raw, noise: NoiseConfig, key: RngKey, frame: int | None = None,
             out_dtype: str = "float32"):
    """Background offset + per-pixel Gaussian noise, clamped to [0, 1]
    (raster.py:154-161); noise from Philox keyed by (seed, batch, pair, frame).
    ``raw`` may be (H, W) or (P, H, W); numpy in, numpy out."""
    frame = key.frame if frame is None else frame
    dev = cuda_device()
    src = to_dev(raw, torch.float32, dev)
    shape = src.shape
    if src.ndim == 2:
        src = src.unsqueeze(0)
    pairs, height, width = src.shape
    dtype = torch.uint16 if out_dtype == "uint16" else torch.float32
    out = torch.empty(src.shape, dtype=dtype, device=dev)
    bg, sd = _noise_args(noise)
    mode = _lib.OUT_U16 if out_dtype == "uint16" else _lib.OUT_F32
    _lib.call("pgb_finalize_dev", src.data_ptr(), pairs, height, width, bg, sd, key.seed,
              key.batch, key.pair, frame, mode, out.data_ptr(), stream_ptr(dev))
    return like_input(out.reshape(shape), raw)


def quantize_u16(img):
    """rint(clip(x, 0, 1) * 65535) in float32 -> uint16 (export.py:19-20), bit-exact."""
    dev = cuda_device()
    src = to_dev(img, torch.float32, dev)
    out = torch.empty(src.shape, dtype=torch.uint16, device=dev)
    _lib.call("pgb_quantize_u16_dev", src.data_ptr(), src.numel(), out.data_ptr(), stream_ptr(dev))
    return like_input(out, img)


def target_cdf(target) -> np.ndarray:
    """cumsum(hist) / sum(hist) in float64, exactly as the reference (raster.py:181)."""
    hist = np.asarray(target, dtype=np.float64)
    if hist.shape != (256,):
        raise ValueError(f"target histogram must have 256 bins, got {hist.shape}")
    if (hist < 0).any() or not np.isfinite(hist).all() or hist.sum() <= 0:
        raise ValueError("target histogram must be non-negative with positive sum")
    return np.cumsum(hist) / hist.sum()


def match_histogram(img, target, out=None):
    """Histogram specification on 256 levels (raster.py:164-187), one CUDA
    block per image (csrc/histmatch.cuh), bit-identical to the reference.

    img: (H, W) or (N, H, W) float32 (numpy or torch); returns the same kind.
    `out` (a CUDA float32 tensor of img's shape, may be img itself) receives
    the result in place."""
    cdf = target_cdf(target)
    is_tensor = isinstance(img, torch.Tensor)
    dev = img.device if is_tensor and img.is_cuda else cuda_device()
    x = to_dev(img, torch.float32, dev).contiguous()
    if x.dim() < 2:
        raise ValueError("match_histogram expects an (H, W) or (N, H, W) image")
    pixels = x.shape[-1] * x.shape[-2]
    images = x.numel() // pixels if pixels else 0
    dst = out if out is not None else torch.empty_like(x)
    if dst.dtype != torch.float32 or not dst.is_contiguous() or dst.shape != x.shape or dst.device != x.device:
        raise ValueError("out must be a contiguous float32 tensor of the image's shape on its device")
    cdf_dev = torch.from_numpy(cdf).to(dev)
    _lib.call("pgb_match_histogram_dev", x.data_ptr(), dst.data_ptr(), images, pixels, cdf_dev.data_ptr(),
              stream_ptr(dev))
    return dst if is_tensor else dst.cpu().numpy()


def render_pair(pset: ParticleSet, height: int, width: int, side: int, noise: NoiseConfig,
                target_histogram, key: RngKey, pool=None, bands: int = 1,
                psf: str = "point") -> tuple[np.ndarray, np.ndarray]:
    """Splat + finalize (+ histogram) for both frames (raster.py:190-204),
    in one inject-kernel launch."""
    dev = cuda_device()
    frames = []
    for f in (1, 2):
        pos, app, _ = _frame(pset, f)
        frames.append(dict(
            pos=to_dev(pos, torch.float64, dev).reshape(1, -1, 2),
            i0=to_dev(app.i0, torch.float32, dev), sx=to_dev(app.sigma_x, torch.float32, dev),
            sy=to_dev(app.sigma_y, torch.float32, dev), rho=to_dev(app.rho, torch.float32, dev),
            mask=to_dev(contribution_mask(pset, f), torch.uint8, dev)))
    n = frames[0]["pos"].shape[1]
    outs = [torch.empty((1, height, width), dtype=torch.float32, device=dev) for _ in range(2)]
    structs = [_lib.PgbParticles(fr["pos"].data_ptr(), fr["i0"].data_ptr(), fr["sx"].data_ptr(),
                                 fr["sy"].data_ptr(), fr["rho"].data_ptr(), fr["mask"].data_ptr())
               for fr in frames]
    import ctypes

    sides = (ctypes.c_int * 1)(int(side))
    bg, sd = _noise_args(noise)
    _lib.call("pgb_render_pairs_dev", ctypes.byref(structs[0]), ctypes.byref(structs[1]), n, 1,
              sides, height, width, _lib.PSF_CODES[psf], _lib.OUT_F32, bg, sd, key.seed,
              key.batch, key.pair, outs[0].data_ptr(), outs[1].data_ptr(), None, None,
              stream_ptr(dev))
    imgs = []
    for o in outs:
        img = o[0]
        if target_histogram is not None:
            img = match_histogram(img, target_histogram)
        imgs.append(img.cpu().numpy())
    return imgs[0], imgs[1]
