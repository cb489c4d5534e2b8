// fused.cuh -- the batched image-pair generator as ONE cluster kernel.
//
// Replaces the body of Sampler._render_batch (reference pipeline.py:278-329):
// per pair, sample_particles / perturb_frame2 / advect / apply_hiding
// (particles.py:61-147), patch_side (raster.py:30-38, pipeline.py:291-294),
// splat (raster.py:108-126 -> _native.pyx:14-66) and finalize
// (raster.py:154-161) + quantize_u16 (export.py:19-20).
//
// Decomposition (B200-first):
//   * one thread-block CLUSTER per (pair, pass); CTA r of the cluster owns
//     screen tile (pass * CL + r) of the image for BOTH frames;
//   * seeding: CTA r generates the particle slice [r*N/CL, (r+1)*N/CL) with
//     Philox (or reads injected oracle arrays), advects it (bilinear, float64)
//     and bins it by destination tile -- a distributed counting sort:
//       count pass -> per-(frame, tile) counts in smem,
//       one remote atomicAdd per (frame, tile) on the owner's fill counter
//       reserves a contiguous slot range in the owner's shared memory,
//       write pass -> records are stored straight into the owner CTA's
//       shared memory through DSMEM (st.shared::cluster), overflow spills to
//       a per-CTA global region;
//   * render: each CTA splats its tile's particle list into a shared-memory
//     fixed-point (int32, 2^-s units) accumulator; contributions are integers,
//     so the per-pixel sum is exact and ORDER-INDEPENDENT -> the output bits
//     do not depend on scheduling, tiling, cluster size or GPU count;
//   * fused epilogue: offset + Philox noise + clamp (+ uint16 quantisation),
//     128-bit coalesced stores of the tile for each frame.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace pgb {

constexpr int kThreads = 512;
constexpr int kMaxCluster = 16;
constexpr int kAccShift = 22;     // default fixed-point fraction bits
constexpr int kCellMin = 8;       // coverage-guard cell size floor
constexpr float kLog2e = 1.4426950408889634f;

enum OutMode { kOutRaw = 0, kOutF32 = 1, kOutU16 = 2, kOutAccum = 3 };
enum Psf { kPsfPoint = 0, kPsfErf = 1 };

// 32-byte particle record exchanged between CTAs.
// After setup (point PSF) the fields (amp, sx, sy, rho) hold (L, A, B, C):
//   value * 2^s = exp2(L - (A dx^2 + B dx dy + C dy^2)),  L = log2(amp) + s.
// After setup (erf PSF): (amp', isx, isy, slope) -- see setup_erf().
struct __align__(16) Cand {
  int axy;      // anchor: ax in low 16 bits, ay in high 16 bits (both signed)
  float fx, fy; // sub-pixel offset from the anchor: x - ax, y - ay
  float amp;
  float sx, sy, rho;
  float aux;
};

struct GenCfg {
  int H, W, n;
  uint32_t k0, k1;
  double ppp_lo, ppp_hi, d_lo, d_hi, i0_lo, i0_hi, rho_lo, rho_hi;
  double sigma_ratio, patch_mult, hide_p;
  double z_lo, z_hi;
  float f2_sigma_std, f2_rho_std, f2_i0_std;
  float dz0, shape, q, w;
  int laser;
  int need_b, need_perturb;
};

struct InjFrame {
  const double* pos;
  const float* i0;
  const float* sx;
  const float* sy;
  const float* rho;
  const uint8_t* mask;
};

struct FusedParams {
  int H, W, row_lo, row_hi;
  int TH, TW, tiles_y, tiles_x, tiles, CL, passes;
  int cap, spill_cap, halo, nframes, cells_cap;
  int n, pairs;
  long long pair_base;
  uint32_t batch_lo;
  int psf, out_mode;
  float bg_offset, noise_std;
  int mode;  // 0 generate, 1 inject
  GenCfg g;
  const float2* flows;
  int pairs_per_field, num_fields;
  long long field_elems;
  InjFrame inj[2];
  const int* side_in;  // device, per pair (inject mode)
  void* out[2];
  long long out_pair_elems;
  double* st_ppp;
  int* st_M;
  int* st_side;
  float* st_dmax;
  int* bin_counts;
  Cand* spill;
  int* overflow;
};

struct SharedHdr {
  int fill[2];
  int cnt[2][kMaxCluster];
  int base[2][kMaxCluster];
  int cursor[2][kMaxCluster];
  unsigned dmax_bits;
  unsigned amp_bits;
  int cov_max;
  int M;
  double ppp;
};

struct Particle {
  double x[2], y[2];
  float amp[2], sx[2], sy[2], rho[2];
  bool on[2];
  float diam;
  bool active;
};

__device__ __forceinline__ float laser_profile(const GenCfg& g, float z) {
  // I0(z) = q exp(-(1/sqrt(2 pi)) |2 z^2 / dZ0^2|^s)
  const float t = 2.0f * z * z / (g.dz0 * g.dz0);
  const float p = t > 0.f ? powf(t, g.shape) : 0.f;
  return g.q * expf(-0.3989422804014327f * p);
}

// Per-particle seeding (generate mode) or injection (oracle mode).
template <int MODE>
__device__ __forceinline__ void make_particle(const FusedParams& P, int pl, int i, int M,
                                              Particle& pt) {
  if (MODE == 1) {
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      if (f >= P.nframes) { pt.on[f] = false; continue; }
      const InjFrame& F = P.inj[f];
      const size_t o = (size_t)pl * P.n + i;
      pt.x[f] = F.pos[2 * o];
      pt.y[f] = F.pos[2 * o + 1];
      pt.amp[f] = F.i0[o];
      pt.sx[f] = F.sx[o];
      pt.sy[f] = F.sy[o];
      pt.rho[f] = F.rho[o];
      pt.on[f] = F.mask[o] != 0;
    }
    pt.diam = 0.f;
    pt.active = false;
    return;
  }
  const GenCfg& g = P.g;
  const uint32_t gpair = (uint32_t)(P.pair_base + pl);
  const RngKey key{g.k0, g.k1, gpair, P.batch_lo};
  // sample_particles (particles.py:61-101): positions, diameter, intensity.
  const uint4 a = draw(key, (uint32_t)i, kTagParticleA);
  const double x1 = dmul(u32_to_unit(a.x), (double)g.W);
  const double y1 = dmul(u32_to_unit(a.y), (double)g.H);
  const double d = lerp_exact(g.d_lo, g.d_hi, u32_to_unit(a.z));
  const double i0 = lerp_exact(g.i0_lo, g.i0_hi, u32_to_unit(a.w));
  const bool active = i < M;
  double rho = g.rho_lo, z1 = 0.0;
  bool vis1 = true, vis2 = true;
  if (g.need_b) {
    const uint4 b = draw(key, (uint32_t)i, kTagParticleB);
    rho = lerp_exact(g.rho_lo, g.rho_hi, u32_to_unit(b.x));
    // apply_hiding (particles.py:139-147): visible iff U >= p_hide.
    vis1 = u32_to_unit(b.y) >= g.hide_p;
    vis2 = u32_to_unit(b.z) >= g.hide_p;
    z1 = lerp_exact(g.z_lo, g.z_hi, u32_to_unit(b.w));
  }
  const float i0f = active ? (float)i0 : 0.f;
  const float sig = (float)ddiv(d, g.sigma_ratio);
  const float rhof = (float)rho;
  float sx2 = sig, sy2 = sig, i02 = i0f, rho2 = rhof;
  if (g.need_perturb) {
    // perturb_frame2 (particles.py:104-126): zero-mean Gaussian jitter, floors/clamps.
    const uint4 c = draw(key, (uint32_t)i, kTagPerturb);
    const float2 n01 = box_muller(c.x, c.y);
    const float2 n23 = box_muller(c.z, c.w);
    if (g.f2_sigma_std > 0.f) {
      sx2 = (float)fmax((double)sig + (double)g.f2_sigma_std * (double)n01.x, 1e-3);
      sy2 = (float)fmax((double)sig + (double)g.f2_sigma_std * (double)n01.y, 1e-3);
    }
    if (g.f2_i0_std > 0.f) {
      const double t = fmin(fmax((double)i0f + (double)g.f2_i0_std * (double)n23.x, 0.0), 1.0);
      i02 = i0f == 0.f ? 0.f : (float)t;
    }
    if (g.f2_rho_std > 0.f) {
      const double lim = 1.0 - 1e-3;
      rho2 = (float)fmin(fmax((double)rhof + (double)g.f2_rho_std * (double)n23.y, -lim), lim);
    }
  }
  float amp1 = i0f, amp2 = i02;
  if (g.laser) {
    amp1 *= laser_profile(g, (float)z1);
    amp2 *= laser_profile(g, (float)z1 + g.w);
  }
  // advect (particles.py:129-136): one forward-Euler step through the
  // bilinear field, float64 exactly as the reference.
  const long long field = (P.pair_base + pl) / P.pairs_per_field;
  const float2* flow = P.flows + (size_t)field * P.field_elems;
  double u, v;
  sample_flow_exact(flow, g.H, g.W, x1, y1, &u, &v);
  pt.x[0] = x1;
  pt.y[0] = y1;
  pt.x[1] = dadd(x1, u);
  pt.y[1] = dadd(y1, v);
  pt.amp[0] = amp1;
  pt.amp[1] = amp2;
  pt.sx[0] = sig;
  pt.sy[0] = sig;
  pt.rho[0] = rhof;
  pt.sx[1] = sx2;
  pt.sy[1] = sy2;
  pt.rho[1] = rho2;
  // contribution_mask (raster.py:86-88): active & visible & i0 > 0.
  pt.on[0] = active && vis1 && amp1 > 0.f;
  pt.on[1] = active && vis2 && amp2 > 0.f;
  pt.diam = (float)d;
  pt.active = active;
}

// Anchor = nearest pixel floor(x + 0.5) (_native.pyx:31-32); returns false
// when the (2*halo+1)^2 window misses the covered region entirely.
__device__ __forceinline__ bool anchor_of(const FusedParams& P, double x, double y, int& ax,
                                          int& ay) {
  const double fxa = floor(dadd(x, 0.5));
  const double fya = floor(dadd(y, 0.5));
  const int hx = P.halo;
  if (!(fxa >= (double)(-hx) && fxa <= (double)(P.W - 1 + hx))) return false;
  if (!(fya >= (double)(P.row_lo - hx) && fya <= (double)(P.row_hi - 1 + hx))) return false;
  ax = (int)fxa;
  ay = (int)fya;
  return true;
}

// Destination tiles of a window, restricted to this pass. Calls fn(rank).
template <typename Fn>
__device__ __forceinline__ void for_each_dest(const FusedParams& P, int pass, int ax, int ay,
                                              Fn&& fn) {
  const int hx = P.halo;
  const int rlo = max(ay - hx, P.row_lo) - P.row_lo;
  const int rhi = min(ay + hx, P.row_hi - 1) - P.row_lo;
  const int clo = max(ax - hx, 0);
  const int chi = min(ax + hx, P.W - 1);
  const int ty0 = rlo / P.TH, ty1 = rhi / P.TH;
  const int tx0 = clo / P.TW, tx1 = chi / P.TW;
  const int t_lo = pass * P.CL;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) {
      const int d = ty * P.tiles_x + tx - t_lo;
      if (d >= 0 && d < P.CL) fn(d);
    }
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Round a non-negative value < 2^22 (+ a few ulp) to the nearest integer
// with two full-rate ALU ops (magic-number add), avoiding the F2I pipe.
__device__ __forceinline__ int round_small(float v) {
  return __float_as_int(v + 12582912.0f) - 0x4B400000;
}

__device__ __forceinline__ void setup_point(Cand& c, float s_scale_log2) {
  const float sx = c.sx, sy = c.sy, r = c.rho;
  const float q = 1.0f - r * r;
  const float a = 0.5f / (q * sx * sx);
  const float b = r / (q * sx * sy);
  const float cc = 0.5f / (q * sy * sy);
  c.sx = a * kLog2e;
  c.sy = -b * kLog2e;
  c.rho = cc * kLog2e;
  c.amp = (c.amp > 0.f ? __log2f(c.amp) : -INFINITY) + s_scale_log2;
}

// erf PSF: pixel-area mean of Eq. (1) over [c-1/2, c+1/2] x [r-1/2, r+1/2].
//   x | y is Gaussian with mean x0 + slope (y - y0), std sc = sx sqrt(1 - rho^2):
//   value = amp * int_dy exp(-dy^2 / (2 sy^2)) * sc sqrt(pi/2) [erf(.)-erf(.)] dy
// rho == 0: closed form in y as well.
constexpr int kGLPoints = 8;
__constant__ float kGLx[kGLPoints] = {-0.4801449282487681f, -0.3983332387068134f,
                                       -0.2627662050032837f, -0.0916173212478249f,
                                       0.0916173212478249f,  0.2627662050032837f,
                                       0.3983332387068134f,  0.4801449282487681f};
__constant__ float kGLw[kGLPoints] = {0.0506142681451881f, 0.1111905172266872f,
                                       0.1568533229389436f, 0.1813418916891810f,
                                       0.1813418916891810f, 0.1568533229389436f,
                                       0.1111905172266872f, 0.0506142681451881f};

__device__ __forceinline__ void setup_erf(Cand& c, float scale) {
  const float sx = c.sx, sy = c.sy, r = c.rho;
  const float sc = sx * sqrtf(fmaxf(1.0f - r * r, 0.f));
  const float k = 1.2533141373155001f;  // sqrt(pi/2)
  c.aux = (r == 0.f) ? 1.f : 0.f;
  if (r == 0.f) c.amp = c.amp * scale * (k * sx) * (k * sy);
  else c.amp = c.amp * scale * (k * sc);
  c.sx = 0.70710678118654752f / sc;        // 1 / (sc sqrt 2)
  c.rho = r * sx / sy;                       // slope of the conditional mean
  c.sy = 0.70710678118654752f / sy;        // 1 / (sy sqrt 2)
}

__device__ __forceinline__ const Cand* cand_at(const Cand* local, const Cand* spill, int cap,
                                               int k) {
  return k < cap ? local + k : spill + (k - cap);
}

// Accumulate one (candidate, patch row) work item.
template <int SIDE, int PSF>
__device__ __forceinline__ void splat_row(int* __restrict__ acc, const Cand& c, int side_rt,
                                          int i, int r0, int nr, int c0, int nc, int TW) {
  const int side = SIDE > 0 ? SIDE : side_rt;
  const int h = side >> 1;
  const int ay = c.axy >> 16;
  const int ax = (int)(short)(c.axy & 0xffff);
  const int row = ay - h + i - r0;
  if ((unsigned)row >= (unsigned)nr) return;
  const int col0 = ax - h - c0;
  int* base = acc + row * TW + col0;
  const float dy = (float)(i - h) - c.fy;
  if (PSF == kPsfPoint) {
    const float Ly = fmaf(-c.rho * dy, dy, c.amp);
    const float By = c.sy * dy;
#pragma unroll
    for (int j = 0; j < (SIDE > 0 ? SIDE : 64); ++j) {
      if (SIDE == 0 && j >= side) break;
      const float dx = (float)(j - h) - c.fx;
      const float t = fmaf(c.sx, dx, By);
      const float e = fmaf(-t, dx, Ly);
      const int q = round_small(ex2_approx(e));
      if ((unsigned)(col0 + j) < (unsigned)nc) atomicAdd(base + j, q);
    }
  } else {
    // erf PSF
    float wrow = 1.f;
    const bool sep = c.aux != 0.f;
    if (sep) wrow = erff((dy + 0.5f) * c.sy) - erff((dy - 0.5f) * c.sy);
    float eprev = 0.f;
    for (int j = 0; j <= side; ++j) {
      const float dxl = (float)(j - h) - c.fx - 0.5f;  // left edge of column j
      float val = 0.f;
      if (sep) {
        const float e = erff(dxl * c.sx);
        if (j > 0) val = (e - eprev) * wrow;
        eprev = e;
      } else if (j > 0) {
        const float dxc = dxl - 0.5f;  // centre of column j-1 relative to x0
        float s = 0.f;
#pragma unroll
        for (int g = 0; g < kGLPoints; ++g) {
          const float yy = dy + kGLx[g];
          const float mu = c.rho * yy;               // conditional mean offset
          const float gy = __expf(-yy * yy * (c.sy * c.sy));  // exp(-yy^2/(2 sy^2))
          const float hi = erff((dxc + 0.5f - mu) * c.sx);
          const float lo = erff((dxc - 0.5f - mu) * c.sx);
          s = fmaf(kGLw[g] * gy, hi - lo, s);
        }
        val = s;
      }
      if (j > 0) {
        const int jj = j - 1;
        const int q = __float2int_rn(val * c.amp);
        if ((unsigned)(col0 + jj) < (unsigned)nc && q != 0) atomicAdd(base + jj, q);
      }
    }
  }
}

template <int SIDE, int PSF>
__device__ void splat_items(int* __restrict__ acc, const Cand* __restrict__ local,
                            const Cand* __restrict__ spill, int cap, int K, int side, int r0,
                            int nr, int c0, int nc, int TW) {
  const int total = K * side;
  const float inv = 1.0f / (float)side;
  for (int w = threadIdx.x; w < total; w += kThreads) {
    int k = (int)(((float)w + 0.5f) * inv);  // exact for w < 2^22
    int i = w - k * side;
    const Cand c = *cand_at(local, spill, cap, k);
    splat_row<SIDE, PSF>(acc, c, side, i, r0, nr, c0, nc, TW);
  }
}

template <int PSF>
__device__ void splat_dispatch(int* acc, const Cand* local, const Cand* spill, int cap, int K,
                               int side, int r0, int nr, int c0, int nc, int TW) {
  if (PSF == kPsfPoint) {
    switch (side) {
      case 3: splat_items<3, PSF>(acc, local, spill, cap, K, side, r0, nr, c0, nc, TW); return;
      case 5: splat_items<5, PSF>(acc, local, spill, cap, K, side, r0, nr, c0, nc, TW); return;
      case 7: splat_items<7, PSF>(acc, local, spill, cap, K, side, r0, nr, c0, nc, TW); return;
      case 9: splat_items<9, PSF>(acc, local, spill, cap, K, side, r0, nr, c0, nc, TW); return;
      case 13: splat_items<13, PSF>(acc, local, spill, cap, K, side, r0, nr, c0, nc, TW); return;
      default: break;
    }
  }
  splat_items<0, PSF>(acc, local, spill, cap, K, side, r0, nr, c0, nc, TW);
}

// Pixel noise: Philox(quad = p >> 2, pair, batch, kTagNoise + frame) ->
// two Box-Muller pairs -> normals for pixels 4q .. 4q+3.
__device__ __forceinline__ float4 noise4(uint32_t k0, uint32_t k1, uint32_t gpair,
                                         uint32_t batch, uint32_t frame, uint32_t quad) {
  const uint4 w = philox4x32_10(make_uint4(quad, gpair, batch, kTagNoise + frame), k0, k1);
  const float2 a = box_muller(w.x, w.y);
  const float2 b = box_muller(w.z, w.w);
  return make_float4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ float finalize_px(float raw, float bg, float std_, float nz) {
  float x = raw + bg;
  if (std_ > 0.f) x = fmaf(std_, nz, x);
  return fminf(fmaxf(x, 0.0f), 1.0f);
}

__device__ __forceinline__ uint16_t quant_u16(float x) {
  // rint(clip(x, 0, 1) * 65535) in float32 (export.py:19-20)
  const float y = __fmul_rn(fminf(fmaxf(x, 0.0f), 1.0f), 65535.0f);
  return (uint16_t)__float2int_rn(y);
}

// Epilogue for one frame of one tile: convert, finalize, store, re-zero acc.
__device__ void store_tile(const FusedParams& P, int* __restrict__ acc, int pl, int f, int r0,
                           int nr, int c0, int nc, float inv_scale) {
  const uint32_t gpair = (uint32_t)(P.pair_base + pl);
  const int TW = P.TW;
  const size_t pair_off = (size_t)pl * (size_t)P.out_pair_elems;
  const bool vec = ((nc & 3) == 0) && ((P.W & 3) == 0) && ((c0 & 3) == 0) && ((TW & 3) == 0);
  const int mode = P.out_mode;
  const float bg = P.bg_offset, sd = P.noise_std;
  if (vec) {
    const int qpr = nc >> 2;  // quads per row
    const int total = nr * qpr;
    for (int e = threadIdx.x; e < total; e += kThreads) {
      const int row = e / qpr;
      const int cq = e - row * qpr;
      int4* ap = reinterpret_cast<int4*>(acc + row * TW + cq * 4);
      const int4 a = *ap;
      *ap = make_int4(0, 0, 0, 0);
      float4 v = make_float4((float)a.x * inv_scale, (float)a.y * inv_scale,
                             (float)a.z * inv_scale, (float)a.w * inv_scale);
      const size_t p = (size_t)(r0 + row) * P.W + (size_t)(c0 + cq * 4);
      if (mode == kOutRaw) {
        reinterpret_cast<float4*>(static_cast<float*>(P.out[f]) + pair_off + p)[0] = v;
      } else if (mode == kOutAccum) {
        float4* o = reinterpret_cast<float4*>(static_cast<float*>(P.out[f]) + pair_off + p);
        float4 old = *o;
        old.x += v.x; old.y += v.y; old.z += v.z; old.w += v.w;
        *o = old;
      } else {
        float4 nz = make_float4(0.f, 0.f, 0.f, 0.f);
        if (sd > 0.f) nz = noise4(P.g.k0, P.g.k1, gpair, P.batch_lo, (uint32_t)f + 1, (uint32_t)(p >> 2));
        v.x = finalize_px(v.x, bg, sd, nz.x);
        v.y = finalize_px(v.y, bg, sd, nz.y);
        v.z = finalize_px(v.z, bg, sd, nz.z);
        v.w = finalize_px(v.w, bg, sd, nz.w);
        if (mode == kOutF32) {
          reinterpret_cast<float4*>(static_cast<float*>(P.out[f]) + pair_off + p)[0] = v;
        } else {
          ushort4 u = make_ushort4(quant_u16(v.x), quant_u16(v.y), quant_u16(v.z), quant_u16(v.w));
          reinterpret_cast<ushort4*>(static_cast<uint16_t*>(P.out[f]) + pair_off + p)[0] = u;
        }
      }
    }
  } else {
    const int total = nr * nc;
    for (int e = threadIdx.x; e < total; e += kThreads) {
      const int row = e / nc;
      const int col = e - row * nc;
      int* ap = acc + row * TW + col;
      float v = (float)(*ap) * inv_scale;
      *ap = 0;
      const size_t p = (size_t)(r0 + row) * P.W + (size_t)(c0 + col);
      if (mode == kOutRaw) {
        static_cast<float*>(P.out[f])[pair_off + p] = v;
      } else if (mode == kOutAccum) {
        static_cast<float*>(P.out[f])[pair_off + p] += v;
      } else {
        float nzv = 0.f;
        if (sd > 0.f) {
          const float4 nz = noise4(P.g.k0, P.g.k1, gpair, P.batch_lo, (uint32_t)f + 1, (uint32_t)(p >> 2));
          const int j = (int)(p & 3);
          nzv = j == 0 ? nz.x : (j == 1 ? nz.y : (j == 2 ? nz.z : nz.w));
        }
        v = finalize_px(v, bg, sd, nzv);
        if (mode == kOutF32) static_cast<float*>(P.out[f])[pair_off + p] = v;
        else static_cast<uint16_t*>(P.out[f])[pair_off + p] = quant_u16(v);
      }
    }
  }
}

template <int MODE, int PSF>
__global__ void __launch_bounds__(kThreads, 2) fused_generate_kernel(const FusedParams P) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = P.CL;
  const int rank = (int)cluster.block_rank();
  const int cid = blockIdx.x / CL;
  const int nclusters = gridDim.x / CL;
  const int cluster_first = blockIdx.x - rank;
  const int tid = threadIdx.x;

  extern __shared__ __align__(16) unsigned char smem[];
  int* acc = reinterpret_cast<int*>(smem);
  Cand* cand = reinterpret_cast<Cand*>(smem + (size_t)P.TH * P.TW * sizeof(int));
  SharedHdr* sh = reinterpret_cast<SharedHdr*>(cand + (size_t)P.nframes * P.cap);
  int* cells = reinterpret_cast<int*>(sh + 1);
  // this CTA's private spill region (persistent grid => bounded footprint)
  Cand* my_spill = P.spill + (size_t)blockIdx.x * 2 * P.spill_cap;

  {
    int4* a4 = reinterpret_cast<int4*>(acc);
    const int n4 = (P.TH * P.TW) >> 2;
    for (int e = tid; e < n4; e += kThreads) a4[e] = make_int4(0, 0, 0, 0);
  }

  const int items = P.pairs * P.passes;
  for (int item = cid; item < items; item += nclusters) {
    const int pl = item / P.passes;
    const int pass = item - pl * P.passes;

    // ---- init (local state only; remote traffic starts after the sync) -----
    if (tid < 2 * kMaxCluster) {
      (&sh->cnt[0][0])[tid] = 0;
      (&sh->cursor[0][0])[tid] = 0;
    }
    if (tid == 0) {
      sh->fill[0] = sh->fill[1] = 0;
      sh->dmax_bits = 0u;
      sh->amp_bits = 0u;
      sh->cov_max = 0;
      int M = 0;
      double ppp = 0.0;
      if (MODE == 0) {
        const RngKey key{P.g.k0, P.g.k1, (uint32_t)(P.pair_base + pl), P.batch_lo};
        const uint4 w = draw(key, 0u, kTagPair);
        ppp = lerp_exact(P.g.ppp_lo, P.g.ppp_hi, u53_to_unit(w.x, w.y));
        // m = round(ppp * H * W) clamped to [0, N]   (particles.py:80-83)
        double m = rint(dmul(dmul(ppp, (double)P.g.H), (double)P.g.W));
        m = fmin(fmax(m, 0.0), (double)P.n);
        M = (int)m;
      }
      sh->M = M;
      sh->ppp = ppp;
    }
    cluster.sync();
    const int M = sh->M;

    const long long n = P.n;
    const int i_lo = (int)((long long)rank * n / CL);
    const int i_hi = (int)((long long)(rank + 1) * n / CL);

    // ---- count pass: bin this slice by destination tile --------------------
    unsigned dmax_local = 0u;
    for (int i = i_lo + tid; i < i_hi; i += kThreads) {
      Particle pt;
      make_particle<MODE>(P, pl, i, M, pt);
      if (MODE == 0 && pt.active) dmax_local = max(dmax_local, __float_as_uint(pt.diam));
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        if (f >= P.nframes || !pt.on[f]) continue;
        int ax, ay;
        if (!anchor_of(P, pt.x[f], pt.y[f], ax, ay)) continue;
        for_each_dest(P, pass, ax, ay, [&](int d) { atomicAdd(&sh->cnt[f][d], 1); });
      }
    }
    if (MODE == 0) {
      for (int o = 16; o > 0; o >>= 1)
        dmax_local = max(dmax_local, __shfl_xor_sync(~0u, dmax_local, o));
      if ((tid & 31) == 0 && dmax_local) atomicMax(&sh->dmax_bits, dmax_local);
    }
    __syncthreads();
    // ---- reserve contiguous slot ranges in the owners' shared memory -------
    if (tid < P.nframes * CL) {
      const int f = tid / CL, d = tid - (tid / CL) * CL;
      const int c = sh->cnt[f][d];
      if (c > 0) sh->base[f][d] = atomicAdd(cluster.map_shared_rank(&sh->fill[f], d), c);
    } else if (MODE == 0 && tid >= 64 && tid < 64 + CL) {
      const unsigned m = sh->dmax_bits;
      if (m) atomicMax(cluster.map_shared_rank(&sh->dmax_bits, tid - 64), m);
    }
    __syncthreads();

    // ---- write pass: regenerate, store records into the owners' smem -------
    for (int i = i_lo + tid; i < i_hi; i += kThreads) {
      Particle pt;
      make_particle<MODE>(P, pl, i, M, pt);
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        if (f >= P.nframes || !pt.on[f]) continue;
        int ax, ay;
        if (!anchor_of(P, pt.x[f], pt.y[f], ax, ay)) continue;
        Cand rec;
        rec.axy = (ay << 16) | (ax & 0xffff);
        rec.fx = (float)dsub(pt.x[f], (double)ax);
        rec.fy = (float)dsub(pt.y[f], (double)ay);
        rec.amp = pt.amp[f];
        rec.sx = pt.sx[f];
        rec.sy = pt.sy[f];
        rec.rho = pt.rho[f];
        rec.aux = 0.f;
        for_each_dest(P, pass, ax, ay, [&](int d) {
          const int slot = sh->base[f][d] + atomicAdd(&sh->cursor[f][d], 1);
          Cand* dst;
          if (slot < P.cap) {
            dst = cluster.map_shared_rank(cand, d) + (size_t)f * P.cap + slot;
          } else if (slot - P.cap < P.spill_cap) {
            dst = P.spill + ((size_t)(cluster_first + d) * 2 + f) * P.spill_cap + (slot - P.cap);
          } else {
            atomicAdd(P.overflow, 1);
            return;
          }
          const float4* s4 = reinterpret_cast<const float4*>(&rec);
          float4* d4 = reinterpret_cast<float4*>(dst);
          d4[0] = s4[0];
          d4[1] = s4[1];
        });
      }
    }
    cluster.sync();

    // ---- render --------------------------------------------------------------
    const int t = pass * CL + rank;
    int side;
    float dmax = 0.f;
    if (MODE == 0) {
      dmax = __uint_as_float(sh->dmax_bits);
      if (M == 0) dmax = (float)P.g.d_hi;
      side = patch_side_exact((double)dmax, P.g.patch_mult);
    } else {
      side = P.side_in[pl];
    }
    if (MODE == 0 && rank == 0 && pass == 0 && tid == 0) {
      if (P.st_ppp) P.st_ppp[pl] = sh->ppp;
      if (P.st_M) P.st_M[pl] = M;
      if (P.st_side) P.st_side[pl] = side;
      if (P.st_dmax) P.st_dmax[pl] = dmax;
    }
    if (t >= P.tiles) continue;
    const int ty = t / P.tiles_x, tx = t - (t / P.tiles_x) * P.tiles_x;
    const int r0 = P.row_lo + ty * P.TH;
    const int nr = min(P.TH, P.row_hi - r0);
    const int c0 = tx * P.TW;
    const int nc = min(P.TW, P.W - c0);
    const int h = side >> 1;

    for (int f = 0; f < P.nframes; ++f) {
      int K = sh->fill[f];
      if (P.bin_counts && tid == 0) P.bin_counts[((size_t)pl * 2 + f) * P.tiles + t] = K;
      if (K > P.cap + P.spill_cap) K = P.cap + P.spill_cap;
      Cand* local = cand + (size_t)f * P.cap;
      Cand* spill = my_spill + (size_t)f * P.spill_cap;
      // -- coverage guard: per-pixel particle count bound from a cell
      //    histogram (cells >= 2h+1 wide: a pixel's anchor window lies in a
      //    2x2 block); picks the fixed-point shift so int32 cannot overflow.
      const int S = max(2 * h + 1, kCellMin);
      const int ncy = (nr + 2 * h + S - 1) / S, ncx = (nc + 2 * h + S - 1) / S;
      const bool cells_ok = ncy * ncx <= P.cells_cap;
      if (cells_ok)
        for (int e = tid; e < ncy * ncx; e += kThreads) cells[e] = 0;
      __syncthreads();
      unsigned amp_local = 0u;
      for (int k = tid; k < K; k += kThreads) {
        const Cand* c = cand_at(local, spill, P.cap, k);
        amp_local = max(amp_local, __float_as_uint(fmaxf(c->amp, 0.f)));
        if (cells_ok) {
          const int ay = c->axy >> 16, ax = (int)(short)(c->axy & 0xffff);
          const int cy = ay - (r0 - h), cx = ax - (c0 - h);
          if (cy >= 0 && cy < nr + 2 * h && cx >= 0 && cx < nc + 2 * h)
            atomicAdd(&cells[(cy / S) * ncx + cx / S], 1);
        }
      }
      for (int o = 16; o > 0; o >>= 1)
        amp_local = max(amp_local, __shfl_xor_sync(~0u, amp_local, o));
      if ((tid & 31) == 0) atomicMax(&sh->amp_bits, amp_local);
      __syncthreads();
      if (cells_ok) {
        int cm = 0;
        for (int e = tid; e < ncy * ncx; e += kThreads) {
          const int cy = e / ncx, cx = e - (e / ncx) * ncx;
          int s = cells[e];
          if (cx + 1 < ncx) s += cells[e + 1];
          if (cy + 1 < ncy) s += cells[e + ncx];
          if (cx + 1 < ncx && cy + 1 < ncy) s += cells[e + ncx + 1];
          cm = max(cm, s);
        }
        for (int o = 16; o > 0; o >>= 1) cm = max(cm, __shfl_xor_sync(~0u, cm, o));
        if ((tid & 31) == 0) atomicMax(&sh->cov_max, cm);
      }
      __syncthreads();
      const float amp_max = __uint_as_float(sh->amp_bits);
      int shift = kAccShift;
      if (amp_max > 1.0f) shift -= (int)ceilf(log2f(amp_max));
      {
        const float cov = cells_ok ? (float)sh->cov_max : (float)K;
        const float units = cov * fmaxf(amp_max, 1e-30f);
        if (units > 0.f) {
          // keep cov * amp_max * 2^shift + cov < 2^31
          const int lim = 30 - (int)ceilf(log2f(units + 1.0f));
          if (shift > lim) shift = lim;
        }
      }
      // -- per-candidate coefficients, in place
      for (int k = tid; k < K; k += kThreads) {
        Cand* c = const_cast<Cand*>(cand_at(local, spill, P.cap, k));
        if (PSF == kPsfPoint) setup_point(*c, (float)shift);
        else setup_erf(*c, exp2f((float)shift));
      }
      __syncthreads();
      if (tid == 0) {
        sh->amp_bits = 0u;
        sh->cov_max = 0;
      }
      // -- splat: integer accumulation in shared memory
      splat_dispatch<PSF>(acc, local, spill, P.cap, K, side, r0, nr, c0, nc, P.TW);
      __syncthreads();
      // -- fused epilogue
      store_tile(P, acc, pl, f, r0, nr, c0, nc, exp2f(-(float)shift));
      __syncthreads();
    }
  }
}

}  // namespace pgb
