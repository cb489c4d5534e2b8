// fused.cuh -- the batched image-pair generator as ONE persistent kernel.
//
// Replaces the body of Sampler._render_batch (reference pipeline.py:278-329):
// per pair, sample_particles / perturb_frame2 / advect / apply_hiding
// (particles.py:61-147), patch_side (raster.py:30-38, pipeline.py:291-294),
// splat (raster.py:108-126 -> _native.pyx:14-66) and finalize
// (raster.py:154-161) + quantize_u16 (export.py:19-20).
//
// Schedule (B200-first): a persistent grid pulls work tickets
// from one global counter. Two kinds of work item:
//   * GENERATE (pair p, chunk c): Philox seeding in fixed point + float32 (or
//     oracle injection), bilinear advection, and a counting sort of the
//     chunk's particles into per-(frame, screen tile) record lists of pair
//     slot p % ring -- local shared-memory ranks, ONE global atomicAdd per
//     (frame, tile) per round reserves the slots, coalesced record stores.
//   * RENDER (pair p, tile t): waits until all chunks of p are binned, splats
//     the tile's records into a padded shared-memory fixed-point accumulator
//     (int32, 2^-s units; integer addition is associative, so pixel sums are
//     exact and order-independent -> bit-identical output for any schedule,
//     tiling or GPU count), then the fused epilogue (offset + Philox noise +
//     clamp, optional uint16 quantisation) with 128-bit streaming stores.
// Tickets are ordered so every wait targets an earlier ticket (deadlock-free):
// generation runs `lookahead` pairs ahead of rendering; the record ring stays
// L2-resident. Patch pixels whose value provably rounds to zero in the
// fixed-point accumulator are skipped (tight window), which cannot change a bit.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace pgb {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kAccShift = 22;     // max fixed-point fraction bits
constexpr int kCellMin = 8;       // coverage-guard cell size floor
constexpr float kLog2e = 1.4426950408889634f;

enum OutMode { kOutRaw = 0, kOutF32 = 1, kOutU16 = 2, kOutAccum = 3 };
enum Psf { kPsfPoint = 0, kPsfErf = 1 };

// 32-byte render-ready particle record, addressed for its owning tile.
//   point PSF:  value * 2^s = exp2(L + s - (A dx^2 + B dx dy + C dy^2)), with
//               dx = dx0 + j, dy = dy0 + i for window lane column j / row i
//   erf PSF:    L = amp', A = 1/(sc sqrt2), B = 1/(sy sqrt2), C = slope (0: separable)
// The window (Wr x Hr pixels starting at anchor offset (jlo, ilo)) is the
// record's TIGHT window: every pixel outside it would contribute an integer 0
// at the maximum fixed-point shift, so skipping it cannot change a bit.
struct __align__(16) Rec {
  int addr;      // accumulator offset (ints) of the window's first pixel in the owning tile
  float dx0;     // jlo - fx
  float dy0;     // ilo - fy
  float L;
  float A, B, C;
  int meta;      // jlo (int8) | ilo (int8) << 8 | Wr << 16 | Hr << 24
};

struct GenCfg {
  int H, W, n;
  uint32_t k0, k1;
  PhiloxKeys rk;             // round keys of (k0, k1)
  double ppp_lo, ppp_hi;
  float d_lo, d_span, i0_lo, i0_span, rho_lo, rho_span, inv_ratio;
  double patch_mult, d_hi;
  uint64_t hide_thr;         // visible iff word >= hide_thr  (exactly U >= p)
  float z_lo, z_span;
  float f2_sigma_std, f2_rho_std, f2_i0_std;
  float dz0, shape, q, w, inv_dz0sq;
  int laser;
  int need_b, need_perturb;
};

// Tight-window radius factor: R = sigma * kR, kR = sqrt(2 ln(2^22 / 0.49)) * 1.0001
// (records with amp <= 1; larger amplitudes widen R by ln(amp), see record_radius).
constexpr float kTightR = 5.6508017f;

struct InjFrame {
  const double* pos;
  const float* i0;
  const float* sx;
  const float* sy;
  const float* rho;
  const uint8_t* mask;
};

// Per pair-slot bookkeeping in global memory (ring of `ring` slots).
struct __align__(16) SlotHdr {
  int gen_done;        // generate items of the current occupant finished
  int render_done;     // render items finished
  int epoch;           // number of occupants retired (slot of pair p is free when epoch == p / ring)
  unsigned amp;        // max record amplitude (float bits)
  int wmax[2];         // per frame max record window width (columns or rows)
  int pad0, pad1;
};

struct FusedParams {
  int H, W, row_lo, row_hi;
  int TH, TW, tiles_y, tiles_x, tiles, th_shift, tw_shift;
  int cap;                 // record capacity per (slot, frame, tile, chunk) segment
  int rbuf;                // shared-memory record buffer per frame (render)
  int halo, nframes, cells_cap;
  int pad, AH, AS;         // accumulator: AH rows x AS ints (tile + pad on each side)
  int n, pairs, chunk, chunks, ring, lookahead;
  long long pair_base;
  uint32_t batch_lo;
  int psf, out_mode;
  float bg_offset, noise_std;
  uint32_t k0, k1;     // seed (noise keys)
  InjFrame inj[2];
  const int* side_in;  // device, per pair (inject mode)
  void* out[2];
  long long out_pair_elems;
  int* bin_counts;
  // workspace
  Rec* recs;           // [ring][nframes][tiles][chunks][cap]
  int* fills;          // [ring][nframes][tiles][chunks] segment counts
  SlotHdr* slots;      // [ring]
  int* ticket;         // work counter (zeroed before launch)
  int* overflow;
};

// Per-CTA shared control block.
struct __align__(16) SharedHdr {
  unsigned long long bar;   // mbarrier: TMA bulk loads of a render item's records
  int item;                 // current ticket
  unsigned amp;
  int wmax[2];
  int cov_max, shift;
  int K[2];                 // records per frame of the current render item
};

// ----------------------------------------------------------------------------
// Seeding (generate mode): fixed-point positions, float32 attributes.
//   x1 = (2 w + 1) W / 2^33 exactly; anchor = floor(x1 + 1/2); the fraction is
//   rounded once to float32. Advection and all attribute arithmetic are
//   separately rounded float32 ops (no contraction), restated bit-exactly by
//   oracle/generate.py.
// ----------------------------------------------------------------------------
struct Frame {
  int ax, ay;
  float fx, fy;
  float amp, sx, sy, rho;
  bool on;
};

struct Particle {
  Frame fr[2];
  float diam, z1;
  bool active, vis1, vis2;
};

// Open-interval float32 uniform ((w >> 9) + 1/2) 2^-23: exact, strictly inside (0, 1).
PGB_HD float unit23(uint32_t w) { return ((float)(w >> 9) + 0.5f) * 0x1p-23f; }

__device__ __forceinline__ float lerpf_exact(float lo, float span, float u) {
  return __fadd_rn(lo, __fmul_rn(span, u));
}

// Fixed-point coordinates (Q17): value = X / 2^17 with X odd, i.e. the centre
// of a 2^-16 px bin; all position arithmetic is 32-bit integer (images < 16384 px).
// Coordinate -> (anchor floor(v + 1/2), float32 fraction; exact, |f| <= 1/2).
__device__ __forceinline__ void fixed_anchor(uint32_t X, int& a, float& f) {
  const uint32_t an = (X + (1u << 16)) >> 17;
  a = (int)an;
  f = (float)(int)(X - (an << 17)) * 0x1p-17f;
}

// Clamped bilinear cell: x = min(v, N-1), c = min(floor x, N-2), t = x - c (exact).
__device__ __forceinline__ void fixed_cell(uint32_t X, int N, int& c, float& t) {
  const uint32_t lim = (uint32_t)(N - 1) << 17;
  const uint32_t xc = X < lim ? X : lim;
  int cc = (int)(xc >> 17);
  const int cmax = N - 2 > 0 ? N - 2 : 0;
  cc = cc < cmax ? cc : cmax;
  c = cc;
  t = (float)(int)(xc - ((uint32_t)cc << 17)) * 0x1p-17f;
}

// Uniform Q17 coordinate inside seeding cell `cell` of width CW = size / 2^bits
// px (CW << 16 is an integer for bits <= 16): X = 2 (cell CW16 + floor(w CW16 / 2^32)) + 1.
__device__ __forceinline__ uint32_t cell_coord(uint32_t cell, uint32_t w, int size, int bits) {
  const uint32_t cw = (uint32_t)size << (16 - bits);
  return ((cell * cw + __umulhi(w, cw)) << 1) | 1u;
}

__device__ __forceinline__ float bilerp(float g00, float g01, float g10, float g11, float tx,
                                        float ty) {
  const float sx = __fsub_rn(1.0f, tx), sy = __fsub_rn(1.0f, ty);
  const float top = __fadd_rn(__fmul_rn(sx, g00), __fmul_rn(tx, g01));
  const float bot = __fadd_rn(__fmul_rn(sx, g10), __fmul_rn(tx, g11));
  return __fadd_rn(__fmul_rn(sy, top), __fmul_rn(ty, bot));
}

// Advection in fixed point: the frame-1 fraction (Q17, exact) and the
// displacement rint(d * 2^20) are added in Q20 (the displacement is quantised
// to 2^-20 px, exactly); then anchor + floor(t + 1/2) and the exact float32
// fraction (<= 20 fractional bits, so window offsets dy = i - f stay exact for
// |i| < 16 and images are bit-identical for every tiling).
__device__ __forceinline__ void advect_anchor(uint32_t X, int a, float d, int& a2, float& f2) {
  const int t = ((int)(X - ((uint32_t)a << 17)) << 3) + __float2int_rn(d * 1048576.0f);
  const int k = (t + (1 << 19)) >> 20;   // arithmetic shift: floor
  a2 = a + k;
  f2 = (float)(t - (k << 20)) * 0x1p-20f;
}

__device__ __forceinline__ float laser_profile(const GenCfg& g, float z) {
  // I0(z) = q exp(-(1/sqrt(2 pi)) |2 z^2 / dZ0^2|^s).
  // MUFU lg2/ex2 instead of powf/expf (measured 11% of C4's instructions):
  // amplitude relative error ~1e-6 (tests: rtol 2e-5 vs the float64 oracle);
  // the common shapes 1 and 2 are exact products. Warp-uniform branches.
  float lg, e2;
  const float t = 2.0f * z * z * g.inv_dz0sq;
  float p;
  if (g.shape == 2.0f) {
    p = t * t;
  } else if (g.shape == 1.0f) {
    p = t;
  } else {
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(t));
    float ep;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ep) : "f"(g.shape * lg));
    p = t > 0.f ? ep : 0.f;
  }
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e2) : "f"(-0.3989422804014327f * kLog2e * p));
  return g.q * e2;
}

// Oracle mode: float64 positions from the reference; anchor = floor(x + 1/2)
// (_native.pyx:31-32), fraction rounded once to float32.
__device__ __forceinline__ void inject_particle(const FusedParams& P, int pl, int i,
                                                Particle& pt) {
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    Frame& fr = pt.fr[f];
    fr.on = false;
    if (f >= P.nframes) continue;
    const InjFrame& F = P.inj[f];
    const size_t o = (size_t)pl * P.n + i;
    if (!F.mask[o]) continue;
    const double x = F.pos[2 * o], y = F.pos[2 * o + 1];
    const double fxa = floor(dadd(x, 0.5)), fya = floor(dadd(y, 0.5));
    // far-away particles are rejected by the window test; keep int conversion safe
    if (!(fabs(fxa) < 1e8 && fabs(fya) < 1e8)) continue;
    fr.ax = (int)fxa;
    fr.ay = (int)fya;
    fr.fx = (float)dsub(x, fxa);
    fr.fy = (float)dsub(y, fya);
    fr.amp = F.i0[o];
    fr.sx = F.sx[o];
    fr.sy = F.sy[o];
    fr.rho = F.rho[o];
    fr.on = true;
  }
  pt.diam = 0.f;
  pt.active = false;
}

// Tight-window radius of a record (pixels); exact-reproducible for amp <= 1
// (one float32 multiply); larger amplitudes add ln(amp) to the exponent budget.
__device__ __forceinline__ float record_radius(const Frame& fr, int psf) {
  const float sm = fmaxf(fr.sx, fr.sy);
  float R = __fmul_rn(sm, kTightR);
  if (fr.amp > 1.0f) R = sm * sqrtf(2.0f * (15.962588f + logf(fr.amp))) * 1.0001f;
  if (psf != kPsfPoint) R += 0.5f;     // pixel-area mean: nearest point of the pixel
  return R;
}

// Coefficients + window of a record; addr is filled in per destination tile.
__device__ __forceinline__ Rec make_rec(const Frame& fr, int psf, int jlo, int ilo, int Wr, int Hr) {
  Rec r;
  r.addr = 0;
  r.dx0 = (float)jlo - fr.fx;
  r.dy0 = (float)ilo - fr.fy;
  r.meta = (jlo & 0xff) | ((ilo & 0xff) << 8) | (Wr << 16) | (Hr << 24);
  const float sx = fr.sx, sy = fr.sy, rho = fr.rho;
  if (psf == kPsfPoint) {
    const float q = 1.0f - rho * rho;
    const float isx = __frcp_rn(sx), isy = __frcp_rn(sy), iq = __frcp_rn(q);
    r.A = (0.5f * kLog2e) * iq * isx * isx;
    r.C = (0.5f * kLog2e) * iq * isy * isy;
    r.B = -kLog2e * rho * iq * isx * isy;
    r.L = __log2f(fr.amp);
  } else {
    const float k = 1.2533141373155001f;  // sqrt(pi/2)
    const float sc = sx * sqrtf(fmaxf(1.0f - rho * rho, 0.f));
    const bool sep = rho == 0.f;
    r.L = sep ? fr.amp * (k * sx) * (k * sy) : fr.amp * (k * sc);
    r.A = 0.70710678118654752f / sc;
    r.B = 0.70710678118654752f / sy;
    r.C = sep ? 0.f : rho * sx / sy;
  }
  return r;
}

// ----------------------------------------------------------------------------
// Render: lanes = (record slot, window column); each lane walks the rows.
// ----------------------------------------------------------------------------
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Round a non-negative value <= 2^22 (+ a few ulp) to the nearest integer with
// two full-rate ALU ops (magic-number add), avoiding the conversion pipe.
__device__ __forceinline__ int round_small(float v) {
  return __float_as_int(v + 12582912.0f) - 0x4B400000;
}

constexpr int kGLPoints = 8;
__constant__ float kGLx[kGLPoints] = {-0.48014492824876809f, -0.39833323870681336f, -0.2627662049581645f, -0.09171732124782489f, 0.091717321247824893f, 0.2627662049581645f, 0.39833323870681336f, 0.48014492824876809f};
__constant__ float kGLw[kGLPoints] = {0.050614268145188532f, 0.11119051722668721f, 0.15685332293894344f, 0.18134189168918083f, 0.18134189168918083f, 0.15685332293894344f, 0.11119051722668721f, 0.050614268145188532f};

// One lane: column j of the record's window, rows 0..Hr-1; columns/rows beyond
// the pair's patch half-width h are the reference's truncation (_native.pyx:34-49).
template <int WC, int PSF>
__device__ __forceinline__ void splat_lane(int* __restrict__ acc, const Rec& r, int Wrt, int j,
                                           int h, int AS, float s_log2, float scale) {
  const int W = WC > 0 ? WC : Wrt;
  const int jlo = (int)(signed char)(r.meta & 0xff);
  const int ilo = (int)(signed char)((r.meta >> 8) & 0xff);
  const int Wr = (r.meta >> 16) & 0xff;
  const int Hr = (r.meta >> 24) & 0xff;
  const int jo = jlo + j;
  if (j >= Wr || jo < -h || jo > h) return;
  const int ib = max(0, -h - ilo);
  const int ie = min(Hr, h - ilo + 1);
  int* p = acc + r.addr + j;
  const float dx = r.dx0 + (float)j;
  if (PSF == kPsfPoint) {
    const float Lx = fmaf(-r.A * dx, dx, r.L + s_log2);
    const float Bdx = r.B * dx;
#pragma unroll 5
    for (int i = 0; i < (WC > 0 ? WC : 64); ++i) {
      if (WC == 0 && i >= W) break;
      if (i < ib || i >= ie) continue;
      const float dy = r.dy0 + (float)i;
      const float t = fmaf(r.C, dy, Bdx);
      const float e = fmaf(-t, dy, Lx);
      atomicAdd(p + i * AS, round_small(ex2_approx(e)));
    }
  } else {
    const bool sep = r.C == 0.f;
    float ex = 0.f;
    if (sep) ex = erff((dx + 0.5f) * r.A) - erff((dx - 0.5f) * r.A);
    for (int i = ib; i < ie; ++i) {
      const float dy = r.dy0 + (float)i;
      float val;
      if (sep) {
        val = ex * (erff((dy + 0.5f) * r.B) - erff((dy - 0.5f) * r.B));
      } else {
        float s = 0.f;
#pragma unroll
        for (int gq = 0; gq < kGLPoints; ++gq) {
          const float yy = dy + kGLx[gq];
          const float mu = r.C * yy;
          const float gy = __expf(-yy * yy * (r.B * r.B));
          const float hi = erff((dx + 0.5f - mu) * r.A);
          const float lo = erff((dx - 0.5f - mu) * r.A);
          s = fmaf(kGLw[gq] * gy, hi - lo, s);
        }
        val = s;
      }
      const int q = __float2int_rn(val * r.L * scale);
      if (q) atomicAdd(p + i * AS, q);
    }
  }
}

// Records come from shared memory (TMA-staged) or, for oversized lists, L2.
__device__ __forceinline__ Rec load_rec(const Rec* q) {
  float4 a, b;
  if (__isShared(q)) {
    a = reinterpret_cast<const float4*>(q)[0];
    b = reinterpret_cast<const float4*>(q)[1];
  } else {
    a = __ldcg(reinterpret_cast<const float4*>(q));
    b = __ldcg(reinterpret_cast<const float4*>(q) + 1);
  }
  Rec r;
  r.addr = __float_as_int(a.x); r.dx0 = a.y; r.dy0 = a.z; r.L = a.w;
  r.A = b.x; r.B = b.y; r.C = b.z; r.meta = __float_as_int(b.w);
  return r;
}

template <int WC, int PSF>
__device__ void splat_tile(int* __restrict__ acc, const Rec* __restrict__ recs, int K, int Wrt,
                           int h, int AS, float s_log2, float scale) {
  const int W = WC > 0 ? WC : Wrt;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (W <= 32) {
    const int cpw = 32 / W;                         // records per warp-step
    const int slot = lane / W;
    const int j = lane - slot * W;
    if (slot >= cpw) return;
    for (int k = warp * cpw + slot; k < K; k += kWarps * cpw)
      splat_lane<WC, PSF>(acc, load_rec(recs + k), W, j, h, AS, s_log2, scale);
  } else {
    // very large windows: the warp walks one record, lanes stride the columns
    for (int k = warp; k < K; k += kWarps) {
      const Rec r = load_rec(recs + k);
      for (int jj = lane; jj < W; jj += 32)
        splat_lane<0, PSF>(acc, r, W, jj, h, AS, s_log2, scale);
    }
  }
}

template <int PSF>
__device__ void splat_dispatch(int* acc, const Rec* recs, int K, int W, int h, int AS,
                               float s_log2, float scale) {
#define PGB_SPLAT(WW) splat_tile<WW, PSF>(acc, recs, K, W, h, AS, s_log2, scale)
  if (PSF == kPsfPoint) {
    switch (W) {
      case 2: PGB_SPLAT(2); return;
      case 3: PGB_SPLAT(3); return;
      case 4: PGB_SPLAT(4); return;
      case 5: PGB_SPLAT(5); return;
      case 6: PGB_SPLAT(6); return;
      case 7: PGB_SPLAT(7); return;
      case 8: PGB_SPLAT(8); return;
      case 9: PGB_SPLAT(9); return;
      case 11: PGB_SPLAT(11); return;
      case 13: PGB_SPLAT(13); return;
      default: break;
    }
  }
  PGB_SPLAT(0);
#undef PGB_SPLAT
}

// Largest fixed-point shift s <= kAccShift with cnt * (amp_max * 2^s + 1/2) < 2^31.
__device__ __forceinline__ int shift_for(int cnt, float amp_max) {
  const double per = (2147483648.0 / (double)cnt - 0.5) / (double)amp_max;
  if (!(per >= 1.0)) return 0;
  int e = ilogb(per);                      // floor(log2(per)), exact
  return e < kAccShift ? e : kAccShift;
}

// ----------------------------------------------------------------------------
// Epilogue
// ----------------------------------------------------------------------------
// Pixel noise: Philox(quad = p >> 2, pair, batch, kTagNoise + frame) ->
// two Box-Muller pairs -> normals for pixels 4q .. 4q+3.
__device__ __forceinline__ float4 noise4_rk(const PhiloxKeys& K, uint32_t gpair, uint32_t batch,
                                            uint32_t frame, uint32_t quad) {
  const uint4 w = philox_rk(make_uint4(quad, gpair, batch, kTagNoise + frame), K);
  const float2 a = box_muller(w.x, w.y);
  const float2 b = box_muller(w.z, w.w);
  return make_float4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ float4 noise4(uint32_t k0, uint32_t k1, uint32_t gpair,
                                         uint32_t batch, uint32_t frame, uint32_t quad) {
  const uint4 w = philox4x32_10(make_uint4(quad, gpair, batch, kTagNoise + frame), k0, k1);
  const float2 a = box_muller(w.x, w.y);
  const float2 b = box_muller(w.z, w.w);
  return make_float4(a.x, a.y, b.x, b.y);
}

// clip(raw + offset + std * n, 0, 1) (raster.py:154-161): offset + std * n in
// one FFMA, then one saturating add. The fused epilogue computes the same
// value as FFMA.SAT(acc, 2^-s, offset + std * n) (acc * 2^-s is exact), so the
// standalone and the fused finalize are bit-identical.
__device__ __forceinline__ float finalize_px(float raw, float bg, float std_, float nz) {
  return __saturatef(raw + fmaf(std_, nz, bg));
}

__device__ __forceinline__ uint16_t quant_u16(float x) {
  // rint(clip(x, 0, 1) * 65535) in float32 (export.py:19-20)
  const float y = __fmul_rn(fminf(fmaxf(x, 0.0f), 1.0f), 65535.0f);
  return (uint16_t)__float2int_rn(y);
}

// int accumulator (>= 0, < 2^23) -> float with two ALU ops.
__device__ __forceinline__ float acc_to_float(int a) {
  return __int_as_float(a | 0x4B000000) - 8388608.0f;
}
// One output quad (4 pixels) of frame f.
template <int OUT, bool NOISE>
__device__ __forceinline__ void store_quad(const FusedParams& P, const int4 a, char* dst,
                                           size_t pix, int f, uint32_t gpair, float inv_scale) {
  float4 v;
  if ((a.x | a.y | a.z | a.w) >= (1 << 23)) {
    v = make_float4((float)a.x, (float)a.y, (float)a.z, (float)a.w);
  } else {
    v = make_float4(acc_to_float(a.x), acc_to_float(a.y), acc_to_float(a.z), acc_to_float(a.w));
  }
  if (OUT == kOutRaw) {
    v.x *= inv_scale; v.y *= inv_scale; v.z *= inv_scale; v.w *= inv_scale;
    __stcs(reinterpret_cast<float4*>(dst), v);
  } else if (OUT == kOutAccum) {
    float4* o = reinterpret_cast<float4*>(dst);
    float4 old = *o;
    old.x = fmaf(v.x, inv_scale, old.x); old.y = fmaf(v.y, inv_scale, old.y);
    old.z = fmaf(v.z, inv_scale, old.z); old.w = fmaf(v.w, inv_scale, old.w);
    *o = old;
  } else {
    const float bg = P.bg_offset;
    if (NOISE) {
      const float sd = P.noise_std;
      const float4 nz = noise4(P.k0, P.k1, gpair, P.batch_lo, (uint32_t)f + 1, (uint32_t)(pix >> 2));
      v.x = finalize_px(v.x * inv_scale, bg, sd, nz.x);
      v.y = finalize_px(v.y * inv_scale, bg, sd, nz.y);
      v.z = finalize_px(v.z * inv_scale, bg, sd, nz.z);
      v.w = finalize_px(v.w * inv_scale, bg, sd, nz.w);
    } else {
      v.x = fminf(fmaxf(fmaf(v.x, inv_scale, bg), 0.f), 1.f);
      v.y = fminf(fmaxf(fmaf(v.y, inv_scale, bg), 0.f), 1.f);
      v.z = fminf(fmaxf(fmaf(v.z, inv_scale, bg), 0.f), 1.f);
      v.w = fminf(fmaxf(fmaf(v.w, inv_scale, bg), 0.f), 1.f);
    }
    if (OUT == kOutF32) {
      __stcs(reinterpret_cast<float4*>(dst), v);
    } else {
      ushort4 u = make_ushort4(quant_u16(v.x), quant_u16(v.y), quant_u16(v.z), quant_u16(v.w));
      __stcs(reinterpret_cast<ushort4*>(dst), u);
    }
  }
}

template <int OUT, bool NOISE>
__device__ void store_tile_vec(const FusedParams& P, const int* __restrict__ acc, int pl, int f,
                               int r0, int nr, int c0, int nc, float inv_scale) {
  constexpr int ESZ = OUT == kOutU16 ? 2 : 4;
  const uint32_t gpair = (uint32_t)(P.pair_base + pl);
  const int qpr = nc >> 2;
  char* outb = static_cast<char*>(P.out[f]) + (size_t)pl * (size_t)P.out_pair_elems * ESZ;
  if ((qpr & (qpr - 1)) == 0 && qpr <= kThreads) {
    // each thread owns one column quad and walks rows with constant pointer steps
    const int cq = threadIdx.x & (qpr - 1);
    const int row0 = threadIdx.x / qpr;
    const int rstep = kThreads / qpr;
    const int* ap = acc + (row0 + P.pad) * P.AS + P.pad + cq * 4;
    const int astep = rstep * P.AS;
    size_t pix = (size_t)(r0 + row0) * P.W + (size_t)(c0 + cq * 4);
    const size_t pstep = (size_t)rstep * P.W;
    for (int row = row0; row < nr; row += rstep, ap += astep, pix += pstep)
      store_quad<OUT, NOISE>(P, *reinterpret_cast<const int4*>(ap), outb + pix * ESZ, pix, f,
                             gpair, inv_scale);
  } else {
    const int total = nr * qpr;
    for (int e = threadIdx.x; e < total; e += kThreads) {
      const int row = e / qpr;
      const int c = e - row * qpr;
      const size_t pix = (size_t)(r0 + row) * P.W + (size_t)(c0 + c * 4);
      store_quad<OUT, NOISE>(P, *reinterpret_cast<const int4*>(acc + (row + P.pad) * P.AS + P.pad + c * 4),
                             outb + pix * ESZ, pix, f, gpair, inv_scale);
    }
  }
}

__device__ void store_tile(const FusedParams& P, const int* __restrict__ acc, int pl, int f,
                           int r0, int nr, int c0, int nc, float inv_scale) {
  const int AS = P.AS, pad = P.pad;
  const bool vec = ((nc & 3) == 0) && ((P.W & 3) == 0) && ((c0 & 3) == 0);
  const bool noise = P.noise_std > 0.f;
  if (vec) {
    switch (P.out_mode) {
      case kOutRaw: store_tile_vec<kOutRaw, false>(P, acc, pl, f, r0, nr, c0, nc, inv_scale); return;
      case kOutAccum: store_tile_vec<kOutAccum, false>(P, acc, pl, f, r0, nr, c0, nc, inv_scale); return;
      case kOutF32:
        if (noise) store_tile_vec<kOutF32, true>(P, acc, pl, f, r0, nr, c0, nc, inv_scale);
        else store_tile_vec<kOutF32, false>(P, acc, pl, f, r0, nr, c0, nc, inv_scale);
        return;
      default:
        if (noise) store_tile_vec<kOutU16, true>(P, acc, pl, f, r0, nr, c0, nc, inv_scale);
        else store_tile_vec<kOutU16, false>(P, acc, pl, f, r0, nr, c0, nc, inv_scale);
        return;
    }
  }
  const uint32_t gpair = (uint32_t)(P.pair_base + pl);
  const size_t pair_off = (size_t)pl * (size_t)P.out_pair_elems;
  const int mode = P.out_mode;
  const float bg = P.bg_offset, sd = P.noise_std;
  const int total = nr * nc;
  for (int e = threadIdx.x; e < total; e += kThreads) {
    const int row = e / nc;
    const int col = e - row * nc;
    float v = (float)acc[(row + pad) * AS + pad + col] * inv_scale;
    const size_t p = (size_t)(r0 + row) * P.W + (size_t)(c0 + col);
    if (mode == kOutRaw) {
      static_cast<float*>(P.out[f])[pair_off + p] = v;
    } else if (mode == kOutAccum) {
      static_cast<float*>(P.out[f])[pair_off + p] += v;
    } else {
      float nzv = 0.f;
      if (sd > 0.f) {
        const float4 nz = noise4(P.k0, P.k1, gpair, P.batch_lo, (uint32_t)f + 1, (uint32_t)(p >> 2));
        const int jn = (int)(p & 3);
        nzv = jn == 0 ? nz.x : (jn == 1 ? nz.y : (jn == 2 ? nz.z : nz.w));
      }
      v = finalize_px(v, bg, sd, nzv);
      if (mode == kOutF32) static_cast<float*>(P.out[f])[pair_off + p] = v;
      else static_cast<uint16_t*>(P.out[f])[pair_off + p] = quant_u16(v);
    }
  }
}

// ----------------------------------------------------------------------------
// Work items
// ----------------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void spin_until_geq(const int* p, int target) {
  int ns = 32;
  while (ld_acquire(p) < target) {
    __nanosleep(ns);
    ns = ns < 1024 ? ns * 2 : 1024;
  }
}

__device__ __forceinline__ void store_rec_global(Rec* dst, const Rec& r) {
  const float4* s4 = reinterpret_cast<const float4*>(&r);
  __stcg(reinterpret_cast<float4*>(dst), s4[0]);
  __stcg(reinterpret_cast<float4*>(dst) + 1, s4[1]);
}

// GENERATE (pair pl, chunk c): counting sort of the chunk's particles into
// its PRIVATE per-(frame, tile) segments of the pair's slot. Ranks come from
// shared-memory atomics only: no global round trips, no barriers per round.
__device__ void generate_item(const FusedParams& P, SharedHdr* sh, int* cnt, int pl, int c) {
  const int tid = threadIdx.x;
  const int slot = pl % P.ring;
  SlotHdr* S = P.slots + slot;
  const int T = P.tiles, G = P.chunks;
  const int nf = P.nframes;
  if (tid == 0) {
    // the slot is free once its previous occupant (pair pl - ring) is fully rendered
    spin_until_geq(&S->epoch, pl / P.ring);
    sh->amp = 0u;
    sh->wmax[0] = sh->wmax[1] = 0;
  }
  for (int e = tid; e < nf * T; e += kThreads) cnt[e] = 0;
  __syncthreads();
  Rec* recs = P.recs + (size_t)slot * nf * T * G * P.cap;
  const int i_lo = c * P.chunk;
  const int i_hi = min(P.n, i_lo + P.chunk);
  const int hx = P.halo;
  unsigned amp_l = 0u;
  int wmax_l[2] = {0, 0};
  for (int i = i_lo + tid; i < i_hi; i += kThreads) {
    Particle pt;
    inject_particle(P, pl, i, pt);
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      if (f >= nf) continue;
      const Frame& fr = pt.fr[f];
      if (!fr.on) continue;
      // tight window (anchor offsets), clipped to the config half-width hx
      const float R = record_radius(fr, P.psf);
      const int jlo = max(-hx, (int)ceilf(__fsub_rn(fr.fx, R)));
      const int jhi = min(hx, (int)floorf(__fadd_rn(fr.fx, R)));
      const int ilo = max(-hx, (int)ceilf(__fsub_rn(fr.fy, R)));
      const int ihi = min(hx, (int)floorf(__fadd_rn(fr.fy, R)));
      if (jlo > jhi || ilo > ihi) continue;
      const int rlo = max(fr.ay + ilo, P.row_lo), rhi = min(fr.ay + ihi, P.row_hi - 1);
      const int clo = max(fr.ax + jlo, 0), chi = min(fr.ax + jhi, P.W - 1);
      if (rlo > rhi || clo > chi) continue;
      const int ty0 = (rlo - P.row_lo) >> P.th_shift, ty1 = (rhi - P.row_lo) >> P.th_shift;
      const int tx0 = clo >> P.tw_shift, tx1 = chi >> P.tw_shift;
      Rec r = make_rec(fr, P.psf, jlo, ilo, jhi - jlo + 1, ihi - ilo + 1);
      amp_l = max(amp_l, __float_as_uint(fr.amp));
      wmax_l[f] = max(wmax_l[f], max(jhi - jlo, ihi - ilo) + 1);
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const int ty = ty0 + dy, tx = tx0 + dx;
          if (ty > ty1 || tx > tx1) continue;
          const int t = ty * P.tiles_x + tx;
          const int k = atomicAdd(&cnt[f * T + t], 1);
          // accumulator offset of the window's first pixel in tile (ty, tx)
          r.addr = (fr.ay + ilo - (P.row_lo + ty * P.TH - P.pad)) * P.AS +
                   (fr.ax + jlo - (tx * P.TW - P.pad));
          if (k < P.cap) store_rec_global(recs + (((size_t)f * T + t) * G + c) * P.cap + k, r);
          else atomicAdd(P.overflow, 1);
        }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    amp_l = max(amp_l, __shfl_xor_sync(~0u, amp_l, o));
    wmax_l[0] = max(wmax_l[0], __shfl_xor_sync(~0u, wmax_l[0], o));
    wmax_l[1] = max(wmax_l[1], __shfl_xor_sync(~0u, wmax_l[1], o));
  }
  if ((tid & 31) == 0) {
    atomicMax(&sh->amp, amp_l);
    atomicMax(&sh->wmax[0], wmax_l[0]);
    atomicMax(&sh->wmax[1], wmax_l[1]);
  }
  __syncthreads();
  int* counts = P.fills + (size_t)slot * nf * T * G;
  for (int e = tid; e < nf * T; e += kThreads) counts[(size_t)e * G + c] = min(cnt[e], P.cap);
  __syncthreads();
  if (tid == 0) {
    if (sh->amp) atomicMax(&S->amp, sh->amp);
    if (sh->wmax[0]) atomicMax(&S->wmax[0], sh->wmax[0]);
    if (sh->wmax[1]) atomicMax(&S->wmax[1], sh->wmax[1]);
    __threadfence();   // records + counts before the release
    atomicAdd(&S->gen_done, 1);
  }
}

// ----------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk) + mbarrier transaction counting
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1D bulk copy global -> shared, completion signalled on `bar` (complete_tx).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// RENDER (pair pl, tile t): both frames of one screen tile. The tile's
// record segments (one per generate chunk) are pulled into shared memory with
// TMA bulk copies (one elected thread, mbarrier transaction count), then
// splatted from shared memory.
template <int PSF>
__device__ void render_item(const FusedParams& P, SharedHdr* sh, int* acc, Rec* rbuf, int* cells,
                            int pl, int t, uint32_t& bar_phase) {
  const int tid = threadIdx.x;
  const int slot = pl % P.ring;
  SlotHdr* S = P.slots + slot;
  const int T = P.tiles, G = P.chunks;
  const int nf = P.nframes;
  const int* counts = P.fills + (size_t)slot * nf * T * G;
  const Rec* recs = P.recs + (size_t)slot * nf * T * G * P.cap;
  if (tid == 0) {
    spin_until_geq(&S->gen_done, G);
    // records per frame, then one transaction-counted barrier for all copies
    uint32_t bytes = 0;
    for (int f = 0; f < nf; ++f) {
      int K = 0;
      for (int c = 0; c < G; ++c) K += __ldcg(&counts[((size_t)f * T + t) * G + c]);
      sh->K[f] = K;
      if (K <= P.rbuf) bytes += (uint32_t)K * sizeof(Rec);
    }
    mbar_arrive_expect_tx(&sh->bar, bytes);
    // the buffer was last read through the generic proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int f = 0; f < nf; ++f) {
      if (sh->K[f] > P.rbuf) continue;
      int off = 0;
      for (int c = 0; c < G; ++c) {
        const int n = __ldcg(&counts[((size_t)f * T + t) * G + c]);
        if (n) {
          bulk_g2s(rbuf + (size_t)f * P.rbuf + off, recs + (((size_t)f * T + t) * G + c) * P.cap,
                   (uint32_t)n * sizeof(Rec), &sh->bar);
          off += n;
        }
      }
    }
  }
  __syncthreads();
  const int side = P.side_in[pl];
  const int ty = t / P.tiles_x, tx = t - (t / P.tiles_x) * P.tiles_x;
  const int r0 = P.row_lo + ty * P.TH;
  const int nr = min(P.TH, P.row_hi - r0);
  const int c0 = tx * P.TW;
  const int nc = min(P.TW, P.W - c0);
  const int h = side >> 1;
  const float amp_max = fmaxf(__uint_as_float(__ldcg(&S->amp)), 1e-30f);
  const int acc_ints = P.AH * P.AS;
  mbar_wait(&sh->bar, bar_phase);
  bar_phase ^= 1u;
  for (int f = 0; f < nf; ++f) {
    const int K = sh->K[f];
    const bool staged = K <= P.rbuf;
    const Rec* rl = rbuf + (size_t)f * P.rbuf;
    if (P.bin_counts && tid == 0) P.bin_counts[((size_t)pl * 2 + f) * T + t] = K;
    // -- fixed-point shift: per-pixel sum of rounded contributions < 2^31.
    //    Cheap bound from K; cell histogram only if it would cost precision
    //    (cells >= 2h+1 wide, so a pixel's anchor window lies in 2x2 cells).
    if (tid == 0) sh->shift = shift_for(max(K, 1), amp_max);
    __syncthreads();
    int shift = sh->shift;
    if (shift < kAccShift - 1) {
      // cells >= 2*hx+1 over the accumulator: a pixel's contributing window
      // starts lie in a 2x2 block of cells
      const int Sc = max(2 * P.halo + 1, kCellMin);
      const int ncy = (P.AH + Sc - 1) / Sc, ncx = (P.AS + Sc - 1) / Sc;
      if (ncy * ncx <= P.cells_cap) {
        if (tid == 0) sh->cov_max = 0;
        for (int e = tid; e < ncy * ncx; e += kThreads) cells[e] = 0;
        __syncthreads();
        for (int c = 0; c < G; ++c) {
          const int n = staged ? (c == 0 ? K : 0) : __ldcg(&counts[((size_t)f * T + t) * G + c]);
          const Rec* seg = staged ? rl : recs + (((size_t)f * T + t) * G + c) * P.cap;
          for (int k = tid; k < n; k += kThreads) {
            const int addr = staged ? seg[k].addr : __ldcg(&seg[k].addr);
            const int wr = addr / P.AS, wc = addr - (addr / P.AS) * P.AS;
            atomicAdd(&cells[(wr / Sc) * ncx + wc / Sc], 1);
          }
        }
        __syncthreads();
        int cm = 0;
        for (int e = tid; e < ncy * ncx; e += kThreads) {
          const int cy = e / ncx, cx = e - (e / ncx) * ncx;
          int sm = cells[e];
          if (cx + 1 < ncx) sm += cells[e + 1];
          if (cy + 1 < ncy) sm += cells[e + ncx];
          if (cx + 1 < ncx && cy + 1 < ncy) sm += cells[e + ncx + 1];
          cm = max(cm, sm);
        }
        for (int o = 16; o > 0; o >>= 1) cm = max(cm, __shfl_xor_sync(~0u, cm, o));
        if ((tid & 31) == 0) atomicMax(&sh->cov_max, cm);
        __syncthreads();
        if (tid == 0) sh->shift = shift_for(max(sh->cov_max, 1), amp_max);
        __syncthreads();
        shift = sh->shift;
      }
    }
    // lanes per record = widest tight window of the frame (exact skipping)
    const int W = max(1, min(2 * h + 1, __ldcg(&S->wmax[f])));
    if (staged) {
      splat_dispatch<PSF>(acc, rl, K, W, h, P.AS, (float)shift, exp2f((float)shift));
    } else {
      for (int c = 0; c < G; ++c)
        splat_dispatch<PSF>(acc, recs + (((size_t)f * T + t) * G + c) * P.cap,
                            __ldcg(&counts[((size_t)f * T + t) * G + c]), W, h, P.AS,
                            (float)shift, exp2f((float)shift));
    }
    __syncthreads();
    store_tile(P, acc, pl, f, r0, nr, c0, nc, exp2f(-(float)shift));
    __syncthreads();
    for (int e = tid; e < acc_ints >> 2; e += kThreads)
      reinterpret_cast<int4*>(acc)[e] = make_int4(0, 0, 0, 0);
    __syncthreads();
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&S->render_done, 1) == T - 1) {
      // last renderer retires the slot: reset it, then publish the new epoch
      S->gen_done = 0;
      S->render_done = 0;
      S->amp = 0u;
      S->wmax[0] = S->wmax[1] = 0;
      __threadfence();
      atomicAdd(&S->epoch, 1);
    }
  }
}

// ----------------------------------------------------------------------------
// The kernel: persistent CTAs pulling ordered tickets.
//   [gen items of pairs 0 .. L-1] then, per pair p: [render tiles of p][gen chunks of p + L]
// ----------------------------------------------------------------------------
template <int PSF>
__global__ void __launch_bounds__(kThreads, 4) inject_render_kernel(const FusedParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  int* acc = reinterpret_cast<int*>(smem);
  const int acc_ints = P.AH * P.AS;
  Rec* rbuf = reinterpret_cast<Rec*>(acc + acc_ints);                 // [nframes][rbuf]
  SharedHdr* sh = reinterpret_cast<SharedHdr*>(rbuf + (size_t)P.nframes * P.rbuf);
  int* cnt = reinterpret_cast<int*>(sh + 1);                          // [nframes * tiles]
  int* cells = cnt + P.nframes * P.tiles;                             // [cells_cap]
  const int tid = threadIdx.x;
  for (int e = tid; e < acc_ints >> 2; e += kThreads)
    reinterpret_cast<int4*>(acc)[e] = make_int4(0, 0, 0, 0);
  if (tid == 0) mbar_init(&sh->bar, 1);
  uint32_t bar_phase = 0;
  const int T = P.tiles, G = P.chunks, L = P.lookahead, NP = P.pairs;
  const long long pre = (long long)min(L, NP) * G;
  const long long total = pre + (long long)NP * (T + G);
  for (;;) {
    __syncthreads();
    if (tid == 0) sh->item = atomicAdd(P.ticket, 1);
    __syncthreads();
    const long long tk = sh->item;
    if (tk >= total) break;
    if (tk < pre) {
      generate_item(P, sh, cnt, (int)(tk / G), (int)(tk % G));
    } else {
      const long long u = tk - pre;
      const int p = (int)(u / (T + G));
      const int r = (int)(u - (long long)p * (T + G));
      if (r < T) {
        render_item<PSF>(P, sh, acc, rbuf, cells, p, r, bar_phase);
      } else if (p + L < NP) {
        generate_item(P, sh, cnt, p + L, r - T);
      }
    }
  }
}

}  // namespace pgb
