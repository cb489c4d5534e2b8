// common.cuh -- shared device helpers for the B200-native PIV generator.
//
// * Philox4x32-10 counter-based RNG (Salmon et al., SC'11), keyed by the
//   64-bit seed; counters carry (index, global pair, batch, stream tag), so
//   every draw is a pure function of (seed, batch, pair, purpose, index) --
//   the same determinism contract as the reference RNG (rng.py:1-9,
//   pipeline.py:8-11), with Philox replacing the splitmix64 mix.
// * Exact float64 arithmetic (no FMA contraction) for the parts that must be
//   bit-identical with the numpy reference: position sampling, advection
//   (flowfield.py:207-232) and the active-count / patch-side rules.
#pragma once
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

#ifndef PGB_HD
#define PGB_HD __host__ __device__ __forceinline__
#endif

namespace pgb {

// ----------------------------------------------------------------------------
// Philox4x32-10
// ----------------------------------------------------------------------------
constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

// Stream tags (counter word 3). Distinct tags = independent streams.
constexpr uint32_t kTagParticleA = 0x01;  // x, y, diameter, i0
constexpr uint32_t kTagParticleB = 0x02;  // rho, hide1, hide2, z
constexpr uint32_t kTagPerturb = 0x03;    // 4 normals for frame-2 jitter
constexpr uint32_t kTagPair = 0x04;       // per-pair seeding density
constexpr uint32_t kTagNoise = 0x10;      // + frame (1, 2): pixel noise
constexpr uint32_t kTagCell = 0x20;       // seeding-cell labels (stratified positions)

PGB_HD uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

PGB_HD uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = mulhi32(kPhiloxM0, c.x), lo0 = kPhiloxM0 * c.x;
    const uint32_t hi1 = mulhi32(kPhiloxM1, c.z), lo1 = kPhiloxM1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  return c;
}

// Device Philox with precomputed round keys (kernel parameters: each round's
// key is a constant-bank operand) and one 32x32->64 multiply per product.
struct PhiloxKeys {
  uint32_t k0[10], k1[10];
};

PGB_HD PhiloxKeys philox_keys(uint32_t k0, uint32_t k1) {
  PhiloxKeys K;
  for (int r = 0; r < 10; ++r) {
    K.k0[r] = k0;
    K.k1[r] = k1;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  return K;
}

__device__ __forceinline__ uint4 philox_rk(uint4 c, const PhiloxKeys& K) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)kPhiloxM0 * c.x;
    const uint64_t p1 = (uint64_t)kPhiloxM1 * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ K.k0[r], (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ K.k1[r],
                   (uint32_t)p0);
  }
  return c;
}

struct RngKey {
  uint32_t k0, k1;   // seed (lo, hi)
  uint32_t pair;     // global pair index within the batch
  uint32_t batch;    // batch index (low 32 bits)
};

PGB_HD uint4 draw(const RngKey& k, uint32_t index, uint32_t tag) {
  return philox4x32_10(make_uint4(index, k.pair, k.batch, tag), k.k0, k.k1);
}

// Open-interval uniform from one 32-bit word, exact in float64:
// u = (w + 0.5) * 2^-32  in (0, 1).
PGB_HD double u32_to_unit(uint32_t w) { return ((double)w + 0.5) * 0x1p-32; }

// 53-bit open-interval uniform from two words (mirrors rng.py:87-96 precision).
PGB_HD double u53_to_unit(uint32_t lo, uint32_t hi) {
  const uint64_t bits = (((uint64_t)hi << 32) | lo) >> 11;
  return ((double)bits + 0.5) * 0x1p-53;
}

// float32 open-interval uniform with 23-bit resolution (for Box-Muller);
// (2^23 - 1) + 0.5 is exact in float32, so the interval is truly open.
PGB_HD float u32_to_unitf(uint32_t w) { return ((float)(w >> 9) + 0.5f) * 0x1p-23f; }

// ----------------------------------------------------------------------------
// Exact float64 ops (no contraction) -- host fallbacks keep the code usable
// in host-side unit checks.
// ----------------------------------------------------------------------------
#ifdef __CUDA_ARCH__
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
#else
inline double dadd(double a, double b) { volatile double r = a + b; return r; }
inline double dsub(double a, double b) { volatile double r = a - b; return r; }
inline double dmul(double a, double b) { volatile double r = a * b; return r; }
inline double ddiv(double a, double b) { volatile double r = a / b; return r; }
#endif

// low + (high - low) * u   (rng.py:96)
PGB_HD double lerp_exact(double lo, double hi, double u) { return dadd(lo, dmul(dsub(hi, lo), u)); }

// Reproducible float64 log / exp: only correctly rounded +, -, *, / and exact
// scalings, so oracle/generate.py (plain Python floats) reproduces every bit.
// Accuracy ~1e-15 relative (they only draw the per-pair maximum diameter).
PGB_HD double rlog(double x) {
  int e = 0;
  double f = frexp(x, &e);                       // x = f 2^e, f in [1/2, 1)
  if (f < 0.70710678118654752) { f = dmul(f, 2.0); e -= 1; }
  const double s = ddiv(dsub(f, 1.0), dadd(f, 1.0));
  const double z = dmul(s, s);
  // 2 atanh(s) = 2 s sum z^k / (2k + 1); constants folded at compile time
  constexpr double kInvOdd[13] = {1.0, 1.0 / 3, 1.0 / 5, 1.0 / 7, 1.0 / 9, 1.0 / 11, 1.0 / 13,
                                  1.0 / 15, 1.0 / 17, 1.0 / 19, 1.0 / 21, 1.0 / 23, 1.0 / 25};
  double p = kInvOdd[12];
  for (int k = 11; k >= 0; --k) p = dadd(dmul(p, z), kInvOdd[k]);
  return dadd(dmul((double)e, 0.6931471805599453), dmul(2.0, dmul(s, p)));
}

PGB_HD double rexp(double y) {
  const double k = rint(dmul(y, 1.4426950408889634));
  const double r = dsub(y, dmul(k, 0.6931471805599453));
  constexpr double kInv[17] = {0.0, 1.0, 1.0 / 2, 1.0 / 3, 1.0 / 4, 1.0 / 5, 1.0 / 6, 1.0 / 7, 1.0 / 8,
                               1.0 / 9, 1.0 / 10, 1.0 / 11, 1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15,
                               1.0 / 16};
  double p = 1.0;
  for (int i = 16; i >= 1; --i) p = dadd(1.0, dmul(dmul(r, p), kInv[i]));
  return ldexp(p, (int)k);
}

// Smallest odd side >= ceil(round(mult * dmax + 1, 9)), at least 1 (raster.py:30-38).
PGB_HD int patch_side_exact(double dmax, double mult) {
  const double v = dadd(dmul(mult, dmax), 1.0);
  const double f = floor(v);
  // round(v, 9) followed by ceil(): values within 5e-10 above an integer
  // round down onto it; everything else ceils normally.
  double c = (v - f <= 5e-10) ? f : ceil(v);
  int side = (int)c;
  if ((side & 1) == 0) side += 1;
  return side < 1 ? 1 : side;
}

// Bilinear, edge-clamped sample of an interleaved (u, v) float32 grid,
// evaluated in float64 exactly as flowfield.sample_flow (flowfield.py:217-231).
PGB_HD void sample_flow_exact(const float2* __restrict__ flow, int H, int W, double px,
                              double py, double* u_out, double* v_out) {
  const double x = fmin(fmax(px, 0.0), (double)W - 1.0);
  const double y = fmin(fmax(py, 0.0), (double)H - 1.0);
  const double xmax = (double)(W - 2 > 0 ? W - 2 : 0);
  const double ymax = (double)(H - 2 > 0 ? H - 2 : 0);
  const int x0 = (int)fmin(fmax(floor(x), 0.0), xmax);
  const int y0 = (int)fmin(fmax(floor(y), 0.0), ymax);
  const int x1 = x0 + 1 < W - 1 ? x0 + 1 : W - 1;
  const int y1 = y0 + 1 < H - 1 ? y0 + 1 : H - 1;
  const double fx = dsub(x, (double)x0);
  const double fy = dsub(y, (double)y0);
  const double gx = dsub(1.0, fx), gy = dsub(1.0, fy);
#ifdef __CUDA_ARCH__
  const float2 a = __ldg(flow + (size_t)y0 * W + x0);
  const float2 b = __ldg(flow + (size_t)y0 * W + x1);
  const float2 c = __ldg(flow + (size_t)y1 * W + x0);
  const float2 d = __ldg(flow + (size_t)y1 * W + x1);
#else
  const float2 a = flow[(size_t)y0 * W + x0], b = flow[(size_t)y0 * W + x1];
  const float2 c = flow[(size_t)y1 * W + x0], d = flow[(size_t)y1 * W + x1];
#endif
  const double tu = dadd(dmul(gx, (double)a.x), dmul(fx, (double)b.x));
  const double bu = dadd(dmul(gx, (double)c.x), dmul(fx, (double)d.x));
  const double tv = dadd(dmul(gx, (double)a.y), dmul(fx, (double)b.y));
  const double bv = dadd(dmul(gx, (double)c.y), dmul(fx, (double)d.y));
  *u_out = dadd(dmul(gy, tu), dmul(fy, bu));
  *v_out = dadd(dmul(gy, tv), dmul(fy, bv));
}

// ----------------------------------------------------------------------------
// Box-Muller pair from two words (float32; distributional semantics only).
// ----------------------------------------------------------------------------
// Radius uniform u1 = f32((float)wa 2^-32 + 2^-33) in (0, 1] (32-bit resolution:
// the tail reaches sqrt(2 ln 2^33) = 6.76 sigma); angle uniform u2 =
// ((wb >> 9) + 1/2) 2^-23 built from its bits (exact). r = sqrt(-2 ln 2 lg2 u1)
// with MUFU lg2/sqrt, no slow-path branch. ~14 instructions per normal pair.
__device__ __forceinline__ float2 box_muller(uint32_t wa, uint32_t wb) {
  const float u1 = fmaf((float)wa, 0x1p-32f, 0x1p-33f);
  const float u2 = __fadd_rn(__uint_as_float((wb >> 9) | 0x3f800000u), -0.99999994f);
  float l, r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(u1));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(l * -1.3862943611198906f));
  float s, c;
  __sincosf(6.28318530717958647692f * u2, &s, &c);
  return make_float2(r * c, r * s);
}

}  // namespace pgb
