// refrng.cuh -- reference-RNG mode: the reference's
// splitmix64 counter streams (rng.py:33-106) and its particle sampling
// (particles.py:61-147) restated on the GPU, so that a batch is generated
// end to end with the reference's own random numbers (no oracle injection).
//
//   key(seed; stream, batch, pair, lane) = fold(...fold(seed, stream)..., lane),
//     fold(k, w) = mix64(k ^ mix64(w + phi))                       (rng.py:41-44)
//   word_i = mix64(base + (i + 1) phi)   (uint64 wrap)            (rng.py:81-85)
//   U_i    = lo + (hi - lo) ((word_i >> 11) + 1/2) 2^-53           (rng.py:87-96)
//   N_i    = std * ndtri(U_i)                                      (rng.py:98-101)
//
// Uniform-derived quantities (positions, density, M, I0, diameters, sigma,
// rho, hiding, advection) are bit-identical to the reference (float64 ops in
// the reference's order, no contraction). Normals use CUDA's normcdfinv in
// place of scipy's ndtri (agree to a few ulp of float64), so frame-2 jitter
// and pixel noise match to ~1e-15 relative before the float32 rounding.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace pgb {

constexpr uint64_t kSmGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kSmMixA = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kSmMixB = 0x94D049BB133111EBull;
enum { kSmPosition = 1, kSmAppearance = 2, kSmPerturb = 3, kSmHide = 4, kSmNoise = 5 };

__host__ __device__ __forceinline__ uint64_t sm_mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * kSmMixA;
  x = (x ^ (x >> 27)) * kSmMixB;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t sm_key(uint64_t seed, uint64_t stream, uint64_t batch, uint64_t pair,
                                                    uint64_t lane) {
  uint64_t k = seed;
  const uint64_t w[4] = {stream, batch, pair, lane};
  for (int i = 0; i < 4; ++i) k = sm_mix64(k ^ sm_mix64(w[i] + kSmGolden));
  return k;
}

// Counter index i (0-based, offset included): U on (lo, hi).
__device__ __forceinline__ double sm_uniform(uint64_t base, uint64_t i, double lo, double hi) {
  const uint64_t w = sm_mix64(base + (i + 1) * kSmGolden);
  const double u = ((double)(w >> 11) + 0.5) * 0x1p-53;
  return dadd(lo, dmul(dsub(hi, lo), u));
}

__device__ __forceinline__ double sm_normal(uint64_t base, uint64_t i, double std_) {
  return dmul(std_, normcdfinv(sm_uniform(base, i, 0.0, 1.0)));
}

struct SmParams {
  int H, W, n, pairs;
  uint64_t seed, batch;
  long long pair_base;
  double ppp_lo, ppp_hi, d_lo, d_hi, i0_lo, i0_hi, rho_lo, rho_hi, ratio, mult;
  double s_std, i_std, r_std, hide_p;
  const float2* flows;
  long long field_elems;
  int pairs_per_field;
};

// One thread per particle slot of one pair (blockIdx.y = pair).
__global__ void sm_particles_kernel(const SmParams S, pgb_particle_out O, double* st_ppp, int* st_M,
                                    unsigned* st_dmax_bits) {
  const int pl = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S.n) return;
  const uint64_t gp = (uint64_t)(S.pair_base + pl);
  // sample_particles (particles.py:61-101)
  const uint64_t kpos = sm_key(S.seed, kSmPosition, S.batch, gp, 0);
  const double x = dmul(sm_uniform(kpos, (uint64_t)i, 0.0, 1.0), (double)S.W);
  const double y = dmul(sm_uniform(kpos, (uint64_t)(S.n + i), 0.0, 1.0), (double)S.H);
  const double ppp = sm_uniform(sm_key(S.seed, kSmAppearance, S.batch, gp, 0), 0, S.ppp_lo, S.ppp_hi);
  double mm = rint(dmul(dmul(ppp, (double)S.H), (double)S.W));
  mm = fmin(fmax(mm, 0.0), (double)S.n);
  const int M = (int)mm;
  const bool active = i < M;
  const double i0 = sm_uniform(sm_key(S.seed, kSmAppearance, S.batch, gp, 1), (uint64_t)i, S.i0_lo, S.i0_hi);
  const double diam = sm_uniform(sm_key(S.seed, kSmAppearance, S.batch, gp, 2), (uint64_t)i, S.d_lo, S.d_hi);
  const double rho = sm_uniform(sm_key(S.seed, kSmAppearance, S.batch, gp, 3), (uint64_t)i, S.rho_lo, S.rho_hi);
  const float i0f = active ? (float)i0 : 0.0f;
  const float sig = (float)ddiv(diam, S.ratio);
  const float rhof = (float)rho;
  const float df = (float)diam;
  // perturb_frame2 (particles.py:104-126): float32 + float64 jitter in float64
  float sx2 = sig, sy2 = sig, i02 = i0f, rho2 = rhof;
  if (S.s_std > 0.0) {
    const uint64_t k1 = sm_key(S.seed, kSmPerturb, S.batch, gp, 1), k2 = sm_key(S.seed, kSmPerturb, S.batch, gp, 2);
    sx2 = (float)fmax(dadd((double)sig, sm_normal(k1, (uint64_t)i, S.s_std)), 1e-3);
    sy2 = (float)fmax(dadd((double)sig, sm_normal(k2, (uint64_t)i, S.s_std)), 1e-3);
  }
  if (S.i_std > 0.0) {
    const uint64_t k3 = sm_key(S.seed, kSmPerturb, S.batch, gp, 3);
    const double t = fmin(fmax(dadd((double)i0f, sm_normal(k3, (uint64_t)i, S.i_std)), 0.0), 1.0);
    i02 = i0f == 0.0f ? 0.0f : (float)t;
  }
  if (S.r_std > 0.0) {
    const uint64_t k4 = sm_key(S.seed, kSmPerturb, S.batch, gp, 4);
    const double lim = 1.0 - 1e-3;
    rho2 = (float)fmin(fmax(dadd((double)rhof, sm_normal(k4, (uint64_t)i, S.r_std)), -lim), lim);
  }
  // apply_hiding (particles.py:139-147)
  const bool vis1 = sm_uniform(sm_key(S.seed, kSmHide, S.batch, gp, 1), (uint64_t)i, 0.0, 1.0) >= S.hide_p;
  const bool vis2 = sm_uniform(sm_key(S.seed, kSmHide, S.batch, gp, 2), (uint64_t)i, 0.0, 1.0) >= S.hide_p;
  // advect (particles.py:129-136): float64 bilinear, edge-clamped
  const float2* flow = S.flows + (size_t)((S.pair_base + pl) / S.pairs_per_field) * (size_t)S.field_elems;
  double u, v;
  sample_flow_exact(flow, S.H, S.W, x, y, &u, &v);
  const size_t o = (size_t)pl * S.n + i;
  if (O.pos1) { O.pos1[2 * o] = x; O.pos1[2 * o + 1] = y; }
  if (O.pos2) { O.pos2[2 * o] = dadd(x, u); O.pos2[2 * o + 1] = dadd(y, v); }
  if (O.i0_1) O.i0_1[o] = i0f;
  if (O.sx_1) O.sx_1[o] = sig;
  if (O.sy_1) O.sy_1[o] = sig;
  if (O.rho_1) O.rho_1[o] = rhof;
  if (O.i0_2) O.i0_2[o] = i02;
  if (O.sx_2) O.sx_2[o] = sx2;
  if (O.sy_2) O.sy_2[o] = sy2;
  if (O.rho_2) O.rho_2[o] = rho2;
  if (O.diameter) O.diameter[o] = df;
  if (O.z1) O.z1[o] = 0.0f;
  if (O.active) O.active[o] = active ? 1 : 0;
  if (O.visible1) O.visible1[o] = (vis1 && active) ? 1 : 0;
  if (O.visible2) O.visible2[o] = (vis2 && active) ? 1 : 0;
  if (active && st_dmax_bits) atomicMax(st_dmax_bits + pl, __float_as_uint(df));
  if (i == 0) {
    if (st_ppp) st_ppp[pl] = ppp;
    if (st_M) st_M[pl] = M;
  }
}

// Per pair: the patch side from the maximum active diameter (pipeline.py:291-294).
__global__ void sm_side_kernel(const SmParams S, const int* st_M, unsigned* st_dmax_bits, int* st_side) {
  const int pl = blockIdx.x * blockDim.x + threadIdx.x;
  if (pl >= S.pairs) return;
  double dmax = S.d_hi;   // no active particle: diameter_range[1]
  if (st_M[pl] > 0) dmax = (double)__uint_as_float(st_dmax_bits[pl]);
  else st_dmax_bits[pl] = __float_as_uint((float)S.d_hi);
  st_side[pl] = patch_side_exact(dmax, S.mult);
}

// finalize (raster.py:154-161) with the reference noise stream (NOISE, lane = frame).
__global__ void sm_finalize_kernel(const float* __restrict__ raw, float* out, long long pixels, int images,
                                   double bg, double std_, uint64_t seed, uint64_t batch, long long pair_base,
                                   int frame) {
  const int img = blockIdx.y;
  const uint64_t base = sm_key(seed, kSmNoise, batch, (uint64_t)(pair_base + img), (uint64_t)frame);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < pixels;
       p += (long long)gridDim.x * blockDim.x) {
    const size_t o = (size_t)img * (size_t)pixels + (size_t)p;
    double x = (double)raw[o];
    if (bg != 0.0) x = dadd(x, bg);
    if (std_ > 0.0) x = dadd(x, sm_normal(base, (uint64_t)p, std_));
    out[o] = (float)fmin(fmax(x, 0.0), 1.0);
  }
}

}  // namespace pgb
