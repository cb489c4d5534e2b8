// wide.cuh -- oracle-mode renders without a shared-memory tile plan.
//
// * wide_splat_kernel: the reference splat (_native.pyx:14-66) for patch sides
//   too large for the tiled inject kernel (fused.cuh: a window must fit 2x2
//   shared-memory tiles). One warp per particle, lanes over the window
//   columns, the reference's float64 arithmetic per pixel, contributions
//   rounded to 2^-32 and summed with 64-bit integer atomics: exact,
//   order-independent, no side limit.
// * oracle_render_kernel: render_oracle (raster.py:129-151), the untruncated
//   O(N H W) float64 sum; one thread per pixel, particles staged through
//   shared memory in chunks.
#pragma once
#include "common.cuh"
#include "fused.cuh"

namespace pgb {

constexpr double kWideScale = 4294967296.0;   // 2^32 fixed point

struct WideParams {
  int H, W, row_lo, row_hi;
  long long n;                 // particles per pair
  int pl;                      // pair (offset into the [pairs][n] arrays)
  int side;
  int psf;
  InjFrame fr;
  unsigned long long* acc;     // [H][W], rows [row_lo, row_hi) used
};

__device__ __forceinline__ double wide_value(int psf, double amp, double sx, double sy, double rr, double dx,
                                             double dy) {
  if (psf == kPsfPoint) {
    // _native.pyx:54-66 (float64)
    const double q = 1.0 - rr * rr;
    const double a = 1.0 / (2.0 * q * sx * sx);
    const double b = rr / (q * sx * sy);
    const double cc = 1.0 / (2.0 * q * sy * sy);
    return amp * exp(-(a * dx * dx - b * dx * dy + cc * dy * dy));
  }
  // pixel-area mean of Eq. (1) over [dx - 1/2, dx + 1/2] x [dy - 1/2, dy + 1/2]
  // (oracle/render.py render_erf): separable for rho == 0, else x | y is
  // Gaussian with mean rho sx / sy y and sd sx sqrt(1 - rho^2); 8-point
  // Gauss-Legendre in y.
  const double k = 1.2533141373155001;   // sqrt(pi / 2)
  const double r2 = 0.70710678118654752;
  if (rr == 0.0) {
    const double ex = erf((dx + 0.5) * r2 / sx) - erf((dx - 0.5) * r2 / sx);
    const double ey = erf((dy + 0.5) * r2 / sy) - erf((dy - 0.5) * r2 / sy);
    return amp * (k * sx) * (k * sy) * ex * ey;
  }
  const double sc = sx * sqrt(fmax(1.0 - rr * rr, 0.0));
  const double kx[8] = {-0.48014492824876809, -0.39833323870681336, -0.2627662049581645, -0.09171732124782489,
                        0.091717321247824893, 0.2627662049581645, 0.39833323870681336, 0.48014492824876809};
  const double kw[8] = {0.050614268145188532, 0.11119051722668721, 0.15685332293894344, 0.18134189168918083,
                        0.18134189168918083, 0.15685332293894344, 0.11119051722668721, 0.050614268145188532};
  double s = 0.0;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const double yy = dy + kx[g];
    const double mu = rr * sx / sy * yy;
    const double gy = exp(-yy * yy / (2.0 * sy * sy));
    s += kw[g] * gy * (erf((dx + 0.5 - mu) * r2 / sc) - erf((dx - 0.5 - mu) * r2 / sc));
  }
  return amp * (k * sc) * s;
}

// One warp per particle: the window [a - h, a + h] clipped to the band and the
// image (_native.pyx:31-49), lanes over columns, rows in a loop.
__global__ void __launch_bounds__(256) wide_splat_kernel(const WideParams P) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int h = P.side >> 1;
  for (long long i = warp; i < P.n; i += nwarps) {
    const size_t o = (size_t)P.pl * P.n + i;
    if (!P.fr.mask[o]) continue;
    const double x = P.fr.pos[2 * o], y = P.fr.pos[2 * o + 1];
    const double fxa = floor(x + 0.5), fya = floor(y + 0.5);
    if (!(fabs(fxa) < 1e8 && fabs(fya) < 1e8)) continue;
    const long long ax = (long long)fxa, ay = (long long)fya;
    const long long r0 = max(ay - h, (long long)P.row_lo), r1 = min(ay + h, (long long)P.row_hi - 1);
    const long long c0 = max(ax - h, 0ll), c1 = min(ax + h, (long long)P.W - 1);
    if (r0 > r1 || c0 > c1) continue;
    const double amp = P.fr.i0[o], sx = P.fr.sx[o], sy = P.fr.sy[o], rr = P.fr.rho[o];
    const int nc = (int)(c1 - c0 + 1);
    for (long long r = r0; r <= r1; ++r) {
      const double dy = (double)r - y;
      unsigned long long* row = P.acc + (size_t)r * P.W;
      for (int j = lane; j < nc; j += 32) {
        const long long c = c0 + j;
        const double v = wide_value(P.psf, amp, sx, sy, rr, (double)c - x, dy);
        const unsigned long long q = (unsigned long long)llrint(v * kWideScale);
        if (q) atomicAdd(row + c, q);
      }
    }
  }
}

// Fixed-point rows [row_lo, row_hi) -> the caller's image, every out mode of
// the tiled kernel (raw, += accumulate, finalize to float32 / uint16 with the
// same Philox noise keyed by the row-major pixel quad).
__global__ void wide_store_kernel(const unsigned long long* __restrict__ acc, int H, int W, int row_lo,
                                  int row_hi, int out_mode, float bg, float sd, uint32_t k0, uint32_t k1,
                                  uint32_t gpair, uint32_t batch, int frame, void* out) {
  const long long p0 = (long long)row_lo * W, p1 = (long long)row_hi * W;
  const long long q0 = p0 >> 2, q1 = (p1 + 3) >> 2;
  for (long long q = q0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < q1;
       q += (long long)gridDim.x * blockDim.x) {
    float4 nz = make_float4(0.f, 0.f, 0.f, 0.f);
    if ((out_mode == kOutF32 || out_mode == kOutU16) && sd > 0.f)
      nz = noise4(k0, k1, gpair, batch, (uint32_t)frame, (uint32_t)q);
    const float nzs[4] = {nz.x, nz.y, nz.z, nz.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long p = 4 * q + j;
      if (p < p0 || p >= p1) continue;
      const float v = (float)((double)acc[p] * (1.0 / kWideScale));
      if (out_mode == kOutRaw) {
        static_cast<float*>(out)[p] = v;
      } else if (out_mode == kOutAccum) {
        static_cast<float*>(out)[p] += v;
      } else {
        const float f = finalize_px(v, bg, sd, nzs[j]);
        if (out_mode == kOutF32) static_cast<float*>(out)[p] = f;
        else static_cast<uint16_t*>(out)[p] = quant_u16(f);
      }
    }
  }
}

// render_oracle (raster.py:129-151): every masked particle at every pixel,
// float64, no truncation, summed in particle-index order (masked particles
// add an exact 0). 16 x 16 pixel blocks; particles staged in chunks.
constexpr int kOracleChunk = 256;

__global__ void __launch_bounds__(256) oracle_render_kernel(const double* __restrict__ pos,
                                                            const float* __restrict__ i0,
                                                            const float* __restrict__ sxa,
                                                            const float* __restrict__ sya,
                                                            const float* __restrict__ rhoa,
                                                            const uint8_t* __restrict__ mask, long long n,
                                                            int H, int W, float* __restrict__ out) {
  __shared__ double sp[kOracleChunk][6];
  const int c = blockIdx.x * 16 + (threadIdx.x & 15);
  const int r = blockIdx.y * 16 + (threadIdx.x >> 4);
  double acc = 0.0;
  for (long long base = 0; base < n; base += kOracleChunk) {
    const long long i = base + threadIdx.x;
    if (i < n) {
      sp[threadIdx.x][0] = pos[2 * i];
      sp[threadIdx.x][1] = pos[2 * i + 1];
      sp[threadIdx.x][2] = sxa[i];
      sp[threadIdx.x][3] = sya[i];
      sp[threadIdx.x][4] = rhoa[i];
      sp[threadIdx.x][5] = mask[i] ? (double)i0[i] : 0.0;
    }
    __syncthreads();
    const int kn = (int)min((long long)kOracleChunk, n - base);
    for (int k = 0; k < kn; ++k) {
      const double amp = sp[k][5];
      if (amp == 0.0) continue;
      const double dx = (double)c - sp[k][0];
      const double dy = (double)r - sp[k][1];
      const double sx = sp[k][2], sy = sp[k][3], rr = sp[k][4];
      const double q = 1.0 - rr * rr;
      const double expo = (__dmul_rn(dx, dx) / __dmul_rn(sx, sx) -
                           __dmul_rn(__dmul_rn(__dmul_rn(2.0, rr), dy), dx) / __dmul_rn(sx, sy) +
                           __dmul_rn(dy, dy) / __dmul_rn(sy, sy)) / (2.0 * q);
      acc = __dadd_rn(acc, __dmul_rn(amp, exp(-expo)));
    }
    __syncthreads();
  }
  if (r < H && c < W) out[(size_t)r * W + c] = (float)acc;
}

}  // namespace pgb
