// histmatch.cuh -- histogram specification on 256 levels, one CTA per image
// (reference raster.py:164-187 match_histogram).
//
//   level(x)  = clip(rint(f32(x * 255)), 0, 255)            (float32, half-even)
//   q[L]      = (cum[L] - counts[L] / 2) / total            (float64, exact ints)
//   map[L]    = first i with target_cdf[i] >= q[L]          (searchsorted 'left')
//   out(x)    = f32(map[level(x)] / 255.0)                  (float64 division)
//
// target_cdf = cumsum(hist) / sum(hist) is computed on the host exactly as
// numpy does (sequential float64 sums) and passed in (256 doubles). Every
// step is exact or correctly rounded in the same order as the reference, so
// the output is bit-identical to it.
//
// Per image: one read pass (per-warp shared histograms, merged), a 256-entry
// LUT (one thread per level; 9-step binary search over the CDF in shared
// memory), one read + write pass applying the LUT with 128-bit accesses.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pgb {

constexpr int kHistThreads = 512;
constexpr int kHistWarps = kHistThreads / 32;

__device__ __forceinline__ int hist_level(float x) {
  const float y = rintf(__fmul_rn(x, 255.0f));
  return (int)fminf(fmaxf(y, 0.0f), 255.0f);   // NaN -> 0 (fmaxf)
}

__global__ void __launch_bounds__(kHistThreads) hist_match_kernel(const float* __restrict__ in, float* out,
                                                                  long long pixels,
                                                                  const double* __restrict__ target_cdf) {
  __shared__ int wh[kHistWarps][256];   // per-warp histograms
  __shared__ double cdf[256];
  __shared__ float lut[256];
  const int tid = threadIdx.x, warp = tid >> 5;
  const float* src = in + (size_t)blockIdx.x * (size_t)pixels;
  float* dst = out + (size_t)blockIdx.x * (size_t)pixels;
  for (int i = tid; i < kHistWarps * 256; i += kHistThreads) (&wh[0][0])[i] = 0;
  if (tid < 256) cdf[tid] = target_cdf[tid];
  __syncthreads();
  const bool vec = (pixels & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  if (vec) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    for (long long q = tid; q < pixels / 4; q += kHistThreads) {
      const float4 v = __ldg(s4 + q);
      atomicAdd(&wh[warp][hist_level(v.x)], 1);
      atomicAdd(&wh[warp][hist_level(v.y)], 1);
      atomicAdd(&wh[warp][hist_level(v.z)], 1);
      atomicAdd(&wh[warp][hist_level(v.w)], 1);
    }
  } else {
    for (long long p = tid; p < pixels; p += kHistThreads) atomicAdd(&wh[warp][hist_level(__ldg(src + p))], 1);
  }
  __syncthreads();
  if (tid < 256) {
    int c = 0;
#pragma unroll
    for (int w = 0; w < kHistWarps; ++w) c += wh[w][tid];
    wh[0][tid] = c;   // merged counts (row 0 is only read back by this thread)
  }
  __syncthreads();
  __shared__ int wtot[8];
  int cnt = 0, cum = 0;
  if (tid < 256) {
    // inclusive cumulative count up to level tid (exact integers): warp scans
    cnt = wh[0][tid];
    cum = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(~0u, cum, o);
      if ((tid & 31) >= o) cum += y;
    }
    if ((tid & 31) == 31) wtot[warp] = cum;
  }
  __syncthreads();
  if (tid < 256) {
    for (int w = 0; w < warp; ++w) cum += wtot[w];
    const double q = __ddiv_rn(__dsub_rn((double)cum, __dmul_rn(0.5, (double)cnt)), (double)pixels);
    // searchsorted(side='left'): first i with cdf[i] >= q (256 if none, clipped to 255)
    int lo = 0, hi = 256;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cdf[mid] < q) lo = mid + 1;
      else hi = mid;
    }
    const int m = lo < 255 ? lo : 255;
    lut[tid] = (float)__ddiv_rn((double)m, 255.0);
  }
  __syncthreads();
  if (vec && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (long long q = tid; q < pixels / 4; q += kHistThreads) {
      const float4 v = s4[q];   // plain load: in may alias out
      d4[q] = make_float4(lut[hist_level(v.x)], lut[hist_level(v.y)], lut[hist_level(v.z)], lut[hist_level(v.w)]);
    }
  } else {
    for (long long p = tid; p < pixels; p += kHistThreads) dst[p] = lut[hist_level(src[p])];
  }
}

}  // namespace pgb
