// probes.cuh -- microbenchmarks for the roofline denominators that
// MEASURED_PEAKS.json does not carry: MUFU.EX2 issue rate (the SFU roofline of
// the Gaussian splat).
#pragma once
#include <cstdint>

namespace pgb {

// 8 independent ex2.approx chains per thread: x <- -ex2(x) stays in [-1, -1/2]
// (the negation folds into the MUFU operand), so the loop body is 8 MUFU.EX2.
__global__ void __launch_bounds__(256) ex2_probe_kernel(float* sink, int iters) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = -0.5f - 0.0625f * (float)k - 1e-6f * (float)threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(-x[k]));
      x[k] = -y;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 123.f) sink[threadIdx.x] = s;   // never true; keeps the chains live
}

#ifdef PGB_TRACE
// Shared-atomic issue rate by address pattern (debug builds): mode 0 lanes in
// consecutive words (distinct banks), 1 stride 2 words, 2 stride 32 words (one
// bank), 3 hashed addresses, 4 consecutive words with per-warp offsets
// (k * 37 words: the sorted-splat round pattern).
__global__ void __launch_bounds__(256) atoms_probe_kernel(int* sink, int iters, int mode) {
  __shared__ int a[8192];
  for (int i = threadIdx.x; i < 8192; i += 256) a[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int off;
  switch (mode) {
    case 0: off = warp * 512 + lane; break;
    case 1: off = warp * 512 + 2 * lane; break;
    case 2: off = warp * 8 + 32 * lane; break;
    case 3: off = (int)((((unsigned)threadIdx.x * 2654435761u) >> 7) & 4095u); break;
    default: off = warp * 512 + ((lane * 37) & 511); break;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) atomicAdd(&a[(off + k * 256) & 8191], 1);
  }
  __syncthreads();
  if (a[threadIdx.x] == 123456789) sink[threadIdx.x] = 1;
}
#endif

}  // namespace pgb
