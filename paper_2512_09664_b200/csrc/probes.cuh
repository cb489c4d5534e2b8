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

}  // namespace pgb
