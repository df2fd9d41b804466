// FP64 pipe peak probe (the FP64 roofline denominator: MEASURED_PEAKS.json has no FP64 entry).
// 8 independent dependency chains per thread, grid = 8 x 148 SMs x 256 threads; DFMA chains via
// explicit __fma_rn (the library is built with -fmad=false), and DMUL+DADD chains for the
// no-contraction arithmetic the parity build actually executes.
#pragma once

#include "common.cuh"

namespace cisdc_b200 {

__global__ void __launch_bounds__(256) k_peak_dfma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __fma_rn(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) k_peak_dmul_dadd(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

}  // namespace cisdc_b200
