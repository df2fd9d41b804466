// Shared device-side definitions of the sweep engine.
//
// Arithmetic contract: every kernel evaluates the reference's expressions in the reference's
// operand order with no FMA contraction (the library is built with -fmad=false), so pointwise
// results are bit-identical to the CPU oracle / the reference's no-FMA x86-64 build.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cisdc_gpu.h"

namespace cisdc_b200 {

constexpr int kMaxM = CISDC_MAX_M;
constexpr int kMaxS = CISDC_MAX_SPECIES;
constexpr int kMaxR = CISDC_MAX_REACTIONS;

// Device status word, one per context (written by kernels, read once per sweep).
struct DevStatus {
  unsigned long long first_bad_cell;  // smallest failing cell index (atomicMin), ~0ull if none
  int code;                           // CISDC_E_* of the first recorded failure kind
  int stage;                          // CISDC_STAGE_* of the failure
  unsigned long long newton_trips;    // Newton residual evaluations (atomicAdd)
  unsigned long long mg_cycles;       // multigrid V-cycles
  double incr_partial_unused;
};

// Grid geometry of one field (species-major, x fastest).
struct Geom {
  int nx, ny, nz;  // cells per axis (1 for unused axes)
  int ndim;
  int S;
  long long ncell;  // nx * ny * nz
  long long n;      // S * ncell
};

// Separable face-velocity tables and stencil coefficients (problem constants).
struct Ops {
  const double* vel[3][3];  // nullptr = 1.0
  int adv[3];               // axis a advects
  double cadv[3];           // 1 / (12 h_a)
  double cdiff[kMaxS][3];   // d_s / (12 h_a^2)
  // reference Dirichlet problem (CISDC_PROBLEM_REFERENCE_RD)
  int ref_rd;
  double rd_cadv, rd_cdiff, rd_w[2][5];
};

__device__ __forceinline__ int wrapi(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

__device__ __forceinline__ double face_u(const Ops& o, int a, int i, int j, int k) {
  const double t0 = o.vel[a][0] ? __ldg(o.vel[a][0] + i) : 1.0;
  const double t1 = o.vel[a][1] ? __ldg(o.vel[a][1] + j) : 1.0;
  const double t2 = o.vel[a][2] ? __ldg(o.vel[a][2] + k) : 1.0;
  return (t0 * t1) * t2;
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr), __double_as_longlong(v));
}

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace cisdc_b200
