// K1: operator evaluations F_A, F_D, F_R (OperatorSplitProblem::eval_*).
//
// Periodic ADR problem (configs 1-5): 4th-order finite-volume advection flux form and the
// reference's 4th-order Laplacian stencil (proj/core/src/problems/reaction_diffusion.cpp:84,97)
// per axis with periodic wrap.  Reference Dirichlet problem (config-0 gate): the same stencils
// with the quartic ghost fill of reaction_diffusion.cpp:58-67.
//
// One thread per field element; neighbours come through the read-only/L1 path (the 5-point
// star along each axis re-reads each value 1 + 4*ndim times, which L1/L2 absorb: the kernels
// are HBM-bound on the compulsory read of phi and the writes of F_A, F_D).
#pragma once

#include "common.cuh"

namespace cisdc_b200 {

// value at (i,j,k) displaced by o along axis a (periodic), species plane f
__device__ __forceinline__ double at_off(const double* __restrict__ f, const Geom& g, int i, int j, int k, int a,
                                         int o) {
  if (a == 0) i = wrapi(i + o, g.nx);
  else if (a == 1) j = wrapi(j + o, g.ny);
  else k = wrapi(k + o, g.nz);
  return __ldg(f + ((long long)k * g.ny + j) * g.nx + i);
}

// The reference's stencil -g0 + 16 g1 - 30 g2 + 16 g3 - g4 (reaction_diffusion.cpp:97), evaluated left
// to right.  16 g is exact (a power of two; |g| < 2^1019), so round(16 g1 + (-g0)) is one fused
// multiply-add, and likewise the + 16 g3 term: the same bits with 5 FP64 operations instead of 7.
__device__ __forceinline__ double lap5(double g0, double g1, double g2, double g3, double g4) {
  return __fma_rn(16.0, g3, __fma_rn(16.0, g1, -g0) - 30.0 * g2) - g4;
}

template <int DIM>
__device__ __forceinline__ double adv_periodic(const Ops& o, const Geom& g, const double* __restrict__ f, int i,
                                               int j, int k) {
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    if (!o.adv[a]) continue;
    const double v0 = at_off(f, g, i, j, k, a, -2), v1 = at_off(f, g, i, j, k, a, -1);
    const double v2 = at_off(f, g, i, j, k, a, 0), v3 = at_off(f, g, i, j, k, a, 1);
    const double v4 = at_off(f, g, i, j, k, a, 2);
    const int ia = a == 0 ? wrapi(i - 1, g.nx) : i;
    const int ja = a == 1 ? wrapi(j - 1, g.ny) : j;
    const int ka = a == 2 ? wrapi(k - 1, g.nz) : k;
    const double fr = face_u(o, a, i, j, k) * (7.0 * (v2 + v3) - (v1 + v4));
    const double fl = face_u(o, a, ia, ja, ka) * (7.0 * (v1 + v2) - (v0 + v3));
    acc = acc + (fr - fl) * o.cadv[a];
  }
  return -acc;
}

template <int DIM>
__device__ __forceinline__ double diff_periodic(const Ops& o, const Geom& g, const double* __restrict__ f, int s,
                                                int i, int j, int k) {
  double lap = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const double v0 = at_off(f, g, i, j, k, a, -2), v1 = at_off(f, g, i, j, k, a, -1);
    const double v2 = at_off(f, g, i, j, k, a, 0), v3 = at_off(f, g, i, j, k, a, 1);
    const double v4 = at_off(f, g, i, j, k, a, 2);
    lap = lap + o.cdiff[s][a] * lap5(v0, v1, v2, v3, v4);
  }
  return lap;
}

// ghost-extended value ext[i + 2] of the reference Dirichlet grid (fill_ghosts, :58-67)
__device__ __forceinline__ double rd_ext(const Ops& o, const double* __restrict__ f, int n, int e /* -2..n+1 */) {
  if (e >= 0 && e < n) return __ldg(f + e);
  if (e < 0) {
    const double* w = o.rd_w[-e - 1];
    return w[0] * 1.0 + w[1] * __ldg(f + 0) + w[2] * __ldg(f + 1) + w[3] * __ldg(f + 2) + w[4] * __ldg(f + 3);
  }
  const double* w = o.rd_w[e - n];
  return w[0] * 0.0 + w[1] * __ldg(f + n - 1) + w[2] * __ldg(f + n - 2) + w[3] * __ldg(f + n - 3) +
         w[4] * __ldg(f + n - 4);
}

__device__ __forceinline__ double rd_adv(const Ops& o, const double* __restrict__ f, int n, int i) {
  return o.rd_cadv * (rd_ext(o, f, n, i - 2) - 8.0 * rd_ext(o, f, n, i - 1) + 8.0 * rd_ext(o, f, n, i + 1) -
                      rd_ext(o, f, n, i + 2));
}

__device__ __forceinline__ double rd_diff(const Ops& o, const double* __restrict__ f, int n, int i) {
  return o.rd_cdiff * (-rd_ext(o, f, n, i - 2) + 16.0 * rd_ext(o, f, n, i - 1) - 30.0 * rd_ext(o, f, n, i) +
                       16.0 * rd_ext(o, f, n, i + 1) - rd_ext(o, f, n, i + 2));
}

// 3-D launch over (x, y, z * S): block (256,1) in 1-D, (32,8) otherwise; the point comes straight
// from the block/thread indices (no 64-bit integer division per element).
struct Pt {
  int i, j, k, s;
  long long cell;  // index within one species plane
};

__device__ __forceinline__ bool grid_point(int nx, int ny, int nz, Pt& p) {
  p.i = blockIdx.x * blockDim.x + threadIdx.x;
  p.j = blockIdx.y * blockDim.y + threadIdx.y;
  const unsigned zs = blockIdx.z;
  p.k = (int)(zs % (unsigned)nz);
  p.s = (int)(zs / (unsigned)nz);
  p.cell = ((long long)p.k * ny + p.j) * nx + p.i;
  return p.i < nx && p.j < ny;
}

#ifndef __CUDACC_RTC__
inline dim3 stencil_block(int ndim) { return ndim == 1 ? dim3(256, 1, 1) : dim3(32, 8, 1); }
inline dim3 stencil_grid(int nx, int ny, int nz, int S, int ndim) {
  const dim3 b = stencil_block(ndim);
  return dim3((unsigned)((nx + b.x - 1) / b.x), (unsigned)((ny + b.y - 1) / b.y), (unsigned)(nz * S));
}
#endif

// F_A and/or F_D of phi (either output may be null)
template <int DIM>
__global__ void __launch_bounds__(256) k_eval_ad(Ops o, Geom g, const double* __restrict__ phi,
                                                 double* __restrict__ fa, double* __restrict__ fd) {
  Pt p;
  if (!grid_point(g.nx, g.ny, g.nz, p)) return;
  const int s = p.s, i = p.i, j = p.j, k = p.k;
  const long long e = (long long)s * g.ncell + p.cell;
  const double* f = phi + (long long)s * g.ncell;
  if (o.ref_rd) {
    if (fa) {
      const double v = rd_adv(o, f, g.nx, i);
      fa[e] = v;
      flag_wild(o.wild, wild_bits(v));
    }
    if (fd) fd[e] = rd_diff(o, f, g.nx, i);
    return;
  }
  if (fa) {
    const double v = adv_periodic<DIM>(o, g, f, i, j, k);
    fa[e] = v;
    flag_wild(o.wild, wild_bits(v));
  }
  if (fd) fd[e] = diff_periodic<DIM>(o, g, f, s, i, j, k);
}

}  // namespace cisdc_b200
