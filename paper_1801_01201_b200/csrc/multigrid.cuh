// K3 (2-D/3-D): implicit diffusion solve (I - coef d_s Lap4) x = b by cell-centred geometric
// multigrid, all species batched in every launch (grid.y = species; a converged species is
// masked out with a device flag).  The algorithm and its per-point arithmetic are specified in
// oracle/co_problems.c ("multigrid") and DESIGN.md; the CPU oracle runs the identical cycles so the
// GPU result is bit-identical, and the reference's residual tolerance semantics apply:
// stop when ||b - A x||_inf <= mg_tol * ||b||_inf per species (max-norms are order-independent, so
// the stop decisions are exact).
//
// Kernels (each HBM-bound on its own level):
//   k_mg_absmax    ||b||_inf per species
//   k_mg_resmax    ||b - A x||_inf per species on level 0
//   k_mg_update    per-species convergence / cycle bookkeeping (1 block)
//   k_mg_smooth    weighted Jacobi sweep (13-point 3-D / 9-point 2-D star, radius 2)
//   k_mg_restrict  residual + 2^d-child average, fused
//   k_mg_prolong   (bi/tri)linear cell-centred interpolation + correction, fused
#pragma once

#include <algorithm>
#include <cstdlib>
#include <utility>
#include <vector>

#include "common.cuh"
#include "stencil.cuh"
#include "stencil2d.cuh"
#include "stencil3d.cuh"
#include "tma.cuh"

namespace cisdc_b200 {

constexpr int kMgMaxLevels = 16;

struct MgLevel {
  int nx, ny, nz;
  long long ncell;
  double* x;
  double* t;
  double* b;
};

struct MgHierarchy {
  int L = 0;
  int ndim = 0, S = 0;
  MgLevel lv[kMgMaxLevels] = {};
  int* d_active = nullptr;        // [S]
  int* d_cycles = nullptr;        // [S]
  double* d_bmax = nullptr;       // [S]
  double* d_rmax = nullptr;       // [S]
  int* d_flag = nullptr;          // [2]: any_active, failed species + 1
  unsigned* d_tag = nullptr;      // failure tag of the running solve (DevStatus::fail_key)
  int* h_flag = nullptr;          // pinned mirror
  std::vector<std::pair<double, int>> predicted;  // cycles the last solve with this coef needed
  // Captured V-cycles (the cycles after the first of a solve are identical launch sequences for a
  // given coefficient and output buffer): one graph launch replaces a cycle's tens of kernels.
  struct CycleGraph {
    double coef;
    const void *rhs, *out;
    int L;
    cudaGraphExec_t exec;
    long long kernels;
  };
  std::vector<CycleGraph> graphs;
  // Device-looped solves (mg_solve_graph): the first cycle, a WHILE node whose body is one cycle
  // (its decision kernel sets the condition), and the copy for species that needed no cycle.
  struct SolveGraph {
    double coef;
    const void *rhs, *out;
    int L;
    cudaGraphExec_t exec;
    long long kernels;  // launched by every replay (the body's cycles are counted on the device)
  };
  std::vector<SolveGraph> solve_graphs;
  cudaStream_t s_body = nullptr;  // capture stream of the WHILE bodies
  std::vector<void*> allocs;
};

struct MgCoef {
  int ndim;
  double coef;
  double c[kMaxS][3];
  double wD[kMaxS];
};

__device__ __forceinline__ double mg_at(const double* __restrict__ f, int nx, int ny, int nz, int i, int j, int k, int a,
                                        int o) {
  if (a == 0) i = wrapi(i + o, nx);
  else if (a == 1) j = wrapi(j + o, ny);
  else k = wrapi(k + o, nz);
  return __ldg(f + ((long long)k * ny + j) * nx + i);
}

template <int DIM>
__device__ __forceinline__ double mg_ax(const MgCoef& C, int s, const double* __restrict__ x, int nx, int ny, int nz,
                                        int i, int j, int k) {
  double lap = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const double g0 = mg_at(x, nx, ny, nz, i, j, k, a, -2);
    const double g1 = mg_at(x, nx, ny, nz, i, j, k, a, -1);
    const double g2 = mg_at(x, nx, ny, nz, i, j, k, a, 0);
    const double g3 = mg_at(x, nx, ny, nz, i, j, k, a, 1);
    const double g4 = mg_at(x, nx, ny, nz, i, j, k, a, 2);
    lap = lap + C.c[s][a] * lap5(g0, g1, g2, g3, g4);
  }
  return __ldg(x + ((long long)k * ny + j) * nx + i) - C.coef * lap;
}

// All level kernels run on the 3-D grid of stencil.cuh (x, y, z * S): no integer division per point.

__global__ void k_mg_absmax(const double* __restrict__ b, long long ncell, double* __restrict__ out) {
  const int s = blockIdx.y;
  const double* f = b + (long long)s * ncell;
  double m = 0.0;
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(f[c]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out + s, m);
}

// grid (tiles_x, tiles_y, S); every thread walks its (i, j) column over all k, one atomic per block
template <int DIM>
__global__ void __launch_bounds__(256) k_mg_resmax(const __grid_constant__ MgCoef C, const double* __restrict__ x,
                                                   const double* __restrict__ b, int nx, int ny, int nz,
                                                   const int* __restrict__ active, double* __restrict__ out,
                                                   double* __restrict__ bmax) {
  __shared__ double red[8];
  __shared__ double redb[8];
  const int s = blockIdx.z;
  if (!active[s]) return;  // uniform per block
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y * blockDim.y + threadIdx.y;
  const long long ncell = (long long)nx * ny * nz;
  const double* xs = x + (long long)s * ncell;
  const double* bs = b + (long long)s * ncell;
  double m = 0.0, mb = 0.0;
  if (i < nx && j < ny)
    for (int k = 0; k < nz; ++k) {
      const double bv = bs[((long long)k * ny + j) * nx + i];
      m = fmax(m, fabs(bv - mg_ax<DIM>(C, s, xs, nx, ny, nz, i, j, k)));
      mb = fmax(mb, fabs(bv));
    }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    m = fmax(m, __shfl_down_sync(0xffffffffu, m, off));
    mb = fmax(mb, __shfl_down_sync(0xffffffffu, mb, off));
  }
  const int t = threadIdx.y * blockDim.x + threadIdx.x;
  if ((t & 31) == 0) {
    red[t >> 5] = m;
    redb[t >> 5] = mb;
  }
  __syncthreads();
  if (t == 0) {
    for (int w = 1; w < (int)(blockDim.x * blockDim.y) / 32; ++w) {
      m = fmax(m, red[w]);
      mb = fmax(mb, redb[w]);
    }
    if (m > 0.0) atomic_max_nonneg(out + s, m);
    if (bmax && mb > 0.0) atomic_max_nonneg(bmax + s, mb);
  }
}

// out = b for the species that needed no cycle (x = b met the tolerance)
__global__ void k_mg_copy_unswept(const double* __restrict__ b, double* __restrict__ out, long long ncell,
                                  const int* __restrict__ cycles) {
  const int s = blockIdx.y;
  if (cycles[s] != 0) return;
  const long long base = (long long)s * ncell;
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += (long long)gridDim.x * blockDim.x)
    out[base + c] = b[base + c];
}

// per-species stop decision of the oracle's loop: rn <= tol*bn -> done; cap -> failure
// count == 0: the decision of a check-only pass (no cycle follows it in the same launch sequence;
// the next cycle's fused check repeats the same decision and counts).  Returns "some species goes on".
__device__ __forceinline__ int mg_update_body(int S, double tol, int max_cycles, int* active, int* cycles,
                                              const double* bmax, double* rmax, int* flag, DevStatus* st,
                                              const unsigned* tag, int count) {
  int any = 0;
  for (int s = 0; s < S; ++s) {
    if (!active[s]) continue;
    const double thr = tol * bmax[s];
    if (rmax[s] <= thr) {
      active[s] = 0;
      continue;
    }
    if (!count) {
      any = 1;
      continue;
    }
    if (cycles[s] >= max_cycles) {
      active[s] = 0;
      if (flag[1] == 0) flag[1] = s + 1;
      record_failure(st, *tag, CISDC_E_NUMERIC, (unsigned long long)s);
      continue;
    }
    cycles[s] += 1;
    st->mg_cycles += 1;
    any = 1;
  }
  for (int s = 0; s < S; ++s) rmax[s] = 0.0;
  flag[0] = any;
  return any;
}
__global__ void k_mg_update(int S, double tol, int max_cycles, int* active, int* cycles, const double* bmax,
                            double* rmax, int* flag, DevStatus* st, const unsigned* tag, int count = 1) {
  if (threadIdx.x != 0) return;
  mg_update_body(S, tol, max_cycles, active, cycles, bmax, rmax, flag, st, tag, count);
}
// The same decision inside a device-looped solve graph (mg_solve_graph): it also sets the WHILE
// node's condition -- run another cycle iff some species goes on and none failed, the host loop's
// exit test -- and counts the kernels of that next cycle into the status word (the host learns
// the launch count at the step's status read).
__global__ void k_mg_update_loop(int S, double tol, int max_cycles, int* active, int* cycles, const double* bmax,
                                 double* rmax, int* flag, DevStatus* st, const unsigned* tag,
                                 cudaGraphConditionalHandle loop, unsigned long long cycle_kernels) {
  if (threadIdx.x != 0) return;
  const int any = mg_update_body(S, tol, max_cycles, active, cycles, bmax, rmax, flag, st, tag, 1);
  const unsigned go = (any && flag[1] == 0) ? 1u : 0u;
  if (go) st->loop_kernels += cycle_kernels;
  cudaGraphSetConditional(loop, go);
}

// per-solve reset of the bookkeeping (one launch instead of memsets and a host copy); the solve's
// failure tag goes to device memory because captured cycle graphs are replayed across solves
__global__ void k_mg_begin(int S, int* active, int* cycles, double* bmax, double* rmax, int* flag, unsigned* tag,
                           unsigned tag_value) {
  const int s = threadIdx.x;
  if (s < S) {
    active[s] = 1;
    cycles[s] = 0;
    bmax[s] = 0.0;
    rmax[s] = 0.0;
  }
  if (s == 0) {
    flag[0] = flag[1] = 0;
    *tag = tag_value;
  }
}

// max of non-negative values, NaN ignored (the oracle's `if (r > m) m = r`)
__device__ __forceinline__ double max_keep(double m, double r) { return r > m ? r : m; }
// The running max of |v| kept as a signed value ms whose magnitude is max_keep's (|v| > |ms| ? v :
// ms; NaN never wins): the compare takes both magnitudes as operand modifiers, so no |v| is
// materialised per cell (an FP64 add on sm_100a).  The norm is fabs(ms).
__device__ __forceinline__ double max_keep_abs(double ms, double v) { return fabs(v) > fabs(ms) ? v : ms; }

// block max of m (and mb) -> one atomic per block into out[s] (bmax[s]); all threads participate
template <bool BMAX>
__device__ __forceinline__ void block_max_atomic(double m, double mb, double* red, double* redb, double* out,
                                                 double* bmax) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    m = max_keep(m, __shfl_down_sync(0xffffffffu, m, off));
    if (BMAX) mb = max_keep(mb, __shfl_down_sync(0xffffffffu, mb, off));
  }
  const int t = threadIdx.y * blockDim.x + threadIdx.x, nw = (int)(blockDim.x * blockDim.y) / 32;
  if ((t & 31) == 0) {
    red[t >> 5] = m;
    redb[t >> 5] = mb;
  }
  __syncthreads();
  if (t == 0) {
    for (int w = 1; w < nw; ++w) {
      m = max_keep(m, red[w]);
      mb = max_keep(mb, redb[w]);
    }
    if (m > 0.0) atomic_max_nonneg(out, m);
    if (BMAX && mb > 0.0) atomic_max_nonneg(bmax, mb);
  }
}

// Weighted Jacobi sweep x -> xo.  NORM: the sweep's residual r = b - A x is also the residual of
// its INPUT iterate, so ||r||_inf (and ||b||_inf with BMAX) of the input is reduced on the fly:
// the convergence check of x and the cycle's first sweep from x are one pass (the decision kernel
// runs after it; a species found converged keeps x, see mg_solve_dim).
template <int DIM, bool NORM = false, bool BMAX = false>
__global__ void __launch_bounds__(256) k_mg_smooth(const __grid_constant__ MgCoef C, const double* __restrict__ x,
                                                   const double* __restrict__ b, double* __restrict__ xo, int nx,
                                                   int ny, int nz, int from_zero, const int* __restrict__ active,
                                                   double* __restrict__ out = nullptr,
                                                   double* __restrict__ bmax = nullptr) {
  Pt p;
  const bool inr = grid_point(nx, ny, nz, p);
  if (!active[p.s]) return;  // uniform per block
  const long long ncell = (long long)nx * ny * nz;
  const long long e = (long long)p.s * ncell + p.cell;
  if (!NORM) {
    if (!inr) return;
    if (from_zero) {
      xo[e] = C.wD[p.s] * b[e];
      return;
    }
  }
  double m = 0.0, mb = 0.0;
  if (inr) {
    const double* xs = x + (long long)p.s * ncell;
    const double bv = b[e];
    const double r = bv - mg_ax<DIM>(C, p.s, xs, nx, ny, nz, p.i, p.j, p.k);
    xo[e] = xs[p.cell] + C.wD[p.s] * r;
    if (NORM) {
      m = fabs(r);
      if (BMAX) mb = fabs(bv);
    }
  }
  if (NORM) {
    __shared__ double red[8], redb[8];
    block_max_atomic<BMAX>(m, mb, red, redb, out + p.s, bmax + p.s);
  }
}

// 3-D levels: 2.5-D blocked versions (stencil3d.cuh) of the smoother and the residual norm.
// A x at (i,j,k) from the tile / z-queue taps, same expression as mg_ax.
__device__ __forceinline__ double mg_ax_taps(const MgCoef& C, int s, const double (&v)[3][5]) {
  double lap = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    lap = lap + C.c[s][a] * lap5(v[a][0], v[a][1], v[a][2], v[a][3], v[a][4]);
  return v[0][2] - C.coef * lap;
}

// SMOOTH: x -> xo (not from zero); NORM: ||b - A x||_inf per species into out[s] (of the input
// x; fused with SMOOTH this is the check + first sweep of a cycle); BMAX: also ||b||_inf into bmax[s]
template <bool SMOOTH, bool NORM, bool BMAX>
__global__ void __launch_bounds__(kTX* kTY, kMgMinBlocks) k_mg3_tiled(const __grid_constant__ MgCoef C, const double* __restrict__ x,
                                                         const double* __restrict__ b, double* __restrict__ xo,
                                                         int nx, int ny, int nz, int kc, const int* __restrict__ active,
                                                         double* __restrict__ out, double* __restrict__ bmax) {
  __shared__ TileRing ring;
  __shared__ AuxRing aring;
  __shared__ double red[kTX * kTY / 32];
  __shared__ double redb[kTX * kTY / 32];
  const ZChunk z = zchunk(nz, kc);
  if (!active[z.s]) return;  // uniform per block
  const long long ncell = (long long)nx * ny * nz;
  const long long sbase = (long long)z.s * ncell;
  double* xos = SMOOTH ? opaque(xo + sbase) : nullptr;
  const int s = z.s;
  const double cs0 = C.c[s][0], cs1 = C.c[s][1], cs2 = C.c[s][2], coef = C.coef, wd = C.wD[s];
  double m = 0.0, mb = 0.0;
  walk_tiled<!BMAX>(x + sbase, b + sbase, nx, ny, nz, z, ring, &aring, [](int) {},
                   [&](int, unsigned cell, const double (&v)[3][5], double bva, bool ok) {
                     const double bv = BMAX ? v[0][2] : bva;  // BMAX: x is b (the solve's first check)
                     // mg_ax_taps with the species coefficients hoisted (same expression)
                     double lap = 0.0;
                     lap = lap + cs0 * lap5(v[0][0], v[0][1], v[0][2], v[0][3], v[0][4]);
                     lap = lap + cs1 * lap5(v[1][0], v[1][1], v[1][2], v[1][3], v[1][4]);
                     lap = lap + cs2 * lap5(v[2][0], v[2][1], v[2][2], v[2][3], v[2][4]);
                     const double r = bv - (v[0][2] - coef * lap);
                     if (!ok) return;
                     if (SMOOTH) __stcg(xos + cell, v[2][2] + wd * r);
                     if (NORM) m = max_keep_abs(m, r);
                     if (BMAX) mb = max_keep_abs(mb, bv);
                   });
  if (NORM) block_max_atomic<BMAX>(fabs(m), fabs(mb), red, redb, out + z.s, bmax + z.s);
}

// The same level-0 sweep / check with two x-adjacent cells per thread (even nx; walk_pair): 128-bit
// shared loads of the staged tiles, the rhs staged as pairs; per cell the identical expression.
// Dynamic shared memory: kMgPairSmem (6-plane rings, 3 blocks per SM).
template <bool SMOOTH, bool NORM, bool BMAX>
__global__ void __launch_bounds__(kTX* kTY, 3) k_mg3_pair(const __grid_constant__ MgCoef C, const double* __restrict__ x,
                                                          const double* __restrict__ b, double* __restrict__ xo, int nx,
                                                          int ny, int nz, int kc, const int* __restrict__ active,
                                                          double* __restrict__ out, double* __restrict__ bmax) {
  extern __shared__ __align__(16) double mg_pring[];
  __shared__ double red[kTX * kTY / 32];
  __shared__ double redb[kTX * kTY / 32];
  const ZChunk z = zchunk(nz, kc);
  if (!active[z.s]) return;  // uniform per block
  const long long ncell = (long long)nx * ny * nz;
  const long long sbase = (long long)z.s * ncell;
  double* xos = SMOOTH ? opaque(xo + sbase) : nullptr;
  const int s = z.s;
  const double cs0 = C.c[s][0], cs1 = C.c[s][1], cs2 = C.c[s][2], coef = C.coef, wd = C.wD[s];
  double m = 0.0, mb = 0.0;
  walk_pair<!BMAX, kMgRing, kMgRing - 2>(x + sbase, b + sbase, nx, ny, nz, z, mg_pring, mg_pring + kMgRing * kPPlaneSlot, [](int) {},
                  [&](int, unsigned cell, const PairTaps& v, const double (&bva)[2], bool ok) {
                    double xn[2];
                    // BMAX: x is b (the solve's first check), so b comes from the x tile's centre taps
                    const double bv[2] = {BMAX ? v.x[2] : bva[0], BMAX ? v.x[3] : bva[1]};
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                      double lap = 0.0;
                      lap = lap + cs0 * lap5(v.x[c], v.x[c + 1], v.x[c + 2], v.x[c + 3], v.x[c + 4]);
                      lap = lap + cs1 * lap5(v.y[c][0], v.y[c][1], v.y[c][2], v.y[c][3], v.y[c][4]);
                      lap = lap + cs2 * lap5(v.z[c][0], v.z[c][1], v.z[c][2], v.z[c][3], v.z[c][4]);
                      const double r = bv[c] - (v.x[c + 2] - coef * lap);
                      xn[c] = v.z[c][2] + wd * r;
                      if (NORM && ok) m = max_keep_abs(m, r);
                      if (BMAX && ok) mb = max_keep_abs(mb, bv[c]);
                    }
                    if (SMOOTH && ok) __stcg(reinterpret_cast<double2*>(xos + cell), make_double2(xn[0], xn[1]));
                  });
  if (NORM) block_max_atomic<BMAX>(fabs(m), fabs(mb), red, redb, out + z.s, bmax + z.s);
}

// The same level-0 sweep / check with the planes staged by TMA (tma.cuh walk_pair_tma; whole 64 x 8
// tiles only): per cell the identical expression, so the same bits as k_mg3_pair.
template <bool SMOOTH, bool NORM, bool BMAX>
__global__ void __launch_bounds__(kTX* kTY, 3) k_mg3_tma(const __grid_constant__ MgCoef C,
                                                         const __grid_constant__ TmaMaps maps, double* __restrict__ xo,
                                                         int nx, int ny, int nz, int kc, const int* __restrict__ active,
                                                         double* __restrict__ out, double* __restrict__ bmax) {
  extern __shared__ __align__(128) double mg_tring[];
  __shared__ double red[kTX * kTY / 32];
  __shared__ double redb[kTX * kTY / 32];
  const ZChunk z = zchunk(nz, kc);
  if (!active[z.s]) return;  // uniform per block
  const long long ncell = (long long)nx * ny * nz;
  double* xos = SMOOTH ? opaque(xo + (long long)z.s * ncell) : nullptr;
  const int s = z.s;
  const double cs0 = C.c[s][0], cs1 = C.c[s][1], cs2 = C.c[s][2], coef = C.coef, wd = C.wD[s];
  double m = 0.0, mb = 0.0;
  walk_pair_tma<!BMAX, false>(maps, nx, ny, nz, z, mg_tring, [](int) {},
                                    [&](int, unsigned cell, const PairTaps& v, const double (&bva)[2], bool) {
                                      double xn[2];
                                      const double bv[2] = {BMAX ? v.x[2] : bva[0], BMAX ? v.x[3] : bva[1]};
#pragma unroll
                                      for (int c = 0; c < 2; ++c) {
                                        double lap = 0.0;
                                        lap = lap + cs0 * lap5(v.x[c], v.x[c + 1], v.x[c + 2], v.x[c + 3], v.x[c + 4]);
                                        lap = lap + cs1 * lap5(v.y[c][0], v.y[c][1], v.y[c][2], v.y[c][3], v.y[c][4]);
                                        lap = lap + cs2 * lap5(v.z[c][0], v.z[c][1], v.z[c][2], v.z[c][3], v.z[c][4]);
                                        const double r = bv[c] - (v.x[c + 2] - coef * lap);
                                        xn[c] = v.z[c][2] + wd * r;
                                        if (NORM) m = max_keep_abs(m, r);
                                        if (BMAX) mb = max_keep_abs(mb, bv[c]);
                                      }
                                      if (SMOOTH) __stcg(reinterpret_cast<double2*>(xos + cell), make_double2(xn[0], xn[1]));
                                    });
  if (NORM) block_max_atomic<BMAX>(fabs(m), fabs(mb), red, redb, out + z.s, bmax + z.s);
}

// 2-D level sweep / check on the row-streaming walker (stencil2d.cuh; nx even): per cell the
// expression of k_mg_smooth<2> / mg_ax<2>.  Dynamic shared memory kRowSmem.
template <bool SMOOTH, bool NORM, bool BMAX>
__global__ void __launch_bounds__(kRowWarps * 32, 2) k_mg2_rows(const __grid_constant__ MgCoef C, const double* __restrict__ x,
                                                                const double* __restrict__ b, double* __restrict__ xo,
                                                                int nx, int ny, int chunk, const int* __restrict__ active,
                                                                double* __restrict__ out, double* __restrict__ bmax) {
  extern __shared__ __align__(16) double mg_rsm[];
  __shared__ double red[kRowWarps], redb[kRowWarps];
  const int s = blockIdx.z;
  if (!active[s]) return;  // uniform per block
  const long long ncell = (long long)nx * ny;
  const long long sbase = (long long)s * ncell;
  double* xos = SMOOTH ? opaque(xo + sbase) : nullptr;
  const double c0 = C.c[s][0], c1 = C.c[s][1], coef = C.coef, wd = C.wD[s];
  const int j0 = blockIdx.y * chunk, j1 = min(ny, j0 + chunk);
  double m = 0.0, mb = 0.0;
  walk_rows<true>(x + sbase, b + sbase, nx, ny, j0, j1, mg_rsm, [](int) {},
                  [&](int, unsigned cell, const RowTaps& v, const double (&bv)[2], bool ok) {
                    double xn[2];
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                      double lap = 0.0;
                      lap = lap + c0 * lap5(v.x[c], v.x[c + 1], v.x[c + 2], v.x[c + 3], v.x[c + 4]);
                      lap = lap + c1 * lap5(v.y[c][0], v.y[c][1], v.y[c][2], v.y[c][3], v.y[c][4]);
                      const double r = bv[c] - (v.x[c + 2] - coef * lap);
                      xn[c] = v.x[c + 2] + wd * r;
                      if (NORM && ok) m = max_keep_abs(m, r);
                      if (BMAX && ok) mb = max_keep_abs(mb, bv[c]);
                    }
                    if (SMOOTH && ok) __stcg(reinterpret_cast<double2*>(xos + cell), make_double2(xn[0], xn[1]));
                  });
  if (NORM) block_max_atomic<BMAX>(fabs(m), fabs(mb), red, redb, out + s, bmax + s);
}

// launched on the COARSE grid
template <int DIM>
__global__ void __launch_bounds__(256) k_mg_restrict(const __grid_constant__ MgCoef C, const double* __restrict__ x,
                                                     const double* __restrict__ b, int nx, int ny, int nz,
                                                     double* __restrict__ bc, int cx, int cy, int cz,
                                                     const int* __restrict__ active) {
  Pt p;
  if (!grid_point(cx, cy, cz, p)) return;
  const int s = p.s;
  if (!active[s]) return;
  const int I = p.i, J = p.j, K = p.k;
  const long long nc = (long long)cx * cy * cz;
  const long long nf = (long long)nx * ny * nz;
  const double* xs = x + (long long)s * nf;
  const double* bs = b + (long long)s * nf;
  const double scale = DIM == 1 ? 0.5 : (DIM == 2 ? 0.25 : 0.125);
  double acc = 0.0;
#pragma unroll
  for (int dz = 0; dz < (DIM >= 3 ? 2 : 1); ++dz)
#pragma unroll
    for (int dy = 0; dy < (DIM >= 2 ? 2 : 1); ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const int i = 2 * I + dx, j = DIM >= 2 ? 2 * J + dy : J, k = DIM >= 3 ? 2 * K + dz : K;
        const long long id = ((long long)k * ny + j) * nx + i;
        acc = acc + (bs[id] - mg_ax<DIM>(C, s, xs, nx, ny, nz, i, j, k));
      }
  bc[(long long)s * nc + p.cell] = acc * scale;
}

template <int DIM>
__global__ void __launch_bounds__(256) k_mg_prolong(double* __restrict__ x, int nx, int ny, int nz,
                                                    const double* __restrict__ ec, int cx, int cy, int cz,
                                                    const int* __restrict__ active) {
  Pt p;
  if (!grid_point(nx, ny, nz, p)) return;
  const int s = p.s;
  if (!active[s]) return;
  const int i = p.i, j = p.j, k = p.k;
  const long long nf = (long long)nx * ny * nz;
  const double* e = ec + (long long)s * cx * cy * cz;
  const int I = i >> 1, I2 = wrapi((i & 1) ? I + 1 : I - 1, cx);
  int J = j, J2 = j, K = k, K2 = k;
  if (DIM >= 2) {
    J = j >> 1;
    J2 = wrapi((j & 1) ? J + 1 : J - 1, cy);
  }
  if (DIM >= 3) {
    K = k >> 1;
    K2 = wrapi((k & 1) ? K + 1 : K - 1, cz);
  }
#define E_(a, b_, c_) __ldg(e + ((long long)(c_) * cy + (b_)) * cx + (a))
  double v;
  if (DIM == 1) {
    v = 0.75 * E_(I, 0, 0) + 0.25 * E_(I2, 0, 0);
  } else if (DIM == 2) {
    const double a0 = 0.75 * E_(I, J, 0) + 0.25 * E_(I2, J, 0);
    const double a1 = 0.75 * E_(I, J2, 0) + 0.25 * E_(I2, J2, 0);
    v = 0.75 * a0 + 0.25 * a1;
  } else {
    const double a00 = 0.75 * E_(I, J, K) + 0.25 * E_(I2, J, K);
    const double a10 = 0.75 * E_(I, J2, K) + 0.25 * E_(I2, J2, K);
    const double a01 = 0.75 * E_(I, J, K2) + 0.25 * E_(I2, J, K2);
    const double a11 = 0.75 * E_(I, J2, K2) + 0.25 * E_(I2, J2, K2);
    const double b0 = 0.75 * a00 + 0.25 * a10;
    const double b1 = 0.75 * a01 + 0.25 * a11;
    v = 0.75 * b0 + 0.25 * b1;
  }
#undef E_
  const long long id = (long long)s * nf + p.cell;
  x[id] = x[id] + v;
}

// k_mg_restrict on 2-D levels, one coarse cell per thread with its 2 x 2 fine children's taps
// loaded as 128-bit pairs (columns 2I, 2I+1 are adjacent; fine nx is even): 12 vector loads per
// coarse cell instead of 4 x 9 scalar ones.  Per child the expression of mg_ax<2>, children summed
// in k_mg_restrict's order (dy outer, dx inner): same bits.  Grid: (ceil(cx/32), ceil(cy/8), S).
__global__ void __launch_bounds__(256) k_mg_restrict2_pair(const __grid_constant__ MgCoef C,
                                                           const double* __restrict__ x,
                                                           const double* __restrict__ b, int nx, int ny,
                                                           double* __restrict__ bc, int cx, int cy,
                                                           const int* __restrict__ active) {
  const int I = blockIdx.x * 32 + threadIdx.x, J = blockIdx.y * 8 + threadIdx.y, s = blockIdx.z;
  if (I >= cx || J >= cy || !active[s]) return;
  const long long nf = (long long)nx * ny;
  const double* xs = x + (long long)s * nf;
  const double* bs = b + (long long)s * nf;
  const int i = 2 * I;
  auto ld2 = [&](const double* base, int jj, int ii) {
    return __ldg(reinterpret_cast<const double2*>(base + (unsigned)jj * (unsigned)nx + (unsigned)ii));
  };
  const int im2 = wrapi(i - 2, nx), ip2 = wrapi(i + 2, nx);
  double acc = 0.0;
#pragma unroll
  for (int dy = 0; dy < 2; ++dy) {
    const int j = 2 * J + dy;
    // row j: x at i-2 .. i+3 ; column taps at rows j-2, j-1, j+1, j+2 for both cells
    const double2 xl = ld2(xs, j, im2), xc = ld2(xs, j, i), xr = ld2(xs, j, ip2);
    const double2 ym2 = ld2(xs, wrapi(j - 2, ny), i), ym1 = ld2(xs, wrapi(j - 1, ny), i);
    const double2 yp1 = ld2(xs, wrapi(j + 1, ny), i), yp2 = ld2(xs, wrapi(j + 2, ny), i);
    const double2 bv = ld2(bs, j, i);
    const double g[6] = {xl.x, xl.y, xc.x, xc.y, xr.x, xr.y};  // x taps i-2 .. i+3
    const double ya[4] = {ym2.x, ym1.x, yp1.x, yp2.x}, yb[4] = {ym2.y, ym1.y, yp1.y, yp2.y};
#pragma unroll
    for (int dx = 0; dx < 2; ++dx) {
      const double* yy = dx == 0 ? ya : yb;
      const double xcc = g[2 + dx];
      double lap = 0.0;
      lap = lap + C.c[s][0] * lap5(g[dx], g[dx + 1], xcc, g[dx + 3], g[dx + 4]);
      lap = lap + C.c[s][1] * lap5(yy[0], yy[1], xcc, yy[2], yy[3]);
      const double ax = xcc - C.coef * lap;
      acc = acc + ((dx == 0 ? bv.x : bv.y) - ax);
    }
  }
  bc[(long long)s * cx * cy + (long long)J * cx + I] = acc * 0.25;
}

// k_mg_prolong for two x-adjacent fine cells per thread (2-D / 3-D; fine nx is even on every level
// that has a coarser one): fine cells 2I and 2I+1 share the coarse column I, their second columns
// are I-1 and I+1; 32-bit in-plane offsets, the fine pair read and written as 128-bit words.  Per
// cell the expression of k_mg_prolong (same bits).  Grid: (ceil(nx/64), ceil(ny/8), nz * S).
template <int DIM>
__global__ void __launch_bounds__(256) k_mg_prolong_pair(double* __restrict__ x, int nx, int ny, int nz,
                                                         const double* __restrict__ ec, int cx, int cy, int cz,
                                                         const int* __restrict__ active) {
  const int I = blockIdx.x * 32 + threadIdx.x;  // coarse column = fine pair
  const int j = blockIdx.y * 8 + threadIdx.y;
  const unsigned zs = blockIdx.z;
  const int k = (int)(zs % (unsigned)nz), s = (int)(zs / (unsigned)nz);
  if (2 * I >= nx || j >= ny || !active[s]) return;
  const double* e = ec + (long long)s * cx * cy * cz;
  const int Il = wrapi(I - 1, cx), Ir = wrapi(I + 1, cx);  // second columns of cells 2I and 2I+1
  int J = j, J2 = j, K = k, K2 = k;
  if (DIM >= 2) {
    J = j >> 1;
    J2 = wrapi((j & 1) ? J + 1 : J - 1, cy);
  }
  if (DIM >= 3) {
    K = k >> 1;
    K2 = wrapi((k & 1) ? K + 1 : K - 1, cz);
  }
  const unsigned cp = (unsigned)cx * (unsigned)cy;
  auto row = [&](int jj, int kk) { return e + ((unsigned)kk * cp + (unsigned)jj * (unsigned)cx); };
  double v[2];
  if (DIM == 2) {
    const double* r0 = row(J, 0);
    const double* r1 = row(J2, 0);
    const double e0 = __ldg(r0 + I), e1 = __ldg(r1 + I);
    {
      const double a0 = 0.75 * e0 + 0.25 * __ldg(r0 + Il);
      const double a1 = 0.75 * e1 + 0.25 * __ldg(r1 + Il);
      v[0] = 0.75 * a0 + 0.25 * a1;
    }
    {
      const double a0 = 0.75 * e0 + 0.25 * __ldg(r0 + Ir);
      const double a1 = 0.75 * e1 + 0.25 * __ldg(r1 + Ir);
      v[1] = 0.75 * a0 + 0.25 * a1;
    }
  } else {
    const double* r00 = row(J, K);
    const double* r10 = row(J2, K);
    const double* r01 = row(J, K2);
    const double* r11 = row(J2, K2);
    const double e00 = __ldg(r00 + I), e10 = __ldg(r10 + I), e01 = __ldg(r01 + I), e11 = __ldg(r11 + I);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int I2 = c == 0 ? Il : Ir;
      const double a00 = 0.75 * e00 + 0.25 * __ldg(r00 + I2);
      const double a10 = 0.75 * e10 + 0.25 * __ldg(r10 + I2);
      const double a01 = 0.75 * e01 + 0.25 * __ldg(r01 + I2);
      const double a11 = 0.75 * e11 + 0.25 * __ldg(r11 + I2);
      const double b0 = 0.75 * a00 + 0.25 * a10;
      const double b1 = 0.75 * a01 + 0.25 * a11;
      v[c] = 0.75 * b0 + 0.25 * b1;
    }
  }
  double2* xp = reinterpret_cast<double2*>(x + (long long)s * ((long long)nx * ny * nz) +
                                           ((unsigned)k * (unsigned)nx * (unsigned)ny + (unsigned)j * (unsigned)nx +
                                            (unsigned)(2 * I)));
  const double2 xv = *xp;
  *xp = make_double2(xv.x + v[0], xv.y + v[1]);
}

// The coarse end of a V-cycle in one kernel: levels lc .. L-1 (each at most a few thousand cells)
// for one species per block, with __syncthreads between the steps instead of a launch per step.
// Per point the operations of k_mg_smooth / k_mg_restrict / k_mg_prolong, in the order of
// MgRunner::vcycle; the ping-pong pointers of every level make an even number of swaps, so the
// host-side assignment is unchanged afterwards.
constexpr int kMgCoarseThreads = 1024;
struct MgCoarseArgs {
  int lc, L, pre, post, coarse;
  int nx[kMgMaxLevels], ny[kMgMaxLevels], nz[kMgMaxLevels];
  double *x[kMgMaxLevels], *t[kMgMaxLevels], *b[kMgMaxLevels];
  MgCoef C[kMgMaxLevels];
  const int* active;
};

template <int DIM>
__global__ void __launch_bounds__(kMgCoarseThreads) k_mg_coarse(const __grid_constant__ MgCoarseArgs A) {
  const int s = blockIdx.x;
  if (!A.active[s]) return;
  // the levels' current (x, t) pointers, swapped after every sweep (block-uniform, in shared memory)
  __shared__ double* xs[kMgMaxLevels];
  __shared__ double* ts[kMgMaxLevels];
  if (threadIdx.x == 0)
    for (int l = A.lc; l < A.L; ++l) {
      xs[l] = A.x[l];
      ts[l] = A.t[l];
    }
  __syncthreads();
  auto sweep = [&](int l, bool from_zero) {
    const int nx = A.nx[l], ny = A.ny[l], nz = A.nz[l];
    const int nc = nx * ny * nz;
    const long long base = (long long)s * nc;
    const MgCoef& C = A.C[l];
    double* to = ts[l] + base;
    const double* xsp = xs[l] + base;
    const double* bs = A.b[l] + base;
    for (int c = threadIdx.x; c < nc; c += blockDim.x) {
      if (from_zero) {
        to[c] = C.wD[s] * bs[c];
      } else {
        const int i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
        const double r = bs[c] - mg_ax<DIM>(C, s, xsp, nx, ny, nz, i, j, k);
        to[c] = xsp[c] + C.wD[s] * r;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double* tmp = xs[l];
      xs[l] = ts[l];
      ts[l] = tmp;
    }
    __syncthreads();
  };
  for (int l = A.lc; l < A.L - 1; ++l) {
    for (int it = 0; it < A.pre; ++it) sweep(l, l > 0 && it == 0);
    // restriction into level l+1 (k_mg_restrict)
    const int nx = A.nx[l], ny = A.ny[l], nz = A.nz[l];
    const int cx = A.nx[l + 1], cy = A.ny[l + 1], cz = A.nz[l + 1];
    const int nf = nx * ny * nz, nc = cx * cy * cz;
    const double* xsp = xs[l] + (long long)s * nf;
    const double* bsp = A.b[l] + (long long)s * nf;
    const double scale = DIM == 1 ? 0.5 : (DIM == 2 ? 0.25 : 0.125);
    for (int c = threadIdx.x; c < nc; c += blockDim.x) {
      const int I = c % cx, J = (c / cx) % cy, K = c / (cx * cy);
      double acc = 0.0;
#pragma unroll
      for (int dz = 0; dz < (DIM >= 3 ? 2 : 1); ++dz)
#pragma unroll
        for (int dy = 0; dy < (DIM >= 2 ? 2 : 1); ++dy)
#pragma unroll
          for (int dx = 0; dx < 2; ++dx) {
            const int i = 2 * I + dx, j = DIM >= 2 ? 2 * J + dy : J, k = DIM >= 3 ? 2 * K + dz : K;
            const long long id = ((long long)k * ny + j) * nx + i;
            acc = acc + (bsp[id] - mg_ax<DIM>(A.C[l], s, xsp, nx, ny, nz, i, j, k));
          }
      A.b[l + 1][(long long)s * nc + c] = acc * scale;
    }
    __syncthreads();
  }
  {
    const int l = A.L - 1;
    const int ns = A.L == 1 ? A.pre : A.coarse;
    for (int it = 0; it < ns; ++it) sweep(l, l > 0 && it == 0);
  }
  for (int l = A.L - 2; l >= A.lc; --l) {
    // prolongation of level l+1 into level l (k_mg_prolong)
    const int nx = A.nx[l], ny = A.ny[l], nz = A.nz[l];
    const int cx = A.nx[l + 1], cy = A.ny[l + 1], cz = A.nz[l + 1];
    const int nf = nx * ny * nz;
    const double* e = xs[l + 1] + (long long)s * cx * cy * cz;
    double* xl = xs[l] + (long long)s * nf;
    for (int c = threadIdx.x; c < nf; c += blockDim.x) {
      const int i = c % nx, j = (c / nx) % ny, k = c / (nx * ny);
      const int I = i >> 1, I2 = wrapi((i & 1) ? I + 1 : I - 1, cx);
      int J = j, J2 = j, K = k, K2 = k;
      if (DIM >= 2) {
        J = j >> 1;
        J2 = wrapi((j & 1) ? J + 1 : J - 1, cy);
      }
      if (DIM >= 3) {
        K = k >> 1;
        K2 = wrapi((k & 1) ? K + 1 : K - 1, cz);
      }
#define E_(a, b_, c_) e[((long long)(c_) * cy + (b_)) * cx + (a)]
      double v;
      if (DIM == 1) {
        v = 0.75 * E_(I, 0, 0) + 0.25 * E_(I2, 0, 0);
      } else if (DIM == 2) {
        const double a0 = 0.75 * E_(I, J, 0) + 0.25 * E_(I2, J, 0);
        const double a1 = 0.75 * E_(I, J2, 0) + 0.25 * E_(I2, J2, 0);
        v = 0.75 * a0 + 0.25 * a1;
      } else {
        const double a00 = 0.75 * E_(I, J, K) + 0.25 * E_(I2, J, K);
        const double a10 = 0.75 * E_(I, J2, K) + 0.25 * E_(I2, J2, K);
        const double a01 = 0.75 * E_(I, J, K2) + 0.25 * E_(I2, J, K2);
        const double a11 = 0.75 * E_(I, J2, K2) + 0.25 * E_(I2, J2, K2);
        const double b0 = 0.75 * a00 + 0.25 * a10;
        const double b1 = 0.75 * a01 + 0.25 * a11;
        v = 0.75 * b0 + 0.25 * b1;
      }
#undef E_
      xl[c] = xl[c] + v;
    }
    __syncthreads();
    for (int it = 0; it < A.post; ++it) sweep(l, false);
  }
}

// ------------------------------------------------------------------ host side

inline int mg_init(MgHierarchy& h, const Geom& g, const cisdc_problem_desc& d) {
  h.ndim = g.ndim;
  h.S = g.S;
  int n[3] = {g.nx, g.ny, g.nz};
  const int minc = d.mg_min_coarse > 2 ? d.mg_min_coarse : 4;
  if (d.mg_pre < 2 || d.mg_coarse_sweeps < 2 || d.mg_post < 0 || d.mg_max_cycles < 1 || d.mg_pre % 2 ||
      d.mg_post % 2 || d.mg_coarse_sweeps % 2)
    return CISDC_E_INVALID_ARGUMENT;  // even sweep counts: see MgRunner
  h.L = 0;
  for (;;) {
    MgLevel& L = h.lv[h.L];
    L.nx = n[0];
    L.ny = n[1];
    L.nz = n[2];
    L.ncell = (long long)n[0] * n[1] * n[2];
    const size_t bytes = sizeof(double) * (size_t)L.ncell * g.S;
    for (double** p : {&L.x, &L.t, &L.b}) {
      void* v = nullptr;
      if (cudaMalloc(&v, bytes) != cudaSuccess) return CISDC_E_CUDA;
      h.allocs.push_back(v);
      *p = static_cast<double*>(v);
    }
    h.L++;
    bool ok = h.L < kMgMaxLevels;
    for (int a = 0; a < g.ndim; ++a)
      if (n[a] % 2 != 0 || n[a] / 2 < minc) ok = false;
    if (!ok) break;
    for (int a = 0; a < g.ndim; ++a) n[a] /= 2;
  }
  void* v = nullptr;
  auto al = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    h.allocs.push_back(p);
    return p;
  };
  h.d_active = static_cast<int*>(al(sizeof(int) * g.S));
  h.d_cycles = static_cast<int*>(al(sizeof(int) * g.S));
  h.d_bmax = static_cast<double*>(al(sizeof(double) * g.S));
  h.d_rmax = static_cast<double*>(al(sizeof(double) * g.S));
  h.d_flag = static_cast<int*>(al(sizeof(int) * 2));
  h.d_tag = static_cast<unsigned*>(al(sizeof(unsigned)));
  if (!h.d_active || !h.d_cycles || !h.d_bmax || !h.d_rmax || !h.d_flag || !h.d_tag) return CISDC_E_CUDA;
  if (cudaMallocHost(&v, sizeof(int) * 2) != cudaSuccess) return CISDC_E_CUDA;
  h.h_flag = static_cast<int*>(v);
  if (cudaStreamCreateWithFlags(&h.s_body, cudaStreamNonBlocking) != cudaSuccess) return CISDC_E_CUDA;
  return CISDC_OK;
}

inline void mg_free(MgHierarchy& h) {
  for (auto& g : h.graphs) cudaGraphExecDestroy(g.exec);
  h.graphs.clear();
  for (auto& g : h.solve_graphs) cudaGraphExecDestroy(g.exec);
  h.solve_graphs.clear();
  if (h.s_body) cudaStreamDestroy(h.s_body);
  h.s_body = nullptr;
  for (void* p : h.allocs) cudaFree(p);
  h.allocs.clear();
  if (h.h_flag) cudaFreeHost(h.h_flag);
  h.h_flag = nullptr;
}

// Per-solve plan: levels used and optimal Jacobi weights (identical arithmetic to the oracle's
// mg_plan, oracle/co_problems.c).  Returns the number of levels used.
inline int mg_plan(const MgHierarchy& h, const cisdc_problem_desc& d, double coef, MgCoef* C) {
  double rho[kMgMaxLevels];
  double emax[kMgMaxLevels][kMaxS], ehf[kMgMaxLevels][kMaxS];
  for (int l = 0; l < h.L; ++l) {
    C[l] = MgCoef{};
    C[l].ndim = d.ndim;
    C[l].coef = coef;
    rho[l] = 0.0;
    for (int s = 0; s < d.nspecies; ++s) {
      double csum = 0.0, cmin = 0.0;
      for (int a = 0; a < d.ndim; ++a) {
        const double hl = d.h[a] * (double)(1 << l);
        C[l].c[s][a] = d.diffusivity[s] / (12.0 * hl * hl);
        csum = csum + C[l].c[s][a];
        cmin = (a == 0 || C[l].c[s][a] < cmin) ? C[l].c[s][a] : cmin;
      }
      emax[l][s] = 1.0 + coef * (64.0 * csum);
      ehf[l][s] = 1.0 + coef * (28.0 * cmin);
      const double r = (emax[l][s] - 1.0) / (emax[l][s] + 1.0);
      rho[l] = r > rho[l] ? r : rho[l];
    }
  }
  int L = 1;
  while (L < h.L && rho[L - 1] > 0.1) ++L;
  for (int l = 0; l < L; ++l)
    for (int s = 0; s < d.nspecies; ++s) C[l].wD[s] = 2.0 / ((l < L - 1 ? ehf[l][s] : 1.0) + emax[l][s]);
  return L;
}

// the last check of a predicted batch as a residual-only pass (CISDC_MG_CHECKONLY=0: fused)
inline bool mg_check_only_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("CISDC_MG_CHECKONLY");
    return !(e && e[0] == '0');
  }();
  return v;
}

// levels of at most this many cells run inside one k_mg_coarse launch (CISDC_MG_COARSE=0: off)
constexpr long long kMgCoarseCells = 1024;
inline bool mg_coarse_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("CISDC_MG_COARSE");
    return !(e && e[0] == '0');
  }();
  return v;
}

// prolongation with two fine cells per thread and the 2-D restriction with vector taps
// (CISDC_MG_PROLONG_PAIR=0: the per-point kernels)
inline bool mg_pair_prolong() {
  static const bool v = [] {
    const char* e = std::getenv("CISDC_MG_PROLONG_PAIR");
    return !(e && e[0] == '0');
  }();
  return v;
}

// row-streaming 2-D sweeps (CISDC_MG_ROWS=0: the per-point kernel)
inline bool mg_rows_enabled() {
  static const bool env = [] {
    const char* e = std::getenv("CISDC_MG_ROWS");
    return !(e && e[0] == '0');
  }();
  if (!env) return false;
  const int sm = (int)kRowSmem;
  return func_attr_once(k_mg2_rows<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess &&
         func_attr_once(k_mg2_rows<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess &&
         func_attr_once(k_mg2_rows<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess &&
         func_attr_once(k_mg2_rows<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess;
}

// two cells per thread for the level-0 sweeps on even-nx 3-D grids (CISDC_MG_PAIR=0: one per thread)
inline bool mg_pair_enabled() {
  static const bool env = [] {
    const char* e = std::getenv("CISDC_MG_PAIR");
    return !(e && e[0] == '0');
  }();
  if (!env) return false;
  const int sm = (int)kMgPairSmem;
  return func_attr_once(k_mg3_pair<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess &&
         func_attr_once(k_mg3_pair<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess &&
         func_attr_once(k_mg3_pair<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess &&
         func_attr_once(k_mg3_pair<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess;
}

// TMA-staged level-0 sweeps on whole-tile 3-D grids (tma.cuh; CISDC_MG_TMA=0: the cp.async walker).
// Read per launch so that a process can compare the two (tests do).
inline bool mg_tma_enabled() {
  const char* e = std::getenv("CISDC_MG_TMA");
  if (e && e[0] == '0') return false;
  if (!tma_encoder()) return false;
  const int sm = (int)kTmaSmem;
  return func_attr_once(k_mg3_tma<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess &&
         func_attr_once(k_mg3_tma<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess &&
         func_attr_once(k_mg3_tma<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess &&
         func_attr_once(k_mg3_tma<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
             cudaSuccess;
}

// Wraps the engine's hook while a cycle is captured: counts the kernels (the replays are charged
// that many launches) and forwards nothing else (no timing events inside a graph).
struct CountingHook final : LaunchHook {
  long long n = 0;
  void before(int, cudaStream_t) override {}
  void after(int, cudaStream_t, double) override { ++n; }
};

template <int DIM>
struct MgRunner {
  MgHierarchy& h;
  const cisdc_problem_desc& d;
  MgCoef C[kMgMaxLevels];
  int L;  // levels used by this solve
  cudaStream_t s;
  LaunchHook* hook;
  // level-0 x lives in h.lv[0].x (ping-pong with .t); b0 = rhs.  Sweep counts are even, so after
  // every pair of sweeps .x holds the iterate again for active AND masked (converged) species.
  const double* b0;
  const double* first_x = nullptr;  // the initial iterate x = b is read straight from the rhs
  bool check_next = false;          // the next level-0 sweep also reduces the residual norm of its input
  bool first_check = true;          // ... and ||b||_inf (the first check of the solve)
  DevStatus* st = nullptr;
  // Compulsory bytes of one cycle for ALL species, per kernel class: the checking sweep (run for
  // every species still active before the check) and the rest of the cycle (run for the species
  // that continue).  Launches are charged 0 bytes; the solve charges sum_s of its per-species
  // cycle counts afterwards (masked species move no data).
  bool recording = false;
  double fs_bytes = 0.0;
  double rest_bytes[kNumKernelClasses] = {};
  void charge(int cls, double b, bool is_check) {
    if (!recording) return;
    if (is_check) fs_bytes += b;
    else rest_bytes[cls] += b;
  }

  const double* bof(int l) const { return l == 0 ? b0 : h.lv[l].b; }
  dim3 grid(const MgLevel& Lv) const { return stencil_grid(Lv.nx, Lv.ny, Lv.nz, h.S, DIM); }
  dim3 block() const { return stencil_block(DIM); }

  // device-looped solve graph being captured (mg_solve_graph): decisions also drive the WHILE node
  bool loop = false;
  cudaGraphConditionalHandle loop_handle{};
  unsigned long long loop_cycle_kernels = 0;

  // per-species decision of the oracle's loop on the reduced norms (enables the rest of the cycle)
  void update(int count = 1) {
    hook->before(kKMgNorm, s);
    if (loop)
      k_mg_update_loop<<<1, 32, 0, s>>>(h.S, d.mg_tol, d.mg_max_cycles, h.d_active, h.d_cycles, h.d_bmax, h.d_rmax,
                                        h.d_flag, st, h.d_tag, loop_handle, loop_cycle_kernels);
    else
      k_mg_update<<<1, 32, 0, s>>>(h.S, d.mg_tol, d.mg_max_cycles, h.d_active, h.d_cycles, h.d_bmax, h.d_rmax,
                                   h.d_flag, st, h.d_tag, count);
    hook->after(kKMgNorm, s, 0.0);
  }

  // The predicted last check of a solve without the sweep fused to it: ||b - A x||_inf of the
  // level-0 iterate (reads x and b, writes nothing; the fused form also writes a sweep that a
  // converged species discards), then the decision without counting a cycle.
  void check_only() {
    MgLevel& Lv = h.lv[0];
    const bool pair = DIM == 3 && tile3d_ok(Lv.ncell) && Lv.nx % 2 == 0 && mg_pair_enabled();
    const bool rows2 = DIM == 2 && Lv.nx % 2 == 0 && Lv.nx >= 64 && tile3d_ok(Lv.ncell) && mg_rows_enabled();
    TmaMaps maps;
    const bool tma = pair && tma_grid_ok(Lv.nx, Lv.ny, Lv.nz, Lv.ncell) && mg_tma_enabled() &&
                     tma_maps(maps, Lv.x, b0, Lv.nx, Lv.ny, Lv.nz * h.S);
    hook->before(kKMgSmooth, s);
    if (rows2) {
      const int ch = rows_chunk(Lv.ncell, h.S);
      k_mg2_rows<false, true, false><<<rows_grid(Lv.nx, Lv.ny, h.S, ch), kRowWarps * 32, kRowSmem, s>>>(
          C[0], Lv.x, b0, nullptr, Lv.nx, Lv.ny, ch, h.d_active, h.d_rmax, nullptr);
    } else if (tma) {
      k_mg3_tma<false, true, false><<<tile3d_pair_grid(Lv.nx, Lv.ny, Lv.nz, h.S), dim3(kTX, kTY), kTmaSmem, s>>>(
          C[0], maps, nullptr, Lv.nx, Lv.ny, Lv.nz, kZChunk, h.d_active, h.d_rmax, nullptr);
    } else if (pair) {
      k_mg3_pair<false, true, false><<<tile3d_pair_grid(Lv.nx, Lv.ny, Lv.nz, h.S), dim3(kTX, kTY), kMgPairSmem, s>>>(
          C[0], Lv.x, b0, nullptr, Lv.nx, Lv.ny, Lv.nz, kZChunk, h.d_active, h.d_rmax, nullptr);
    } else if (DIM == 3 && tile3d_ok(Lv.ncell)) {
      k_mg3_tiled<false, true, false><<<tile3d_grid(Lv.nx, Lv.ny, Lv.nz, h.S), dim3(kTX, kTY), 0, s>>>(
          C[0], Lv.x, b0, nullptr, Lv.nx, Lv.ny, Lv.nz, kZChunk, h.d_active, h.d_rmax, nullptr);
    } else {
      const dim3 rb = block();
      const dim3 rg((Lv.nx + rb.x - 1) / rb.x, (Lv.ny + rb.y - 1) / rb.y, h.S);
      k_mg_resmax<DIM><<<rg, rb, 0, s>>>(C[0], Lv.x, b0, Lv.nx, Lv.ny, Lv.nz, h.d_active, h.d_rmax, nullptr);
    }
    hook->after(kKMgSmooth, s, 0.0);
    update(0);
  }

  void smooth(int l, bool from_zero) {
    MgLevel& Lv = h.lv[l];
    const double* xin = (l == 0 && first_x) ? first_x : Lv.x;
    if (l == 0) first_x = nullptr;
    const bool chk = l == 0 && check_next;
    const bool bm = chk && first_check;  // the solve's first check: x is b (the BMAX kernels read b from the x tile)
    const bool tiled = DIM == 3 && !from_zero && tile3d_ok(Lv.ncell);
    const bool pair = tiled && Lv.nx % 2 == 0 && mg_pair_enabled();
    const double n8 = 8.0 * Lv.ncell * h.S;
    TmaMaps maps;
    hook->before(kKMgSmooth, s);  // a checking sweep is still a sweep (its norm is a by-product)
    const bool rows2 = DIM == 2 && !from_zero && Lv.nx % 2 == 0 && Lv.nx >= 64 && tile3d_ok(Lv.ncell) &&
                       mg_rows_enabled();
    if (rows2) {
      const int ch = rows_chunk(Lv.ncell, h.S);
      const dim3 rg = rows_grid(Lv.nx, Lv.ny, h.S, ch);
      if (bm)
        k_mg2_rows<true, true, true><<<rg, kRowWarps * 32, kRowSmem, s>>>(C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, ch,
                                                                            h.d_active, h.d_rmax, h.d_bmax);
      else if (chk)
        k_mg2_rows<true, true, false><<<rg, kRowWarps * 32, kRowSmem, s>>>(C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, ch,
                                                                             h.d_active, h.d_rmax, nullptr);
      else
        k_mg2_rows<true, false, false><<<rg, kRowWarps * 32, kRowSmem, s>>>(C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, ch,
                                                                              h.d_active, nullptr, nullptr);
    } else if (pair && tma_grid_ok(Lv.nx, Lv.ny, Lv.nz, Lv.ncell) && mg_tma_enabled() &&
               tma_maps(maps, xin, bof(l), Lv.nx, Lv.ny, Lv.nz * h.S)) {
      const dim3 pg = tile3d_pair_grid(Lv.nx, Lv.ny, Lv.nz, h.S);
      const size_t sm = kTmaSmem;
      if (bm)
        k_mg3_tma<true, true, true><<<pg, dim3(kTX, kTY), sm, s>>>(C[l], maps, Lv.t, Lv.nx, Lv.ny, Lv.nz, kZChunk,
                                                                    h.d_active, h.d_rmax, h.d_bmax);
      else if (chk)
        k_mg3_tma<true, true, false><<<pg, dim3(kTX, kTY), sm, s>>>(C[l], maps, Lv.t, Lv.nx, Lv.ny, Lv.nz, kZChunk,
                                                                     h.d_active, h.d_rmax, nullptr);
      else
        k_mg3_tma<true, false, false><<<pg, dim3(kTX, kTY), sm, s>>>(C[l], maps, Lv.t, Lv.nx, Lv.ny, Lv.nz, kZChunk,
                                                                      h.d_active, nullptr, nullptr);
    } else if (pair) {
      const dim3 pg = tile3d_pair_grid(Lv.nx, Lv.ny, Lv.nz, h.S);
      const size_t sm = kMgPairSmem;
      if (bm)
        k_mg3_pair<true, true, true><<<pg, dim3(kTX, kTY), sm, s>>>(C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, Lv.nz,
                                                                     kZChunk, h.d_active, h.d_rmax, h.d_bmax);
      else if (chk)
        k_mg3_pair<true, true, false><<<pg, dim3(kTX, kTY), sm, s>>>(C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, Lv.nz,
                                                                      kZChunk, h.d_active, h.d_rmax, nullptr);
      else
        k_mg3_pair<true, false, false><<<pg, dim3(kTX, kTY), sm, s>>>(C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, Lv.nz,
                                                                       kZChunk, h.d_active, nullptr, nullptr);
    } else if (tiled && bm)
      k_mg3_tiled<true, true, true><<<tile3d_grid(Lv.nx, Lv.ny, Lv.nz, h.S), dim3(kTX, kTY), 0, s>>>(
          C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, Lv.nz, kZChunk, h.d_active, h.d_rmax, h.d_bmax);
    else if (tiled && chk)
      k_mg3_tiled<true, true, false><<<tile3d_grid(Lv.nx, Lv.ny, Lv.nz, h.S), dim3(kTX, kTY), 0, s>>>(
          C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, Lv.nz, kZChunk, h.d_active, h.d_rmax, nullptr);
    else if (tiled)
      k_mg3_tiled<true, false, false><<<tile3d_grid(Lv.nx, Lv.ny, Lv.nz, h.S), dim3(kTX, kTY), 0, s>>>(
          C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, Lv.nz, kZChunk, h.d_active, nullptr, nullptr);
    else if (bm)
      k_mg_smooth<DIM, true, true><<<grid(Lv), block(), 0, s>>>(C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, Lv.nz, 0,
                                                                 h.d_active, h.d_rmax, h.d_bmax);
    else if (chk)
      k_mg_smooth<DIM, true, false><<<grid(Lv), block(), 0, s>>>(C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, Lv.nz, 0,
                                                                  h.d_active, h.d_rmax, nullptr);
    else
      k_mg_smooth<DIM><<<grid(Lv), block(), 0, s>>>(C[l], xin, bof(l), Lv.t, Lv.nx, Lv.ny, Lv.nz, from_zero ? 1 : 0,
                                                    h.d_active);
    hook->after(kKMgSmooth, s, 0.0);
    charge(kKMgSmooth, n8 * (from_zero ? 2 : 3), chk);
    std::swap(Lv.x, Lv.t);
    if (chk) {
      check_next = false;
      first_check = false;
      update();
    }
  }
  int lc = kMgMaxLevels;  // first level handled by k_mg_coarse (levels of <= kMgCoarseCells cells)
  void vcycle(int l) {
    MgLevel& Lv = h.lv[l];
    if (l >= 1 && l >= lc) {  // the rest of the cycle in one launch
      MgCoarseArgs A{};
      A.lc = l;
      A.L = L;
      A.pre = d.mg_pre;
      A.post = d.mg_post;
      A.coarse = d.mg_coarse_sweeps;
      for (int q = l; q < L; ++q) {
        A.nx[q] = h.lv[q].nx;
        A.ny[q] = h.lv[q].ny;
        A.nz[q] = h.lv[q].nz;
        A.x[q] = h.lv[q].x;
        A.t[q] = h.lv[q].t;
        A.b[q] = h.lv[q].b;
        A.C[q] = C[q];
      }
      A.active = h.d_active;
      hook->before(kKMgSmooth, s);
      k_mg_coarse<DIM><<<h.S, kMgCoarseThreads, 0, s>>>(A);
      hook->after(kKMgSmooth, s, 0.0);
      return;
    }
    if (l == L - 1) {
      const int ns = L == 1 ? d.mg_pre : d.mg_coarse_sweeps;
      for (int it = 0; it < ns; ++it) smooth(l, l > 0 && it == 0);
      return;
    }
    for (int it = 0; it < d.mg_pre; ++it) smooth(l, l > 0 && it == 0);
    MgLevel& Cl = h.lv[l + 1];
    hook->before(kKMgRestrict, s);
    if (DIM == 2 && Lv.nx % 2 == 0 && tile3d_ok(Lv.ncell) && mg_pair_prolong())
      k_mg_restrict2_pair<<<dim3((unsigned)((Cl.nx + 31) / 32), (unsigned)((Cl.ny + 7) / 8), (unsigned)h.S),
                            dim3(32, 8), 0, s>>>(C[l], Lv.x, bof(l), Lv.nx, Lv.ny, Cl.b, Cl.nx, Cl.ny, h.d_active);
    else
      k_mg_restrict<DIM><<<grid(Cl), block(), 0, s>>>(C[l], Lv.x, bof(l), Lv.nx, Lv.ny, Lv.nz, Cl.b, Cl.nx, Cl.ny,
                                                        Cl.nz, h.d_active);
    hook->after(kKMgRestrict, s, 0.0);
    charge(kKMgRestrict, 8.0 * h.S * (2.0 * Lv.ncell + Cl.ncell), false);
    vcycle(l + 1);
    hook->before(kKMgProlong, s);
    if (DIM >= 2 && Lv.nx % 2 == 0 && tile3d_ok(Lv.ncell) && mg_pair_prolong())
      k_mg_prolong_pair<DIM><<<dim3((unsigned)((Lv.nx / 2 + 31) / 32), (unsigned)((Lv.ny + 7) / 8),
                                    (unsigned)(Lv.nz * h.S)),
                               dim3(32, 8), 0, s>>>(Lv.x, Lv.nx, Lv.ny, Lv.nz, Cl.x, Cl.nx, Cl.ny, Cl.nz, h.d_active);
    else
      k_mg_prolong<DIM><<<grid(Lv), block(), 0, s>>>(Lv.x, Lv.nx, Lv.ny, Lv.nz, Cl.x, Cl.nx, Cl.ny, Cl.nz,
                                                     h.d_active);
    hook->after(kKMgProlong, s, 0.0);
    charge(kKMgProlong, 8.0 * h.S * (2.0 * Lv.ncell + Cl.ncell), false);
    for (int it = 0; it < d.mg_post; ++it) smooth(l, false);
  }
};

inline bool graphs_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("CISDC_MG_GRAPHS");
    return !(e && e[0] == '0');
  }();
  return v;
}

// The cached graph of one checking V-cycle (cycles >= 1 of a solve) for (coef, rhs, out, L); built
// by capturing R.vcycle(0) on the stream.  nullptr if capture is unavailable (the caller then
// launches the cycle directly).
template <int DIM>
inline MgHierarchy::CycleGraph* cycle_graph(MgHierarchy& h, MgRunner<DIM>& R, double coef, const double* rhs,
                                            const double* out, cudaStream_t s) {
  for (auto& g : h.graphs)
    if (g.coef == coef && g.rhs == rhs && g.out == out && g.L == R.L) return &g;
  CountingHook counter;
  LaunchHook* saved = R.hook;
  R.hook = &counter;
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    R.hook = saved;
    return nullptr;
  }
  R.check_next = true;
  R.recording = false;
  R.vcycle(0);
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(s, &graph);
  R.hook = saved;
  if (e != cudaSuccess || !graph) return nullptr;
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) return nullptr;
  if (h.graphs.size() >= 64) {
    cudaGraphExecDestroy(h.graphs.front().exec);
    h.graphs.erase(h.graphs.begin());
  }
  h.graphs.push_back({coef, rhs, out, R.L, exec, counter.n});
  return &h.graphs.back();
}

// Device-side convergence loops for fused-check solves (CISDC_MG_LOOP=1).  Off by default: measured
// on B200 (profiles/r2/r2d_*), the loop removes the per-solve host wait but gives up the predicted
// residual-only last check (a WHILE body cannot know which check is the last), and the host wait
// was already hidden behind the batches it enqueues: C5 549.4 -> 552.6 ms per step, C4 117.7 ->
// 119.7, C3 35.61 -> 35.57.  It is the form a graph-captured sweep needs (no host decision inside).
inline bool mg_loop_enabled() {  // read per solve, so a process can switch it (tests do)
  const char* e = std::getenv("CISDC_MG_LOOP");
  return e && e[0] == '1';
}

// The whole solve as one graph, cached per (coef, rhs, out, L): the first cycle (check of x = b and
// ||b||, sweeps from b), a WHILE node whose body is one checking cycle -- its decision kernel
// (k_mg_update_loop) sets the condition to the host loop's "go on" test -- and the copy of b for
// species that met the tolerance at x = b.  The host enqueues k_mg_begin + one graph launch and
// never waits: no per-solve synchronisation, and the cycle count is whatever the device decides
// (the oracle's loop exactly; the cap is the decision kernel's).  R must be in its pre-solve state
// (level-0 x = out, first_x = rhs); the capture launches nothing.  nullptr if capture fails.
template <int DIM>
inline MgHierarchy::SolveGraph* mg_solve_graph(MgHierarchy& h, MgRunner<DIM>& R, const Geom& g, double coef,
                                               const double* rhs, double* out, cudaStream_t s) {
  for (auto& e : h.solve_graphs)
    if (e.coef == coef && e.rhs == rhs && e.out == out && e.L == R.L) return &e;
  CountingHook counter;
  LaunchHook* saved = R.hook;
  R.hook = &counter;
  auto reset = [&]() {
    R.first_x = rhs;
    R.check_next = true;
    R.first_check = true;
    R.recording = false;
  };
  // kernels of one cycle (a throwaway capture of the same launch sequence)
  reset();
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    R.hook = saved;
    return nullptr;
  }
  R.vcycle(0);
  cudaGraph_t tmp = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &tmp);
  if (tmp) cudaGraphDestroy(tmp);
  const long long per_cycle = counter.n;
  cudaGraph_t graph = nullptr;
  cudaGraphConditionalHandle hnd{};
  bool ok = e == cudaSuccess && cudaGraphCreate(&graph, 0) == cudaSuccess &&
            cudaGraphConditionalHandleCreate(&hnd, graph, 0, cudaGraphCondAssignDefault) == cudaSuccess;
  if (ok) ok = cudaStreamBeginCaptureToGraph(s, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
               cudaSuccess;
  if (ok) {
    reset();
    R.loop = true;
    R.loop_handle = hnd;
    R.loop_cycle_kernels = (unsigned long long)per_cycle;
    R.vcycle(0);  // the first cycle
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    cudaGraph_t cg = nullptr;
    cudaGraphNode_t wnode = nullptr;
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = hnd;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    ok = cudaStreamGetCaptureInfo(s, &cs, nullptr, &cg, &deps, &nd) == cudaSuccess &&
         cudaGraphAddNode(&wnode, cg, deps, nd, &p) == cudaSuccess;
    if (ok) {  // the body: one checking cycle, captured on the body stream
      const cudaStream_t s_saved = R.s;
      R.s = h.s_body;
      ok = cudaStreamBeginCaptureToGraph(h.s_body, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal) == cudaSuccess;
      if (ok) {
        R.check_next = true;
        R.vcycle(0);
        cudaGraph_t bg = nullptr;
        ok = cudaStreamEndCapture(h.s_body, &bg) == cudaSuccess;
      }
      R.s = s_saved;
      ok = ok && cudaStreamUpdateCaptureDependencies(s, &wnode, 1, cudaStreamSetCaptureDependencies) == cudaSuccess;
    }
    // species that met the tolerance at x = b: out = b (the kernel reads the cycle counts)
    const dim3 cgrid((unsigned)std::min<long long>((g.ncell + 255) / 256, 4096), (unsigned)g.S, 1);
    k_mg_copy_unswept<<<cgrid, 256, 0, s>>>(rhs, out, g.ncell, h.d_cycles);
    cudaGraph_t done = nullptr;
    ok = (cudaStreamEndCapture(s, &done) == cudaSuccess) && ok && done == graph;
  }
  R.loop = false;
  R.hook = saved;
  cudaGraphExec_t exec = nullptr;
  if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
  if (graph) cudaGraphDestroy(graph);
  cudaGetLastError();
  if (!ok) return nullptr;
  if (h.solve_graphs.size() >= 64) {
    cudaGraphExecDestroy(h.solve_graphs.front().exec);
    h.solve_graphs.erase(h.solve_graphs.begin());
  }
  h.solve_graphs.push_back({coef, rhs, out, R.L, exec, per_cycle + 1});
  return &h.solve_graphs.back();
}

// The oracle's loop per species: x = b; while (||b - A x|| > tol ||b||) { cap check; V-cycle }.
// Device form: every enqueued V-cycle starts with a level-0 sweep that also reduces the residual
// norm of its input iterate (k_mg3_tiled<.., NORM> / k_mg_smooth<.., NORM>), followed by the
// decision kernel; a species found converged is masked out for the rest of the cycle and keeps
// its iterate (the sweep wrote the ping-pong partner, which an even sweep count never hands back).
// So n real cycles cost n + 1 enqueued cycles, the last one a masked no-op after its first sweep.
// The host enqueues cycles in batches (predicted from the last solve with this coefficient) and
// only then reads the device flag.  Without a level-0 pre-sweep (mg_pre == 0) the check is a
// separate residual-norm pass.
template <int DIM>
inline int mg_solve_dim(MgHierarchy& h, const Geom& g, const cisdc_problem_desc& d, double coef, const double* rhs,
                        double* out, DevStatus* st, unsigned tag, cudaStream_t s, LaunchHook* hook) {
  const long long n = g.n;
  if (coef == 0.0) {
    if (cudaMemcpyAsync(out, rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return CISDC_E_CUDA;
    return CISDC_OK;
  }
  MgRunner<DIM> R{h, d, {}, 1, s, hook, rhs};
  R.st = st;
  R.L = mg_plan(h, d, coef, R.C);
  if (mg_coarse_enabled())
    for (int l = 1; l + 1 < R.L; ++l)  // only when it replaces at least two levels
      if (h.lv[l].ncell <= kMgCoarseCells) {
        R.lc = l;
        break;
      }
  hook->before(kKMgNorm, s);
  k_mg_begin<<<1, 32, 0, s>>>(g.S, h.d_active, h.d_cycles, h.d_bmax, h.d_rmax, h.d_flag, h.d_tag, tag);
  hook->after(kKMgNorm, s, 0.0);
  // Level 0 iterates directly in `out` (ping-pong with the level-0 workspace; even sweep counts
  // leave the iterate in `out`), and the initial iterate x = b is read straight from the rhs:
  // no copy in, no copy out.
  MgLevel& L0 = h.lv[0];
  double* own_x = L0.x;
  double* own_t = L0.t;
  L0.x = out;
  R.first_x = rhs;
  const bool fused = d.mg_pre >= 1;
  const double* x_check = rhs;  // separate-check path: the first check sees x = b
  auto check = [&]() {
    hook->before(kKMgNorm, s);
    const dim3 rb = R.block();
    const dim3 rg((L0.nx + rb.x - 1) / rb.x, (L0.ny + rb.y - 1) / rb.y, g.S);
    double* bmax = x_check == rhs ? h.d_bmax : nullptr;
    if (DIM == 3 && tile3d_ok(L0.ncell) && bmax)
      k_mg3_tiled<false, true, true><<<tile3d_grid(L0.nx, L0.ny, L0.nz, g.S), dim3(kTX, kTY), 0, s>>>(
          R.C[0], x_check, rhs, nullptr, L0.nx, L0.ny, L0.nz, kZChunk, h.d_active, h.d_rmax, bmax);
    else if (DIM == 3 && tile3d_ok(L0.ncell))
      k_mg3_tiled<false, true, false><<<tile3d_grid(L0.nx, L0.ny, L0.nz, g.S), dim3(kTX, kTY), 0, s>>>(
          R.C[0], x_check, rhs, nullptr, L0.nx, L0.ny, L0.nz, kZChunk, h.d_active, h.d_rmax, nullptr);
    else
      k_mg_resmax<DIM><<<rg, rb, 0, s>>>(R.C[0], x_check, rhs, L0.nx, L0.ny, L0.nz, h.d_active, h.d_rmax, bmax);
    hook->after(kKMgNorm, s, 0.0);
    if (R.recording || x_check == rhs) R.fs_bytes = (x_check == rhs ? 8.0 : 16.0) * n;
    x_check = L0.x;
    R.update();
  };
  if (fused && mg_loop_enabled() && !hook->timing()) {
    MgHierarchy::SolveGraph* sg = mg_solve_graph<DIM>(h, R, g, coef, rhs, out, s);
    if (sg) {
      if (cudaGraphLaunch(sg->exec, s) != cudaSuccess) return CISDC_E_CUDA;
      hook->add_launches(sg->kernels);
      L0.x = own_x;
      L0.t = own_t;
      return cudaGetLastError() == cudaSuccess ? CISDC_OK : CISDC_E_CUDA;
    }
    R.first_x = rhs;  // capture unavailable: the host-driven loop below
    R.check_next = false;
    R.first_check = true;
  }
  int batch = 1;
  for (const auto& pc : h.predicted)
    if (pc.first == coef) batch = std::max(1, pc.second);
  int launched = 0;   // V-cycles enqueued
  int chk_only = -1;  // real cycles enqueued before the check-only pass (-1: none)
  if (fused) {
    // cycle i checks x_{i-1} first: n real cycles need n + 1 enqueued ones.  Cycles after the first
    // replay a captured graph of the cycle (same kernels, same pointers: the sweep counts per level
    // are even, so the ping-pong pointers are back in place after every cycle).
    batch += 1;
    const bool use_graph = !hook->timing() && graphs_enabled();
    MgHierarchy::CycleGraph* cg = nullptr;
    bool first_batch = true;
    for (;;) {
      for (int b = 0; b < batch && launched <= d.mg_max_cycles; ++b, ++launched) {
        if (first_batch && b == batch - 1 && b >= 1 && mg_check_only_enabled()) {
          // the predicted convergence check: residual only (a misprediction costs this pass; the
          // next cycle's fused check repeats the decision)
          R.check_only();
          chk_only = b;
          --launched;  // not a V-cycle: the cap counts real cycles only (the (N+1)-th fused check
                       // must still test x_N and flag the cap)
          continue;
        }
        if (launched >= 1 && use_graph) {
          if (!cg) cg = cycle_graph(h, R, coef, rhs, out, s);
          if (cg) {
            if (cudaGraphLaunch(cg->exec, s) != cudaSuccess) return CISDC_E_CUDA;
            hook->add_launches(cg->kernels);
            continue;
          }
        }
        R.check_next = true;
        R.recording = launched == 0;
        R.vcycle(0);
        R.recording = false;
      }
      cudaMemcpyAsync(h.h_flag, h.d_flag, sizeof(int) * 2, cudaMemcpyDeviceToHost, s);
      if (cudaStreamSynchronize(s) != cudaSuccess) return CISDC_E_CUDA;
      if (!h.h_flag[0] || h.h_flag[1] || launched > d.mg_max_cycles) break;
      batch = 1;
      first_batch = false;
    }
  } else {
    check();
    for (;;) {
      for (int b = 0; b < batch && launched < d.mg_max_cycles; ++b, ++launched) {
        R.recording = launched == 0;
        R.vcycle(0);
        check();
        R.recording = false;
      }
      cudaMemcpyAsync(h.h_flag, h.d_flag, sizeof(int) * 2, cudaMemcpyDeviceToHost, s);
      if (cudaStreamSynchronize(s) != cudaSuccess) return CISDC_E_CUDA;
      if (!h.h_flag[0] || h.h_flag[1] || launched >= d.mg_max_cycles) break;
      batch = 1;
    }
  }
  // remember how many cycles this coefficient needed (flag[0] == 0 after the last check)
  bool any_unswept = false;
  {
    std::vector<int> cyc(g.S);
    cudaMemcpy(cyc.data(), h.d_cycles, sizeof(int) * g.S, cudaMemcpyDeviceToHost);
    int used = 0;
    for (int v : cyc) used = std::max(used, v);
    // exact compulsory bytes: species s ran c_s full cycles and c_s + 1 checks; unswept species
    // are copied (2 fields of one species)
    double checks = 0.0, cycles = 0.0, unswept = 0.0;
    for (int v : cyc) {
      checks += v + 1;
      cycles += v;
      unswept += v == 0;
      any_unswept = any_unswept || v == 0;
    }
    const double per = 1.0 / g.S;
    if (fused) {
      // the first check sweeps x = b (rhs read once + the partner written), later ones 3 fields;
      // the check-only pass (after P = chk_only cycles) reads 2 fields: a species that stopped
      // there saved one field, one that went on paid it on top
      double fields = 0.0;
      for (int v : cyc) {
        fields += 2.0 + 3.0 * v;
        if (chk_only >= 1 && v == chk_only) fields -= 1.0;
        if (chk_only >= 1 && v > chk_only) fields += 2.0;
      }
      hook->add_bytes(kKMgSmooth, 8.0 * (double)g.ncell * fields);
    } else {
      hook->add_bytes(kKMgNorm, (8.0 * n * g.S + 16.0 * n * cycles) * per);
    }
    (void)checks;
    for (int c = 0; c < kNumKernelClasses; ++c)
      if (R.rest_bytes[c] > 0.0) hook->add_bytes(c, R.rest_bytes[c] * cycles * per);
    hook->add_bytes(kKMgNorm, 16.0 * (double)g.ncell * unswept);
    used = std::max(used, 1);
    bool found = false;
    for (auto& pc : h.predicted)
      if (pc.first == coef) {
        pc.second = used;
        found = true;
      }
    if (!found) {
      if (h.predicted.size() >= 64) h.predicted.erase(h.predicted.begin());
      h.predicted.push_back({coef, used});
    }
  }
  const bool in_out = L0.x == out;
  L0.x = own_x;
  L0.t = own_t;
  if (!in_out) return CISDC_E_CUDA;  // unreachable with even sweep counts
  // species that met the tolerance at x = b never had a sweep write `out` (the host read the cycle
  // counts above, so the copy is launched only when there is one)
  if (any_unswept) {
    const dim3 cg((unsigned)std::min<long long>((g.ncell + 255) / 256, 4096), (unsigned)g.S, 1);
    hook->before(kKMgNorm, s);
    k_mg_copy_unswept<<<cg, 256, 0, s>>>(rhs, out, g.ncell, h.d_cycles);
    hook->after(kKMgNorm, s, 0.0);
  }
  if (cudaGetLastError() != cudaSuccess) return CISDC_E_CUDA;
  return CISDC_OK;
}

inline int mg_solve(MgHierarchy& h, const Geom& g, const cisdc_problem_desc& d, double coef, const double* rhs,
                    double* out, DevStatus* st, unsigned tag, cudaStream_t s, LaunchHook* hook) {
  switch (g.ndim) {
    case 1: return mg_solve_dim<1>(h, g, d, coef, rhs, out, st, tag, s, hook);
    case 2: return mg_solve_dim<2>(h, g, d, coef, rhs, out, st, tag, s, hook);
    default: return mg_solve_dim<3>(h, g, d, coef, rhs, out, st, tag, s, hook);
  }
}

}  // namespace cisdc_b200
