// K3 (1-D): implicit diffusion solve (I - coef F_D) phi = rhs.
//
// Periodic 1-D (configs 1-2).  With the reference's 4th-order stencil the system is cyclic
// pentadiagonal and, for constant coefficients, circulant:
//     A = (1+30c) I - 16c (Z + Z^-1) + c (Z^2 + Z^-2),    c = coef * d / (12 h^2),
// Z the cyclic shift.  It factors EXACTLY as A = K * P(Z) * P(Z^-1) with P(z) = 1 - p z + q z^2,
// both roots of P outside the unit circle (host: cisdc_b200::factor_circulant).  The direct solve
// is therefore two periodic second-order linear recurrences (a forward and a backward bidiagonal
// pair) and a scale -- the "batched tri/bidiagonal" direct-solver family of the reference's
// banded LU (proj/core/src/linalg.cpp:105-155), without its O(n) serial dependency chain.
//
// Each recurrence is evaluated as a parallel scan of 2x2 affine maps over ONE thread-block
// cluster (up to 8 CTAs x 1024 threads x E elements): per-thread local recurrence -> CTA scan
// (shared memory) -> cluster scan through distributed shared memory (DSMEM) -> periodic closure
// s_{-1} = (I - T^N)^{-1} c_N -> per-thread re-run of the recurrence from its exact incoming
// state.  The field is read once and written once; everything else stays on chip.
//
// Reference Dirichlet problem (config-0 gate): assemble_diffusion_system + banded_solve of
// proj/core/src/problems/reaction_diffusion.cpp:127-164 executed verbatim by one thread
// (bit-identical to the reference; the gate is n_x <= a few thousand).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace cisdc_b200 {

namespace cg = cooperative_groups;

struct Circ {
  int npass;
  double p[4], q[4];
  int reverse[4];
  int kind[4];  // 0: second-order (p, q); 1: two coupled first-order (zeta1 = p, zeta2 = q)
  double invK;
};

struct Solve1dArgs {
  const double* rhs;
  double* out;
  int N;
  int active[kMaxS];  // 0: coef == 0 or d == 0 -> identity (copy)
  Circ c[kMaxS];
};

struct Aff {  // s -> A s + c on the state (u_i, u_{i-1})
  double a00, a01, a10, a11, c0, c1;
};

__device__ __forceinline__ Aff aff_identity() { return {1.0, 0.0, 0.0, 1.0, 0.0, 0.0}; }

// later o earlier
__device__ __forceinline__ Aff aff_then(const Aff& later, const Aff& earlier) {
  Aff r;
  r.a00 = later.a00 * earlier.a00 + later.a01 * earlier.a10;
  r.a01 = later.a00 * earlier.a01 + later.a01 * earlier.a11;
  r.a10 = later.a10 * earlier.a00 + later.a11 * earlier.a10;
  r.a11 = later.a10 * earlier.a01 + later.a11 * earlier.a11;
  r.c0 = later.a00 * earlier.c0 + later.a01 * earlier.c1 + later.c0;
  r.c1 = later.a10 * earlier.c0 + later.a11 * earlier.c1 + later.c1;
  return r;
}

template <int T>
struct Solve1dSmem {
  Aff wtot[T / 32];   // warp totals (visiting order)
  Aff wincl[T / 32];  // their inclusive scan
  Aff peer[16];       // CTA totals of the cluster, by rank
  Aff total[4];       // per pass: this CTA's total map (read by the cluster peers through DSMEM)
};

__device__ __forceinline__ double shfl_dir(double v, int delta, bool down) {
  return down ? __shfl_down_sync(0xffffffffu, v, delta) : __shfl_up_sync(0xffffffffu, v, delta);
}
__device__ __forceinline__ Aff shfl_aff(const Aff& m, int delta, bool down) {
  return {shfl_dir(m.a00, delta, down), shfl_dir(m.a01, delta, down), shfl_dir(m.a10, delta, down),
          shfl_dir(m.a11, delta, down), shfl_dir(m.c0, delta, down),  shfl_dir(m.c1, delta, down)};
}

// One step of a pass's recurrence on the state (s0, s1); returns the element's new value.
//   kind 0 (second order):        u = (x + p s0) - q s1;           state (u_i, u_{i-1})
//   kind 1 (two coupled 1st order): u = x + p s0; v = u + q s1;   state (u_i, v_i), output v
__device__ __forceinline__ double rec_step(int kind, double x, double p, double q, double& s0, double& s1) {
  if (kind == 0) {
    const double un = (x + p * s0) - q * s1;
    s1 = s0;
    s0 = un;
    return un;
  }
  const double u = x + p * s0;
  const double v = u + q * s1;
  s0 = u;
  s1 = v;
  return v;
}

// One pass of a periodic recurrence over the cluster's elements in visiting order (reverse = from
// the last element down).  Scan of 2x2 affine maps: thread-local chain -> warp Kogge-Stone scan
// (shuffles) -> scan of the warp totals -> cluster prefix from the CTA totals (DSMEM) -> periodic
// closure s_{-1} = (I - A_N)^{-1} c_N -> re-run of the chain from the exact incoming state.
// oracle/co_problems.c (scan_pass) emulates this evaluation order exactly.
template <int E, int T, bool reverse>
__device__ __forceinline__ void periodic_pass(double (&u)[E], int len, int kind, double p, double q,
                                              Solve1dSmem<T>& sm, int pass, cg::cluster_group& cluster,
                                              int cl_size) {
  constexpr int NW = T / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lp = reverse ? 31 - lane : lane;
  const int wp = reverse ? NW - 1 - warp : warp;
  const int my_rank = static_cast<int>(cluster.block_rank());
  const int vrank = reverse ? (cl_size - 1 - my_rank) : my_rank;
  // local map with zero incoming state (element index t is a compile-time constant in both
  // directions, so u[] stays in registers)
  Aff m;
  {
    double s0 = 0.0, s1 = 0.0;
    double a00 = 1.0, a01 = 0.0, a10 = 0.0, a11 = 1.0;
#pragma unroll
    for (int tt = 0; tt < E; ++tt) {
      const int t = reverse ? (E - 1 - tt) : tt;
      if (t < len) {
        rec_step(kind, u[t], p, q, s0, s1);
        double n00, n01, n10, n11;
        if (kind == 0) {  // A <- [[p, -q], [1, 0]] A
          n00 = p * a00 - q * a10;
          n01 = p * a01 - q * a11;
          n10 = a00;
          n11 = a01;
        } else {  // A <- [[p, 0], [p, q]] A
          n00 = p * a00;
          n01 = p * a01;
          n10 = p * a00 + q * a10;
          n11 = p * a01 + q * a11;
        }
        a00 = n00;
        a01 = n01;
        a10 = n10;
        a11 = n11;
      }
    }
    m = {a00, a01, a10, a11, s0, s1};
  }
  // warp inclusive scan over lane positions lp
  Aff incl = m;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Aff o = shfl_aff(incl, off, reverse);
    if (lp >= off) incl = aff_then(incl, o);
  }
  Aff excl_lane = shfl_aff(incl, 1, reverse);
  if (lp == 0) excl_lane = aff_identity();
  if (lp == 31) sm.wtot[wp] = incl;
  __syncthreads();
  if (warp == 0) {
    Aff w = lane < NW ? sm.wtot[lane] : aff_identity();
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const Aff o = shfl_aff(w, off, false);
      if (lane >= off) w = aff_then(w, o);
    }
    if (lane < NW) sm.wincl[lane] = w;
  }
  __syncthreads();
  const Aff wexcl = wp > 0 ? sm.wincl[wp - 1] : aff_identity();
  const Aff excl = aff_then(excl_lane, wexcl);
  if (cl_size == 1) {  // single CTA: no cluster barrier, no DSMEM
    if (tid == 0) sm.peer[0] = sm.wincl[NW - 1];
    __syncthreads();
  } else {
    if (tid == 0) sm.total[pass] = sm.wincl[NW - 1];
    cluster.sync();
    if (tid < cl_size) {
      Solve1dSmem<T>* peer = cluster.map_shared_rank(&sm, tid);
      sm.peer[tid] = peer->total[pass];
    }
    __syncthreads();
  }
  // cluster prefix (CTAs before me in visiting order) and global total
  Aff pre = aff_identity(), tot = aff_identity();
  for (int v = 0; v < cl_size; ++v) {
    const Aff tv = sm.peer[reverse ? (cl_size - 1 - v) : v];
    if (v < vrank) pre = aff_then(tv, pre);
    tot = aff_then(tv, tot);
  }
  // periodic closure: s = (I - A_N)^{-1} c_N
  const double m00 = 1.0 - tot.a00, m01 = -tot.a01, m10 = -tot.a10, m11 = 1.0 - tot.a11;
  const double det = m00 * m11 - m01 * m10;
  const double sa = (m11 * tot.c0 - m01 * tot.c1) / det;
  const double sb = (m00 * tot.c1 - m10 * tot.c0) / det;
  // incoming state of this CTA, then of this thread
  const double ca = pre.a00 * sa + pre.a01 * sb + pre.c0;
  const double cb = pre.a10 * sa + pre.a11 * sb + pre.c1;
  double s0 = excl.a00 * ca + excl.a01 * cb + excl.c0;
  double s1 = excl.a10 * ca + excl.a11 * cb + excl.c1;
#pragma unroll
  for (int tt = 0; tt < E; ++tt) {
    const int t = reverse ? (E - 1 - tt) : tt;
    if (t < len) u[t] = rec_step(kind, u[t], p, q, s0, s1);
  }
}

// grid: (cluster_size * nsys) CTAs of T threads; cluster dims (cluster_size, 1, 1); one cluster per
// species system (blockIdx.x / cluster_size).
template <int E, int T>
__global__ void __launch_bounds__(T) k_solve1d_periodic(const __grid_constant__ Solve1dArgs a) {
  __shared__ Solve1dSmem<T> sm;
  cg::cluster_group cluster = cg::this_cluster();
  const int cl_size = static_cast<int>(cluster.num_blocks());
  const int sys = blockIdx.x / cl_size;
  const int rank = static_cast<int>(cluster.block_rank());
  const int N = a.N;
  const double* b = a.rhs + (long long)sys * N;
  double* y = a.out + (long long)sys * N;
  const int a0 = (rank * T + threadIdx.x) * E;
  const int len = max(0, min(E, N - a0));
  if (!a.active[sys]) {  // coef == 0: copy (reaction_diffusion.cpp:159)
    for (int t = 0; t < len; ++t) y[a0 + t] = b[a0 + t];
    return;  // uniform over the cluster: no cluster.sync below is reached by any CTA
  }
  const Circ& c = a.c[sys];
  double u[E];
#pragma unroll
  for (int t = 0; t < E; ++t) u[t] = t < len ? b[a0 + t] : 0.0;
  for (int k = 0; k < c.npass; ++k)
    if (c.reverse[k]) periodic_pass<E, T, true>(u, len, c.kind[k], c.p[k], c.q[k], sm, k, cluster, cl_size);
    else periodic_pass<E, T, false>(u, len, c.kind[k], c.p[k], c.q[k], sm, k, cluster, cl_size);
#pragma unroll
  for (int t = 0; t < E; ++t)
    if (t < len) y[a0 + t] = u[t] * c.invK;
  if (cl_size > 1) cluster.sync();  // peers may still read this CTA's totals through DSMEM
}

// Reference Dirichlet system, one thread (bit-identical to assemble_diffusion_system + banded_solve)
struct RdSolveArgs {
  int n;
  double c;  // coef * d / (12 dx^2), host-computed like the reference
  double w[2][5];
  const double* rhs;
  double* out;
  double* work;  // n * 10 doubles
  unsigned tag;  // failure tag (DevStatus::fail_key)
};

__global__ void k_rd_banded_solve(RdSolveArgs a, DevStatus* st) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int n = a.n, kl = 3, ku = 3, width = 2 * kl + ku + 1;
  const double kLap[5] = {-1.0, 16.0, -30.0, 16.0, -1.0};
  double* w = a.work;
  double* x = a.out;
  for (long long i = 0; i < (long long)n * width; ++i) w[i] = 0.0;
  // banded_solve copies A (band kl=ku=3) into a working band of width 2kl+ku+1 (row-major)
#define W_(i, j) w[(long long)(i) * width + ((j) - (i) + kl)]
  for (int i = 0; i < n; ++i) {
    x[i] = a.rhs[i];
    W_(i, i) = 1.0;
  }
  for (int i = 0; i < n; ++i) {
    for (int o = -2; o <= 2; ++o) {
      const double s = -a.c * kLap[o + 2];
      const int j = i + o;
      if (j >= 0 && j < n) {
        W_(i, j) += s;
      } else if (j < 0) {
        const double* wg = a.w[-j - 1];
        for (int q = 0; q < 4; ++q) W_(i, q) += s * wg[q + 1];
        x[i] -= s * wg[0] * 1.0;
      } else {
        const double* wg = a.w[j - n];
        for (int q = 0; q < 4; ++q) W_(i, n - 1 - q) += s * wg[q + 1];
        x[i] -= s * wg[0] * 0.0;
      }
    }
  }
  for (int k = 0; k < n; ++k) {
    const int last = min(n - 1, k + kl);
    int p = k;
    double best = fabs(W_(k, k));
    for (int i = k + 1; i <= last; ++i) {
      if (fabs(W_(i, k)) > best) {
        best = fabs(W_(i, k));
        p = i;
      }
    }
    if (best == 0.0) {
      record_failure(st, a.tag, CISDC_E_SOLVE, (unsigned long long)k);
      return;
    }
    const int jmax = min(n - 1, k + kl + ku);
    if (p != k) {
      for (int j = k; j <= jmax; ++j) {
        const double t = W_(k, j);
        W_(k, j) = W_(p, j);
        W_(p, j) = t;
      }
      const double t = x[k];
      x[k] = x[p];
      x[p] = t;
    }
    const double pivot = W_(k, k);
    for (int i = k + 1; i <= last; ++i) {
      const double m = W_(i, k) / pivot;
      if (m != 0.0) {
        for (int j = k + 1; j <= jmax; ++j) W_(i, j) -= m * W_(k, j);
        x[i] -= m * x[k];
      }
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    const int jmax = min(n - 1, i + kl + ku);
    for (int j = i + 1; j <= jmax; ++j) s -= W_(i, j) * x[j];
    x[i] = s / W_(i, i);
  }
#undef W_
}

}  // namespace cisdc_b200
