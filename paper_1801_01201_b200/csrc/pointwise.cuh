// K2: spectral quadrature and sweep right-hand-side assembly, plus the increment norm (K5).
//
//  k_quad_base  -- quadrature_base (proj/core/src/integrators.cpp:52-65) for ALL M rows in one
//                  pass: per element the M+1 node sums s_j = (fa+fd+fr)_j are formed once in
//                  registers and contracted with the M x (M+1) matrix dt*Q (kernel parameter),
//                  i.e. the S.F / Q.F product as a per-cell small-matrix contraction, not M passes.
//  k_rhs        -- the stage right-hand sides of misdc_sweep (:86-87), misdcq_sweep (:115-122,
//                  :127-134) and run_diffusion_cell (:201-226) in the reference's operand order.
//  k_incr_*     -- increment_norm (proj/core/src/sweep_state.cpp:60-66): fixed-tree, run-to-run
//                  deterministic sum (differs from the serial sum by rounding only).
#pragma once

#include "common.cuh"
#include "rhs.cuh"

namespace cisdc_b200 {

struct QuadArgs {
  int M;
  double c[kMaxM][kMaxM + 1];  // dt * Q(m, j)
  const double* phi0;
  const double* fa[kMaxM + 1];
  const double* fd[kMaxM + 1];
  const double* fr[kMaxM + 1];
  double* base[kMaxM];  // base[0] may be null (no reader: fused into rhs0 below)
  // The first stage right-hand side of the sweep, which reads base row 0 and otherwise only fields
  // this pass loads anyway, assembled here (k_rhs's expression, same bits): rhs0_kind 1 =
  // misdcq_sweep m = 0 (base - fc*X), 2 = run_diffusion_cell m = 1 (base + (fc*(X - Y) - fc*Z)).
  int rhs0_kind;
  double fc;
  const double *X, *Y, *Z;
  double* rhs0;
};

__global__ void __launch_bounds__(256) k_quad_base(const __grid_constant__ QuadArgs q, long long n) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double s[kMaxM + 1];
#pragma unroll
  for (int j = 0; j <= kMaxM; ++j)
    if (j <= q.M) s[j] = q.fa[j][e] + q.fd[j][e] + q.fr[j][e];
  const double p0 = q.phi0[e];
  double acc0 = 0.0;
#pragma unroll
  for (int m = 0; m < kMaxM; ++m) {
    if (m >= q.M) break;
    double acc = p0;
#pragma unroll
    for (int j = 0; j <= kMaxM; ++j)
      if (j <= q.M) acc += q.c[m][j] * s[j];
    if (m == 0) acc0 = acc;
    if (q.base[m]) q.base[m][e] = acc;
  }
  if (q.rhs0_kind == 1) q.rhs0[e] = acc0 - q.fc * q.X[e];
  else if (q.rhs0_kind == 2) q.rhs0[e] = acc0 + (q.fc * (q.X[e] - q.Y[e]) - q.fc * q.Z[e]);
}

__global__ void __launch_bounds__(256) k_rhs(const __grid_constant__ RhsArgs a, long long n) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  if (a.kind == kRhsMisdc) {
    double base = a.phim[e];
#pragma unroll
    for (int j = 0; j <= kMaxM; ++j)
      if (j <= a.M) base += a.sc[j] * (a.sfa[j][e] + a.sfd[j][e] + a.sfr[j][e]);
    a.base_out[e] = base;
    a.out[e] = base + a.fc * (a.X[e] - a.Y[e] - a.Z[e]);
    return;
  }
  const bool tame = a.wild == nullptr || *a.wild == 0;
  const double base = a.base[e];
  if (a.kind == kRhsImexq) {  // the MISDCQ reaction-stage sum, then rhs -= coef * (fd_p + fr_p)
    double rr = base;
#pragma unroll
    for (int t = 0; t < kMaxM; ++t) {
      if (t >= a.nt) break;
      const RhsTerm& T = a.t[t];
      const double tI2 = T.cI * (T.D[e] - T.Dp[e] + T.R[e] - T.Rp[e]);
      rr += rhs_term_a(T, e, tI2, T.skipA && tame);
    }
    rr -= a.fc * (a.X[e] + a.Y[e]);
    a.out[e] = rr;
    return;
  }
  if (a.kind == kRhsMisdcq) {
    double rd = base, rr = base;
#pragma unroll
    for (int t = 0; t < kMaxM; ++t) {
      if (t >= a.nt) break;
      const RhsTerm& T = a.t[t];
      const bool skip = T.skipA && tame;
      const double dD = T.D[e] - T.Dp[e];
      const double tI = T.cI * dD;
      if (!a.out2) {
        rd += rhs_term_a(T, e, tI, skip);
        continue;
      }
      const double tI2 = T.cI * (dD + T.R[e] - T.Rp[e]);
      if (skip && tI != 0.0 && tI2 != 0.0) {
        rd += tI;
        rr += tI2;
      } else {
        const double cA = T.cE * (T.A[e] - T.Ap[e]);
        rd += cA + tI;
        rr += cA + tI2;
      }
    }
    rd -= a.fc * a.X[e];
    a.out[e] = rd;
    if (a.out2) a.out2[e] = rr;
    return;
  }
  // kRhsCisdcq
  double r = base;
#pragma unroll
  for (int t = 0; t < kMaxM; ++t) {
    if (t >= a.nt) break;
    const RhsTerm& T = a.t[t];
    double dDR;
    if (T.diff) {
      dDR = T.D[e];
    } else {
      dDR = T.D[e] - T.Dp[e] + T.R[e] - T.Rp[e];
      if (T.outDR) T.outDR[e] = dDR;
    }
    const double tI = T.cI * dDR;
    if (T.skipA && tame) {
      r += rhs_term_a(T, e, tI, true);
    } else {
      const double dA = (T.diff && T.dA) ? T.dA[e] : T.A[e] - T.Ap[e];
      if (!T.diff && T.outA) T.outA[e] = dA;
      r += T.cE * dA + tI;
    }
  }
  if (rhs_same_xy(a, tame)) r += a.fc * 0.0 - a.fc * a.Z[e];  // X - Y = +0.0 exactly (rhs.cuh)
  else r += a.fc * (a.X[e] - a.Y[e]) - a.fc * a.Z[e];
  a.out[e] = r;
}

// LinearScalarProblem (proj/core/src/problems/linear.cpp:19-50), per element of a batch of
// independent copies: F_A = a phi, F_D = d phi (either output may be null), and the exact stage
// solves out = rhs / denom with denom = 1 - coef * (d | r | d + r) formed and checked on the host.
__global__ void __launch_bounds__(256) k_lin_eval(const double* __restrict__ phi, double* __restrict__ fa,
                                                  double* __restrict__ fd, double a, double d, long long n,
                                                  int* wild) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const double v = phi[e];
  if (fa) {
    const double va = a * v;
    fa[e] = va;
    flag_wild(wild, wild_bits(va));  // F_A values k_rhs's exact-zero shortcut must not skip
  }
  if (fd) fd[e] = d * v;
}
__global__ void __launch_bounds__(256) k_lin_div(const double* __restrict__ rhs, double* __restrict__ out,
                                                 double denom, long long n) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) out[e] = rhs[e] / denom;
}

// Coupled stage of the periodic ADR class (cisdc_gpu.h): f <- rhs + coef * f, the stage right-hand
// side of the alternating iteration (no contraction: the oracle's a + c * b is a product, then a sum)
__global__ void __launch_bounds__(256) k_axpy_inplace(const double* __restrict__ rhs, double coef, double* __restrict__ f,
                                                      long long n) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) f[e] = __dadd_rn(rhs[e], __dmul_rn(coef, f[e]));
}
// out2[0] = max |yn - y|, out2[1] = max |yn| as the bit patterns of non-negative doubles (ordered like
// the values; maxima are exact, so the order of the reduction does not matter).  out2 zeroed before.
__global__ void __launch_bounds__(256) k_coupled_delta(const double* __restrict__ yn, const double* __restrict__ y,
                                                       long long n, unsigned long long* __restrict__ out2) {
  double d = 0.0, a = 0.0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const double v = yn[e];
    d = fmax(d, fabs(v - y[e]));
    a = fmax(a, fabs(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out2, (unsigned long long)__double_as_longlong(d));
    atomicMax(out2 + 1, (unsigned long long)__double_as_longlong(a));
  }
}

constexpr int kIncrBlocks = 1184;  // 8 x 148 SMs; fixed so the reduction tree is fixed
constexpr int kIncrThreads = 256;
static_assert(kIncrBlocks <= 2048, "k_incr_final folds at most two partials per thread");

__global__ void __launch_bounds__(kIncrThreads) k_incr_partial(const double* __restrict__ a,
                                                              const double* __restrict__ b, long long n,
                                                              double* __restrict__ partial) {
  __shared__ double sh[kIncrThreads];
  double s = 0.0;
  for (long long e = (long long)blockIdx.x * kIncrThreads + threadIdx.x; e < n; e += (long long)kIncrBlocks * kIncrThreads)
    s += fabs(a[e] - b[e]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = kIncrThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(1024) k_incr_final(const double* __restrict__ a, const double* __restrict__ b,
                                                     long long n, const double* __restrict__ partial,
                                                     double* __restrict__ out) {
  __shared__ double sh[1024];
  const int t = threadIdx.x;
  double v = t < kIncrBlocks ? partial[t] : 0.0;
  if (t + 1024 < kIncrBlocks) v = v + partial[t + 1024];
  sh[t] = v;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (t < w) sh[t] = sh[t] + sh[t + w];
    __syncthreads();
  }
  if (t == 0) *out = (n == 1) ? fabs(a[0] - b[0]) : sh[0] / (double)n;
}

}  // namespace cisdc_b200
