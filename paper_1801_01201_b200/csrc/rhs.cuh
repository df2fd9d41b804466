// Stage right-hand-side terms shared by the pointwise rhs kernel (pointwise.cuh, k_rhs) and the
// Newton kernel's next-cell epilogue (newton.cuh, k_react_next).
//
// One correction term: cE*(A - Ap) + cI*(D - Dp)                 (R == nullptr)
//                   or cE*(A - Ap) + cI*(D - Dp + R - Rp)
// CISDCQ difference cache: a term whose differences dA = A - Ap and dDR = ((D - Dp) + R) - Rp were
// stored by an earlier launch reads just those (diff != 0: D = dDR, dA = the cached dA or null); a
// term read in full can store them (outA/outDR) for the later nodes.  Same operations, same bits.
//
// Exact zeros (skipA): in the literal Euler convention the configs use, QtE(m, j) is non-zero only
// on the subdiagonal (reference quadrature.cpp:137-139), so most terms have cE == 0.0.  For finite
// A - Ap, cE * (A - Ap) is then a signed zero, and t = (+-0) + tI equals tI bit for bit whenever
// tI = cI * (...) != 0.  Such a term skips the A / Ap reads (and the dA cache): A and Ap are read
// only at the elements where tI is itself a zero (the sign of the sum then depends on both), and
// everywhere once an F_A evaluation flagged a value >= 2^1022, an Inf or a NaN (Ops::wild), where
// the difference could overflow or carry a NaN.  A and Ap are always the original fields.
#pragma once

#include "common.cuh"

namespace cisdc_b200 {

struct RhsTerm {
  double cE, cI;
  const double *A, *Ap, *D, *Dp, *R, *Rp;
  const double* dA;  // cached A - Ap (diff terms whose cE != 0)
  int diff;
  int skipA;
  double *outA, *outDR;
};

enum RhsKind {
  kRhsMisdcq = 0,  // out = base + sum(AD terms) - fc*X ; out2 = base + sum(ADR terms)
  kRhsCisdcq = 1,  // out = base + sum(ADR terms) + (fc*(X - Y) - fc*Z)
  kRhsMisdc = 2,   // base = phi_m + sum_j sc_j*(fa+fd+fr)_j ; out = base + fc*(X - Y - Z)
  kRhsImexq = 3    // out = base + sum(ADR terms) - fc*(X + Y)   (imexq_sweep, integrators.cpp:155-164)
};

struct RhsArgs {
  int kind;
  int nt;
  RhsTerm t[kMaxM];
  double fc;
  const double *X, *Y, *Z;
  const double* base;  // kRhsMisdcq / kRhsCisdcq
  double* out;
  double* out2;        // kRhsMisdcq: reaction-stage partial rhs (may be null)
  // kRhsMisdc
  int M;
  double sc[kMaxM + 1];
  const double* phim;
  const double *sfa[kMaxM + 1], *sfd[kMaxM + 1], *sfr[kMaxM + 1];
  double* base_out;
  const int* wild;  // Ops::wild of the context
};

// kRhsCisdcq's lagged-reaction term fc * (X - Y): for ell == 1 (always, when nu == 1) X and Y are the
// SAME field, F_R of the previous sweep at this node (integrators.cpp:222-224 with fr_lag == fr_p).
// For a finite value x - x is +0.0 exactly, so the term is fc * 0.0 (a zero with fc's sign) and X is
// not read: one field less per launch.  Every F_R store flags non-finite values in Ops::wild as well
// (newton.cuh react_finish, k_eval_r); once flagged, X - Y is evaluated as written (Inf - Inf = NaN).
__device__ __forceinline__ bool rhs_same_xy(const RhsArgs& a, bool tame) { return tame && a.X == a.Y; }

// cE * (A - Ap) + tI with the skipA shortcut above
__device__ __forceinline__ double rhs_term_a(const RhsTerm& T, long long e, double tI, bool skip) {
  if (skip && tI != 0.0) return tI;
  const double dA = (T.diff && T.dA) ? T.dA[e] : T.A[e] - T.Ap[e];
  return T.cE * dA + tI;
}

// k_rhs's kRhsCisdcq expression (run_diffusion_cell's right-hand side, integrators.cpp:201-226)
// for the S species of cell c at once: element s * ncell + c for s = 0 .. S-1.  Every field of a
// term is loaded for all S species before the first value is used, so one thread keeps S to 4 S
// loads in flight per term -- the form the Newton kernel's epilogue needs, whose 16 warps per SM
// could not cover one load at a time.  Per element the operations and their order are k_rhs's.
template <int S>
__device__ __forceinline__ void rhs_cisdcq_cell(const RhsArgs& a, long long c, long long ncell) {
  const bool tame = a.wild == nullptr || *a.wild == 0;
  double r[S];
#pragma unroll
  for (int s = 0; s < S; ++s) r[s] = a.base[(long long)s * ncell + c];
#pragma unroll 1
  for (int t = 0; t < a.nt; ++t) {
    const RhsTerm& T = a.t[t];
    double d[S];
    if (T.diff) {
#pragma unroll
      for (int s = 0; s < S; ++s) d[s] = T.D[(long long)s * ncell + c];
    } else {
      double dp[S], rr[S], rp[S];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const long long e = (long long)s * ncell + c;
        d[s] = T.D[e];
        dp[s] = T.Dp[e];
        rr[s] = T.R[e];
        rp[s] = T.Rp[e];
      }
#pragma unroll
      for (int s = 0; s < S; ++s) d[s] = d[s] - dp[s] + rr[s] - rp[s];
      if (T.outDR) {
#pragma unroll
        for (int s = 0; s < S; ++s) T.outDR[(long long)s * ncell + c] = d[s];
      }
    }
    if (T.skipA && tame) {
#pragma unroll
      for (int s = 0; s < S; ++s) r[s] += rhs_term_a(T, (long long)s * ncell + c, T.cI * d[s], true);
    } else {
      double dA[S];
      if (T.diff && T.dA) {
#pragma unroll
        for (int s = 0; s < S; ++s) dA[s] = T.dA[(long long)s * ncell + c];
      } else {
        double ap[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          dA[s] = T.A[(long long)s * ncell + c];
          ap[s] = T.Ap[(long long)s * ncell + c];
        }
#pragma unroll
        for (int s = 0; s < S; ++s) dA[s] = dA[s] - ap[s];
        if (!T.diff && T.outA) {
#pragma unroll
          for (int s = 0; s < S; ++s) T.outA[(long long)s * ncell + c] = dA[s];
        }
      }
#pragma unroll
      for (int s = 0; s < S; ++s) r[s] += T.cE * dA[s] + T.cI * d[s];
    }
  }
  double x[S], y[S], z[S];
  if (rhs_same_xy(a, tame)) {  // X - Y = +0.0 exactly: X is not read (header comment)
#pragma unroll
    for (int s = 0; s < S; ++s) z[s] = a.Z[(long long)s * ncell + c];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      r[s] += a.fc * 0.0 - a.fc * z[s];
      a.out[(long long)s * ncell + c] = r[s];
    }
    return;
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const long long e = (long long)s * ncell + c;
    x[s] = a.X[e];
    y[s] = a.Y[e];
    z[s] = a.Z[e];
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    r[s] += a.fc * (x[s] - y[s]) - a.fc * z[s];
    a.out[(long long)s * ncell + c] = r[s];
  }
}

}  // namespace cisdc_b200
