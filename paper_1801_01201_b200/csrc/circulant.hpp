// Host-side exact factorisation of the periodic 4th-order diffusion matrix (see solve1d.cuh):
//   (1+30c) - 16c (z + 1/z) + c (z^2 + 1/z^2) = K * (1 - p z + q z^2) * (1 - p/z + q/z^2)
// With w = z + 1/z the symbol is c w^2 - 16 c w + (1 + 28 c), roots w = 8 -+ sqrt(36 - 1/c).
// Each root gives zeta + 1/zeta = w with |zeta| < 1; p = zeta1 + zeta2, q = zeta1 zeta2 (real for
// real roots and for a complex-conjugate pair), K = c / q.
//
// Written with explicit real arithmetic only (sqrt, +, -, *, /; no complex library calls) so the
// CPU oracle (oracle/co_problems.c: circ_factor) reproduces the same bits.  The block
// decomposition of the scan (solve1d_blocking) is part of the algorithm's definition for the same
// reason: the oracle emulates the identical evaluation order.
#pragma once

#include <cmath>

namespace cisdc_b200 {

// Up to four recurrence passes u_i = (x_i + p u_{i-1}) - q u_{i-2} (forward) / mirrored
// (backward), then y = invK * u.  Real roots (c > 1/36, the stiff case) are applied as four
// first-order passes (q = 0) so that 1 - zeta carries full relative precision for the slowly
// decaying constant mode; a complex-conjugate pair as one second-order pass per direction.
// Real roots: one forward and one backward pass, each running the two first-order recurrences
// (zeta1 then zeta2) coupled in a single scan (kind 1).
struct CircFactor {
  int npass;
  double p[4], q[4];
  int reverse[4];
  int kind[4];
  double invK;
};

inline CircFactor factor_circulant(double c) {
  CircFactor f{};
  const double disc = 36.0 - 1.0 / c;
  if (disc >= 0.0) {
    const double r = std::sqrt(disc);
    // w1 - 2 = 6 - r computed without cancellation; w^2 - 4 = (w - 2)(w + 2)
    const double e1 = (1.0 / c) / (6.0 + r);
    const double w1 = 2.0 + e1, w2 = 8.0 + r;
    const double z1 = 2.0 / (w1 + std::sqrt(e1 * (w1 + 2.0)));
    const double z2 = 2.0 / (w2 + std::sqrt((w2 - 2.0) * (w2 + 2.0)));
    f.npass = 2;
    for (int k = 0; k < 2; ++k) {
      f.p[k] = z1;
      f.q[k] = z2;
      f.reverse[k] = k;
      f.kind[k] = 1;
    }
    f.invK = (z1 * z2) / c;
  } else {
    // w = 8 + i wi; s = principal sqrt(w^2 - 4) = sqrt(ar + i ai)
    const double wi = std::sqrt(-disc);
    const double ar = 60.0 - wi * wi, ai = 16.0 * wi;
    const double mod = std::sqrt(ar * ar + ai * ai);
    double sr, si;
    if (ar >= 0.0) {
      sr = std::sqrt((mod + ar) * 0.5);
      si = ai / (2.0 * sr);
    } else {
      si = std::sqrt((mod - ar) * 0.5);  // ai > 0
      sr = ai / (2.0 * si);
    }
    // the denominator of larger modulus gives |zeta| < 1: zeta = 2 / (w +- s)
    const double d1r = 8.0 + sr, d1i = wi + si, d2r = 8.0 - sr, d2i = wi - si;
    const double m1 = d1r * d1r + d1i * d1i, m2 = d2r * d2r + d2i * d2i;
    const double dr = m1 >= m2 ? d1r : d2r, di = m1 >= m2 ? d1i : d2i, dm = m1 >= m2 ? m1 : m2;
    const double zr = (2.0 * dr) / dm, zi = (-2.0 * di) / dm;
    f.npass = 2;
    f.p[0] = f.p[1] = 2.0 * zr;
    f.q[0] = f.q[1] = zr * zr + zi * zi;
    f.reverse[0] = 0;
    f.reverse[1] = 1;
    f.kind[0] = f.kind[1] = 0;
    f.invK = f.q[0] / c;
  }
  return f;
}

// Block decomposition of the scan: T threads per CTA, E elements per thread, CL CTAs per cluster
// (up to 16, the non-portable cluster size: more SMs before the per-thread chains grow).
constexpr int kSolve1dThreads = 512;
constexpr int kSolve1dMaxCluster = 16;
inline void solve1d_blocking(int N, int* E, int* CL) {
  int e = 1;
  while (e < 32 && (long long)e * kSolve1dThreads * kSolve1dMaxCluster < N) e *= 2;
  *E = e;
  *CL = (N + e * kSolve1dThreads - 1) / (e * kSolve1dThreads);
}

}  // namespace cisdc_b200
