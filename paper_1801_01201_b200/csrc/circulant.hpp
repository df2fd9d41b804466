// Host-side exact factorisation of the periodic 4th-order diffusion matrix (see solve1d.cuh):
//   (1+30c) - 16c (z + 1/z) + c (z^2 + 1/z^2) = K * (1 - p z + q z^2) * (1 - p/z + q/z^2)
// With w = z + 1/z the symbol is c w^2 - 16 c w + (1 + 28 c), roots w = 8 -+ sqrt(36 - 1/c).
// Each root gives zeta + 1/zeta = w with |zeta| < 1; p = zeta1 + zeta2, q = zeta1 zeta2 (real for
// real roots and for a complex-conjugate pair), K = c / q.
#pragma once

#include <cmath>
#include <complex>

namespace cisdc_b200 {

// Up to four recurrence passes u_i = (x_i + p u_{i-1}) - q u_{i-2} (forward) / mirrored
// (backward), then y = invK * u.  Real roots (c > 1/36, the stiff case) are applied as four
// first-order passes (q = 0) so that 1 - zeta carries full relative precision for the slowly
// decaying constant mode; a complex-conjugate pair as one second-order pass per direction.
struct CircFactor {
  int npass;
  double p[4], q[4];
  int reverse[4];
  double invK;
};

inline std::complex<double> small_root(std::complex<double> w) {
  // zeta = 2 / (w + sqrt(w^2 - 4)) with the sqrt branch that maximises |w + sqrt| (|zeta| < 1)
  const std::complex<double> s = std::sqrt(w * w - 4.0);
  const std::complex<double> d1 = w + s, d2 = w - s;
  return 2.0 / (std::abs(d1) >= std::abs(d2) ? d1 : d2);
}

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
    f.npass = 4;
    const double zs[4] = {z1, z2, z1, z2};
    for (int k = 0; k < 4; ++k) {
      f.p[k] = zs[k];
      f.q[k] = 0.0;
      f.reverse[k] = k >= 2;
    }
    f.invK = (z1 * z2) / c;
  } else {
    const std::complex<double> z = small_root(std::complex<double>(8.0, std::sqrt(-disc)));
    f.npass = 2;
    f.p[0] = f.p[1] = 2.0 * z.real();
    f.q[0] = f.q[1] = std::norm(z);
    f.reverse[0] = 0;
    f.reverse[1] = 1;
    f.invK = f.q[0] / c;
  }
  return f;
}

}  // namespace cisdc_b200
