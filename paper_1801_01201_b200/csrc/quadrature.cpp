// Host-side quadrature tables of the sweep engine (the constant operands of every RHS kernel).
//
// B200 design: the M x (M+1) tables are built ONCE on the host, in the reference's exact
// floating-point operation order, and uploaded as kernel parameters -- never recomputed on the
// device, so the GPU shares the reference's round-off (e.g. the ~1e-13 row-sum error of Q at
// M = 6, SURVEY.md finding 3).  Algorithms follow:
//   gauss_lobatto_nodes     proj/core/src/quadrature.cpp:40-76  (Newton on P'_M, symmetry forced)
//   build_Q                 proj/core/src/quadrature.cpp:78-108 (monomial Lagrange integration)
//   build_S                 proj/core/src/quadrature.cpp:110-119
//   build_QtI               proj/core/src/quadrature.cpp:121-132 (U^T of unpivoted LU of Qt^T)
//   build_QtE               proj/core/src/quadrature.cpp:134-145
//   make_quadrature_tables  proj/core/src/quadrature.cpp:147-162
// Built with -ffp-contract=off (no FMA), matching the reference's -march=x86-64 build.
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/cisdc_gpu.h"

namespace cisdc_b200 {

namespace {

struct Legendre {
  double p, dp;
};

Legendre legendre_at(int M, double x) {
  if (M == 0) return {1.0, 0.0};
  double prev = 1.0, cur = x;
  for (int k = 2; k <= M; ++k) {
    const double next = ((2.0 * k - 1.0) * x * cur - (k - 1.0) * prev) / k;
    prev = cur;
    cur = next;
  }
  return {cur, M * (x * cur - prev) / (x * x - 1.0)};
}

void lobatto_nodes(int M, double* tau, double* dtau) {
  std::vector<double> x(M + 1);
  x.front() = -1.0;
  x.back() = 1.0;
  for (int i = 1; i < M; ++i) {
    double xi = -std::cos(M_PI * i / M);
    for (int it = 0; it < 100; ++it) {
      const Legendre L = legendre_at(M, xi);
      const double ddp = (2.0 * xi * L.dp - M * (M + 1.0) * L.p) / (1.0 - xi * xi);
      const double step = L.dp / ddp;
      xi -= step;
      if (std::abs(step) <= 1e-16 * (1.0 + std::abs(xi))) break;
    }
    x[i] = xi;
  }
  for (int i = 0; i <= M / 2; ++i) {
    const double half = 0.5 * (x[i] - x[M - i]);
    x[i] = half;
    x[M - i] = -half;
  }
  if (M % 2 == 0) x[M / 2] = 0.0;
  for (int i = 0; i <= M; ++i) tau[i] = 0.5 * (x[i] + 1.0);
  tau[0] = 0.0;
  tau[M] = 1.0;
  for (int m = 0; m < M; ++m) dtau[m] = tau[m + 1] - tau[m];
}

}  // namespace

int make_tables(int M, int convention, cisdc_tables* t) {
  if (M < 1 || M > CISDC_MAX_M) return CISDC_E_INVALID_ARGUMENT;
  std::memset(t, 0, sizeof(*t));
  t->M = M;
  t->convention = convention;
  lobatto_nodes(M, t->tau, t->dtau);
  const int W = M + 1;
  // Q: L_j in ascending monomial coefficients, integrated analytically over [0, tau[m+1]]
  for (int j = 0; j <= M; ++j) {
    std::vector<double> poly{1.0};
    double denom = 1.0;
    for (int i = 0; i <= M; ++i) {
      if (i == j) continue;
      std::vector<double> grown(poly.size() + 1, 0.0);
      for (std::size_t c = 0; c < poly.size(); ++c) {
        grown[c + 1] += poly[c];
        grown[c] -= t->tau[i] * poly[c];
      }
      poly.swap(grown);
      denom *= t->tau[j] - t->tau[i];
    }
    for (int m = 0; m < M; ++m) {
      const double upper = t->tau[m + 1];
      double integral = 0.0, power = upper;
      for (std::size_t c = 0; c < poly.size(); ++c) {
        integral += poly[c] * power / static_cast<double>(c + 1);
        power *= upper;
      }
      t->Q[m * W + j] = integral / denom;
    }
  }
  for (int m = 0; m < M; ++m) {
    t->q[m] = t->Q[m * W];
    for (int j = 1; j <= M; ++j) t->Qt[m * M + j - 1] = t->Q[m * W + j];
  }
  for (int j = 0; j <= M; ++j) {
    t->S[j] = t->Q[j];
    for (int m = 1; m < M; ++m) t->S[m * W + j] = t->Q[m * W + j] - t->Q[(m - 1) * W + j];
  }
  // QtI = U^T where Qt^T = L U (Doolittle, no pivoting)
  std::vector<double> a(M * M);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) a[i * M + j] = t->Qt[j * M + i];
  for (int k = 0; k < M; ++k) {
    const double pivot = a[k * M + k];
    if (pivot == 0.0) return CISDC_E_FACTORIZATION;
    for (int i = k + 1; i < M; ++i) {
      const double mult = a[i * M + k] / pivot;
      a[i * M + k] = mult;
      for (int j = k + 1; j < M; ++j) a[i * M + j] -= mult * a[k * M + j];
    }
  }
  for (int i = 0; i < M; ++i)
    for (int j = i; j < M; ++j) t->QtI[j * M + i] = a[i * M + j];
  for (int m = 1; m < M; ++m) {
    if (convention == CISDC_EULER_LITERAL) {
      t->QtE[m * M + m - 1] = t->dtau[m];
    } else {
      for (int j = 1; j <= m; ++j) t->QtE[m * M + j - 1] = t->dtau[j];
    }
  }
  return CISDC_OK;
}

}  // namespace cisdc_b200

extern "C" int cisdc_make_quadrature_tables(int M, int convention, cisdc_tables* out) {
  if (!out) return CISDC_E_INVALID_ARGUMENT;
  return cisdc_b200::make_tables(M, convention, out);
}
