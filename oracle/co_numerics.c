/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY (see cisdc_oracle.h).
 * Quadrature tables and linear algebra, restated from the reference:
 *   gauss_lobatto_nodes   proj/core/src/quadrature.cpp:40-76
 *   build_Q               proj/core/src/quadrature.cpp:78-108
 *   build_S               proj/core/src/quadrature.cpp:110-119
 *   build_QtI             proj/core/src/quadrature.cpp:121-132
 *   build_QtE             proj/core/src/quadrature.cpp:134-145
 *   make_quadrature_tables proj/core/src/quadrature.cpp:147-162
 *   lu_factor_dense       proj/core/src/linalg.cpp:24-57
 *   lu_solve              proj/core/src/linalg.cpp:59-75
 *   banded_solve          proj/core/src/linalg.cpp:105-155
 * Same floating-point operation order as the reference (bitwise-equal outputs are asserted by
 * tests/test_oracle_vs_ref.py).  Compiled with -ffp-contract=off like the reference's no-FMA build.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "cisdc_oracle.h"

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* P_M and P'_M by the three-term recurrence (quadrature.cpp:26-36) */
static void legendre_pd(int M, double x, double* p, double* dp) {
  double a = 1.0, b = x;
  if (M == 0) {
    *p = 1.0;
    *dp = 0.0;
    return;
  }
  for (int k = 2; k <= M; ++k) {
    const double c = ((2.0 * k - 1.0) * x * b - (k - 1.0) * a) / k;
    a = b;
    b = c;
  }
  *p = b;
  *dp = M * (x * b - a) / (x * x - 1.0);
}

static void lobatto(int M, double* tau, double* dtau) {
  double x[CISDC_MAX_M + 1];
  x[0] = -1.0;
  x[M] = 1.0;
  for (int i = 1; i < M; ++i) {
    double xi = -cos(M_PI * i / M);
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      legendre_pd(M, xi, &p, &dp);
      const double ddp = (2.0 * xi * dp - M * (M + 1.0) * p) / (1.0 - xi * xi);
      const double step = dp / ddp;
      xi -= step;
      if (fabs(step) <= 1e-16 * (1.0 + fabs(xi))) break;
    }
    x[i] = xi;
  }
  for (int i = 0; i <= M / 2; ++i) {
    const double s = 0.5 * (x[i] - x[M - i]);
    x[i] = s;
    x[M - i] = -s;
  }
  if (M % 2 == 0) x[M / 2] = 0.0;
  for (int i = 0; i <= M; ++i) tau[i] = 0.5 * (x[i] + 1.0);
  tau[0] = 0.0;
  tau[M] = 1.0;
  for (int m = 0; m < M; ++m) dtau[m] = tau[m + 1] - tau[m];
}

int co_lu_factor_dense(int n, double* a, int* perm, int pivoting, char* err) {
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) {
    if (pivoting) {
      int p = k;
      double best = fabs(a[k * n + k]);
      for (int i = k + 1; i < n; ++i) {
        if (fabs(a[i * n + k]) > best) {
          best = fabs(a[i * n + k]);
          p = i;
        }
      }
      if (p != k) {
        for (int j = 0; j < n; ++j) {
          const double t = a[k * n + j];
          a[k * n + j] = a[p * n + j];
          a[p * n + j] = t;
        }
        const int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
      }
    }
    const double pivot = a[k * n + k];
    if (pivot == 0.0) {
      if (err) snprintf(err, 512, "lu_factor_dense: zero pivot at index %d", k);
      return CISDC_E_FACTORIZATION;
    }
    for (int i = k + 1; i < n; ++i) {
      const double m = a[i * n + k] / pivot;
      a[i * n + k] = m;
      for (int j = k + 1; j < n; ++j) a[i * n + j] -= m * a[k * n + j];
    }
  }
  return CISDC_OK;
}

void co_lu_solve(int n, const double* lu, const int* perm, const double* b, double* x) {
  for (int i = 0; i < n; ++i) x[i] = b[perm[i]];
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int j = 0; j < i; ++j) s -= lu[i * n + j] * x[j];
    x[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int j = i + 1; j < n; ++j) s -= lu[i * n + j] * x[j];
    x[i] = s / lu[i * n + i];
  }
}

int co_make_tables(int M, int convention, cisdc_tables* tb) {
  if (M < 1 || M > CISDC_MAX_M) return CISDC_E_INVALID_ARGUMENT;
  memset(tb, 0, sizeof(*tb));
  tb->M = M;
  tb->convention = convention;
  lobatto(M, tb->tau, tb->dtau);
  const int W = M + 1;
  /* build_Q: Lagrange basis in monomial form, integrated from 0 to tau[m+1] */
  for (int j = 0; j <= M; ++j) {
    double coef[CISDC_MAX_M + 2];
    int len = 1;
    coef[0] = 1.0;
    double denom = 1.0;
    for (int i = 0; i <= M; ++i) {
      if (i == j) continue;
      double next[CISDC_MAX_M + 2];
      for (int c = 0; c <= len; ++c) next[c] = 0.0;
      for (int c = 0; c < len; ++c) {
        next[c + 1] += coef[c];
        next[c] -= tb->tau[i] * coef[c];
      }
      ++len;
      for (int c = 0; c < len; ++c) coef[c] = next[c];
      denom *= tb->tau[j] - tb->tau[i];
    }
    for (int m = 0; m < M; ++m) {
      const double t = tb->tau[m + 1];
      double integral = 0.0, tp = t;
      for (int c = 0; c < len; ++c) {
        integral += coef[c] * tp / (double)(c + 1);
        tp *= t;
      }
      tb->Q[m * W + j] = integral / denom;
    }
  }
  for (int m = 0; m < M; ++m) {
    tb->q[m] = tb->Q[m * W + 0];
    for (int j = 1; j <= M; ++j) tb->Qt[m * M + (j - 1)] = tb->Q[m * W + j];
  }
  /* build_S: rowwise difference of Q */
  for (int j = 0; j <= M; ++j) {
    tb->S[0 * W + j] = tb->Q[0 * W + j];
    for (int m = 1; m < M; ++m) tb->S[m * W + j] = tb->Q[m * W + j] - tb->Q[(m - 1) * W + j];
  }
  /* build_QtI: U^T of the unpivoted Doolittle LU of Qt^T */
  double At[CISDC_MAX_M * CISDC_MAX_M];
  int perm[CISDC_MAX_M];
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) At[i * M + j] = tb->Qt[j * M + i];
  if (co_lu_factor_dense(M, At, perm, 0, NULL) != CISDC_OK) return CISDC_E_FACTORIZATION;
  for (int i = 0; i < M; ++i)
    for (int j = i; j < M; ++j) tb->QtI[j * M + i] = At[i * M + j];
  /* build_QtE */
  for (int m = 1; m < M; ++m) {
    if (convention == CISDC_EULER_LITERAL) {
      tb->QtE[m * M + (m - 1)] = tb->dtau[m];
    } else {
      for (int j = 1; j <= m; ++j) tb->QtE[m * M + (j - 1)] = tb->dtau[j];
    }
  }
  return CISDC_OK;
}

/* banded_solve (linalg.cpp:105-155): partial pivoting inside the band, working width 2kl+ku+1 */
int co_banded_solve(int n, int kl, int ku, const double* band, const double* b, double* x, char* err) {
  const int width = 2 * kl + ku + 1;
  double* w = (double*)calloc((size_t)n * width, sizeof(double));
  if (!w) return CISDC_E_CUDA;
#define W_(i, j) w[(size_t)(i) * width + ((j) - (i) + kl)]
  for (int i = 0; i < n; ++i) {
    const int j0 = i - kl > 0 ? i - kl : 0;
    const int j1 = i + ku < n - 1 ? i + ku : n - 1;
    for (int j = j0; j <= j1; ++j) W_(i, j) = band[(size_t)(j - i + kl) * n + i];
  }
  for (int i = 0; i < n; ++i) x[i] = b[i];
  for (int k = 0; k < n; ++k) {
    const int last = k + kl < n - 1 ? k + kl : n - 1;
    int p = k;
    double best = fabs(W_(k, k));
    for (int i = k + 1; i <= last; ++i) {
      if (fabs(W_(i, k)) > best) {
        best = fabs(W_(i, k));
        p = i;
      }
    }
    if (best == 0.0) {
      if (err) snprintf(err, 512, "banded_solve: singular band at column %d", k);
      free(w);
      return CISDC_E_SOLVE;
    }
    const int jmax = k + kl + ku < n - 1 ? k + kl + ku : n - 1;
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
    const int jmax = i + kl + ku < n - 1 ? i + kl + ku : n - 1;
    for (int j = i + 1; j <= jmax; ++j) s -= W_(i, j) * x[j];
    x[i] = s / W_(i, i);
  }
#undef W_
  free(w);
  return CISDC_OK;
}
