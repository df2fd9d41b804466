// Batched iteration-matrix scans: spectral_radius_scan on the GPU, one thread
// per (scheme, nu, r) point.
//
// Reference semantics, restated per point in the reference's operation order:
//   AffineEngine (affine maps of (phi0, Phi^(k)) through one sweep)  proj/core/src/analysis.cpp:25-195
//   affine_iteration_matrix / spectral_radius_scan                     analysis.cpp:215-293
//   hessenberg_reduce + spectral_radius (Francis double-shift QR)      proj/core/src/linalg.cpp:157-332
// A point whose stage factor vanishes, whose G has a non-finite entry, or whose QR iteration hits its
// cap is recorded with ok = 0 (the reference catches those exceptions and records the point).
// Every operation of the affine engine and of the Householder / QR steps is a +, -, *, / or sqrt in
// the reference's order (the library builds with -fmad=false), so G is bit-identical; the one
// library call, hypot for a complex eigenvalue pair's modulus, is CUDA's, not glibc's, so gamma is
// compared to the reference within round-off (tests/test_spectral_scan.py).
#pragma once

#include <cfloat>

#include "common.cuh"

namespace cisdc_b200 {

struct ScanTables {
  int M;
  double Q[kMaxM][kMaxM + 1];
  double S[kMaxM][kMaxM + 1];
  double QtI[kMaxM][kMaxM];
  double QtE[kMaxM][kMaxM];
  double dtau[kMaxM];
};

struct ScanArgs {
  int n_points;
  int n_r;
  int n_groups;              // (scheme, nu) pairs in scan order
  int scheme[64], nu[64];    // per group
  const double* r_grid;
  int d_rule;                // 0 = half_of_r, 1 = fixed
  double fixed_d, a, dt;
  double* gamma;             // [n_points]
  int* ok;                   // [n_points]
  double* G;                 // optional [n_points][M][M]
};

// Affine value c0 * phi0 + sum_j w[j] Phi_j (analysis.cpp:26-31)
struct AffV {
  double c0;
  double w[kMaxM];
};

struct AffVOps {
  int M;
  __device__ __forceinline__ void sub(AffV& y, const AffV& a, const AffV& b) const {  // y = a - b
    y.c0 = a.c0 - b.c0;
    for (int i = 0; i < M; ++i) y.w[i] = a.w[i] - b.w[i];
  }
  __device__ __forceinline__ void scale(AffV& y, double c, const AffV& v) const {  // y = c * v
    y.c0 = c * v.c0;
    for (int i = 0; i < M; ++i) y.w[i] = c * v.w[i];
  }
  __device__ __forceinline__ void axpy(AffV& y, double c, const AffV& x) const {  // y += c x
    y.c0 += c * x.c0;
    for (int i = 0; i < M; ++i) y.w[i] += c * x.w[i];
  }
};

// stage_solve (analysis.cpp:51-58): (1 / (1 - coef kappa)) * rhs; false on a vanishing factor
__device__ __forceinline__ bool aff_stage(const AffVOps& o, AffV& out, const AffV& rhs, double coef, double kappa) {
  const double denom = 1.0 - coef * kappa;
  if (denom == 0.0) return false;
  o.scale(out, 1.0 / denom, rhs);
  return true;
}

// One sweep's affine map (AffineEngine::run); cur[1..M] receive the node maps.  false = singular.
__device__ bool affine_sweep(const ScanTables& tb, int scheme, int nu, double a, double d, double r, double dt,
                             AffV (&cur)[kMaxM + 1]) {
  const int M = tb.M;
  if (scheme == 2 && nu < 1) return false;  // affine_sweep_map throws invalid_argument (analysis.cpp:200)
  const AffVOps o{M};
  AffV prev[kMaxM + 1];
  for (int j = 0; j <= M; ++j) {
    prev[j].c0 = j == 0 ? 1.0 : 0.0;
    for (int i = 0; i < M; ++i) prev[j].w[i] = (j >= 1 && i == j - 1) ? 1.0 : 0.0;
  }
  const double s = a + d + r;  // StiffnessTriple::sum
  auto quadrature_base = [&](int row, AffV& base) {
    base = prev[0];
    for (int j = 0; j <= M; ++j) o.axpy(base, dt * tb.Q[row][j] * s, prev[j]);
  };
  AffV rhs, rhs2, delta, phi_ad, tmp;
  for (int j = 0; j <= M; ++j) cur[j] = prev[j];
  if (scheme == 1) {  // misdcq
    for (int m = 0; m < M; ++m) {
      AffV base;
      quadrature_base(m, base);
      const double coef = dt * tb.QtI[m][m];
      rhs = base;
      for (int j = 1; j <= m; ++j) {
        o.sub(delta, cur[j], prev[j]);
        o.axpy(rhs, dt * tb.QtE[m][j - 1] * a, delta);
        o.axpy(rhs, dt * tb.QtI[m][j - 1] * d, delta);
      }
      o.axpy(rhs, -coef * d, prev[m + 1]);
      if (!aff_stage(o, phi_ad, rhs, coef, d)) return false;
      rhs2 = base;
      for (int j = 1; j <= m; ++j) {
        o.sub(delta, cur[j], prev[j]);
        o.axpy(rhs2, dt * tb.QtE[m][j - 1] * a, delta);
        o.axpy(rhs2, dt * tb.QtI[m][j - 1] * (d + r), delta);
      }
      o.axpy(rhs2, coef * d, phi_ad);
      o.axpy(rhs2, -coef * (d + r), prev[m + 1]);
      if (!aff_stage(o, cur[m + 1], rhs2, coef, r)) return false;
    }
    return true;
  }
  if (scheme == 0) {  // misdc
    for (int m = 0; m < M; ++m) {
      const double dtm = dt * tb.dtau[m];
      AffV base = cur[m];
      for (int j = 0; j <= M; ++j) o.axpy(base, dt * tb.S[m][j] * s, prev[j]);
      rhs = base;
      o.sub(delta, cur[m], prev[m]);
      o.axpy(rhs, dtm * a, delta);
      o.axpy(rhs, -dtm * d, prev[m + 1]);
      if (!aff_stage(o, phi_ad, rhs, dtm, d)) return false;
      rhs2 = base;
      o.sub(delta, cur[m], prev[m]);
      o.axpy(rhs2, dtm * a, delta);
      o.sub(tmp, phi_ad, prev[m + 1]);
      o.axpy(rhs2, dtm * d, tmp);
      o.axpy(rhs2, -dtm * r, prev[m + 1]);
      if (!aff_stage(o, cur[m + 1], rhs2, dtm, r)) return false;
    }
    return true;
  }
  if (scheme == 3) {  // imexq
    for (int m = 0; m < M; ++m) {
      quadrature_base(m, rhs);
      for (int j = 1; j <= m; ++j) {
        o.sub(delta, cur[j], prev[j]);
        o.axpy(rhs, dt * tb.QtE[m][j - 1] * a, delta);
        o.axpy(rhs, dt * tb.QtI[m][j - 1] * (d + r), delta);
      }
      const double coef = dt * tb.QtI[m][m];
      o.axpy(rhs, -coef * (d + r), prev[m + 1]);
      if (!aff_stage(o, cur[m + 1], rhs, coef, d + r)) return false;
    }
    return true;
  }
  // cisdcq(nu)
  AffV lag_r[kMaxM + 1], lag_ad[kMaxM + 1], new_r[kMaxM + 1], pad[kMaxM + 1];
  for (int j = 0; j <= M; ++j) lag_r[j] = lag_ad[j] = prev[j];
  for (int ell = 1; ell <= nu; ++ell) {
    for (int j = 0; j <= M; ++j) new_r[j] = prev[j];
    for (int m = 0; m < M; ++m) {
      const int node = m + 1;
      quadrature_base(m, rhs);
      for (int j = 1; j <= m - 1; ++j) {
        o.sub(delta, new_r[j], prev[j]);
        o.axpy(rhs, dt * tb.QtE[m][j - 1] * a, delta);
        o.axpy(rhs, dt * tb.QtI[m][j - 1] * (d + r), delta);
      }
      if (m >= 1) {
        o.sub(delta, lag_ad[m], prev[m]);
        o.axpy(rhs, dt * tb.QtE[m][m - 1] * a, delta);
        o.sub(delta, lag_ad[m], prev[m]);
        o.axpy(rhs, dt * tb.QtI[m][m - 1] * d, delta);
        o.sub(delta, lag_r[m], prev[m]);
        o.axpy(rhs, dt * tb.QtI[m][m - 1] * r, delta);
      }
      const double coef = dt * tb.QtI[m][m];
      o.sub(delta, lag_r[node], prev[node]);
      o.axpy(rhs, coef * r, delta);
      o.axpy(rhs, -coef * d, prev[node]);
      if (!aff_stage(o, pad[node], rhs, coef, d)) return false;
      if (ell == 1) lag_ad[node] = pad[node];
      rhs2 = pad[node];
      if (m >= 1) {
        o.sub(delta, new_r[m], lag_r[m]);
        o.axpy(rhs2, dt * tb.QtI[m][m - 1] * r, delta);
      }
      o.axpy(rhs2, -coef * r, lag_r[node]);
      if (!aff_stage(o, new_r[node], rhs2, coef, r)) return false;
    }
    for (int j = 0; j <= M; ++j) lag_r[j] = lag_ad[j] = new_r[j];
  }
  for (int j = 0; j <= M; ++j) cur[j] = new_r[j];
  return true;
}

__device__ __forceinline__ double max_ref(double a, double b) { return (a < b) ? b : a; }  // std::max

// spectral_radius (linalg.cpp:197-332) of the n x n matrix h (row-major, n <= kMaxM), destroyed.
// Returns 0 = ok, 1 = non-finite entry (invalid_argument), 2 = QR iteration cap (NumericError).
__device__ int spectral_radius_dev(double (&h)[kMaxM][kMaxM], int n, double& rho_out) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (!isfinite(h[i][j])) return 1;
  if (n == 1) {
    rho_out = fabs(h[0][0]);
    return 0;
  }
  // hessenberg_reduce (linalg.cpp:159-193)
  double v[kMaxM];
  for (int k = 1; k < n - 1; ++k) {
    double scale = 0.0;
    for (int i = k; i < n; ++i) scale += fabs(h[i][k - 1]);
    if (scale == 0.0) continue;
    double ssq = 0.0;
    for (int i = k; i < n; ++i) {
      v[i] = h[i][k - 1] / scale;
      ssq += v[i] * v[i];
    }
    double alpha = sqrt(ssq);
    if (v[k] > 0.0) alpha = -alpha;
    const double beta = ssq - v[k] * alpha;
    if (beta == 0.0) continue;
    v[k] -= alpha;
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int i = k; i < n; ++i) s += v[i] * h[i][j];
      s /= beta;
      for (int i = k; i < n; ++i) h[i][j] -= s * v[i];
    }
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = k; j < n; ++j) s += h[i][j] * v[j];
      s /= beta;
      for (int j = k; j < n; ++j) h[i][j] -= s * v[j];
    }
    h[k][k - 1] = scale * alpha;
    for (int i = k + 1; i < n; ++i) h[i][k - 1] = 0.0;
  }
  const double eps = DBL_EPSILON;
  const long cap = 10000L * n;
  long iters = 0;
  double rho = 0.0, anorm = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = (i - 1 > 0 ? i - 1 : 0); j < n; ++j) anorm += fabs(h[i][j]);
  if (anorm == 0.0) {
    rho_out = 0.0;
    return 0;
  }
  int nn = n - 1;
  double t = 0.0;
  while (nn >= 0) {
    int its = 0;
    int l;
    do {
      for (l = nn; l >= 1; --l) {
        const double s = fabs(h[l - 1][l - 1]) + fabs(h[l][l]);
        const double thr = (s == 0.0 ? anorm : s) * eps;
        if (fabs(h[l][l - 1]) <= thr) {
          h[l][l - 1] = 0.0;
          break;
        }
      }
      double x = h[nn][nn];
      if (l == nn) {
        rho = max_ref(rho, fabs(x + t));
        --nn;
        break;
      }
      double y = h[nn - 1][nn - 1];
      double w = h[nn][nn - 1] * h[nn - 1][nn];
      if (l == nn - 1) {
        const double p2 = 0.5 * (y - x);
        const double q2 = p2 * p2 + w;
        const double z2 = sqrt(fabs(q2));
        x += t;
        if (q2 >= 0.0) {
          const double zz = p2 + (p2 >= 0.0 ? z2 : -z2);
          rho = max_ref(rho, fabs(x + zz));
          if (zz != 0.0) rho = max_ref(rho, fabs(x - w / zz));
        } else {
          rho = max_ref(rho, hypot(x + p2, z2));
        }
        nn -= 2;
        break;
      }
      if (iters++ >= cap) return 2;
      if (its == 10 || its == 20) {
        t += x;
        for (int i = 0; i <= nn; ++i) h[i][i] -= x;
        const double s = fabs(h[nn][nn - 1]) + fabs(h[nn - 1][nn - 2]);
        x = y = 0.75 * s;
        w = -0.4375 * s * s;
      }
      ++its;
      int m;
      double p = 0.0, q = 0.0, r = 0.0;
      for (m = nn - 2; m >= l; --m) {
        const double z = h[m][m];
        const double rr = x - z;
        const double ss = y - z;
        p = (rr * ss - w) / h[m + 1][m] + h[m][m + 1];
        q = h[m + 1][m + 1] - z - rr - ss;
        r = h[m + 2][m + 1];
        const double scl = fabs(p) + fabs(q) + fabs(r);
        p /= scl;
        q /= scl;
        r /= scl;
        if (m == l) break;
        const double u = fabs(h[m][m - 1]) * (fabs(q) + fabs(r));
        const double vv = fabs(p) * (fabs(h[m - 1][m - 1]) + fabs(z) + fabs(h[m + 1][m + 1]));
        if (u <= eps * vv) break;
      }
      for (int i = m + 2; i <= nn; ++i) h[i][i - 2] = 0.0;
      for (int i = m + 3; i <= nn; ++i) h[i][i - 3] = 0.0;
      for (int k = m; k <= nn - 1; ++k) {
        double scl = 0.0;
        if (k != m) {
          p = h[k][k - 1];
          q = h[k + 1][k - 1];
          r = (k != nn - 1) ? h[k + 2][k - 1] : 0.0;
          scl = fabs(p) + fabs(q) + fabs(r);
          if (scl != 0.0) {
            p /= scl;
            q /= scl;
            r /= scl;
          }
        }
        double s = sqrt(p * p + q * q + r * r);
        if (p < 0.0) s = -s;
        if (s == 0.0) continue;
        if (k == m) {
          if (l != m) h[k][k - 1] = -h[k][k - 1];
        } else {
          h[k][k - 1] = -s * scl;
        }
        p += s;
        const double xh = p / s;
        const double yh = q / s;
        const double zh = r / s;
        q /= p;
        r /= p;
        for (int j = k; j <= nn; ++j) {
          double pp = h[k][j] + q * h[k + 1][j];
          if (k != nn - 1) {
            pp += r * h[k + 2][j];
            h[k + 2][j] -= pp * zh;
          }
          h[k + 1][j] -= pp * yh;
          h[k][j] -= pp * xh;
        }
        const int mmin = nn < k + 3 ? nn : k + 3;
        for (int i = l; i <= mmin; ++i) {
          double pp = xh * h[i][k] + yh * h[i][k + 1];
          if (k != nn - 1) {
            pp += zh * h[i][k + 2];
            h[i][k + 2] -= pp * r;
          }
          h[i][k + 1] -= pp * q;
          h[i][k] -= pp;
        }
      }
    } while (l < nn - 1);
  }
  rho_out = rho;
  return 0;
}

// spectral_radius of `count` independent n x n matrices (row-major, n <= 8), one per thread;
// status 0 = ok, 1 = non-finite entry (std::invalid_argument), 2 = QR cap (NumericError)
__global__ void __launch_bounds__(64) k_spectral_batch(const double* __restrict__ A, int n, int count,
                                                       double* __restrict__ rho, int* __restrict__ status) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= count) return;
  double h[kMaxM][kMaxM];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) h[i][j] = A[((long long)p * n + i) * n + j];
  double r = 0.0;
  status[p] = spectral_radius_dev(h, n, r);
  rho[p] = r;
}

// one thread per point, points ordered like the reference's loops (scheme, nu, r)
__global__ void __launch_bounds__(64) k_spectral_scan(const __grid_constant__ ScanTables tb,
                                                      const __grid_constant__ ScanArgs a) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.n_points) return;
  const int g = p / a.n_r, ir = p - g * a.n_r;
  const double r = a.r_grid[ir];
  const double d = a.d_rule == 0 ? r / 2.0 : a.fixed_d;
  const int M = tb.M;
  AffV cur[kMaxM + 1];
  double h[kMaxM][kMaxM];
  int ok = affine_sweep(tb, a.scheme[g], a.nu[g], a.a, d, r, a.dt, cur) ? 1 : 0;
  double gamma = 0.0;
  if (ok) {
    for (int m = 1; m <= M; ++m)
      for (int j = 0; j < M; ++j) h[m - 1][j] = cur[m].w[j];
    if (a.G)
      for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) a.G[((long long)p * M + i) * M + j] = h[i][j];
    ok = spectral_radius_dev(h, M, gamma) == 0 ? 1 : 0;
    if (!ok) gamma = 0.0;
  }
  a.gamma[p] = gamma;
  a.ok[p] = ok;
}

}  // namespace cisdc_b200
