/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY (see cisdc_oracle.h).
 * Problem classes behind the OperatorSplitProblem contract
 * (proj/core/include/cisdc/operator_split.hpp:36-54):
 *
 *  - CISDC_PROBLEM_REFERENCE_RD: restatement of the reference's own 1-D Dirichlet PDE
 *      ReactionDiffusionGrid / ghost weights   proj/core/src/problems/reaction_diffusion.cpp:30-67
 *      advection_operator                      :76-87
 *      laplacian_operator                      :89-100
 *      reaction_term                           :102-109
 *      assemble_diffusion_system / solve       :127-164  (banded_solve, linalg.cpp:105-155)
 *      solve_reaction_implicit                 :166-183  (newton_scalar, linalg.cpp:333-349)
 *  - CISDC_PROBLEM_LINEAR_SCALAR: LinearScalarProblem, proj/core/src/problems/linear.cpp:19-50
 *  - CISDC_PROBLEM_PERIODIC_ADR: NEW problem class for BASELINE configs 1-5 (no reference
 *    implementation exists).  It follows reaction_diffusion.cpp's structure: the same 4th-order
 *    stencils (:84,:97) per axis with periodic wrap, advection in flux form, a cyclic banded direct
 *    diffusion solve in 1-D (the ring folded into a band of half-width 4 and handed to the
 *    restated banded_solve), a geometric multigrid in 2-D/3-D, and the per-cell Newton of
 *    solve_reaction_implicit generalised to S species with lu_factor_dense(pivoting) / lu_solve
 *    (linalg.cpp:24-75) and newton_scalar's two exit tests (linalg.cpp:339,346) in inf-norms.
 *    The GPU kernels implement exactly the arithmetic written here (same operation order, no
 *    FMA contraction); DESIGN.md "Problem class" is the specification.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "cisdc_oracle.h"

/* Optional threads for the per-cell loops (env CISDC_ORACLE_THREADS, default 1): every parallel
   loop below has independent iterations writing disjoint cells, and the reductions are max-norms
   (order-free) or integer sums, so the results are bit-identical at any thread count.  Used to
   generate the full-size golden fixtures (tests/golden/make_golden.py --full) in reasonable time;
   the CPU baselines in bench.py run with 1 thread (the reference's problem stages are serial). */
static int co_threads(void) {
  static int t = -1;
  if (t < 0) {
    const char* e = getenv("CISDC_ORACLE_THREADS");
    t = e ? atoi(e) : 1;
    if (t < 1) t = 1;
  }
  return t;
}
#define CO_PRAGMA(x) _Pragma(#x)
#define CO_PAR_ROWS(n) \
  CO_PRAGMA(omp parallel for schedule(static) collapse(2) if (co_threads() > 1 && (n) > 16384) num_threads(co_threads()))
#define CO_PAR(n) CO_PRAGMA(omp parallel for schedule(static) if (co_threads() > 1 && (n) > 16384) num_threads(co_threads()))

#define MAXS CISDC_MAX_SPECIES
#define MAXR CISDC_MAX_REACTIONS
#define MAXL 16

struct co_problem {
  cisdc_problem_desc d;
  size_t dim, ncell;
  int S, nx, ny, nz;
  double* vel[3][3];      /* owned copies of the separable face-velocity tables (NULL = 1.0) */
  int adv[3];             /* axis a advects */
  double cadv[3];         /* 1 / (12 h_a) */
  double cdiff[MAXS][3];  /* d_s / (12 h_a h_a) */
  double diffusivity[MAXS];
  /* mass action */
  int nr;
  int reac[MAXR][2], prod[MAXR][2];
  double k[MAXR];
  int nu[MAXS][MAXR];     /* net stoichiometric change of species s in reaction r */
  /* reference RD */
  double rd_dx, rd_w[2][5];
  /* multigrid workspace */
  int L;
  int ln[MAXL][3];
  double* mg_x[MAXL];
  double* mg_b[MAXL];
  double* mg_t[MAXL];
  char err[512];
};

static int fail(co_problem* p, int code, const char* msg) {
  snprintf(p->err, sizeof(p->err), "%s", msg);
  return code;
}

/* ------------------------------------------------------------------ creation */

static void lagrange_weights_at(double xg, double* w) {
  static const double pts[5] = {0.0, 0.5, 1.5, 2.5, 3.5};
  for (int j = 0; j < 5; ++j) {
    double num = 1.0, den = 1.0;
    for (int i = 0; i < 5; ++i) {
      if (i == j) continue;
      num *= xg - pts[i];
      den *= pts[j] - pts[i];
    }
    w[j] = num / den;
  }
}

int co_problem_create(const cisdc_problem_desc* desc, co_problem** out, char* err) {
  co_problem* p = (co_problem*)calloc(1, sizeof(co_problem));
  if (!p) return CISDC_E_CUDA;
  p->d = *desc;
  int rc = CISDC_OK;
#define BAD(msg)                                         \
  do {                                                   \
    if (err) snprintf(err, 512, "%s", msg);              \
    rc = CISDC_E_INVALID_ARGUMENT;                       \
    goto fail_;                                          \
  } while (0)
  if (desc->kind == CISDC_PROBLEM_LINEAR_SCALAR) {
    /* n[0] >= 1 independent copies of the scalar model (the reference's dimension-1 problem per
       element; n[0] = 1 is LinearScalarProblem itself) */
    p->dim = p->ncell = (size_t)(desc->n[0] >= 1 ? desc->n[0] : 1);
    p->S = 1;
  } else if (desc->kind == CISDC_PROBLEM_REFERENCE_RD) {
    p->nx = desc->n[0];
    if (p->nx < 8) BAD("ReactionDiffusionGrid: n_x must be >= 8");
    p->ny = p->nz = 1;
    p->S = 1;
    p->dim = p->ncell = (size_t)p->nx;
    p->rd_dx = (20.0 - 0.0) / p->nx;
    lagrange_weights_at(-0.5, p->rd_w[0]);
    lagrange_weights_at(-1.5, p->rd_w[1]);
  } else if (desc->kind == CISDC_PROBLEM_PERIODIC_ADR) {
    if (desc->ndim < 1 || desc->ndim > 3) BAD("periodic ADR: ndim must be 1..3");
    if (desc->nspecies < 1 || desc->nspecies > MAXS) BAD("periodic ADR: nspecies out of range");
    p->S = desc->nspecies;
    p->nx = desc->n[0];
    p->ny = desc->ndim >= 2 ? desc->n[1] : 1;
    p->nz = desc->ndim >= 3 ? desc->n[2] : 1;
    int nn[3] = {p->nx, p->ny, p->nz};
    for (int a = 0; a < desc->ndim; ++a)
      if (nn[a] < 8) BAD("periodic ADR: every active axis needs >= 8 cells");
    p->ncell = (size_t)p->nx * p->ny * p->nz;
    p->dim = p->ncell * p->S;
    for (int a = 0; a < 3; ++a) {
      int any = 0;
      for (int b = 0; b < 3; ++b) {
        if (desc->vel[a][b] && b < desc->ndim) {
          p->vel[a][b] = (double*)malloc(sizeof(double) * nn[b]);
          memcpy(p->vel[a][b], desc->vel[a][b], sizeof(double) * nn[b]);
          any = 1;
        }
      }
      p->adv[a] = any && a < desc->ndim;
      if (a < desc->ndim) p->cadv[a] = 1.0 / (12.0 * desc->h[a]);
    }
    for (int s = 0; s < p->S; ++s) {
      const double ds = desc->diffusivity ? desc->diffusivity[s] : 0.0;
      p->diffusivity[s] = ds;
      for (int a = 0; a < desc->ndim; ++a) p->cdiff[s][a] = ds / (12.0 * desc->h[a] * desc->h[a]);
    }
    if (desc->reaction_kind == CISDC_REACTION_LINEAR_DECAY || desc->reaction_kind == CISDC_REACTION_BISTABLE) {
      if (p->S != 1) BAD("scalar reaction kinds need nspecies == 1");
    } else if (desc->reaction_kind == CISDC_REACTION_MASS_ACTION) {
      if (desc->n_reactions < 0 || desc->n_reactions > MAXR) BAD("mass action: too many reactions");
      p->nr = desc->n_reactions;
      for (int r = 0; r < p->nr; ++r) {
        for (int t = 0; t < 2; ++t) {
          p->reac[r][t] = desc->reactants[2 * r + t];
          p->prod[r][t] = desc->products[2 * r + t];
          if (p->reac[r][t] >= p->S || p->prod[r][t] >= p->S) BAD("mass action: species index out of range");
        }
        if (p->reac[r][0] < 0) BAD("mass action: every reaction needs a first reactant");
        p->k[r] = desc->rate_constants[r];
        for (int t = 0; t < 2; ++t) {
          if (p->reac[r][t] >= 0) p->nu[p->reac[r][t]][r] -= 1;
          if (p->prod[r][t] >= 0) p->nu[p->prod[r][t]][r] += 1;
        }
      }
    } else if (desc->reaction_kind != CISDC_REACTION_NONE) {
      BAD("unknown reaction kind");
    }
    if (desc->diffusion_solver == CISDC_DIFFUSION_DIRECT) {
      if (desc->ndim != 1) BAD("direct diffusion solve is 1-D only; use multigrid");
      if (p->nx > 8 * 512 * 32) BAD("1-D direct solve supports n <= 131072");
    } else if (desc->diffusion_solver == CISDC_DIFFUSION_BANDED_ORACLE) {
      if (desc->ndim != 1) BAD("banded diffusion solve is 1-D only");
    } else if (desc->diffusion_solver == CISDC_DIFFUSION_MULTIGRID) {
      int n0[3] = {p->nx, p->ny, p->nz};
      p->L = 1;
      for (int a = 0; a < 3; ++a) p->ln[0][a] = n0[a];
      const int minc = desc->mg_min_coarse > 2 ? desc->mg_min_coarse : 4;
      for (;;) {
        int ok = p->L < MAXL;
        for (int a = 0; a < desc->ndim; ++a) {
          const int na = p->ln[p->L - 1][a];
          if (na % 2 != 0 || na / 2 < minc) ok = 0;
        }
        if (!ok) break;
        for (int a = 0; a < 3; ++a) p->ln[p->L][a] = a < desc->ndim ? p->ln[p->L - 1][a] / 2 : 1;
        p->L++;
      }
      for (int l = 0; l < p->L; ++l) {
        const size_t nc = (size_t)p->ln[l][0] * p->ln[l][1] * p->ln[l][2];
        p->mg_x[l] = (double*)calloc(nc, sizeof(double));
        p->mg_b[l] = (double*)calloc(nc, sizeof(double));
        p->mg_t[l] = (double*)calloc(nc, sizeof(double));
      }
      if (desc->mg_pre < 2 || desc->mg_coarse_sweeps < 2 || desc->mg_post < 0 || desc->mg_max_cycles < 1 ||
          desc->mg_pre % 2 || desc->mg_post % 2 || desc->mg_coarse_sweeps % 2)
        BAD("multigrid: need even mg_pre >= 2, mg_post >= 0, mg_coarse_sweeps >= 2 and mg_max_cycles >= 1");
    } else {
      BAD("unknown diffusion solver");
    }
  } else {
    BAD("unknown problem kind");
  }
  *out = p;
  return CISDC_OK;
fail_:
  co_problem_destroy(p);
  return rc;
#undef BAD
}

void co_problem_destroy(co_problem* p) {
  if (!p) return;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) free(p->vel[a][b]);
  for (int l = 0; l < MAXL; ++l) {
    free(p->mg_x[l]);
    free(p->mg_b[l]);
    free(p->mg_t[l]);
  }
  free(p);
}

size_t co_problem_dim(const co_problem* p) { return p->dim; }
int co_problem_has_coupled(const co_problem* p) {
  return p->d.kind == CISDC_PROBLEM_LINEAR_SCALAR ||
         (p->d.kind == CISDC_PROBLEM_PERIODIC_ADR && p->d.coupled_max_iter > 0);
}
const char* co_problem_error(const co_problem* p) { return p->err; }

/* ------------------------------------------------------------------ periodic ADR operators */

static inline int wrap(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

/* separable face velocity of component a at the + face (along a) of cell (i,j,k) */
static inline double face_u(const co_problem* p, int a, int i, int j, int k) {
  const double t0 = p->vel[a][0] ? p->vel[a][0][i] : 1.0;
  const double t1 = p->vel[a][1] ? p->vel[a][1][j] : 1.0;
  const double t2 = p->vel[a][2] ? p->vel[a][2][k] : 1.0;
  return (t0 * t1) * t2;
}

/* value of field f (one species plane) at (i,j,k) displaced by o along axis a, periodic */
static inline double at_off(const co_problem* p, const double* f, int i, int j, int k, int a, int o) {
  if (a == 0) i = wrap(i + o, p->nx);
  else if (a == 1) j = wrap(j + o, p->ny);
  else k = wrap(k + o, p->nz);
  return f[((size_t)k * p->ny + j) * p->nx + i];
}

/* unscaled 4th-order face value times velocity, + face of the cell displaced by o along a */
static inline double face_flux(const co_problem* p, const double* f, int i, int j, int k, int a, int o) {
  const double pm1 = at_off(p, f, i, j, k, a, o - 1);
  const double p0 = at_off(p, f, i, j, k, a, o);
  const double p1 = at_off(p, f, i, j, k, a, o + 1);
  const double p2 = at_off(p, f, i, j, k, a, o + 2);
  int ii = i, jj = j, kk = k;
  if (a == 0) ii = wrap(i + o, p->nx);
  else if (a == 1) jj = wrap(j + o, p->ny);
  else kk = wrap(k + o, p->nz);
  return face_u(p, a, ii, jj, kk) * (7.0 * (p0 + p1) - (pm1 + p2));
}

static void adr_advection(const co_problem* p, const double* phi, double* out) {
  for (int s = 0; s < p->S; ++s) {
    const double* f = phi + (size_t)s * p->ncell;
    double* o = out + (size_t)s * p->ncell;
    CO_PAR_ROWS(p->ncell)
    for (int k = 0; k < p->nz; ++k)
      for (int j = 0; j < p->ny; ++j)
        for (int i = 0; i < p->nx; ++i) {
          double acc = 0.0;
          for (int a = 0; a < p->d.ndim; ++a) {
            if (!p->adv[a]) continue;
            const double fr = face_flux(p, f, i, j, k, a, 0);
            const double fl = face_flux(p, f, i, j, k, a, -1);
            acc = acc + (fr - fl) * p->cadv[a];
          }
          o[((size_t)k * p->ny + j) * p->nx + i] = -acc;
        }
  }
}

static inline double lap_axis(const co_problem* p, const double* f, int i, int j, int k, int a) {
  const double g0 = at_off(p, f, i, j, k, a, -2);
  const double g1 = at_off(p, f, i, j, k, a, -1);
  const double g2 = at_off(p, f, i, j, k, a, 0);
  const double g3 = at_off(p, f, i, j, k, a, 1);
  const double g4 = at_off(p, f, i, j, k, a, 2);
  return -g0 + 16.0 * g1 - 30.0 * g2 + 16.0 * g3 - g4;
}

static void adr_diffusion(const co_problem* p, const double* phi, double* out) {
  for (int s = 0; s < p->S; ++s) {
    const double* f = phi + (size_t)s * p->ncell;
    double* o = out + (size_t)s * p->ncell;
    CO_PAR_ROWS(p->ncell)
    for (int k = 0; k < p->nz; ++k)
      for (int j = 0; j < p->ny; ++j)
        for (int i = 0; i < p->nx; ++i) {
          double lap = 0.0;
          for (int a = 0; a < p->d.ndim; ++a) lap = lap + p->cdiff[s][a] * lap_axis(p, f, i, j, k, a);
          o[((size_t)k * p->ny + j) * p->nx + i] = lap;
        }
  }
}

/* mass-action rates and net production R_s = sum_r nu_sr w_r (zero nu skipped) */
static void ma_rates(const co_problem* p, const double* x, double* R) {
  double w[MAXR];
  for (int r = 0; r < p->nr; ++r) {
    const int a = p->reac[r][0], b = p->reac[r][1];
    w[r] = b >= 0 ? (p->k[r] * x[a]) * x[b] : p->k[r] * x[a];
  }
  for (int s = 0; s < p->S; ++s) {
    double acc = 0.0;
    for (int r = 0; r < p->nr; ++r)
      if (p->nu[s][r] != 0) acc = acc + (double)p->nu[s][r] * w[r];
    R[s] = acc;
  }
}

/* J[s][q] = sum over r (ascending), reactant slot t (ascending) of nu_sr * dw_r/dx_q */
static void ma_jacobian(const co_problem* p, const double* x, double* J) {
  const int S = p->S;
  for (int i = 0; i < S * S; ++i) J[i] = 0.0;
  for (int r = 0; r < p->nr; ++r) {
    const int a = p->reac[r][0], b = p->reac[r][1];
    for (int t = 0; t < 2; ++t) {
      const int q = p->reac[r][t];
      if (q < 0) continue;
      const double g = (t == 0) ? (b >= 0 ? p->k[r] * x[b] : p->k[r]) : p->k[r] * x[a];
      for (int s = 0; s < S; ++s)
        if (p->nu[s][r] != 0) J[s * S + q] = J[s * S + q] + (double)p->nu[s][r] * g;
    }
  }
}

static inline double bistable_R(double lam, double th, double x) { return ((lam * x) * (1.0 - x)) * (x - th); }
static inline double bistable_dR(double lam, double th, double x) {
  return lam * ((-3.0 * x * x + 2.0 * (1.0 + th) * x) - th);
}

static void adr_reaction(const co_problem* p, const double* phi, double* out) {
  const size_t nc = p->ncell;
  switch (p->d.reaction_kind) {
    case CISDC_REACTION_NONE:
      for (size_t i = 0; i < p->dim; ++i) out[i] = 0.0;
      break;
    case CISDC_REACTION_LINEAR_DECAY:
      for (size_t i = 0; i < nc; ++i) out[i] = -p->d.lambda * phi[i];
      break;
    case CISDC_REACTION_BISTABLE:
      for (size_t i = 0; i < nc; ++i) out[i] = bistable_R(p->d.lambda, p->d.theta, phi[i]);
      break;
    case CISDC_REACTION_MASS_ACTION: {
      CO_PAR(nc)
      for (size_t c = 0; c < nc; ++c) {
        double x[MAXS] = {0}, R[MAXS];
        for (int s = 0; s < p->S; ++s) x[s] = phi[(size_t)s * nc + c];
        ma_rates(p, x, R);
        for (int s = 0; s < p->S; ++s) out[(size_t)s * nc + c] = R[s];
      }
      break;
    }
  }
}

/* newton_scalar (linalg.cpp:333-349) on f(x) = (x - coef*R(x)) - b; returns trips or <0 */
static int newton_scalar_cell(const co_problem* p, double coef, double b, double* xout, long long* trips) {
  const double tol = p->d.newton_tol;
  const double lam = p->d.lambda, th = p->d.theta;
  double x = b;
  for (int it = 0; it < p->d.newton_max_iter; ++it) {
    ++*trips;
    double fx, d;
    if (p->d.reaction_kind == CISDC_REACTION_LINEAR_DECAY) {
      fx = (x - coef * (-lam * x)) - b;
    } else {
      fx = (x - coef * bistable_R(lam, th, x)) - b;
    }
    if (fabs(fx) <= tol) {
      *xout = x;
      return CISDC_OK;
    }
    if (p->d.reaction_kind == CISDC_REACTION_LINEAR_DECAY) d = 1.0 - coef * (-lam);
    else d = 1.0 - coef * bistable_dR(lam, th, x);
    if (fabs(d) < 1e-300) return -CISDC_E_SOLVE;
    const double step = fx / d;
    x -= step;
    if (fabs(step) <= tol * (1.0 + fabs(x))) {
      *xout = x;
      return CISDC_OK;
    }
  }
  return -CISDC_E_NUMERIC;
}

/* vector Newton: newton_scalar's control flow with inf-norms, Jacobian solve by
   lu_factor_dense(pivoting=true) + lu_solve; a pivot below 1e-300 is a singular Jacobian */
/* diagnostic: row interchanges performed by the vector Newton's LU (process-wide) */
long long co_pivot_swaps = 0;
long long co_get_pivot_swaps(void) { return co_pivot_swaps; }

static int newton_vector_cell(const co_problem* p, double coef, const double* b, double* x, long long* trips) {
  const int S = p->S;
  const double tol = p->d.newton_tol;
  double R[MAXS], f[MAXS], J[MAXS * MAXS], dlt[MAXS];
  int perm[MAXS];
  for (int s = 0; s < S; ++s) x[s] = b[s];
  for (int it = 0; it < p->d.newton_max_iter; ++it) {
    ++*trips;
    ma_rates(p, x, R);
    double fn = 0.0;
    for (int s = 0; s < S; ++s) {
      f[s] = (x[s] - coef * R[s]) - b[s];
      if (fabs(f[s]) > fn) fn = fabs(f[s]);
    }
    if (fn <= tol) return CISDC_OK;
    ma_jacobian(p, x, J);
    for (int s = 0; s < S; ++s)
      for (int q = 0; q < S; ++q) J[s * S + q] = (s == q ? 1.0 : 0.0) - coef * J[s * S + q];
    /* lu_factor_dense with pivoting, singular threshold as newton_scalar */
    for (int i = 0; i < S; ++i) perm[i] = i;
    for (int kk = 0; kk < S; ++kk) {
      int pv = kk;
      double best = fabs(J[kk * S + kk]);
      for (int i = kk + 1; i < S; ++i)
        if (fabs(J[i * S + kk]) > best) {
          best = fabs(J[i * S + kk]);
          pv = i;
        }
      if (pv != kk) {
        ++co_pivot_swaps;
        for (int j = 0; j < S; ++j) {
          const double t = J[kk * S + j];
          J[kk * S + j] = J[pv * S + j];
          J[pv * S + j] = t;
        }
        const int t = perm[kk];
        perm[kk] = perm[pv];
        perm[pv] = t;
      }
      const double pivot = J[kk * S + kk];
      if (fabs(pivot) < 1e-300) return -CISDC_E_SOLVE;
      for (int i = kk + 1; i < S; ++i) {
        const double m = J[i * S + kk] / pivot;
        J[i * S + kk] = m;
        for (int j = kk + 1; j < S; ++j) J[i * S + j] -= m * J[kk * S + j];
      }
    }
    co_lu_solve(S, J, perm, f, dlt);
    double sn = 0.0, xn = 0.0;
    for (int s = 0; s < S; ++s) {
      x[s] -= dlt[s];
      if (fabs(dlt[s]) > sn) sn = fabs(dlt[s]);
    }
    for (int s = 0; s < S; ++s)
      if (fabs(x[s]) > xn) xn = fabs(x[s]);
    if (sn <= tol * (1.0 + xn)) return CISDC_OK;
  }
  return -CISDC_E_NUMERIC;
}

static int adr_solve_reaction(co_problem* p, double coef, const double* rhs, double* out, cisdc_counters* c) {
  const size_t nc = p->ncell;
  long long trips = 0;
  int rc = CISDC_OK;
  if (p->d.reaction_kind == CISDC_REACTION_NONE) {
    memcpy(out, rhs, sizeof(double) * p->dim);
    return CISDC_OK;
  }
  /* cells are independent: the first failing cell (the one the reference's serial loop stops at)
     is the smallest failing index */
  size_t bad = (size_t)-1;
  int bad_r = CISDC_OK;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : trips) if (co_threads() > 1 && nc > 16384) \
    num_threads(co_threads())
  for (size_t cell = 0; cell < nc; ++cell) {
    int r;
    long long t = 0;
    if (p->d.reaction_kind == CISDC_REACTION_MASS_ACTION) {
      double b[MAXS], x[MAXS];
      for (int s = 0; s < p->S; ++s) b[s] = rhs[(size_t)s * nc + cell];
      r = newton_vector_cell(p, coef, b, x, &t);
      for (int s = 0; s < p->S; ++s) out[(size_t)s * nc + cell] = x[s];
    } else {
      r = newton_scalar_cell(p, coef, rhs[cell], &out[cell], &t);
    }
    trips += t;
    if (r != CISDC_OK) {
#pragma omp critical(co_newton_fail)
      if (cell < bad) {
        bad = cell;
        bad_r = r;
      }
    }
  }
  if (bad != (size_t)-1) {
    rc = -bad_r;
    snprintf(p->err, sizeof(p->err), "solve_reaction_implicit: cell %zu: %s", bad,
             rc == CISDC_E_SOLVE ? "newton: singular jacobian" : "newton: no convergence within the iteration cap");
    rc = CISDC_E_SOLVE; /* reaction_diffusion.cpp:178-180 wraps every failure as SolveError */
  }
  if (c) c->newton_iterations += trips;
  return rc;
}

/* 1-D periodic direct solve: (I - c Lap) on the ring, c = coef * d_s / (12 h^2), folded into a
   band of half-width 4 (order 0, n-1, 1, n-2, ...) and solved by the restated banded_solve */
static int adr_solve_diffusion_direct(co_problem* p, double coef, const double* rhs, double* out) {
  const int n = p->nx;
  const int kl = 4, ku = 4;
  static const double st[5] = {-1.0, 16.0, -30.0, 16.0, -1.0};
  int* ord = (int*)malloc(sizeof(int) * n);
  int* inv = (int*)malloc(sizeof(int) * n);
  double* band = (double*)malloc(sizeof(double) * (size_t)(kl + ku + 1) * n);
  double* bb = (double*)malloc(sizeof(double) * n);
  double* xx = (double*)malloc(sizeof(double) * n);
  int rc = CISDC_OK;
  for (int q = 0; q < n; ++q) {
    ord[q] = (q % 2 == 0) ? q / 2 : n - 1 - (q - 1) / 2;
    inv[ord[q]] = q;
  }
  for (int s = 0; s < p->S && rc == CISDC_OK; ++s) {
    const double* b = rhs + (size_t)s * n;
    double* o = out + (size_t)s * n;
    if (coef == 0.0) {
      memcpy(o, b, sizeof(double) * n);
      continue;
    }
    const double c = coef * p->cdiff[s][0];
    memset(band, 0, sizeof(double) * (size_t)(kl + ku + 1) * n);
#define BAND(i, j) band[(size_t)((j) - (i) + kl) * n + (i)]
    for (int i = 0; i < n; ++i) BAND(inv[i], inv[i]) = 1.0;
    for (int i = 0; i < n; ++i)
      for (int off = -2; off <= 2; ++off) {
        const double sv = -c * st[off + 2];
        BAND(inv[i], inv[wrap(i + off, n)]) += sv;
      }
#undef BAND
    for (int q = 0; q < n; ++q) bb[q] = b[ord[q]];
    rc = co_banded_solve(n, kl, ku, band, bb, xx, p->err);
    for (int q = 0; q < n; ++q) o[ord[q]] = xx[q];
  }
  free(ord);
  free(inv);
  free(band);
  free(bb);
  free(xx);
  return rc;
}

/* 1-D periodic direct solve as defined by the product: the exact
   circulant factorisation A = K P(Z) P(Z^-1) applied as up to four periodic linear recurrences,
   each evaluated with the blocked affine-map scan of solve1d.cuh -- same block decomposition, same
   operation order -- so the GPU result is reproduced bit for bit.  (The independent cross-check is
   the cyclic banded LU above, CISDC_DIFFUSION_BANDED_ORACLE.) */
typedef struct {
  double a00, a01, a10, a11, c0, c1;
} aff_t;

static aff_t aff_id(void) {
  aff_t r = {1.0, 0.0, 0.0, 1.0, 0.0, 0.0};
  return r;
}

static aff_t aff_then(aff_t later, aff_t earlier) {
  aff_t r;
  r.a00 = later.a00 * earlier.a00 + later.a01 * earlier.a10;
  r.a01 = later.a00 * earlier.a01 + later.a01 * earlier.a11;
  r.a10 = later.a10 * earlier.a00 + later.a11 * earlier.a10;
  r.a11 = later.a10 * earlier.a01 + later.a11 * earlier.a11;
  r.c0 = later.a00 * earlier.c0 + later.a01 * earlier.c1 + later.c0;
  r.c1 = later.a10 * earlier.c0 + later.a11 * earlier.c1 + later.c1;
  return r;
}

typedef struct {
  int npass;
  double p[4], q[4];
  int reverse[4];
  int kind[4];
  double invK;
} circ_t;

/* same explicit arithmetic as csrc/circulant.hpp factor_circulant */
static circ_t circ_factor(double c) {
  circ_t f;
  memset(&f, 0, sizeof(f));
  const double disc = 36.0 - 1.0 / c;
  if (disc >= 0.0) {
    const double r = sqrt(disc);
    const double e1 = (1.0 / c) / (6.0 + r);
    const double w1 = 2.0 + e1, w2 = 8.0 + r;
    const double z1 = 2.0 / (w1 + sqrt(e1 * (w1 + 2.0)));
    const double z2 = 2.0 / (w2 + sqrt((w2 - 2.0) * (w2 + 2.0)));
    f.npass = 2;
    for (int k = 0; k < 2; ++k) {
      f.p[k] = z1;
      f.q[k] = z2;
      f.reverse[k] = k;
      f.kind[k] = 1;
    }
    f.invK = (z1 * z2) / c;
  } else {
    const double wi = sqrt(-disc);
    const double ar = 60.0 - wi * wi, ai = 16.0 * wi;
    const double mod = sqrt(ar * ar + ai * ai);
    double sr, si;
    if (ar >= 0.0) {
      sr = sqrt((mod + ar) * 0.5);
      si = ai / (2.0 * sr);
    } else {
      si = sqrt((mod - ar) * 0.5);
      sr = ai / (2.0 * si);
    }
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

#define SCAN_T 512
#define SCAN_MAXCL 16 /* CTAs per cluster before the elements per thread grow (circulant.hpp) */
#define SCAN_NW (SCAN_T / 32)

/* rec_step of solve1d.cuh */
static double rec_step(int kind, double x, double p, double q, double* s0, double* s1) {
  if (kind == 0) {
    const double un = (x + p * *s0) - q * *s1;
    *s1 = *s0;
    *s0 = un;
    return un;
  }
  const double uu = x + p * *s0;
  const double v = uu + q * *s1;
  *s0 = uu;
  *s1 = v;
  return v;
}

/* one periodic recurrence pass over u[0..N) in exactly the evaluation order of solve1d.cuh
   (periodic_pass): per-thread chain, warp Kogge-Stone scan (32 lanes), scan of the SCAN_NW warp
   totals, cluster prefix, periodic closure, re-run */
static void scan_pass(double* u, int N, int E, int CL, int reverse, int kind, double p, double q, aff_t* excl,
                      aff_t* tot_cta) {
  aff_t m[SCAN_T], incl[32], tmp[32], wtot[32], wincl[32];
  for (int rank = 0; rank < CL; ++rank) {
    for (int tid = 0; tid < SCAN_T; ++tid) {
      const int a0 = (rank * SCAN_T + tid) * E;
      int len = N - a0;
      if (len < 0) len = 0;
      if (len > E) len = E;
      double s0 = 0.0, s1 = 0.0, a00 = 1.0, a01 = 0.0, a10 = 0.0, a11 = 1.0;
      for (int k = 0; k < len; ++k) {
        const int e = reverse ? (len - 1 - k) : k;
        rec_step(kind, u[a0 + e], p, q, &s0, &s1);
        double n00, n01, n10, n11;
        if (kind == 0) {
          n00 = p * a00 - q * a10;
          n01 = p * a01 - q * a11;
          n10 = a00;
          n11 = a01;
        } else {
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
      aff_t mm = {a00, a01, a10, a11, s0, s1};
      m[tid] = mm;
    }
    aff_t excl_lane[SCAN_T];
    for (int warp = 0; warp < SCAN_NW; ++warp) {
      const int wp = reverse ? SCAN_NW - 1 - warp : warp;
      for (int lp = 0; lp < 32; ++lp) incl[lp] = m[warp * 32 + (reverse ? 31 - lp : lp)];
      for (int off = 1; off < 32; off <<= 1) {
        for (int lp = 0; lp < 32; ++lp) tmp[lp] = lp >= off ? aff_then(incl[lp], incl[lp - off]) : incl[lp];
        memcpy(incl, tmp, sizeof(incl));
      }
      for (int lp = 0; lp < 32; ++lp) excl_lane[warp * 32 + (reverse ? 31 - lp : lp)] = lp > 0 ? incl[lp - 1] : aff_id();
      wtot[wp] = incl[31];
    }
    for (int l = 0; l < 32; ++l) wincl[l] = l < SCAN_NW ? wtot[l] : aff_id();
    for (int off = 1; off < 32; off <<= 1) {
      for (int l = 0; l < 32; ++l) tmp[l] = l >= off ? aff_then(wincl[l], wincl[l - off]) : wincl[l];
      memcpy(wincl, tmp, sizeof(wincl));
    }
    for (int tid = 0; tid < SCAN_T; ++tid) {
      const int warp = tid >> 5;
      const int wp = reverse ? SCAN_NW - 1 - warp : warp;
      const aff_t wexcl = wp > 0 ? wincl[wp - 1] : aff_id();
      excl[rank * SCAN_T + tid] = aff_then(excl_lane[tid], wexcl);
    }
    tot_cta[rank] = wincl[SCAN_NW - 1];
  }
  for (int rank = 0; rank < CL; ++rank) {
    const int vrank = reverse ? (CL - 1 - rank) : rank;
    aff_t pre = aff_id(), tot = aff_id();
    for (int v = 0; v < CL; ++v) {
      const int r = reverse ? (CL - 1 - v) : v;
      if (v < vrank) pre = aff_then(tot_cta[r], pre);
      tot = aff_then(tot_cta[r], tot);
    }
    const double m00 = 1.0 - tot.a00, m01 = -tot.a01, m10 = -tot.a10, m11 = 1.0 - tot.a11;
    const double det = m00 * m11 - m01 * m10;
    const double sa = (m11 * tot.c0 - m01 * tot.c1) / det;
    const double sb = (m00 * tot.c1 - m10 * tot.c0) / det;
    const double ca = pre.a00 * sa + pre.a01 * sb + pre.c0;
    const double cb = pre.a10 * sa + pre.a11 * sb + pre.c1;
    for (int tid = 0; tid < SCAN_T; ++tid) {
      const int a0 = (rank * SCAN_T + tid) * E;
      int len = N - a0;
      if (len < 0) len = 0;
      if (len > E) len = E;
      const aff_t ex = excl[rank * SCAN_T + tid];
      double s0 = ex.a00 * ca + ex.a01 * cb + ex.c0;
      double s1 = ex.a10 * ca + ex.a11 * cb + ex.c1;
      for (int k = 0; k < len; ++k) {
        const int e = reverse ? (len - 1 - k) : k;
        u[a0 + e] = rec_step(kind, u[a0 + e], p, q, &s0, &s1);
      }
    }
  }
}

static int adr_solve_diffusion_scan(co_problem* p, double coef, const double* rhs, double* out) {
  const int N = p->nx;
  int E = 1;
  while (E < 32 && (long long)E * SCAN_T * SCAN_MAXCL < N) E *= 2;
  const int CL = (N + E * SCAN_T - 1) / (E * SCAN_T);
  aff_t* ex = (aff_t*)malloc(sizeof(aff_t) * CL * SCAN_T);
  aff_t tot[64];
  for (int s = 0; s < p->S; ++s) {
    const double* b = rhs + (size_t)s * N;
    double* o = out + (size_t)s * N;
    const double c = coef * p->cdiff[s][0];
    memcpy(o, b, sizeof(double) * N);
    if (!(coef != 0.0 && c != 0.0)) continue;
    const circ_t f = circ_factor(c);
    for (int k = 0; k < f.npass; ++k) scan_pass(o, N, E, CL, f.reverse[k], f.kind[k], f.p[k], f.q[k], ex, tot);
    for (int i = 0; i < N; ++i) o[i] = o[i] * f.invK;
  }
  free(ex);
  return CISDC_OK;
}

/* ------------------------------------------------------------------ multigrid (2-D/3-D) */
/*
 * Cell-centred geometric multigrid for (I - coef d_s Lap4) x = b, per species, batched on the GPU
 * with identical per-point arithmetic:
 *   level l: n_l = n >> l per active axis, h_l = h * 2^l, c_la = d / (12 h_l h_l)
 *   A x   = x - coef * lap,  lap = sum_a c_la * stencil_a(x)   (stencil as Lap4 above)
 *   Jacobi: x' = x + wD * (b - A x), wD from the spectral plan (mg_plan below);
 *           from a zero guess x' = wD * b; levels used per solve = mg_plan's L
 *   restriction: mean of the 2^ndim children of (b - A x), summed x-fastest then y then z
 *   prolongation: cell-centred (bi/tri)linear, 3/4-1/4 per axis, x then y then z, periodic
 *   V-cycle: pre-smooth (first from zero below the top), restrict, recurse, correct, post-smooth;
 *            coarsest level: mg_coarse_sweeps Jacobi sweeps (first from zero)
 *   loop: x = b; while ||b - A x||_inf > tol * ||b||_inf: V-cycle (cap mg_max_cycles)
 */

typedef struct {
  int nx, ny, nz, ndim;
  double c[3];
  double coef, wD;
} mg_level_op;

static inline double mg_ax(const mg_level_op* L, const double* x, int i, int j, int k) {
  double lap = 0.0;
  for (int a = 0; a < L->ndim; ++a) {
    int n = a == 0 ? L->nx : (a == 1 ? L->ny : L->nz);
    double g[5];
    for (int o = -2; o <= 2; ++o) {
      int ii = i, jj = j, kk = k;
      if (a == 0) ii = wrap(i + o, n);
      else if (a == 1) jj = wrap(j + o, n);
      else kk = wrap(k + o, n);
      g[o + 2] = x[((size_t)kk * L->ny + jj) * L->nx + ii];
    }
    lap = lap + L->c[a] * (-g[0] + 16.0 * g[1] - 30.0 * g[2] + 16.0 * g[3] - g[4]);
  }
  return x[((size_t)k * L->ny + j) * L->nx + i] - L->coef * lap;
}

static void mg_smooth(const mg_level_op* L, const double* b, double* x, double* tmp, int from_zero) {
  const size_t n = (size_t)L->nx * L->ny * L->nz;
  if (from_zero) {
    for (size_t i = 0; i < n; ++i) x[i] = L->wD * b[i];
    return;
  }
  CO_PAR_ROWS(n)
  for (int k = 0; k < L->nz; ++k)
    for (int j = 0; j < L->ny; ++j)
      for (int i = 0; i < L->nx; ++i) {
        const size_t id = ((size_t)k * L->ny + j) * L->nx + i;
        const double r = b[id] - mg_ax(L, x, i, j, k);
        tmp[id] = x[id] + L->wD * r;
      }
  memcpy(x, tmp, sizeof(double) * n);
}

static double mg_resnorm(const mg_level_op* L, const double* b, const double* x) {
  double m = 0.0;
  const size_t n = (size_t)L->nx * L->ny * L->nz;
  /* `if (r > m) m = r` keeps the largest non-NaN residual in any order: per-thread maxima combined
     with the same rule give the serial result */
#pragma omp parallel if (co_threads() > 1 && n > 16384) num_threads(co_threads())
  {
    double mt = 0.0;
#pragma omp for schedule(static) collapse(2) nowait
  for (int k = 0; k < L->nz; ++k)
    for (int j = 0; j < L->ny; ++j)
      for (int i = 0; i < L->nx; ++i) {
        const size_t id = ((size_t)k * L->ny + j) * L->nx + i;
        const double r = fabs(b[id] - mg_ax(L, x, i, j, k));
        if (r > mt) mt = r;
      }
#pragma omp critical(co_resnorm)
    if (mt > m) m = mt;
  }
  return m;
}

static void mg_restrict(const mg_level_op* F, const double* b, const double* x, const mg_level_op* C, double* bc) {
  const double scale = F->ndim == 1 ? 0.5 : (F->ndim == 2 ? 0.25 : 0.125);
  const int ez = F->ndim >= 3 ? 2 : 1, ey = F->ndim >= 2 ? 2 : 1;
  CO_PAR_ROWS((size_t)F->nx * F->ny * F->nz)
  for (int K = 0; K < C->nz; ++K)
    for (int J = 0; J < C->ny; ++J)
      for (int I = 0; I < C->nx; ++I) {
        double acc = 0.0;
        for (int dz = 0; dz < ez; ++dz)
          for (int dy = 0; dy < ey; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
              const int i = 2 * I + dx, j = ey == 2 ? 2 * J + dy : J, k = ez == 2 ? 2 * K + dz : K;
              const size_t id = ((size_t)k * F->ny + j) * F->nx + i;
              acc = acc + (b[id] - mg_ax(F, x, i, j, k));
            }
        bc[((size_t)K * C->ny + J) * C->nx + I] = acc * scale;
      }
}

static void mg_prolong_add(const mg_level_op* F, double* x, const mg_level_op* C, const double* e) {
  CO_PAR_ROWS((size_t)F->nx * F->ny * F->nz)
  for (int k = 0; k < F->nz; ++k)
    for (int j = 0; j < F->ny; ++j)
      for (int i = 0; i < F->nx; ++i) {
        const int I = i >> 1, I2 = wrap((i & 1) ? I + 1 : I - 1, C->nx);
        int J = j, J2 = j, K = k, K2 = k;
        if (F->ndim >= 2) {
          J = j >> 1;
          J2 = wrap((j & 1) ? J + 1 : J - 1, C->ny);
        }
        if (F->ndim >= 3) {
          K = k >> 1;
          K2 = wrap((k & 1) ? K + 1 : K - 1, C->nz);
        }
#define E_(a, b_, c_) e[((size_t)(c_) * C->ny + (b_)) * C->nx + (a)]
        double v;
        if (F->ndim == 1) {
          v = 0.75 * E_(I, 0, 0) + 0.25 * E_(I2, 0, 0);
        } else if (F->ndim == 2) {
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
        const size_t id = ((size_t)k * F->ny + j) * F->nx + i;
        x[id] = x[id] + v;
      }
}

static void mg_vcycle(co_problem* p, mg_level_op* ops, int l) {
  const cisdc_problem_desc* d = &p->d;
  double* x = p->mg_x[l];
  double* b = p->mg_b[l];
  double* t = p->mg_t[l];
  if (l == p->L - 1) {
    for (int it = 0; it < d->mg_coarse_sweeps; ++it) mg_smooth(&ops[l], b, x, t, l > 0 && it == 0);
    return;
  }
  for (int it = 0; it < d->mg_pre; ++it) mg_smooth(&ops[l], b, x, t, l > 0 && it == 0);
  mg_restrict(&ops[l], b, x, &ops[l + 1], p->mg_b[l + 1]);
  mg_vcycle(p, ops, l + 1);
  mg_prolong_add(&ops[l], x, &ops[l + 1], p->mg_x[l + 1]);
  for (int it = 0; it < d->mg_post; ++it) mg_smooth(&ops[l], b, x, t, 0);
}

/* Per-solve multigrid plan (csrc/multigrid.cuh mg_plan does the same arithmetic):
 *   A_l = I - coef F_D,l has spectrum [1, Emax], Emax = 1 + coef * 64 * sum_a c_la; the modes that are
 *   high-frequency in some axis sit above Ehf = 1 + coef * 28 * min_a c_la.
 *   Weighted Jacobi with the optimal weight for the targeted interval [Elo, Emax]:
 *     wD = 2 / (Elo + Emax),  Elo = Ehf on levels that hand the smooth modes to a coarser grid,
 *                             Elo = 1 on the coarsest level used (it must reduce every mode).
 *   Coarsen below level l only while the level is stiff: (Emax - 1) / (Emax + 1) > 0.1 for the
 *   stiffest species (a well-conditioned level is solved by its own sweeps; a near-identity
 *   system -- small coef d / h^2 -- uses no coarse grid at all).
 *   The coarsest level does mg_coarse_sweeps sweeps, or mg_pre sweeps when it is the only level. */
static int mg_plan(const co_problem* p, double coef, double wD[MAXL][MAXS], double c3[MAXL][MAXS][3]) {
  const cisdc_problem_desc* d = &p->d;
  double rho[MAXL];
  double emax[MAXL][MAXS], ehf[MAXL][MAXS];
  for (int l = 0; l < p->L; ++l) {
    rho[l] = 0.0;
    for (int s = 0; s < p->S; ++s) {
      double csum = 0.0, cmin = 0.0;
      for (int a = 0; a < 3; ++a) c3[l][s][a] = 0.0;
      for (int a = 0; a < d->ndim; ++a) {
        const double hl = d->h[a] * (double)(1 << l);
        c3[l][s][a] = d->diffusivity[s] / (12.0 * hl * hl);
        csum = csum + c3[l][s][a];
        cmin = (a == 0 || c3[l][s][a] < cmin) ? c3[l][s][a] : cmin;
      }
      emax[l][s] = 1.0 + coef * (64.0 * csum);
      ehf[l][s] = 1.0 + coef * (28.0 * cmin);
      const double r = (emax[l][s] - 1.0) / (emax[l][s] + 1.0);
      rho[l] = r > rho[l] ? r : rho[l];
    }
  }
  int L = 1;
  while (L < p->L && rho[L - 1] > 0.1) ++L;
  for (int l = 0; l < L; ++l)
    for (int s = 0; s < p->S; ++s) wD[l][s] = 2.0 / ((l < L - 1 ? ehf[l][s] : 1.0) + emax[l][s]);
  return L;
}

static int adr_solve_diffusion_mg(co_problem* p, double coef, const double* rhs, double* out, cisdc_counters* c) {
  const size_t nc = p->ncell;
  double wD[MAXL][MAXS], c3[MAXL][MAXS][3];
  const int Lsave = p->L;
  const int Luse = coef == 0.0 ? 1 : mg_plan(p, coef, wD, c3);
  const int coarse_save = p->d.mg_coarse_sweeps;
  p->L = Luse;
  if (Luse == 1) p->d.mg_coarse_sweeps = p->d.mg_pre;
  for (int s = 0; s < p->S; ++s) {
    const double* b = rhs + (size_t)s * nc;
    double* o = out + (size_t)s * nc;
    if (coef == 0.0) {
      memcpy(o, b, sizeof(double) * nc);
      continue;
    }
    mg_level_op ops[MAXL];
    for (int l = 0; l < Luse; ++l) {
      ops[l].nx = p->ln[l][0];
      ops[l].ny = p->ln[l][1];
      ops[l].nz = p->ln[l][2];
      ops[l].ndim = p->d.ndim;
      ops[l].coef = coef;
      for (int a = 0; a < 3; ++a) ops[l].c[a] = c3[l][s][a];
      ops[l].wD = wD[l][s];
    }
    double bn = 0.0;
    for (size_t i = 0; i < nc; ++i)
      if (fabs(b[i]) > bn) bn = fabs(b[i]);
    memcpy(p->mg_b[0], b, sizeof(double) * nc);
    memcpy(p->mg_x[0], b, sizeof(double) * nc);
    const double thr = p->d.mg_tol * bn;
    int cyc = 0;
    for (;;) {
      const double rn = mg_resnorm(&ops[0], p->mg_b[0], p->mg_x[0]);
      if (rn <= thr) break;
      if (cyc >= p->d.mg_max_cycles) {
        snprintf(p->err, sizeof(p->err),
                 "solve_diffusion: multigrid: species %d: no convergence in %d cycles (residual %.3e, target %.3e)",
                 s, cyc, rn, thr);
        p->L = Lsave;
        p->d.mg_coarse_sweeps = coarse_save;
        return CISDC_E_NUMERIC;
      }
      mg_vcycle(p, ops, 0);
      ++cyc;
    }
    if (c) c->mg_cycles += cyc;
    memcpy(o, p->mg_x[0], sizeof(double) * nc);
  }
  p->L = Lsave;
  p->d.mg_coarse_sweeps = coarse_save;
  return CISDC_OK;
}

/* ------------------------------------------------------------------ reference RD problem */

static void rd_fill_ghosts(const co_problem* p, const double* phi, double* ext) {
  const int n = p->nx;
  memcpy(ext + 2, phi, sizeof(double) * n);
  const double phi_left = 1.0, phi_right = 0.0;
  for (int k = 0; k < 2; ++k) {
    const double* w = p->rd_w[k];
    ext[1 - k] = w[0] * phi_left + w[1] * phi[0] + w[2] * phi[1] + w[3] * phi[2] + w[4] * phi[3];
    ext[n + 2 + k] = w[0] * phi_right + w[1] * phi[n - 1] + w[2] * phi[n - 2] + w[3] * phi[n - 3] + w[4] * phi[n - 4];
  }
}

static int rd_eval(co_problem* p, int stage, const double* phi, double* out) {
  const int n = p->nx;
  if (stage == CISDC_STAGE_REACTION) {
    const double r = p->d.ref_r;
    for (int i = 0; i < n; ++i) {
      const double q = phi[i];
      out[i] = r * q * (q - 1.0) * (q - 0.5);
    }
    return CISDC_OK;
  }
  double* g = (double*)malloc(sizeof(double) * (n + 4));
  rd_fill_ghosts(p, phi, g);
  if (stage == CISDC_STAGE_ADVECTION) {
    const double c = p->d.ref_a / (12.0 * p->rd_dx);
    for (int i = 0; i < n; ++i) {
      const int k = i + 2;
      out[i] = c * (g[k - 2] - 8.0 * g[k - 1] + 8.0 * g[k + 1] - g[k + 2]);
    }
  } else {
    const double c = p->d.ref_d / (12.0 * p->rd_dx * p->rd_dx);
    for (int i = 0; i < n; ++i) {
      const int k = i + 2;
      out[i] = c * (-g[k - 2] + 16.0 * g[k - 1] - 30.0 * g[k] + 16.0 * g[k + 1] - g[k + 2]);
    }
  }
  free(g);
  return CISDC_OK;
}

static int rd_solve_diffusion(co_problem* p, double coef, const double* rhs, double* out) {
  const int n = p->nx;
  if (coef == 0.0) {
    memcpy(out, rhs, sizeof(double) * n);
    return CISDC_OK;
  }
  static const double kLap[5] = {-1.0, 16.0, -30.0, 16.0, -1.0};
  const int kl = 3, ku = 3;
  double* band = (double*)calloc((size_t)(kl + ku + 1) * n, sizeof(double));
  double* b = (double*)malloc(sizeof(double) * n);
  const double c = coef * p->d.ref_d / (12.0 * p->rd_dx * p->rd_dx);
  memcpy(b, rhs, sizeof(double) * n);
#define A_(i, j) band[(size_t)((j) - (i) + kl) * n + (i)]
  for (int i = 0; i < n; ++i) A_(i, i) = 1.0;
  for (int i = 0; i < n; ++i) {
    for (int o = -2; o <= 2; ++o) {
      const double s = -c * kLap[o + 2];
      const int j = i + o;
      if (j >= 0 && j < n) {
        A_(i, j) += s;
      } else if (j < 0) {
        const double* w = p->rd_w[-j - 1];
        for (int q = 0; q < 4; ++q) A_(i, q) += s * w[q + 1];
        b[i] -= s * w[0] * 1.0;
      } else {
        const double* w = p->rd_w[j - n];
        for (int q = 0; q < 4; ++q) A_(i, n - 1 - q) += s * w[q + 1];
        b[i] -= s * w[0] * 0.0;
      }
    }
  }
#undef A_
  const int rc = co_banded_solve(n, kl, ku, band, b, out, p->err);
  free(band);
  free(b);
  return rc;
}

static int rd_solve_reaction(co_problem* p, double coef, const double* rhs, double* out, cisdc_counters* cnt) {
  const int n = p->nx;
  const double r = p->d.ref_r;
  const double tol = 1e-14;
  const int max_iter = 50;
  long long trips = 0;
  for (int i = 0; i < n; ++i) {
    const double bi = rhs[i];
    double x = bi;
    int done = 0, code = CISDC_E_NUMERIC;
    for (int it = 0; it < max_iter; ++it) {
      ++trips;
      const double fx = x - coef * r * x * (x - 1.0) * (x - 0.5) - bi;
      if (fabs(fx) <= tol) {
        done = 1;
        break;
      }
      const double d = 1.0 - coef * r * (3.0 * x * x - 3.0 * x + 0.5);
      if (fabs(d) < 1e-300) {
        code = CISDC_E_SOLVE;
        break;
      }
      const double step = fx / d;
      x -= step;
      if (fabs(step) <= tol * (1.0 + fabs(x))) {
        done = 1;
        break;
      }
    }
    if (!done) {
      snprintf(p->err, sizeof(p->err), "solve_reaction_implicit: cell %d: %s", i,
               code == CISDC_E_SOLVE ? "newton_scalar: singular jacobian"
                                     : "newton_scalar: no convergence in 50 iterations");
      if (cnt) cnt->newton_iterations += trips;
      return CISDC_E_SOLVE;
    }
    out[i] = x;
  }
  if (cnt) cnt->newton_iterations += trips;
  return CISDC_OK;
}

/* ------------------------------------------------------------------ coupled D+R stage (periodic ADR)
 *
 * OperatorSplitProblem::solve_coupled (operator_split.hpp:49-53): phi - coef (F_D(phi) + F_R(phi)) = rhs.
 * The reference PDE class provides none; the periodic ADR class defines it (cisdc_gpu.h, "coupled
 * stage") as the fixed point of the alternating diffusion / reaction stage solves -- the nested
 * iteration of cisdcq_cells at one node (integrators.cpp:195-258), whose limit is the coupled solve
 * (test_integrators.cpp:195-213) -- run to convergence:
 *   y_0 = rhs;  z = solve_D(coef, rhs + coef F_R(y_k));  y_{k+1} = solve_R(coef, rhs + coef F_D(z));
 *   stop when max|y_{k+1} - y_k| <= coupled_tol * max|y_{k+1}|; SolveError after coupled_max_iter. */
static int adr_solve_diffusion_any(co_problem* p, double coef, const double* rhs, double* out, cisdc_counters* c) {
  if (p->d.diffusion_solver == CISDC_DIFFUSION_DIRECT) return adr_solve_diffusion_scan(p, coef, rhs, out);
  if (p->d.diffusion_solver == CISDC_DIFFUSION_BANDED_ORACLE) return adr_solve_diffusion_direct(p, coef, rhs, out);
  return adr_solve_diffusion_mg(p, coef, rhs, out, c);
}

static int adr_solve_coupled(co_problem* p, double coef, const double* rhs, double* out, cisdc_counters* c) {
  const size_t n = p->dim;
  if (coef == 0.0) {
    memmove(out, rhs, sizeof(double) * n);
    return CISDC_OK;
  }
  double* y = (double*)malloc(sizeof(double) * n);
  double* f = (double*)malloc(sizeof(double) * n);
  double* b = (double*)malloc(sizeof(double) * n);
  double* z = (double*)malloc(sizeof(double) * n);
  double* yn = (double*)malloc(sizeof(double) * n);
  int rc = CISDC_OK, converged = 0;
  memcpy(y, rhs, sizeof(double) * n);
  for (int it = 0; it < p->d.coupled_max_iter && !converged; ++it) {
    adr_reaction(p, y, f);
    for (size_t i = 0; i < n; ++i) b[i] = rhs[i] + coef * f[i];
    rc = adr_solve_diffusion_any(p, coef, b, z, c);
    if (rc) break;
    adr_diffusion(p, z, f);
    for (size_t i = 0; i < n; ++i) b[i] = rhs[i] + coef * f[i];
    rc = adr_solve_reaction(p, coef, b, yn, c);
    if (rc) break;
    double delta = 0.0, scale = 0.0;
    for (size_t i = 0; i < n; ++i) {
      const double d = fabs(yn[i] - y[i]), a = fabs(yn[i]);
      if (d > delta) delta = d;
      if (a > scale) scale = a;
    }
    double* t = y;
    y = yn;
    yn = t;
    converged = delta <= p->d.coupled_tol * scale;
  }
  if (!rc && !converged) rc = fail(p, CISDC_E_SOLVE, "periodic ADR: coupled solve did not converge");
  if (!rc) memcpy(out, y, sizeof(double) * n);
  free(y);
  free(f);
  free(b);
  free(z);
  free(yn);
  return rc;
}

/* ------------------------------------------------------------------ dispatch */

int co_eval(co_problem* p, int stage, const double* phi, double* out) {
  switch (p->d.kind) {
    case CISDC_PROBLEM_LINEAR_SCALAR: {
      const double c = stage == CISDC_STAGE_ADVECTION ? p->d.ref_a : (stage == CISDC_STAGE_DIFFUSION ? p->d.ref_d : p->d.ref_r);
      for (size_t i = 0; i < p->dim; ++i) out[i] = c * phi[i];  /* linear.cpp:19-30 per element */
      return CISDC_OK;
    }
    case CISDC_PROBLEM_REFERENCE_RD:
      return rd_eval(p, stage, phi, out);
    default:
      if (stage == CISDC_STAGE_ADVECTION) adr_advection(p, phi, out);
      else if (stage == CISDC_STAGE_DIFFUSION) adr_diffusion(p, phi, out);
      else adr_reaction(p, phi, out);
      return CISDC_OK;
  }
}

int co_solve(co_problem* p, int stage, double coef, const double* rhs, double* out, cisdc_counters* c) {
  switch (p->d.kind) {
    case CISDC_PROBLEM_LINEAR_SCALAR: {
      double denom;
      const char* what;
      if (stage == CISDC_STAGE_DIFFUSION) {
        denom = 1.0 - coef * p->d.ref_d;
        what = "LinearScalarProblem: singular diffusion stage";
      } else if (stage == CISDC_STAGE_REACTION) {
        denom = 1.0 - coef * p->d.ref_r;
        what = "LinearScalarProblem: singular reaction stage";
      } else {
        denom = 1.0 - coef * (p->d.ref_d + p->d.ref_r);
        what = "LinearScalarProblem: singular coupled stage";
      }
      if (denom == 0.0) return fail(p, CISDC_E_SOLVE, what);
      for (size_t i = 0; i < p->dim; ++i) out[i] = rhs[i] / denom;  /* linear.cpp:32-50 per element */
      return CISDC_OK;
    }
    case CISDC_PROBLEM_REFERENCE_RD:
      if (stage == CISDC_STAGE_DIFFUSION) return rd_solve_diffusion(p, coef, rhs, out);
      if (stage == CISDC_STAGE_REACTION) return rd_solve_reaction(p, coef, rhs, out, c);
      return fail(p, CISDC_E_CAPABILITY, "OperatorSplitProblem: coupled diffusion-reaction solve not provided");
    default:
      if (stage == CISDC_STAGE_DIFFUSION) {
        if (p->d.diffusion_solver == CISDC_DIFFUSION_DIRECT) return adr_solve_diffusion_scan(p, coef, rhs, out);
        if (p->d.diffusion_solver == CISDC_DIFFUSION_BANDED_ORACLE) return adr_solve_diffusion_direct(p, coef, rhs, out);
        return adr_solve_diffusion_mg(p, coef, rhs, out, c);
      }
      if (stage == CISDC_STAGE_REACTION) return adr_solve_reaction(p, coef, rhs, out, c);
      if (p->d.coupled_max_iter > 0) return adr_solve_coupled(p, coef, rhs, out, c);
      return fail(p, CISDC_E_CAPABILITY, "OperatorSplitProblem: coupled diffusion-reaction solve not provided");
  }
}
