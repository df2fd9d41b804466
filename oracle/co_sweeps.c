/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY (see cisdc_oracle.h).
 * Sweep state and sweep engines restated from the reference, same operand order:
 *   SweepState ctor / initialize / set_node_values  proj/core/src/sweep_state.cpp:22-58
 *   increment_norm                                   proj/core/src/sweep_state.cpp:60-66
 *   quadrature_base                                  proj/core/src/integrators.cpp:52-65
 *   misdc_sweep                                      proj/core/src/integrators.cpp:69-101
 *   misdcq_sweep                                     proj/core/src/integrators.cpp:103-143
 *   imexq_sweep                                      proj/core/src/integrators.cpp:145-173
 *   cisdcq_cells::{resize,run_diffusion_cell,run_reaction_cell,finalize}
 *                                                    proj/core/src/integrators.cpp:175-271
 *   cisdcq_sweep / run_sweep / integrate             proj/core/src/integrators.cpp:273-333
 * (execute_pipelined, pipeline.cpp:171-320, is bitwise identical to cisdcq_sweep by construction;
 *  the oracle runs the serial cell order.)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "cisdc_oracle.h"

struct co_state {
  int M;
  size_t dim;
  double* buf;  /* 5 (M+1) fields */
};

static double* F(co_state* s, int which, int m) { return s->buf + ((size_t)which * (s->M + 1) + m) * s->dim; }

co_state* co_state_create(int M, size_t dim) {
  if (M < 1 || dim == 0) return NULL;
  co_state* s = (co_state*)malloc(sizeof(co_state));
  s->M = M;
  s->dim = dim;
  s->buf = (double*)calloc((size_t)5 * (M + 1) * dim, sizeof(double));
  if (!s->buf) {
    free(s);
    return NULL;
  }
  return s;
}

void co_state_destroy(co_state* s) {
  if (!s) return;
  free(s->buf);
  free(s);
}

double* co_state_field(co_state* s, int which, int node) { return F(s, which, node); }

int co_state_initialize(co_state* s, co_problem* p, const double* phi0) {
  const size_t n = s->dim;
  double* a = (double*)malloc(sizeof(double) * n);
  double* d = (double*)malloc(sizeof(double) * n);
  double* r = (double*)malloc(sizeof(double) * n);
  int rc = co_eval(p, CISDC_STAGE_ADVECTION, phi0, a);
  if (!rc) rc = co_eval(p, CISDC_STAGE_DIFFUSION, phi0, d);
  if (!rc) rc = co_eval(p, CISDC_STAGE_REACTION, phi0, r);
  for (int m = 0; m <= s->M && !rc; ++m) {
    memcpy(F(s, CISDC_FIELD_PHI, m), phi0, sizeof(double) * n);
    memcpy(F(s, CISDC_FIELD_FA, m), a, sizeof(double) * n);
    memcpy(F(s, CISDC_FIELD_FD, m), d, sizeof(double) * n);
    memcpy(F(s, CISDC_FIELD_FR, m), r, sizeof(double) * n);
  }
  free(a);
  free(d);
  free(r);
  return rc;
}

int co_state_set_nodes(co_state* s, co_problem* p, const double* values) {
  for (int m = 0; m <= s->M; ++m) {
    memcpy(F(s, CISDC_FIELD_PHI, m), values + (size_t)m * s->dim, sizeof(double) * s->dim);
    int rc = co_eval(p, CISDC_STAGE_ADVECTION, F(s, CISDC_FIELD_PHI, m), F(s, CISDC_FIELD_FA, m));
    if (!rc) rc = co_eval(p, CISDC_STAGE_DIFFUSION, F(s, CISDC_FIELD_PHI, m), F(s, CISDC_FIELD_FD, m));
    if (!rc) rc = co_eval(p, CISDC_STAGE_REACTION, F(s, CISDC_FIELD_PHI, m), F(s, CISDC_FIELD_FR, m));
    if (rc) return rc;
  }
  return CISDC_OK;
}

double co_increment_norm(const double* a, const double* b, size_t n) {
  if (n == 1) return fabs(a[0] - b[0]);
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += fabs(a[i] - b[i]);
  return s / (double)n;
}

/* ------------------------------------------------------------------ helpers */

typedef struct {
  int M;
  size_t n;
  double* fa;  /* (M+1) x n snapshots of sweep (k) */
  double* fd;
  double* fr;
} snap_t;

static int snap_take(co_state* s, snap_t* sn) {
  const size_t sz = sizeof(double) * (size_t)(s->M + 1) * s->dim;
  sn->M = s->M;
  sn->n = s->dim;
  sn->fa = (double*)malloc(sz);
  sn->fd = (double*)malloc(sz);
  sn->fr = (double*)malloc(sz);
  memcpy(sn->fa, F(s, CISDC_FIELD_FA, 0), sz);
  memcpy(sn->fd, F(s, CISDC_FIELD_FD, 0), sz);
  memcpy(sn->fr, F(s, CISDC_FIELD_FR, 0), sz);
  return 0;
}
static void snap_free(snap_t* sn) {
  free(sn->fa);
  free(sn->fd);
  free(sn->fr);
}
#define SN(arr, j) ((arr) + (size_t)(j) * n)

#define QT(t, m, j) ((t)->Q[(m) * ((t)->M + 1) + (j)])
#define ST(t, m, j) ((t)->S[(m) * ((t)->M + 1) + (j)])
#define QI(t, m, j) ((t)->QtI[(m) * (t)->M + (j)])
#define QE(t, m, j) ((t)->QtE[(m) * (t)->M + (j)])

/* quadrature_base (integrators.cpp:52-65) */
static void quadrature_base(const double* phi0, const cisdc_tables* tb, int row, double dt, const double* fa,
                            const double* fd, const double* fr, size_t n, double* rhs) {
  const int M = tb->M;
  for (size_t i = 0; i < n; ++i) rhs[i] = phi0[i];
  for (int j = 0; j <= M; ++j) {
    const double c = dt * QT(tb, row, j);
    const double* a = SN(fa, j);
    const double* d = SN(fd, j);
    const double* r = SN(fr, j);
    for (size_t i = 0; i < n; ++i) rhs[i] += c * (a[i] + d[i] + r[i]);
  }
}

#define CALL(x)             \
  do {                      \
    rc = (x);               \
    if (rc) goto done;      \
  } while (0)

static int eval3(co_problem* p, const double* phi, double* a, double* d, double* r) {
  int rc = co_eval(p, CISDC_STAGE_ADVECTION, phi, a);
  if (!rc) rc = co_eval(p, CISDC_STAGE_DIFFUSION, phi, d);
  if (!rc) rc = co_eval(p, CISDC_STAGE_REACTION, phi, r);
  return rc;
}

/* ------------------------------------------------------------------ misdc (integrators.cpp:69-101) */
static int misdc_sweep(co_state* s, const cisdc_tables* tb, co_problem* p, double dt, cisdc_counters* c) {
  const int M = s->M;
  const size_t n = s->dim;
  int rc = 0;
  snap_t sp;
  snap_take(s, &sp);
  double* base = (double*)malloc(sizeof(double) * n);
  double* rhs = (double*)malloc(sizeof(double) * n);
  double* fd_ad = (double*)malloc(sizeof(double) * n);
  for (int m = 0; m < M; ++m) {
    const double dtm = dt * tb->dtau[m];
    const double* phim = F(s, CISDC_FIELD_PHI, m);
    for (size_t i = 0; i < n; ++i) base[i] = phim[i];
    for (int j = 0; j <= M; ++j) {
      const double cc = dt * ST(tb, m, j);
      for (size_t i = 0; i < n; ++i) base[i] += cc * (SN(sp.fa, j)[i] + SN(sp.fd, j)[i] + SN(sp.fr, j)[i]);
    }
    const double* fam = F(s, CISDC_FIELD_FA, m);
    for (size_t i = 0; i < n; ++i) rhs[i] = base[i] + dtm * (fam[i] - SN(sp.fa, m)[i] - SN(sp.fd, m + 1)[i]);
    CALL(co_solve(p, CISDC_STAGE_DIFFUSION, dtm, rhs, F(s, CISDC_FIELD_PHI_AD, m + 1), c));
    if (c) ++c->diffusion;
    CALL(co_eval(p, CISDC_STAGE_DIFFUSION, F(s, CISDC_FIELD_PHI_AD, m + 1), fd_ad));
    for (size_t i = 0; i < n; ++i)
      rhs[i] = base[i] + dtm * (fam[i] - SN(sp.fa, m)[i] + fd_ad[i] - SN(sp.fd, m + 1)[i] - SN(sp.fr, m + 1)[i]);
    CALL(co_solve(p, CISDC_STAGE_REACTION, dtm, rhs, F(s, CISDC_FIELD_PHI, m + 1), c));
    if (c) ++c->reaction;
    CALL(eval3(p, F(s, CISDC_FIELD_PHI, m + 1), F(s, CISDC_FIELD_FA, m + 1), F(s, CISDC_FIELD_FD, m + 1),
               F(s, CISDC_FIELD_FR, m + 1)));
  }
done:
  snap_free(&sp);
  free(base);
  free(rhs);
  free(fd_ad);
  return rc;
}

/* ------------------------------------------------------------------ misdcq (integrators.cpp:103-143) */
static int misdcq_sweep(co_state* s, const cisdc_tables* tb, co_problem* p, double dt, cisdc_counters* c) {
  const int M = s->M;
  const size_t n = s->dim;
  int rc = 0;
  snap_t sp;
  snap_take(s, &sp);
  double* base = (double*)malloc(sizeof(double) * n);
  double* rhs = (double*)malloc(sizeof(double) * n);
  double* fd_ad = (double*)malloc(sizeof(double) * n);
  for (int m = 0; m < M; ++m) {
    quadrature_base(F(s, CISDC_FIELD_PHI, 0), tb, m, dt, sp.fa, sp.fd, sp.fr, n, base);
    const double coef = dt * QI(tb, m, m);
    for (size_t i = 0; i < n; ++i) rhs[i] = base[i];
    for (int j = 1; j <= m; ++j) {
      const double cE = dt * QE(tb, m, j - 1);
      const double cI = dt * QI(tb, m, j - 1);
      const double* faj = F(s, CISDC_FIELD_FA, j);
      const double* fdj = F(s, CISDC_FIELD_FD, j);
      for (size_t i = 0; i < n; ++i)
        rhs[i] += cE * (faj[i] - SN(sp.fa, j)[i]) + cI * (fdj[i] - SN(sp.fd, j)[i]);
    }
    for (size_t i = 0; i < n; ++i) rhs[i] -= coef * SN(sp.fd, m + 1)[i];
    CALL(co_solve(p, CISDC_STAGE_DIFFUSION, coef, rhs, F(s, CISDC_FIELD_PHI_AD, m + 1), c));
    if (c) ++c->diffusion;
    CALL(co_eval(p, CISDC_STAGE_DIFFUSION, F(s, CISDC_FIELD_PHI_AD, m + 1), fd_ad));
    for (size_t i = 0; i < n; ++i) rhs[i] = base[i];
    for (int j = 1; j <= m; ++j) {
      const double cE = dt * QE(tb, m, j - 1);
      const double cI = dt * QI(tb, m, j - 1);
      const double* faj = F(s, CISDC_FIELD_FA, j);
      const double* fdj = F(s, CISDC_FIELD_FD, j);
      const double* frj = F(s, CISDC_FIELD_FR, j);
      for (size_t i = 0; i < n; ++i)
        rhs[i] += cE * (faj[i] - SN(sp.fa, j)[i]) + cI * (fdj[i] - SN(sp.fd, j)[i] + frj[i] - SN(sp.fr, j)[i]);
    }
    for (size_t i = 0; i < n; ++i) rhs[i] += coef * (fd_ad[i] - SN(sp.fd, m + 1)[i] - SN(sp.fr, m + 1)[i]);
    CALL(co_solve(p, CISDC_STAGE_REACTION, coef, rhs, F(s, CISDC_FIELD_PHI, m + 1), c));
    if (c) ++c->reaction;
    CALL(eval3(p, F(s, CISDC_FIELD_PHI, m + 1), F(s, CISDC_FIELD_FA, m + 1), F(s, CISDC_FIELD_FD, m + 1),
               F(s, CISDC_FIELD_FR, m + 1)));
  }
done:
  snap_free(&sp);
  free(base);
  free(rhs);
  free(fd_ad);
  return rc;
}

/* ------------------------------------------------------------------ imexq (integrators.cpp:145-173) */
static int imexq_sweep(co_state* s, const cisdc_tables* tb, co_problem* p, double dt, cisdc_counters* c) {
  if (!co_problem_has_coupled(p)) return CISDC_E_CAPABILITY;
  const int M = s->M;
  const size_t n = s->dim;
  int rc = 0;
  snap_t sp;
  snap_take(s, &sp);
  double* rhs = (double*)malloc(sizeof(double) * n);
  for (int m = 0; m < M; ++m) {
    quadrature_base(F(s, CISDC_FIELD_PHI, 0), tb, m, dt, sp.fa, sp.fd, sp.fr, n, rhs);
    for (int j = 1; j <= m; ++j) {
      const double cE = dt * QE(tb, m, j - 1);
      const double cI = dt * QI(tb, m, j - 1);
      const double* faj = F(s, CISDC_FIELD_FA, j);
      const double* fdj = F(s, CISDC_FIELD_FD, j);
      const double* frj = F(s, CISDC_FIELD_FR, j);
      for (size_t i = 0; i < n; ++i)
        rhs[i] += cE * (faj[i] - SN(sp.fa, j)[i]) + cI * (fdj[i] - SN(sp.fd, j)[i] + frj[i] - SN(sp.fr, j)[i]);
    }
    const double coef = dt * QI(tb, m, m);
    for (size_t i = 0; i < n; ++i) rhs[i] -= coef * (SN(sp.fd, m + 1)[i] + SN(sp.fr, m + 1)[i]);
    CALL(co_solve(p, 3, coef, rhs, F(s, CISDC_FIELD_PHI, m + 1), c));
    if (c) ++c->coupled;
    memcpy(F(s, CISDC_FIELD_PHI_AD, m + 1), F(s, CISDC_FIELD_PHI, m + 1), sizeof(double) * n);
    CALL(eval3(p, F(s, CISDC_FIELD_PHI, m + 1), F(s, CISDC_FIELD_FA, m + 1), F(s, CISDC_FIELD_FD, m + 1),
               F(s, CISDC_FIELD_FR, m + 1)));
  }
done:
  snap_free(&sp);
  free(rhs);
  return rc;
}

/* ------------------------------------------------------------------ cisdcq (integrators.cpp:175-288) */
typedef struct {
  int M, nu;
  size_t n;
  double *phi_ad, *fa_ad, *fd_ad, *phi_r, *fa_r, *fd_r, *fr_r; /* (M*nu) x n each */
} ws_t;

static size_t slot(const ws_t* w, int m, int ell) { return (size_t)(ell - 1) * w->M + (m - 1); }
#define WS(arr, sl) ((arr) + (sl) * n)

static int run_diffusion_cell(int m, int ell, co_state* in, const cisdc_tables* tb, co_problem* p, double dt,
                              ws_t* ws, cisdc_counters* c) {
  const size_t n = ws->n;
  const int row = m - 1;
  const int M = in->M;
  double* rhs = (double*)malloc(sizeof(double) * n);
  int rc = 0;
  const double* fa = F(in, CISDC_FIELD_FA, 0);
  const double* fd = F(in, CISDC_FIELD_FD, 0);
  const double* fr = F(in, CISDC_FIELD_FR, 0);
  (void)M;
  quadrature_base(F(in, CISDC_FIELD_PHI, 0), tb, row, dt, fa, fd, fr, n, rhs);
  for (int j = 1; j <= m - 2; ++j) {
    const double cE = dt * QE(tb, row, j - 1);
    const double cI = dt * QI(tb, row, j - 1);
    const size_t sj = slot(ws, j, ell);
    for (size_t i = 0; i < n; ++i)
      rhs[i] += cE * (WS(ws->fa_r, sj)[i] - SN(fa, j)[i]) +
                cI * (WS(ws->fd_r, sj)[i] - SN(fd, j)[i] + WS(ws->fr_r, sj)[i] - SN(fr, j)[i]);
  }
  if (m >= 2) {
    const double cE = dt * QE(tb, row, m - 2);
    const double cI = dt * QI(tb, row, m - 2);
    const double* lag_fa = (ell == 1) ? WS(ws->fa_ad, slot(ws, m - 1, 1)) : WS(ws->fa_r, slot(ws, m - 1, ell - 1));
    const double* lag_fd = (ell == 1) ? WS(ws->fd_ad, slot(ws, m - 1, 1)) : WS(ws->fd_r, slot(ws, m - 1, ell - 1));
    const double* lag_fr = (ell == 1) ? SN(fr, m - 1) : WS(ws->fr_r, slot(ws, m - 1, ell - 1));
    for (size_t i = 0; i < n; ++i)
      rhs[i] += cE * (lag_fa[i] - SN(fa, m - 1)[i]) +
                cI * (lag_fd[i] - SN(fd, m - 1)[i] + lag_fr[i] - SN(fr, m - 1)[i]);
  }
  const double coef = dt * QI(tb, row, m - 1);
  const double* lag_fr_m = (ell == 1) ? SN(fr, m) : WS(ws->fr_r, slot(ws, m, ell - 1));
  for (size_t i = 0; i < n; ++i) rhs[i] += coef * (lag_fr_m[i] - SN(fr, m)[i]) - coef * SN(fd, m)[i];
  const size_t s = slot(ws, m, ell);
  rc = co_solve(p, CISDC_STAGE_DIFFUSION, coef, rhs, WS(ws->phi_ad, s), c);
  if (!rc && c) ++c->diffusion;
  if (!rc && ell == 1) {
    rc = co_eval(p, CISDC_STAGE_ADVECTION, WS(ws->phi_ad, s), WS(ws->fa_ad, s));
    if (!rc) rc = co_eval(p, CISDC_STAGE_DIFFUSION, WS(ws->phi_ad, s), WS(ws->fd_ad, s));
  }
  free(rhs);
  return rc;
}

static int run_reaction_cell(int m, int ell, co_state* in, const cisdc_tables* tb, co_problem* p, double dt,
                             ws_t* ws, cisdc_counters* c) {
  const size_t n = ws->n;
  const int row = m - 1;
  const size_t s = slot(ws, m, ell);
  const double* fr = F(in, CISDC_FIELD_FR, 0);
  double* rhs = (double*)malloc(sizeof(double) * n);
  memcpy(rhs, WS(ws->phi_ad, s), sizeof(double) * n);
  if (m >= 2) {
    const double cI = dt * QI(tb, row, m - 2);
    const double* fr_new = WS(ws->fr_r, slot(ws, m - 1, ell));
    const double* lag_fr = (ell == 1) ? SN(fr, m - 1) : WS(ws->fr_r, slot(ws, m - 1, ell - 1));
    for (size_t i = 0; i < n; ++i) rhs[i] += cI * (fr_new[i] - lag_fr[i]);
  }
  const double coef = dt * QI(tb, row, m - 1);
  const double* lag_fr_m = (ell == 1) ? SN(fr, m) : WS(ws->fr_r, slot(ws, m, ell - 1));
  for (size_t i = 0; i < n; ++i) rhs[i] -= coef * lag_fr_m[i];
  int rc = co_solve(p, CISDC_STAGE_REACTION, coef, rhs, WS(ws->phi_r, s), c);
  if (!rc && c) ++c->reaction;
  if (!rc) rc = eval3(p, WS(ws->phi_r, s), WS(ws->fa_r, s), WS(ws->fd_r, s), WS(ws->fr_r, s));
  free(rhs);
  return rc;
}

static int cisdcq_sweep(co_state* st, const cisdc_tables* tb, co_problem* p, double dt, int nu, cisdc_counters* c) {
  if (nu < 1) return CISDC_E_INVALID_ARGUMENT;
  const int M = st->M;
  const size_t n = st->dim;
  ws_t ws;
  ws.M = M;
  ws.nu = nu;
  ws.n = n;
  const size_t cells = (size_t)M * nu;
  double** arrs[7] = {&ws.phi_ad, &ws.fa_ad, &ws.fd_ad, &ws.phi_r, &ws.fa_r, &ws.fd_r, &ws.fr_r};
  for (int a = 0; a < 7; ++a) *arrs[a] = (double*)calloc(cells * n, sizeof(double));
  int rc = 0;
  for (int ell = 1; ell <= nu && !rc; ++ell) {
    for (int m = 1; m <= M && !rc; ++m) {
      rc = run_diffusion_cell(m, ell, st, tb, p, dt, &ws, c);
      if (!rc) rc = run_reaction_cell(m, ell, st, tb, p, dt, &ws, c);
    }
  }
  if (!rc) {
    for (int m = 1; m <= M; ++m) {
      const size_t s = slot(&ws, m, nu);
      memcpy(F(st, CISDC_FIELD_PHI, m), WS(ws.phi_r, s), sizeof(double) * n);
      memcpy(F(st, CISDC_FIELD_FA, m), WS(ws.fa_r, s), sizeof(double) * n);
      memcpy(F(st, CISDC_FIELD_FD, m), WS(ws.fd_r, s), sizeof(double) * n);
      memcpy(F(st, CISDC_FIELD_FR, m), WS(ws.fr_r, s), sizeof(double) * n);
      memcpy(F(st, CISDC_FIELD_PHI_AD, m), WS(ws.phi_ad, s), sizeof(double) * n);
    }
  }
  for (int a = 0; a < 7; ++a) free(*arrs[a]);
  return rc;
}

int co_run_sweep(int scheme, co_state* s, const cisdc_tables* tb, co_problem* p, double dt, int nu,
                 cisdc_counters* c) {
  if (s->M != tb->M) return CISDC_E_INVALID_ARGUMENT;
  if (s->dim != co_problem_dim(p)) return CISDC_E_INVALID_ARGUMENT;
  switch (scheme) {
    case CISDC_SCHEME_MISDC: return misdc_sweep(s, tb, p, dt, c);
    case CISDC_SCHEME_MISDCQ: return misdcq_sweep(s, tb, p, dt, c);
    case CISDC_SCHEME_CISDCQ: return cisdcq_sweep(s, tb, p, dt, nu, c);
    case CISDC_SCHEME_IMEXQ: return imexq_sweep(s, tb, p, dt, c);
  }
  return CISDC_E_INVALID_ARGUMENT;
}

/* integrate (integrators.cpp:301-333) */
int co_integrate(co_problem* p, const double* phi0, const cisdc_integrate_options* opt, double* final_state,
                 cisdc_step_report* reports, double* increments, char* err) {
  if (opt->n_sweeps < 1) {
    if (err) snprintf(err, 1024, "integrate: n_sweeps must be >= 1");
    return CISDC_E_INVALID_ARGUMENT;
  }
  if (opt->scheme == CISDC_SCHEME_CISDCQ && opt->nu < 1) {
    if (err) snprintf(err, 1024, "integrate: nu must be >= 1");
    return CISDC_E_INVALID_ARGUMENT;
  }
  cisdc_tables tb;
  if (co_make_tables(opt->M, opt->convention, &tb)) {
    if (err) snprintf(err, 1024, "make_quadrature_tables failed");
    return CISDC_E_INVALID_ARGUMENT;
  }
  const size_t n = co_problem_dim(p);
  co_state* st = co_state_create(opt->M, n);
  double* start = (double*)malloc(sizeof(double) * n);
  double* prev = (double*)malloc(sizeof(double) * n);
  memcpy(start, phi0, sizeof(double) * n);
  int rc = 0;
  for (int step = 0; step < opt->n_steps && !rc; ++step) {
    rc = co_state_initialize(st, p, start);
    if (rc) break;
    cisdc_step_report rep;
    memset(&rep, 0, sizeof(rep));
    memcpy(prev, F(st, CISDC_FIELD_PHI, opt->M), sizeof(double) * n);
    int k;
    for (k = 1; k <= opt->n_sweeps; ++k) {
      rc = co_run_sweep(opt->scheme, st, &tb, p, opt->dt, opt->nu, &rep.counters);
      if (rc) {
        if (err)
          snprintf(err, 1024, "integrate: step %d, sweep %d: %s", step + 1, k,
                   rc == CISDC_E_CAPABILITY ? "imexq_sweep: problem provides no coupled diffusion-reaction solve"
                                            : co_problem_error(p));
        rc = CISDC_E_SOLVE; /* integrate rethrows every stage failure as SolveError (:317-322) */
        break;
      }
      const double inc = co_increment_norm(F(st, CISDC_FIELD_PHI, opt->M), prev, n);
      if (increments) increments[(size_t)step * opt->n_sweeps + (k - 1)] = inc;
      memcpy(prev, F(st, CISDC_FIELD_PHI, opt->M), sizeof(double) * n);
      if (opt->has_stop_tol && inc <= opt->stop_tol) {
        ++k;
        break;
      }
    }
    if (rc) break;
    rep.sweeps = k - 1;
    if (reports) reports[step] = rep;
    memcpy(start, F(st, CISDC_FIELD_PHI, opt->M), sizeof(double) * n);
  }
  if (!rc) memcpy(final_state, start, sizeof(double) * n);
  co_state_destroy(st);
  free(start);
  free(prev);
  return rc;
}
