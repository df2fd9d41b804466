// ORACLE -- TEST INFRASTRUCTURE ONLY (see cisdc_oracle.h).
//
// C entry points over the UNMODIFIED reference library compiled from /root/reference/proj/core
// (oracle/Makefile builds both into oracle/_ref/libcisdc_ref.so; nothing of the reference is
// copied into this repository).  Used to pin the C restatement (tests/test_oracle_vs_ref.py),
// to generate golden fixtures (tests/golden/make_golden.py) and as the CPU baseline in
// bench.py (cpu_baseline.kind = "reference").
//
// The periodic multi-D ADR problem of BASELINE configs 1-5 does not exist in the reference; it is
// wrapped here as a cisdc::OperatorSplitProblem subclass (AdrProblem) whose stages call the
// oracle's problem class, so the reference's own integrators (cisdc::integrate, run_sweep,
// execute_pipelined) drive it unmodified.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "cisdc/analysis.hpp"
#include "cisdc/errors.hpp"
#include "cisdc/integrators.hpp"
#include "cisdc/linalg.hpp"
#include "cisdc/pipeline.hpp"
#include "cisdc/problems/linear.hpp"
#include "cisdc/problems/reaction_diffusion.hpp"
#include "cisdc/quadrature.hpp"
#include "cisdc/sweep_state.hpp"
#include "adr_problem.hpp"
#include "cisdc_oracle.h"

namespace {

using cisdc_oracle::AdrProblem;

struct Holder {
  co_problem* cp = nullptr;
  std::unique_ptr<cisdc::OperatorSplitProblem> prob;
  AdrProblem* adr = nullptr;
  ~Holder() {
    prob.reset();
    if (cp) co_problem_destroy(cp);
  }
};

int make_problem(const cisdc_problem_desc* d, Holder& h, char* err) {
  if (d->kind == CISDC_PROBLEM_REFERENCE_RD) {
    cisdc::ReactionDiffusionGrid grid(d->n[0], d->ref_a, d->ref_d, d->ref_r);
    h.prob = std::make_unique<cisdc::ReactionDiffusionProblem>(grid);
  } else if (d->kind == CISDC_PROBLEM_LINEAR_SCALAR) {
    h.prob = std::make_unique<cisdc::LinearScalarProblem>(cisdc::StiffnessTriple{d->ref_a, d->ref_d, d->ref_r}, 1.0);
  } else {
    const int rc = co_problem_create(d, &h.cp, err);
    if (rc) return rc;
    auto a = std::make_unique<AdrProblem>(h.cp);
    h.adr = a.get();
    h.prob = std::move(a);
  }
  return CISDC_OK;
}

int code_of(const std::exception& e) {
  if (dynamic_cast<const std::invalid_argument*>(&e)) return CISDC_E_INVALID_ARGUMENT;
  if (dynamic_cast<const cisdc::FactorizationError*>(&e)) return CISDC_E_FACTORIZATION;
  if (dynamic_cast<const cisdc::NumericError*>(&e)) return CISDC_E_NUMERIC;
  if (dynamic_cast<const cisdc::CapabilityError*>(&e)) return CISDC_E_CAPABILITY;
  return CISDC_E_SOLVE;
}

void fill_tables(const cisdc::QuadratureTables& t, cisdc_tables* out) {
  std::memset(out, 0, sizeof(*out));
  const int M = t.nodes.M;
  out->M = M;
  out->convention = t.euler_convention == cisdc::EulerConvention::literal ? 0 : 1;
  for (int i = 0; i <= M; ++i) out->tau[i] = t.nodes.tau[i];
  for (int i = 0; i < M; ++i) out->dtau[i] = t.nodes.dtau[i];
  for (int m = 0; m < M; ++m) {
    out->q[m] = t.q[m];
    for (int j = 0; j <= M; ++j) {
      out->Q[m * (M + 1) + j] = t.Q(m, j);
      out->S[m * (M + 1) + j] = t.S(m, j);
    }
    for (int j = 0; j < M; ++j) {
      out->Qt[m * M + j] = t.Qt(m, j);
      out->QtI[m * M + j] = t.QtI(m, j);
      out->QtE[m * M + j] = t.QtE(m, j);
    }
  }
}

cisdc::EulerConvention conv_of(int c) {
  return c == CISDC_EULER_CUMULATIVE ? cisdc::EulerConvention::cumulative : cisdc::EulerConvention::literal;
}

}  // namespace

extern "C" {

int ref_make_tables(int M, int convention, cisdc_tables* out) {
  try {
    fill_tables(cisdc::make_quadrature_tables(M, conv_of(convention)), out);
    return CISDC_OK;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_banded_solve(int n, int kl, int ku, const double* band, const double* b, double* x) {
  try {
    cisdc::BandedMatrix A(n, kl, ku);
    for (int i = 0; i < n; ++i)
      for (int j = std::max(0, i - kl); j <= std::min(n - 1, i + ku); ++j) A.at(i, j) = band[(j - i + kl) * n + i];
    const auto v = cisdc::banded_solve(A, std::span<const double>(b, n));
    std::memcpy(x, v.data(), sizeof(double) * n);
    return CISDC_OK;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// cisdc::integrate (serial sweeps) or, with workers > 0 and scheme cisdcq, the same step loop
// with execute_pipelined for every sweep (pipeline.cpp:171-320).
int ref_integrate(const cisdc_problem_desc* d, const double* phi0, const cisdc_integrate_options* o,
                  double* final_state, cisdc_step_report* reports, double* increments, char* err) {
  Holder h;
  int rc = make_problem(d, h, err);
  if (rc) return rc;
  const std::size_t n = h.prob->dimension();
  try {
    cisdc::IntegrateOptions opt;
    opt.scheme = static_cast<cisdc::Scheme>(o->scheme);
    opt.dt = o->dt;
    opt.n_steps = o->n_steps;
    opt.M = o->M;
    opt.n_sweeps = o->n_sweeps;
    opt.nu = o->nu;
    if (o->has_stop_tol) opt.stop_tol = o->stop_tol;
    opt.convention = conv_of(o->convention);
    cisdc::IntegrateResult res;
    if (o->workers > 0 && opt.scheme == cisdc::Scheme::cisdcq) {
      // integrators.cpp:301-333 with run_sweep replaced by execute_pipelined
      const auto tables = cisdc::make_quadrature_tables(opt.M, opt.convention);
      cisdc::SweepState state(opt.M, n);
      cisdc::NodeVector start(phi0, phi0 + n);
      for (int step = 0; step < opt.n_steps; ++step) {
        state.initialize(*h.prob, start);
        cisdc::SweepReport rep;
        cisdc::NodeVector prev_end = state.phi[opt.M];
        for (int k = 1; k <= opt.n_sweeps; ++k) {
          try {
            cisdc::execute_pipelined(state, tables, *h.prob, opt.dt, opt.nu, o->workers, &rep.counters);
          } catch (const std::exception& e) {
            throw cisdc::SolveError("integrate: step " + std::to_string(step + 1) + ", sweep " +
                                    std::to_string(k) + ": " + e.what());
          }
          rep.increments.push_back(cisdc::increment_norm(state.phi[opt.M], prev_end));
          prev_end = state.phi[opt.M];
          if (opt.stop_tol && rep.increments.back() <= *opt.stop_tol) break;
        }
        rep.sweeps = static_cast<int>(rep.increments.size());
        res.steps.push_back(std::move(rep));
        start = state.phi[opt.M];
      }
      res.final_state = std::move(start);
    } else {
      res = cisdc::integrate(*h.prob, std::span<const double>(phi0, n), opt);
    }
    std::memcpy(final_state, res.final_state.data(), sizeof(double) * n);
    for (std::size_t s = 0; s < res.steps.size(); ++s) {
      if (reports) {
        reports[s].sweeps = res.steps[s].sweeps;
        reports[s].counters.diffusion = res.steps[s].counters.diffusion;
        reports[s].counters.reaction = res.steps[s].counters.reaction;
        reports[s].counters.coupled = res.steps[s].counters.coupled;
        reports[s].counters.newton_iterations = -1;
        reports[s].counters.mg_cycles = -1;
      }
      if (increments)
        for (std::size_t k = 0; k < res.steps[s].increments.size(); ++k)
          increments[s * o->n_sweeps + k] = res.steps[s].increments[k];
    }
    if (h.adr && reports && !res.steps.empty()) {
      // per-run totals (the reference counts no Newton work; the adapter does)
      reports[0].counters.newton_iterations = h.adr->newton();
      reports[0].counters.mg_cycles = h.adr->mg();
    }
    return CISDC_OK;
  } catch (const std::exception& e) {
    if (err) std::snprintf(err, 1024, "%s", e.what());
    return code_of(e);
  }
}

// Sweep-level driver: initialise (values == NULL: SweepState::initialize(phi0); else
// set_node_values(values)), run n_sweeps sweeps (workers > 0: execute_pipelined), then copy out
// phi, fa, fd, fr, phi_ad at every node: out[(which*(M+1) + m)*n + i].
int ref_sweeps(const cisdc_problem_desc* d, int M, int convention, int scheme, double dt, int nu, int workers,
               int n_sweeps, const double* phi0, const double* values, double* out, cisdc_counters* counters,
               char* err) {
  Holder h;
  int rc = make_problem(d, h, err);
  if (rc) return rc;
  const std::size_t n = h.prob->dimension();
  try {
    const auto tables = cisdc::make_quadrature_tables(M, conv_of(convention));
    cisdc::SweepState st(M, n);
    if (values) {
      std::vector<cisdc::NodeVector> v(M + 1);
      for (int m = 0; m <= M; ++m) v[m].assign(values + m * n, values + (m + 1) * n);
      st.set_node_values(*h.prob, v);
    } else {
      st.initialize(*h.prob, std::span<const double>(phi0, n));
    }
    cisdc::SolveCounters sc;
    for (int k = 0; k < n_sweeps; ++k) {
      if (workers > 0 && scheme == CISDC_SCHEME_CISDCQ)
        cisdc::execute_pipelined(st, tables, *h.prob, dt, nu, workers, &sc);
      else
        cisdc::run_sweep(static_cast<cisdc::Scheme>(scheme), st, tables, *h.prob, dt, nu, &sc);
    }
    const std::vector<cisdc::NodeVector>* f[5] = {&st.phi, &st.fa, &st.fd, &st.fr, &st.phi_ad};
    for (int w = 0; w < 5; ++w)
      for (int m = 0; m <= M; ++m) std::memcpy(out + ((std::size_t)w * (M + 1) + m) * n, (*f[w])[m].data(), sizeof(double) * n);
    if (counters) {
      counters->diffusion = sc.diffusion;
      counters->reaction = sc.reaction;
      counters->coupled = sc.coupled;
      counters->newton_iterations = h.adr ? h.adr->newton() : -1;
      counters->mg_cycles = h.adr ? h.adr->mg() : -1;
    }
    return CISDC_OK;
  } catch (const std::exception& e) {
    if (err) std::snprintf(err, 1024, "%s", e.what());
    return code_of(e);
  }
}

// One problem stage on one field (OperatorSplitProblem::eval_* / solve_*).
int ref_stage(const cisdc_problem_desc* d, int solve, int stage, double coef, const double* in, double* out,
              char* err) {
  Holder h;
  int rc = make_problem(d, h, err);
  if (rc) return rc;
  const std::size_t n = h.prob->dimension();
  try {
    std::span<const double> x(in, n);
    std::span<double> o(out, n);
    if (!solve) {
      if (stage == CISDC_STAGE_ADVECTION) h.prob->eval_advection(x, o);
      else if (stage == CISDC_STAGE_DIFFUSION) h.prob->eval_diffusion(x, o);
      else h.prob->eval_reaction(x, o);
    } else {
      if (stage == CISDC_STAGE_DIFFUSION) h.prob->solve_diffusion(coef, x, o);
      else if (stage == CISDC_STAGE_REACTION) h.prob->solve_reaction(coef, x, o);
      else h.prob->solve_coupled(coef, x, o);
    }
    return CISDC_OK;
  } catch (const std::exception& e) {
    if (err) std::snprintf(err, 1024, "%s", e.what());
    return code_of(e);
  }
}

// Reference initial condition of the Dirichlet PDE (reaction_diffusion.cpp:69-74).
int ref_rd_initial_condition(int n_x, double a, double d, double r, double* out) {
  try {
    cisdc::ReactionDiffusionGrid grid(n_x, a, d, r);
    const auto v = cisdc::initial_condition(grid);
    std::memcpy(out, v.data(), sizeof(double) * n_x);
    return CISDC_OK;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// SDC1 snapshot IO of the reference (reaction_diffusion.cpp:230-259), for byte-level checks.
int ref_write_field_snapshot(const char* path, int n_x, double dx, const double* data, size_t n, char* err) {
  try {
    cisdc::write_field_snapshot(path, n_x, dx, std::span<const double>(data, n));
    return CISDC_OK;
  } catch (const std::invalid_argument& e) {
    if (err) std::snprintf(err, 1024, "%s", e.what());
    return CISDC_E_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    if (err) std::snprintf(err, 1024, "%s", e.what());
    return CISDC_E_IO;
  }
}

int ref_read_field_snapshot(const char* path, int* n_x, double* dx, double* data, size_t cap, char* err) {
  try {
    const cisdc::FieldSnapshot s = cisdc::read_field_snapshot(path);
    *n_x = s.n_x;
    *dx = s.dx;
    if (data) std::memcpy(data, s.data.data(), sizeof(double) * std::min<size_t>(cap, s.data.size()));
    return CISDC_OK;
  } catch (const std::exception& e) {
    if (err) std::snprintf(err, 1024, "%s", e.what());
    return CISDC_E_IO;
  }
}

// The reference's validate_schedule_trace (pipeline.cpp:322-350) on a trace given as arrays in
// cell-id order; msg receives its verdict ("" = valid).
static cisdc::ScheduleTrace to_ref_trace(int M, int nu, int workers, const cisdc_cell_trace* cells, int n) {
  const cisdc::TaskGraph g = cisdc::build_task_graph(M, nu);
  cisdc::ScheduleTrace t;
  t.workers = workers;
  for (int i = 0; i < n; ++i) {
    cisdc::CellTrace c;
    c.cell = g.cells[i];
    c.worker = cells[i].worker;
    c.start_ns = cells[i].start_ns;
    c.end_ns = cells[i].end_ns;
    c.seq_start = cells[i].seq_start;
    c.seq_end = cells[i].seq_end;
    t.cells.push_back(c);
  }
  return t;
}

int ref_validate_trace(int M, int nu, int workers, const cisdc_cell_trace* cells, int n, char* msg, size_t cap) {
  try {
    const cisdc::TaskGraph g = cisdc::build_task_graph(M, nu);
    const std::string v = cisdc::validate_schedule_trace(g, to_ref_trace(M, nu, workers, cells, n));
    std::snprintf(msg, cap, "%s", v.c_str());
    return CISDC_OK;
  } catch (const std::exception& e) {
    std::snprintf(msg, cap, "%s", e.what());
    return code_of(e);
  }
}

// cisdc::spectral_radius (linalg.cpp:197-332) of one n x n row-major matrix
int ref_spectral_radius(const double* A, int n, double* rho) {
  try {
    cisdc::DenseMatrix M(n, n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) M(i, j) = A[i * n + j];
    *rho = cisdc::spectral_radius(M);
    return CISDC_OK;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// cisdc::spectral_radius_scan (analysis.cpp:270-293) with the C-ABI's point layout; G_out
// (optional) receives affine_iteration_matrix(...).G of every point that has one (zeros otherwise).
int ref_spectral_radius_scan(const int* schemes, int n_schemes, const int* nu_list, int n_nu, const double* r_grid,
                             int n_r, int d_rule, double fixed_d, double a, double dt, int M, int convention,
                             cisdc_scan_point* out, size_t cap, size_t* n_out, double* G_out, char* err) {
  try {
    cisdc::ScanOptions o;
    for (int i = 0; i < n_schemes; ++i) o.schemes.push_back(static_cast<cisdc::Scheme>(schemes[i]));
    for (int i = 0; i < n_nu; ++i) o.nu_list.push_back(nu_list[i]);
    for (int i = 0; i < n_r; ++i) o.r_grid.push_back(r_grid[i]);
    o.d_rule = d_rule == 0 ? cisdc::DRule::half_of_r : cisdc::DRule::fixed;
    o.fixed_d = fixed_d;
    o.a = a;
    o.dt = dt;
    o.M = M;
    o.convention = conv_of(convention);
    const std::vector<cisdc::ScanPoint> pts = cisdc::spectral_radius_scan(o);
    if (n_out) *n_out = pts.size();
    if (cap < pts.size()) return CISDC_E_INVALID_ARGUMENT;
    for (size_t i = 0; i < pts.size(); ++i) {
      const cisdc::ScanPoint& p = pts[i];
      out[i] = cisdc_scan_point{static_cast<int>(p.scheme), p.M, p.nu, p.a, p.d, p.r, p.dt, p.gamma, p.ok ? 1 : 0};
      if (G_out) {
        double* g = G_out + i * (size_t)M * M;
        std::memset(g, 0, sizeof(double) * M * M);
        try {
          const cisdc::IterationMatrixResult res =
              cisdc::affine_iteration_matrix(p.scheme, {p.a, p.d, p.r}, p.dt, p.M, p.nu, o.convention);
          for (int r = 0; r < M; ++r)
            for (int c = 0; c < M; ++c) g[r * M + c] = res.G(r, c);
        } catch (const std::exception&) {
          // singular stage / non-finite G / QR cap: the point is ok = false; G where it exists
          try {
            const cisdc::AffineMap mp = cisdc::affine_sweep_map(p.scheme, {p.a, p.d, p.r}, p.dt, p.M, p.nu, o.convention);
            for (int r = 0; r < M; ++r)
              for (int c = 0; c < M; ++c) g[r * M + c] = mp.W(r, c);
          } catch (const std::exception&) {
          }
        }
      }
    }
    return CISDC_OK;
  } catch (const std::exception& e) {
    if (err) std::snprintf(err, 1024, "%s", e.what());
    return code_of(e);
  }
}

}  // extern "C"
