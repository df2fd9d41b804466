// cisdc/gpu.hpp -- the reference-side binding of the B200 sweep engine.
//
// What a maintainer of the reference (cisdc, C++20, proj/core) adds to use the GPU path: a thin
// C++ adapter over the C-ABI of include/cisdc_gpu.h that speaks the reference's own types
//   cisdc::QuadratureTables  (proj/core/include/cisdc/quadrature.hpp:47-60)  -> cisdc_tables
//   cisdc::IntegrateOptions  (proj/core/include/cisdc/integrators.hpp:64-73) -> cisdc_integrate_options
//   cisdc::IntegrateResult   (integrators.hpp:75-79) / cisdc::SweepReport (sweep_state.hpp:56-60)
// and rethrows the engine's status codes as the reference's exceptions (errors.hpp:24-45).
// Engine::integrate is the drop-in for cisdc::integrate (integrators.hpp:84-85,
// integrators.cpp:301-333): same options in, same state, reports and exception types out.
// The tables come from the reference's own make_quadrature_tables, so the engine runs on exactly
// the reference's bits.  Compiled and tested against the unmodified reference headers by
// integration/engine_check.cpp (tests/test_engine_adapter.py).
#pragma once

#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "cisdc/errors.hpp"
#include "cisdc/integrators.hpp"
#include "cisdc/quadrature.hpp"
#include "cisdc_gpu.h"

namespace cisdc::gpu {

inline void check(int rc, const cisdc_gpu_ctx* ctx) {
  if (rc == CISDC_OK) return;
  const std::string msg = ctx ? cisdc_gpu_last_error(ctx) : "cisdc_gpu: error " + std::to_string(rc);
  switch (rc) {
    case CISDC_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case CISDC_E_FACTORIZATION: throw FactorizationError(msg);
    case CISDC_E_NUMERIC: throw NumericError(msg);
    case CISDC_E_CAPABILITY: throw CapabilityError(msg);
    case CISDC_E_SOLVE: throw SolveError(msg);
    default: throw std::runtime_error(msg);  // CUDA failure / IO
  }
}

// cisdc::QuadratureTables -> the C-ABI's row-major copy (bit for bit).
inline cisdc_tables to_c(const QuadratureTables& t) {
  cisdc_tables c;
  std::memset(&c, 0, sizeof(c));
  const int M = t.nodes.M;
  if (M < 1 || M > CISDC_MAX_M) throw std::invalid_argument("cisdc::gpu: M must be in 1..8");
  c.M = M;
  c.convention = t.euler_convention == EulerConvention::literal ? CISDC_EULER_LITERAL : CISDC_EULER_CUMULATIVE;
  for (int i = 0; i <= M; ++i) c.tau[i] = t.nodes.tau[i];
  for (int i = 0; i < M; ++i) c.dtau[i] = t.nodes.dtau[i];
  for (int m = 0; m < M; ++m) {
    c.q[m] = t.q[m];
    for (int j = 0; j <= M; ++j) {
      c.Q[m * (M + 1) + j] = t.Q(m, j);
      c.S[m * (M + 1) + j] = t.S(m, j);
    }
    for (int j = 0; j < M; ++j) {
      c.Qt[m * M + j] = t.Qt(m, j);
      c.QtI[m * M + j] = t.QtI(m, j);
      c.QtE[m * M + j] = t.QtE(m, j);
    }
  }
  return c;
}

// Device-resident SweepState + problem.  One host thread per instance (like SweepState).
class Engine {
 public:
  Engine(const cisdc_problem_desc& desc, const QuadratureTables& tables) : conv_(tables.euler_convention) {
    const cisdc_tables t = to_c(tables);
    cisdc_gpu_ctx* raw = nullptr;
    const int rc = cisdc_gpu_create(&desc, &t, &raw);
    ctx_.reset(raw);
    check(rc, raw);
  }

  std::size_t dimension() const { return cisdc_gpu_dimension(ctx_.get()); }

  // cisdc::integrate(problem, phi0, opt); workers > 0 runs CISDCQ sweeps as execute_pipelined's DAG
  // on two CUDA streams (bitwise equal to the serial cell order).  The engine's tables must be
  // make_quadrature_tables(opt.M, opt.convention) -- as in integrators.cpp:306.
  IntegrateResult integrate(std::span<const double> phi0, const IntegrateOptions& opt, int workers = 0) {
    if (opt.n_sweeps < 1) throw std::invalid_argument("integrate: n_sweeps must be >= 1");
    cisdc_integrate_options o{};
    o.scheme = static_cast<int>(opt.scheme);
    o.dt = opt.dt;
    o.n_steps = opt.n_steps;
    o.M = opt.M;
    o.n_sweeps = opt.n_sweeps;
    o.nu = opt.nu;
    o.has_stop_tol = opt.stop_tol.has_value() ? 1 : 0;
    o.stop_tol = opt.stop_tol.value_or(0.0);
    o.convention = opt.convention == EulerConvention::literal ? CISDC_EULER_LITERAL : CISDC_EULER_CUMULATIVE;
    o.workers = workers;
    IntegrateResult res;
    res.final_state.resize(phi0.size());
    std::vector<cisdc_step_report> reps(opt.n_steps > 0 ? opt.n_steps : 1);
    std::vector<double> incs(static_cast<std::size_t>(reps.size()) * opt.n_sweeps);
    check(cisdc_gpu_integrate(ctx_.get(), phi0.data(), phi0.size(), &o, res.final_state.data(), reps.data(),
                              incs.data()),
          ctx_.get());
    if (opt.n_steps <= 0) res.final_state.assign(phi0.begin(), phi0.end());
    for (int s = 0; s < opt.n_steps; ++s) {
      SweepReport r;
      r.sweeps = reps[s].sweeps;
      r.counters.diffusion = reps[s].counters.diffusion;
      r.counters.reaction = reps[s].counters.reaction;
      r.counters.coupled = reps[s].counters.coupled;
      const auto* first = incs.data() + static_cast<std::size_t>(s) * opt.n_sweeps;
      r.increments.assign(first, first + r.sweeps);
      res.steps.push_back(std::move(r));
      newton_.push_back(reps[s].counters.newton_iterations);
      mg_.push_back(reps[s].counters.mg_cycles);
    }
    return res;
  }

  // per-step Newton trips / multigrid cycles of the integrate calls so far (no reference counterpart)
  const std::vector<long long>& newton_iterations() const { return newton_; }
  const std::vector<long long>& mg_cycles() const { return mg_; }

 private:
  struct Del {
    void operator()(cisdc_gpu_ctx* c) const { cisdc_gpu_destroy(c); }
  };
  std::unique_ptr<cisdc_gpu_ctx, Del> ctx_;
  EulerConvention conv_;
  std::vector<long long> newton_, mg_;
};

}  // namespace cisdc::gpu
