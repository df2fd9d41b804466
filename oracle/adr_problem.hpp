// ORACLE -- TEST INFRASTRUCTURE ONLY (see cisdc_oracle.h).
//
// cisdc::OperatorSplitProblem (proj/core/include/cisdc/operator_split.hpp:36-54) over the oracle's
// periodic ADR problem class, so the reference's own integrators (cisdc::integrate, run_sweep,
// execute_pipelined) drive it unmodified.  Shared by ref_adapter.cpp and the compiled C++
// consumer of the GPU engine (integration/engine_check.cpp).
#pragma once

#include <atomic>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>

#include "cisdc/errors.hpp"
#include "cisdc/operator_split.hpp"
#include "cisdc_oracle.h"

namespace cisdc_oracle {

inline void throw_for(int rc, const std::string& what) {
  switch (rc) {
    case CISDC_E_INVALID_ARGUMENT: throw std::invalid_argument(what);
    case CISDC_E_FACTORIZATION: throw cisdc::FactorizationError(what);
    case CISDC_E_NUMERIC: throw cisdc::NumericError(what);
    case CISDC_E_CAPABILITY: throw cisdc::CapabilityError(what);
    default: throw cisdc::SolveError(what);
  }
}

// OperatorSplitProblem over the oracle's periodic ADR class.  Diffusion solves share the
// multigrid workspace and are serialised by a mutex (execute_pipelined may run two D cells at
// once for nu > 1); Newton/multigrid work counts are accumulated atomically.
class AdrProblem final : public cisdc::OperatorSplitProblem {
 public:
  explicit AdrProblem(co_problem* p) : p_(p) {}
  std::size_t dimension() const override { return co_problem_dim(p_); }
  void eval_advection(std::span<const double> x, std::span<double> o) const override { ev(CISDC_STAGE_ADVECTION, x, o); }
  void eval_diffusion(std::span<const double> x, std::span<double> o) const override { ev(CISDC_STAGE_DIFFUSION, x, o); }
  void eval_reaction(std::span<const double> x, std::span<double> o) const override { ev(CISDC_STAGE_REACTION, x, o); }
  void solve_diffusion(double coef, std::span<const double> b, std::span<double> o) const override {
    std::lock_guard<std::mutex> lk(mu_);
    sv(CISDC_STAGE_DIFFUSION, coef, b, o);
  }
  void solve_reaction(double coef, std::span<const double> b, std::span<double> o) const override {
    sv(CISDC_STAGE_REACTION, coef, b, o);
  }
  // the periodic ADR class's coupled stage (cisdc_gpu.h: alternating stage solves to convergence);
  // it runs diffusion solves inside, so it takes the multigrid-workspace lock as well
  bool has_coupled_solve() const override { return co_problem_has_coupled(p_) != 0; }
  void solve_coupled(double coef, std::span<const double> b, std::span<double> o) const override {
    if (!co_problem_has_coupled(p_)) {
      cisdc::OperatorSplitProblem::solve_coupled(coef, b, o);
      return;
    }
    std::lock_guard<std::mutex> lk(mu_);
    sv(3, coef, b, o);
  }
  long long newton() const { return newton_.load(); }
  long long mg() const { return mg_.load(); }
  void reset() {
    newton_ = 0;
    mg_ = 0;
  }

 private:
  void ev(int st, std::span<const double> x, std::span<double> o) const {
    const int rc = co_eval(p_, st, x.data(), o.data());
    if (rc) throw_for(rc, co_problem_error(p_));
  }
  void sv(int st, double coef, std::span<const double> b, std::span<double> o) const {
    cisdc_counters c{};
    const int rc = co_solve(p_, st, coef, b.data(), o.data(), &c);
    newton_ += c.newton_iterations;
    mg_ += c.mg_cycles;
    if (rc) throw_for(rc, co_problem_error(p_));
  }
  co_problem* p_;
  mutable std::mutex mu_;
  mutable std::atomic<long long> newton_{0}, mg_{0};
};

}  // namespace cisdc_oracle
