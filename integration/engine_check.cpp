// A compiled reference-side consumer of the GPU engine (VERDICT r1 "make the drop-in real").
//
// Built against the UNMODIFIED reference headers (/root/reference/proj/core/include) and library
// (oracle/_ref/libcisdc_ref.so) plus libcisdc_gpu.so by `make -C oracle engine`; called from
// tests/test_engine_adapter.py.  Each entry point runs the same problem twice:
//   reference: cisdc::integrate (integrators.hpp:84-85) on the reference's own
//              cisdc::ReactionDiffusionProblem (config-0) or on the oracle's periodic ADR class
//              (cisdc_oracle::AdrProblem) for configs 1-5;
//   GPU:       cisdc::gpu::Engine::integrate (integration/cisdc/gpu.hpp) with the tables from the
//              reference's own cisdc::make_quadrature_tables.
// and hands both results back for a bitwise comparison.  TEST INFRASTRUCTURE (links the oracle).
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "adr_problem.hpp"
#include "cisdc/errors.hpp"
#include "cisdc/integrators.hpp"
#include "cisdc/problems/reaction_diffusion.hpp"
#include "cisdc/quadrature.hpp"
#include "cisdc/gpu.hpp"

namespace {

struct RefProblem {
  co_problem* cp = nullptr;
  std::unique_ptr<cisdc::OperatorSplitProblem> prob;
  ~RefProblem() {
    prob.reset();
    if (cp) co_problem_destroy(cp);
  }
};

void make_ref_problem(const cisdc_problem_desc* d, RefProblem& h) {
  if (d->kind == CISDC_PROBLEM_REFERENCE_RD) {
    h.prob = std::make_unique<cisdc::ReactionDiffusionProblem>(
        cisdc::ReactionDiffusionGrid(d->n[0], d->ref_a, d->ref_d, d->ref_r));
  } else {
    char err[512] = {0};
    const int rc = co_problem_create(d, &h.cp, err);
    if (rc) throw std::invalid_argument(err);
    h.prob = std::make_unique<cisdc_oracle::AdrProblem>(h.cp);
  }
}

cisdc::IntegrateOptions to_ref(const cisdc_integrate_options* o) {
  cisdc::IntegrateOptions opt;
  opt.scheme = static_cast<cisdc::Scheme>(o->scheme);
  opt.dt = o->dt;
  opt.n_steps = o->n_steps;
  opt.M = o->M;
  opt.n_sweeps = o->n_sweeps;
  opt.nu = o->nu;
  if (o->has_stop_tol) opt.stop_tol = o->stop_tol;
  opt.convention = o->convention == CISDC_EULER_CUMULATIVE ? cisdc::EulerConvention::cumulative
                                                           : cisdc::EulerConvention::literal;
  return opt;
}

// 0 invalid_argument, 1 FactorizationError, 2 SolveError, 3 NumericError, 4 CapabilityError, 5 other
int kind_of(const std::exception& e) {
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 0;
  if (dynamic_cast<const cisdc::FactorizationError*>(&e)) return 1;
  if (dynamic_cast<const cisdc::SolveError*>(&e)) return 2;
  if (dynamic_cast<const cisdc::NumericError*>(&e)) return 3;
  if (dynamic_cast<const cisdc::CapabilityError*>(&e)) return 4;
  return 5;
}

void put(long long* c, const cisdc::SweepReport& r) {
  c[0] = r.sweeps;
  c[1] = r.counters.diffusion;
  c[2] = r.counters.reaction;
  c[3] = r.counters.coupled;
}

}  // namespace

extern "C" {

// Runs both sides; per step s: counts[4 s .. 4 s + 3] = sweeps, diffusion, reaction, coupled solves;
// incs[s * n_sweeps + k].  Returns 0, or -1 with the message in err when a side threw.
int engine_vs_reference(const cisdc_problem_desc* d, const double* phi0, size_t n, const cisdc_integrate_options* o,
                        int workers, double* gpu_final, double* ref_final, long long* gpu_counts,
                        long long* ref_counts, double* gpu_incs, double* ref_incs, long long* gpu_newton,
                        char* err, size_t cap) {
  try {
    const cisdc::IntegrateOptions opt = to_ref(o);
    RefProblem h;
    make_ref_problem(d, h);
    const cisdc::IntegrateResult ref = cisdc::integrate(*h.prob, std::span<const double>(phi0, n), opt);
    cisdc::gpu::Engine eng(*d, cisdc::make_quadrature_tables(opt.M, opt.convention));
    const cisdc::IntegrateResult gpu = eng.integrate(std::span<const double>(phi0, n), opt, workers);
    std::memcpy(ref_final, ref.final_state.data(), sizeof(double) * n);
    std::memcpy(gpu_final, gpu.final_state.data(), sizeof(double) * n);
    for (std::size_t s = 0; s < ref.steps.size(); ++s) {
      put(ref_counts + 4 * s, ref.steps[s]);
      put(gpu_counts + 4 * s, gpu.steps[s]);
      for (std::size_t k = 0; k < ref.steps[s].increments.size(); ++k)
        ref_incs[s * o->n_sweeps + k] = ref.steps[s].increments[k];
      for (std::size_t k = 0; k < gpu.steps[s].increments.size(); ++k)
        gpu_incs[s * o->n_sweeps + k] = gpu.steps[s].increments[k];
      gpu_newton[s] = eng.newton_iterations()[s];
    }
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(err, cap, "%s", e.what());
    return -1;
  }
}

// The same integrate on both sides when one of them is expected to throw: the exception kinds
// (kind_of above, -1 = none) and messages.
int engine_exceptions(const cisdc_problem_desc* d, const double* phi0, size_t n, const cisdc_integrate_options* o,
                      int workers, int* ref_kind, char* ref_what, int* gpu_kind, char* gpu_what, size_t cap) {
  const cisdc::IntegrateOptions opt = to_ref(o);
  *ref_kind = *gpu_kind = -1;
  ref_what[0] = gpu_what[0] = 0;
  try {
    RefProblem h;
    make_ref_problem(d, h);
    (void)cisdc::integrate(*h.prob, std::span<const double>(phi0, n), opt);
  } catch (const std::exception& e) {
    *ref_kind = kind_of(e);
    std::snprintf(ref_what, cap, "%s", e.what());
  }
  try {
    cisdc::gpu::Engine eng(*d, cisdc::make_quadrature_tables(opt.M, opt.convention));
    (void)eng.integrate(std::span<const double>(phi0, n), opt, workers);
  } catch (const std::exception& e) {
    *gpu_kind = kind_of(e);
    std::snprintf(gpu_what, cap, "%s", e.what());
  }
  return 0;
}

}  // extern "C"
