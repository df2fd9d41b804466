// B200-native MISDC / MISDCQ / CISDCQ ("PMISDC") sweep engine: context, sweep drivers and the
// C-ABI of include/cisdc_gpu.h.
//
// The host keeps the reference's control flow verbatim (node loop of misdc_sweep /
// misdcq_sweep, cell order or DAG of cisdcq_sweep / execute_pipelined, step loop of integrate);
// every per-element loop of the reference becomes one of the kernels in *.cuh.  Sweep state is
// device resident for the whole run: node fields of sweep (k) and (k+1) are two pointer sets that
// swap after every sweep (the reference's fa_p = state.fa copy, integrators.cpp:74/108, becomes a
// pointer swap), and node 0 is shared by both sets.  After SweepState::initialize every node of
// the current set aliases node 0 (no M-fold copy).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cisdc_gpu.h"
#include "analysis.cuh"
#include "circulant.hpp"
#include "common.cuh"
#include "multigrid.cuh"
#include "newton.cuh"
#include "peak.cuh"
#include "pointwise.cuh"
#include "rtc.cuh"
#include "solve1d.cuh"
#include "stencil.cuh"

namespace cisdc_b200 {
int make_tables(int M, int convention, cisdc_tables* t);
}

using namespace cisdc_b200;

namespace {

constexpr int kPhi = 0, kFa = 1, kFd = 2, kFr = 3;

const char* kClassNames[kNumKernelClasses] = {"quad_base", "rhs", "solve1d", "mg_smooth", "mg_restrict",
                                              "mg_prolong", "mg_norm", "react_newton", "eval_ad", "eval_r",
                                              "increment", "react_newton_rhs"};

// Launch accounting + optional live CUDA-event timing per kernel class.
struct Timing final : LaunchHook {
  bool on = false;
  long long launches = 0;
  double ms[kNumKernelClasses] = {};
  double bytes[kNumKernelClasses] = {};
  long long count[kNumKernelClasses] = {};
  struct Pending {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<Pending> pending;
  cudaEvent_t cur = nullptr;

  cudaEvent_t take() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  void before(int, cudaStream_t s) override {
    if (!on) return;
    cur = take();
    cudaEventRecord(cur, s);
  }
  void add_bytes(int cls, double b) override { bytes[cls] += b; }
  void add_launches(long long n) override { launches += n; }
  bool timing() const override { return on; }
  void after(int cls, cudaStream_t s, double b) override {
    ++launches;
    ++count[cls];
    bytes[cls] += b;
    if (!on) return;
    cudaEvent_t e = take();
    cudaEventRecord(e, s);
    pending.push_back({cls, cur, e});
  }
  // call after the streams are synchronised
  void resolve() {
    for (const Pending& p : pending) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess) ms[p.cls] += t;
    }
    pending.clear();
    used = 0;
  }
  void reset() {
    for (int c = 0; c < kNumKernelClasses; ++c) {
      ms[c] = bytes[c] = 0.0;
      count[c] = 0;
    }
    launches = 0;
  }
  ~Timing() override {
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
};

}  // namespace

struct cisdc_gpu_ctx {
  cisdc_problem_desc desc{};  // borrowed pointers are dropped after create; diffusivity is owned
  std::vector<double> diffusivity;
  cisdc_tables tb{};
  int M = 0;
  Geom g{};
  Ops ops{};
  Reaction rx{};
  int S = 1;
  bool ref_rd = false;
  bool linear = false;  // CISDC_PROBLEM_LINEAR_SCALAR: (a, d, r) per element, exact stage solves
  double lin_a = 0.0, lin_d = 0.0, lin_r = 0.0;
  // device memory
  std::vector<void*> allocs;
  double* node0[4] = {};                       // phi0, fa0, fd0, fr0 (shared by both sets)
  double* own[2][4][kMaxM + 1] = {};           // [set][field][node 1..M]
  const double* view[2][4][kMaxM + 1] = {};    // current views (node 0 -> node0)
  int cur = 0;
  double* phi_ad[kMaxM + 1] = {};              // state.phi_ad (entry 0 unused, zeros)
  double* base[kMaxM] = {};                    // quadrature bases per row
  double* rhs_d = nullptr;
  double* rhs_r = nullptr;
  double* scratch = nullptr;
  // CISDCQ workspace (ell = 1 evaluations at phi_ad, and the slots of ell < nu)
  double* fa_ad[kMaxM + 1] = {};
  double* fd_ad[kMaxM + 1] = {};
  std::vector<double*> slot_bufs;  // (nu-1) * M * 5: phi_ad, phi_r, fa_r, fd_r, fr_r
  std::vector<double*> diff_bufs;  // CISDCQ rhs difference cache: (M - 3) nodes x {dA, dDR}
  // coupled stage of the periodic ADR class (allocated on first use): y, y_next, f / stage rhs, z;
  // the convergence maxima on the device and their pinned mirror (delta, scale, fail_key)
  double* cpl[4] = {};
  unsigned long long* d_cpl = nullptr;
  unsigned long long* h_cpl = nullptr;
  // solvers
  double* rd_work = nullptr;
  MgHierarchy mg;
  RtcNewton rtc;  // network-specialised Newton kernels (mass action)
  unsigned* defer_list = nullptr;  // cells the specialised kernel hands to the dense fixup
  int* defer_count = nullptr;
  // status / reductions
  DevStatus* d_st = nullptr;
  DevStatus* h_st = nullptr;  // pinned
  double* d_partial = nullptr;
  double* d_incr = nullptr;   // [kMaxSweepsPerStep] increments of the current step
  double* h_incr = nullptr;   // pinned mirror
  int incr_slot = 0;
  unsigned long long newton_seen = 0, mg_seen = 0;
  unsigned long long newton_res_exits = 0;  // device counter as of the last check_status
  unsigned long long loop_seen = 0;         // DevStatus::loop_kernels already counted
  cudaStream_t s_main = nullptr, s_r = nullptr;
  int num_sms = 148;
  // PMISDC schedule trace (cisdc_gpu_set_trace / cisdc_gpu_last_trace)
  bool trace_on = false, trace_pending = false;
  int trace_M = 0, trace_nu = 0, trace_workers = 0;
  std::vector<cudaEvent_t> trace_ev;  // [2 * cell id + 0/1] start/end, last = base
  std::vector<cisdc_cell_trace> trace;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t ev_base = nullptr, ev_join = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
  Timing tm;
  double device_ms = 0.0;
  std::string err;
  double last_incr = 0.0;
  bool have_incr = false;
  // failure tags (DevStatus::fail_key): tag t-1 -> (sweep of the running integrate step, stage)
  std::vector<std::pair<int, int>> tags;
  int cur_sweep = 0;   // 1-based sweep of the integrate step being enqueued, 0 outside integrate
  int fail_sweep = 0;  // sweep of the failure the last check_status decoded
  // Whole integrate steps captured as CUDA graphs (steps without host decisions inside: no stop
  // tolerance, no host-synchronised multigrid, no live timing or tracing).  A replay stands for the
  // host enqueue of initialize + n sweeps + the node-0 copy; the host bookkeeping the enqueue did
  // (tags, stage counts, views, cur) is restored from the capture.
  struct StepGraph {
    int scheme, nu, workers, n_sweeps, convention;
    double dt;
    cudaGraphExec_t exec;
    long long kernels;
    std::vector<std::pair<int, int>> tags;
    cisdc_counters counts;
    int cur;
    const double* view[2][4][kMaxM + 1];
  };
  std::vector<StepGraph> step_graphs;
  long long steps_direct = 0;  // steps enqueued directly (the first one is never captured)
};

namespace {

constexpr int kMaxSweepsPerStep = 4096;

int set_err(cisdc_gpu_ctx* c, int code, const std::string& m) {
  if (c) c->err = m;
  return code;
}

#define CU(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess)                                                                       \
      return set_err(ctx, CISDC_E_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                            " at " #x);                                          \
  } while (0)

#define TRY(x)             \
  do {                     \
    const int rc_ = (x);   \
    if (rc_) return rc_;   \
  } while (0)

int dalloc(cisdc_gpu_ctx* ctx, double** p, size_t count) {
  void* v = nullptr;
  CU(cudaMalloc(&v, std::max<size_t>(count, 1) * sizeof(double)));
  ctx->allocs.push_back(v);
  *p = static_cast<double*>(v);
  return CISDC_OK;
}

const double* V(cisdc_gpu_ctx* c, int set, int field, int node) { return c->view[set][field][node]; }

void reset_views(cisdc_gpu_ctx* c, int set) {
  for (int f = 0; f < 4; ++f) {
    c->view[set][f][0] = c->node0[f];
    for (int m = 1; m <= c->M; ++m) c->view[set][f][m] = c->own[set][f][m];
  }
}

void alias_views_to_node0(cisdc_gpu_ctx* c, int set) {
  for (int f = 0; f < 4; ++f)
    for (int m = 0; m <= c->M; ++m) c->view[set][f][m] = c->node0[f];
}

unsigned next_tag(cisdc_gpu_ctx* c, int stage) {
  c->tags.push_back({c->cur_sweep, stage});
  return (unsigned)c->tags.size();
}

int grid_of(long long n, int block) { return static_cast<int>((n + block - 1) / block); }

double F8(const cisdc_gpu_ctx* c) { return 8.0 * (double)c->g.n; }  // bytes of one field

// ---------------------------------------------------------------- kernel launchers

// two cells per thread for F_A/F_D on even-nx 3-D grids (CISDC_EVAL_PAIR=0: one cell per thread)
bool eval_pair() {
  static const bool v = [] {
    const char* e = std::getenv("CISDC_EVAL_PAIR");
    return !(e && e[0] == '0');
  }();
  return v;
}

// TMA-staged planes for F_A/F_D on whole-tile 3-D grids (CISDC_EVAL_TMA=0: the cp.async pair walker);
// read per launch so that a process can compare the two (tests do)
bool eval_tma() {
  const char* e = std::getenv("CISDC_EVAL_TMA");
  return !(e && e[0] == '0') && tma_encoder() != nullptr;
}

int launch_eval_ad(cisdc_gpu_ctx* ctx, const double* phi, double* fa, double* fd, cudaStream_t s) {
  const Geom& g = ctx->g;
  if (ctx->linear) {
    ctx->tm.before(kKEvalAD, s);
    k_lin_eval<<<grid_of(g.n, 256), 256, 0, s>>>(phi, fa, fd, ctx->lin_a, ctx->lin_d, g.n, ctx->ops.wild);
    ctx->tm.after(kKEvalAD, s, F8(ctx) * (1 + (fa != nullptr) + (fd != nullptr)));
    CU(cudaGetLastError());
    return CISDC_OK;
  }
  const dim3 grid = stencil_grid(g.nx, g.ny, g.nz, g.S, g.ndim), block = stencil_block(g.ndim);
  ctx->tm.before(kKEvalAD, s);
  switch (g.ndim) {
    case 1: k_eval_ad<1><<<grid, block, 0, s>>>(ctx->ops, g, phi, fa, fd); break;
    case 2:
      if (g.nx % 2 == 0 && g.nx >= 64 && tile3d_ok(g.ncell) && eval_pair()) {
        CU(func_attr_once(k_eval_ad2_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRowSmem));
        const int ch = rows_chunk(g.ncell, g.S);
        k_eval_ad2_rows<<<rows_grid(g.nx, g.ny, g.S, ch), kRowWarps * 32, kRowSmem, s>>>(ctx->ops, g, phi, fa, fd, ch);
      } else {
        k_eval_ad<2><<<grid, block, 0, s>>>(ctx->ops, g, phi, fa, fd);
      }
      break;
    default:
      if (!tile3d_ok(g.ncell)) {
        k_eval_ad<3><<<grid, block, 0, s>>>(ctx->ops, g, phi, fa, fd);
        break;
      }
      TmaMaps maps;
      if (g.nx % 2 == 0 && eval_pair() && tma_grid_ok(g.nx, g.ny, g.nz, g.ncell) && eval_tma() &&
          tma_maps(maps, phi, nullptr, g.nx, g.ny, g.nz * g.S)) {
        CU(func_attr_once(k_eval_ad3_tma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaEvalSmem));
        CU(func_attr_once(k_eval_ad3_tma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaEvalSmem));
        const dim3 eg = tile3d_pair_grid(g.nx, g.ny, g.nz, g.S);
        if (ctx->ops.vconst)
          k_eval_ad3_tma<true><<<eg, dim3(kTX, kTY), kTmaEvalSmem, s>>>(ctx->ops, g, maps, fa, fd, kZChunk);
        else
          k_eval_ad3_tma<false><<<eg, dim3(kTX, kTY), kTmaEvalSmem, s>>>(ctx->ops, g, maps, fa, fd, kZChunk);
      } else if (g.nx % 2 == 0 && eval_pair()) {
        CU(func_attr_once(k_eval_ad3_pair<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPairSmem));
        CU(func_attr_once(k_eval_ad3_pair<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPairSmem));
        if (ctx->ops.vconst)
          k_eval_ad3_pair<true><<<tile3d_pair_grid(g.nx, g.ny, g.nz, g.S), dim3(kTX, kTY), kPairSmem, s>>>(
              ctx->ops, g, phi, fa, fd, kZChunk);
        else
          k_eval_ad3_pair<false><<<tile3d_pair_grid(g.nx, g.ny, g.nz, g.S), dim3(kTX, kTY), kPairSmem, s>>>(
              ctx->ops, g, phi, fa, fd, kZChunk);
      } else if (ctx->ops.vconst)
        k_eval_ad3_tiled<2, true><<<tile3d_grid(g.nx, g.ny, g.nz, g.S), dim3(kTX, kTY), 0, s>>>(ctx->ops, g, phi, fa,
                                                                                                 fd, kZChunk);
      else
        k_eval_ad3_tiled<2, false><<<tile3d_grid(g.nx, g.ny, g.nz, g.S), dim3(kTX, kTY), 0, s>>>(ctx->ops, g, phi, fa,
                                                                                                  fd, kZChunk);
      break;
  }
  ctx->tm.after(kKEvalAD, s, F8(ctx) * (1 + (fa != nullptr) + (fd != nullptr)));
  CU(cudaGetLastError());
  return CISDC_OK;
}

template <int S>
int launch_eval_r_s(cisdc_gpu_ctx* ctx, const double* phi, double* fr, cudaStream_t s) {
  ctx->tm.before(kKEvalR, s);
  k_eval_r<S><<<grid_of(ctx->g.ncell, 128), 128, 0, s>>>(ctx->rx, ctx->g, phi, fr, ctx->ops.wild);
  ctx->tm.after(kKEvalR, s, 2.0 * F8(ctx));
  CU(cudaGetLastError());
  return CISDC_OK;
}

int launch_eval_r(cisdc_gpu_ctx* ctx, const double* phi, double* fr, cudaStream_t s) {
  switch (ctx->S) {
    case 1: return launch_eval_r_s<1>(ctx, phi, fr, s);
    case 2: return launch_eval_r_s<2>(ctx, phi, fr, s);
    case 3: return launch_eval_r_s<3>(ctx, phi, fr, s);
    case 4: return launch_eval_r_s<4>(ctx, phi, fr, s);
    case 9: return launch_eval_r_s<9>(ctx, phi, fr, s);
  }
  return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "unsupported species count");
}

// compulsory fields touched by one reaction-stage launch
double react_fields(int mode, const ReactArgs& a) {
  const double w = 1.0 + (a.fr_out != nullptr);
  switch (mode) {
    case kModeMisdcq: return 4.0 + w;
    case kModeMisdc: return 6.0 + w;
    case kModeCisdcq: return (a.has_incr ? 4.0 : 2.0) + w;
    default: return 1.0 + w;
  }
}

template <int S, int MODE>
int launch_react_sm(cisdc_gpu_ctx* ctx, const ReactArgs& a, cudaStream_t s) {
  const int blocks = grid_of(ctx->g.ncell, 128);
  ctx->tm.before(kKReact, s);
  if constexpr (MODE == kModeMisdcq || MODE == kModeMisdc) {
    if (a.fd_ad) k_react<S, 0, MODE><<<blocks, 128, 0, s>>>(ctx->rx, ctx->ops, ctx->g, a, ctx->d_st);
    else k_react<S, 1, MODE><<<blocks, 128, 0, s>>>(ctx->rx, ctx->ops, ctx->g, a, ctx->d_st);  // 1-D only
  } else {
    k_react<S, 1, MODE><<<blocks, 128, 0, s>>>(ctx->rx, ctx->ops, ctx->g, a, ctx->d_st);
  }
  ctx->tm.after(kKReact, s, F8(ctx) * react_fields(MODE, a));
  CU(cudaGetLastError());
  return CISDC_OK;
}

template <int MODE>
int launch_react_m(cisdc_gpu_ctx* ctx, const ReactArgs& a, cudaStream_t s) {
  switch (ctx->S) {
    case 1: return launch_react_sm<1, MODE>(ctx, a, s);
    case 2: return launch_react_sm<2, MODE>(ctx, a, s);
    case 3: return launch_react_sm<3, MODE>(ctx, a, s);
    case 4: return launch_react_sm<4, MODE>(ctx, a, s);
    case 9: return launch_react_sm<9, MODE>(ctx, a, s);
  }
  return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "unsupported species count");
}

template <int S, int MODE>
void launch_fixup_sm(cisdc_gpu_ctx* ctx, const ReactArgs& a, cudaStream_t s) {
  const dim3 grid(148), block(128);
  if constexpr (MODE == kModeMisdcq || MODE == kModeMisdc) {
    if (a.fd_ad) k_react_fixup<S, 0, MODE><<<grid, block, 0, s>>>(ctx->rx, ctx->ops, ctx->g, a, ctx->d_st);
    else k_react_fixup<S, 1, MODE><<<grid, block, 0, s>>>(ctx->rx, ctx->ops, ctx->g, a, ctx->d_st);
  } else {
    k_react_fixup<S, 1, MODE><<<grid, block, 0, s>>>(ctx->rx, ctx->ops, ctx->g, a, ctx->d_st);
  }
}

template <int MODE>
void launch_fixup_m(cisdc_gpu_ctx* ctx, const ReactArgs& a, cudaStream_t s) {
  switch (ctx->S) {
    case 1: launch_fixup_sm<1, MODE>(ctx, a, s); break;
    case 2: launch_fixup_sm<2, MODE>(ctx, a, s); break;
    case 3: launch_fixup_sm<3, MODE>(ctx, a, s); break;
    case 4: launch_fixup_sm<4, MODE>(ctx, a, s); break;
    default: launch_fixup_sm<9, MODE>(ctx, a, s); break;
  }
}

double rhs_fields(const RhsArgs& a);

// next: the right-hand side of the following diffusion cell, assembled by the same kernel
// (k_react_next; the network-specialised CISDCQ kernel only -- see can_fuse_next_rhs)
int launch_react(cisdc_gpu_ctx* ctx, int mode, const ReactArgs& a_in, cudaStream_t s, const RhsArgs* next = nullptr) {
  if (ctx->linear && 1.0 - a_in.coef * ctx->lin_r == 0.0)
    return set_err(ctx, CISDC_E_SOLVE, "LinearScalarProblem: singular reaction stage");
  ReactArgs a = a_in;
  a.tag = next_tag(ctx, CISDC_STAGE_REACTION);
  if (ctx->rtc.ready) {
    Reaction rx = ctx->rx;
    Ops o = ctx->ops;
    Geom g = ctx->g;
    ReactArgs aa = a;
    aa.defer_list = ctx->defer_list;
    aa.defer_count = ctx->defer_count;
    DevStatus* st = ctx->d_st;
    RhsArgs nx{};
    if (next) {
      nx = *next;
      nx.wild = ctx->ops.wild;
    }
    void* args[6] = {&rx, &o, &g, &aa, &st, &nx};
    const int cls = next ? kKReactRhs : kKReact;
    ctx->tm.before(cls, s);
    CU(cudaLaunchKernel(reinterpret_cast<const void*>(ctx->rtc.fn[next ? 4 : mode]), dim3(grid_of(ctx->g.ncell, 128)),
                        dim3(128), args, 0, s));
    ctx->tm.after(cls, s, F8(ctx) * (react_fields(mode, a) + (next ? rhs_fields(nx) : 0.0)));
    // cells whose LU needed a row interchange: dense generic kernel, then reset the list
    ctx->tm.before(kKReact, s);
    switch (mode) {
      case kModeMisdcq: launch_fixup_m<kModeMisdcq>(ctx, aa, s); break;
      case kModeMisdc: launch_fixup_m<kModeMisdc>(ctx, aa, s); break;
      case kModeCisdcq: launch_fixup_m<kModeCisdcq>(ctx, aa, s); break;
      default: launch_fixup_m<kModePlain>(ctx, aa, s); break;
    }
    ctx->tm.after(kKReact, s, 0.0);
    CU(cudaGetLastError());
    CU(cudaMemsetAsync(ctx->defer_count, 0, sizeof(int), s));
    return CISDC_OK;
  }
  if (next) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "launch_react: fused next rhs needs the specialised kernel");
  switch (mode) {
    case kModeMisdcq: return launch_react_m<kModeMisdcq>(ctx, a, s);
    case kModeMisdc: return launch_react_m<kModeMisdc>(ctx, a, s);
    case kModeCisdcq: return launch_react_m<kModeCisdcq>(ctx, a, s);
    default: return launch_react_m<kModePlain>(ctx, a, s);
  }
}

// compulsory traffic = distinct arrays (right after initialize every node view aliases node 0)
double distinct_fields(std::vector<const void*> p) {
  p.erase(std::remove(p.begin(), p.end(), nullptr), p.end());
  std::sort(p.begin(), p.end());
  return (double)(std::unique(p.begin(), p.end()) - p.begin());
}

// compulsory fields (distinct inputs + outputs) of one stage right-hand side
double rhs_fields(const RhsArgs& a) {
  std::vector<const void*> in;
  if (a.kind == kRhsMisdc) {
    in.push_back(a.phim);
    for (int j = 0; j <= a.M; ++j) in.insert(in.end(), {a.sfa[j], a.sfd[j], a.sfr[j]});
  } else {
    in.push_back(a.base);
    for (int t = 0; t < a.nt; ++t) {
      const RhsTerm& T = a.t[t];
      if (!T.skipA && T.diff && T.dA) in.push_back(T.dA);
      else if (!T.skipA) in.insert(in.end(), {T.A, T.Ap});
      if (T.diff) in.push_back(T.D);
      else in.insert(in.end(), {T.D, T.Dp, T.R, T.Rp});
    }
  }
  if (a.kind == kRhsCisdcq && a.X == a.Y) in.push_back(a.Z);  // X - Y = +0.0: X is not read (rhs.cuh)
  else in.insert(in.end(), {a.X, a.Y, a.Z});
  double outs = 1 + (a.out2 != nullptr) + (a.base_out != nullptr);
  for (int t = 0; t < a.nt; ++t) outs += (a.t[t].outA != nullptr) + (a.t[t].outDR != nullptr);
  return distinct_fields(in) + outs;
}

int launch_rhs(cisdc_gpu_ctx* ctx, const RhsArgs& a, cudaStream_t s) {
  const double fields = rhs_fields(a);
  RhsArgs aw = a;
  aw.wild = ctx->ops.wild;
  ctx->tm.before(kKRhs, s);
  k_rhs<<<grid_of(ctx->g.n, 256), 256, 0, s>>>(aw, ctx->g.n);
  ctx->tm.after(kKRhs, s, F8(ctx) * fields);
  CU(cudaGetLastError());
  return CISDC_OK;
}

// quadrature_base for all M rows; fuse (optional): the first stage rhs (k_rhs arguments with
// nt == 0 and base == base[0]), assembled in the same pass; skip_base0: base row 0 has no other
// reader and is not stored
int launch_quad_base(cisdc_gpu_ctx* ctx, int set, double dt, cudaStream_t s, const RhsArgs* fuse = nullptr,
                     bool skip_base0 = false) {
  QuadArgs q{};
  const int M = ctx->M;
  q.M = M;
  for (int m = 0; m < M; ++m)
    for (int j = 0; j <= M; ++j) q.c[m][j] = dt * ctx->tb.Q[m * (M + 1) + j];
  q.phi0 = ctx->node0[kPhi];
  for (int j = 0; j <= M; ++j) {
    q.fa[j] = V(ctx, set, kFa, j);
    q.fd[j] = V(ctx, set, kFd, j);
    q.fr[j] = V(ctx, set, kFr, j);
  }
  for (int m = 0; m < M; ++m) q.base[m] = ctx->base[m];
  std::vector<const void*> in{q.phi0};
  for (int j = 0; j <= M; ++j) in.insert(in.end(), {q.fa[j], q.fd[j], q.fr[j]});
  double outs = M;
  if (fuse) {
    q.rhs0_kind = fuse->kind == kRhsMisdcq ? 1 : 2;
    q.fc = fuse->fc;
    q.X = fuse->X;
    q.Y = fuse->Y;
    q.Z = fuse->Z;
    q.rhs0 = fuse->out;
    in.insert(in.end(), {q.X, q.Y, q.Z});
    outs += 1;
    if (skip_base0) {
      q.base[0] = nullptr;
      outs -= 1;
    }
  }
  ctx->tm.before(kKQuad, s);
  k_quad_base<<<grid_of(ctx->g.n, 256), 256, 0, s>>>(q, ctx->g.n);
  ctx->tm.after(kKQuad, s, F8(ctx) * (distinct_fields(in) + outs));
  CU(cudaGetLastError());
  return CISDC_OK;
}

template <int E>
int launch_solve1d_e(cisdc_gpu_ctx* ctx, const Solve1dArgs& a, int cl, cudaStream_t s) {
  constexpr int T = kSolve1dThreads;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cl * ctx->S, 1, 1);
  cfg.blockDim = dim3(T, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cl > 8)  // clusters above 8 CTAs are opt-in
    CU(func_attr_once(k_solve1d_periodic<E, T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  ctx->tm.before(kKSolve1d, s);
  CU(cudaLaunchKernelEx(&cfg, k_solve1d_periodic<E, T>, a));
  ctx->tm.after(kKSolve1d, s, 2.0 * F8(ctx));
  return CISDC_OK;
}

// LinearScalarProblem stage solves (linear.cpp:32-50): denom = 1 - coef * c, checked here (the
// reference throws SolveError before touching the output)
int linear_solve(cisdc_gpu_ctx* ctx, int stage, double coef, const double* rhs, double* out, cudaStream_t s) {
  double denom;
  const char* what;
  if (stage == CISDC_STAGE_DIFFUSION) {
    denom = 1.0 - coef * ctx->lin_d;
    what = "LinearScalarProblem: singular diffusion stage";
  } else if (stage == CISDC_STAGE_REACTION) {
    denom = 1.0 - coef * ctx->lin_r;
    what = "LinearScalarProblem: singular reaction stage";
  } else {
    denom = 1.0 - coef * (ctx->lin_d + ctx->lin_r);
    what = "LinearScalarProblem: singular coupled stage";
  }
  if (denom == 0.0) return set_err(ctx, CISDC_E_SOLVE, what);
  const int cls = stage == CISDC_STAGE_REACTION ? kKReact : kKSolve1d;
  ctx->tm.before(cls, s);
  k_lin_div<<<grid_of(ctx->g.n, 256), 256, 0, s>>>(rhs, out, denom, ctx->g.n);
  ctx->tm.after(cls, s, 2.0 * F8(ctx));
  CU(cudaGetLastError());
  return CISDC_OK;
}

int solve_diffusion(cisdc_gpu_ctx* ctx, double coef, const double* rhs, double* out, cudaStream_t s) {
  const long long n = ctx->g.n;
  if (ctx->linear) return linear_solve(ctx, CISDC_STAGE_DIFFUSION, coef, rhs, out, s);
  if (ctx->ref_rd) {
    if (coef == 0.0) {
      CU(cudaMemcpyAsync(out, rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      return CISDC_OK;
    }
    RdSolveArgs a{};
    a.n = ctx->g.nx;
    const double dx = (20.0 - 0.0) / ctx->g.nx;
    a.c = coef * ctx->desc.ref_d / (12.0 * dx * dx);
    std::memcpy(a.w, ctx->ops.rd_w, sizeof(a.w));
    a.rhs = rhs;
    a.out = out;
    a.work = ctx->rd_work;
    a.tag = next_tag(ctx, CISDC_STAGE_DIFFUSION);
    ctx->tm.before(kKSolve1d, s);
    k_rd_banded_solve<<<1, 32, 0, s>>>(a, ctx->d_st);
    ctx->tm.after(kKSolve1d, s, 2.0 * F8(ctx));
    CU(cudaGetLastError());
    return CISDC_OK;
  }
  if (ctx->desc.diffusion_solver == CISDC_DIFFUSION_MULTIGRID) {
    const int rc = mg_solve(ctx->mg, ctx->g, ctx->desc, coef, rhs, out, ctx->d_st,
                            next_tag(ctx, CISDC_STAGE_DIFFUSION), s, &ctx->tm);
    if (rc) return set_err(ctx, rc, "multigrid launch failed");
    return CISDC_OK;
  }
  // periodic 1-D direct solve, one cluster per species
  Solve1dArgs a{};
  a.rhs = rhs;
  a.out = out;
  a.N = ctx->g.nx;
  for (int sp = 0; sp < ctx->S; ++sp) {
    const double c = coef * ctx->ops.cdiff[sp][0];
    a.active[sp] = (coef != 0.0 && c != 0.0);
    if (a.active[sp]) {
      const CircFactor f = factor_circulant(c);
      a.c[sp].npass = f.npass;
      for (int k = 0; k < 4; ++k) {
        a.c[sp].p[k] = f.p[k];
        a.c[sp].q[k] = f.q[k];
        a.c[sp].reverse[k] = f.reverse[k];
        a.c[sp].kind[k] = f.kind[k];
      }
      a.c[sp].invK = f.invK;
    }
  }
  int E = 1, cl = 1;
  solve1d_blocking(ctx->g.nx, &E, &cl);
  switch (E) {
    case 1: return launch_solve1d_e<1>(ctx, a, cl, s);
    case 2: return launch_solve1d_e<2>(ctx, a, cl, s);
    case 4: return launch_solve1d_e<4>(ctx, a, cl, s);
    case 8: return launch_solve1d_e<8>(ctx, a, cl, s);
    case 16: return launch_solve1d_e<16>(ctx, a, cl, s);
    default: return launch_solve1d_e<32>(ctx, a, cl, s);
  }
}

int launch_incr(cisdc_gpu_ctx* ctx, const double* a, const double* b, double* out, cudaStream_t s) {
  ctx->tm.before(kKIncr, s);
  k_incr_partial<<<kIncrBlocks, kIncrThreads, 0, s>>>(a, b, ctx->g.n, ctx->d_partial);
  ctx->tm.after(kKIncr, s, 2.0 * F8(ctx));
  ctx->tm.before(kKIncr, s);
  k_incr_final<<<1, 1024, 0, s>>>(a, b, ctx->g.n, ctx->d_partial, out);
  ctx->tm.after(kKIncr, s, 0.0);
  CU(cudaGetLastError());
  return CISDC_OK;
}

// ---------------------------------------------------------------- status

// Synchronises s_main, harvests timing and the device status word.
int check_status(cisdc_gpu_ctx* ctx, cisdc_counters* counters) {
  cudaStream_t s = ctx->s_main;
  CU(cudaMemcpyAsync(ctx->h_st, ctx->d_st, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  ctx->tm.resolve();
  const DevStatus h = *ctx->h_st;
  if (counters) {
    counters->newton_iterations += (long long)(h.newton_trips - ctx->newton_seen);
    counters->mg_cycles += (long long)(h.mg_cycles - ctx->mg_seen);
  }
  ctx->newton_seen = h.newton_trips;
  ctx->newton_res_exits = h.newton_res_exits;
  ctx->tm.add_launches((long long)(h.loop_kernels - ctx->loop_seen));
  ctx->loop_seen = h.loop_kernels;
  ctx->mg_seen = h.mg_cycles;
  ctx->fail_sweep = 0;
  if (h.fail_key != ~0ull) {
    const unsigned tag = (unsigned)(h.fail_key >> 35);
    const int code = (int)((h.fail_key >> 32) & 7);
    const unsigned long long cell = h.fail_key & 0xffffffffull;
    const int stage = (tag >= 1 && tag <= ctx->tags.size()) ? ctx->tags[tag - 1].second : CISDC_STAGE_REACTION;
    ctx->fail_sweep = (tag >= 1 && tag <= ctx->tags.size()) ? ctx->tags[tag - 1].first : 0;
    char buf[256];
    if (stage == CISDC_STAGE_REACTION) {
      std::snprintf(buf, sizeof(buf), "solve_reaction_implicit: cell %llu: %s", cell,
                    code == CISDC_E_SOLVE ? "newton: singular jacobian"
                                          : "newton: no convergence within the iteration cap");
    } else if (ctx->ref_rd) {
      std::snprintf(buf, sizeof(buf), "banded_solve: singular band at column %llu", cell);
    } else {
      std::snprintf(buf, sizeof(buf), "solve_diffusion: multigrid: species %llu: no convergence in %d cycles", cell,
                    ctx->desc.mg_max_cycles);
    }
    DevStatus z{};  // reset the status word so the context stays usable
    z.fail_key = ~0ull;
    z.newton_trips = h.newton_trips;
    z.newton_res_exits = h.newton_res_exits;
    z.loop_kernels = h.loop_kernels;
    z.mg_cycles = h.mg_cycles;
    CU(cudaMemcpy(ctx->d_st, &z, sizeof(z), cudaMemcpyHostToDevice));
    ctx->tags.clear();
    const int rc = (stage == CISDC_STAGE_REACTION || ctx->ref_rd) ? CISDC_E_SOLVE : code;
    return set_err(ctx, rc, buf);
  }
  ctx->tags.clear();
  return CISDC_OK;
}

// ---------------------------------------------------------------- coupled stage (periodic ADR)

bool has_coupled(const cisdc_gpu_ctx* ctx) {
  return ctx->linear || (!ctx->ref_rd && ctx->desc.coupled_max_iter > 0);
}

// OperatorSplitProblem::solve_coupled (operator_split.hpp:49-53) of the periodic ADR class, as
// cisdc_gpu.h defines it: y_0 = rhs; z = solve_D(coef, rhs + coef F_R(y_k)); y_{k+1} =
// solve_R(coef, rhs + coef F_D(z)) until max|y_{k+1} - y_k| <= coupled_tol max|y_{k+1}|.  Every step is
// one of the engine's stage kernels (F_R, the multigrid or 1-D direct solve, F_D, the Newton
// kernel); the host reads the two maxima (exact, so bit-equal to the oracle's serial loop) and the
// failure word once per iteration.  A stage failure inside ends the iteration and is reported by
// check_status with the failing stage's message, as the oracle returns it.
int solve_coupled_adr(cisdc_gpu_ctx* ctx, double coef, const double* rhs, double* out, cudaStream_t s,
                      cisdc_counters* c) {
  const long long n = ctx->g.n;
  if (coef == 0.0) {
    if (out != rhs) CU(cudaMemcpyAsync(out, rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    return CISDC_OK;
  }
  if (!ctx->cpl[0]) {
    for (int b = 0; b < 4; ++b) TRY(dalloc(ctx, &ctx->cpl[b], n));
    double* d2 = nullptr;
    TRY(dalloc(ctx, &d2, 2));
    ctx->d_cpl = reinterpret_cast<unsigned long long*>(d2);
    CU(cudaMallocHost(&ctx->h_cpl, 3 * sizeof(unsigned long long)));
  }
  double *y = ctx->cpl[0], *yn = ctx->cpl[1], *f = ctx->cpl[2], *z = ctx->cpl[3];
  const double* cur = rhs;  // y_0 = rhs, read in place
  const int blocks = grid_of(n, 256);
  bool converged = false;
  for (int it = 0; it < ctx->desc.coupled_max_iter && !converged; ++it) {
    TRY(launch_eval_r(ctx, cur, f, s));
    ctx->tm.before(kKRhs, s);
    k_axpy_inplace<<<blocks, 256, 0, s>>>(rhs, coef, f, n);
    ctx->tm.after(kKRhs, s, 3.0 * F8(ctx));
    TRY(solve_diffusion(ctx, coef, f, z, s));
    TRY(launch_eval_ad(ctx, z, nullptr, f, s));
    ctx->tm.before(kKRhs, s);
    k_axpy_inplace<<<blocks, 256, 0, s>>>(rhs, coef, f, n);
    ctx->tm.after(kKRhs, s, 3.0 * F8(ctx));
    ReactArgs a{};
    a.coef = coef;
    a.p0 = f;
    a.phi_out = yn;
    a.fr_out = nullptr;
    TRY(launch_react(ctx, kModePlain, a, s));
    CU(cudaMemsetAsync(ctx->d_cpl, 0, 2 * sizeof(unsigned long long), s));
    ctx->tm.before(kKIncr, s);
    k_coupled_delta<<<std::min(blocks, 8 * ctx->num_sms), 256, 0, s>>>(yn, cur, n, ctx->d_cpl);
    ctx->tm.after(kKIncr, s, 2.0 * F8(ctx));
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(ctx->h_cpl, ctx->d_cpl, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(ctx->h_cpl + 2, &ctx->d_st->fail_key, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (ctx->h_cpl[2] != ~0ull) return check_status(ctx, c);  // a stage solve inside failed
    double delta, scale;
    std::memcpy(&delta, ctx->h_cpl, sizeof(double));
    std::memcpy(&scale, ctx->h_cpl + 1, sizeof(double));
    converged = delta <= ctx->desc.coupled_tol * scale;
    std::swap(y, yn);  // the new iterate is y
    cur = y;
  }
  if (!converged) return set_err(ctx, CISDC_E_SOLVE, "periodic ADR: coupled solve did not converge");
  CU(cudaMemcpyAsync(out, cur, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  return CISDC_OK;
}

// ---------------------------------------------------------------- sweeps

double QI(const cisdc_tables& t, int m, int j) { return t.QtI[m * t.M + j]; }
double QE(const cisdc_tables& t, int m, int j) { return t.QtE[m * t.M + j]; }

// The reaction stage of MISDC/MISDCQ adds F_D(phi_AD[m+1]) (integrators.cpp:90,125: a separate
// eval_diffusion in the reference too).  It is evaluated by the tiled stencil kernels into a
// scratch field that the Newton kernel then reads pointwise (its DIM = 0 instantiation), instead of
// a (4 ndim + 1)-tap stencil per species inside the FP64-bound Newton kernel: C4 33.3 -> 22.4 ms of
// Newton per step for 4.2 ms of evaluation.  1-D grids (L2-resident, launch-bound) keep the
// stencil inside.
bool react_fd_separate(const cisdc_gpu_ctx* ctx) { return ctx->linear || ctx->g.ndim >= 2; }
int prepare_fd_ad(cisdc_gpu_ctx* ctx, ReactArgs& a, cudaStream_t s) {
  if (!react_fd_separate(ctx)) return CISDC_OK;
  a.fd_ad = ctx->fd_ad[1];
  return launch_eval_ad(ctx, a.phi_ad, nullptr, ctx->fd_ad[1], s);
}

// misdcq_sweep (integrators.cpp:103-143)
int sweep_misdcq(cisdc_gpu_ctx* ctx, double dt, cisdc_counters* c) {
  const int M = ctx->M, prev = ctx->cur, nxt = 1 - ctx->cur;
  cudaStream_t s = ctx->s_main;
  reset_views(ctx, nxt);
  {  // node 0's diffusion rhs (base - coef fd_p[1]) in the quadrature pass
    RhsArgs r0{};
    r0.kind = kRhsMisdcq;
    r0.fc = dt * QI(ctx->tb, 0, 0);
    r0.X = V(ctx, prev, kFd, 1);
    r0.out = ctx->rhs_d;
    TRY(launch_quad_base(ctx, prev, dt, s, &r0));
  }
  for (int m = 0; m < M; ++m) {
    const double coef = dt * QI(ctx->tb, m, m);
    RhsArgs r{};
    r.kind = kRhsMisdcq;
    r.nt = m;
    for (int j = 1; j <= m; ++j) {
      RhsTerm& t = r.t[j - 1];
      t.cE = dt * QE(ctx->tb, m, j - 1);
      t.cI = dt * QI(ctx->tb, m, j - 1);
      t.skipA = t.cE == 0.0;
      t.A = V(ctx, nxt, kFa, j);
      t.Ap = V(ctx, prev, kFa, j);
      t.D = V(ctx, nxt, kFd, j);
      t.Dp = V(ctx, prev, kFd, j);
      t.R = V(ctx, nxt, kFr, j);
      t.Rp = V(ctx, prev, kFr, j);
    }
    r.fc = coef;
    r.X = V(ctx, prev, kFd, m + 1);
    r.base = ctx->base[m];
    r.out = ctx->rhs_d;
    r.out2 = m > 0 ? ctx->rhs_r : nullptr;
    if (m > 0) TRY(launch_rhs(ctx, r, s));
    TRY(solve_diffusion(ctx, coef, ctx->rhs_d, ctx->phi_ad[m + 1], s));
    if (c) ++c->diffusion;
    ReactArgs a{};
    a.coef = coef;
    a.p0 = m > 0 ? ctx->rhs_r : ctx->base[m];
    a.phi_ad = ctx->phi_ad[m + 1];
    a.fdp1 = V(ctx, prev, kFd, m + 1);
    a.frp1 = V(ctx, prev, kFr, m + 1);
    a.phi_out = ctx->own[nxt][kPhi][m + 1];
    a.fr_out = ctx->own[nxt][kFr][m + 1];
    TRY(prepare_fd_ad(ctx, a, s));
    TRY(launch_react(ctx, kModeMisdcq, a, s));
    if (c) ++c->reaction;
    TRY(launch_eval_ad(ctx, ctx->own[nxt][kPhi][m + 1], ctx->own[nxt][kFa][m + 1], ctx->own[nxt][kFd][m + 1], s));
  }
  return CISDC_OK;
}

// imexq_sweep (integrators.cpp:145-173): per node, rhs = base + sum_j [cE (fa - fa_p) + cI (fd - fd_p +
// fr - fr_p)]_j - coef (fd_p + fr_p)_{m+1}, the coupled solve phi - coef (F_D + F_R)(phi) = rhs,
// phi_AD = phi, and the three evaluations at phi.  Only problems with a coupled solve (the
// linear scalar model, as in the reference) run it.
int sweep_imexq(cisdc_gpu_ctx* ctx, double dt, cisdc_counters* c) {
  if (!has_coupled(ctx))
    return set_err(ctx, CISDC_E_CAPABILITY, "imexq_sweep: problem provides no coupled diffusion-reaction solve");
  const int M = ctx->M, prev = ctx->cur, nxt = 1 - ctx->cur;
  cudaStream_t s = ctx->s_main;
  reset_views(ctx, nxt);
  TRY(launch_quad_base(ctx, prev, dt, s));
  for (int m = 0; m < M; ++m) {
    const double coef = dt * QI(ctx->tb, m, m);
    RhsArgs r{};
    r.kind = kRhsImexq;
    r.nt = m;
    for (int j = 1; j <= m; ++j) {
      RhsTerm& t = r.t[j - 1];
      t.cE = dt * QE(ctx->tb, m, j - 1);
      t.cI = dt * QI(ctx->tb, m, j - 1);
      t.skipA = t.cE == 0.0;
      t.A = V(ctx, nxt, kFa, j);
      t.Ap = V(ctx, prev, kFa, j);
      t.D = V(ctx, nxt, kFd, j);
      t.Dp = V(ctx, prev, kFd, j);
      t.R = V(ctx, nxt, kFr, j);
      t.Rp = V(ctx, prev, kFr, j);
    }
    r.fc = coef;
    r.X = V(ctx, prev, kFd, m + 1);
    r.Y = V(ctx, prev, kFr, m + 1);
    r.base = ctx->base[m];
    r.out = ctx->rhs_d;
    TRY(launch_rhs(ctx, r, s));
    double* phi = ctx->own[nxt][kPhi][m + 1];
    if (ctx->linear) TRY(linear_solve(ctx, CISDC_STAGE_COUPLED, coef, ctx->rhs_d, phi, s));
    else TRY(solve_coupled_adr(ctx, coef, ctx->rhs_d, phi, s, c));
    if (c) ++c->coupled;
    CU(cudaMemcpyAsync(ctx->phi_ad[m + 1], phi, sizeof(double) * ctx->g.n, cudaMemcpyDeviceToDevice, s));
    TRY(launch_eval_ad(ctx, phi, ctx->own[nxt][kFa][m + 1], ctx->own[nxt][kFd][m + 1], s));
    TRY(launch_eval_r(ctx, phi, ctx->own[nxt][kFr][m + 1], s));
  }
  return CISDC_OK;
}

// misdc_sweep (integrators.cpp:69-101)
int sweep_misdc(cisdc_gpu_ctx* ctx, double dt, cisdc_counters* c) {
  const int M = ctx->M, prev = ctx->cur, nxt = 1 - ctx->cur;
  cudaStream_t s = ctx->s_main;
  reset_views(ctx, nxt);
  for (int m = 0; m < M; ++m) {
    const double dtm = dt * ctx->tb.dtau[m];
    RhsArgs r{};
    r.kind = kRhsMisdc;
    r.M = M;
    for (int j = 0; j <= M; ++j) {
      r.sc[j] = dt * ctx->tb.S[m * (M + 1) + j];
      r.sfa[j] = V(ctx, prev, kFa, j);
      r.sfd[j] = V(ctx, prev, kFd, j);
      r.sfr[j] = V(ctx, prev, kFr, j);
    }
    r.phim = V(ctx, nxt, kPhi, m);
    r.fc = dtm;
    r.X = V(ctx, nxt, kFa, m);
    r.Y = V(ctx, prev, kFa, m);
    r.Z = V(ctx, prev, kFd, m + 1);
    r.out = ctx->rhs_d;
    r.base_out = ctx->base[0];
    TRY(launch_rhs(ctx, r, s));
    TRY(solve_diffusion(ctx, dtm, ctx->rhs_d, ctx->phi_ad[m + 1], s));
    if (c) ++c->diffusion;
    ReactArgs a{};
    a.coef = dtm;
    a.p0 = ctx->base[0];
    a.phi_ad = ctx->phi_ad[m + 1];
    a.fam = V(ctx, nxt, kFa, m);
    a.fapm = V(ctx, prev, kFa, m);
    a.fdp1 = V(ctx, prev, kFd, m + 1);
    a.frp1 = V(ctx, prev, kFr, m + 1);
    a.phi_out = ctx->own[nxt][kPhi][m + 1];
    a.fr_out = ctx->own[nxt][kFr][m + 1];
    TRY(prepare_fd_ad(ctx, a, s));
    TRY(launch_react(ctx, kModeMisdc, a, s));
    if (c) ++c->reaction;
    TRY(launch_eval_ad(ctx, ctx->own[nxt][kPhi][m + 1], ctx->own[nxt][kFa][m + 1], ctx->own[nxt][kFd][m + 1], s));
  }
  return CISDC_OK;
}

// CISDCQ slot fields (integrators.hpp:93-107): ell == nu maps onto the next state set.
struct Slots {
  cisdc_gpu_ctx* ctx;
  int nxt, nu;
  double* get(int kind, int m, int ell) const {  // kind: 0 phi_ad, 1 phi_r, 2 fa_r, 3 fd_r, 4 fr_r
    if (ell == nu) {
      switch (kind) {
        case 0: return ctx->phi_ad[m];
        case 1: return ctx->own[nxt][kPhi][m];
        case 2: return ctx->own[nxt][kFa][m];
        case 3: return ctx->own[nxt][kFd][m];
        default: return ctx->own[nxt][kFr][m];
      }
    }
    return ctx->slot_bufs[((size_t)(ell - 1) * ctx->M + (m - 1)) * 5 + kind];
  }
};

int ensure_slots(cisdc_gpu_ctx* ctx, int nu) {
  const size_t need = (size_t)(nu - 1) * ctx->M * 5;
  while (ctx->slot_bufs.size() < need) {
    double* p = nullptr;
    TRY(dalloc(ctx, &p, ctx->g.n));
    ctx->slot_bufs.push_back(p);
  }
  const size_t dneed = ctx->M > 3 ? (size_t)(ctx->M - 3) * 2 : 0;
  while (ctx->diff_bufs.size() < dneed) {
    double* p = nullptr;
    TRY(dalloc(ctx, &p, ctx->g.n));
    ctx->diff_bufs.push_back(p);
  }
  return CISDC_OK;
}

// the right-hand side of run_diffusion_cell (integrators.cpp:201-226) as k_rhs arguments
RhsArgs diffusion_rhs(cisdc_gpu_ctx* ctx, const Slots& W, int m, int ell, double dt) {
  const int prev = ctx->cur, row = m - 1;
  RhsArgs r{};
  r.kind = kRhsCisdcq;
  int nt = 0;
  // the differences of node j's term are read in full by the first row that needs them (m = j+2),
  // which stores them when rows m+1 .. M will read them again (nodes j <= M-3)
  const bool cache = (int)ctx->diff_bufs.size() >= 2 * (ctx->M - 3) && ctx->M > 3;
  for (int j = 1; j <= m - 2; ++j) {
    RhsTerm& t = r.t[nt++];
    t.cE = dt * QE(ctx->tb, row, j - 1);
    t.cI = dt * QI(ctx->tb, row, j - 1);
    t.skipA = t.cE == 0.0;  // literal convention: every j <= m - 2 (k_rhs reads A, Ap only where needed)
    t.A = W.get(2, j, ell);
    t.Ap = V(ctx, prev, kFa, j);
    // the dA cache is needed only when some row reads cE * dA (cumulative convention)
    const bool cache_a = !t.skipA;
    if (cache && j < m - 2) {
      t.diff = 1;
      t.dA = cache_a ? ctx->diff_bufs[2 * (j - 1)] : nullptr;
      t.D = ctx->diff_bufs[2 * (j - 1) + 1];
      continue;
    }
    t.D = W.get(3, j, ell);
    t.Dp = V(ctx, prev, kFd, j);
    t.R = W.get(4, j, ell);
    t.Rp = V(ctx, prev, kFr, j);
    if (cache && j <= ctx->M - 3) {
      t.outA = cache_a ? ctx->diff_bufs[2 * (j - 1)] : nullptr;
      t.outDR = ctx->diff_bufs[2 * (j - 1) + 1];
    }
  }
  if (m >= 2) {
    RhsTerm& t = r.t[nt++];
    t.cE = dt * QE(ctx->tb, row, m - 2);
    t.cI = dt * QI(ctx->tb, row, m - 2);
    t.A = ell == 1 ? ctx->fa_ad[m - 1] : W.get(2, m - 1, ell - 1);
    t.Ap = V(ctx, prev, kFa, m - 1);
    t.D = ell == 1 ? ctx->fd_ad[m - 1] : W.get(3, m - 1, ell - 1);
    t.Dp = V(ctx, prev, kFd, m - 1);
    t.R = ell == 1 ? V(ctx, prev, kFr, m - 1) : W.get(4, m - 1, ell - 1);
    t.Rp = V(ctx, prev, kFr, m - 1);
  }
  r.nt = nt;
  const double coef = dt * QI(ctx->tb, row, m - 1);
  r.fc = coef;
  r.X = ell == 1 ? V(ctx, prev, kFr, m) : W.get(4, m, ell - 1);
  r.Y = V(ctx, prev, kFr, m);
  r.Z = V(ctx, prev, kFd, m);
  r.base = ctx->base[row];
  r.out = ctx->rhs_d;
  return r;
}

// cisdcq_cells::run_diffusion_cell (integrators.cpp:195-235); rhs_ready: D(1, 1)'s rhs was
// assembled by the sweep's quadrature pass
int diffusion_cell(cisdc_gpu_ctx* ctx, const Slots& W, int m, int ell, double dt, cudaStream_t s, cisdc_counters* c,
                   bool rhs_ready = false) {
  const int row = m - 1;
  const double coef = dt * QI(ctx->tb, row, m - 1);
  if (!rhs_ready) TRY(launch_rhs(ctx, diffusion_rhs(ctx, W, m, ell, dt), s));
  double* out = W.get(0, m, ell);
  TRY(solve_diffusion(ctx, coef, ctx->rhs_d, out, s));
  if (c) ++c->diffusion;
  // fa_ad / fd_ad of slot (m, 1) are read only by D(m+1, 1) (integrators.cpp:215-216): the
  // reference's evaluation at m = M has no reader and is skipped
  if (ell == 1 && m < ctx->M) TRY(launch_eval_ad(ctx, out, ctx->fa_ad[m], ctx->fd_ad[m], s));
  return CISDC_OK;
}

// cisdcq_cells::run_reaction_cell (integrators.cpp:237-258)
// next_rhs: the right-hand side of D(m+1, ell), assembled by this cell's Newton kernel; ev_newton is
// recorded right after that kernel (the D stream waits on it instead of on the whole cell)
int reaction_cell(cisdc_gpu_ctx* ctx, const Slots& W, int m, int ell, double dt, cudaStream_t s, cisdc_counters* c,
                  const RhsArgs* next_rhs = nullptr, cudaEvent_t ev_newton = nullptr) {
  const int prev = ctx->cur, row = m - 1;
  ReactArgs a{};
  a.coef = dt * QI(ctx->tb, row, m - 1);
  a.has_incr = m >= 2;
  if (m >= 2) {
    a.c2 = dt * QI(ctx->tb, row, m - 2);
    a.fr_new = W.get(4, m - 1, ell);
    a.lag_fr = ell == 1 ? V(ctx, prev, kFr, m - 1) : W.get(4, m - 1, ell - 1);
  }
  a.lag_frm = ell == 1 ? V(ctx, prev, kFr, m) : W.get(4, m, ell - 1);
  a.p0 = W.get(0, m, ell);
  a.phi_out = W.get(1, m, ell);
  a.fr_out = W.get(4, m, ell);
  TRY(launch_react(ctx, kModeCisdcq, a, s, next_rhs));
  if (ev_newton) CU(cudaEventRecord(ev_newton, s));
  if (c) ++c->reaction;
  TRY(launch_eval_ad(ctx, a.phi_out, W.get(2, m, ell), W.get(3, m, ell), s));
  return CISDC_OK;
}

// k_react_next serves the NVRTC-specialised mass-action kernel (CISDC_FUSE_RHS=0: separate k_rhs)
bool can_fuse_next_rhs(const cisdc_gpu_ctx* ctx) {
  static const bool env_on = [] {
    const char* e = std::getenv("CISDC_FUSE_RHS");
    return !e || std::atoi(e) != 0;
  }();
  return env_on && ctx->rtc.ready && !ctx->trace_on;
}

// cisdcq_sweep (workers == 0, integrators.cpp:273-288) or execute_pipelined (pipeline.cpp:171-320)
int sweep_cisdcq(cisdc_gpu_ctx* ctx, double dt, int nu, int workers, cisdc_counters* c) {
  if (nu < 1) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "cisdcq_sweep: nu must be >= 1");
  const int M = ctx->M, nxt = 1 - ctx->cur;
  TRY(ensure_slots(ctx, nu));
  reset_views(ctx, nxt);
  Slots W{ctx, nxt, nu};
  cudaStream_t sd = ctx->s_main;
  // D(1, 1)'s rhs reads base row 0 and node-1 fields only: assembled by the quadrature pass, and
  // base row 0 (read by D(1, ell) alone) is then not stored when nu == 1
  const RhsArgs r11 = diffusion_rhs(ctx, W, 1, 1, dt);
  TRY(launch_quad_base(ctx, ctx->cur, dt, sd, &r11, nu == 1));
  // R(m, ell)'s Newton kernel also assembles D(m+1, ell)'s right-hand side (k_react_next): the
  // network-specialised kernel only; off while a schedule trace is recorded (the D cell's rhs would
  // run inside the R cell's interval)
  const bool fuse = can_fuse_next_rhs(ctx);
  RhsArgs nr{};
  if (workers <= 0) {
    bool ready = true;  // D(1, 1): the quadrature pass
    for (int ell = 1; ell <= nu; ++ell)
      for (int m = 1; m <= M; ++m) {
        TRY(diffusion_cell(ctx, W, m, ell, dt, sd, c, ready));
        ready = fuse && m < M;
        if (ready) nr = diffusion_rhs(ctx, W, m + 1, ell, dt);
        TRY(reaction_cell(ctx, W, m, ell, dt, sd, c, ready ? &nr : nullptr));
      }
    return CISDC_OK;
  }
  // DAG of build_task_graph (pipeline.cpp:36-70): D cells on s_main, R cells on s_r; the
  // cross-stream edges D(m,l) -> R(m,l) and R(m-2,l), R(m-1,l-1), R(m,l-1) -> D(m,l) are events.
  // D cells are totally ordered on their stream (single rhs buffer); R cells write only their slots.
  cudaStream_t sr = ctx->s_r;
  const size_t ncells = (size_t)M * nu;
  while (ctx->ev_pool.size() < 3 * ncells) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->ev_pool.push_back(e);
  }
  auto evD = [&](int m, int ell) { return ctx->ev_pool[3 * ((size_t)(ell - 1) * M + (m - 1))]; };
  auto evR = [&](int m, int ell) { return ctx->ev_pool[3 * ((size_t)(ell - 1) * M + (m - 1)) + 1]; };
  // after R(m, ell)'s Newton kernel, which wrote D(m+1, ell)'s right-hand side (fuse)
  auto evN = [&](int m, int ell) { return ctx->ev_pool[3 * ((size_t)(ell - 1) * M + (m - 1)) + 2]; };
  // trace: start/end events of cell id (TaskGraph::cell_id = 2 ((ell-1) M + (m-1)) + kind)
  const bool tr = ctx->trace_on;
  if (tr) {
    while (ctx->trace_ev.size() < 4 * ncells + 1) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      ctx->trace_ev.push_back(e);
    }
    ctx->trace_M = M;
    ctx->trace_nu = nu;
    ctx->trace_workers = 2;
    ctx->trace_pending = true;
  }
  auto tev = [&](int kind, int m, int ell, int end) {
    return ctx->trace_ev[2 * (2 * ((size_t)(ell - 1) * M + (m - 1)) + kind) + end];
  };
  CU(cudaEventRecord(ctx->ev_base, sd));
  CU(cudaStreamWaitEvent(sr, ctx->ev_base, 0));
  bool ready = true;  // D(1, 1): the quadrature pass
  for (int ell = 1; ell <= nu; ++ell) {
    for (int m = 1; m <= M; ++m) {
      if (m >= 3) CU(cudaStreamWaitEvent(sd, evR(m - 2, ell), 0));
      if (ell >= 2) {
        if (m >= 2) CU(cudaStreamWaitEvent(sd, evR(m - 1, ell - 1), 0));
        CU(cudaStreamWaitEvent(sd, evR(m, ell - 1), 0));
      }
      if (ready && m >= 2) CU(cudaStreamWaitEvent(sd, evN(m - 1, ell), 0));
      if (tr) CU(cudaEventRecord(tev(0, m, ell, 0), sd));
      TRY(diffusion_cell(ctx, W, m, ell, dt, sd, c, ready));
      if (tr) CU(cudaEventRecord(tev(0, m, ell, 1), sd));
      CU(cudaEventRecord(evD(m, ell), sd));
      CU(cudaStreamWaitEvent(sr, evD(m, ell), 0));
      if (tr) CU(cudaEventRecord(tev(1, m, ell, 0), sr));
      ready = fuse && m < M;
      if (ready) nr = diffusion_rhs(ctx, W, m + 1, ell, dt);
      TRY(reaction_cell(ctx, W, m, ell, dt, sr, c, ready ? &nr : nullptr, ready ? evN(m, ell) : nullptr));
      if (tr) CU(cudaEventRecord(tev(1, m, ell, 1), sr));
      CU(cudaEventRecord(evR(m, ell), sr));
    }
  }
  CU(cudaEventRecord(ctx->ev_join, sr));
  CU(cudaStreamWaitEvent(sd, ctx->ev_join, 0));
  return CISDC_OK;
}

int check_ctx(cisdc_gpu_ctx* ctx) { return ctx ? CISDC_OK : CISDC_E_INVALID_ARGUMENT; }

// mass-action network of the descriptor -> Reaction (nu_sr = products - reactants)
int fill_mass_action(const cisdc_problem_desc* d, Reaction& rx, std::string& why) {
  const int S = d->nspecies;
  if (d->n_reactions < 0 || d->n_reactions > kMaxR) {
    why = "mass action: too many reactions";
    return 1;
  }
  rx.nr = d->n_reactions;
  for (int r = 0; r < rx.nr; ++r) {
    for (int t = 0; t < 2; ++t) {
      const int a = d->reactants[2 * r + t], p = d->products[2 * r + t];
      if (a >= S || p >= S) {
        why = "mass action: species index out of range";
        return 1;
      }
      rx.reac[r][t] = (signed char)(a < 0 ? -1 : a);
      if (a >= 0) rx.nu[a][r] -= 1;
      if (p >= 0) rx.nu[p][r] += 1;
    }
    if (rx.reac[r][0] < 0) {
      why = "mass action: every reaction needs a first reactant";
      return 1;
    }
    rx.k[r] = d->rate_constants[r];
  }
  return 0;
}

int do_initialize(cisdc_gpu_ctx* ctx) {
  cudaStream_t s = ctx->s_main;
  CU(cudaMemsetAsync(ctx->ops.wild, 0, sizeof(int), s));  // every F_A is evaluated afresh from here
  TRY(launch_eval_ad(ctx, ctx->node0[kPhi], ctx->node0[kFa], ctx->node0[kFd], s));
  TRY(launch_eval_r(ctx, ctx->node0[kPhi], ctx->node0[kFr], s));
  ctx->cur = 0;
  alias_views_to_node0(ctx, 0);
  reset_views(ctx, 1);
  ctx->have_incr = false;
  return CISDC_OK;
}

// one sweep, asynchronous; the increment lands in d_incr[slot]
int run_one_sweep(cisdc_gpu_ctx* ctx, int scheme, double dt, int nu, int workers, cisdc_counters* c, int slot) {
  const int prev = ctx->cur;
  const double* prev_end = V(ctx, prev, kPhi, ctx->M);
  switch (scheme) {
    case CISDC_SCHEME_MISDC: TRY(sweep_misdc(ctx, dt, c)); break;
    case CISDC_SCHEME_MISDCQ: TRY(sweep_misdcq(ctx, dt, c)); break;
    case CISDC_SCHEME_CISDCQ: TRY(sweep_cisdcq(ctx, dt, nu, workers, c)); break;
    case CISDC_SCHEME_IMEXQ: TRY(sweep_imexq(ctx, dt, c)); break;
    default: return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "unknown scheme");
  }
  const int nxt = 1 - prev;
  TRY(launch_incr(ctx, V(ctx, nxt, kPhi, ctx->M), prev_end, ctx->d_incr + slot, ctx->s_main));
  ctx->cur = nxt;
  return CISDC_OK;
}

int begin_timed(cisdc_gpu_ctx* ctx) {
  CU(cudaEventRecord(ctx->ev_t0, ctx->s_main));
  return CISDC_OK;
}

int end_timed(cisdc_gpu_ctx* ctx) {
  CU(cudaEventRecord(ctx->ev_t1, ctx->s_main));
  CU(cudaEventSynchronize(ctx->ev_t1));
  float t = 0.f;
  CU(cudaEventElapsedTime(&t, ctx->ev_t0, ctx->ev_t1));
  ctx->device_ms += t;
  return CISDC_OK;
}

}  // namespace

// ================================================================== C-ABI

extern "C" {

const char* cisdc_gpu_last_error(const cisdc_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
size_t cisdc_gpu_dimension(const cisdc_gpu_ctx* ctx) { return ctx ? (size_t)ctx->g.n : 0; }
long long cisdc_gpu_launch_count(const cisdc_gpu_ctx* ctx) { return ctx ? ctx->tm.launches : 0; }
long long cisdc_gpu_newton_residual_exits(const cisdc_gpu_ctx* ctx) {
  return ctx ? (long long)ctx->newton_res_exits : 0;
}

void cisdc_gpu_destroy(cisdc_gpu_ctx* ctx) {
  if (!ctx) return;
  cudaDeviceSynchronize();
  for (auto& g : ctx->step_graphs) cudaGraphExecDestroy(g.exec);
  for (void* p : ctx->allocs) cudaFree(p);
  mg_free(ctx->mg);
  rtc_free(ctx->rtc);
  if (ctx->h_st) cudaFreeHost(ctx->h_st);
  if (ctx->h_cpl) cudaFreeHost(ctx->h_cpl);
  if (ctx->h_incr) cudaFreeHost(ctx->h_incr);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->trace_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : {ctx->ev_base, ctx->ev_join, ctx->ev_t0, ctx->ev_t1})
    if (e) cudaEventDestroy(e);
  if (ctx->s_main) cudaStreamDestroy(ctx->s_main);
  if (ctx->s_r) cudaStreamDestroy(ctx->s_r);
  delete ctx;
}

static int build_ctx(cisdc_gpu_ctx* ctx, const cisdc_problem_desc* d, const cisdc_tables* tb) {
  ctx->desc = *d;
  ctx->tb = *tb;
  ctx->M = tb->M;
  if (ctx->M < 1 || ctx->M > kMaxM) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "M must be in 1..8");
  Geom& g = ctx->g;
  Ops& o = ctx->ops;
  Reaction& rx = ctx->rx;
  std::memset(&o, 0, sizeof(o));
  std::memset(&rx, 0, sizeof(rx));
  if (d->kind == CISDC_PROBLEM_REFERENCE_RD) {
    if (d->n[0] < 8) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "ReactionDiffusionGrid: n_x must be >= 8");
    ctx->ref_rd = true;
    g.nx = d->n[0];
    g.ny = g.nz = 1;
    g.ndim = 1;
    g.S = 1;
    o.ref_rd = 1;
    const double dx = (20.0 - 0.0) / g.nx;
    o.rd_cadv = d->ref_a / (12.0 * dx);
    o.rd_cdiff = d->ref_d / (12.0 * dx * dx);
    static const double pts[5] = {0.0, 0.5, 1.5, 2.5, 3.5};
    const double xg[2] = {-0.5, -1.5};
    for (int k = 0; k < 2; ++k)
      for (int j = 0; j < 5; ++j) {  // lagrange_weights_at, reaction_diffusion.cpp:34-46
        double num = 1.0, den = 1.0;
        for (int i = 0; i < 5; ++i) {
          if (i == j) continue;
          num *= xg[k] - pts[i];
          den *= pts[j] - pts[i];
        }
        o.rd_w[k][j] = num / den;
      }
    rx.ref_rd = 1;
    rx.ref_r = d->ref_r;
    rx.tol = 1e-14;
    rx.max_iter = 50;
  } else if (d->kind == CISDC_PROBLEM_PERIODIC_ADR) {
    if (d->ndim < 1 || d->ndim > 3) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "periodic ADR: ndim must be 1..3");
    const int S = d->nspecies;
    if (!(S == 1 || S == 2 || S == 3 || S == 4 || S == 9))
      return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "GPU path supports nspecies in {1,2,3,4,9}");
    g.S = S;
    g.ndim = d->ndim;
    g.nx = d->n[0];
    g.ny = d->ndim >= 2 ? d->n[1] : 1;
    g.nz = d->ndim >= 3 ? d->n[2] : 1;
    const int nn[3] = {g.nx, g.ny, g.nz};
    for (int a = 0; a < d->ndim; ++a)
      if (nn[a] < 8) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "periodic ADR: every active axis needs >= 8 cells");
    for (int a = 0; a < 3; ++a) {
      bool any = false;
      for (int b = 0; b < 3; ++b) {
        if (d->vel[a][b] && b < d->ndim && a < d->ndim) {
          double* p = nullptr;
          TRY(dalloc(ctx, &p, nn[b]));
          CU(cudaMemcpy(p, d->vel[a][b], sizeof(double) * nn[b], cudaMemcpyHostToDevice));
          o.vel[a][b] = p;
          any = true;
        }
      }
      o.adv[a] = any;
      if (a < d->ndim) o.cadv[a] = 1.0 / (12.0 * d->h[a]);
    }
    // uniform-velocity detection (the tiled 3-D F_A kernel then skips the per-face products)
    o.vconst = 1;
    for (int a = 0; a < 3; ++a) {
      double f[3] = {1.0, 1.0, 1.0};
      for (int b = 0; b < 3; ++b) {
        if (!o.vel[a][b]) continue;
        const double* t = d->vel[a][b];
        for (int i = 1; i < nn[b]; ++i)
          if (t[i] != t[0] || std::signbit(t[i]) != std::signbit(t[0])) o.vconst = 0;
        f[b] = t[0];
      }
      o.ucon[a] = (f[0] * f[1]) * f[2];
    }
    for (int s = 0; s < S; ++s) {
      const double ds = d->diffusivity ? d->diffusivity[s] : 0.0;
      for (int a = 0; a < d->ndim; ++a) o.cdiff[s][a] = ds / (12.0 * d->h[a] * d->h[a]);
    }
    rx.kind = d->reaction_kind;
    rx.lambda = d->lambda;
    rx.theta = d->theta;
    rx.tol = d->newton_tol;
    rx.max_iter = d->newton_max_iter;
    if (d->reaction_kind == CISDC_REACTION_LINEAR_DECAY || d->reaction_kind == CISDC_REACTION_BISTABLE) {
      if (S != 1) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "scalar reaction kinds need nspecies == 1");
    } else if (d->reaction_kind == CISDC_REACTION_MASS_ACTION) {
      std::string why;
      if (fill_mass_action(d, rx, why)) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, why);
      const char* env = std::getenv("CISDC_RTC");
      if (!(env && env[0] == '0')) {
        if (rtc_build(ctx->rtc, rx, S, d->ndim, true))
          return set_err(ctx, CISDC_E_CUDA, "NVRTC network kernel build failed:\n" + ctx->rtc.log);
      }
    } else if (d->reaction_kind != CISDC_REACTION_NONE) {
      return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "unknown reaction kind");
    }
    if (d->diffusion_solver == CISDC_DIFFUSION_DIRECT) {
      if (d->ndim != 1) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "direct diffusion solve is 1-D only; use multigrid");
      if (g.nx > 8 * kSolve1dThreads * 32) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "1-D direct solve supports n <= 131072");
    } else if (d->diffusion_solver != CISDC_DIFFUSION_MULTIGRID) {
      return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "diffusion solver not available on the GPU (oracle-only)");
    }
  } else if (d->kind == CISDC_PROBLEM_LINEAR_SCALAR) {
    // LinearScalarProblem (linear.hpp:31-51): n[0] >= 1 independent copies (n[0] = 1 is the
    // reference's dimension-1 problem); the only problem class with the coupled solve IMEXQ needs
    ctx->linear = true;
    g.nx = d->n[0] >= 1 ? d->n[0] : 1;
    g.ny = g.nz = 1;
    g.ndim = 1;
    g.S = 1;
    ctx->lin_a = d->ref_a;
    ctx->lin_d = d->ref_d;
    ctx->lin_r = d->ref_r;
    rx.kind = kReactLinear;
    rx.lambda = d->ref_r;
    rx.max_iter = 1;
  } else {
    return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "unknown problem kind");
  }
  // the caller's arrays are borrowed for the duration of create only (include/cisdc_gpu.h): keep
  // the diffusivities the multigrid plans read at every solve, forget the rest
  if (d->diffusivity && d->nspecies > 0) {
    ctx->diffusivity.assign(d->diffusivity, d->diffusivity + d->nspecies);
    ctx->desc.diffusivity = ctx->diffusivity.data();
  } else {
    ctx->diffusivity.assign(std::max(d->nspecies, 1), 0.0);
    ctx->desc.diffusivity = ctx->diffusivity.data();
  }
  for (auto& row : ctx->desc.vel)
    for (auto& t : row) t = nullptr;
  ctx->desc.reactants = ctx->desc.products = nullptr;
  ctx->desc.rate_constants = nullptr;
  g.ncell = (long long)g.nx * g.ny * g.nz;
  g.n = g.ncell * g.S;
  ctx->S = g.S;
  const long long n = g.n;
  for (int f = 0; f < 4; ++f) TRY(dalloc(ctx, &ctx->node0[f], n));
  for (int set = 0; set < 2; ++set)
    for (int f = 0; f < 4; ++f)
      for (int m = 1; m <= ctx->M; ++m) TRY(dalloc(ctx, &ctx->own[set][f][m], n));
  for (int m = 0; m <= ctx->M; ++m) TRY(dalloc(ctx, &ctx->phi_ad[m], n));
  CU(cudaMemset(ctx->phi_ad[0], 0, sizeof(double) * n));
  for (int m = 0; m < ctx->M; ++m) TRY(dalloc(ctx, &ctx->base[m], n));
  TRY(dalloc(ctx, &ctx->rhs_d, n));
  TRY(dalloc(ctx, &ctx->rhs_r, n));
  TRY(dalloc(ctx, &ctx->scratch, n));
  for (int m = 1; m <= ctx->M; ++m) {
    TRY(dalloc(ctx, &ctx->fa_ad[m], n));
    TRY(dalloc(ctx, &ctx->fd_ad[m], n));
  }
  if (ctx->ref_rd) TRY(dalloc(ctx, &ctx->rd_work, (size_t)g.nx * 10));
  if (ctx->rtc.ready) {
    void* v1 = nullptr;
    CU(cudaMalloc(&v1, sizeof(unsigned) * (size_t)g.ncell + sizeof(int)));
    ctx->allocs.push_back(v1);
    ctx->defer_list = static_cast<unsigned*>(v1);
    ctx->defer_count = reinterpret_cast<int*>(ctx->defer_list + g.ncell);
    CU(cudaMemset(ctx->defer_count, 0, sizeof(int)));
  }
  if (!ctx->ref_rd && !ctx->linear && d->diffusion_solver == CISDC_DIFFUSION_MULTIGRID) {
    const int rc = mg_init(ctx->mg, g, *d);
    if (rc) return set_err(ctx, rc, "multigrid: hierarchy setup failed (" + std::to_string(rc) + ")");
  }
  {
    void* w = nullptr;
    CU(cudaMalloc(&w, sizeof(int)));
    ctx->allocs.push_back(w);
    ctx->ops.wild = static_cast<int*>(w);
    CU(cudaMemset(ctx->ops.wild, 0, sizeof(int)));
  }
  void* v = nullptr;
  CU(cudaMalloc(&v, sizeof(DevStatus)));
  ctx->allocs.push_back(v);
  ctx->d_st = static_cast<DevStatus*>(v);
  DevStatus z{};
  z.fail_key = ~0ull;
  CU(cudaMemcpy(ctx->d_st, &z, sizeof(z), cudaMemcpyHostToDevice));
  CU(cudaMallocHost(&ctx->h_st, sizeof(DevStatus)));
  TRY(dalloc(ctx, &ctx->d_partial, kIncrBlocks));
  TRY(dalloc(ctx, &ctx->d_incr, kMaxSweepsPerStep));
  CU(cudaMallocHost(&ctx->h_incr, sizeof(double) * kMaxSweepsPerStep));
  {
    int dev = 0;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  // PMISDC: the D chain (s_main: rhs, multigrid, F_A/F_D) is the critical path; the R chain (s_r:
  // Newton) fills what it leaves, so s_main gets the higher priority
  {
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(cudaStreamCreateWithPriority(&ctx->s_main, cudaStreamNonBlocking, hi));
    CU(cudaStreamCreateWithPriority(&ctx->s_r, cudaStreamNonBlocking, lo));
  }
  CU(cudaEventCreateWithFlags(&ctx->ev_base, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  CU(cudaEventCreate(&ctx->ev_t0));
  CU(cudaEventCreate(&ctx->ev_t1));
  reset_views(ctx, 0);
  reset_views(ctx, 1);
  return CISDC_OK;
}

int cisdc_gpu_create(const cisdc_problem_desc* desc, const cisdc_tables* tables, cisdc_gpu_ctx** out) {
  if (!desc || !tables || !out) return CISDC_E_INVALID_ARGUMENT;
  *out = nullptr;
  cisdc_gpu_ctx* ctx = new cisdc_gpu_ctx();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    ctx->err = "no CUDA device: the B200 sweep engine has no CPU fallback";
    *out = ctx;  // the caller reads the message, then destroys
    return CISDC_E_CUDA;
  }
  const int rc = build_ctx(ctx, desc, tables);
  *out = ctx;
  return rc;
}

int cisdc_gpu_initialize(cisdc_gpu_ctx* ctx, const double* phi0, size_t n) {
  TRY(check_ctx(ctx));
  if (n != (size_t)ctx->g.n) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "SweepState::initialize: dimension mismatch");
  CU(cudaMemcpyAsync(ctx->node0[kPhi], phi0, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->s_main));
  TRY(do_initialize(ctx));
  return check_status(ctx, nullptr);
}

int cisdc_gpu_initialize_device(cisdc_gpu_ctx* ctx, const double* d_phi0, size_t n) {
  TRY(check_ctx(ctx));
  if (n != (size_t)ctx->g.n) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "SweepState::initialize: dimension mismatch");
  CU(cudaMemcpyAsync(ctx->node0[kPhi], d_phi0, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->s_main));
  TRY(do_initialize(ctx));
  return check_status(ctx, nullptr);
}

int cisdc_gpu_set_nodes(cisdc_gpu_ctx* ctx, const double* values, size_t n) {
  TRY(check_ctx(ctx));
  if (n != (size_t)ctx->g.n) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "SweepState::set_node_values: dimension mismatch");
  cudaStream_t s = ctx->s_main;
  ctx->cur = 0;
  reset_views(ctx, 0);
  reset_views(ctx, 1);
  CU(cudaMemsetAsync(ctx->ops.wild, 0, sizeof(int), s));
  for (int m = 0; m <= ctx->M; ++m) {
    double* phi = m == 0 ? ctx->node0[kPhi] : ctx->own[0][kPhi][m];
    double* fa = m == 0 ? ctx->node0[kFa] : ctx->own[0][kFa][m];
    double* fd = m == 0 ? ctx->node0[kFd] : ctx->own[0][kFd][m];
    double* fr = m == 0 ? ctx->node0[kFr] : ctx->own[0][kFr][m];
    CU(cudaMemcpyAsync(phi, values + (size_t)m * n, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    TRY(launch_eval_ad(ctx, phi, fa, fd, s));
    TRY(launch_eval_r(ctx, phi, fr, s));
  }
  ctx->have_incr = false;
  return check_status(ctx, nullptr);
}

int cisdc_gpu_sweep(cisdc_gpu_ctx* ctx, int scheme, double dt, int nu, int workers, cisdc_counters* inout) {
  TRY(check_ctx(ctx));
  TRY(begin_timed(ctx));
  TRY(run_one_sweep(ctx, scheme, dt, nu, workers, inout, 0));
  CU(cudaMemcpyAsync(ctx->h_incr, ctx->d_incr, sizeof(double), cudaMemcpyDeviceToHost, ctx->s_main));
  TRY(end_timed(ctx));
  TRY(check_status(ctx, inout));
  ctx->last_incr = ctx->h_incr[0];
  ctx->have_incr = true;
  return CISDC_OK;
}

int cisdc_gpu_increment(cisdc_gpu_ctx* ctx, double* out) {
  TRY(check_ctx(ctx));
  if (!ctx->have_incr) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "no sweep has run since initialize");
  *out = ctx->last_incr;
  return CISDC_OK;
}

static int field_ptr(cisdc_gpu_ctx* ctx, int which, int node, const double** p) {
  if (node < 0 || node > ctx->M) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "node out of range");
  if (which == CISDC_FIELD_PHI_AD) *p = ctx->phi_ad[node];
  else if (which >= 0 && which < 4) *p = V(ctx, ctx->cur, which, node);
  else return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "unknown field");
  return CISDC_OK;
}

int cisdc_gpu_get_field(cisdc_gpu_ctx* ctx, int which, int node, double* host, size_t n) {
  TRY(check_ctx(ctx));
  if (n != (size_t)ctx->g.n) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "get_field: dimension mismatch");
  const double* p = nullptr;
  TRY(field_ptr(ctx, which, node, &p));
  CU(cudaStreamSynchronize(ctx->s_main));
  CU(cudaMemcpy(host, p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return CISDC_OK;
}

int cisdc_gpu_get_field_device(cisdc_gpu_ctx* ctx, int which, int node, double* d_out, size_t n) {
  TRY(check_ctx(ctx));
  if (n != (size_t)ctx->g.n) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "get_field: dimension mismatch");
  const double* p = nullptr;
  TRY(field_ptr(ctx, which, node, &p));
  CU(cudaMemcpyAsync(d_out, p, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->s_main));
  CU(cudaStreamSynchronize(ctx->s_main));
  return CISDC_OK;
}

int cisdc_gpu_eval(cisdc_gpu_ctx* ctx, int stage, const double* phi, double* out, size_t n) {
  TRY(check_ctx(ctx));
  if (n != (size_t)ctx->g.n) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "eval: dimension mismatch");
  cudaStream_t s = ctx->s_main;
  CU(cudaMemcpyAsync(ctx->rhs_d, phi, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  if (stage == CISDC_STAGE_ADVECTION) TRY(launch_eval_ad(ctx, ctx->rhs_d, ctx->scratch, nullptr, s));
  else if (stage == CISDC_STAGE_DIFFUSION) TRY(launch_eval_ad(ctx, ctx->rhs_d, nullptr, ctx->scratch, s));
  else if (stage == CISDC_STAGE_REACTION) TRY(launch_eval_r(ctx, ctx->rhs_d, ctx->scratch, s));
  else return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "unknown stage");
  CU(cudaMemcpyAsync(out, ctx->scratch, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  return check_status(ctx, nullptr);
}

int cisdc_gpu_solve(cisdc_gpu_ctx* ctx, int stage, double coef, const double* rhs, double* out, size_t n,
                    cisdc_counters* inout) {
  TRY(check_ctx(ctx));
  if (n != (size_t)ctx->g.n) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "solve: dimension mismatch");
  cudaStream_t s = ctx->s_main;
  CU(cudaMemcpyAsync(ctx->rhs_d, rhs, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  if (stage == CISDC_STAGE_DIFFUSION) {
    TRY(solve_diffusion(ctx, coef, ctx->rhs_d, ctx->scratch, s));
  } else if (stage == CISDC_STAGE_REACTION) {
    ReactArgs a{};
    a.coef = coef;
    a.p0 = ctx->rhs_d;
    a.phi_out = ctx->scratch;
    a.fr_out = nullptr;
    TRY(launch_react(ctx, kModePlain, a, s));
  } else if (ctx->linear) {
    TRY(linear_solve(ctx, CISDC_STAGE_COUPLED, coef, ctx->rhs_d, ctx->scratch, s));
  } else if (has_coupled(ctx)) {
    TRY(solve_coupled_adr(ctx, coef, ctx->rhs_d, ctx->scratch, s, inout));
  } else {
    return set_err(ctx, CISDC_E_CAPABILITY, "OperatorSplitProblem: coupled diffusion-reaction solve not provided");
  }
  TRY(check_status(ctx, inout));
  CU(cudaMemcpy(out, ctx->scratch, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return CISDC_OK;
}

// cisdc::integrate (integrators.cpp:301-333).  Sweeps are enqueued asynchronously; without a
// stop tolerance the host synchronises once per step (increments and counters are harvested
// from device memory), with one it must look at every increment.
// one step's enqueue without host decisions: initialize, n sweeps, node 0 <- phi[M]
static int enqueue_step(cisdc_gpu_ctx* ctx, const cisdc_integrate_options* o, cisdc_counters* counters, int& done) {
  TRY(do_initialize(ctx));
  for (int k = 1; k <= o->n_sweeps; ++k) {
    ctx->cur_sweep = k;
    done = k - 1;
    TRY(run_one_sweep(ctx, o->scheme, o->dt, o->nu, o->workers, counters, k - 1));
  }
  CU(cudaMemcpyAsync(ctx->node0[kPhi], V(ctx, ctx->cur, kPhi, ctx->M), sizeof(double) * ctx->g.n,
                     cudaMemcpyDeviceToDevice, ctx->s_main));
  return CISDC_OK;
}

// whole-step graphs (CISDC_STEP_GRAPH=0: every step enqueued directly)
static bool step_graph_ok(const cisdc_gpu_ctx* ctx, const cisdc_integrate_options* o) {
  const char* e = std::getenv("CISDC_STEP_GRAPH");
  if (e && e[0] == '0') return false;
  const bool host_mg = !ctx->ref_rd && !ctx->linear && ctx->desc.diffusion_solver == CISDC_DIFFUSION_MULTIGRID;
  const bool host_coupled = o->scheme == CISDC_SCHEME_IMEXQ && !ctx->linear;  // the host reads every iteration's maxima
  return !o->has_stop_tol && !ctx->tm.on && !ctx->trace_on && !host_mg && !host_coupled;
}

static cisdc_gpu_ctx::StepGraph* find_step_graph(cisdc_gpu_ctx* ctx, const cisdc_integrate_options* o) {
  for (auto& g : ctx->step_graphs)
    if (g.scheme == o->scheme && g.nu == o->nu && g.workers == o->workers && g.n_sweeps == o->n_sweeps &&
        g.convention == ctx->tb.convention && g.dt == o->dt)
      return &g;
  return nullptr;
}

// capture one step (nothing executes); nullptr when capture is not possible
static cisdc_gpu_ctx::StepGraph* capture_step_graph(cisdc_gpu_ctx* ctx, const cisdc_integrate_options* o) {
  cudaStream_t s = ctx->s_main;
  const long long launches0 = ctx->tm.launches;
  ctx->tags.clear();
  cisdc_counters counts{};
  int done = 0;
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return nullptr;
  const int rc = enqueue_step(ctx, o, &counts, done);
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(s, &graph);
  cudaGetLastError();
  cisdc_gpu_ctx::StepGraph g{};
  g.kernels = ctx->tm.launches - launches0;
  ctx->tm.launches = launches0;
  if (rc || ec != cudaSuccess || !graph) {
    if (graph) cudaGraphDestroy(graph);
    ctx->tags.clear();
    return nullptr;
  }
  const cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) {
    cudaGetLastError();
    ctx->tags.clear();
    return nullptr;
  }
  g.scheme = o->scheme;
  g.nu = o->nu;
  g.workers = o->workers;
  g.n_sweeps = o->n_sweeps;
  g.convention = ctx->tb.convention;
  g.dt = o->dt;
  g.tags = ctx->tags;
  g.counts = counts;
  g.cur = ctx->cur;
  std::memcpy(g.view, ctx->view, sizeof(g.view));
  ctx->tags.clear();
  if (ctx->step_graphs.size() >= 8) {
    cudaGraphExecDestroy(ctx->step_graphs.front().exec);
    ctx->step_graphs.erase(ctx->step_graphs.begin());
  }
  ctx->step_graphs.push_back(g);
  return &ctx->step_graphs.back();
}

static int integrate_impl(cisdc_gpu_ctx* ctx, const double* phi0, bool phi0_device, size_t n,
                          const cisdc_integrate_options* o, double* final_state, bool final_device,
                          cisdc_step_report* reports, double* increments) {
  TRY(check_ctx(ctx));
  if (!o) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "integrate: null options");
  if (o->n_sweeps < 1) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "integrate: n_sweeps must be >= 1");
  if (o->n_sweeps > kMaxSweepsPerStep) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "integrate: too many sweeps");
  if (o->scheme == CISDC_SCHEME_CISDCQ && o->nu < 1) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "integrate: nu must be >= 1");
  if (o->M != ctx->M) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "integrate: options.M differs from the context's tables");
  if (n != (size_t)ctx->g.n) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "integrate: dimension mismatch");
  if (o->convention != ctx->tb.convention) {  // tables = make_quadrature_tables(M, convention)
    cisdc_tables t;
    if (make_tables(o->M, o->convention, &t)) return set_err(ctx, CISDC_E_INVALID_ARGUMENT, "bad tables");
    ctx->tb = t;
  }
  cudaStream_t s = ctx->s_main;
  TRY(begin_timed(ctx));
  CU(cudaMemcpyAsync(ctx->node0[kPhi], phi0, sizeof(double) * n,
                     phi0_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  for (int step = 0; step < o->n_steps; ++step) {
    cisdc_step_report rep{};
    int done = 0;
    // the reference's context prefix (integrators.cpp:320-321); the sweep comes from the failure's
    // tag (the status word is read once per step) or from the sweep that failed to enqueue
    auto fail = [&](int rc) {
      const int k = ctx->fail_sweep > 0 ? ctx->fail_sweep : done + 1;
      ctx->cur_sweep = 0;
      ctx->err = "integrate: step " + std::to_string(step + 1) + ", sweep " + std::to_string(k) + ": " + ctx->err;
      return rc == CISDC_E_CUDA ? rc : CISDC_E_SOLVE;
    };
    ctx->fail_sweep = 0;
    if (o->has_stop_tol) {
      TRY(do_initialize(ctx));
      for (int k = 1; k <= o->n_sweeps; ++k) {
        ctx->cur_sweep = k;
        int rc = run_one_sweep(ctx, o->scheme, o->dt, o->nu, o->workers, &rep.counters, k - 1);
        if (!rc) {
          CU(cudaMemcpyAsync(ctx->h_incr + (k - 1), ctx->d_incr + (k - 1), sizeof(double), cudaMemcpyDeviceToHost, s));
          rc = check_status(ctx, &rep.counters);
        }
        if (rc) return fail(rc);
        done = k;
        if (ctx->h_incr[k - 1] <= o->stop_tol) break;
      }
      // start = state.phi[M] becomes node 0 of the next step
      CU(cudaMemcpyAsync(ctx->node0[kPhi], V(ctx, ctx->cur, kPhi, ctx->M), sizeof(double) * n,
                         cudaMemcpyDeviceToDevice, s));
    } else {
      cisdc_gpu_ctx::StepGraph* sg = nullptr;
      if (step_graph_ok(ctx, o) && ctx->steps_direct > 0) {
        sg = find_step_graph(ctx, o);
        if (!sg) sg = capture_step_graph(ctx, o);
      }
      if (sg) {  // replay: the captured enqueue, and the host bookkeeping it did
        CU(cudaGraphLaunch(sg->exec, s));
        ctx->tm.add_launches(sg->kernels);
        ctx->tags = sg->tags;
        rep.counters.diffusion += sg->counts.diffusion;
        rep.counters.reaction += sg->counts.reaction;
        rep.counters.coupled += sg->counts.coupled;
        ctx->cur = sg->cur;
        std::memcpy(ctx->view, sg->view, sizeof(ctx->view));
        ctx->have_incr = false;
        done = o->n_sweeps - 1;
      } else {
        const int rc = enqueue_step(ctx, o, &rep.counters, done);
        ++ctx->steps_direct;
        if (rc) return fail(rc);
      }
      CU(cudaMemcpyAsync(ctx->h_incr, ctx->d_incr, sizeof(double) * o->n_sweeps, cudaMemcpyDeviceToHost, s));
      const int rc = check_status(ctx, &rep.counters);
      if (rc) return fail(rc);
      done = o->n_sweeps;
    }
    ctx->cur_sweep = 0;
    for (int k = 0; k < done; ++k)
      if (increments) increments[(size_t)step * o->n_sweeps + k] = ctx->h_incr[k];
    ctx->last_incr = ctx->h_incr[done - 1];
    ctx->have_incr = true;
    rep.sweeps = done;
    if (reports) reports[step] = rep;
  }
  CU(cudaMemcpyAsync(final_state, ctx->node0[kPhi], sizeof(double) * n,
                     final_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  TRY(end_timed(ctx));
  return CISDC_OK;
}

int cisdc_gpu_integrate(cisdc_gpu_ctx* ctx, const double* phi0, size_t n, const cisdc_integrate_options* opt,
                        double* final_state, cisdc_step_report* reports, double* increments) {
  return integrate_impl(ctx, phi0, false, n, opt, final_state, false, reports, increments);
}

int cisdc_gpu_integrate_device(cisdc_gpu_ctx* ctx, const double* d_phi0, size_t n, const cisdc_integrate_options* opt,
                               double* d_final_state, cisdc_step_report* reports, double* increments) {
  return integrate_impl(ctx, d_phi0, true, n, opt, d_final_state, true, reports, increments);
}

int cisdc_gpu_set_timing(cisdc_gpu_ctx* ctx, int on) {
  TRY(check_ctx(ctx));
  ctx->tm.on = on != 0;
  return CISDC_OK;
}

int cisdc_gpu_kernel_times(cisdc_gpu_ctx* ctx, double* ms, double* bytes, long long* launches, int max_classes,
                           int reset) {
  if (!ctx) return 0;
  const int nc = std::min<int>(max_classes, kNumKernelClasses);
  for (int c = 0; c < nc; ++c) {
    if (ms) ms[c] = ctx->tm.ms[c];
    if (bytes) bytes[c] = ctx->tm.bytes[c];
    if (launches) launches[c] = ctx->tm.count[c];
  }
  if (reset) {
    ctx->tm.reset();
    ctx->device_ms = 0.0;
  }
  return nc;
}

int cisdc_rtc_compile_check(const cisdc_problem_desc* d, char* log, size_t cap) {
  if (!d || d->reaction_kind != CISDC_REACTION_MASS_ACTION) return CISDC_E_INVALID_ARGUMENT;
  Reaction rx{};
  std::string why;
  if (fill_mass_action(d, rx, why)) {
    if (log && cap) std::snprintf(log, cap, "%s", why.c_str());
    return CISDC_E_INVALID_ARGUMENT;
  }
  rx.kind = CISDC_REACTION_MASS_ACTION;
  RtcNewton r;
  const int rc = rtc_build(r, rx, d->nspecies, d->ndim, false);
  if (log && cap) std::snprintf(log, cap, "%s", (rc ? r.log : std::string("ok\n") + r.log).c_str());
  return rc;
}

// ---------------------------------------------------------------- iteration-matrix scans

static thread_local std::string g_last_err;
const char* cisdc_last_error(void) { return g_last_err.c_str(); }

int cisdc_log_r_grid(double lo_exp, double hi_exp, int points_per_decade, double* out, size_t cap) {
  if (points_per_decade < 1) {
    g_last_err = "log_r_grid: points_per_decade >= 1";
    return -1;
  }
  const int n = static_cast<int>(std::lround((hi_exp - lo_exp) * points_per_decade));
  for (int i = 0; i <= n; ++i) {
    const double e = lo_exp + (hi_exp - lo_exp) * i / n;
    if (out && (size_t)i < cap) out[i] = -std::pow(10.0, e);
  }
  return n + 1;
}

int cisdc_gpu_spectral_radius_scan(const int* schemes, int n_schemes, const int* nu_list, int n_nu,
                                   const double* r_grid, int n_r, int d_rule, double fixed_d, double a, double dt,
                                   int M, int convention, cisdc_scan_point* out, size_t cap, size_t* n_out,
                                   double* G_out) {
  if (!r_grid || n_r < 1) {
    g_last_err = "spectral_radius_scan: empty r grid";
    return CISDC_E_INVALID_ARGUMENT;
  }
  if (!schemes || n_schemes < 1) {
    g_last_err = "spectral_radius_scan: no schemes";
    return CISDC_E_INVALID_ARGUMENT;
  }
  if (M < 1 || M > kMaxM) {
    g_last_err = "spectral_radius_scan: M must be in 1..8";
    return CISDC_E_INVALID_ARGUMENT;
  }
  ScanArgs A{};
  std::vector<std::pair<int, int>> groups;
  for (int i = 0; i < n_schemes; ++i) {
    if (schemes[i] < 0 || schemes[i] > 3) {
      g_last_err = "spectral_radius_scan: unknown scheme";
      return CISDC_E_INVALID_ARGUMENT;
    }
    if (schemes[i] == CISDC_SCHEME_CISDCQ) {
      for (int k = 0; k < n_nu; ++k) groups.push_back({schemes[i], nu_list[k]});
    } else {
      groups.push_back({schemes[i], 1});
    }
  }
  if (groups.size() > 64) {
    g_last_err = "spectral_radius_scan: at most 64 (scheme, nu) groups per call";
    return CISDC_E_INVALID_ARGUMENT;
  }
  const size_t np = groups.size() * (size_t)n_r;
  if (n_out) *n_out = np;
  if (!out || cap < np) {
    g_last_err = "spectral_radius_scan: output capacity";
    return CISDC_E_INVALID_ARGUMENT;
  }
  cisdc_tables t;
  if (make_tables(M, convention, &t)) {
    g_last_err = "spectral_radius_scan: quadrature tables";
    return CISDC_E_INVALID_ARGUMENT;
  }
  ScanTables tb{};
  tb.M = M;
  for (int m = 0; m < M; ++m) {
    tb.dtau[m] = t.dtau[m];
    for (int j = 0; j <= M; ++j) {
      tb.Q[m][j] = t.Q[m * (M + 1) + j];
      tb.S[m][j] = t.S[m * (M + 1) + j];
    }
    for (int j = 0; j < M; ++j) {
      tb.QtI[m][j] = t.QtI[m * M + j];
      tb.QtE[m][j] = t.QtE[m * M + j];
    }
  }
  A.n_points = (int)np;
  A.n_r = n_r;
  A.n_groups = (int)groups.size();
  for (size_t g = 0; g < groups.size(); ++g) {
    A.scheme[g] = groups[g].first;
    A.nu[g] = groups[g].second;
  }
  A.d_rule = d_rule;
  A.fixed_d = fixed_d;
  A.a = a;
  A.dt = dt;
  double *d_r = nullptr, *d_gamma = nullptr, *d_G = nullptr;
  int* d_ok = nullptr;
  auto fail = [&](cudaError_t e) {
    cudaFree(d_r);
    cudaFree(d_gamma);
    cudaFree(d_ok);
    cudaFree(d_G);
    g_last_err = std::string("CUDA error: ") + cudaGetErrorString(e);
    return CISDC_E_CUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&d_r, sizeof(double) * n_r)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&d_gamma, sizeof(double) * np)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&d_ok, sizeof(int) * np)) != cudaSuccess) return fail(e);
  if (G_out && (e = cudaMalloc(&d_G, sizeof(double) * np * M * M)) != cudaSuccess) return fail(e);
  if ((e = cudaMemcpy(d_r, r_grid, sizeof(double) * n_r, cudaMemcpyHostToDevice)) != cudaSuccess) return fail(e);
  A.r_grid = d_r;
  A.gamma = d_gamma;
  A.ok = d_ok;
  A.G = d_G;
  k_spectral_scan<<<(unsigned)((np + 63) / 64), 64>>>(tb, A);
  if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
  std::vector<double> gam(np);
  std::vector<int> ok(np);
  if ((e = cudaMemcpy(gam.data(), d_gamma, sizeof(double) * np, cudaMemcpyDeviceToHost)) != cudaSuccess) return fail(e);
  if ((e = cudaMemcpy(ok.data(), d_ok, sizeof(int) * np, cudaMemcpyDeviceToHost)) != cudaSuccess) return fail(e);
  if (G_out && (e = cudaMemcpy(G_out, d_G, sizeof(double) * np * M * M, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return fail(e);
  for (size_t p = 0; p < np; ++p) {
    const int g = (int)(p / n_r);
    const double r = r_grid[p % n_r];
    cisdc_scan_point& o = out[p];
    o.scheme = groups[g].first;
    o.M = M;
    o.nu = groups[g].second;
    o.a = a;
    o.d = d_rule == 0 ? r / 2.0 : fixed_d;
    o.r = r;
    o.dt = dt;
    o.gamma = gam[p];
    o.ok = ok[p];
  }
  cudaFree(d_r);
  cudaFree(d_gamma);
  cudaFree(d_ok);
  cudaFree(d_G);
  return CISDC_OK;
}

int cisdc_gpu_spectral_radius_batch(const double* A, int n, int count, double* rho, int* status) {
  if (n < 1 || n > kMaxM || count < 0 || (count > 0 && (!A || !rho || !status))) {
    g_last_err = "spectral_radius_batch: n must be in 1..8";
    return CISDC_E_INVALID_ARGUMENT;
  }
  if (count == 0) return CISDC_OK;
  double *dA = nullptr, *dr = nullptr;
  int* ds = nullptr;
  cudaError_t e = cudaMalloc(&dA, sizeof(double) * (size_t)count * n * n);
  if (e == cudaSuccess) e = cudaMalloc(&dr, sizeof(double) * count);
  if (e == cudaSuccess) e = cudaMalloc(&ds, sizeof(int) * count);
  if (e == cudaSuccess) e = cudaMemcpy(dA, A, sizeof(double) * (size_t)count * n * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    k_spectral_batch<<<(unsigned)((count + 63) / 64), 64>>>(dA, n, count, dr, ds);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(rho, dr, sizeof(double) * count, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(status, ds, sizeof(int) * count, cudaMemcpyDeviceToHost);
  cudaFree(dA);
  cudaFree(dr);
  cudaFree(ds);
  if (e != cudaSuccess) {
    g_last_err = std::string("CUDA error: ") + cudaGetErrorString(e);
    return CISDC_E_CUDA;
  }
  return CISDC_OK;
}

const char* cisdc_gpu_kernel_class_name(int cls) {
  return (cls >= 0 && cls < kNumKernelClasses) ? kClassNames[cls] : "?";
}

double cisdc_gpu_device_time_ms(cisdc_gpu_ctx* ctx, int reset) {
  if (!ctx) return 0.0;
  const double t = ctx->device_ms;
  if (reset) ctx->device_ms = 0.0;
  return t;
}

int cisdc_gpu_fp64_peak(double* tflops_dfma, double* tflops_dmul_dadd) {
  cisdc_gpu_ctx* ctx = nullptr;  // for the CU() macro's error path
  int dev = 0, sms = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out = nullptr;
  CU(cudaMalloc(&out, sizeof(double)));
  cudaEvent_t a, b;
  CU(cudaEventCreate(&a));
  CU(cudaEventCreate(&b));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  const double ops = (double)blocks * threads * iters * 8;  // instructions (chains x iterations)
  for (int variant = 0; variant < 2; ++variant) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CU(cudaEventRecord(a));
      if (variant == 0) k_peak_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      else k_peak_dmul_dadd<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      CU(cudaEventRecord(b));
      CU(cudaEventSynchronize(b));
      float t = 0.f;
      CU(cudaEventElapsedTime(&t, a, b));
      best = std::min(best, t);
    }
    // DFMA: 2 flops per instruction; DMUL+DADD: 2 instructions per 2 flops
    const double tf = (variant == 0 ? 2.0 * ops : 2.0 * ops) / (best * 1e-3) / 1e12;
    if (variant == 0 && tflops_dfma) *tflops_dfma = tf;
    if (variant == 1 && tflops_dmul_dadd) *tflops_dmul_dadd = tf;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  return CISDC_OK;
}

int cisdc_gpu_set_trace(cisdc_gpu_ctx* ctx, int on) {
  if (!ctx) return CISDC_E_INVALID_ARGUMENT;
  ctx->trace_on = on != 0;
  return CISDC_OK;
}

int cisdc_gpu_last_trace(cisdc_gpu_ctx* ctx, cisdc_cell_trace* cells, int max_cells, int* n_cells, int* workers) {
  if (!ctx) return CISDC_E_INVALID_ARGUMENT;
  if (ctx->trace_pending) {
    const int M = ctx->trace_M, nu = ctx->trace_nu, n = 2 * M * nu;
    CU(cudaStreamSynchronize(ctx->s_main));
    CU(cudaStreamSynchronize(ctx->s_r));
    std::vector<double> t(2 * (size_t)n);
    const cudaEvent_t base = ctx->trace_ev[0];  // start of D(1,1): the sweep's first cell
    for (int id = 0; id < n; ++id)
      for (int e = 0; e < 2; ++e) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, base, ctx->trace_ev[2 * id + e]));
        t[2 * id + e] = (double)ms;
      }
    // one global order of all start/end events: by time, ends before starts on ties, then by id
    std::vector<int> ord(2 * (size_t)n);
    for (int i = 0; i < 2 * n; ++i) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](int a, int b) {
      if (t[a] != t[b]) return t[a] < t[b];
      if ((a & 1) != (b & 1)) return (a & 1) > (b & 1);
      return a < b;
    });
    ctx->trace.assign(n, cisdc_cell_trace{});
    for (int id = 0; id < n; ++id) {
      cisdc_cell_trace& c = ctx->trace[id];
      c.kind = id & 1;
      c.m = (id >> 1) % M + 1;
      c.ell = (id >> 1) / M + 1;
      c.worker = c.kind;
      c.start_ns = (long long)std::llround(t[2 * id] * 1e6);
      c.end_ns = (long long)std::llround(t[2 * id + 1] * 1e6);
    }
    for (int r = 0; r < 2 * n; ++r) {
      cisdc_cell_trace& c = ctx->trace[ord[r] >> 1];
      if (ord[r] & 1) c.seq_end = r;
      else c.seq_start = r;
    }
    ctx->trace_pending = false;
  }
  const int n = (int)ctx->trace.size();
  if (n_cells) *n_cells = n;
  if (workers) *workers = n ? ctx->trace_workers : 0;
  if (cells)
    for (int i = 0; i < n && i < max_cells; ++i) cells[i] = ctx->trace[i];
  return CISDC_OK;
}

// ---- SDC1 field snapshots (reaction_diffusion.cpp:230-259), host only
static thread_local std::string g_io_err;

const char* cisdc_io_last_error(void) { return g_io_err.c_str(); }

int cisdc_write_field_snapshot(const char* path, int n_x, double dx, const double* data, size_t n) {
  if (!path || n_x < 0 || (size_t)n_x != n || (n && !data)) {
    g_io_err = "write_field_snapshot: size mismatch";
    return CISDC_E_INVALID_ARGUMENT;
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) {
    g_io_err = std::string("write_field_snapshot: cannot open ") + path;
    return CISDC_E_IO;
  }
  const char magic[4] = {'S', 'D', 'C', '1'};
  const uint32_t nn = (uint32_t)n_x;
  bool ok = std::fwrite(magic, 1, 4, f) == 4 && std::fwrite(&nn, sizeof(nn), 1, f) == 1 &&
            std::fwrite(&dx, sizeof(dx), 1, f) == 1 && (n == 0 || std::fwrite(data, sizeof(double), n, f) == n);
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) {
    g_io_err = std::string("write_field_snapshot: write failed for ") + path;
    return CISDC_E_IO;
  }
  return CISDC_OK;
}

int cisdc_read_field_snapshot(const char* path, int* n_x, double* dx, double* data, size_t cap) {
  FILE* f = path ? std::fopen(path, "rb") : nullptr;
  if (!f) {
    g_io_err = std::string("read_field_snapshot: cannot open ") + (path ? path : "");
    return CISDC_E_IO;
  }
  char magic[4];
  if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "SDC1", 4) != 0) {
    std::fclose(f);
    g_io_err = std::string("read_field_snapshot: bad magic in ") + path;
    return CISDC_E_IO;
  }
  uint32_t nn = 0;
  double h = 0.0;
  bool ok = std::fread(&nn, sizeof(nn), 1, f) == 1 && std::fread(&h, sizeof(h), 1, f) == 1;
  std::vector<double> v;
  if (ok) {
    v.resize(nn);
    ok = nn == 0 || std::fread(v.data(), sizeof(double), nn, f) == nn;
  }
  std::fclose(f);
  if (!ok) {
    g_io_err = std::string("read_field_snapshot: truncated file ") + path;
    return CISDC_E_IO;
  }
  if (n_x) *n_x = (int)nn;
  if (dx) *dx = h;
  if (data) std::memcpy(data, v.data(), sizeof(double) * std::min<size_t>(cap, nn));
  return CISDC_OK;
}

}  // extern "C"
