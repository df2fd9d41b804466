/*
 * cisdc_gpu.h -- C-ABI of the B200-native MISDC / MISDCQ / CISDCQ ("PMISDC") sweep engine.
 *
 * Plain C: pointers, sizes and ints only, no C++ or CUDA types in any signature.
 * Every entry point below replaces one call of the reference's C++ sweep/integrator API
 * (paths relative to the reference repo root; see INTEGRATION.md for the binding):
 *
 *   cisdc_make_quadrature_tables  <- cisdc::make_quadrature_tables   proj/core/src/quadrature.cpp:147-162
 *   cisdc_gpu_create              <- constructing an OperatorSplitProblem + SweepState
 *                                    proj/core/include/cisdc/operator_split.hpp:36-54,
 *                                    proj/core/src/sweep_state.cpp:22-30
 *   cisdc_gpu_initialize          <- cisdc::SweepState::initialize     proj/core/src/sweep_state.cpp:32-44
 *   cisdc_gpu_set_nodes           <- cisdc::SweepState::set_node_values proj/core/src/sweep_state.cpp:46-58
 *   cisdc_gpu_sweep               <- cisdc::run_sweep (misdc/misdcq/cisdcq dispatch)
 *                                    proj/core/src/integrators.cpp:290-299; with
 *                                    workers > 0 the CISDCQ DAG runs as in cisdc::execute_pipelined
 *                                    proj/core/src/pipeline.cpp:171-320
 *   cisdc_gpu_increment           <- cisdc::increment_norm(phi[M], prev) proj/core/src/sweep_state.cpp:60-66
 *   cisdc_gpu_get_field           <- reading SweepState::{phi,fa,fd,fr,phi_ad}[m]
 *   cisdc_gpu_integrate           <- cisdc::integrate                  proj/core/src/integrators.cpp:301-333
 *   cisdc_gpu_eval / cisdc_gpu_solve
 *                                 <- OperatorSplitProblem::eval_* / solve_* (one stage on one field)
 *   cisdc_gpu_last_trace          <- the ScheduleTrace returned by cisdc::execute_pipelined
 *                                    proj/core/include/cisdc/pipeline.hpp:72-93
 *   cisdc_write_field_snapshot / cisdc_read_field_snapshot
 *                                 <- cisdc::write_field_snapshot / read_field_snapshot
 *                                    proj/core/src/problems/reaction_diffusion.cpp:230-259
 *
 * Error behaviour mirrors the reference's exception taxonomy (proj/core/include/cisdc/errors.hpp:24-45):
 * every function returns a cisdc_status; the message (stage, node, first failing cell) is
 * available from cisdc_gpu_last_error().  Calls are synchronous at return, like run_sweep.
 * One host thread per context (a context is not thread-safe, like SweepState).
 */
#ifndef CISDC_GPU_H_
#define CISDC_GPU_H_

#ifndef __CUDACC_RTC__
#include <stddef.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: exception types of proj/core/include/cisdc/errors.hpp + std::invalid_argument */
typedef enum {
  CISDC_OK = 0,
  CISDC_E_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  CISDC_E_FACTORIZATION = 2,    /* cisdc::FactorizationError */
  CISDC_E_SOLVE = 3,            /* cisdc::SolveError */
  CISDC_E_NUMERIC = 4,          /* cisdc::NumericError (Newton / multigrid cap) */
  CISDC_E_CAPABILITY = 5,       /* cisdc::CapabilityError */
  CISDC_E_CUDA = 6,             /* CUDA runtime failure, out of memory */
  CISDC_E_IO = 7                /* std::runtime_error of the snapshot / trace file IO */
} cisdc_status;

/* cisdc::Scheme, same order (proj/core/include/cisdc/integrators.hpp:30) */
enum { CISDC_SCHEME_MISDC = 0, CISDC_SCHEME_MISDCQ = 1, CISDC_SCHEME_CISDCQ = 2, CISDC_SCHEME_IMEXQ = 3 };
/* cisdc::EulerConvention (proj/core/include/cisdc/quadrature.hpp:42) */
enum { CISDC_EULER_LITERAL = 0, CISDC_EULER_CUMULATIVE = 1 };

/* problem kinds */
enum {
  CISDC_PROBLEM_PERIODIC_ADR = 0,   /* periodic 1-D/2-D/3-D advection-diffusion-reaction, S species */
  CISDC_PROBLEM_REFERENCE_RD = 1,   /* the reference's own 1-D Dirichlet PDE on [0,20]
                                       (proj/core/include/cisdc/problems/reaction_diffusion.hpp:28-99) */
  CISDC_PROBLEM_LINEAR_SCALAR = 2   /* phi' = (a+d+r) phi (proj/core/include/cisdc/problems/linear.hpp:31-51);
                                       oracle only (known-answer tests), rejected by cisdc_gpu_create */
};
enum {
  CISDC_REACTION_NONE = 0,
  CISDC_REACTION_LINEAR_DECAY = 1,  /* R = -lambda * phi                      (S = 1) */
  CISDC_REACTION_BISTABLE = 2,      /* R = lambda * phi (1 - phi) (phi - theta) (S = 1) */
  CISDC_REACTION_MASS_ACTION = 3    /* network of <=2-reactant/<=2-product mass-action reactions */
};
/* DIRECT: 1-D periodic exact circulant factorisation (blocked scan); MULTIGRID: 2-D/3-D;
   BANDED_ORACLE: cyclic banded LU (reference banded_solve semantics), CPU oracle only (cross-check) */
enum { CISDC_DIFFUSION_DIRECT = 0, CISDC_DIFFUSION_MULTIGRID = 1, CISDC_DIFFUSION_BANDED_ORACLE = 2 };
enum { CISDC_FIELD_PHI = 0, CISDC_FIELD_FA = 1, CISDC_FIELD_FD = 2, CISDC_FIELD_FR = 3, CISDC_FIELD_PHI_AD = 4 };
enum { CISDC_STAGE_ADVECTION = 0, CISDC_STAGE_DIFFUSION = 1, CISDC_STAGE_REACTION = 2, CISDC_STAGE_COUPLED = 3 };

#define CISDC_MAX_M 8
#define CISDC_MAX_SPECIES 16
#define CISDC_MAX_REACTIONS 64

/*
 * Problem description.  Field layout (host and device): species-major, x fastest:
 *   phi[((s * n[2] + k) * n[1] + j) * n[0] + i],   dimension = S * n[0] * n[1] * n[2].
 *
 * Advection F_A = -div(u phi) in finite-volume flux form with 4th-order face values
 * phi_{i+1/2} = (7(phi_i + phi_{i+1}) - (phi_{i-1} + phi_{i+2}))/12.  The face velocity of
 * component a at the + face of cell (i,j,k) is the separable product
 *   u_a = (vel[a][0][i] * vel[a][1][j]) * vel[a][2][k]
 * (a NULL table counts as 1.0; if all three tables of component a are NULL there is no
 * advection along a).  Tables are filled by the caller so CPU and GPU share the same bits.
 * Diffusion F_D = d_s * Lap4 (the reference's (-1,16,-30,16,-1)/(12 h^2) stencil per axis).
 */
typedef struct cisdc_problem_desc {
  int kind;                 /* CISDC_PROBLEM_* */
  int ndim;                 /* 1..3 */
  int n[3];                 /* cells per axis; unused axes = 1 */
  int nspecies;             /* S */
  double h[3];              /* cell widths */
  const double* vel[3][3];  /* separable face-velocity tables (see above) */
  const double* diffusivity;/* [S] */
  int reaction_kind;        /* CISDC_REACTION_* */
  double lambda, theta;     /* LINEAR_DECAY / BISTABLE parameters */
  int n_reactions;          /* MASS_ACTION: reactions r = 0..n_reactions-1 */
  const int* reactants;     /* [2*n_reactions], species index or -1 */
  const int* products;      /* [2*n_reactions], species index or -1 */
  const double* rate_constants; /* [n_reactions] */
  double newton_tol;        /* reference default 1e-14 (proj/core/include/cisdc/linalg.hpp:97-100) */
  int newton_max_iter;      /* reference default 50 */
  int diffusion_solver;     /* CISDC_DIFFUSION_DIRECT (1-D) or CISDC_DIFFUSION_MULTIGRID (2-D/3-D) */
  double mg_tol;            /* stop when ||b - A x||_inf <= mg_tol * ||b||_inf (per species) */
  int mg_max_cycles, mg_pre, mg_post, mg_coarse_sweeps, mg_min_coarse;
  double mg_omega;          /* weighted-Jacobi damping */
  /* CISDC_PROBLEM_REFERENCE_RD / LINEAR_SCALAR coefficients (a, d, r); n[0] = n_x for RD */
  double ref_a, ref_d, ref_r;
  /* Coupled stage of the periodic ADR class (OperatorSplitProblem::solve_coupled,
   * operator_split.hpp:49-53; imexq_sweep's stage solve, integrators.cpp:166):
   *   phi - coef (F_D(phi) + F_R(phi)) = rhs
   * as the fixed point of the alternating stage solves (the nested iteration of cisdcq_cells at one
   * node, integrators.cpp:195-258, run to convergence):
   *   y_0 = rhs;  z = solve_diffusion(coef, rhs + coef F_R(y_k));  y_{k+1} = solve_reaction(coef, rhs + coef F_D(z))
   * until max|y_{k+1} - y_k| <= coupled_tol * max|y_{k+1}|; SolveError after coupled_max_iter
   * iterations.  coupled_max_iter == 0: no coupled solve (has_coupled_solve() == false, imexq_sweep
   * raises CapabilityError, as for the reference's ReactionDiffusionProblem). */
  double coupled_tol;
  int coupled_max_iter;
} cisdc_problem_desc;

/* cisdc::QuadratureTables, row-major, M <= CISDC_MAX_M (proj/core/include/cisdc/quadrature.hpp:47-60) */
typedef struct cisdc_tables {
  int M;
  int convention;
  double tau[CISDC_MAX_M + 1];
  double dtau[CISDC_MAX_M];
  double Q[CISDC_MAX_M * (CISDC_MAX_M + 1)];   /* M x (M+1), stride M+1 */
  double q[CISDC_MAX_M];
  double Qt[CISDC_MAX_M * CISDC_MAX_M];        /* M x M, stride M */
  double S[CISDC_MAX_M * (CISDC_MAX_M + 1)];   /* M x (M+1), stride M+1 */
  double QtI[CISDC_MAX_M * CISDC_MAX_M];       /* M x M, stride M */
  double QtE[CISDC_MAX_M * CISDC_MAX_M];       /* M x M, stride M */
} cisdc_tables;

/* cisdc::SolveCounters (operator_split.hpp:57-68) plus the Newton/multigrid work counts */
typedef struct cisdc_counters {
  long long diffusion, reaction, coupled;
  long long newton_iterations;  /* residual evaluations summed over cells and reaction solves */
  long long mg_cycles;          /* V-cycles summed over species and diffusion solves */
} cisdc_counters;

/* cisdc::IntegrateOptions (integrators.hpp:64-73) */
typedef struct cisdc_integrate_options {
  int scheme;
  double dt;
  int n_steps;
  int M;
  int n_sweeps;
  int nu;
  int has_stop_tol;
  double stop_tol;
  int convention;
  int workers;  /* CISDCQ only: 0 = serial cell order (cisdcq_sweep), >0 = concurrent D/R streams
                   (execute_pipelined semantics; results are bitwise identical) */
} cisdc_integrate_options;

/* cisdc::SweepReport (sweep_state.hpp:56-60); increments are written separately */
typedef struct cisdc_step_report {
  int sweeps;
  cisdc_counters counters;
} cisdc_step_report;

#ifndef __CUDACC_RTC__ /* device-side runtime compilation sees only the types above */
typedef struct cisdc_gpu_ctx cisdc_gpu_ctx;

int cisdc_make_quadrature_tables(int M, int convention, cisdc_tables* out);

int cisdc_gpu_create(const cisdc_problem_desc* desc, const cisdc_tables* tables, cisdc_gpu_ctx** out);
void cisdc_gpu_destroy(cisdc_gpu_ctx* ctx);
const char* cisdc_gpu_last_error(const cisdc_gpu_ctx* ctx);
size_t cisdc_gpu_dimension(const cisdc_gpu_ctx* ctx);

/* host-pointer state upload; *_device variants take device pointers (no PCIe copy) */
int cisdc_gpu_initialize(cisdc_gpu_ctx* ctx, const double* phi0, size_t n);
int cisdc_gpu_initialize_device(cisdc_gpu_ctx* ctx, const double* d_phi0, size_t n);
int cisdc_gpu_set_nodes(cisdc_gpu_ctx* ctx, const double* values /* (M+1) x n */, size_t n);

int cisdc_gpu_sweep(cisdc_gpu_ctx* ctx, int scheme, double dt, int nu, int workers, cisdc_counters* inout);
int cisdc_gpu_increment(cisdc_gpu_ctx* ctx, double* out);
int cisdc_gpu_get_field(cisdc_gpu_ctx* ctx, int which, int node, double* host, size_t n);
int cisdc_gpu_get_field_device(cisdc_gpu_ctx* ctx, int which, int node, double* d_out, size_t n);

/* one stage on one field (OperatorSplitProblem::eval_* / solve_*), host pointers */
int cisdc_gpu_eval(cisdc_gpu_ctx* ctx, int stage, const double* phi, double* out, size_t n);
int cisdc_gpu_solve(cisdc_gpu_ctx* ctx, int stage, double coef, const double* rhs, double* out, size_t n,
                    cisdc_counters* inout);

/* cisdc::integrate: phi0 / final_state host buffers of n doubles; reports[n_steps];
   increments[n_steps * n_sweeps] (unused tail entries when stop_tol ends a step early are 0) */
int cisdc_gpu_integrate(cisdc_gpu_ctx* ctx, const double* phi0, size_t n, const cisdc_integrate_options* opt,
                        double* final_state, cisdc_step_report* reports, double* increments);
/* same with device-resident phi0 / final_state (no host<->device copies of fields) */
int cisdc_gpu_integrate_device(cisdc_gpu_ctx* ctx, const double* d_phi0, size_t n,
                               const cisdc_integrate_options* opt, double* d_final_state,
                               cisdc_step_report* reports, double* increments);

/* ---- measurement (no reference counterpart; used by bench.py) ----
 * Live per-kernel-class CUDA-event timing on the launching stream (off by default), the
 * algorithmic (compulsory) bytes each class moved and its launch count, accumulated since the
 * last reset; the device time of sweep/integrate calls (events on the context's stream). */
int cisdc_gpu_set_timing(cisdc_gpu_ctx* ctx, int on);
int cisdc_gpu_kernel_times(cisdc_gpu_ctx* ctx, double* ms, double* bytes, long long* launches, int max_classes,
                           int reset);
const char* cisdc_gpu_kernel_class_name(int cls);
double cisdc_gpu_device_time_ms(cisdc_gpu_ctx* ctx, int reset);
/* kernel launches issued since creation (or the last kernel_times reset) */
long long cisdc_gpu_launch_count(const cisdc_gpu_ctx* ctx);
/* cell Newton solves since creation that ended at the residual test |f| <= tol (their last trip
   built no Jacobian); with newton_iterations this splits the trips for the flop model (bench.py) */
long long cisdc_gpu_newton_residual_exits(const cisdc_gpu_ctx* ctx);
/* ---- batched iteration-matrix scans (analysis.hpp:72-95; analysis.cpp:215-293) ----------------
   cisdc::spectral_radius_scan on the GPU, one thread per point: for every scheme, every nu of
   nu_list (CISDCQ only; 1 otherwise) and every r of r_grid, in that order, the affine iteration
   matrix G of one sweep on the linear model (a, d, r) -- d = r / 2 (d_rule 0, DRule::half_of_r) or
   fixed_d (d_rule 1) -- and its spectral radius.  A point whose stage factor vanishes, whose G is
   not finite, or whose QR iteration reaches its cap gets ok = 0 (gamma 0), as the reference records
   it.  G_out (optional): the n_points M x M matrices, row-major.  Empty schemes / r_grid ->
   CISDC_E_INVALID_ARGUMENT with the reference's message (cisdc_last_error). */
typedef struct cisdc_scan_point {
  int scheme, M, nu;
  double a, d, r, dt;
  double gamma;
  int ok;
} cisdc_scan_point;
int cisdc_gpu_spectral_radius_scan(const int* schemes, int n_schemes, const int* nu_list, int n_nu,
                                   const double* r_grid, int n_r, int d_rule, double fixed_d, double a, double dt,
                                   int M, int convention, cisdc_scan_point* out, size_t cap, size_t* n_out,
                                   double* G_out);
/* cisdc::spectral_radius (linalg.cpp:197-332) of `count` n x n matrices (row-major, n <= 8), one GPU
   thread each: rho[i], status[i] = 0 ok, 1 non-finite entry (std::invalid_argument), 2 QR iteration
   cap (cisdc::NumericError) */
int cisdc_gpu_spectral_radius_batch(const double* A, int n, int count, double* rho, int* status);
/* cisdc::log_r_grid (analysis.cpp:255-266): -10^e for n + 1 exponents from lo_exp to hi_exp,
   n = round((hi - lo) * points_per_decade); returns the count (or -1: points_per_decade < 1) */
int cisdc_log_r_grid(double lo_exp, double hi_exp, int points_per_decade, double* out, size_t cap);
const char* cisdc_last_error(void);

/* FP64 pipe peak on the current device: DFMA chains and DMUL+DADD chains, TFLOP/s */
int cisdc_gpu_fp64_peak(double* tflops_dfma, double* tflops_dmul_dadd);
/* ---- PMISDC schedule trace (cisdc::CellTrace / ScheduleTrace, pipeline.hpp:72-84) ----
   With tracing on, every CISDCQ sweep run with workers > 0 records GPU timestamps at the start and
   end of each DAG cell on its stream (worker 0 = diffusion stream, 1 = reaction stream).
   cisdc_gpu_last_trace returns the cells of the last such sweep in cell-id order
   (TaskGraph::cell_id); times are ns from the sweep's first cell, seq_* a single global order of
   the start/end events (ends before starts on equal times). */
typedef struct {
  int kind; /* 0 = diffusion (D), 1 = reaction (R) */
  int m;
  int ell;
  int worker;
  long long start_ns, end_ns;
  long long seq_start, seq_end;
} cisdc_cell_trace;
int cisdc_gpu_set_trace(cisdc_gpu_ctx* ctx, int on);
/* copies min(n, max_cells) cells; *n_cells = n, *workers = streams used (0 if no traced sweep) */
int cisdc_gpu_last_trace(cisdc_gpu_ctx* ctx, cisdc_cell_trace* cells, int max_cells, int* n_cells, int* workers);

/* ---- field snapshots (host only; reaction_diffusion.hpp:101-112) ----
   File: magic "SDC1", u32 n_x, f64 dx, then n_x doubles, little-endian.  write: n must equal n_x
   (CISDC_E_INVALID_ARGUMENT, "size mismatch"), IO failure -> CISDC_E_IO.  read: header into
   *n_x, *dx, then min(n_x, cap) values into data (data may be NULL to query the size); bad magic or
   a truncated file -> CISDC_E_IO.  cisdc_io_last_error(): the message of the calling thread's last
   failed snapshot call, worded as the reference's exceptions. */
int cisdc_write_field_snapshot(const char* path, int n_x, double dx, const double* data, size_t n);
int cisdc_read_field_snapshot(const char* path, int* n_x, double* dx, double* data, size_t cap);
const char* cisdc_io_last_error(void);

/* Generate and NVRTC-compile the network-specialised Newton kernels of a mass-action problem for
   sm_100a without loading them (no GPU needed); the compiler log goes to log[cap]. */
int cisdc_rtc_compile_check(const cisdc_problem_desc* desc, char* log, size_t cap);

#endif /* __CUDACC_RTC__ */

#ifdef __cplusplus
}
#endif

#endif /* CISDC_GPU_H_ */
