/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference's MISDC / MISDCQ / CISDCQ / IMEXQ sweep path
 * (reference: /root/reference/proj/core, cited file:line per function in the .c files).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load it, and only as the checker or the CPU baseline -- never as the product path.
 *
 * Pinning: the quadrature tables, linear algebra, integrator algebra and the reference's own
 * 1-D Dirichlet problem are checked bit-for-bit against the UNMODIFIED reference compiled from
 * /root/reference into oracle/_ref (oracle/Makefile, tests/test_oracle_vs_ref.py), and against
 * the reference's known-answer tests (tests/test_oracle_known_answers.py) and the golden
 * fixtures in tests/golden/.  The periodic multi-D / multi-species problem class (configs 1-5)
 * has no reference implementation; it is new code following reaction_diffusion.cpp's
 * structure and is driven by the unmodified reference integrators in oracle/_ref, so for those
 * configs only the problem class is unpinned.
 */
#ifndef CISDC_ORACLE_H_
#define CISDC_ORACLE_H_

#include <stddef.h>

#include "../include/cisdc_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- quadrature (quadrature.cpp) ---- */
int co_make_tables(int M, int convention, cisdc_tables* out);

/* ---- linear algebra (linalg.cpp) ---- */
/* band[(j - i + kl) * n + i] holds A(i,j) (BandedMatrix storage, linalg.hpp:63-85) */
int co_banded_solve(int n, int kl, int ku, const double* band, const double* b, double* x, char* err);
int co_lu_factor_dense(int n, double* a /* row-major, in/out */, int* perm, int pivoting, char* err);
void co_lu_solve(int n, const double* lu, const int* perm, const double* b, double* x);

/* ---- problems (operator_split.hpp contract) ---- */
typedef struct co_problem co_problem;
int co_problem_create(const cisdc_problem_desc* desc, co_problem** out, char* err /* >= 512 */);
void co_problem_destroy(co_problem* p);
size_t co_problem_dim(const co_problem* p);
int co_problem_has_coupled(const co_problem* p);
/* stage: CISDC_STAGE_* */
int co_eval(co_problem* p, int stage, const double* phi, double* out);
/* stage: CISDC_STAGE_DIFFUSION / CISDC_STAGE_REACTION, or 3 = coupled */
int co_solve(co_problem* p, int stage, double coef, const double* rhs, double* out, cisdc_counters* c);
const char* co_problem_error(const co_problem* p);

/* ---- sweep state (sweep_state.cpp) ---- */
typedef struct co_state co_state;
co_state* co_state_create(int M, size_t dim);
void co_state_destroy(co_state* s);
int co_state_initialize(co_state* s, co_problem* p, const double* phi0);
int co_state_set_nodes(co_state* s, co_problem* p, const double* values /* (M+1) x dim */);
double* co_state_field(co_state* s, int which, int node);
double co_increment_norm(const double* a, const double* b, size_t n);

/* ---- sweeps / driver (integrators.cpp) ---- */
int co_run_sweep(int scheme, co_state* s, const cisdc_tables* tb, co_problem* p, double dt, int nu,
                 cisdc_counters* c);
int co_integrate(co_problem* p, const double* phi0, const cisdc_integrate_options* opt, double* final_state,
                 cisdc_step_report* reports, double* increments, char* err /* >= 1024 */);

#ifdef __cplusplus
}
#endif

#endif /* CISDC_ORACLE_H_ */
