// Shared device-side definitions of the sweep engine.
//
// Arithmetic contract: every kernel evaluates the reference's expressions in the reference's
// operand order with no FMA contraction (the library is built with -fmad=false), so pointwise
// results are bit-identical to the CPU oracle / the reference's no-FMA x86-64 build.
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <set>
#include <tuple>
#endif

#include "../../include/cisdc_gpu.h"

namespace cisdc_b200 {

constexpr int kMaxM = CISDC_MAX_M;
constexpr int kMaxS = CISDC_MAX_SPECIES;
constexpr int kMaxR = CISDC_MAX_REACTIONS;

// Device status word, one per context (written by kernels, read once per step).
// fail_key orders failures the way the reference meets them: the host gives every launch that can
// fail a tag in enqueue (= the reference's serial) order, and a failing kernel records
//   key = tag << 35 | code << 32 | cell   (atomicMin)
// so the earliest failing stage wins and, within it, the smallest cell (species for multigrid).
struct DevStatus {
  unsigned long long fail_key;        // ~0ull if nothing failed
  unsigned long long newton_trips;    // Newton residual evaluations (atomicAdd)
  unsigned long long mg_cycles;       // multigrid V-cycles
  unsigned long long newton_res_exits;  // cell solves that ended at the residual test (atomicAdd)
  unsigned long long loop_kernels;      // kernels run by device-looped multigrid cycles (multigrid.cuh)
};

#ifdef __CUDACC__
__device__ __forceinline__ void record_failure(DevStatus* st, unsigned tag, int code, unsigned long long cell) {
  atomicMin(&st->fail_key, ((unsigned long long)tag << 35) | ((unsigned long long)(code & 7) << 32) |
                               (cell & 0xffffffffull));
}
#endif

// Grid geometry of one field (species-major, x fastest).
struct Geom {
  int nx, ny, nz;  // cells per axis (1 for unused axes)
  int ndim;
  int S;
  long long ncell;  // nx * ny * nz
  long long n;      // S * ncell
};

// Separable face-velocity tables and stencil coefficients (problem constants).
struct Ops {
  const double* vel[3][3];  // nullptr = 1.0
  int adv[3];               // axis a advects
  double cadv[3];           // 1 / (12 h_a)
  double cdiff[kMaxS][3];   // d_s / (12 h_a^2)
  // uniform face velocities: every table of every advecting axis is constant (or absent), and
  // ucon[a] = (T_a0 T_a1) T_a2 -- the per-face product face_u forms, same bits
  int vconst;
  double ucon[3];
  // reference Dirichlet problem (CISDC_PROBLEM_REFERENCE_RD)
  int ref_rd;
  double rd_cadv, rd_cdiff, rd_w[2][5];
  // set (sticky until the next initialize) when an F_A evaluation stores a value with |v| >= 2^1022,
  // an Inf or a NaN: k_rhs then evaluates cE*(A - Ap) even where cE == 0 (see k_rhs)
  int* wild;
};

// |v| >= 2^1022, Inf or NaN (exponent field >= 2045): a difference of two values below this bound
// is finite, so 0.0 * (A - Ap) is a signed zero
__device__ __forceinline__ unsigned wild_bits(double v) {
  return (unsigned)(((unsigned)__double2hiint(v) & 0x7ff00000u) >= (2045u << 20));
}
__device__ __forceinline__ void flag_wild(int* flag, unsigned w) {
  if (w && flag) atomicOr(flag, 1);
}

// Kernel classes for the live per-class CUDA-event timing (cisdc_gpu_kernel_times).
enum KernelClass {
  kKQuad = 0,      // k_quad_base
  kKRhs = 1,       // k_rhs
  kKSolve1d = 2,   // k_solve1d_periodic / k_rd_banded_solve
  kKMgSmooth = 3,  // k_mg_smooth
  kKMgRestrict = 4,
  kKMgProlong = 5,
  kKMgNorm = 6,    // k_mg_absmax / k_mg_resmax / k_mg_update
  kKReact = 7,     // k_react (Newton)
  kKEvalAD = 8,    // k_eval_ad
  kKEvalR = 9,     // k_eval_r
  kKIncr = 10,     // k_incr_*
  kKReactRhs = 11,  // k_react_next (Newton of R(m, l) + the right-hand side of D(m+1, l))
  kNumKernelClasses = 12
};

#ifndef __CUDACC_RTC__
// Called around every kernel launch (timing is a no-op unless enabled).
struct LaunchHook {
  virtual void before(int cls, cudaStream_t s) = 0;
  virtual void after(int cls, cudaStream_t s, double bytes) = 0;
  // bytes known only after the fact (multigrid: per-species masking decided on the device)
  virtual void add_bytes(int, double) {}
  // kernels launched through a CUDA graph replay (counted, not individually timed)
  virtual void add_launches(long long) {}
  // per-launch timing active (graph replays are then not used, so every launch is timed)
  virtual bool timing() const { return false; }
  virtual ~LaunchHook() = default;
};
#endif

__device__ __forceinline__ int wrapi(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

__device__ __forceinline__ double face_u(const Ops& o, int a, int i, int j, int k) {
  const double t0 = o.vel[a][0] ? __ldg(o.vel[a][0] + i) : 1.0;
  const double t1 = o.vel[a][1] ? __ldg(o.vel[a][1] + j) : 1.0;
  const double t2 = o.vel[a][2] ? __ldg(o.vel[a][2] + k) : 1.0;
  return (t0 * t1) * t2;
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr), __double_as_longlong(v));
}

#ifndef __CUDACC_RTC__
inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// cudaFuncSetAttribute once per (kernel, attribute, value, device): CUDA applies function
// attributes per device, so a second context on another device sets them again.
inline cudaError_t func_attr_once(const void* fn, cudaFuncAttribute attr, int value) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int, int>> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
  const auto key = std::make_tuple(fn, (int)attr, value, dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(key)) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, attr, value);
  if (e == cudaSuccess) done.insert(key);
  return e;
}
template <class F>
inline cudaError_t func_attr_once(F* fn, cudaFuncAttribute attr, int value) {
  return func_attr_once(reinterpret_cast<const void*>(fn), attr, value);
}
#endif

}  // namespace cisdc_b200
