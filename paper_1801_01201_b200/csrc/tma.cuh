// Tensor-memory-accelerator (TMA) staging for the 3-D pair walker (stencil3d.cuh walk_pair): the
// Blackwell-native form of the multigrid level-0 sweep / residual check on tile-aligned grids.
//
// walk_pair stages every plane's 68 x 12 halo tile with per-thread 16-byte cp.async: 2 LDGSTS per
// thread per plane plus their address arithmetic and a wait_group, about a third of the sweep
// kernel's instructions (profiles/r2, k_mg3_pair SASS: the residual-check variants are
// issue-bound).  Here one elected thread moves a plane with five cp.async.bulk.tensor boxes of a
// 3-D tensor map over (x, y, z * S) -- interior 64 x 8, top and bottom halo rows 64 x 2, left and
// right halo columns 2 x 8 (a star stencil needs no corners) -- each box at its periodically
// wrapped origin, so no box ever crosses a seam and nothing is zero-filled.  The right-hand side
// rides in the same transaction (one 64 x 8 box).  Completion is an mbarrier per ring slot
// (arrive.expect_tx by the producer, complete_tx by the copies, try_wait.parity by all threads);
// slot reuse (WAR) is fenced by the walker's per-plane __syncthreads (multigrid sweeps) or by a second
// "empty" mbarrier per slot (F_A/F_D: FREE, below).
//
// Shared-memory plane slot (doubles; every region 128-byte aligned, as the bulk tensor copy needs;
// rows -2 .. 9 are contiguous at pitch 64, so a thread's five y taps and its centre are one base
// register plus compile-time offsets):
//   [0, 128)    rows -2, -1, pitch 64
//   [128, 640)  interior rows 0..7, pitch 64
//   [640, 768)  rows 8, 9, pitch 64
//   [768, 784)  columns -2, -1 of rows 0..7, pitch 2
//   [784, 800)  columns 64, 65 of rows 0..7, pitch 2
// A thread's taps are the same values walk_pair reads (same operand order in the body): only the
// shared-memory address of each tap changes, so the results are bit-identical.
//
// Requirements (else the launcher keeps walk_pair): nx % 64 == 0, ny % 8 == 0, 16-byte aligned
// fields; tensor maps from the driver's cuTensorMapEncodeTiled through the runtime's entry-point
// query (no libcuda link).
#pragma once

#include <cuda.h>

#include "stencil3d.cuh"

namespace cisdc_b200 {

constexpr int kTmaTop = 0, kTmaMain = 128, kTmaBot = 640, kTmaLeft = 768, kTmaRight = 784;
constexpr int kTmaSlot = 800;                               // doubles per plane slot
constexpr unsigned kTmaPlaneBytes = kTmaSlot * 8u;          // 6400 bytes of x per plane
constexpr unsigned kTmaAuxBytes = kPTX * kTY * 8u;          // 4096 bytes of rhs per plane
constexpr int kTmaRing = 6;
constexpr size_t kTmaSmem = (size_t)kTmaRing * (kTmaSlot + kPTX * kTY) * sizeof(double) + 128 + 128;
constexpr size_t kTmaEvalSmem = (size_t)kTmaRing * kTmaSlot * sizeof(double) + 128 + 128;  // no rhs ring

// The tensor maps one walk needs: x with the three box shapes, and the rhs (interior box).
struct TmaMaps {
  CUtensorMap x_main;  // box {64, 8, 1}
  CUtensorMap x_rows;  // box {64, 2, 1}
  CUtensorMap x_cols;  // box {2, 8, 1}
  CUtensorMap b_main;  // box {64, 8, 1}
};

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// one lane of a converged warp (warp-uniform branch around it): straight-line UTMALDG issue
__device__ __forceinline__ bool elect_one() {
  unsigned pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tma_load3(unsigned dst, const CUtensorMap* map, int x, int y, int z, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}

// 128-bit shared load at a 32-bit shared-space address plus a compile-time byte offset (LDS.128 with
// an immediate: a pointer rounded up through an integer loses its address space and compiles to
// generic loads with 64-bit address arithmetic).  volatile: stays behind the mbarrier wait.
template <int IMM>
__device__ __forceinline__ void lds2(unsigned addr, double& a, double& b) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(a), "=d"(b) : "r"(addr), "n"(IMM));
}

// walk_pair's contract (stencil3d.cuh) on TMA-staged planes; HAS_AUX stages the rhs (z-folded field
// index s * nz + k).  plane(k) runs once per plane before the body, as in walk_pair.
//
// The plane loop is unrolled by the ring size (6) and the z taps sit in a 6-deep register queue, so
// inside the unrolled body every ring slot, mbarrier and phase parity is a compile-time constant:
// plane k0 - 2 + j lives in slot j % 6 and is that slot's (j / 6)-th fill.  Staging distance 4:
// the step of plane k waits for plane k + 2 and stages plane k + 4 into the slot of plane k - 2.
//
// FREE: no block barrier in the plane loop.  Slot reuse is then gated by a second mbarrier per slot
// ("empty", one arrival per warp after the warp's last read of the slot: its x/y taps and rhs pair of
// that plane; the two z-tap-only planes below the chunk are released after the prologue); the staging
// lane waits for the empty phase of the slot it refills -- the plane two steps back, so warps drift up
// to two planes apart and their FP64 bursts stop being phase-locked.  Measured on C5 (r3a, same box,
// alternating runs): F_A/F_D 103.0 -> 96.1 ms per step (on), multigrid sweeps 125.8 -> 133.8 (off).
template <bool HAS_AUX, bool FREE, class PlaneFn, class Body>
__device__ __forceinline__ void walk_pair_tma(const TmaMaps& maps, int nx, int ny, int nz, const ZChunk& z,
                                              double* smem, PlaneFn plane, Body body) {
  constexpr bool free_run = FREE;
  static_assert(kTmaRing == 6, "the unrolled walker is written for a 6-slot ring");
  constexpr int kSlotB = kTmaSlot * 8, kAuxB = kPTX * kTY * 8;
  const int i0 = blockIdx.x * kPTX, j0 = blockIdx.y * kTY;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int t = ty * kTX + tx;
  const unsigned pl = (unsigned)nx * (unsigned)ny;
  const unsigned col = (unsigned)(j0 + ty) * (unsigned)nx + (unsigned)(i0 + 2 * tx);
  // ring: 6 x-slots, then 6 rhs slots, then the mbarriers (base rounded up to the 128 bytes the bulk
  // tensor copies need; kTmaSmem has the slack)
  const unsigned xs = ((unsigned)__cvta_generic_to_shared(smem) + 127u) & ~127u;
  const unsigned as = xs + kTmaRing * kSlotB;
  const unsigned bars = as + (HAS_AUX ? kTmaRing * kAuxB : 0);  // no rhs ring without a rhs
  const int zoff = z.s * nz;
  const int jt = j0 - 2 < 0 ? j0 - 2 + ny : j0 - 2;   // rows -2, -1 (wrapped)
  const int jb = j0 + kTY >= ny ? j0 + kTY - ny : j0 + kTY;  // rows 8, 9 (wrapped)
  const int il = i0 - 2 < 0 ? i0 - 2 + nx : i0 - 2;   // columns -2, -1
  const int ir = i0 + kPTX >= nx ? i0 + kPTX - nx : i0 + kPTX;  // columns 64, 65
  if (t == 0) {
#pragma unroll
    for (int r = 0; r < kTmaRing; ++r) {
      mbar_init(bars + 8u * r, 1);
      mbar_init(bars + 8u * (kTmaRing + r), kTY);  // "empty": one arrival per warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // stage plane kk into slot R (compile-time)
  // refill: the slot held an earlier plane; in free-run mode wait until every warp released it
  // (completion `empty_par` of the slot's empty barrier)
  auto issue = [&](auto slot, int kk, bool refill = false, unsigned empty_par = 0u) {
    constexpr int R = decltype(slot)::value;
    if (ty != 0 || kk > z.k1 + 1) return;  // warp 0 stages (a warp is one tile row)
    if (!elect_one()) return;
    const unsigned bar = bars + 8u * R;
    if (free_run && refill) mbar_wait(bars + 8u * (kTmaRing + R), empty_par);
    const bool aux = HAS_AUX && kk >= z.k0 && kk < z.k1;
    mbar_expect_tx(bar, kTmaPlaneBytes + (aux ? kTmaAuxBytes : 0u));
    const int zz = zoff + wrapi(kk, nz);
    const unsigned d = xs + (unsigned)(R * kSlotB);
    tma_load3(d + kTmaMain * 8u, &maps.x_main, i0, j0, zz, bar);
    tma_load3(d + kTmaTop * 8u, &maps.x_rows, i0, jt, zz, bar);
    tma_load3(d + kTmaBot * 8u, &maps.x_rows, i0, jb, zz, bar);
    tma_load3(d + kTmaLeft * 8u, &maps.x_cols, il, j0, zz, bar);
    tma_load3(d + kTmaRight * 8u, &maps.x_cols, ir, j0, zz, bar);
    if (aux) tma_load3(as + (unsigned)(R * kAuxB), &maps.b_main, i0, j0, zz, bar);
  };
  // this thread's tap addresses inside slot 0 (shared-space bytes): x taps (pairs at c-2, c, c+2),
  // y taps (rows ty-2 .. ty+2 at column c), its rhs pair
  const int c = 2 * tx;
  const unsigned ax0 = xs + 8u * (unsigned)(tx == 0 ? kTmaLeft + 2 * ty : kTmaMain + ty * kPTX + c - 2);
  const unsigned ay0 = xs + 8u * (unsigned)(kTmaTop + ty * kPTX + c);  // row ty - 2; row ty + o - 2 at + o * kRowB
  const unsigned ax2 = xs + 8u * (unsigned)(tx == kTX - 1 ? kTmaRight + 2 * ty : kTmaMain + ty * kPTX + c + 2);
  constexpr int kRowB = kPTX * 8, kCtr = 2 * kRowB;  // the centre pair sits at ay0 + kCtr
  const unsigned aa = as + 16u * (unsigned)t;
  issue(Phase<0>{}, z.k0 - 2);
  issue(Phase<1>{}, z.k0 - 1);
  issue(Phase<2>{}, z.k0);
  issue(Phase<3>{}, z.k0 + 1);
  issue(Phase<4>{}, z.k0 + 2);
  issue(Phase<5>{}, z.k0 + 3);
  double q[2][6];  // z taps: planes k-2 .. k+2 of phase P sit in q[.][(P + o) % 6]
#pragma unroll
  for (int r = 0; r < 4; ++r) mbar_wait(bars + 8u * r, 0u);
  lds2<0 * kSlotB + kCtr>(ay0, q[0][0], q[1][0]);
  lds2<1 * kSlotB + kCtr>(ay0, q[0][1], q[1][1]);
  lds2<2 * kSlotB + kCtr>(ay0, q[0][2], q[1][2]);
  lds2<3 * kSlotB + kCtr>(ay0, q[0][3], q[1][3]);
  if (free_run) {  // planes k0-2 and k0-1 are z taps only: their slots are released here
    __syncwarp();
    if (tx == 0) {
      mbar_arrive(bars + 8u * (kTmaRing + 0));
      mbar_arrive(bars + 8u * (kTmaRing + 1));
    }
  }
  // phase P of iteration it handles plane k = k0 + 6 it + P = fill it of slot (P + 2) % 6
  auto step = [&](auto ph, int k, unsigned par) {
    constexpr int P = decltype(ph)::value;
    constexpr int SK = (P + 2) % 6;   // slot of plane k
    constexpr int S2 = (P + 4) % 6;   // slot of plane k + 2: fill it + (P >= 2)
    mbar_wait(bars + 8u * S2, par ^ (P >= 2 ? 1u : 0u));  // plane k+2 has landed
    if (!free_run) __syncthreads();  // every thread is past plane k-1: the slot of plane k-2 is free
    issue(Phase<P>{}, k + 4, true, par);  // slot P: its fill (it + 1) follows release number it
    lds2<S2 * kSlotB + kCtr>(ay0, q[0][(P + 4) % 6], q[1][(P + 4) % 6]);
    plane(k);
    PairTaps v;
    lds2<SK * kSlotB>(ax0, v.x[0], v.x[1]);
    lds2<SK * kSlotB + kCtr>(ay0, v.x[2], v.x[3]);
    lds2<SK * kSlotB>(ax2, v.x[4], v.x[5]);
    lds2<SK * kSlotB + 0 * kRowB>(ay0, v.y[0][0], v.y[1][0]);
    lds2<SK * kSlotB + 1 * kRowB>(ay0, v.y[0][1], v.y[1][1]);
    v.y[0][2] = v.x[2];
    v.y[1][2] = v.x[3];
    lds2<SK * kSlotB + 3 * kRowB>(ay0, v.y[0][3], v.y[1][3]);
    lds2<SK * kSlotB + 4 * kRowB>(ay0, v.y[0][4], v.y[1][4]);
#pragma unroll
    for (int o = 0; o < 5; ++o) {
      v.z[0][o] = q[0][(P + o) % 6];
      v.z[1][o] = q[1][(P + o) % 6];
    }
    double av[2] = {0.0, 0.0};
    if (HAS_AUX) lds2<SK * kAuxB>(aa, av[0], av[1]);
    if (free_run) {  // this warp's last read of plane k's slot
      __syncwarp();
      if (tx == 0) mbar_arrive(bars + 8u * (kTmaRing + SK));
    }
    body(k, (unsigned)k * pl + col, v, av, true);
  };
  unsigned par = 0;
  for (int k = z.k0; k < z.k1; k += 6, par ^= 1u) {
    step(Phase<0>{}, k, par);
    if (k + 1 >= z.k1) break;
    step(Phase<1>{}, k + 1, par);
    if (k + 2 >= z.k1) break;
    step(Phase<2>{}, k + 2, par);
    if (k + 3 >= z.k1) break;
    step(Phase<3>{}, k + 3, par);
    if (k + 4 >= z.k1) break;
    step(Phase<4>{}, k + 4, par);
    if (k + 5 >= z.k1) break;
    step(Phase<5>{}, k + 5, par);
  }
  // nothing in flight remains: planes up to k1 + 1 were waited for, later ones were never issued
}

// F_A and/or F_D, 3-D periodic, two cells per thread on TMA-staged planes (whole 64 x 8 tiles): the
// body of k_eval_ad3_pair (stencil3d.cuh) on walk_pair_tma, so the same operations and the same bits.
template <bool UCONST>
__global__ void __launch_bounds__(kTX* kTY, UCONST ? 3 : 2) k_eval_ad3_tma(Ops o, Geom g, const __grid_constant__ TmaMaps maps,
                                                                           double* __restrict__ fa, double* __restrict__ fd,
                                                                           int kc) {
  extern __shared__ __align__(128) double ev_tring[];
  const ZChunk z = zchunk(g.nz, kc);
  const long long sbase = (long long)z.s * g.ncell;
  double* fas = fa ? opaque(fa + sbase) : nullptr;
  double* fds = fd ? opaque(fd + sbase) : nullptr;
  const int s = z.s;
  double cd[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) cd[a] = o.cdiff[s][a];
  AdvPair<UCONST> ad;
  ad.init(o, g);
  walk_pair_tma<false, true>(
      maps, g.nx, g.ny, g.nz, z, ev_tring, [&](int k) { ad.plane(g, k); },
      [&](int k, unsigned cell, const PairTaps& v, const double (&)[2], bool) {
        if (fas) {
          double acc[2];
          ad.acc(o, k, v, acc);
          __stcg(reinterpret_cast<double2*>(fas + cell), make_double2(-acc[0], -acc[1]));
          flag_wild(o.wild, wild_bits(acc[0]) | wild_bits(acc[1]));
        }
        if (fds) {
          double lap[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            lap[c] = 0.0;
            lap[c] = lap[c] + cd[0] * lap5(v.x[c], v.x[c + 1], v.x[c + 2], v.x[c + 3], v.x[c + 4]);
            lap[c] = lap[c] + cd[1] * lap5(v.y[c][0], v.y[c][1], v.y[c][2], v.y[c][3], v.y[c][4]);
            lap[c] = lap[c] + cd[2] * lap5(v.z[c][0], v.z[c][1], v.z[c][2], v.z[c][3], v.z[c][4]);
          }
          __stcg(reinterpret_cast<double2*>(fds + cell), make_double2(lap[0], lap[1]));
        }
        ad.carry_k = k + 1;
      });
}

#ifndef __CUDACC_RTC__
// cuTensorMapEncodeTiled through the runtime's driver entry-point query
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline PFN_encodeTiled tma_encoder() {
  static PFN_encodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_encodeTiled>(p);
  }();
  return fn;
}
// a 3-D map over one field of S species (x, y, z * S), double elements
inline bool tma_encode(CUtensorMap* m, const double* base, int nx, int ny, int nzs, unsigned bx, unsigned by) {
  PFN_encodeTiled enc = tma_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nzs};
  const cuuint64_t strides[2] = {(cuuint64_t)nx * 8u, (cuuint64_t)nx * (cuuint64_t)ny * 8u};
  const cuuint32_t box[3] = {bx, by, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// grids the TMA walker handles: whole 64 x 8 tiles, 16-byte aligned fields
inline bool tma_grid_ok(int nx, int ny, int nz, long long ncell) {
  return nx % kPTX == 0 && ny % kTY == 0 && nx >= kPTX && ny >= kTY && nz >= 4 && tile3d_ok(ncell);
}
inline bool tma_maps(TmaMaps& M, const double* x, const double* b, int nx, int ny, int nzs) {
  if (((uintptr_t)x & 15u) || (b && ((uintptr_t)b & 15u))) return false;
  bool ok = tma_encode(&M.x_main, x, nx, ny, nzs, kPTX, kTY) && tma_encode(&M.x_rows, x, nx, ny, nzs, kPTX, 2) &&
            tma_encode(&M.x_cols, x, nx, ny, nzs, 2, kTY);
  if (ok && b) ok = tma_encode(&M.b_main, b, nx, ny, nzs, kPTX, kTY);
  return ok;
}
#endif

}  // namespace cisdc_b200
