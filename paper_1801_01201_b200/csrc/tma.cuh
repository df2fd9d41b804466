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
// the per-plane __syncthreads of the walker stays as the slot-reuse (WAR) fence.
//
// Shared-memory plane slot (doubles; every region 128-byte aligned, as the bulk tensor copy needs):
//   [0, 512)    interior rows 0..7, pitch 64
//   [512, 640)  rows -2, -1, pitch 64
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

constexpr int kTmaMain = 0, kTmaTop = 512, kTmaBot = 640, kTmaLeft = 768, kTmaRight = 784;
constexpr int kTmaSlot = 800;                               // doubles per plane slot
constexpr unsigned kTmaPlaneBytes = kTmaSlot * 8u;          // 6400 bytes of x per plane
constexpr unsigned kTmaAuxBytes = kPTX * kTY * 8u;          // 4096 bytes of rhs per plane
constexpr int kTmaRing = 6;
constexpr size_t kTmaSmem = (size_t)kTmaRing * (kTmaSlot + kPTX * kTY) * sizeof(double) + 128;

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
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load3(unsigned dst, const CUtensorMap* map, int x, int y, int z, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}

// walk_pair's contract (stencil3d.cuh) on TMA-staged planes; HAS_AUX stages the rhs (z-folded field
// index s * nz + k).  The plane(k) hook of walk_pair is not needed by the multigrid kernels.
template <bool HAS_AUX, int AHEAD, class Body>
__device__ __forceinline__ void walk_pair_tma(const TmaMaps& maps, int nx, int ny, int nz, const ZChunk& z,
                                              double* smem, Body body) {
  static_assert(AHEAD >= 4 && AHEAD + 2 <= kTmaRing, "ring too small for the staging distance");
  const int i0 = blockIdx.x * kPTX, j0 = blockIdx.y * kTY;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int t = ty * kTX + tx;
  const unsigned pl = (unsigned)nx * (unsigned)ny;
  const unsigned col = (unsigned)(j0 + ty) * (unsigned)nx + (unsigned)(i0 + 2 * tx);
  // ring: kTmaRing x-slots, then kTmaRing rhs slots, then the mbarriers (base rounded up to the
  // 128 bytes the bulk tensor copies need; kTmaSmem has the slack)
  smem = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem) + 127) & ~static_cast<uintptr_t>(127));
  double* xring = smem;
  double* aring = smem + kTmaRing * kTmaSlot;
  const unsigned xs = (unsigned)__cvta_generic_to_shared(xring);
  const unsigned as = (unsigned)__cvta_generic_to_shared(aring);
  const unsigned bars = (unsigned)__cvta_generic_to_shared(aring + kTmaRing * kPTX * kTY);
  const int zoff = z.s * nz;
  const int jt = j0 - 2 < 0 ? j0 - 2 + ny : j0 - 2;   // rows -2, -1 (wrapped)
  const int jb = j0 + kTY >= ny ? j0 + kTY - ny : j0 + kTY;  // rows 8, 9 (wrapped)
  const int il = i0 - 2 < 0 ? i0 - 2 + nx : i0 - 2;   // columns -2, -1
  const int ir = i0 + kPTX >= nx ? i0 + kPTX - nx : i0 + kPTX;  // columns 64, 65
  if (t == 0) {
    for (int r = 0; r < kTmaRing; ++r) mbar_init(bars + 8u * r, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int kk) {
    if (t != 0 || kk > z.k1 + 1) return;
    const int r = ring_slot<kTmaRing>(kk);
    const unsigned bar = bars + 8u * r;
    const bool aux = HAS_AUX && kk >= z.k0 && kk < z.k1;
    mbar_expect_tx(bar, kTmaPlaneBytes + (aux ? kTmaAuxBytes : 0u));
    const int zz = zoff + wrapi(kk, nz);
    const unsigned d = xs + (unsigned)(r * kTmaSlot) * 8u;
    tma_load3(d + kTmaMain * 8u, &maps.x_main, i0, j0, zz, bar);
    tma_load3(d + kTmaTop * 8u, &maps.x_rows, i0, jt, zz, bar);
    tma_load3(d + kTmaBot * 8u, &maps.x_rows, i0, jb, zz, bar);
    tma_load3(d + kTmaLeft * 8u, &maps.x_cols, il, j0, zz, bar);
    tma_load3(d + kTmaRight * 8u, &maps.x_cols, ir, j0, zz, bar);
    if (aux) tma_load3(as + (unsigned)(r * kPTX * kTY) * 8u, &maps.b_main, i0, j0, zz, bar);
  };
  // per-slot phase bits (every thread tracks the same sequence of completions)
  unsigned phase = 0;
  auto wait = [&](int kk) {
    const int r = ring_slot<kTmaRing>(kk);
    mbar_wait(bars + 8u * r, (phase >> r) & 1u);
    phase ^= 1u << r;
  };
  // this thread's tap addresses inside a slot (doubles): x taps (pairs at c-2, c, c+2), y taps
  // (rows ty-2 .. ty+2 at column c), centre
  const int c = 2 * tx;
  const int ox0 = tx == 0 ? kTmaLeft + 2 * ty : kTmaMain + ty * kPTX + c - 2;
  const int oxc = kTmaMain + ty * kPTX + c;
  const int ox2 = tx == kTX - 1 ? kTmaRight + 2 * ty : kTmaMain + ty * kPTX + c + 2;
  int oy[5];
#pragma unroll
  for (int o = 0; o < 5; ++o) {
    const int rr = ty + o - 2;
    oy[o] = rr < 0 ? kTmaTop + (rr + 2) * kPTX + c : (rr >= kTY ? kTmaBot + (rr - kTY) * kPTX + c : kTmaMain + rr * kPTX + c);
  }
  auto ld2 = [&](const double* p, double& a, double& b) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    a = v.x;
    b = v.y;
  };
#pragma unroll
  for (int kk = -2; kk < AHEAD; ++kk) issue(z.k0 + kk);
  double q[2][5];
  for (int kk = -2; kk < 2; ++kk) wait(z.k0 + kk);
#pragma unroll
  for (int o = 0; o < 4; ++o) ld2(xring + ring_slot<kTmaRing>(z.k0 + o - 2) * kTmaSlot + oxc, q[0][o], q[1][o]);
  auto step = [&](auto ph, int k) {
    constexpr int P = decltype(ph)::value;
    wait(k + 2);      // plane k+2 has landed
    __syncthreads();  // every thread is past plane k-1: the slot of plane k+AHEAD-kTmaRing is free
    issue(k + AHEAD);
    const double* tk = xring + ring_slot<kTmaRing>(k) * kTmaSlot;
    ld2(xring + ring_slot<kTmaRing>(k + 2) * kTmaSlot + oxc, q[0][(P + 4) % 5], q[1][(P + 4) % 5]);
    PairTaps v;
    ld2(tk + ox0, v.x[0], v.x[1]);
    ld2(tk + oxc, v.x[2], v.x[3]);
    ld2(tk + ox2, v.x[4], v.x[5]);
#pragma unroll
    for (int o = 0; o < 5; ++o) {
      if (o == 2) {
        v.y[0][2] = v.x[2];
        v.y[1][2] = v.x[3];
      } else {
        ld2(tk + oy[o], v.y[0][o], v.y[1][o]);
      }
      v.z[0][o] = q[0][(P + o) % 5];
      v.z[1][o] = q[1][(P + o) % 5];
    }
    double av[2] = {0.0, 0.0};
    if (HAS_AUX) ld2(aring + ring_slot<kTmaRing>(k) * kPTX * kTY + 2 * t, av[0], av[1]);
    body(k, (unsigned)k * pl + col, v, av, true);
  };
  for (int k = z.k0; k < z.k1; k += 5) {
    step(Phase<0>{}, k);
    if (k + 1 >= z.k1) break;
    step(Phase<1>{}, k + 1);
    if (k + 2 >= z.k1) break;
    step(Phase<2>{}, k + 2);
    if (k + 3 >= z.k1) break;
    step(Phase<3>{}, k + 3);
    if (k + 4 >= z.k1) break;
    step(Phase<4>{}, k + 4);
  }
  // drain: the planes issued past the last wait (k1 .. k1+1 were waited for; later ones were never
  // issued) -- nothing in flight remains, since issue() stops at k1 + 1
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
