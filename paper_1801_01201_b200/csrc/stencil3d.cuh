// 2.5-D blocked radius-2 star stencils for 3-D grids (K1 F_A/F_D, and the multigrid smoother /
// residual of K3).
//
// A (32, 8) thread block owns a 32 x 8 x-y tile and walks a chunk of z-planes.  The x-y tile of
// every plane, with its 2-cell periodic halo, is staged in a shared-memory ring of kRing planes by
// cp.async (8-byte LDGSTS, no register staging): while plane k is computed, planes k+3 .. k+5 are
// in flight, which is what keeps enough bytes outstanding per SM to run at HBM bandwidth (one
// plane of prefetch through registers measured 1.8 TB/s).  An auxiliary per-point field (the
// multigrid right-hand side) rides in a second ring.  The z taps live in a 5-deep register queue
// fed from the ring's plane k+2; the plane loop is unrolled by 5 so the queue rotates by renaming.
// Every input value comes from HBM once per chunk (plus the tile halo, from L2) instead of once per
// stencil tap.  The arithmetic is the generic kernels' expressions in the same operand order (same
// bits): only the data source of each tap changes.
#pragma once

#include "common.cuh"
#include "stencil.cuh"

namespace cisdc_b200 {

constexpr int kTX = 32, kTY = 8, kHalo = 2;
constexpr int kTileW = kTX + 2 * kHalo, kTileH = kTY + 2 * kHalo;
constexpr int kTileP = kTileW + 1;                                 // padded row pitch
constexpr int kTileN = kTileW * kTileH;                            // 432 staged values per plane
constexpr int kTilePer = (kTileN + kTX * kTY - 1) / (kTX * kTY);   // 2 per thread
constexpr int kRing = 8;                                           // planes k-2 .. k+5
constexpr int kPlaneSlot = kTileH * kTileP;                        // doubles per ring slot

__device__ __forceinline__ int wrap_any(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

// hides a pointer's provenance from the optimiser so that `p + 32-bit offset` stays a single
// wide multiply-add instead of being re-associated into 64-bit index arithmetic
template <class T>
__device__ __forceinline__ T* opaque(T* p) {
  asm("" : "+l"(p));
  return p;
}

__device__ __forceinline__ void cp_async8(unsigned smem, const double* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// The tile elements this thread stages: smem slot and in-plane offset (32-bit: one species' field
// is < 2^32 cells, checked by the launcher).  Only the last element can fall outside the tile.
struct TileLoader {
  int slot[kTilePer];
  unsigned off[kTilePer];
  __device__ __forceinline__ void init(int nx, int ny, int i0, int j0) {
    const int t = threadIdx.y * kTX + threadIdx.x;
#pragma unroll
    for (int u = 0; u < kTilePer; ++u) {
      const int idx = t + u * kTX * kTY;
      if (idx < kTileN) {
        const int r = idx / kTileW, c = idx - r * kTileW;
        slot[u] = r * kTileP + c;
        off[u] = (unsigned)wrap_any(j0 + r - kHalo, ny) * (unsigned)nx + (unsigned)wrap_any(i0 + c - kHalo, nx);
      } else {
        slot[u] = -1;
        off[u] = 0;
      }
    }
  }
  __device__ __forceinline__ static bool full(int u) { return (u + 1) * kTX * kTY <= kTileN; }
};

// z-chunking: blockIdx.z = s * nzc + zc
struct ZChunk {
  int s, k0, k1;
};
__device__ __forceinline__ ZChunk zchunk(int nz, int kc) {
  const int nzc = (nz + kc - 1) / kc;
  ZChunk z;
  z.s = blockIdx.z / nzc;
  const int zc = blockIdx.z - z.s * nzc;
  z.k0 = zc * kc;
  z.k1 = min(nz, z.k0 + kc);
  return z;
}

#ifndef __CUDACC_RTC__
constexpr int kZChunk = 32;
inline dim3 tile3d_grid(int nx, int ny, int nz, int S) {
  return dim3((unsigned)((nx + kTX - 1) / kTX), (unsigned)((ny + kTY - 1) / kTY),
              (unsigned)(S * ((nz + kZChunk - 1) / kZChunk)));
}
// the tiled kernels index one species' field with 32-bit offsets
inline bool tile3d_ok(long long ncell) { return ncell < (1LL << 32); }
#endif

struct TileRing {
  double t[kRing][kPlaneSlot];  // 8 x 12 x 37 doubles = 28.4 KB
};
struct AuxRing {
  double a[kRing][kTX * kTY];  // 16 KB
};

constexpr int kMgMinBlocks = 3;

template <int P>
struct Phase {
  static constexpr int value = P;
};

// Walks the z-chunk of one species field f (and the matching auxiliary field aux when HAS_AUX);
// for every plane k calls plane(k) once, then body(k, cell, v, aux, ok) (cell = in-field offset,
// ok = the point is inside the grid: threads past the edge run on clamped data and must not
// write) with the 3 x 5 taps v[axis][offset + 2] and aux[cell].
template <bool HAS_AUX, class PlaneFn, class Body>
__device__ __forceinline__ void walk_tiled(const double* __restrict__ f, const double* __restrict__ aux, int nx,
                                           int ny, int nz, const ZChunk& z, TileRing& ring, AuxRing* aring,
                                           PlaneFn plane, Body body) {
  const int i0 = blockIdx.x * kTX, j0 = blockIdx.y * kTY;
  const int i = i0 + threadIdx.x, j = j0 + threadIdx.y;
  const int t = threadIdx.y * kTX + threadIdx.x;
  const unsigned pl = (unsigned)nx * (unsigned)ny;
  const bool in = i < nx && j < ny;
  const unsigned col = in ? (unsigned)j * (unsigned)nx + (unsigned)i : 0u;
  f = opaque(f);
  if (HAS_AUX) aux = opaque(aux);
  TileLoader L;
  L.init(nx, ny, i0, j0);
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(&ring.t[0][0]);
  const unsigned aux_s = HAS_AUX ? (unsigned)__cvta_generic_to_shared(&aring->a[0][t]) : 0u;
  // stage plane kk (chunk-relative planes k0-2 .. k1+1 exist; others commit an empty group so the
  // group count stays uniform)
  auto issue = [&](int kk) {
    if (kk <= z.k1 + 1) {
      const double* fp = opaque(f + (unsigned)wrapi(kk, nz) * pl);
      const unsigned sb = ring_s + (unsigned)((kk & (kRing - 1)) * kPlaneSlot) * 8u;
#pragma unroll
      for (int u = 0; u < kTilePer; ++u)
        if (TileLoader::full(u) || L.slot[u] >= 0) cp_async8(sb + (unsigned)L.slot[u] * 8u, fp + L.off[u]);
      if (HAS_AUX && kk >= z.k0 && kk < z.k1)
        cp_async8(aux_s + (unsigned)((kk & (kRing - 1)) * kTX * kTY) * 8u, aux + (unsigned)kk * pl + col);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int kk = -2; kk <= 4; ++kk) issue(z.k0 + kk);
  const int tx = threadIdx.x + kHalo, ty = threadIdx.y + kHalo;
  const int cidx = ty * kTileP + tx;
  double q[5];  // z taps of this column; planes k0-2 .. k0+1 first
  // planes k-2 .. k+2 sit in q[(P + o) % 5]; the step loads plane k+2 into q[(P + 4) % 5]
  auto step = [&](auto ph, int k) {
    constexpr int P = decltype(ph)::value;
    cp_async_wait<2>();  // this thread's copies of plane k+2 have landed
    __syncthreads();     // ... and everyone's; plane k-3 is free
    issue(k + 5);
    const double* tk = &ring.t[k & (kRing - 1)][0];
    q[(P + 4) % 5] = ring.t[(k + 2) & (kRing - 1)][cidx];
    plane(k);
    double v[3][5];
#pragma unroll
    for (int o = 0; o < 5; ++o) {
      v[0][o] = tk[cidx + o - 2];
      v[1][o] = o == 2 ? v[0][2] : tk[cidx + (o - 2) * kTileP];
      v[2][o] = q[(P + o) % 5];
    }
    const double av = HAS_AUX ? aring->a[k & (kRing - 1)][t] : 0.0;
    body(k, (unsigned)k * pl + col, v, av, in);
  };
  // the queue's first four planes (k0-2 .. k0+1) are complete once plane k0+1 is
  cp_async_wait<3>();
  __syncthreads();
#pragma unroll
  for (int o = 0; o < 4; ++o) q[o] = ring.t[(z.k0 + o - 2) & (kRing - 1)][cidx];
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
  cp_async_wait<0>();  // no copy may be outstanding when the block exits
}

// F_A and/or F_D, 3-D periodic; MINB = resident blocks per SM the registers are budgeted for;
// UCONST: uniform face velocities (Ops::vconst), u_a = Ops::ucon[a] on every face
template <int MINB, bool UCONST>
__global__ void __launch_bounds__(kTX* kTY, MINB) k_eval_ad3_tiled(Ops o, Geom g, const double* __restrict__ phi,
                                                              double* __restrict__ fa, double* __restrict__ fd,
                                                              int kc) {
  __shared__ TileRing ring;
  const ZChunk z = zchunk(g.nz, kc);
  const long long sbase = (long long)z.s * g.ncell;
  const double* f = phi + sbase;
  double* fas = fa ? opaque(fa + sbase) : nullptr;
  double* fds = fd ? opaque(fd + sbase) : nullptr;
  const int s = z.s;
  // Face velocities u_a = (T_a0[i] T_a1[j]) T_a2[k] (face_u): the (i, j) factors of the right and
  // left faces are formed once per thread, times T_a2 once per plane (same bits as face_u).
  const int ic = min(blockIdx.x * kTX + threadIdx.x, g.nx - 1);
  const int jc = min(blockIdx.y * kTY + threadIdx.y, g.ny - 1);
  double pr[3], pl[3];
  const double* t2[3];
  bool adv[3];
  double cd[3], ca[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    adv[a] = o.adv[a] != 0;
    cd[a] = o.cdiff[s][a];
    ca[a] = o.cadv[a];
    t2[a] = o.vel[a][2];
    if (UCONST) continue;
    const double* t0 = o.vel[a][0];
    const double* t1 = o.vel[a][1];
    const int il = a == 0 ? wrapi(ic - 1, g.nx) : ic, jl = a == 1 ? wrapi(jc - 1, g.ny) : jc;
    pr[a] = (t0 ? __ldg(t0 + ic) : 1.0) * (t1 ? __ldg(t1 + jc) : 1.0);
    pl[a] = (t0 ? __ldg(t0 + il) : 1.0) * (t1 ? __ldg(t1 + jl) : 1.0);
  }
  double t2r[3], t2l[3];
  // z faces: the right-face flux of plane k is the left-face flux of plane k+1 in the same column
  // (same velocity bits: for a = 2 pl == pr and T2 index k; same bracket operands), so it is carried
  double fz_carry = 0.0;
  int carry_k = -1;
  walk_tiled<false>(
      f, nullptr, g.nx, g.ny, g.nz, z, ring, nullptr,
      [&](int k) {
        if (UCONST) return;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          t2r[a] = t2[a] ? __ldg(t2[a] + k) : 1.0;
          t2l[a] = t2[a] ? __ldg(t2[a] + (a == 2 ? wrapi(k - 1, g.nz) : k)) : 1.0;
        }
      },
      [&](int k, unsigned cell, const double (&v)[3][5], double, bool ok) {
        if (fas) {
          double acc = 0.0;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            if (!adv[a]) continue;
            const double ur = UCONST ? o.ucon[a] : pr[a] * t2r[a];
            const double fr = ur * (7.0 * (v[a][2] + v[a][3]) - (v[a][1] + v[a][4]));
            double fl;
            if (a == 2 && carry_k == k) {
              fl = fz_carry;
            } else {
              const double ul = UCONST ? o.ucon[a] : pl[a] * t2l[a];
              fl = ul * (7.0 * (v[a][1] + v[a][2]) - (v[a][0] + v[a][3]));
            }
            if (a == 2) fz_carry = fr;
            acc = acc + (fr - fl) * ca[a];
          }
          if (ok) __stcg(fas + cell, -acc);
        }
        if (fds) {
          double lap = 0.0;
#pragma unroll
          for (int a = 0; a < 3; ++a) lap = lap + cd[a] * lap5(v[a][0], v[a][1], v[a][2], v[a][3], v[a][4]);
          if (ok) __stcg(fds + cell, lap);
        }
        carry_k = k + 1;
      });
}

}  // namespace cisdc_b200
