// 2.5-D blocked radius-2 star stencils for 3-D grids (K1 F_A/F_D, and the multigrid smoother /
// residual of K3).
//
// A (32, 8) thread block owns a 32 x (8 R) x-y tile (R rows per thread) and walks a chunk of
// z-planes.  Each thread keeps its columns' five z-values (k-2 .. k+2) in register queues; the x/y
// neighbours of plane k come from a shared-memory tile with a 2-cell periodic halo.  Everything the
// next plane needs -- its tile, the z-value k+3 and an auxiliary per-point input (the multigrid
// right-hand side) -- is fetched into registers while the current plane is computed, so HBM/L2
// latency overlaps the arithmetic; the periodic tile offsets are computed once per block.  Every
// input value comes from HBM once per chunk (plus the tile halo, from L2) instead of once per
// stencil tap.  The arithmetic is the generic kernels' expressions in the same operand order (same
// bits): only the data source of each tap changes.
#pragma once

#include "common.cuh"
#include "stencil.cuh"

namespace cisdc_b200 {

#ifndef CISDC_TILE_ROWS
#define CISDC_TILE_ROWS 1
#endif
constexpr int kTX = 32, kTY = 8, kHalo = 2, kRows = CISDC_TILE_ROWS;
constexpr int kTileW = kTX + 2 * kHalo, kTileH = kTY * kRows + 2 * kHalo;
constexpr int kTileN = kTileW * kTileH;                           // 432
constexpr int kTilePer = (kTileN + kTX * kTY - 1) / (kTX * kTY);  // 2 elements per thread

__device__ __forceinline__ int wrap_any(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
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
        slot[u] = r * (kTileW + 1) + c;
        off[u] = (unsigned)wrap_any(j0 + r - kHalo, ny) * (unsigned)nx + (unsigned)wrap_any(i0 + c - kHalo, nx);
      } else {
        slot[u] = -1;
        off[u] = 0;
      }
    }
  }
  __device__ __forceinline__ static bool full(int u) { return (u + 1) * kTX * kTY <= kTileN; }
  __device__ __forceinline__ void fetch(const double* __restrict__ plane, double (&v)[kTilePer]) const {
#pragma unroll
    for (int u = 0; u < kTilePer; ++u) v[u] = (full(u) || slot[u] >= 0) ? __ldg(plane + off[u]) : 0.0;
  }
  __device__ __forceinline__ void store(double* tile, const double (&v)[kTilePer]) const {
#pragma unroll
    for (int u = 0; u < kTilePer; ++u)
      if (full(u) || slot[u] >= 0) tile[slot[u]] = v[u];
  }
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
  return dim3((unsigned)((nx + kTX - 1) / kTX), (unsigned)((ny + kTY * kRows - 1) / (kTY * kRows)),
              (unsigned)(S * ((nz + kZChunk - 1) / kZChunk)));
}
// the tiled kernels index one species' field with 32-bit offsets
inline bool tile3d_ok(long long ncell) { return ncell < (1LL << 32); }
#endif

using TileArr = double[kTileH][kTileW + 1];

// occupancy targets (blocks of 256 per SM); forcing more resident blocks spills and was measured
// slower (C5: F_A/F_D 1.6 -> 2.0 ms per launch at 3 blocks)
constexpr int kEvalMinBlocks = 1, kMgMinBlocks = 1;

// hides a pointer's provenance from the optimiser so that `p + 32-bit offset` stays a single
// wide multiply-add instead of being re-associated into 64-bit index arithmetic
template <class T>
__device__ __forceinline__ T* opaque(T* p) {
  asm("" : "+l"(p));
  return p;
}

template <int P>
struct Phase {
  static constexpr int value = P;
};

// Walks the z-chunk of one species field f (and the matching auxiliary field aux, may be null);
// for every plane k calls plane(k) once, then for every point of the thread's rows
// body(r, k, cell, v, aux, ok) (r = the thread's row slot, cell = in-field offset, ok = the point
// is inside the grid: rows past the edge run on clamped data and must not write) with the 3 x 5
// taps v[axis][offset + 2] and aux[cell] (0 without aux).
//
// The z taps live in a 5-deep register queue per row.  The plane loop is unrolled by 5 with the
// queue phase a compile-time constant, so the queue "rotates" by renaming instead of register
// moves.  All addressing is 32-bit inside the species field.
template <class PlaneFn, class Body>
__device__ __forceinline__ void walk_tiled(const double* __restrict__ f, const double* __restrict__ aux, int nx,
                                           int ny, int nz, const ZChunk& z, TileArr& tile, PlaneFn plane,
                                           Body body) {
  const int i0 = blockIdx.x * kTX, j0 = blockIdx.y * kTY * kRows;
  const int i = i0 + threadIdx.x;
  const unsigned pl = (unsigned)nx * (unsigned)ny;
  f = opaque(f);
  if (aux) aux = opaque(aux);
  bool in[kRows];
  unsigned col[kRows];
  double q[kRows][5], a_nx[kRows];
#pragma unroll
  for (int r = 0; r < kRows; ++r) {
    const int jr = j0 + threadIdx.y + r * kTY;
    in[r] = i < nx && jr < ny;
    col[r] = in[r] ? (unsigned)jr * (unsigned)nx + (unsigned)i : 0u;
#pragma unroll
    for (int o = 0; o < 5; ++o) q[r][o] = __ldg(f + (unsigned)wrapi(z.k0 + o - 2, nz) * pl + col[r]);
    a_nx[r] = aux ? __ldg(aux + (unsigned)z.k0 * pl + col[r]) : 0.0;
  }
  TileLoader L;
  L.init(nx, ny, i0, j0);
  double pre[kTilePer];
  L.fetch(f + (unsigned)z.k0 * pl, pre);
  L.store(&tile[0][0], pre);
  const int tx = threadIdx.x + kHalo;
  // planes k-2 .. k+2 sit in q[r][(P + o) % 5]; afterwards slot P (plane k-2) takes plane k+3
  auto step = [&](auto ph, int k) {
    constexpr int P = decltype(ph)::value;
    __syncthreads();  // tile(k) complete
    const bool more = k + 1 < z.k1;
    const unsigned kp = (unsigned)k * pl, kn = kp + pl;
    const double* f3 = opaque(f + (unsigned)wrapi(k + 3, nz) * pl);
    const double* fn = opaque(f + kn);
    const double* an = aux ? opaque(aux + kn) : nullptr;
    double q5[kRows], a_cur[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {  // prefetch for plane k+1
      a_cur[r] = a_nx[r];
      q5[r] = more ? __ldg(f3 + col[r]) : 0.0;
      if (aux && more) a_nx[r] = __ldg(an + col[r]);
    }
    if (more) L.fetch(fn, pre);
    plane(k);
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int ty = threadIdx.y + r * kTY + kHalo;
      double v[3][5];
#pragma unroll
      for (int o = 0; o < 5; ++o) {
        v[0][o] = tile[ty][tx + o - 2];
        v[1][o] = o == 2 ? v[0][2] : tile[ty + o - 2][tx];
        v[2][o] = q[r][(P + o) % 5];
      }
      body(r, k, kp + col[r], v, a_cur[r], in[r]);
    }
    __syncthreads();  // everyone is done with tile(k)
    if (more) L.store(&tile[0][0], pre);
#pragma unroll
    for (int r = 0; r < kRows; ++r) q[r][P] = q5[r];
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
}

// F_A and/or F_D, 3-D periodic
__global__ void __launch_bounds__(kTX* kTY, kEvalMinBlocks) k_eval_ad3_tiled(Ops o, Geom g, const double* __restrict__ phi,
                                                              double* __restrict__ fa, double* __restrict__ fd,
                                                              int kc) {
  __shared__ TileArr tile;
  const ZChunk z = zchunk(g.nz, kc);
  const long long sbase = (long long)z.s * g.ncell;
  const double* f = phi + sbase;
  double* fas = fa ? opaque(fa + sbase) : nullptr;
  double* fds = fd ? opaque(fd + sbase) : nullptr;
  const int s = z.s;
  // Face velocities u_a = (T_a0[i] T_a1[j]) T_a2[k] (face_u): the (i, j) factors of the right and
  // left faces are formed once per thread-row, times T_a2 once per plane (same bits as face_u).
  const int ic = min(blockIdx.x * kTX + threadIdx.x, g.nx - 1);
  double pr[kRows][3], pl[kRows][3];
  const double* t2[3];
  bool adv[3];
  double cd[3], ca[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    adv[a] = o.adv[a] != 0;
    cd[a] = o.cdiff[s][a];
    ca[a] = o.cadv[a];
    t2[a] = o.vel[a][2];
    const double* t0 = o.vel[a][0];
    const double* t1 = o.vel[a][1];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int jc = min(blockIdx.y * kTY * kRows + threadIdx.y + r * kTY, g.ny - 1);
      const int il = a == 0 ? wrapi(ic - 1, g.nx) : ic, jl = a == 1 ? wrapi(jc - 1, g.ny) : jc;
      pr[r][a] = (t0 ? __ldg(t0 + ic) : 1.0) * (t1 ? __ldg(t1 + jc) : 1.0);
      pl[r][a] = (t0 ? __ldg(t0 + il) : 1.0) * (t1 ? __ldg(t1 + jl) : 1.0);
    }
  }
  double t2r[3], t2l[3];
  // z faces: the right-face flux of plane k is the left-face flux of plane k+1 in the same column
  // (same velocity bits: for a = 2 pl == pr and T2 index k; same bracket operands), so it is carried
  double fz_carry[kRows];
  int carry_k = -1;
  walk_tiled(
      f, nullptr, g.nx, g.ny, g.nz, z, tile,
      [&](int k) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          t2r[a] = t2[a] ? __ldg(t2[a] + k) : 1.0;
          t2l[a] = t2[a] ? __ldg(t2[a] + (a == 2 ? wrapi(k - 1, g.nz) : k)) : 1.0;
        }
      },
      [&](int r, int k, unsigned cell, const double (&v)[3][5], double, bool ok) {
        if (fas) {
          double acc = 0.0;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            if (!adv[a]) continue;
            const double ur = pr[r][a] * t2r[a];
            const double fr = ur * (7.0 * (v[a][2] + v[a][3]) - (v[a][1] + v[a][4]));
            double fl;
            if (a == 2 && carry_k == k) {
              fl = fz_carry[r];
            } else {
              const double ul = pl[r][a] * t2l[a];
              fl = ul * (7.0 * (v[a][1] + v[a][2]) - (v[a][0] + v[a][3]));
            }
            if (a == 2) fz_carry[r] = fr;
            acc = acc + (fr - fl) * ca[a];
          }
          if (ok) fas[cell] = -acc;
        }
        if (fds) {
          double lap = 0.0;
#pragma unroll
          for (int a = 0; a < 3; ++a) lap = lap + cd[a] * lap5(v[a][0], v[a][1], v[a][2], v[a][3], v[a][4]);
          if (ok) fds[cell] = lap;
        }
        if (r == kRows - 1) carry_k = k + 1;
      });
}

}  // namespace cisdc_b200
