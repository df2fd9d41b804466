// 2.5-D blocked radius-2 star stencils for 3-D grids (K1 F_A/F_D, and the multigrid smoother /
// residual of K3).
//
// A (32, 8) thread block owns an x-y tile and walks a chunk of z-planes.  Each thread keeps its
// column's five z-values (k-2 .. k+2) in a register queue; the x/y neighbours of plane k come from a
// shared-memory tile with a 2-cell periodic halo.  The next plane's tile is prefetched into
// registers while the current plane is computed (its L2 latency overlaps the arithmetic), and the
// periodic tile offsets are computed once per block, not per plane.  Every input value is fetched
// from HBM once per chunk (plus the tile halo, from L2) instead of once per stencil tap.  The
// arithmetic is the generic kernels' expressions in the same operand order (same bits): only the
// data source of each tap changes.
#pragma once

#include "common.cuh"
#include "stencil.cuh"

namespace cisdc_b200 {

constexpr int kTX = 32, kTY = 8, kHalo = 2;
constexpr int kTileW = kTX + 2 * kHalo, kTileH = kTY + 2 * kHalo;
constexpr int kTileN = kTileW * kTileH;                         // 432
constexpr int kTilePer = (kTileN + kTX * kTY - 1) / (kTX * kTY);  // 2 elements per thread

__device__ __forceinline__ int wrap_any(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

// The (up to) two tile elements this thread stages: smem slot and in-plane global offset.
struct TileLoader {
  int slot[kTilePer];
  long long off[kTilePer];
  __device__ __forceinline__ void init(int nx, int ny, int i0, int j0) {
    const int t = threadIdx.y * kTX + threadIdx.x;
#pragma unroll
    for (int u = 0; u < kTilePer; ++u) {
      const int idx = t + u * kTX * kTY;
      if (idx < kTileN) {
        const int r = idx / kTileW, c = idx - r * kTileW;
        slot[u] = r * (kTileW + 1) + c;
        off[u] = (long long)wrap_any(j0 + r - kHalo, ny) * nx + wrap_any(i0 + c - kHalo, nx);
      } else {
        slot[u] = -1;
        off[u] = 0;
      }
    }
  }
  __device__ __forceinline__ void fetch(const double* __restrict__ plane, double (&v)[kTilePer]) const {
#pragma unroll
    for (int u = 0; u < kTilePer; ++u) v[u] = slot[u] >= 0 ? __ldg(plane + off[u]) : 0.0;
  }
  __device__ __forceinline__ void store(double* tile, const double (&v)[kTilePer]) const {
#pragma unroll
    for (int u = 0; u < kTilePer; ++u)
      if (slot[u] >= 0) tile[slot[u]] = v[u];
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
  return dim3((unsigned)((nx + kTX - 1) / kTX), (unsigned)((ny + kTY - 1) / kTY),
              (unsigned)(S * ((nz + kZChunk - 1) / kZChunk)));
}
#endif

// Walks the z-chunk of one species stack f, calling body(k, v) for every in-range point with the
// 3 x 5 taps v[axis][offset + 2] of plane k.
template <class Body>
__device__ __forceinline__ void walk_tiled(const double* __restrict__ f, int nx, int ny, int nz, const ZChunk& z,
                                           double (*tile)[kTileW + 1], Body body) {
  const int i0 = blockIdx.x * kTX, j0 = blockIdx.y * kTY;
  const int i = i0 + threadIdx.x, j = j0 + threadIdx.y;
  const bool in = i < nx && j < ny;
  const long long pl = (long long)nx * ny;
  const long long col = (long long)(in ? j : 0) * nx + (in ? i : 0);
  TileLoader L;
  L.init(nx, ny, i0, j0);
  double pre[kTilePer];
  L.fetch(f + (long long)z.k0 * pl, pre);
  double q0 = __ldg(f + wrapi(z.k0 - 2, nz) * pl + col);
  double q1 = __ldg(f + wrapi(z.k0 - 1, nz) * pl + col);
  double q2 = __ldg(f + (long long)z.k0 * pl + col);
  double q3 = __ldg(f + wrapi(z.k0 + 1, nz) * pl + col);
  L.store(&tile[0][0], pre);
  const int tx = threadIdx.x + kHalo, ty = threadIdx.y + kHalo;
  for (int k = z.k0; k < z.k1; ++k) {
    __syncthreads();  // tile(k) complete
    const double q4 = __ldg(f + wrapi(k + 2, nz) * pl + col);
    if (k + 1 < z.k1) L.fetch(f + (long long)(k + 1) * pl, pre);
    if (in) {
      double v[3][5];
#pragma unroll
      for (int o2 = 0; o2 < 5; ++o2) {
        v[0][o2] = tile[ty][tx + o2 - 2];
        v[1][o2] = tile[ty + o2 - 2][tx];
      }
      v[2][0] = q0;
      v[2][1] = q1;
      v[2][2] = q2;
      v[2][3] = q3;
      v[2][4] = q4;
      body(k, (long long)k * pl + col, i, j, v);
    }
    __syncthreads();  // everyone is done with tile(k)
    if (k + 1 < z.k1) L.store(&tile[0][0], pre);
    q0 = q1;
    q1 = q2;
    q2 = q3;
    q3 = q4;
  }
}

// F_A and/or F_D, 3-D periodic
__global__ void __launch_bounds__(kTX* kTY) k_eval_ad3_tiled(Ops o, Geom g, const double* __restrict__ phi,
                                                              double* __restrict__ fa, double* __restrict__ fd,
                                                              int kc) {
  __shared__ double tile[kTileH][kTileW + 1];
  const ZChunk z = zchunk(g.nz, kc);
  const double* f = phi + (long long)z.s * g.ncell;
  const long long sbase = (long long)z.s * g.ncell;
  const int s = z.s;
  // Face velocities u_a = (T_a0[i] T_a1[j]) T_a2[k] (face_u): the (i, j) factor of the right and
  // left faces is fixed for this thread's column -- formed once, times T_a2 per plane (same bits).
  const int ic = min(blockIdx.x * kTX + threadIdx.x, g.nx - 1), jc = min(blockIdx.y * kTY + threadIdx.y, g.ny - 1);
  double pr[3], pl[3];
  const double* t2[3];
  bool adv[3];
  double cd[3], ca[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    adv[a] = o.adv[a] != 0;
    cd[a] = o.cdiff[s][a];
    ca[a] = o.cadv[a];
    const int il = a == 0 ? wrapi(ic - 1, g.nx) : ic, jl = a == 1 ? wrapi(jc - 1, g.ny) : jc;
    const double* t0 = o.vel[a][0];
    const double* t1 = o.vel[a][1];
    pr[a] = (t0 ? __ldg(t0 + ic) : 1.0) * (t1 ? __ldg(t1 + jc) : 1.0);
    pl[a] = (t0 ? __ldg(t0 + il) : 1.0) * (t1 ? __ldg(t1 + jl) : 1.0);
    t2[a] = o.vel[a][2];
  }
  walk_tiled(f, g.nx, g.ny, g.nz, z, tile, [&](int k, long long cell, int, int, const double (&v)[3][5]) {
    const long long e = sbase + cell;
    if (fa) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (!adv[a]) continue;
        const double ur = pr[a] * (t2[a] ? __ldg(t2[a] + k) : 1.0);
        const double ul = pl[a] * (t2[a] ? __ldg(t2[a] + (a == 2 ? wrapi(k - 1, g.nz) : k)) : 1.0);
        const double fr = ur * (7.0 * (v[a][2] + v[a][3]) - (v[a][1] + v[a][4]));
        const double fl = ul * (7.0 * (v[a][1] + v[a][2]) - (v[a][0] + v[a][3]));
        acc = acc + (fr - fl) * ca[a];
      }
      fa[e] = -acc;
    }
    if (fd) {
      double lap = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) lap = lap + cd[a] * lap5(v[a][0], v[a][1], v[a][2], v[a][3], v[a][4]);
      fd[e] = lap;
    }
  });
}

}  // namespace cisdc_b200
