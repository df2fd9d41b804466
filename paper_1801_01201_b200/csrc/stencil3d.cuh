// 2.5-D blocked radius-2 star stencils for 3-D grids (K1 F_A/F_D, and the multigrid smoother /
// residual of K3).
//
// A (32, 8) thread block owns an x-y tile and walks a chunk of z-planes.  Each thread keeps its
// column's five z-values (k-2 .. k+2) in a register queue; the x/y neighbours of plane k come from a
// shared-memory tile with a 2-cell periodic halo.  Every input value is fetched from HBM once per
// chunk (plus the tile halo, from L2), instead of once per stencil tap.  The arithmetic is the
// generic kernels' expressions with the same operand order (same bits): only the data source of
// each tap changes.
#pragma once

#include "common.cuh"
#include "stencil.cuh"

namespace cisdc_b200 {

constexpr int kTX = 32, kTY = 8, kHalo = 2;
constexpr int kTileW = kTX + 2 * kHalo, kTileH = kTY + 2 * kHalo;

__device__ __forceinline__ int wrap_any(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

// tile[r][c] = f(i0 + c - 2, j0 + r - 2, k) periodic; called by all threads of the block
__device__ __forceinline__ void load_tile(double (*tile)[kTileW + 1], const double* __restrict__ f, int nx, int ny,
                                          int i0, int j0, int k) {
  const int t = threadIdx.y * kTX + threadIdx.x;
  const long long plane = (long long)k * ny * nx;
  for (int idx = t; idx < kTileW * kTileH; idx += kTX * kTY) {
    const int r = idx / kTileW, c = idx - r * kTileW;
    const int gi = wrap_any(i0 + c - kHalo, nx), gj = wrap_any(j0 + r - kHalo, ny);
    tile[r][c] = __ldg(f + plane + (long long)gj * nx + gi);
  }
}

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

// F_A and/or F_D, 3-D periodic
__global__ void __launch_bounds__(kTX* kTY) k_eval_ad3_tiled(Ops o, Geom g, const double* __restrict__ phi,
                                                              double* __restrict__ fa, double* __restrict__ fd,
                                                              int kc) {
  __shared__ double tile[kTileH][kTileW + 1];
  const ZChunk z = zchunk(g.nz, kc);
  const int i0 = blockIdx.x * kTX, j0 = blockIdx.y * kTY;
  const int i = i0 + threadIdx.x, j = j0 + threadIdx.y;
  const bool in = i < g.nx && j < g.ny;
  const int ic = in ? i : 0, jc = in ? j : 0;
  const double* f = phi + (long long)z.s * g.ncell;
  const long long col = (long long)jc * g.nx + ic, pl = (long long)g.nx * g.ny;
  double q0 = __ldg(f + wrapi(z.k0 - 2, g.nz) * pl + col);
  double q1 = __ldg(f + wrapi(z.k0 - 1, g.nz) * pl + col);
  double q2 = __ldg(f + (long long)z.k0 * pl + col);
  double q3 = __ldg(f + wrapi(z.k0 + 1, g.nz) * pl + col);
  const int tx = threadIdx.x + kHalo, ty = threadIdx.y + kHalo;
  const int im1 = wrapi(i - 1, g.nx), jm1 = wrapi(j - 1, g.ny);
  for (int k = z.k0; k < z.k1; ++k) {
    const double q4 = __ldg(f + wrapi(k + 2, g.nz) * pl + col);
    __syncthreads();
    load_tile(tile, f, g.nx, g.ny, i0, j0, k);
    __syncthreads();
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
      const long long e = (long long)z.s * g.ncell + (long long)k * pl + col;
      if (fa) {
        double acc = 0.0;
        const int km1 = wrapi(k - 1, g.nz);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (!o.adv[a]) continue;
          const int ia = a == 0 ? im1 : i, ja = a == 1 ? jm1 : j, ka = a == 2 ? km1 : k;
          const double fr = face_u(o, a, i, j, k) * (7.0 * (v[a][2] + v[a][3]) - (v[a][1] + v[a][4]));
          const double fl = face_u(o, a, ia, ja, ka) * (7.0 * (v[a][1] + v[a][2]) - (v[a][0] + v[a][3]));
          acc = acc + (fr - fl) * o.cadv[a];
        }
        fa[e] = -acc;
      }
      if (fd) {
        double lap = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) lap = lap + o.cdiff[z.s][a] * lap5(v[a][0], v[a][1], v[a][2], v[a][3], v[a][4]);
        fd[e] = lap;
      }
    }
    q0 = q1;
    q1 = q2;
    q2 = q3;
    q3 = q4;
  }
}

}  // namespace cisdc_b200
