// Row-streaming radius-2 star stencils for 2-D grids (F_A/F_D, and the multigrid level sweeps).
//
// Every warp owns a 64-column strip (two x-adjacent cells per lane) and walks a chunk of rows:
// each row of the strip, with its 2-cell periodic x halo (68 values), is staged by 16-byte cp.async
// into the warp's own shared-memory ring (8 rows; rows j+3 .. j+5 in flight while row j is
// computed), an auxiliary per-point field (the multigrid rhs) in a second ring.  The y taps live in
// a 5-deep register queue fed from the ring's row j+2; the row loop is unrolled by 5 so the queue
// rotates by renaming.  Warps never wait for each other (no block barrier: __syncwarp only).
// The arithmetic is the generic 2-D kernels' expressions in the same operand order (same bits).
// Needs nx even (a cell pair never straddles the periodic seam).
#pragma once

#include "common.cuh"
#include "stencil.cuh"
#include "stencil3d.cuh"

namespace cisdc_b200 {

constexpr int kRowW = 64;                 // columns per warp strip
constexpr int kRowTileW = kRowW + 4;      // 68 staged values per row
constexpr int kRowRing = 8, kRowAhead = 5;
constexpr int kRowWarps = 8;              // warps (strips) per block
constexpr size_t kRowSmemPerWarp = (size_t)kRowRing * (kRowTileW + kRowW) * sizeof(double);  // 8.4 KB
constexpr size_t kRowSmem = kRowWarps * kRowSmemPerWarp;                                     // 67 KB

#ifndef __CUDACC_RTC__
// grid (strip groups, row chunks, S)
inline int rows_chunk(long long ncell, int S) { return ncell * S >= (16LL << 20) ? 32 : 8; }
inline dim3 rows_grid(int nx, int ny, int S, int chunk) {
  return dim3((unsigned)((nx + kRowW * kRowWarps - 1) / (kRowW * kRowWarps)), (unsigned)((ny + chunk - 1) / chunk),
              (unsigned)S);
}
#endif

// Taps of a cell pair (i, i+1) at row j: x[0..5] = i-2 .. i+3; y[c][o] = row offset o-2.
struct RowTaps {
  double x[6];
  double y[2][5];
};

// f / aux: the species' fields.  body(j, cell, taps, aux_pair, ok), rowfn(j) once per row.
template <bool HAS_AUX, class RowFn, class Body>
__device__ __forceinline__ void walk_rows(const double* __restrict__ f, const double* __restrict__ aux, int nx,
                                          int ny, int j0, int j1, double* smem, RowFn rowfn, Body body) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = (blockIdx.x * kRowWarps + warp) * kRowW;
  if (x0 >= nx) return;  // whole strip outside (warp-uniform)
  const int i = x0 + 2 * lane;
  const bool in_x = i < nx;
  double* ring = smem + (size_t)warp * (kRowSmemPerWarp / sizeof(double));
  double* aring = ring + kRowRing * kRowTileW;
  f = opaque(f);
  if (HAS_AUX) aux = opaque(aux);
  // staged chunks: lane l -> chunk l, lanes 0-1 also chunk 32 + l (34 chunks of 2 values)
  const unsigned off0 = (unsigned)wrap_any(x0 - 2 + 2 * lane, nx);
  const unsigned off1 = (unsigned)wrap_any(x0 - 2 + 2 * (32 + lane), nx);
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
  const unsigned aux_s = HAS_AUX ? (unsigned)__cvta_generic_to_shared(aring + 2 * lane) : 0u;
  const unsigned coli = in_x ? (unsigned)i : 0u;
  auto issue = [&](int jj) {
    if (jj <= j1 + 1) {
      const double* rp = opaque(f + (unsigned)wrapi(jj, ny) * (unsigned)nx);
      const unsigned sb = ring_s + (unsigned)((jj & (kRowRing - 1)) * kRowTileW) * 8u;
      cp_async16(sb + 16u * lane, rp + off0);
      if (lane < 2) cp_async16(sb + 16u * (32 + lane), rp + off1);
      if (HAS_AUX && jj >= j0 && jj < j1)
        cp_async16(aux_s + (unsigned)((jj & (kRowRing - 1)) * kRowW) * 8u, aux + (unsigned)jj * (unsigned)nx + coli);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int jj = -2; jj < kRowAhead; ++jj) issue(j0 + jj);
  const int cidx = 2 + 2 * lane;  // cell i in a staged row
  double q[2][5];
  auto ld2 = [&](const double* p, double& a, double& b) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    a = v.x;
    b = v.y;
  };
  auto step = [&](auto ph, int j) {
    constexpr int P = decltype(ph)::value;
    cp_async_wait<kRowAhead - 3>();  // this lane's copies of row j+2 have landed
    __syncwarp();                    // ... and the other lanes'; row j-3 is free
    issue(j + kRowAhead);
    const double* rj = ring + (j & (kRowRing - 1)) * kRowTileW;
    ld2(ring + ((j + 2) & (kRowRing - 1)) * kRowTileW + cidx, q[0][(P + 4) % 5], q[1][(P + 4) % 5]);
    rowfn(j);
    RowTaps v;
    ld2(rj + cidx - 2, v.x[0], v.x[1]);
    ld2(rj + cidx, v.x[2], v.x[3]);
    ld2(rj + cidx + 2, v.x[4], v.x[5]);
#pragma unroll
    for (int o = 0; o < 5; ++o) {
      v.y[0][o] = q[0][(P + o) % 5];
      v.y[1][o] = q[1][(P + o) % 5];
    }
    double av[2] = {0.0, 0.0};
    if (HAS_AUX) ld2(aring + (j & (kRowRing - 1)) * kRowW + 2 * lane, av[0], av[1]);
    body(j, (unsigned)j * (unsigned)nx + coli, v, av, in_x);
  };
  cp_async_wait<kRowAhead - 2>();  // rows j0-2 .. j0+1
  __syncwarp();
#pragma unroll
  for (int o = 0; o < 4; ++o) ld2(ring + ((j0 + o - 2) & (kRowRing - 1)) * kRowTileW + cidx, q[0][o], q[1][o]);
  for (int j = j0; j < j1; j += 5) {
    step(Phase<0>{}, j);
    if (j + 1 >= j1) break;
    step(Phase<1>{}, j + 1);
    if (j + 2 >= j1) break;
    step(Phase<2>{}, j + 2);
    if (j + 3 >= j1) break;
    step(Phase<3>{}, j + 3);
    if (j + 4 >= j1) break;
    step(Phase<4>{}, j + 4);
  }
  cp_async_wait<0>();
}

// F_A and/or F_D on a 2-D periodic grid (nx even), one species per blockIdx.z, rows
// [blockIdx.y * chunk, ...): adv_periodic / diff_periodic of stencil.cuh, same operations.
__global__ void __launch_bounds__(kRowWarps * 32, 2) k_eval_ad2_rows(Ops o, Geom g, const double* __restrict__ phi,
                                                                     double* __restrict__ fa, double* __restrict__ fd,
                                                                     int chunk) {
  extern __shared__ __align__(16) double rsm[];
  const int s = blockIdx.z;
  const int j0 = blockIdx.y * chunk, j1 = min(g.ny, j0 + chunk);
  const long long sbase = (long long)s * g.ncell;
  double* fas = fa ? opaque(fa + sbase) : nullptr;
  double* fds = fd ? opaque(fd + sbase) : nullptr;
  const bool ax = o.adv[0] != 0, ay = o.adv[1] != 0;
  const double cd0 = o.cdiff[s][0], cd1 = o.cdiff[s][1], ca0 = o.cadv[0], ca1 = o.cadv[1];
  const double *t00 = o.vel[0][0], *t01 = o.vel[0][1], *t10 = o.vel[1][0], *t11 = o.vel[1][1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = min((blockIdx.x * kRowWarps + warp) * kRowW + 2 * lane, g.nx - 2);
  // x-table factors of the three x faces (i-1/2, i+1/2, i+3/2) and the two y-face columns
  const double fx_l = t00 ? __ldg(t00 + wrapi(i - 1, g.nx)) : 1.0;
  const double fx_m = t00 ? __ldg(t00 + i) : 1.0;
  const double fx_r = t00 ? __ldg(t00 + i + 1) : 1.0;
  const double fy0 = t10 ? __ldg(t10 + i) : 1.0, fy1 = t10 ? __ldg(t10 + i + 1) : 1.0;
  double gx = 1.0, gy = 1.0, gyl = 1.0;  // row factors: T01[j], T11[j], T11[j-1]
  double fy_carry[2] = {0.0, 0.0};
  int carry_j = -1;
  walk_rows<false>(
      phi + sbase, nullptr, g.nx, g.ny, j0, j1, rsm,
      [&](int j) {
        gx = t01 ? __ldg(t01 + j) : 1.0;
        gy = t11 ? __ldg(t11 + j) : 1.0;
        gyl = t11 ? __ldg(t11 + wrapi(j - 1, g.ny)) : 1.0;
      },
      [&](int j, unsigned cell, const RowTaps& v, const double (&)[2], bool ok) {
        if (fas) {
          double acc[2] = {0.0, 0.0};
          if (ax) {  // face_u = (T00 T01) * 1.0 (no z table in 2-D: the factor 1.0 is exact)
            const double u_l = fx_l * gx, u_m = fx_m * gx, u_r = fx_r * gx;
            const double f_l = u_l * (7.0 * (v.x[1] + v.x[2]) - (v.x[0] + v.x[3]));
            const double f_m = u_m * (7.0 * (v.x[2] + v.x[3]) - (v.x[1] + v.x[4]));
            const double f_r = u_r * (7.0 * (v.x[3] + v.x[4]) - (v.x[2] + v.x[5]));
            acc[0] = acc[0] + (f_m - f_l) * ca0;
            acc[1] = acc[1] + (f_r - f_m) * ca0;
          }
          if (ay) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const double fyc = c == 0 ? fy0 : fy1;
              const double fr = (fyc * gy) * (7.0 * (v.y[c][2] + v.y[c][3]) - (v.y[c][1] + v.y[c][4]));
              const double fl = carry_j == j ? fy_carry[c]
                                             : (fyc * gyl) * (7.0 * (v.y[c][1] + v.y[c][2]) - (v.y[c][0] + v.y[c][3]));
              fy_carry[c] = fr;
              acc[c] = acc[c] + (fr - fl) * ca1;
            }
          }
          if (ok) {
            __stcg(reinterpret_cast<double2*>(fas + cell), make_double2(-acc[0], -acc[1]));
            flag_wild(o.wild, wild_bits(acc[0]) | wild_bits(acc[1]));
          }
        }
        if (fds) {
          double lap[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            lap[c] = 0.0;
            lap[c] = lap[c] + cd0 * lap5(v.x[c], v.x[c + 1], v.x[c + 2], v.x[c + 3], v.x[c + 4]);
            lap[c] = lap[c] + cd1 * lap5(v.y[c][0], v.y[c][1], v.y[c][2], v.y[c][3], v.y[c][4]);
          }
          if (ok) __stcg(reinterpret_cast<double2*>(fds + cell), make_double2(lap[0], lap[1]));
        }
        carry_j = j + 1;
      });
}

}  // namespace cisdc_b200
