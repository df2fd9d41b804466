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
constexpr int kZChunk = 32;  // planes per block (64 and 128 measured the same, 16 slower: r2s)
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
          if (ok) {
            __stcg(fas + cell, -acc);
            flag_wild(o.wild, wild_bits(acc));
          }
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

// ------------------------------------------------------------------------------------------------
// Two x-adjacent cells per thread (F_A/F_D on grids with even nx): a (32, 8) block owns a 64 x 8
// tile; the 68 x 12 halo tile of a plane is staged with 16-byte cp.async (pairs of cells never
// straddle the periodic seam when nx is even), and each thread reads its x taps i-2 .. i+3 as three
// 128-bit shared loads and its y taps / new z tap as 128-bit pairs: 8 shared loads per 2 cells
// instead of 2 x 10 eight-byte ones.  The face between the two cells is shared (same bits: same
// bracket operands, same face velocity).
constexpr int kPTX = 2 * kTX;                 // 64 cells wide
constexpr int kPTileW = kPTX + 2 * kHalo;     // 68
constexpr int kPTileP = kPTileW;              // pitch (16-byte rows)
constexpr int kPChunks = kPTileW / 2 * kTileH;  // 408 16-byte chunks per plane
constexpr int kPChunkPer = (kPChunks + kTX * kTY - 1) / (kTX * kTY);  // 2
constexpr int kPPlaneSlot = kTileH * kPTileP;   // 816 doubles
constexpr size_t kPairSmem = (size_t)kRing * kPPlaneSlot * sizeof(double);  // 52 KB (dynamic)

__device__ __forceinline__ void cp_async16(unsigned smem, const double* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem), "l"(g) : "memory");
}

#ifndef __CUDACC_RTC__
inline dim3 tile3d_pair_grid(int nx, int ny, int nz, int S) {
  return dim3((unsigned)((nx + kPTX - 1) / kPTX), (unsigned)((ny + kTY - 1) / kTY),
              (unsigned)(S * ((nz + kZChunk - 1) / kZChunk)));
}
#endif

// Taps of a cell pair (i, i+1) at plane k: x[0..5] = i-2 .. i+3; y[c][o], z[c][o] = offsets o-2.
struct PairTaps {
  double x[6];
  double y[2][5];
  double z[2][5];
};

constexpr size_t kPairAuxSmem = (size_t)kRing * kTX * kTY * 2 * sizeof(double);  // 32 KB
// the multigrid sweep's smaller rings (6 planes each: 39 + 24 KB) fit 3 blocks per SM
constexpr int kMgRing = 6;
constexpr size_t kMgPairSmem = (size_t)kMgRing * (kPPlaneSlot + kTX * kTY * 2) * sizeof(double);

// HAS_AUX: a pointwise field (the multigrid rhs) staged as pairs in aux_ring (kRing x 512 doubles);
// body(k, cell, taps, aux_pair[2], ok).
// RING: plane slots (>= 6: planes k .. k+5 are live; 8 uses a mask, others a modulo).
template <int RING>
__device__ __forceinline__ int ring_slot(int kk) {
  if constexpr ((RING & (RING - 1)) == 0) return kk & (RING - 1);
  const int r = kk % RING;
  return r < 0 ? r + RING : r;
}

template <bool HAS_AUX, int RING, int AHEAD, class PlaneFn, class Body>
__device__ __forceinline__ void walk_pair(const double* __restrict__ f, const double* __restrict__ aux, int nx,
                                          int ny, int nz, const ZChunk& z, double* ring, double* aux_ring,
                                          PlaneFn plane, Body body) {
  // AHEAD planes are staged ahead of the one being computed: the prologue stages k0-2 .. k0+AHEAD-1
  // (all of them must fit, since the queue is filled from k0-2 .. k0+1 before the first step), the
  // step of plane k stages k+AHEAD into the slot of plane k+AHEAD-RING (dead).
  static_assert(AHEAD >= 4 && AHEAD + 2 <= RING, "ring too small for the staging distance");
  const int i0 = blockIdx.x * kPTX, j0 = blockIdx.y * kTY;
  const int i = i0 + 2 * threadIdx.x, j = j0 + threadIdx.y;
  const int t = threadIdx.y * kTX + threadIdx.x;
  const unsigned pl = (unsigned)nx * (unsigned)ny;
  const bool in = i < nx && j < ny;  // nx even: i and i+1 are in or out together
  const unsigned col = in ? (unsigned)j * (unsigned)nx + (unsigned)i : 0u;
  f = opaque(f);
  // staged chunks of this thread: smem slot (in doubles) and in-plane offset of the pair
  int slot[kPChunkPer];
  unsigned off[kPChunkPer];
#pragma unroll
  for (int u = 0; u < kPChunkPer; ++u) {
    const int idx = t + u * kTX * kTY;
    if (idx < kPChunks) {
      const int r = idx / (kPTileW / 2), c2 = idx - r * (kPTileW / 2);
      slot[u] = r * kPTileP + 2 * c2;
      off[u] = (unsigned)wrap_any(j0 + r - kHalo, ny) * (unsigned)nx + (unsigned)wrap_any(i0 + 2 * c2 - kHalo, nx);
    } else {
      slot[u] = -1;
      off[u] = 0;
    }
  }
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring);
  const unsigned aux_s = HAS_AUX ? (unsigned)__cvta_generic_to_shared(aux_ring + 2 * t) : 0u;
  if (HAS_AUX) aux = opaque(aux);
  auto issue = [&](int kk) {
    if (kk <= z.k1 + 1) {
      const double* fp = opaque(f + (unsigned)wrapi(kk, nz) * pl);
      const unsigned sb = ring_s + (unsigned)(ring_slot<RING>(kk) * kPPlaneSlot) * 8u;
#pragma unroll
      for (int u = 0; u < kPChunkPer; ++u)
        if ((u + 1) * kTX * kTY <= kPChunks || slot[u] >= 0) cp_async16(sb + (unsigned)slot[u] * 8u, fp + off[u]);
      if (HAS_AUX && kk >= z.k0 && kk < z.k1)
        cp_async16(aux_s + (unsigned)(ring_slot<RING>(kk) * kTX * kTY * 2) * 8u, aux + (unsigned)kk * pl + col);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int kk = -2; kk < AHEAD; ++kk) issue(z.k0 + kk);
  const int cidx = (threadIdx.y + kHalo) * kPTileP + 2 * threadIdx.x + kHalo;  // cell i in the tile
  double q[2][5];
  auto ld2 = [&](const double* p, double& a, double& b) {
    const double2 v = *reinterpret_cast<const double2*>(p);
    a = v.x;
    b = v.y;
  };
  auto step = [&](auto ph, int k) {
    constexpr int P = decltype(ph)::value;
    cp_async_wait<AHEAD - 3>();  // plane k+2 has landed
    __syncthreads();
    issue(k + AHEAD);
    const double* tk = ring + ring_slot<RING>(k) * kPPlaneSlot;
    ld2(ring + ring_slot<RING>(k + 2) * kPPlaneSlot + cidx, q[0][(P + 4) % 5], q[1][(P + 4) % 5]);
    plane(k);
    PairTaps v;
    ld2(tk + cidx - 2, v.x[0], v.x[1]);
    ld2(tk + cidx, v.x[2], v.x[3]);
    ld2(tk + cidx + 2, v.x[4], v.x[5]);
#pragma unroll
    for (int o = 0; o < 5; ++o) {
      if (o == 2) {
        v.y[0][2] = v.x[2];
        v.y[1][2] = v.x[3];
      } else {
        ld2(tk + cidx + (o - 2) * kPTileP, v.y[0][o], v.y[1][o]);
      }
      v.z[0][o] = q[0][(P + o) % 5];
      v.z[1][o] = q[1][(P + o) % 5];
    }
    double av[2] = {0.0, 0.0};
    if (HAS_AUX) ld2(aux_ring + ring_slot<RING>(k) * kTX * kTY * 2 + 2 * t, av[0], av[1]);
    body(k, (unsigned)k * pl + col, v, av, in);
  };
  cp_async_wait<AHEAD - 2>();  // planes k0-2 .. k0+1
  __syncthreads();
#pragma unroll
  for (int o = 0; o < 4; ++o) ld2(ring + ring_slot<RING>(z.k0 + o - 2) * kPPlaneSlot + cidx, q[0][o], q[1][o]);
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
  cp_async_wait<0>();
}

// Per-thread advection state of the pair kernels: face-velocity factors per cell c of the pair
// (face_u order: (T0 T1) T2; for a = 0 the left face of cell 1 is the right face of cell 0, same
// product), the z-face carry, and the F_A of a pair from its taps.  Shared by k_eval_ad3_pair and the
// multigrid check + evaluation kernel (multigrid.cuh), so both compute F_A with the same operations.
template <bool UCONST>
struct AdvPair {
  double pr[2][3], pl[2][3];
  const double* t2[3];
  bool adv[3];
  double ca[3];
  double t2r[3], t2l[3];
  double fz_carry[2];
  int carry_k;
  __device__ __forceinline__ void init(const Ops& o, const Geom& g) {
    const int ic = min(blockIdx.x * kPTX + 2 * threadIdx.x, g.nx - 2);
    const int jc = min(blockIdx.y * kTY + threadIdx.y, g.ny - 1);
    fz_carry[0] = fz_carry[1] = 0.0;
    carry_k = -1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      adv[a] = o.adv[a] != 0;
      ca[a] = o.cadv[a];
      t2[a] = o.vel[a][2];
      if (UCONST) continue;
      const double* t0 = o.vel[a][0];
      const double* t1 = o.vel[a][1];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int icc = ic + c;
        const int il = a == 0 ? wrapi(icc - 1, g.nx) : icc, jl = a == 1 ? wrapi(jc - 1, g.ny) : jc;
        pr[c][a] = (t0 ? __ldg(t0 + icc) : 1.0) * (t1 ? __ldg(t1 + jc) : 1.0);
        pl[c][a] = (t0 ? __ldg(t0 + il) : 1.0) * (t1 ? __ldg(t1 + jl) : 1.0);
      }
    }
  }
  __device__ __forceinline__ void plane(const Geom& g, int k) {
    if (UCONST) return;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      t2r[a] = t2[a] ? __ldg(t2[a] + k) : 1.0;
      t2l[a] = t2[a] ? __ldg(t2[a] + (a == 2 ? wrapi(k - 1, g.nz) : k)) : 1.0;
    }
  }
  // acc = -F_A of the pair at plane k (per-cell 5-tap views: x taps of cell c are v.x[c .. c+4])
  __device__ __forceinline__ void acc(const Ops& o, int k, const PairTaps& v, double (&acc)[2]) {
    acc[0] = 0.0;
    acc[1] = 0.0;
    // axis 0: faces i-1/2, i+1/2, i+3/2
    if (adv[0]) {
      const double u_l0 = UCONST ? o.ucon[0] : pl[0][0] * t2l[0];
      const double u_m = UCONST ? o.ucon[0] : pr[0][0] * t2r[0];
      const double u_r1 = UCONST ? o.ucon[0] : pr[1][0] * t2r[0];
      const double f_l0 = u_l0 * (7.0 * (v.x[1] + v.x[2]) - (v.x[0] + v.x[3]));
      const double f_m = u_m * (7.0 * (v.x[2] + v.x[3]) - (v.x[1] + v.x[4]));
      const double f_r1 = u_r1 * (7.0 * (v.x[3] + v.x[4]) - (v.x[2] + v.x[5]));
      acc[0] = acc[0] + (f_m - f_l0) * ca[0];
      acc[1] = acc[1] + (f_r1 - f_m) * ca[0];
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (adv[1]) {
        const double ur = UCONST ? o.ucon[1] : pr[c][1] * t2r[1];
        const double ul = UCONST ? o.ucon[1] : pl[c][1] * t2l[1];
        const double fr = ur * (7.0 * (v.y[c][2] + v.y[c][3]) - (v.y[c][1] + v.y[c][4]));
        const double fl = ul * (7.0 * (v.y[c][1] + v.y[c][2]) - (v.y[c][0] + v.y[c][3]));
        acc[c] = acc[c] + (fr - fl) * ca[1];
      }
      if (adv[2]) {
        const double ur = UCONST ? o.ucon[2] : pr[c][2] * t2r[2];
        const double fr = ur * (7.0 * (v.z[c][2] + v.z[c][3]) - (v.z[c][1] + v.z[c][4]));
        double fl;
        if (carry_k == k) {
          fl = fz_carry[c];
        } else {
          const double ul = UCONST ? o.ucon[2] : pl[c][2] * t2l[2];
          fl = ul * (7.0 * (v.z[c][1] + v.z[c][2]) - (v.z[c][0] + v.z[c][3]));
        }
        fz_carry[c] = fr;
        acc[c] = acc[c] + (fr - fl) * ca[2];
      }
    }
  }
};

// F_A and/or F_D, 3-D periodic, two cells per thread (nx even); UCONST as k_eval_ad3_tiled.
template <bool UCONST>
__global__ void __launch_bounds__(kTX* kTY, UCONST ? 3 : 2) k_eval_ad3_pair(Ops o, Geom g, const double* __restrict__ phi,
                                                               double* __restrict__ fa, double* __restrict__ fd, int kc) {
  extern __shared__ __align__(16) double pring[];
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
  walk_pair<false, kRing, 5>(
      phi + sbase, nullptr, g.nx, g.ny, g.nz, z, pring, nullptr, [&](int k) { ad.plane(g, k); },
      [&](int k, unsigned cell, const PairTaps& v, const double (&)[2], bool ok) {
        if (fas) {
          double acc[2];
          ad.acc(o, k, v, acc);
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
            lap[c] = lap[c] + cd[0] * lap5(v.x[c], v.x[c + 1], v.x[c + 2], v.x[c + 3], v.x[c + 4]);
            lap[c] = lap[c] + cd[1] * lap5(v.y[c][0], v.y[c][1], v.y[c][2], v.y[c][3], v.y[c][4]);
            lap[c] = lap[c] + cd[2] * lap5(v.z[c][0], v.z[c][1], v.z[c][2], v.z[c][3], v.z[c][4]);
          }
          if (ok) __stcg(reinterpret_cast<double2*>(fds + cell), make_double2(lap[0], lap[1]));
        }
        ad.carry_k = k + 1;
      });
}

}  // namespace cisdc_b200
