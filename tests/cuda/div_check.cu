// div_rcp / rcp_refined (csrc/newton.cuh) against the IEEE division `/`, bit for bit, on random,
// binade-edge, near-midpoint and extreme-range operand pairs.  Built and run by
// tests/test_gpu_parity.py::test_div_rcp_bitexact.
#include <cstdio>
#include <cstdlib>

#include "newton.cuh"

using namespace cisdc_b200;

__device__ unsigned long long mix(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

__device__ double make(unsigned long long r, int emin, int span) {
  const int e = (int)((r >> 52) % (unsigned long long)span) + emin;  // unbiased exponent
  const unsigned long long m = r & 0xfffffffffffffULL;
  double v = __longlong_as_double((long long)(((unsigned long long)(e + 1023) << 52) | m));
  return (r >> 63) ? -v : v;
}

// mode 0: exponents in [-60, 60]; 1: [-1000, 1000] (slow-path territory included);
// 2: mantissas near all-ones; 3: a ~ b * (midpoint) ; 4: zeros, infinities, NaN mixed in
__global__ void k_check(unsigned long long seed, long long n, int mode, unsigned long long* bad, double* ex) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const unsigned long long r1 = mix(seed ^ (2 * t + 1)), r2 = mix(seed + 0x9e3779b97f4a7c15ULL * (t + 7));
    double a, b;
    if (mode == 1) {
      a = make(r1, -1000, 2001);
      b = make(r2, -1000, 2001);
    } else {
      a = make(r1, -60, 121);
      b = make(r2, -60, 121);
    }
    if (mode == 2) {
      a = __longlong_as_double(__double_as_longlong(a) | 0xfff0000000000LL);
      b = __longlong_as_double(__double_as_longlong(b) | 0x7ff0000000000LL);
    }
    if (mode == 3) {
      const double q = make(r1 ^ 0x5555, -30, 61);
      const double h = ldexp(fabs(q), -53);
      a = b * (q + ((r1 >> 9) & 1 ? h : -h));
    }
    if (mode == 4) {
      const int w = (int)(r1 % 8);
      if (w == 0) a = 0.0;
      if (w == 1) a = -0.0;
      if (w == 2) b = __longlong_as_double(0x7ff0000000000000LL);
      if (w == 3) a = __longlong_as_double(0x7ff8000000000000LL);
      if (w == 4) b = ldexp(1.0, -1070);
    }
    const double got = div_rcp(a, b, rcp_refined(b));
    const double want = a / b;
    const bool same = __double_as_longlong(got) == __double_as_longlong(want) || (got != got && want != want);
    if (!same && atomicAdd(bad, 1ULL) == 0) {
      ex[0] = a;
      ex[1] = b;
      ex[2] = got;
      ex[3] = want;
    }
  }
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : (1LL << 26);
  unsigned long long* bad;
  double* ex;
  cudaMallocManaged(&bad, sizeof(unsigned long long));
  cudaMallocManaged(&ex, 4 * sizeof(double));
  unsigned long long total = 0;
  for (int mode = 0; mode < 5; ++mode) {
    *bad = 0;
    k_check<<<148 * 8, 256>>>(0x1234567ULL + mode, n, mode, bad, ex);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      std::printf("cuda error\n");
      return 2;
    }
    std::printf("mode %d: %lld pairs, %llu mismatches\n", mode, n, *bad);
    if (*bad) std::printf("  e.g. a=%a b=%a got=%a want=%a\n", ex[0], ex[1], ex[2], ex[3]);
    total += *bad;
  }
  return total ? 1 : 0;
}
