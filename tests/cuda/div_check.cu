// Bit-exactness check of div_by (csrc/newton.cuh) against the IEEE division, on random and
// adversarial operand pairs.  Built and run by tests/test_gpu_parity.py::test_div_by_bitexact.
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

// mode 0: uniform random bit patterns with exponents in [-420, 420]
// mode 1: near-binade-top mantissas (m_a * m_b close to 2, the q0 error worst case)
// mode 2: quotients near rounding midpoints: a = RN(b * (q + ulp/2 +- tiny))
__global__ void k_check(unsigned long long seed, long long n, int mode, unsigned long long* bad,
                        double* example) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const unsigned long long r1 = mix(seed ^ (2 * t + 1)), r2 = mix(seed + 0x9e3779b97f4a7c15ULL * (t + 7));
    double a, b;
    const int ea = (int)(r1 >> 52) % 841 - 420, eb = (int)(r2 >> 52) % 841 - 420;
    unsigned long long ma = r1 & 0xfffffffffffffULL, mb = r2 & 0xfffffffffffffULL;
    if (mode == 1) {
      ma |= 0xff00000000000ULL;
      mb |= 0x7f00000000000ULL;
    }
    a = __longlong_as_double((long long)(((unsigned long long)(ea + 1023) << 52) | ma));
    b = __longlong_as_double((long long)(((unsigned long long)(eb + 1023) << 52) | mb));
    if (r1 & 1) a = -a;
    if (r2 & 2) b = -b;
    if (mode == 2) {
      // a close to b * midpoint: pick q, form b*(q + half-ulp) rounded (ties broken by the data)
      const double q = __longlong_as_double((long long)(((unsigned long long)((ea % 200) + 1023) << 52) | ma));
      const double half = __longlong_as_double((long long)(((unsigned long long)((ea % 200) + 1023 - 53) << 52)));
      a = b * (q + half * ((r1 >> 7) & 1 ? 1.0 : -1.0)) + ((r1 >> 8) & 1 ? 0.0 : -0.0);
    }
    const double y = 1.0 / b;
    const double got = div_by(a, b, y, div_range_ok(b));
    const double want = a / b;
    if (__double_as_longlong(got) != __double_as_longlong(want)) {
      if (atomicAdd(bad, 1ULL) == 0) {
        example[0] = a;
        example[1] = b;
        example[2] = got;
        example[3] = want;
      }
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
  for (int mode = 0; mode < 3; ++mode) {
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
