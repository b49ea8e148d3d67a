// Bitwise check of div_by (hoisted-reciprocal division) against __ddiv_rn.
// Built and run by tests/test_div_gpu.py on the GPU box.
#include <cstdint>
#include "spcn_device.cuh"

using namespace spcn;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// operand families: random bit patterns, values in the SNMF/coder ranges,
// near-exact quotients (x = q*g +- few ulps) and tiny / huge magnitudes
__device__ double pick(uint64_t r, int fam) {
  switch (fam) {
    case 0: return __longlong_as_double((long long)r);
    case 1: return ((double)(r >> 11) * 0x1.0p-53) * 8.0 - 2.0;
    case 2: return __longlong_as_double((long long)((r & 0x800fffffffffffffull) |
                                                   ((uint64_t)(900 + (r >> 52) % 240) << 52)));
    default: return ((double)(r >> 11) * 0x1.0p-53) * 1e-30;
  }
}

extern "C" __global__ void k_div_check(uint64_t seed, int64_t n, unsigned long long* bad,
                                       double* ex) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r1 = mix64(seed ^ (2 * i)), r2 = mix64(seed ^ (2 * i + 1));
    const int fam = (int)(r1 & 3);
    double g = fabs(pick(r2, fam == 0 ? 0 : (fam == 3 ? 2 : 1)));
    if (fam == 1) g = 0.2 + fabs(g);            // Gram-like divisors
    double x = pick(r1 >> 2, fam);
    if ((r2 & 7) == 0) {                         // near-exact quotient
      const double q = pick(r1 >> 5, 1);
      x = __longlong_as_double(__double_as_longlong(__dmul_rn(q, g)) + (long long)(r2 >> 60) - 8);
    }
    const Recip R = make_recip(g);
    const double a = div_by(x, R), b = __ddiv_rn(x, g);
    const bool same = __double_as_longlong(a) == __double_as_longlong(b) || (a != a && b != b);
    if (!same) {
      const unsigned long long k = atomicAdd(bad, 1ull);
      if (k < 4) { ex[3 * k] = x; ex[3 * k + 1] = g; ex[3 * k + 2] = a; }
    }
  }
}

extern "C" int run_div_check(uint64_t seed, int64_t n, unsigned long long* bad_out,
                             double* examples_out) {
  unsigned long long* bad = nullptr;
  double* ex = nullptr;
  if (cudaMalloc(&bad, sizeof(unsigned long long)) != cudaSuccess) return 1;
  if (cudaMalloc(&ex, 12 * sizeof(double)) != cudaSuccess) return 1;
  cudaMemset(bad, 0, sizeof(unsigned long long));
  cudaMemset(ex, 0, 12 * sizeof(double));
  k_div_check<<<148 * 16, 256>>>(seed, n, bad, ex);
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  cudaMemcpy(bad_out, bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaMemcpy(examples_out, ex, 12 * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(bad);
  cudaFree(ex);
  return 0;
}
