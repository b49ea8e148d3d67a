// coder.cu — fp64 reference-order kernels behind the array-level API:
//   code_densities  (src/stain_sep.py:168-201)
//   normalize_block (src/normalize.py:115-151 + src/optics.py:97-110)
//   beer_lambert    (src/optics.py:71-94, through the 256-entry OD table)
// These are the building blocks the reference exposes publicly; the fused
// transform (xform.cu) is what the hot path runs.
#include "launch_count.h"
#include "spcn_device.cuh"
#include "xform.h"

namespace spcn {

__global__ void __launch_bounds__(256) k_code_densities(const double* __restrict__ od,
                                                        double* __restrict__ h, int64_t n,
                                                        const __grid_constant__ StrictP sp) {
  const NnlsGram G = gram_of(sp);
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) {
    const double v0 = od[i], v1 = od[n + i], v2 = od[2 * n + i];
    const double b0 = strict_dot3(sp.ws[0][0], sp.ws[1][0], sp.ws[2][0], v0, v1, v2);
    const double b1 = strict_dot3(sp.ws[0][1], sp.ws[1][1], sp.ws[2][1], v0, v1, v2);
    double h0, h1;
    strict_nnls(b0, b1, G, sp.lam, sp.max_sweeps, sp.tol, h0, h1);
    h[i] = h0;
    h[n + i] = h1;
  }
}

__global__ void __launch_bounds__(256) k_normalize_block(const double* __restrict__ h,
                                                         uint8_t* __restrict__ out, int64_t n,
                                                         const __grid_constant__ StrictP sp) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) {
    const double s0 = __dmul_rn(sp.f[0], h[i]);
    const double s1 = __dmul_rn(sp.f[1], h[n + i]);
#pragma unroll
    for (int c = 0; c < 3; ++c)
      out[3 * i + c] = (uint8_t)strict_channel(sp.wt[c][0], sp.wt[c][1], s0, s1, sp.i0t[c]);
  }
}

__global__ void __launch_bounds__(256) k_beer_lambert(const uint8_t* __restrict__ px,
                                                      double* __restrict__ od, int64_t n,
                                                      const __grid_constant__ StrictP sp) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) {
#pragma unroll
    for (int c = 0; c < 3; ++c) od[c * n + i] = sp.lut[c][px[3 * i + c]];
  }
}

__global__ void __launch_bounds__(256) k_inverse_bl(const double* __restrict__ od,
                                                    uint8_t* __restrict__ out, int64_t n,
                                                    const __grid_constant__ StrictP sp) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < n; i += 256ll * gridDim.x) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double y = __dmul_rn(sp.i0t[c], exp(-od[3 * i + c]));
      y = floor(__dadd_rn(y, 0.5));
      out[3 * i + c] = (uint8_t)fmin(fmax(y, 0.0), 255.0);
    }
  }
}

static int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  return static_cast<int>(want < (int64_t)sms * 16 ? (want > 0 ? want : 1) : (int64_t)sms * 16);
}

cudaError_t launch_code_densities(const double* od, double* h, int64_t n, const StrictP& sp,
                                  cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_code_densities<<<grid_for(n), 256, 0, st>>>(od, h, n, sp);
  return launched();
}

cudaError_t launch_normalize_block(const double* h, uint8_t* out, int64_t n, const StrictP& sp,
                                   cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_normalize_block<<<grid_for(n), 256, 0, st>>>(h, out, n, sp);
  return launched();
}

cudaError_t launch_beer_lambert(const uint8_t* px, double* od, int64_t n, const StrictP& sp,
                                cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_beer_lambert<<<grid_for(n), 256, 0, st>>>(px, od, n, sp);
  return launched();
}

cudaError_t launch_inverse_bl(const double* od, uint8_t* out, int64_t n, const StrictP& sp,
                              cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_inverse_bl<<<grid_for(n), 256, 0, st>>>(od, out, n, sp);
  return launched();
}

}  // namespace spcn
