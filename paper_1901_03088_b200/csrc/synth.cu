// synth.cu — on-device synthetic H&E slide generator (K8, measurement input).
//
// Same generative model as the reference's fixture generator
// (src/synthetic.py:26-121): tissue mask (scatter: U < tissue_fraction;
// block: a centred square of area tissue_fraction), sparse densities (40 %
// hematoxylin-only, 40 % eosin-only, rest both x0.7, magnitudes U(0.2, 2.0))
// or dense densities (h0 ~ U(0.65, 2), h1 ~ U(0, 1.2), 30 % zero), OD =
// reference basis · h, pixel = floor(i0 · exp(-OD) + 0.5).  The random
// numbers come from a counter-based hash of (seed, pixel index), so any row
// band of a 10-Gpixel slide renders independently and identically on any
// GPU (no numpy PCG64 stream: values differ from the reference's renderer,
// the model does not).  16 pixels per thread, 3 x 128-bit stores.
#include <cstdint>

#include "launch_count.h"
#include "spcn.h"
#include "synth.h"

namespace spcn {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ float u01(uint32_t x) { return (x >> 8) * (1.0f / 16777216.0f); }

__device__ __forceinline__ uint32_t render_px(const spcn_synth_params& p, uint64_t seed,
                                              int64_t y, int64_t x, int64_t width, int64_t height) {
  const uint64_t n = (uint64_t)y * (uint64_t)width + (uint64_t)x;
  const uint64_t r0 = mix64(seed ^ mix64(n));
  const uint64_t r1 = mix64(r0);
  const float ut = u01((uint32_t)r0), uk = u01((uint32_t)(r0 >> 32));
  const float ua = u01((uint32_t)r1), ub = u01((uint32_t)(r1 >> 32));
  bool tissue;
  if (p.layout == 0) {
    tissue = ut < p.tissue_fraction;
  } else {
    const int64_t side = (int64_t)llrint(sqrt((double)p.tissue_fraction * width * height));
    const int64_t bx = (width - side) / 2, by = (height - side) / 2;
    tissue = (x >= bx && x < bx + side && y >= by && y < by + side);
  }
  float h0 = 0.f, h1 = 0.f;
  if (tissue) {
    if (p.dense) {
      h0 = 0.65f + 1.35f * ua;
      h1 = (uk < 0.3f) ? 0.f : 1.2f * ub;
    } else {
      const float m0 = 0.2f + 1.8f * ua, m1 = 0.2f + 1.8f * ub;
      if (uk < 0.4f) h0 = m0;
      else if (uk < 0.8f) h1 = m1;
      else { h0 = 0.7f * m0; h1 = 0.7f * m1; }
    }
  }
  uint32_t out = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float od = p.basis[c * 2] * h0 + p.basis[c * 2 + 1] * h1;
    float v = floorf(p.i0[c] * __expf(-od) + 0.5f);
    v = fminf(fmaxf(v, 0.f), 255.f);
    out |= (uint32_t)v << (8 * c);
  }
  return out;
}

// rows [row0, row0 + rows) of a width x height slide → out (packed RGB8, row-major)
__global__ void __launch_bounds__(256) k_render(uint8_t* __restrict__ out, int64_t width,
                                                int64_t row0, int64_t rows, int64_t height,
                                                uint64_t seed,
                                                const __grid_constant__ spcn_synth_params p) {
  const int64_t npix = width * rows;
  const int64_t groups = npix / 16;
  for (int64_t gi = blockIdx.x * 256ll + threadIdx.x; gi < groups; gi += 256ll * gridDim.x) {
    uint32_t w[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t i = gi * 16 + k;
      const int64_t y = row0 + i / width, x = i % width;
      const uint32_t rgb = render_px(p, seed, y, x, width, height);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int b = 3 * k + c;
        w[b >> 2] |= ((rgb >> (8 * c)) & 255u) << (8 * (b & 3));
      }
    }
    uint4* d = reinterpret_cast<uint4*>(out + 48 * gi);
    d[0] = make_uint4(w[0], w[1], w[2], w[3]);
    d[1] = make_uint4(w[4], w[5], w[6], w[7]);
    d[2] = make_uint4(w[8], w[9], w[10], w[11]);
  }
  // tail (< 16 pixels)
  if (blockIdx.x == 0 && threadIdx.x < (unsigned)(npix - groups * 16)) {
    const int64_t i = groups * 16 + threadIdx.x;
    const int64_t y = row0 + i / width, x = i % width;
    const uint32_t rgb = render_px(p, seed, y, x, width, height);
    out[3 * i] = rgb & 255u;
    out[3 * i + 1] = (rgb >> 8) & 255u;
    out[3 * i + 2] = (rgb >> 16) & 255u;
  }
}

cudaError_t launch_render(uint8_t* out, int64_t width, int64_t row0, int64_t rows, int64_t height,
                          uint64_t seed, const spcn_synth_params& p, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t groups = (width * rows) / 16;
  int64_t grid = (groups + 255) / 256;
  if (grid > (int64_t)sms * 16) grid = (int64_t)sms * 16;
  if (grid < 1) grid = 1;
  k_render<<<(unsigned)grid, 256, 0, st>>>(out, width, row0, rows, height, seed, p);
  return launched();
}

}  // namespace spcn
