// Probe: throughput of a full 2^24-entry colour table gather (64 MB, L2-resident)
// vs the streaming copy, on a synthetic 400 Mpx RGB8 image.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_fill(uint32_t* t, uint8_t* img, int64_t npx, int levels) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (1 << 24); i += (int64_t)gridDim.x * blockDim.x)
    t[i] = (uint32_t)(i * 2654435761u) & 0xffffff;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npx * 3; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = i * 0x9e3779b97f4a7c15ull; z ^= z >> 29;
    img[i] = (uint8_t)(levels >= 256 ? (z & 255) : 120 + (z % levels));   // colour range
  }
}

// each thread: 16 px (48 B) -> 16 gathers -> 48 B out
template <bool GATHER>
__global__ void __launch_bounds__(256) k_map(const uint4* __restrict__ in, uint4* __restrict__ out,
                                             const uint32_t* __restrict__ t, int64_t nblk) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblk; b += (int64_t)gridDim.x * blockDim.x) {
    const uint4 q0 = in[3 * b], q1 = in[3 * b + 1], q2 = in[3 * b + 2];
    uint32_t w[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
    if (GATHER) {
      uint32_t v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int o = 3 * k;
        const uint32_t lo = w[o >> 2], hi = w[(o >> 2) + 1 < 12 ? (o >> 2) + 1 : 11];
        const uint32_t idx = __funnelshift_r(lo, hi, 8 * (o & 3)) & 0xffffff;
        v[k] = __ldg(t + idx);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int o = 3 * k;
        // scatter 3 bytes of v[k] into the output words
        w[o >> 2] = __byte_perm(w[o >> 2], v[k], 0x3210);  // placeholder pack (probe only)
      }
      w[0] ^= v[15]; w[5] ^= v[7]; w[11] ^= v[3];
    }
    out[3 * b] = make_uint4(w[0], w[1], w[2], w[3]);
    out[3 * b + 1] = make_uint4(w[4], w[5], w[6], w[7]);
    out[3 * b + 2] = make_uint4(w[8], w[9], w[10], w[11]);
  }
}

int main(int argc, char** argv) {
  const int levels = argc > 1 ? atoi(argv[1]) : 64;
  const int64_t npx = 400000000;
  uint8_t *img, *out;
  uint32_t* t;
  cudaMalloc(&img, npx * 3);
  cudaMalloc(&out, npx * 3);
  cudaMalloc(&t, sizeof(uint32_t) << 24);
  k_fill<<<148 * 8, 256>>>(t, img, npx, levels);
  printf("levels per channel: %d\n", levels);
  cudaDeviceSynchronize();
  const int64_t nblk = npx / 16;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    for (int grid : {148 * 8, 148 * 16, 148 * 32}) {
      for (int r = 0; r < 2; ++r) {
        cudaEventRecord(a);
        for (int it = 0; it < 10; ++it) {
          if (mode) k_map<true><<<grid, 256>>>((const uint4*)img, (uint4*)out, t, nblk);
          else k_map<false><<<grid, 256>>>((const uint4*)img, (uint4*)out, t, nblk);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 10;
        if (r) printf("%s grid %d: %.3f ms  %.1f Gpx/s  %.1f GB/s (6 B/px)\n", mode ? "gather" : "copy  ",
                      grid, ms, npx / ms / 1e6, 6.0 * npx / ms / 1e6);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
