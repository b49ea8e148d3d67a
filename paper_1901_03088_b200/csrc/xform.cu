// xform.cu — the fused per-pixel recolor kernels (K1, "pass 2").
//
// Replaces the reference's per-strip hot unit `_process_strip`
// (src/pipeline.py:260-272): beer_lambert (src/optics.py:71-94) →
// code_densities (src/stain_sep.py:168-201) → normalize_block
// (src/normalize.py:115-151) → inverse_beer_lambert (src/optics.py:97-110).
//
// Kernels:
//   k_xform_tma<MODE>   persistent, warp-specialised: one producer warp streams
//                       12 KiB tiles (4096 px) into a 4-stage shared-memory ring
//                       with 1-D TMA bulk copies; 8 compute warps run the fp32
//                       path (16 px / thread, OD via a 16-way replicated
//                       shared-memory table) and store with 128-bit STG.
//                       EXACT mode certifies each rounding and appends the
//                       uncertified pixels to a repair list.
//   k_xform_repair      fp64 reference-order recompute of the listed pixels.
//   k_xform_strict      fp64 reference-order path for every pixel (STRICT mode,
//                       head/tail pixels, unaligned buffers).
#include "launch_count.h"
#include "spcn_device.cuh"
#include "xform.h"

namespace spcn {

constexpr int kTilePx = 4096;                 // pixels per tile
constexpr int kTileBytes = 3 * kTilePx;       // 12 KiB
constexpr int kStages = 4;
constexpr int kComputeWarps = 8;
constexpr int kThreads = 32 * (kComputeWarps + 1);
constexpr int kLutRep = 16;                   // table copies (bank-conflict bound 2)
constexpr int kLutBytes = 3 * 256 * kLutRep * 4;
constexpr size_t kXformSmem = kLutBytes + kStages * kTileBytes + 2 * kStages * sizeof(uint64_t);

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

struct RepairList {
  unsigned long long* count;   // device counter
  unsigned long long* items;   // (pixel index << 24) | rgb
  unsigned long long cap;
};

struct ConstLut {              // fp64 table read from kernel parameters
  const StrictP* p;
  __device__ double operator()(int c, uint32_t i) const { return p->lut[c][i]; }
};
struct SmemLut {
  const double* t;
  __device__ double operator()(int c, uint32_t i) const { return t[c * 256 + i]; }
};

// Rare path (repair-list overflow): kept out of line so the hot loop stays small.
__device__ __noinline__ void repair_inline(const StrictP& sp, uint8_t* dst, int64_t gp, uint32_t rgb) {
  const uint32_t out = strict_pixel(sp, ConstLut{&sp}, rgb & 255u, (rgb >> 8) & 255u, rgb >> 16);
  dst[3 * gp] = out & 255u;
  dst[3 * gp + 1] = (out >> 8) & 255u;
  dst[3 * gp + 2] = (out >> 16) & 255u;
}

__device__ __forceinline__ uint32_t byte_of(const uint32_t* w, int idx) {
  return (w[idx >> 2] >> (8 * (idx & 3))) & 0xffu;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 2)
    k_xform_tma(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t npix,
                const __grid_constant__ FastP fp, const __grid_constant__ StrictP sp,
                RepairList rl) {
  extern __shared__ __align__(128) uint8_t smem[];
  float* lut = reinterpret_cast<float*>(smem);
  uint8_t* stages = smem + kLutBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + kStages * kTileBytes);
  uint64_t* empty = full + kStages;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (npix + kTilePx - 1) / kTilePx;

  // replicated OD table: entry (c, x) copy r at float index c*4096 + x*16 + r
  for (int i = tid; i < 3 * 256 * kLutRep; i += kThreads) {
    const int c = i >> 12, x = (i >> 4) & 255;
    lut[i] = fp.lut[c][x];
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kComputeWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kComputeWarps) {
    // ---------------- producer warp: TMA bulk loads into the stage ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int i = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int s = i % kStages;
        if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        const int64_t n = min64(kTilePx, npix - t * kTilePx);
        const uint32_t bytes = static_cast<uint32_t>(3 * n);
        mbar_expect_tx(&full[s], bytes);
        bulk_g2s(stages + s * kTileBytes, src + 3 * t * kTilePx, bytes, &full[s], pol);
      }
    }
    return;
  }

  // ---------------- compute warps
  const int ct = tid;                        // 0..255
  const char* lbase = reinterpret_cast<const char*>(lut) + (lane & 15) * 4;
  int i = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
    const int s = i % kStages;
    mbar_wait(&full[s], (i / kStages) & 1);
    const int64_t tile0 = t * kTilePx;
    const int64_t n = min64(kTilePx, npix - tile0);
    const bool valid = 16 * ct < n;
    uint32_t w[12];
    if (valid) {
      const uint4* q = reinterpret_cast<const uint4*>(stages + s * kTileBytes + 48 * ct);
      const uint4 q0 = q[0], q1 = q[1], q2 = q[2];
      w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w;
      w[4] = q1.x; w[5] = q1.y; w[6] = q1.z; w[7] = q1.w;
      w[8] = q2.x; w[9] = q2.y; w[10] = q2.z; w[11] = q2.w;
    }
    uint32_t o[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) o[k] = 0;
    uint32_t badmask = 0;
    if (valid) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t r = byte_of(w, 3 * k), g = byte_of(w, 3 * k + 1), b = byte_of(w, 3 * k + 2);
      const float v0 = *reinterpret_cast<const float*>(lbase + (r << 6));
      const float v1 = *reinterpret_cast<const float*>(lbase + 16384 + (g << 6));
      const float v2 = *reinterpret_cast<const float*>(lbase + 32768 + (b << 6));
      const FastCore fc = fast_core(fp, v0, v1, v2);
      uint32_t c0, c1, c2;
      if (MODE == 0) {
        const float alpha = __fmaf_rn(fp.a1, fc.T, fp.a0);
        uint32_t bad = 0;
        c0 = cert_channel(fp.i0t[0], alpha, fc.e0, bad);
        c1 = cert_channel(fp.i0t[1], alpha, fc.e1, bad);
        c2 = cert_channel(fp.i0t[2], alpha, fc.e2, bad);
        badmask |= (bad != 0u ? 1u : 0u) << k;
      } else {
        c0 = fast_channel(fp.i0t[0], fc.e0);
        c1 = fast_channel(fp.i0t[1], fc.e1);
        c2 = fast_channel(fp.i0t[2], fc.e2);
      }
      const int bi = 3 * k;
      o[bi >> 2] |= (c0 & 0xffu) << (8 * (bi & 3));
      o[(bi + 1) >> 2] |= (c1 & 0xffu) << (8 * ((bi + 1) & 3));
      o[(bi + 2) >> 2] |= (c2 & 0xffu) << (8 * ((bi + 2) & 3));
    }
    }  // valid (compute)
    // Release the stage only after every loaded word has been consumed: the
    // arrive does not wait for in-flight LDS, and the next TMA write into this
    // stage is an async-proxy write (cross-proxy WAR), hence also the fence.
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (valid) {
    uint4* d = reinterpret_cast<uint4*>(dst + 3 * (tile0 + 16 * ct));
    d[0] = make_uint4(o[0], o[1], o[2], o[3]);
    d[1] = make_uint4(o[4], o[5], o[6], o[7]);
    d[2] = make_uint4(o[8], o[9], o[10], o[11]);

    if (MODE == 0) {
      // warp-aggregated append of uncertified pixels to the repair list
      const unsigned active = __activemask();
      if (__any_sync(active, badmask != 0u)) {
        const uint32_t cnt = __popc(badmask);
        uint32_t incl = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(active, incl, off);
          if (lane >= off) incl += y;
        }
        const int leader = 31 - __clz(active);
        const uint32_t total = __shfl_sync(active, incl, leader);
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(rl.count, (unsigned long long)total);
        base = __shfl_sync(active, base, leader);
        unsigned long long slot = base + incl - cnt;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if (!((badmask >> k) & 1u)) continue;
          const uint32_t rgb = byte_of(w, 3 * k) | (byte_of(w, 3 * k + 1) << 8) |
                               (byte_of(w, 3 * k + 2) << 16);
          const int64_t gp = tile0 + 16 * ct + k;
          if (slot < rl.cap) {
            rl.items[slot] = (static_cast<unsigned long long>(gp) << 24) | rgb;
          } else {  // list overflow: repair inline (same thread, ordered after the STG)
            repair_inline(sp, dst, gp, rgb);
          }
          ++slot;
        }
      }
    }
    }  // valid
  }
}

__global__ void __launch_bounds__(256) k_xform_repair(uint8_t* __restrict__ dst,
                                                      const __grid_constant__ StrictP sp,
                                                      RepairList rl) {
  const unsigned long long n = min(*rl.count, rl.cap);
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n;
       i += 256ull * gridDim.x) {
    const unsigned long long it = rl.items[i];
    const uint32_t rgb = static_cast<uint32_t>(it & 0xffffffu);
    const int64_t gp = static_cast<int64_t>(it >> 24);
    const uint32_t out =
        strict_pixel(sp, ConstLut{&sp}, rgb & 255u, (rgb >> 8) & 255u, rgb >> 16);
    dst[3 * gp] = out & 255u;
    dst[3 * gp + 1] = (out >> 8) & 255u;
    dst[3 * gp + 2] = (out >> 16) & 255u;
  }
}

__global__ void __launch_bounds__(256) k_xform_strict(const uint8_t* __restrict__ src,
                                                      uint8_t* __restrict__ dst, int64_t npix,
                                                      const __grid_constant__ StrictP sp) {
  __shared__ double lut[3 * 256];
  for (int i = threadIdx.x; i < 3 * 256; i += 256) lut[i] = sp.lut[i >> 8][i & 255];
  __syncthreads();
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < npix; i += 256ll * gridDim.x) {
    const uint32_t r = src[3 * i], g = src[3 * i + 1], b = src[3 * i + 2];
    const uint32_t out = strict_pixel(sp, SmemLut{lut}, r, g, b);
    dst[3 * i] = out & 255u;
    dst[3 * i + 1] = (out >> 8) & 255u;
    dst[3 * i + 2] = (out >> 16) & 255u;
  }
}

// ------------------------------------------------------------------ launchers
static int g_sm_count = 0;
static int g_tma_blocks_per_sm = 0;

cudaError_t xform_setup_device() {
  if (g_sm_count) return cudaSuccess;
  int dev;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  for (auto fn : {k_xform_tma<0>, k_xform_tma<1>}) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kXformSmem);
    if (e != cudaSuccess) return e;
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_tma_blocks_per_sm, k_xform_tma<0>,
                                                    kThreads, kXformSmem);
  if (e != cudaSuccess) return e;
  if (g_tma_blocks_per_sm < 1) g_tma_blocks_per_sm = 1;
  return cudaSuccess;
}

cudaError_t launch_xform_tma(int mode, const uint8_t* src, uint8_t* dst, int64_t npix,
                             const FastP& fp, const StrictP& sp, unsigned long long* count,
                             unsigned long long* items, unsigned long long cap,
                             cudaStream_t st) {
  cudaError_t e = xform_setup_device();
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (npix + kTilePx - 1) / kTilePx;
  const int grid = static_cast<int>(min64(ntiles, (int64_t)g_sm_count * g_tma_blocks_per_sm));
  RepairList rl{count, items, cap};
  if (mode == 0)
    k_xform_tma<0><<<grid, kThreads, kXformSmem, st>>>(src, dst, npix, fp, sp, rl);
  else
    k_xform_tma<1><<<grid, kThreads, kXformSmem, st>>>(src, dst, npix, fp, sp, rl);
  return launched();
}

cudaError_t launch_xform_repair(uint8_t* dst, const StrictP& sp, unsigned long long* count,
                                unsigned long long* items, unsigned long long cap,
                                cudaStream_t st) {
  cudaError_t e = xform_setup_device();
  if (e != cudaSuccess) return e;
  RepairList rl{count, items, cap};
  k_xform_repair<<<g_sm_count * 2, 256, 0, st>>>(dst, sp, rl);
  return launched();
}

cudaError_t launch_xform_strict(const uint8_t* src, uint8_t* dst, int64_t npix,
                                const StrictP& sp, cudaStream_t st) {
  cudaError_t e = xform_setup_device();
  if (e != cudaSuccess) return e;
  if (npix <= 0) return cudaSuccess;
  const int64_t want = (npix + 255) / 256;
  const int grid = static_cast<int>(min64(want, (int64_t)g_sm_count * 16));
  k_xform_strict<<<grid, 256, 0, st>>>(src, dst, npix, sp);
  return launched();
}

int xform_tile_pixels() { return kTilePx; }

}  // namespace spcn
