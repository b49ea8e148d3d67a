// stats.cu — whole-slide ("global") per-stain 99th percentile (K2/K3).
//
// Extension of the reference's stain_stats (src/normalize.py:58-100 with
// percentile src/order_stats.py:11-36), which pools the densities of the
// <= 100 k sampled non-white pixels (src/pipeline.py:226,238).  Global mode
// pools the densities of EVERY non-white pixel
// (non-white = not all channels > white threshold, src/pipeline.py:176) of the
// slide, coded with the fitted basis and code_lam exactly as code_densities
// (src/stain_sep.py:168-201) would.  The result is the same order statistic
// the reference's percentile would return on those fp64 densities:
//
//   k_stats_hist    pass over the slide: fp32 densities (fast_density) binned
//                   into a 2 x nbins histogram window of float keys + counts
//                   (non-white pixels, keys below the window).  Run twice: a
//                   coarse level over all keys, then a fine level around the
//                   bins holding the requested ranks.  Approximate by design:
//                   it only places the final window.
//   k_stats_refine  pass over the slide: each density is classified against
//                   the final window [a, b) with its analytic fp32 error bound
//                   (params.cuh density_error_coeffs); only densities that may
//                   lie in the window are recomputed in fp64 in the reference's
//                   operation order (strict_nnls) — once per colour per CTA —
//                   counted exactly, and the in-window values listed as
//                   (value, pixel count) pairs.  The host checks that the ranks
//                   fall inside the window and selects them exactly.
//
// Multi-GPU: histograms and counts are summed across ranks (NCCL all-reduce,
// SURVEY §8(e)); the candidate lists are all-gathered.
#include "launch_count.h"
#include "params.cuh"
#include "recolor.cuh"
#include "spcn_device.cuh"
#include "stats.h"

namespace spcn {

constexpr int kStThreads = 512;
constexpr int kStRep = 16;
constexpr int kStBins = 8192;
constexpr size_t kStSmemHist = LutLayout<kStRep>::kBytes + 2 * kStBins * sizeof(uint32_t);

__device__ __forceinline__ uint32_t st_byte(const uint32_t* w, int idx) {
  return (w[idx >> 2] >> (8 * (idx & 3))) & 0xffu;
}

// 16 pixels of a lane: non-white flags (bit k = pixel k) and fp32 densities.
__device__ __forceinline__ uint32_t st_block(const StatsArgs& a, const uint8_t* lut,
                                             const uint32_t* lc, const uint32_t* w, float* h0,
                                             float* h1, float* T) {
  uint32_t nonwhite = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t r = st_byte(w, 3 * k), g = st_byte(w, 3 * k + 1), b = st_byte(w, 3 * k + 2);
    if (!(r > a.white && g > a.white && b > a.white)) nonwhite |= 1u << k;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int ia = 6 * q, ib = 6 * q + 3;
    const float2 v0 = make_float2(od_lookup(lut, w, ia, lc[0]), od_lookup(lut, w, ib, lc[0]));
    const float2 v1 = make_float2(od_lookup(lut, w, ia + 1, lc[1]), od_lookup(lut, w, ib + 1, lc[1]));
    const float2 v2 = make_float2(od_lookup(lut, w, ia + 2, lc[2]), od_lookup(lut, w, ib + 2, lc[2]));
    const FastDensity d = fast_density(a.fs, v0, v1, v2);
    h0[2 * q] = 0.5f * d.h0x2.x;
    h0[2 * q + 1] = 0.5f * d.h0x2.y;
    h1[2 * q] = 0.5f * d.h1x2.x;
    h1[2 * q + 1] = 0.5f * d.h1x2.y;
    T[2 * q] = d.T.x;
    T[2 * q + 1] = d.T.y;
  }
  return nonwhite;
}

__device__ __forceinline__ void st_load(const uint8_t* src, int64_t blk, uint32_t* w) {
  const uint4* q = reinterpret_cast<const uint4*>(src + 48 * blk);
  const uint4 q0 = __ldcs(q), q1 = __ldcs(q + 1), q2 = __ldcs(q + 2);
  w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w;
  w[4] = q1.x; w[5] = q1.y; w[6] = q1.z; w[7] = q1.w;
  w[8] = q2.x; w[9] = q2.y; w[10] = q2.z; w[11] = q2.w;
}

// tail pixels (npix % 16) as a partial block: missing pixels read as white
__device__ __forceinline__ void st_load_tail(const uint8_t* src, int64_t blk, int64_t npix,
                                             uint32_t* w) {
  for (int t = 0; t < 12; ++t) w[t] = 0xffffffffu;
  const int64_t p0 = 16 * blk;
  for (int k = 0; k < 16 && p0 + k < npix; ++k)
    for (int c = 0; c < 3; ++c) {
      const int idx = 3 * k + c;
      const uint32_t byte = src[3 * (p0 + k) + c];
      w[idx >> 2] = (w[idx >> 2] & ~(0xffu << (8 * (idx & 3)))) | (byte << (8 * (idx & 3)));
    }
}

__global__ void __launch_bounds__(kStThreads, 1)
    k_stats_hist(const uint8_t* __restrict__ src, int64_t npix, const __grid_constant__ StatsArgs a,
                 unsigned long long* __restrict__ hist, unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint8_t* lut = smem;
  uint32_t* sh = reinterpret_cast<uint32_t*>(smem + LutLayout<kStRep>::kBytes);
  LutLayout<kStRep>::fill(smem, &a.lut[0][0], threadIdx.x, kStThreads);
  for (int i = threadIdx.x; i < 2 * kStBins; i += kStThreads) sh[i] = 0;
  __syncthreads();
  uint32_t lc[3];
  LutLayout<kStRep>::lane_consts(threadIdx.x & 31, lc);
  unsigned long long nonwhite = 0, below[2] = {0, 0}, zero[2] = {0, 0};
  const int64_t nblk = (npix + 15) / 16, full = npix / 16;
  const int64_t stride = (int64_t)gridDim.x * kStThreads;
  uint32_t nxt[12];   // software prefetch: the next block is in flight while this one computes
  int64_t blk = blockIdx.x * (int64_t)kStThreads + threadIdx.x;
  if (blk < nblk) {
    if (blk < full) st_load(src, blk, nxt); else st_load_tail(src, blk, npix, nxt);
  }
  for (; blk < nblk; blk += stride) {
    uint32_t w[12];
#pragma unroll
    for (int t = 0; t < 12; ++t) w[t] = nxt[t];
    if (blk + stride < nblk) {
      if (blk + stride < full) st_load(src, blk + stride, nxt);
      else st_load_tail(src, blk + stride, npix, nxt);
    }
    float h0[16], h1[16], T[16];
    const uint32_t nw = st_block(a, lut, lc, w, h0, h1, T);
    nonwhite += __popc(nw);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (!((nw >> k) & 1u)) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint32_t key = __float_as_uint(j ? h1[k] : h0[k]);
        if (key == 0u && a.base[j] == 0u) { ++zero[j]; continue; }   // h = 0: bin 0, no atomics
        if (key < a.base[j]) { ++below[j]; continue; }
        const uint32_t d = (key - a.base[j]) >> a.shift[j];
        if (d < (uint32_t)a.nbins) hist_add_agg(sh + j * kStBins, d);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < a.nbins; i += kStThreads)
    for (int j = 0; j < 2; ++j) {
      uint32_t c = sh[j * kStBins + i];
      if (c) atomicAdd(&hist[j * a.nbins + i], (unsigned long long)c);
    }
  // zeros belong to bin 0 of a window starting at key 0
  for (int off = 16; off; off >>= 1) {
    nonwhite += __shfl_xor_sync(0xffffffffu, nonwhite, off);
    for (int j = 0; j < 2; ++j) {
      below[j] += __shfl_xor_sync(0xffffffffu, below[j], off);
      zero[j] += __shfl_xor_sync(0xffffffffu, zero[j], off);
    }
  }
  if ((threadIdx.x & 31) == 0) {
    if (nonwhite) atomicAdd(&counts[0], nonwhite);
    for (int j = 0; j < 2; ++j) {
      if (below[j]) atomicAdd(&counts[1 + j], below[j]);
      if (zero[j]) atomicAdd(&hist[j * a.nbins], zero[j]);
    }
  }
}

// Per-CTA colour cache of the refine pass: a density is a function of the
// pixel's RGB only, and the pixels that can fall in the narrow window share
// few colours, so each CTA evaluates a colour in fp64 once and keeps in-window
// pixel counts per colour; at the end it lists (value, count) pairs.
constexpr int kSlots = 2048;
constexpr uint32_t kEmpty = 0xffffffffu;
struct ColourSlot {
  uint32_t key;        // rgb, or kEmpty
  uint32_t ready;      // x valid
  uint32_t cnt[2];     // in-window pixels per stain
  double x[2];         // exact densities
};
constexpr size_t kStSmemRefine =
    LutLayout<kStRep>::kBytes + 3 * 256 * sizeof(double) + kSlots * sizeof(ColourSlot);

__device__ __forceinline__ uint32_t colour_hash(uint32_t rgb) {
  return (rgb * 2654435761u) >> (32 - 11);
}

__global__ void __launch_bounds__(kStThreads, 1)
    k_stats_refine(const uint8_t* __restrict__ src, int64_t npix,
                   const __grid_constant__ StatsArgs a, const __grid_constant__ StrictP sp,
                   unsigned long long* __restrict__ counts, double* __restrict__ cand,
                   unsigned long long* __restrict__ wcnt, unsigned long long cap) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint8_t* lut = smem;
  double* dlut = reinterpret_cast<double*>(smem + LutLayout<kStRep>::kBytes);
  ColourSlot* tab = reinterpret_cast<ColourSlot*>(smem + LutLayout<kStRep>::kBytes +
                                                  3 * 256 * sizeof(double));
  LutLayout<kStRep>::fill(smem, &a.lut[0][0], threadIdx.x, kStThreads);
  for (int i = threadIdx.x; i < 3 * 256; i += kStThreads) dlut[i] = sp.lut[i >> 8][i & 255];
  for (int i = threadIdx.x; i < kSlots; i += kStThreads) {
    tab[i].key = kEmpty;
    tab[i].ready = 0;
    tab[i].cnt[0] = tab[i].cnt[1] = 0;
  }
  __syncthreads();
  uint32_t lc[3];
  LutLayout<kStRep>::lane_consts(threadIdx.x & 31, lc);
  const NnlsGram G = gram_of(sp);
  unsigned long long below[2] = {0, 0}, exact_evals = 0;
  const int64_t nblk = (npix + 15) / 16, full = npix / 16;
  auto list = [&](int j, double x, unsigned long long c) {   // one (value, count) entry
    atomicAdd(&counts[2 + j], c);
    const unsigned long long idx = atomicAdd(&counts[5 + j], 1ull);
    if (idx < cap) {
      cand[j * cap + idx] = x;
      wcnt[j * cap + idx] = c;
    }
  };
  const int64_t stride = (int64_t)gridDim.x * kStThreads;
  uint32_t nxt[12];   // software prefetch: the next block is in flight while this one computes
  int64_t blk = blockIdx.x * (int64_t)kStThreads + threadIdx.x;
  if (blk < nblk) {
    if (blk < full) st_load(src, blk, nxt); else st_load_tail(src, blk, npix, nxt);
  }
  for (; blk < nblk; blk += stride) {
    uint32_t w[12];
#pragma unroll
    for (int t = 0; t < 12; ++t) w[t] = nxt[t];
    if (blk + stride < nblk) {
      if (blk + stride < full) st_load(src, blk + stride, nxt);
      else st_load_tail(src, blk + stride, npix, nxt);
    }
    float h0[16], h1[16], T[16];
    const uint32_t nw = st_block(a, lut, lc, w, h0, h1, T);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (!((nw >> k) & 1u)) continue;
      uint32_t need = 0;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const double h = (double)(j ? h1[k] : h0[k]);
        const double eps = (double)a.coef[j] * (double)T[k] * (1.0 + 1e-6) + 1e-30;
        if (h + eps < a.a[j]) ++below[j];          // surely below the window
        else if (!(h - eps >= a.b[j])) need |= 1u << j;   // may lie in [a, b)
      }
      if (!need) continue;
      const uint32_t rgb = st_byte(w, 3 * k) | (st_byte(w, 3 * k + 1) << 8) |
                           (st_byte(w, 3 * k + 2) << 16);
      // colour cache: find or claim a slot; a slot claimed but not yet filled
      // by another thread is simply recomputed here (no waiting)
      int slot = -1;
      double x[2];
      bool have = false;
      uint32_t s = colour_hash(rgb);
      for (int probe = 0; probe < 8; ++probe, s = (s + 1) & (kSlots - 1)) {
        uint32_t key = *(volatile uint32_t*)&tab[s].key;
        if (key == kEmpty) key = atomicCAS(&tab[s].key, kEmpty, rgb) == kEmpty ? kEmpty - 1 : tab[s].key;
        if (key == kEmpty - 1) {                   // claimed by us: fill it below
          slot = (int)s;
          break;
        }
        if (key == rgb) {
          slot = (int)s;
          if (*(volatile uint32_t*)&tab[s].ready) {
            x[0] = tab[s].x[0];
            x[1] = tab[s].x[1];
            have = true;
          }
          break;
        }
      }
      if (!have) {
        ++exact_evals;
        const double v0 = dlut[rgb & 255u], v1 = dlut[256 + ((rgb >> 8) & 255u)],
                     v2 = dlut[512 + (rgb >> 16)];
        const double b0 = strict_dot3(sp.ws[0][0], sp.ws[1][0], sp.ws[2][0], v0, v1, v2);
        const double b1 = strict_dot3(sp.ws[0][1], sp.ws[1][1], sp.ws[2][1], v0, v1, v2);
        strict_nnls(b0, b1, G, sp.lam, sp.max_sweeps, sp.tol, x[0], x[1]);
        if (slot >= 0 && tab[slot].key == rgb && !tab[slot].ready) {
          tab[slot].x[0] = x[0];
          tab[slot].x[1] = x[1];
          __threadfence_block();
          atomicExch(&tab[slot].ready, 1u);
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (!((need >> j) & 1u)) continue;
        if (x[j] < a.a[j]) {
          ++below[j];
        } else if (x[j] < a.b[j]) {
          if (slot >= 0) atomicAdd(&tab[slot].cnt[j], 1u);
          else list(j, x[j], 1ull);                // cache full: list the pixel itself
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kSlots; i += kStThreads)
    for (int j = 0; j < 2; ++j)
      if (tab[i].cnt[j]) {
        // counted only by threads that knew the value; its owner set it
        // (and `ready`) before this barrier
        list(j, tab[i].x[j], tab[i].cnt[j]);
      }
  for (int off = 16; off; off >>= 1) {
    exact_evals += __shfl_xor_sync(0xffffffffu, exact_evals, off);
    for (int j = 0; j < 2; ++j) below[j] += __shfl_xor_sync(0xffffffffu, below[j], off);
  }
  if ((threadIdx.x & 31) == 0) {
    for (int j = 0; j < 2; ++j)
      if (below[j]) atomicAdd(&counts[j], below[j]);
    if (exact_evals) atomicAdd(&counts[4], exact_evals);
  }
}

static int st_grid() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 148;
  }
  return sms;
}

cudaError_t launch_stats_hist(const uint8_t* src, int64_t npix, const StatsArgs& a,
                              unsigned long long* hist, unsigned long long* counts,
                              cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(k_stats_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)kStSmemHist);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (npix <= 0) return cudaSuccess;
  const int64_t nblk = (npix + 15) / 16;
  int64_t grid = (nblk + kStThreads - 1) / kStThreads;
  if (grid > st_grid()) grid = st_grid();
  k_stats_hist<<<(int)grid, kStThreads, kStSmemHist, st>>>(src, npix, a, hist, counts);
  return launched();
}

cudaError_t launch_stats_refine(const uint8_t* src, int64_t npix, const StatsArgs& a,
                                const StrictP& sp, unsigned long long* counts, double* cand,
                                unsigned long long* wcnt, unsigned long long cap,
                                cudaStream_t st) {
  constexpr size_t smem = kStSmemRefine;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(k_stats_refine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (npix <= 0) return cudaSuccess;
  const int64_t nblk = (npix + 15) / 16;
  int64_t grid = (nblk + kStThreads - 1) / kStThreads;
  if (grid > st_grid()) grid = st_grid();
  k_stats_refine<<<(int)grid, kStThreads, smem, st>>>(src, npix, a, sp, counts, cand, wcnt, cap);
  return launched();
}

}  // namespace spcn
