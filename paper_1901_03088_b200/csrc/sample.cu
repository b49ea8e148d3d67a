// sample.cu — device side of the fit's pixel sampling (K4) and background
// estimate (K5).
//
// Reference: sample_pixels src/pipeline.py:128-200 and estimate_max_intensity
// src/optics.py:35-68.  The reference visits seeded random patches in order,
// keeps per channel the first `cap` values > thr in raster order (bright
// pools), and the first `target - collected` non-white pixels in raster order
// of each non-background patch.  The visit logic depends only on per-patch
// counts, so it runs in two data-parallel passes with a tiny host step
// between them:
//   k_sample_count   per-patch, per-4096-pixel-chunk counts (non-white and
//                    bright per channel) — integer work, exact;
//   (host)           replays the reference's visit loop on the counts;
//   k_sample_compact ordered compaction: block scan inside each chunk plus the
//                    prefix of earlier chunks gives every pixel its raster rank,
//                    so "first N in raster order" is reproduced exactly; the
//                    taken bright values go straight into 256-bin histograms.
//   k_i0_from_hist   exact 80th percentile of the bright pools from the counts.
#include "launch_count.h"
#include "spcn_device.cuh"
#include "spcn.h"
#include "sample.h"

namespace spcn {

constexpr int kChunk = SPCN_SAMPLE_CHUNK;     // raster pixels per chunk (4096)
constexpr int kSThreads = 256;
constexpr int kPerThread = kChunk / kSThreads; // 16

// The kPerThread raster-consecutive pixels r0.. of a patch as their 48 RGB
// bytes packed into 12 words (pixel j = bytes 3j..3j+2); returns how many of
// them exist (a prefix: the run ends at the patch's last pixel).  One division
// per thread; a run inside one row at a 16-byte-aligned address is three
// 16-byte loads, anything else pixel by pixel with an incremental (row, col)
// and packed with byte permutes.
__device__ __forceinline__ int patch_run(const uint8_t* img, const spcn_patch& p, int64_t r0,
                                         int64_t npx, uint32_t (&w)[12]) {
  static_assert(kPerThread == 16, "16 px = 48 bytes = 12 words");
  int64_t row, col;
  if (r0 <= 0xffffffffll) {   // 32-bit division (the common case)
    const uint32_t r = (uint32_t)r0 / (uint32_t)p.width;
    row = r;
    col = (int64_t)((uint32_t)r0 - r * (uint32_t)p.width);
  } else {
    row = r0 / p.width;
    col = r0 - row * p.width;
  }
  const uint8_t* q = img + 3 * (p.base + row * p.row_stride + col);
  if (r0 + kPerThread <= npx && col + kPerThread <= p.width &&
      (reinterpret_cast<uintptr_t>(q) & 15) == 0) {
    const uint4* v = reinterpret_cast<const uint4*>(q);
    const uint4 a = __ldg(v), b = __ldg(v + 1), c = __ldg(v + 2);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    w[8] = c.x; w[9] = c.y; w[10] = c.z; w[11] = c.w;
    return kPerThread;
  }
  uint32_t rgb[kPerThread];
  const int nv = (int)min((int64_t)kPerThread, npx - r0);
#pragma unroll
  for (int j = 0; j < kPerThread; ++j) {
    rgb[j] = 0;
    if (j < nv) {
      const uint8_t* t = img + 3 * (p.base + row * p.row_stride + col);
      rgb[j] = t[0] | (t[1] << 8) | (t[2] << 16);
      if (++col == p.width) {
        col = 0;
        ++row;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 12; ++k) {   // word k = bytes 4k..4k+3 = pixel 4k/3 from byte 4k%3 on
    const int j = (4 * k) / 3, o = (4 * k) % 3;
    w[k] = __byte_perm(rgb[j], rgb[j + 1], o == 0 ? 0x4210 : o == 1 ? 0x5421 : 0x6542);
  }
  return nv;
}

// Byte-parallel "value > thr" (SWAR): 0x80 in every byte of x above thr.
// thr is clamped to [-1, 255] (same predicate on 8-bit values); per byte the
// sum stays below 256, so no carry crosses a byte.  HI (thr >= 128):
// x > thr  <=>  x >= 128 and (x & 127) > thr - 128.
__host__ __device__ __forceinline__ int clamp_thr(int thr) { return thr < -1 ? -1 : thr > 255 ? 255 : thr; }
__device__ __forceinline__ uint32_t gt_k(int thr) {
  thr = clamp_thr(thr);
  return (uint32_t)(thr >= 128 ? 255 - thr : 127 - thr) * 0x01010101u;
}
template <bool HI>
__device__ __forceinline__ uint32_t gt80(uint32_t x, uint32_t k) {
  const uint32_t s = (x & 0x7f7f7f7fu) + k;
  return (HI ? (x & s) : (x | s)) & 0x80808080u;
}

// Flags of a thread's 16 pixels: f[g][c] (c = R, G, B: "> thr"; c = 3:
// "non-white"), bit 7 of byte i = pixel 4g+i.  Words 3g..3g+2 hold
// R0 G0 B0 R1 | G1 B1 R2 G2 | B2 R3 G3 B3; missing pixels (j >= nv) flag 0.
template <bool HI>
__device__ __forceinline__ void run_flags(const uint32_t (&w)[12], int nv, uint32_t k,
                                          uint32_t (&f)[4][4]) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const uint32_t m0 = gt80<HI>(w[3 * g], k), m1 = gt80<HI>(w[3 * g + 1], k),
                   m2 = gt80<HI>(w[3 * g + 2], k);
    f[g][0] = __byte_perm(__byte_perm(m0, m1, 0x0630), m2, 0x5210);   // R0 R1 R2 R3
    f[g][1] = __byte_perm(__byte_perm(m0, m1, 0x0741), m2, 0x6210);   // G
    f[g][2] = __byte_perm(__byte_perm(m0, m1, 0x0052), m2, 0x7410);   // B
  }
  if (nv >= kPerThread) {
#pragma unroll
    for (int g = 0; g < 4; ++g) f[g][3] = 0x80808080u ^ (f[g][0] & f[g][1] & f[g][2]);
  } else {
    const uint32_t vbits = (1u << max(nv, 0)) - 1u;
#pragma unroll
    for (int g = 0; g < 4; ++g) {   // 4 bits -> bit 7 of 4 bytes
      const uint32_t vb = (((vbits >> (4 * g)) & 15u) * 0x10204080u) & 0x80808080u;
      f[g][0] &= vb; f[g][1] &= vb; f[g][2] &= vb;
      f[g][3] = vb ^ (f[g][0] & f[g][1] & f[g][2]);
    }
  }
}

__device__ __forceinline__ uint32_t pixel_of(const uint32_t (&w)[12], int j) {
  const int i = 3 * j, k = i >> 2, o = i & 3;   // bytes i..i+2, from word k at offset o
  return __byte_perm(w[k], w[k < 11 ? k + 1 : 11], o == 0 ? 0x210 : o == 1 ? 0x321 : o == 2 ? 0x432 : 0x543);
}

template <bool HI>
__global__ void __launch_bounds__(kSThreads) k_sample_count(const uint8_t* __restrict__ img,
                                                            const spcn_patch* __restrict__ patches,
                                                            int max_chunks, int thr,
                                                            int32_t* __restrict__ counts) {
  const int k = blockIdx.x, pi = blockIdx.y;
  const spcn_patch p = patches[pi];
  const int64_t npx = (int64_t)p.width * p.height;
  const int64_t r0 = (int64_t)k * kChunk + threadIdx.x * kPerThread;
  unsigned c[4] = {0, 0, 0, 0};  // non-white, bright R, G, B
  if (r0 < npx) {
    uint32_t w[12], f[4][4];
    const int nv = patch_run(img, p, r0, npx, w);
    run_flags<HI>(w, nv, gt_k(thr), f);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      c[0] += __popc(f[g][3]);
      c[1] += __popc(f[g][0]);
      c[2] += __popc(f[g][1]);
      c[3] += __popc(f[g][2]);
    }
  }
  __shared__ unsigned scratch[kSThreads / 32][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 4; ++q) c[q] = __reduce_add_sync(0xffffffffu, c[q]);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 4; ++q) scratch[warp][q] = c[q];
  __syncthreads();
  if (threadIdx.x < 4) {
    unsigned v = 0;
#pragma unroll
    for (int i = 0; i < kSThreads / 32; ++i) v += scratch[i][threadIdx.x];
    counts[((int64_t)pi * max_chunks + k) * 4 + threadIdx.x] = (int32_t)v;
  }
}

// The ordered take of one thread's 16 pixels from its flags (already cut to
// what the pools take): STAGE puts the taken non-white pixels at their rank
// in the chunk's stage (the others in a per-lane dump slot); every taken
// bright value goes into its channel's 256-bin histogram.
// Shared-memory increment without a branch: an untaken value goes to the
// lane's own dump word (hist[768 + lane]) instead of being predicated off.
__device__ __forceinline__ void hist_inc(uint32_t addr) {
  asm volatile("red.shared.add.u32 [%0], 1;" :: "r"(addr) : "memory");
}

template <bool STAGE>
__device__ __forceinline__ void compact_run(const uint32_t (&w)[12], const uint32_t (&f)[4][4],
                                            int rank0, uint32_t* stage, int dump, int* hist,
                                            const bool (&act)[3]) {
  if (STAGE) {
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
      const int g = j >> 2, sh = 8 * (j & 3) + 7;
      const int nwf = (f[g][3] >> sh) & 1;
      stage[nwf ? rank0 : dump] = pixel_of(w, j);
      rank0 += nwf;
    }
  }
  const uint32_t hbase = (uint32_t)__cvta_generic_to_shared(hist);
  const uint32_t hdump = hbase + 4 * (3 * 256 + (threadIdx.x & 31));
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    if (!act[c]) continue;   // block-uniform: the channel's pool is full
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
      const int g = j >> 2, sh = 8 * (j & 3) + 7;
      const int b = 3 * j + c;   // byte of channel c of pixel j
      const uint32_t a = hbase + 4 * (256 * c + __byte_perm(w[b >> 2], 0, 0x4440 | (b & 3)));
      hist_inc(f[g][c] & (1u << sh) ? a : hdump);
    }
  }
}

// Keep only the first `m` set flags (raster order) of f[.][q].
__device__ __forceinline__ void limit_flags(uint32_t (&f)[4][4], int q, int m) {
#pragma unroll
  for (int g = 0; g < 4; ++g)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t bit = 0x80u << (8 * i);
      if (f[g][q] & bit) {
        if (m > 0) --m;
        else f[g][q] &= ~bit;
      }
    }
}

// CPB consecutive chunks of one patch per CTA: the histograms are zeroed and
// flushed once and the chunk prefix carried from chunk to chunk.  Many-patch
// launches (batches of tiles) use 8; a slide's few visited patches need only
// their first chunks, which then run in parallel with 1.
constexpr int kCPBMany = 8;
constexpr int kManyPatches = 1024;

template <bool HI, int kCPB>
__global__ void __launch_bounds__(kSThreads) k_sample_compact(
    const uint8_t* __restrict__ img, const spcn_patch* __restrict__ patches, int max_chunks,
    int thr, const int32_t* __restrict__ counts, const spcn_patch_take* __restrict__ takes,
    uint8_t* __restrict__ out_px, int32_t* __restrict__ bright_hist) {
  const int k0 = blockIdx.x * kCPB, pi = blockIdx.y;
  const spcn_patch p = patches[pi];
  const spcn_patch_take tk = takes[pi];
  const int64_t npx = (int64_t)p.width * p.height;
  if ((int64_t)k0 * kChunk >= npx) return;
  __shared__ int s_pre[4];
  __shared__ unsigned scratch[kSThreads / 32][4];
  __shared__ int s_hist[3 * 256 + 32];   // + one dump word per lane
  // per-warp totals of the packed counters (non-white | R << 16, G | B << 16),
  // then their exclusive prefix over warps; s_tot: the chunk's totals
  __shared__ __align__(8) uint32_t s_wsum[kSThreads / 32][2];
  __shared__ __align__(8) uint32_t s_tot[2];
  // the chunk's taken non-white pixels as words in rank order (+ one dump
  // slot per lane for the pixels that are not taken), then written out as
  // one contiguous 3-byte-per-pixel run with coalesced word stores
  __shared__ __align__(16) uint32_t s_stage[kChunk + 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // prefix over earlier chunks of this patch
  unsigned pre[4] = {0, 0, 0, 0};
  for (int j = threadIdx.x; j < k0; j += kSThreads) {
    const int32_t* c = counts + ((int64_t)pi * max_chunks + j) * 4;
    pre[0] += c[0]; pre[1] += c[1]; pre[2] += c[2]; pre[3] += c[3];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) pre[q] = __reduce_add_sync(0xffffffffu, pre[q]);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 4; ++q) scratch[warp][q] = pre[q];
  for (int i = threadIdx.x; i < 3 * 256; i += kSThreads) s_hist[i] = 0;
  __syncthreads();
  if (threadIdx.x < 4) {
    unsigned v = 0;
#pragma unroll
    for (int i = 0; i < kSThreads / 32; ++i) v += scratch[i][threadIdx.x];
    s_pre[threadIdx.x] = (int)v;
  }
  __syncthreads();
  int spre[4] = {s_pre[0], s_pre[1], s_pre[2], s_pre[3]};
  const int lim[4] = {(int)min(tk.take_nonwhite, (int64_t)INT32_MAX), tk.take_bright[0],
                      tk.take_bright[1], tk.take_bright[2]};
  for (int k = k0; k < k0 + kCPB && (int64_t)k * kChunk < npx; ++k) {
    if (!(spre[0] < lim[0] || spre[1] < lim[1] || spre[2] < lim[2] || spre[3] < lim[3]))
      break;  // uniform across the block: every pool is full before this chunk

    const int64_t r0 = (int64_t)k * kChunk + threadIdx.x * kPerThread;
    uint32_t w[12];
    int nv = 0;
    if (r0 < npx) {
      nv = patch_run(img, p, r0, npx, w);
    } else {
#pragma unroll
      for (int i = 0; i < 12; ++i) w[i] = 0;
    }
    uint32_t f[4][4];
    run_flags<HI>(w, nv, gt_k(thr), f);
    uint32_t c01 = 0, c23 = 0;   // packed 16-bit counters: non-white | R << 16, G | B << 16
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      c01 += __popc(f[g][3]) | (__popc(f[g][0]) << 16);
      c23 += __popc(f[g][1]) | (__popc(f[g][2]) << 16);
    }
    // block exclusive scan of the packed counters (chunk totals <= 4096)
    uint32_t i01 = c01, i23 = c23;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y01 = __shfl_up_sync(0xffffffffu, i01, off);
      const uint32_t y23 = __shfl_up_sync(0xffffffffu, i23, off);
      if (lane >= off) {
        i01 += y01;
        i23 += y23;
      }
    }
    if (lane == 31) {
      s_wsum[warp][0] = i01;
      s_wsum[warp][1] = i23;
    }
    __syncthreads();
    if (warp == 0) {   // lane 2w + h: exclusive scan over the 8 warps
      static_assert(kSThreads / 32 * 2 <= 32, "one warp scans the per-warp totals");
      const bool on = lane < 2 * (kSThreads / 32);
      const uint32_t v = on ? (&s_wsum[0][0])[lane] : 0u;
      uint32_t x = v;
#pragma unroll
      for (int off = 2; off < 2 * (kSThreads / 32); off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      __syncwarp();
      if (on) (&s_wsum[0][0])[lane] = x - v;
      if (lane >= 2 * (kSThreads / 32) - 2 && on) s_tot[lane - (2 * (kSThreads / 32) - 2)] = x;
    }
    __syncthreads();
    const uint2 wp = *reinterpret_cast<const uint2*>(s_wsum[warp]);
    const uint2 tt = *reinterpret_cast<const uint2*>(s_tot);
    const uint32_t e01 = wp.x + i01 - c01, e23 = wp.y + i23 - c23;
    const int rank[4] = {spre[0] + (int)(e01 & 0xffffu), spre[1] + (int)(e01 >> 16),
                         spre[2] + (int)(e23 & 0xffffu), spre[3] + (int)(e23 >> 16)};
    const int tot[4] = {(int)(tt.x & 0xffffu), (int)(tt.x >> 16), (int)(tt.y & 0xffffu),
                        (int)(tt.y >> 16)};
#pragma unroll
    for (int q = 0; q < 4; ++q) {   // pool q takes all / none / the first part of the chunk
      const int fq = q == 0 ? 3 : q - 1;
      if (spre[q] >= lim[q]) {                        // block-uniform tests
#pragma unroll
        for (int g = 0; g < 4; ++g) f[g][fq] = 0;
      } else if (spre[q] + tot[q] > lim[q]) {
        limit_flags(f, fq, lim[q] - rank[q]);
      }
    }
    const int blk_r0 = spre[0];                 // the chunk's first non-white rank
    const bool act[3] = {spre[1] < lim[1], spre[2] < lim[2], spre[3] < lim[3]};
    if (spre[0] < lim[0])
      compact_run<true>(w, f, rank[0] - blk_r0, s_stage, kChunk + lane, s_hist, act);
    else
      compact_run<false>(w, f, 0, s_stage, kChunk + lane, s_hist, act);
    __syncthreads();
    {   // the staged run [blk_r0, min(take, blk_r0 + chunk non-white)) to the output
      const int64_t t1 = min((int64_t)tk.take_nonwhite, (int64_t)blk_r0 + tot[0]);
      const int nb = t1 > blk_r0 ? (int)(3 * (t1 - blk_r0)) : 0;
      uint8_t* dstb = out_px + 3 * (tk.out_base + blk_r0);
      const int head = min(nb, (int)((4u - (reinterpret_cast<uintptr_t>(dstb) & 3u)) & 3u));
      if (threadIdx.x < head) dstb[threadIdx.x] = s_stage[threadIdx.x / 3] >> (8 * (threadIdx.x % 3));
      const int nw = (nb - head) >> 2;
      uint32_t* dw = reinterpret_cast<uint32_t*>(dstb + head);
      for (int i = threadIdx.x; i < nw; i += kSThreads) {
        const int b = head + 4 * i, q = b / 3, o = b - 3 * q;   // run bytes b..b+3
        dw[i] = __byte_perm(s_stage[q], s_stage[q + 1], o == 0 ? 0x4210 : o == 1 ? 0x5421 : 0x6542);
      }
      const int tail0 = head + 4 * nw;
      if (threadIdx.x < nb - tail0) {
        const int b = tail0 + threadIdx.x;
        dstb[b] = s_stage[b / 3] >> (8 * (b % 3));
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) spre[q] += tot[q];
    __syncthreads();   // s_stage / s_wsum / s_tot are reused by the next chunk
  }
  int32_t* gh = bright_hist + (int64_t)tk.problem * 3 * 256;
  for (int i = threadIdx.x; i < 3 * 256; i += kSThreads) {
    const int v = s_hist[i];
    if (v) atomicAdd(&gh[i], v);
  }
}

// Exact 80th percentile of 8-bit pools from their 256-bin counts
// (percentile src/order_stats.py:27-36 on the expanded multiset).
// One warp per (problem, channel): 8 bins per lane, a warp prefix sum finds
// the bins holding ranks lo and hi (exact integer counting).
__global__ void k_i0_from_hist(const int32_t* __restrict__ hist, int nprob,
                               double* __restrict__ i0, int32_t* __restrict__ empty) {
  const int idx = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (idx >= nprob * 3) return;                       // whole warps
  const int32_t* h = hist + (int64_t)idx * 256 + lane * 8;
  int64_t c[8], tot = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    c[b] = h[b];
    tot += c[b];
  }
  int64_t incl = tot;
  for (int off = 1; off < 32; off <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  const int64_t n = __shfl_sync(0xffffffffu, incl, 31);
  if (n == 0) {
    if (lane == 0) {
      i0[idx] = 255.0;
      empty[idx] = 1;
    }
    return;
  }
  const double rank = __dmul_rn(80.0 / 100.0, (double)(n - 1));
  const int64_t lo = (int64_t)floor(rank), hi = (int64_t)ceil(rank);
  // the first value whose cumulative count exceeds the rank
  int lov = 256, hiv = 256;
  int64_t cum = incl - tot;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const int64_t before = cum;
    cum += c[b];
    if (before <= lo && cum > lo) lov = lane * 8 + b;
    if (before <= hi && cum > hi) hiv = lane * 8 + b;
  }
  for (int off = 16; off; off >>= 1) {
    lov = min(lov, __shfl_xor_sync(0xffffffffu, lov, off));
    hiv = min(hiv, __shfl_xor_sync(0xffffffffu, hiv, off));
  }
  if (lane == 0) {
    empty[idx] = 0;
    const double frac = __dsub_rn(rank, (double)lo);
    i0[idx] = __dadd_rn((double)lov, __dmul_rn(__dsub_rn((double)hiv, (double)lov), frac));
  }
}

// Per-problem OD tables ln(i0_c / clip(i, 1, i0_c)) (src/optics.py:92-94).
__global__ void k_od_tables(const double* __restrict__ i0, int nprob, double* __restrict__ lut) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nprob * 3 * 256) return;
  const int64_t pc = idx / 256;
  const int i = (int)(idx - pc * 256);
  const double a = i0[pc];
  double x = (double)i;
  x = x < 1.0 ? 1.0 : (x > a ? a : x);
  lut[idx] = log(__ddiv_rn(a, x));
}

// One-patch items (a batch of tiles smaller than a patch): the reference's
// visit rules (src/pipeline.py:156-184) reduce to per-item ones — take the
// first min(non-white, target) non-white pixels if the non-white count
// reaches the background cutoff, and the first min(bright, cap) bright
// values per channel — and the sample offsets are an exclusive scan of the
// takes.  One CTA: totals per item from the chunk counts, the rules, a
// running block scan, the take rows and the per-item non-white takes.
constexpr int kVS = 1024;

// item totals, one warp per item, parked in the item's 32-byte take row
__global__ void __launch_bounds__(256) k_visit_totals(const int32_t* __restrict__ counts, int n,
                                                      int chunks, int64_t* __restrict__ rows) {
  const int item = (int)((blockIdx.x * 256ll + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (item >= n) return;
  int64_t t[4] = {0, 0, 0, 0};
  for (int c = lane; c < chunks; c += 32)
    for (int q = 0; q < 4; ++q) t[q] += counts[((int64_t)item * chunks + c) * 4 + q];
  for (int q = 0; q < 4; ++q)
    for (int off = 16; off; off >>= 1) t[q] += __shfl_xor_sync(0xffffffffu, t[q], off);
  if (lane < 4) rows[4 * (int64_t)item + lane] = t[lane];
}

__global__ void __launch_bounds__(kVS) k_visit_single(const int32_t* __restrict__ counts, int n,
                                                      int chunks, double used_min, int64_t target,
                                                      int64_t cap, spcn_patch_take* __restrict__ takes,
                                                      int64_t* __restrict__ take_nw) {
  __shared__ int64_t s_scan[kVS];
  __shared__ int64_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += kVS) {
    const int i = i0 + threadIdx.x;
    int64_t tot[4] = {0, 0, 0, 0};
    if (i < n)
      for (int q = 0; q < 4; ++q) tot[q] = reinterpret_cast<const int64_t*>(takes)[4 * (int64_t)i + q];
    const bool used = (double)tot[0] >= used_min;
    const int64_t nw = (i < n && used) ? (tot[0] < target ? tot[0] : target) : 0;
    s_scan[threadIdx.x] = nw;
    __syncthreads();
    for (int off = 1; off < kVS; off <<= 1) {           // inclusive block scan
      const int64_t y = threadIdx.x >= off ? s_scan[threadIdx.x - off] : 0;
      __syncthreads();
      s_scan[threadIdx.x] += y;
      __syncthreads();
    }
    const int64_t base = s_carry + s_scan[threadIdx.x] - nw;
    if (i < n) {
      spcn_patch_take t;
      t.take_nonwhite = nw;
      t.out_base = base;
      for (int q = 0; q < 3; ++q) t.take_bright[q] = (int32_t)(tot[1 + q] < cap ? tot[1 + q] : cap);
      t.problem = i;
      takes[i] = t;
      take_nw[i] = nw;
    }
    __syncthreads();
    if (threadIdx.x == kVS - 1) s_carry += s_scan[kVS - 1];
    __syncthreads();
  }
}

cudaError_t launch_visit_single(const int32_t* counts, int n, int chunks, double used_min,
                                int64_t target, int64_t cap, spcn_patch_take* takes,
                                int64_t* take_nw, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_visit_totals<<<(unsigned)((n * 32ll + 255) / 256), 256, 0, st>>>(
      counts, n, chunks, reinterpret_cast<int64_t*>(takes));
  cudaError_t e = launched();
  if (e != cudaSuccess) return e;
  k_visit_single<<<1, kVS, 0, st>>>(counts, n, chunks, used_min, target, cap, takes, take_nw);
  return launched();
}

cudaError_t launch_sample_count(const uint8_t* img, const spcn_patch* patches, int npatches,
                                int max_chunks, int thr, int32_t* counts, cudaStream_t st) {
  if (npatches <= 0 || max_chunks <= 0) return cudaSuccess;
  for (int y0 = 0; y0 < npatches; y0 += kMaxGridY) {   // gridDim.y <= 65535
    const int ny = npatches - y0 < kMaxGridY ? npatches - y0 : kMaxGridY;
    auto kern = clamp_thr(thr) >= 128 ? k_sample_count<true> : k_sample_count<false>;
    kern<<<dim3(max_chunks, ny), kSThreads, 0, st>>>(
        img, patches + y0, max_chunks, thr, counts + (int64_t)y0 * max_chunks * 4);
    const cudaError_t e = launched();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_sample_compact(const uint8_t* img, const spcn_patch* patches, int npatches,
                                  int max_chunks, int thr, const int32_t* counts,
                                  const spcn_patch_take* takes, uint8_t* out_px,
                                  int32_t* bright_hist, cudaStream_t st) {
  if (npatches <= 0 || max_chunks <= 0) return cudaSuccess;
  for (int y0 = 0; y0 < npatches; y0 += kMaxGridY) {   // gridDim.y <= 65535
    const int ny = npatches - y0 < kMaxGridY ? npatches - y0 : kMaxGridY;
    const bool hi = clamp_thr(thr) >= 128, many = npatches >= kManyPatches;
    auto kern = hi ? (many ? k_sample_compact<true, kCPBMany> : k_sample_compact<true, 1>)
                   : (many ? k_sample_compact<false, kCPBMany> : k_sample_compact<false, 1>);
    const int cpb = many ? kCPBMany : 1;
    kern<<<dim3((max_chunks + cpb - 1) / cpb, ny), kSThreads, 0, st>>>(
        img, patches + y0, max_chunks, thr, counts + (int64_t)y0 * max_chunks * 4, takes + y0,
        out_px, bright_hist);
    const cudaError_t e = launched();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_i0_from_hist(const int32_t* hist, int nprob, double* i0, int32_t* empty,
                                cudaStream_t st) {
  if (nprob <= 0) return cudaSuccess;
  k_i0_from_hist<<<(nprob * 3 + 3) / 4, 128, 0, st>>>(hist, nprob, i0, empty);   // warp per pool
  return launched();
}

cudaError_t launch_od_tables(const double* i0, int nprob, double* lut, cudaStream_t st) {
  if (nprob <= 0) return cudaSuccess;
  const int64_t n = (int64_t)nprob * 3 * 256;
  k_od_tables<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(i0, nprob, lut);
  return launched();
}

// ---------------------------------------------------------------------------
// k_visit: the reference's visit loop (src/pipeline.py:156-184) over one batch
// of candidates, on the device so the sampler needs no host round trip in the
// common case.  Block-wide: chunk totals of every candidate, then thread 0
// replays the sequential decisions exactly like pipeline._visit.
__global__ void __launch_bounds__(256) k_visit(const int32_t* __restrict__ counts, int n,
                                               int max_chunks, int k0,
                                               const int32_t* __restrict__ dims,
                                               spcn_visit_plan plan, int64_t* __restrict__ state,
                                               spcn_patch_take* __restrict__ takes,
                                               int64_t* __restrict__ offsets) {
  extern __shared__ int64_t tot[];   // n x 4 totals
  for (int i = threadIdx.x; i < 4 * n; i += blockDim.x) {
    const int k = i >> 2, q = i & 3;
    int64_t t = 0;
    for (int c = 0; c < max_chunks; ++c) t += counts[(k * max_chunks + c) * 4 + q];
    tot[i] = t;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int64_t collected = state[0], visited = state[1], used = state[2];
  int64_t bright_n[3] = {state[3], state[4], state[5]};
  int64_t stopped = state[6];
  const int64_t limit = 10 * (int64_t)plan.max_patches;
  const double min_frac = 1.0 - plan.background_cutoff;
  int k = 0;
  for (; k < n; ++k) {
    spcn_patch_take& tk = takes[k];
    tk.take_nonwhite = 0;
    tk.out_base = 0;
    tk.take_bright[0] = tk.take_bright[1] = tk.take_bright[2] = 0;
    tk.problem = 0;
    if (stopped) continue;
    if (visited >= limit || used >= plan.max_patches || collected >= plan.target_pixels) {
      stopped = 1;
      continue;
    }
    const int64_t nw = tot[4 * k];
    const int64_t npx = (int64_t)dims[2 * k] * dims[2 * k + 1];
    ++visited;
    for (int c = 0; c < 3; ++c) {
      if (bright_n[c] < plan.sample_cap) {
        const int64_t room = plan.sample_cap - bright_n[c];
        const int64_t t = tot[4 * k + 1 + c] < room ? tot[4 * k + 1 + c] : room;
        tk.take_bright[c] = (int32_t)t;
        bright_n[c] += t;
      }
    }
    if ((double)nw < min_frac * (double)npx) continue;   // background patch
    ++used;
    const int64_t room = plan.target_pixels - collected;
    const int64_t take = nw < room ? nw : room;
    tk.take_nonwhite = take;
    tk.out_base = collected;
    collected += take;
  }
  state[0] = collected;
  state[1] = visited;
  state[2] = used;
  for (int c = 0; c < 3; ++c) state[3 + c] = bright_n[c];
  state[6] = stopped;
  state[7] = (!stopped && k0 + n < plan.ncand) ? 1 : 0;   // need more candidates
  offsets[0] = 0;
  offsets[1] = collected;
}

cudaError_t launch_visit(const int32_t* counts, int n, int max_chunks, int k0, const int32_t* dims,
                         const spcn_visit_plan& plan, int64_t* state, spcn_patch_take* takes,
                         int64_t* offsets, cudaStream_t st) {
  const size_t smem = 4 * (size_t)n * sizeof(int64_t);   // n <= 4096: up to 128 KiB
  if (smem > 48 * 1024) {
    const cudaError_t e =
        cudaFuncSetAttribute(k_visit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_visit<<<1, 256, smem, st>>>(counts, n, max_chunks, k0, dims, plan, state, takes, offsets);
  return launched();
}

}  // namespace spcn
