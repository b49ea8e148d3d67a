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

constexpr int kStBins = 8192;
constexpr int kSlicePx = 512;            // one TMA bulk load: 512 px = 1536 B
constexpr int kSliceBytes = 3 * kSlicePx;

// Ring geometry: CW warps per CTA, NSW slots per warp.
template <int CW, int NSW, int NSUB = 1>
struct StRing {
  static constexpr int kThreads = 32 * CW;
  static constexpr size_t kBytes = (size_t)CW * NSW * NSUB * kSliceBytes + (size_t)CW * NSW * 8;
};
// histogram pass: 32 warps (<= 64 registers), 2 slots each
#ifndef SPCN_HIST_CW
#define SPCN_HIST_CW 32
#endif
constexpr int kHistCW = SPCN_HIST_CW, kHistNSW = kHistCW == 32 ? 2 : 3;
// refine pass
#ifndef SPCN_REF_CW
#define SPCN_REF_CW 32
#endif
constexpr int kRefCW = SPCN_REF_CW, kRefNSW = kRefCW == 32 ? 2 : 3;
constexpr size_t kStSmemHist = LutLayout<16>::kBytes + 2 * (kStBins + 8) * sizeof(uint32_t) +
                               StRing<kHistCW, kHistNSW>::kBytes;

__device__ __forceinline__ uint32_t st_byte(const uint32_t* w, int idx) {
  return (w[idx >> 2] >> (8 * (idx & 3))) & 0xffu;
}

// Every warp streams its share of the 512-px slices of the 16-px-aligned body
// [0, nbody) through a private ring of NSW shared-memory slots (1-D TMA bulk
// loads, mbarrier completion; lane 0 refills a slot as soon as the warp has
// read it) and calls body(w, 16, inv, blk) with each lane's 16 pixels (48
// bytes, also readable at blk until body returns; inv = all ones for a lane
// past the end of a short slice, whose pixels must all be ignored).  The
// < 16-px tail is read from global memory by one lane: body(w, nvalid, 0, w).
struct NoAfter {
  __device__ void operator()(const uint8_t*) const {}
};

// NSUB 512-px blocks per slice (each lane: NSUB x 16 px per slice, body once
// per block); after(slot) runs once per slice after its blocks, warp-wide.
template <int CW, int NSW, int NSUB = 1, class Body, class After = NoAfter>
__device__ __forceinline__ void st_scan(const uint8_t* __restrict__ src, int64_t npix,
                                        uint8_t* ring, Body&& body, After&& after = After()) {
  constexpr int kSlicePx = 512 * NSUB, kSliceBytes = 3 * kSlicePx;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* myslots = ring + (size_t)warp * NSW * kSliceBytes;
  uint64_t* mybar = reinterpret_cast<uint64_t*>(ring + (size_t)CW * NSW * kSliceBytes) + warp * NSW;
  const int64_t nbody = npix & ~int64_t(15);
  const int64_t nsl = (nbody + kSlicePx - 1) / kSlicePx;
  const int64_t gw = (int64_t)blockIdx.x * CW + warp, GW = (int64_t)gridDim.x * CW;
  uint64_t pol = 0;
  int ls = 0;              // lane 0: slot of the next load (running counter)
  int64_t lj = gw;         // lane 0: slice of the next load
  auto issue = [&]() {     // lane 0 only
    if (lj < nsl) {
      const int64_t left = nbody - lj * kSlicePx;
      const uint32_t bytes = static_cast<uint32_t>(3 * (left < kSlicePx ? left : kSlicePx));
      mbar_expect_tx(&mybar[ls], bytes);
      bulk_g2s(myslots + ls * kSliceBytes, src + 3 * lj * kSlicePx, bytes, &mybar[ls], pol);
    }
    lj += GW;
    ls = ls + 1 == NSW ? 0 : ls + 1;
  };
  if (lane == 0) {
    for (int s = 0; s < NSW; ++s) mbar_init(&mybar[s], 1);
    mbar_fence_init();
    pol = policy_evict_first();
    for (int k = 0; k < NSW; ++k) issue();
  }
  __syncwarp();
  int s = 0;
  uint32_t phase = 0;
  for (int64_t j = gw; j < nsl; j += GW) {
    mbar_wait(&mybar[s], phase);
    const int64_t left = nbody - j * kSlicePx;
#pragma unroll
    for (int u = 0; u < NSUB; ++u) {
      // no divergent branch: lanes past the end of a short slice run on
      // stale slot bytes with every pixel masked (body's `all_invalid`)
      const uint8_t* blk = myslots + s * kSliceBytes + 1536 * u + 48 * lane;
      const uint4* q = reinterpret_cast<const uint4*>(blk);
      const uint4 q0 = q[0], q1 = q[1], q2 = q[2];
      const uint32_t w[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y,
                              q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
      body(w, 16, 512 * u + 16 * lane < left ? 0u : ~0u, blk);
    }
    after(myslots + s * kSliceBytes);
    __syncwarp();
    if (lane == 0) {
      fence_proxy_async_smem();   // the warp's reads of slot s precede its refill
      issue();                    // slot s again (the loads run NSW slices ahead)
    }
    if (++s == NSW) {
      s = 0;
      phase ^= 1u;
    }
  }
  if (npix > nbody && blockIdx.x == 0 && threadIdx.x == 0) {
    uint32_t w[12];
    for (int t = 0; t < 12; ++t) w[t] = 0;
    for (int64_t p = nbody; p < npix; ++p)
      for (int c = 0; c < 3; ++c) {
        const int idx = 3 * (int)(p - nbody) + c;
        w[idx >> 2] |= (uint32_t)src[3 * p + c] << (8 * (idx & 3));
      }
    body(w, (int)(npix - nbody), 0u, reinterpret_cast<const uint8_t*>(w));
  }
}

// Two pixels (2q, 2q+1) of a lane's block: fp32 densities and non-white flags
// (bit 0: pixel 2q, bit 1: pixel 2q+1).
struct StPair {
  float2 h0x2, h1x2, T;   // 2*h0, 2*h1 (the halving is folded into the consumers' constants)
  uint32_t wx, wy;        // all ones if the pixel is white, else 0
};

// od_lookup through an explicit shared-window address (lets the table base
// ride in the load's uniform-register operand)
__device__ __forceinline__ float st_od(uint32_t lut_s, const uint32_t* w, int idx, uint32_t lc) {
  const uint32_t sel = 0x7604u | ((uint32_t)(idx & 3) << 4);
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(lut_s + __byte_perm(w[idx >> 2], lc, sel)));
  return v;
}

template <bool OD>
__device__ __forceinline__ StPair st_pair(const StatsArgs& a, const uint8_t* lut,
                                          const uint32_t* lc, const uint32_t* w, int q) {
  const int ia = 6 * q, ib = 6 * q + 3;
  const uint32_t ls = smem_u32(lut);
  const float2 v0 = make_float2(st_od(ls, w, ia, lc[0]), st_od(ls, w, ib, lc[0]));
  const float2 v1 = make_float2(st_od(ls, w, ia + 1, lc[1]), st_od(ls, w, ib + 1, lc[1]));
  const float2 v2 = make_float2(st_od(ls, w, ia + 2, lc[2]), st_od(ls, w, ib + 2, lc[2]));
  const FastDensity d = fast_density(a.fs, v0, v1, v2);
  StPair o;
  o.h0x2 = d.h0x2;
  o.h1x2 = d.h1x2;
  o.T = d.T;
  if (OD) {
    // v - OD(white) < 0 (sign bit; RN subtraction keeps the sign) <=> channel > white
    const float2 s0 = __fadd2_rn(v0, bc2(a.nwod[0]));
    const float2 s1 = __fadd2_rn(v1, bc2(a.nwod[1]));
    const float2 s2 = __fadd2_rn(v2, bc2(a.nwod[2]));
    const uint32_t wx = __float_as_uint(s0.x) & __float_as_uint(s1.x) & __float_as_uint(s2.x);
    const uint32_t wy = __float_as_uint(s0.y) & __float_as_uint(s1.y) & __float_as_uint(s2.y);
    o.wx = (uint32_t)((int32_t)wx >> 31);
    o.wy = (uint32_t)((int32_t)wy >> 31);
  } else {
    uint32_t m[2];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int k = 2 * q + p;
      const bool white = st_byte(w, 3 * k) > a.white && st_byte(w, 3 * k + 1) > a.white &&
                         st_byte(w, 3 * k + 2) > a.white;
      m[p] = white ? ~0u : 0u;
    }
    o.wx = m[0];
    o.wy = m[1];
  }
  return o;
}

// fp32 density of one pixel (the fast path's arithmetic, bit-identical to
// st_pair's for that pixel), bytes read from a lane block in memory.
__device__ __forceinline__ FastDensity st_one(const StatsArgs& a, const uint8_t* lut,
                                              const uint32_t* lc, const uint8_t* px) {
  const float v0 = *reinterpret_cast<const float*>(lut + (((uint32_t)px[0] << 8) | lc[0]));
  const float v1 = *reinterpret_cast<const float*>(lut + (((uint32_t)px[1] << 8) | lc[1]));
  const float v2 = *reinterpret_cast<const float*>(lut + (((uint32_t)px[2] << 8) | lc[2]));
  return fast_density(a.fs, bc2(v0), bc2(v1), bc2(v2));
}

// Histogram layout per stain in shared memory: [0] = below the window or
// white (not read), [1 .. nbins] = the bins, [nbins + 1] = above the window.
constexpr int kHistStride = kStBins + 8;

template <bool OD>
__global__ void __launch_bounds__(32 * kHistCW, 1)
    k_stats_hist(const uint8_t* __restrict__ src, int64_t npix, const __grid_constant__ StatsArgs a,
                 unsigned long long* __restrict__ hist, unsigned long long* __restrict__ counts) {
  constexpr int kThreads = 32 * kHistCW;
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* sh = reinterpret_cast<uint32_t*>(smem + LutLayout<16>::kBytes);
  uint8_t* ring = smem + LutLayout<16>::kBytes + 2 * kHistStride * sizeof(uint32_t);
  LutLayout<16>::fill(smem, &a.lut[0][0], threadIdx.x, kThreads);
  for (int i = threadIdx.x; i < 2 * kHistStride; i += kThreads) sh[i] = 0;
  __syncthreads();
  uint32_t lc[3];
  LutLayout<16>::lane_consts(threadIdx.x & 31, lc);
  // Keys are taken of 2h: key(2h) = key(h) + 2^23 over the normal range, so
  // the window start moves instead of every density being halved (the
  // histogram only places the refine window; subnormal h may land a bin off).
  // Slot of a key: min((max(key, lo) - lo) >> shift, nbins + 1) with lo one
  // bin below the window start, so below-the-window keys (and white pixels,
  // whose key is zeroed) land in slot 0 without a branch.  Every pixel does
  // one shared atomic per stain (cheaper here than compacting the few
  // in-window pixels: the kernel is ALU-bound and a divergent loop over
  // candidates costs more than the atomics); "below" = non-white - slots
  // 1..nbins+1, per CTA at the end (with base 0 that is h = 0, i.e. bin 0).
  constexpr uint32_t kTwo = 1u << 23;
  const uint32_t s0 = a.shift[0], s1 = a.shift[1];
  const uint32_t lo0 = a.base[0] + kTwo - (1u << s0), lo1 = a.base[1] + kTwo - (1u << s1);
  const uint32_t top = (uint32_t)a.nbins + 1u;
  uint32_t* hs0 = reinterpret_cast<uint32_t*>(smem + LutLayout<16>::kBytes);
  uint32_t* hs1 = hs0 + kHistStride;
  int32_t nonwhite = 0;
  st_scan<kHistCW, kHistNSW>(src, npix, ring,
                             [&](const uint32_t* w, int nv, uint32_t inv, const uint8_t*) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const StPair d = st_pair<OD>(a, smem, lc, w, q);
      uint32_t wx = d.wx | inv, wy = d.wy | inv;
      if (nv < 16) {
        if (2 * q >= nv) wx = ~0u;
        if (2 * q + 1 >= nv) wy = ~0u;
      }
      nonwhite += 2 + (int32_t)wx + (int32_t)wy;
      const uint32_t k0x = __float_as_uint(d.h0x2.x) & ~wx, k1x = __float_as_uint(d.h1x2.x) & ~wx;
      const uint32_t k0y = __float_as_uint(d.h0x2.y) & ~wy, k1y = __float_as_uint(d.h1x2.y) & ~wy;
      atomicAdd(hs0 + min((max(k0x, lo0) - lo0) >> s0, top), 1u);
      atomicAdd(hs1 + min((max(k1x, lo1) - lo1) >> s1, top), 1u);
      atomicAdd(hs0 + min((max(k0y, lo0) - lo0) >> s0, top), 1u);
      atomicAdd(hs1 + min((max(k1y, lo1) - lo1) >> s1, top), 1u);
    }
  });
  __syncthreads();
  // flush the bins; count this CTA's binned pixels (incl. above) per stain
  const int nb = a.nbins;
  unsigned long long binned0 = 0, binned1 = 0;
  for (int i = 1 + threadIdx.x; i <= nb + 1; i += kThreads) {
    const uint32_t c0 = sh[i], c1 = sh[kHistStride + i];
    binned0 += c0;
    binned1 += c1;
    if (i <= nb) {
      if (c0) atomicAdd(&hist[i - 1], (unsigned long long)c0);
      if (c1) atomicAdd(&hist[nb + i - 1], (unsigned long long)c1);
    }
  }
  __shared__ unsigned long long red[32][3];
  unsigned long long nwl = nonwhite;
  for (int off = 16; off; off >>= 1) {
    nwl += __shfl_xor_sync(0xffffffffu, nwl, off);
    binned0 += __shfl_xor_sync(0xffffffffu, binned0, off);
    binned1 += __shfl_xor_sync(0xffffffffu, binned1, off);
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[warp][0] = nwl;
    red[warp][1] = binned0;
    red[warp][2] = binned1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t[3] = {0, 0, 0};
    for (int k = 0; k < kHistCW; ++k)
      for (int c = 0; c < 3; ++c) t[c] += red[k][c];
    if (t[0]) atomicAdd(&counts[0], t[0]);
    for (int j = 0; j < 2; ++j) {
      const unsigned long long below = t[0] - t[1 + j];
      if (below) atomicAdd(a.base[j] ? &counts[1 + j] : &hist[j * nb], below);
    }
  }
}

// Per-CTA colour cache of the refine pass: a density is a function of the
// pixel's RGB only, and the pixels that can fall in the narrow window share
// few colours, so each CTA evaluates a colour in fp64 once and keeps in-window
// pixel counts per colour; at the end it lists (value, count) pairs.
constexpr int kSlots = kRefCW == 32 ? 1024 : 2048;   // fits next to the ring
constexpr uint32_t kEmpty = 0xffffffffu;
struct ColourSlot {
  uint32_t key;        // rgb, or kEmpty
  uint32_t ready;      // x valid
  uint32_t cnt[2];     // in-window pixels per stain
  double x[2];         // exact densities
};
constexpr size_t kStSmemRefine = LutLayout<16>::kBytes + 3 * 256 * sizeof(double) +
                                 kSlots * sizeof(ColourSlot) + StRing<kRefCW, kRefNSW>::kBytes;

__device__ __forceinline__ uint32_t colour_hash(uint32_t rgb) {
  return (rgb * 2654435761u) >> (32 - (kSlots == 1024 ? 10 : 11));
}

struct RefineCtx {
  const StatsArgs& a;
  const StrictP& sp;
  const NnlsGram& G;
  const double* dlut;
  ColourSlot* tab;
  unsigned long long* counts;
  double* cand;
  unsigned long long* wcnt;
  unsigned long long cap;

  __device__ void list(int j, double x, unsigned long long c) const {   // one (value, count) entry
    atomicAdd(&counts[2 + j], c);
    const unsigned long long idx = atomicAdd(&counts[5 + j], 1ull);
    if (idx < cap) {
      cand[j * cap + idx] = x;
      wcnt[j * cap + idx] = c;
    }
  }

  // fp64 density of a colour that may lie in the window (bit j of `need`),
  // through the colour cache; updates the exact below counts
  // returns bit 0/1: NOT below the window (stain 0/1, among `need`), bit 2:
  // an fp64 evaluation was made
  __device__ __noinline__ uint32_t exact(uint32_t rgb, uint32_t need) const {
    uint32_t r = 0;
    // find or claim a slot; a slot claimed but not yet filled by another
    // thread is simply recomputed here (no waiting)
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
      r |= 4u;
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
      if (x[j] < a.a[j]) continue;
      r |= 1u << j;
      if (x[j] < a.b[j]) {
        if (slot >= 0) atomicAdd(&tab[slot].cnt[j], 1u);
        else list(j, x[j], 1ull);                // cache full: list the pixel itself
      }
    }
    return r;
  }

  // Full classification of one non-white candidate pixel (bytes at px):
  // returns bit 0/1: not below the window (stain 0/1), bit 2: an fp64
  // evaluation was made.  Same bounds as the kernel's fast test.
  __device__ __forceinline__ uint32_t pixel(const uint8_t* lut, const uint32_t* lc,
                                            const uint8_t* px) const {
    const FastDensity d = st_one(a, lut, lc, px);
    const float T = d.T.x;
    float up[2], dn[2];
    up[0] = __fadd_ru(d.h0x2.x, __fmaf_ru(2.0f * a.coef[0], T, 2e-30f));
    up[1] = __fadd_ru(d.h1x2.x, __fmaf_ru(2.0f * a.coef[1], T, 2e-30f));
    dn[0] = __fadd_rd(d.h0x2.x, __fmaf_rd(-2.0f * a.coef[0], T, -2e-30f));
    dn[1] = __fadd_rd(d.h1x2.x, __fmaf_rd(-2.0f * a.coef[1], T, -2e-30f));
    uint32_t r = 0, need = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (up[j] < 2.0f * __double2float_rd(a.a[j])) continue;         // surely below
      if (dn[j] >= 2.0f * __double2float_ru(a.b[j])) r |= 1u << j;    // surely at/above b
      else need |= 1u << j;
    }
    if (need) r |= exact((uint32_t)px[0] | ((uint32_t)px[1] << 8) | ((uint32_t)px[2] << 16), need);
    return r;
  }
};

template <bool OD>
__global__ void __launch_bounds__(32 * kRefCW, 1)
    k_stats_refine(const uint8_t* __restrict__ src, int64_t npix,
                   const __grid_constant__ StatsArgs a, const __grid_constant__ StrictP sp,
                   unsigned long long* __restrict__ counts, double* __restrict__ cand,
                   unsigned long long* __restrict__ wcnt, unsigned long long cap) {
  constexpr int kThreads = 32 * kRefCW;
  extern __shared__ __align__(128) uint8_t smem[];
  double* dlut = reinterpret_cast<double*>(smem + LutLayout<16>::kBytes);
  ColourSlot* tab = reinterpret_cast<ColourSlot*>(smem + LutLayout<16>::kBytes +
                                                  3 * 256 * sizeof(double));
  uint8_t* ring = reinterpret_cast<uint8_t*>(tab + kSlots);
  LutLayout<16>::fill(smem, &a.lut[0][0], threadIdx.x, kThreads);
  for (int i = threadIdx.x; i < 3 * 256; i += kThreads) dlut[i] = sp.lut[i >> 8][i & 255];
  for (int i = threadIdx.x; i < kSlots; i += kThreads) {
    tab[i].key = kEmpty;
    tab[i].ready = 0;
    tab[i].cnt[0] = tab[i].cnt[1] = 0;
  }
  __syncthreads();
  uint32_t lc[3];
  LutLayout<16>::lane_consts(threadIdx.x & 31, lc);
  const NnlsGram G = gram_of(sp);
  const RefineCtx ctx{a, sp, G, dlut, tab, counts, cand, wcnt, cap};
  // Classification in fp32 with directed rounding: with e >= the density
  // error bound, h + e (rounded up) < a (rounded down) proves x < a, and
  // h - e (rounded down) >= b (rounded up) proves x >= b.  Evaluated on 2h
  // against 2e, 2a, 2b (scaling by 2 is exact).  The sign of (h + e) - a
  // (RN keeps the sign of a difference) is the "surely below" flag; a pair
  // whose four flags are set (white pixels count as set) costs no more.
  // Below counts are derived at the end: below = non-white - not-below.
  const float2 ea0 = bc2(2.0f * a.coef[0]), ea1 = bc2(2.0f * a.coef[1]), tiny = bc2(2e-30f);
  const float2 nlo0 = bc2(-2.0f * __double2float_rd(a.a[0])), nlo1 = bc2(-2.0f * __double2float_rd(a.a[1]));
  int32_t nonwhite = 0;
  uint32_t nb0 = 0, nb1 = 0, evals = 0;   // not below, fp64 evaluations
  st_scan<kRefCW, kRefNSW>(src, npix, ring,
                           [&](const uint32_t* w, int nv, uint32_t inv, const uint8_t* blk) {
    // pass 1, branch-free: non-white count and the candidates = non-white
    // pixels not surely below the window in both stains
    uint32_t cand = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const StPair d = st_pair<OD>(a, smem, lc, w, q);
      uint32_t wx = d.wx | inv, wy = d.wy | inv;
      if (nv < 16) {
        if (2 * q >= nv) wx = ~0u;
        if (2 * q + 1 >= nv) wy = ~0u;
      }
      nonwhite += 2 + (int32_t)wx + (int32_t)wy;
      const float2 e0 = __ffma2_ru(ea0, d.T, tiny), e1 = __ffma2_ru(ea1, d.T, tiny);
      const float2 eb0 = __fadd2_rn(__fadd2_ru(d.h0x2, e0), nlo0);
      const float2 eb1 = __fadd2_rn(__fadd2_ru(d.h1x2, e1), nlo1);
      const uint32_t sx = (__float_as_uint(eb0.x) & __float_as_uint(eb1.x)) | wx;
      const uint32_t sy = (__float_as_uint(eb0.y) & __float_as_uint(eb1.y)) | wy;
      cand |= (~sx >> 31) << (2 * q);
      cand |= (~sy >> 31) << (2 * q + 1);
    }
    // pass 2: each lane pops one candidate per iteration
    while (cand) {
      const int k = __ffs(cand) - 1;
      cand &= cand - 1;
      const uint32_t r = ctx.pixel(smem, lc, blk + 3 * k);
      nb0 += r & 1u;
      nb1 += (r >> 1) & 1u;
      evals += r >> 2;
    }
  });
  __syncthreads();
  for (int i = threadIdx.x; i < kSlots; i += kThreads)
    for (int j = 0; j < 2; ++j)
      if (tab[i].cnt[j]) {
        // counted only by threads that knew the value; its owner set it
        // (and `ready`) before this barrier
        ctx.list(j, tab[i].x[j], tab[i].cnt[j]);
      }
  unsigned long long b0 = (unsigned long long)(nonwhite - (int32_t)nb0),
                     b1 = (unsigned long long)(nonwhite - (int32_t)nb1), ev = evals;
  for (int off = 16; off; off >>= 1) {
    ev += __shfl_xor_sync(0xffffffffu, ev, off);
    b0 += __shfl_xor_sync(0xffffffffu, b0, off);
    b1 += __shfl_xor_sync(0xffffffffu, b1, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (b0) atomicAdd(&counts[0], b0);
    if (b1) atomicAdd(&counts[1], b1);
    if (ev) atomicAdd(&counts[4], ev);
  }
}

// ---------------------------------------------------------------------------
// One-pass exact mode (colour table).  A pixel's density depends only on its
// RGB, so the pixels that are not surely below a lower bound a_j (from the
// sample) in some stain are counted per colour in a direct-mapped table of
// 2^24 counters (per-CTA shared-memory cache in front of the global
// atomics).  k_table_scan then evaluates every present colour in fp64 in the
// reference's operation order: pixels off the table are < a_j for sure, so
// the order statistics at or above a_j are exactly those of the table
// entries with x_j >= a_j (the host checks the ranks land there).
constexpr int kTabSlots = 4096;
// Shared-memory layout of the table pass: the OD table sits at the ABSOLUTE
// shared-window address 0x10000, so the PRMT that forms an entry's offset
// (pixel byte << 8 | lane byte, region byte 1) is already its address and
// the load needs no base add (the compiler would otherwise add the window
// base per lookup: 3 instructions per pixel).  Colour cache below it, the
// TMA ring above it.
constexpr uint32_t kTabLutAbs = 0x10000;
constexpr size_t kStSmemTable = kTabLutAbs + LutLayout<16>::kBytes + StRing<kRefCW, kRefNSW>::kBytes;

__device__ __forceinline__ float lds_abs(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ float od_abs(const uint32_t* w, int idx, uint32_t lc) {
  const uint32_t sel = 0x7604u | ((uint32_t)(idx & 3) << 4);
  return lds_abs(__byte_perm(w[idx >> 2], lc, sel));
}

template <bool OD>
__global__ void __launch_bounds__(32 * kRefCW, 1)
    k_stats_table(const uint8_t* __restrict__ src, int64_t npix, const __grid_constant__ StatsArgs a,
                  unsigned long long* __restrict__ table, unsigned long long* __restrict__ counts) {
  constexpr int kThreads = 32 * kRefCW;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t base = smem_u32(smem);
  if (base + kTabSlots * 8 > kTabLutAbs) __trap();   // layout assumption (window base <= 32 KB)
  uint8_t* lut = smem + (kTabLutAbs - base);
  uint32_t* ckey = reinterpret_cast<uint32_t*>(smem);
  uint32_t* ccnt = ckey + kTabSlots;
  uint8_t* ring = lut + LutLayout<16>::kBytes;
  LutLayout<16>::fill(lut, &a.lut[0][0], threadIdx.x, kThreads);
  for (int i = threadIdx.x; i < kTabSlots; i += kThreads) {
    ckey[i] = kEmpty;
    ccnt[i] = 0;
  }
  __syncthreads();
  uint32_t lc[3];
  LutLayout<16>::lane_consts(threadIdx.x & 31, lc);
  for (int c = 0; c < 3; ++c) lc[c] |= kTabLutAbs;   // region byte = 1: absolute address
  // Candidates without solving the NNLS: for two stains the solution has
  // h_j in {0, u_j, t_j/g_jj} (u = G^-1 t, t = W^T v - lam: the three
  // active sets), so h_j <= max(u_j, t_j/g_jj, 0) and a pixel is surely below
  // a_j > 0 when both linear forms u_j - a_j and t_j/g_jj - a_j are negative.
  // The four forms k.v + b are evaluated in fp32 with their rounding bound
  // folded into b (host, stats_linear_forms); a pixel with every form < 0 is
  // off the table.
  int32_t nonwhite = 0;
  st_scan<kRefCW, kRefNSW>(src, npix, ring,
                           [&](const uint32_t* w, int nv, uint32_t inv, const uint8_t* blk) {
    uint32_t cand = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int ia = 6 * q, ib = 6 * q + 3;
      const float2 v0 = make_float2(od_abs(w, ia, lc[0]), od_abs(w, ib, lc[0]));
      const float2 v1 = make_float2(od_abs(w, ia + 1, lc[1]), od_abs(w, ib + 1, lc[1]));
      const float2 v2 = make_float2(od_abs(w, ia + 2, lc[2]), od_abs(w, ib + 2, lc[2]));
      uint32_t wx, wy;
      if (OD) {
        const float2 s0 = __fadd2_rn(v0, bc2(a.nwod[0]));
        const float2 s1 = __fadd2_rn(v1, bc2(a.nwod[1]));
        const float2 s2 = __fadd2_rn(v2, bc2(a.nwod[2]));
        wx = (uint32_t)((int32_t)(__float_as_uint(s0.x) & __float_as_uint(s1.x) & __float_as_uint(s2.x)) >> 31);
        wy = (uint32_t)((int32_t)(__float_as_uint(s0.y) & __float_as_uint(s1.y) & __float_as_uint(s2.y)) >> 31);
      } else {
        uint32_t m[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const int k = 2 * q + p;
          const bool white = st_byte(w, 3 * k) > a.white && st_byte(w, 3 * k + 1) > a.white &&
                             st_byte(w, 3 * k + 2) > a.white;
          m[p] = white ? ~0u : 0u;
        }
        wx = m[0];
        wy = m[1];
      }
      wx |= inv;
      wy |= inv;
      if (nv < 16) {
        if (2 * q >= nv) wx = ~0u;
        if (2 * q + 1 >= nv) wy = ~0u;
      }
      nonwhite += 2 + (int32_t)wx + (int32_t)wy;
      float2 f[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        f[i] = __ffma2_rn(bc2(a.lf[i][0]), v0,
                          __ffma2_rn(bc2(a.lf[i][1]), v1, __ffma2_rn(bc2(a.lf[i][2]), v2, bc2(a.lf[i][3]))));
      const uint32_t sx = (__float_as_uint(f[0].x) & __float_as_uint(f[1].x) &
                           __float_as_uint(f[2].x) & __float_as_uint(f[3].x)) | wx;
      const uint32_t sy = (__float_as_uint(f[0].y) & __float_as_uint(f[1].y) &
                           __float_as_uint(f[2].y) & __float_as_uint(f[3].y)) | wy;
      cand |= (~sx >> 31) << (2 * q);
      cand |= (~sy >> 31) << (2 * q + 1);
    }
    while (cand) {   // each lane counts one candidate colour per iteration
      const int k = __ffs(cand) - 1;
      cand &= cand - 1;
      const uint8_t* px = blk + 3 * k;
      const uint32_t rgb = (uint32_t)px[0] | ((uint32_t)px[1] << 8) | ((uint32_t)px[2] << 16);
      uint32_t sl = (rgb * 2654435761u) >> 20;   // 12-bit hash
      bool done = false;
      for (int probe = 0; probe < 8 && !done; ++probe, sl = (sl + 1) & (kTabSlots - 1)) {
        uint32_t key = ckey[sl];
        if (key == kEmpty) {
          const uint32_t prev = atomicCAS(&ckey[sl], kEmpty, rgb);
          key = prev == kEmpty ? rgb : prev;
        }
        if (key == rgb) {
          atomicAdd(&ccnt[sl], 1u);
          done = true;
        }
      }
      if (!done) atomicAdd(&table[rgb], 1ull);    // cache full around this hash
    }
  });
  __syncthreads();
  for (int i = threadIdx.x; i < kTabSlots; i += kThreads)
    if (ccnt[i]) atomicAdd(&table[ckey[i]], (unsigned long long)ccnt[i]);
  unsigned long long nwl = (unsigned long long)nonwhite;
  for (int off = 16; off; off >>= 1) nwl += __shfl_xor_sync(0xffffffffu, nwl, off);
  if ((threadIdx.x & 31) == 0 && nwl) atomicAdd(&counts[0], nwl);
}

// Every present colour of the table: exact fp64 densities (reference order)
// and its pixel count, compacted to (x[2*i], x[2*i+1], w[i]); n_out[0] = the
// number of present colours (entries past `cap` are dropped), n_out[1] = the
// pixels they hold.
__global__ void __launch_bounds__(256) k_table_scan(const unsigned long long* __restrict__ table,
                                                    const __grid_constant__ StrictP sp,
                                                    double* __restrict__ x,
                                                    unsigned long long* __restrict__ w,
                                                    unsigned long long cap,
                                                    unsigned long long* __restrict__ n_out) {
  __shared__ double dlut[3 * 256];
  for (int i = threadIdx.x; i < 3 * 256; i += 256) dlut[i] = sp.lut[i >> 8][i & 255];
  __syncthreads();
  const NnlsGram G = gram_of(sp);
  unsigned long long pix = 0;
  for (uint32_t c = blockIdx.x * 256u + threadIdx.x; c < (1u << 24); c += 256u * gridDim.x) {
    const unsigned long long n = table[c];
    if (!n) continue;
    pix += n;
    const double v0 = dlut[c & 255u], v1 = dlut[256 + ((c >> 8) & 255u)], v2 = dlut[512 + (c >> 16)];
    const double b0 = strict_dot3(sp.ws[0][0], sp.ws[1][0], sp.ws[2][0], v0, v1, v2);
    const double b1 = strict_dot3(sp.ws[0][1], sp.ws[1][1], sp.ws[2][1], v0, v1, v2);
    double h0, h1;
    strict_nnls(b0, b1, G, sp.lam, sp.max_sweeps, sp.tol, h0, h1);
    const unsigned long long i = atomicAdd(&n_out[0], 1ull);
    if (i < cap) {
      x[2 * i] = h0;
      x[2 * i + 1] = h1;
      w[i] = n;
    }
    // per-stain maximum (densities are >= 0: the bit patterns order like the values)
    atomicMax(&n_out[2], (unsigned long long)__double_as_longlong(h0));
    atomicMax(&n_out[3], (unsigned long long)__double_as_longlong(h1));
  }
  for (int off = 16; off; off >>= 1) pix += __shfl_xor_sync(0xffffffffu, pix, off);
  if ((threadIdx.x & 31) == 0 && pix) atomicAdd(&n_out[1], pix);
}

// ---------------------------------------------------------------------------
// Colour-cube classes in front of the one-pass table (k_stats_cube).  The RGB
// cube is cut into 32^3 cells of 8x8x8 colours; every cell gets one class
// from its 512 colours, evaluated with exactly the per-pixel tests:
//   0  every colour white                      -> the pixel is skipped
//   1  every colour non-white and surely below -> counted as non-white only
//   2  anything else (white and non-white colours, or some candidate)
//      -> per-pixel white test and candidate test (table insert)
// so almost every pixel costs one shared-memory byte lookup instead of three
// OD lookups and four fp32 linear forms.
constexpr int kCubeCells = 1 << 15;

__device__ __forceinline__ uint32_t cube_cell(uint32_t rgb) {   // r | g << 8 | b << 16
  return ((rgb >> 3) & 0x1Fu) | ((rgb >> 6) & 0x3E0u) | ((rgb >> 9) & 0x7C00u);
}

// Not surely below lo in some stain: one of the four linear upper-bound forms
// (stats_linear_forms, fp32 with the rounding bound folded in) is >= 0.  The
// same expression serves the class builder and the pass.
__device__ __forceinline__ bool cube_candidate(const StatsArgs& a, float v0, float v1, float v2) {
  uint32_t all_neg = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    all_neg &= __float_as_uint(__fmaf_rn(a.lf[i][0], v0,
                                         __fmaf_rn(a.lf[i][1], v1, __fmaf_rn(a.lf[i][2], v2, a.lf[i][3]))));
  return !(all_neg >> 31);
}

__global__ void __launch_bounds__(256) k_cube_class(const __grid_constant__ StatsArgs a,
                                                    uint8_t* __restrict__ cls) {
  __shared__ float lut[3 * 256];
  for (int i = threadIdx.x; i < 3 * 256; i += 256) lut[i] = a.lut[i >> 8][i & 255];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int cell = blockIdx.x * 8 + (threadIdx.x >> 5); cell < kCubeCells; cell += gridDim.x * 8) {
    const uint32_t r0 = (cell & 31) << 3, g0 = ((cell >> 5) & 31) << 3, b0 = (cell >> 10) << 3;
    bool any_cand = false, any_white = false, any_nonwhite = false;
    for (int t = 0; t < 16; ++t) {
      const int i = lane * 16 + t;
      const uint32_t r = r0 + (i & 7), g = g0 + ((i >> 3) & 7), b = b0 + (i >> 6);
      const bool white = r > a.white && g > a.white && b > a.white;
      any_white |= white;
      any_nonwhite |= !white;
      if (!white) any_cand |= cube_candidate(a, lut[r], lut[256 + g], lut[512 + b]);
    }
    any_cand = __any_sync(0xffffffffu, any_cand);
    any_white = __any_sync(0xffffffffu, any_white);
    any_nonwhite = __any_sync(0xffffffffu, any_nonwhite);
    if (lane == 0) cls[cell] = any_cand ? 2 : (!any_nonwhite ? 0 : (!any_white ? 1 : 2));
  }
}

// Candidate-colour bitmap (2^24 bits, rgb order): bit = non-white and not
// surely below (cube_candidate) — the same test the cell classes aggregate,
// read per pixel by the few class-2 pixels of k_stats_cube instead of
// evaluating the OD table and the four linear forms.
constexpr size_t kCandBitmapBytes = (size_t)1 << 21;

__global__ void __launch_bounds__(256) k_cand_bitmap(const __grid_constant__ StatsArgs a,
                                                     uint32_t* __restrict__ bits) {
  __shared__ float lut[3 * 256];
  for (int i = threadIdx.x; i < 3 * 256; i += 256) lut[i] = a.lut[i >> 8][i & 255];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // a warp per word: lane t evaluates colour 32 * word + t
  for (uint32_t word = blockIdx.x * 8 + (threadIdx.x >> 5); word < (1u << 19);
       word += gridDim.x * 8) {
    const uint32_t c = 32u * word + lane;
    const uint32_t r = c & 255u, g = (c >> 8) & 255u, b = c >> 16;
    const bool white = r > a.white && g > a.white && b > a.white;
    const bool cand = !white && cube_candidate(a, lut[r], lut[256 + g], lut[512 + b]);
    const uint32_t m = __ballot_sync(0xffffffffu, cand);
    if (lane == 0) bits[word] = m;
  }
}

// The one-pass table of k_stats_table with the cell classes in front: same
// contract (table[rgb] counts the non-white pixels not surely below lo in
// some stain, counts[0] the non-white pixels), pixels in class-0/1 cells
// decided by the class alone.  Shared memory: class table 32 KB, fp32 OD
// table (3 KB, read by the few class-2 pixels only), colour cache, TMA ring.
// 32 warps x 2 ring slots of 512 px (measured at 10 Gpx: 16 warps x 2 slots
// of 1024 px 11.9 ms, 32 x 3 slots 10.2 ms, this 9.6-9.7 ms).
constexpr int kCubeCW = 32, kCubeNSW = 2, kCubeNSUB = 1;
constexpr int kCubeQueue = 256;   // queued marked pixels per warp (flushed when full)
constexpr int kCubeSlots = 2048;           // colour cache (a slide's candidate colours are few)
// Shared-memory layout: colour cache, OD table and queues from the window
// base; the class table at the ABSOLUTE shared address kCubeAbs (so a cell
// index plus an immediate is its address: no base add per pixel); the TMA
// ring above it.
constexpr uint32_t kCubeAbs = 0x9000;
constexpr size_t kCubeLow = (size_t)kCubeSlots * 8 + (size_t)kCubeCW * kCubeQueue * sizeof(uint16_t);
static_assert(kCubeLow <= kCubeAbs - 4096, "cube pass: low region must leave room for the window base");
constexpr size_t kStSmemCube = kCubeAbs + kCubeCells + StRing<kCubeCW, kCubeNSW, kCubeNSUB>::kBytes;

__device__ __forceinline__ uint32_t lds_u8_cube(uint32_t cell) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1+36864];" : "=r"(v) : "r"(cell));   // + kCubeAbs
  return v;
}

__device__ __forceinline__ uint32_t st_rgb(const uint32_t* w, int k) {   // pixel k's r|g<<8|b<<16 (+ junk byte 3)
  const int j = 3 * k, o = j & 3;
  const uint32_t sel = (uint32_t)o | ((uint32_t)(o + 1) << 4) | ((uint32_t)(o + 2) << 8);
  return __byte_perm(w[j >> 2], w[(j >> 2) + (o >= 2 ? 1 : 0)], sel);
}

// One marked (class 2) pixel: exact white test, candidate test (one bit of
// the k_cand_bitmap bitmap: the same test as cube_candidate) and the
// colour-table insert.  Returns 1 if non-white.
__device__ __forceinline__ int32_t cube_marked_pixel(const uint8_t* px, uint32_t white,
                                                     const uint32_t* __restrict__ cbits,
                                                     uint32_t* ckey, uint32_t* ccnt,
                                                     unsigned long long* __restrict__ table) {
  const uint32_t r = px[0], g = px[1], b = px[2];
  if (r > white && g > white && b > white) return 0;
  const uint32_t rgb = r | (g << 8) | (b << 16);
  if (!((__ldg(&cbits[rgb >> 5]) >> (rgb & 31)) & 1u)) return 1;   // surely below (k_cand_bitmap)
  uint32_t sl = (rgb * 2654435761u) >> 21;   // 11-bit hash
  for (int probe = 0; probe < 8; ++probe, sl = (sl + 1) & (kCubeSlots - 1)) {
    uint32_t key = ckey[sl];
    if (key == kEmpty) {
      const uint32_t prev = atomicCAS(&ckey[sl], kEmpty, rgb);
      key = prev == kEmpty ? rgb : prev;
    }
    if (key == rgb) {
      atomicAdd(&ccnt[sl], 1u);
      return 1;
    }
  }
  atomicAdd(&table[rgb], 1ull);    // cache full around this hash
  return 1;
}

__global__ void __launch_bounds__(32 * kCubeCW, 1)
    k_stats_cube(const uint8_t* __restrict__ src, int64_t npix, const __grid_constant__ StatsArgs a,
                 const uint8_t* __restrict__ gcls, unsigned long long* __restrict__ table,
                 unsigned long long* __restrict__ counts) {
  const uint32_t* cbits = reinterpret_cast<const uint32_t*>(gcls + kCubeCells);
  constexpr int kThreads = 32 * kCubeCW;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t base = smem_u32(smem);
  if (base + kCubeLow > kCubeAbs) __trap();   // layout assumption (window base <= 4 KB)
  uint32_t* ckey = reinterpret_cast<uint32_t*>(smem);
  uint32_t* ccnt = ckey + kCubeSlots;
  uint16_t* queue = reinterpret_cast<uint16_t*>(ccnt + kCubeSlots) + (threadIdx.x >> 5) * kCubeQueue;
  uint8_t* cls = smem + (kCubeAbs - base);
  uint8_t* ring = cls + kCubeCells;
  for (int i = threadIdx.x; i < kCubeCells / 16; i += kThreads)
    reinterpret_cast<uint4*>(cls)[i] = reinterpret_cast<const uint4*>(gcls)[i];
  for (int i = threadIdx.x; i < kCubeSlots; i += kThreads) {
    ckey[i] = kEmpty;
    ccnt[i] = 0;
  }
  __syncthreads();
  const uint32_t white = a.white;
  const int lane = threadIdx.x & 31;
  int32_t nonwhite = 0;
  int qn = 0;   // marked pixels queued in this slice (warp-uniform)
  st_scan<kCubeCW, kCubeNSW, kCubeNSUB>(src, npix, ring,
                             [&](const uint32_t* w, int nv, uint32_t inv, const uint8_t* blk) {
    // the 16 classes side by side, 2 bits each (class <= 2: no carries).
    // Cell index with few ALU operations: the 5-bit cell coordinates of every
    // byte first (two operations per word), then per pixel one PRMT (its
    // top byte a sign-replicated zero) and y - 224 (y >> 8) - 7168 (y >> 16)
    // = r5 + 32 g5 + 1024 b5 — the multiply-adds run on the FMA pipe.
    uint32_t w5[12];
#pragma unroll
    for (int t = 0; t < 12; ++t) w5[t] = (w[t] >> 3) & 0x1F1F1F1Fu;
    uint32_t c2 = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int j = 3 * k, o = j & 3;
      const uint32_t sel = (uint32_t)o | ((uint32_t)(o + 1) << 4) | ((uint32_t)(o + 2) << 8) |
                           ((8u | (uint32_t)o) << 12);        // byte 3: sign of byte o = 0
      uint32_t y;   // prmt with the sign-replicate bit (__byte_perm drops it)
      asm("prmt.b32 %0, %1, %2, %3;"
          : "=r"(y) : "r"(w5[j >> 2]), "r"(w5[(j >> 2) + (o >= 2 ? 1 : 0)]), "r"(sel));
      c2 += lds_u8_cube(y - 224u * __umulhi(y, 1u << 24) - 7168u * __umulhi(y, 1u << 16))
            << (2 * k);
    }
    if (nv < 16) c2 &= (1u << (2 * nv)) - 1u;   // the short tail: drop pixels past the end
    c2 &= ~inv;                                 // lanes past the end of a short slice
    nonwhite += __popc(c2 & 0x55555555u);       // class 1: non-white, surely below
    uint32_t mark = c2 & 0xAAAAAAAAu;           // class 2: bit 2k+1
    if (nv < 16) {   // the short tail (one thread): serial path
      while (mark) {
        const int k = (__ffs(mark) - 1) >> 1;
        mark &= mark - 1;
        nonwhite += cube_marked_pixel(blk + 3 * k, white, cbits, ckey, ccnt, table);
      }
      return;
    }
    // queue the marked pixels (byte offsets in the warp's slot) for the
    // warp-cooperative pass after the slice's blocks
    const int cnt = __popc(mark);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t off0 = (uint32_t)(blk - ring) % (uint32_t)(kCubeNSUB * kSliceBytes);
    if (total > kCubeQueue) {        // a block this dense in marks: every lane its own
      while (mark) {
        const int k = (__ffs(mark) - 1) >> 1;
        mark &= mark - 1;
        nonwhite += cube_marked_pixel(blk + 3 * k, white, cbits, ckey, ccnt, table);
      }
      return;
    }
    if (qn + total > kCubeQueue) {   // queue full: work it off now (warp-uniform)
      const uint8_t* slot = blk - off0;
      __syncwarp();
      for (int i = lane; i < qn; i += 32)
        nonwhite += cube_marked_pixel(slot + queue[i], white, cbits, ckey, ccnt, table);
      __syncwarp();
      qn = 0;
    }
    int pos = qn + incl - cnt;
    qn += total;
    while (mark) {
      const int bit = __ffs(mark) - 1;
      mark &= mark - 1;
      queue[pos++] = (uint16_t)(off0 + 3 * (bit >> 1));
    }
  }, [&](const uint8_t* slot) {
    // every lane takes queued pixels in turn: no lane idles while another
    // works through its own list
    __syncwarp();
    for (int i = lane; i < qn; i += 32)
      nonwhite += cube_marked_pixel(slot + queue[i], white, cbits, ckey, ccnt, table);
    qn = 0;
  });
  __syncthreads();
  for (int i = threadIdx.x; i < kCubeSlots; i += kThreads)
    if (ccnt[i]) atomicAdd(&table[ckey[i]], (unsigned long long)ccnt[i]);
  unsigned long long nwl = (unsigned long long)nonwhite;
  for (int off = 16; off; off >>= 1) nwl += __shfl_xor_sync(0xffffffffu, nwl, off);
  if ((threadIdx.x & 31) == 0 && nwl) atomicAdd(&counts[0], nwl);
}

// ---------------------------------------------------------------------------
// Exact selection over the table entries (x[2i+j], w[i]) of k_table_scan,
// without sorting them: a weighted histogram of each stain's entries with
// x >= lo_j over nbins equal bins of [lo_j, lo_j + nbins / scale_j] (the host
// sums it across ranks and finds the bins holding the requested ranks), then
// the entries of bins [b0_j, b1_j] listed as (value, weight) for an exact
// weighted select of the few that remain.  Both kernels compute the bin with
// the same expression, so an entry is listed iff it was counted in those bins.
__device__ __forceinline__ int64_t entry_bin(double x, double lo, double scale, int nbins) {
  if (!(x >= lo)) return -1;
  const double f = (x - lo) * scale;
  return f >= (double)(nbins - 1) ? nbins - 1 : (int64_t)f;
}

__global__ void __launch_bounds__(256) k_entries_hist(const double* __restrict__ x,
                                                      const unsigned long long* __restrict__ w,
                                                      int64_t m, double lo0, double lo1,
                                                      double sc0, double sc1, int nbins,
                                                      unsigned long long* __restrict__ hist) {
  extern __shared__ unsigned long long sh[];   // 2 x nbins
  for (int i = threadIdx.x; i < 2 * nbins; i += 256) sh[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < m; i += 256ll * gridDim.x) {
    const unsigned long long n = w[i];
    const int64_t b0 = entry_bin(x[2 * i], lo0, sc0, nbins);
    const int64_t b1 = entry_bin(x[2 * i + 1], lo1, sc1, nbins);
    if (b0 >= 0) atomicAdd(&sh[b0], n);
    if (b1 >= 0) atomicAdd(&sh[nbins + b1], n);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * nbins; i += 256)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__global__ void __launch_bounds__(256) k_entries_collect(
    const double* __restrict__ x, const unsigned long long* __restrict__ w, int64_t m,
    double lo0, double lo1, double sc0, double sc1, int nbins, int b00, int b01, int b10, int b11,
    double* __restrict__ vals, unsigned long long* __restrict__ wts, unsigned long long cap,
    unsigned long long* __restrict__ nsel) {
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < m; i += 256ll * gridDim.x) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double v = x[2 * i + j];
      const int64_t b = entry_bin(v, j ? lo1 : lo0, j ? sc1 : sc0, nbins);
      if (b >= (j ? b10 : b00) && b <= (j ? b11 : b01)) {
        const unsigned long long k = atomicAdd(&nsel[j], 1ull);
        if (k < cap) {
          vals[j * cap + k] = v;
          wts[j * cap + k] = w[i];
        }
      }
    }
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
    for (auto k : {k_stats_hist<true>, k_stats_hist<false>}) {
      const cudaError_t e =
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStSmemHist);
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  if (npix <= 0) return cudaSuccess;
  const int64_t nsl = (npix + kSlicePx - 1) / kSlicePx;
  int64_t grid = (nsl + kHistCW - 1) / kHistCW;
  if (grid > st_grid()) grid = st_grid();
  (a.white_by_od ? k_stats_hist<true> : k_stats_hist<false>)<<<(int)grid, 32 * kHistCW,
                                                               kStSmemHist, st>>>(src, npix, a, hist, counts);
  return launched();
}

cudaError_t launch_stats_refine(const uint8_t* src, int64_t npix, const StatsArgs& a,
                                const StrictP& sp, unsigned long long* counts, double* cand,
                                unsigned long long* wcnt, unsigned long long cap,
                                cudaStream_t st) {
  constexpr size_t smem = kStSmemRefine;
  static bool attr = false;
  if (!attr) {
    for (auto k : {k_stats_refine<true>, k_stats_refine<false>}) {
      const cudaError_t e =
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  if (npix <= 0) return cudaSuccess;
  const int64_t nsl = (npix + kSlicePx - 1) / kSlicePx;
  int64_t grid = (nsl + kRefCW - 1) / kRefCW;
  if (grid > st_grid()) grid = st_grid();
  (a.white_by_od ? k_stats_refine<true> : k_stats_refine<false>)<<<(int)grid, 32 * kRefCW, smem, st>>>(
      src, npix, a, sp, counts, cand, wcnt, cap);
  return launched();
}

}  // namespace spcn

namespace spcn {
cudaError_t launch_stats_table(const uint8_t* src, int64_t npix, const StatsArgs& a,
                               unsigned long long* table, unsigned long long* counts,
                               cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    for (auto k : {k_stats_table<true>, k_stats_table<false>}) {
      const cudaError_t e =
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStSmemTable);
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  if (npix <= 0) return cudaSuccess;
  const int64_t nsl = (npix + kSlicePx - 1) / kSlicePx;
  int64_t grid = (nsl + kRefCW - 1) / kRefCW;
  if (grid > st_grid()) grid = st_grid();
  (a.white_by_od ? k_stats_table<true> : k_stats_table<false>)<<<(int)grid, 32 * kRefCW,
                                                                 kStSmemTable, st>>>(
      src, npix, a, table, counts);
  return launched();
}

cudaError_t launch_cube_class(const StatsArgs& a, uint8_t* cls, cudaStream_t st) {
  k_cube_class<<<kCubeCells / 8, 256, 0, st>>>(a, cls);
  cudaError_t e = launched();
  if (e != cudaSuccess) return e;
  k_cand_bitmap<<<8 * st_grid(), 256, 0, st>>>(a, reinterpret_cast<uint32_t*>(cls + kCubeCells));
  return launched();
}

cudaError_t launch_stats_cube(const uint8_t* src, int64_t npix, const StatsArgs& a,
                              const uint8_t* cls, unsigned long long* table,
                              unsigned long long* counts, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    const cudaError_t e =
        cudaFuncSetAttribute(k_stats_cube, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStSmemCube);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (npix <= 0) return cudaSuccess;
  const int64_t nsl = (npix + kCubeNSUB * kSlicePx - 1) / (kCubeNSUB * kSlicePx);
  int64_t grid = (nsl + kCubeCW - 1) / kCubeCW;
  if (grid > st_grid()) grid = st_grid();
  k_stats_cube<<<(int)grid, 32 * kCubeCW, kStSmemCube, st>>>(src, npix, a, cls, table, counts);
  return launched();
}

cudaError_t launch_entries_hist(const double* x, const unsigned long long* w, int64_t m,
                                const double* lo, const double* scale, int nbins,
                                unsigned long long* hist, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  int64_t grid = (m + 255) / 256;
  if (grid > 4 * st_grid()) grid = 4 * st_grid();
  const size_t smem = 2 * (size_t)nbins * sizeof(unsigned long long);
  static bool attr = false;
  if (!attr) {
    const cudaError_t e =
        cudaFuncSetAttribute(k_entries_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_entries_hist<<<(int)grid, 256, smem, st>>>(x, w, m, lo[0], lo[1], scale[0], scale[1], nbins,
                                               hist);
  return launched();
}

cudaError_t launch_entries_collect(const double* x, const unsigned long long* w, int64_t m,
                                   const double* lo, const double* scale, int nbins,
                                   const int32_t* bins, double* vals, unsigned long long* wts,
                                   unsigned long long cap, unsigned long long* nsel,
                                   cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  int64_t grid = (m + 255) / 256;
  if (grid > 4 * st_grid()) grid = 4 * st_grid();
  k_entries_collect<<<(int)grid, 256, 0, st>>>(x, w, m, lo[0], lo[1], scale[0], scale[1], nbins,
                                               bins[0], bins[1], bins[2], bins[3], vals, wts, cap,
                                               nsel);
  return launched();
}

cudaError_t launch_table_scan(const unsigned long long* table, const StrictP& sp, double* x,
                              unsigned long long* w, unsigned long long cap,
                              unsigned long long* n_out, cudaStream_t st) {
  k_table_scan<<<4 * st_grid(), 256, 0, st>>>(table, sp, x, w, cap, n_out);
  return launched();
}
}  // namespace spcn
