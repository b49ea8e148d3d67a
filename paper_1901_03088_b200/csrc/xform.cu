// xform.cu — the fused per-pixel recolor kernels (K1, "pass 2").
//
// Replaces the reference's per-strip hot unit `_process_strip`
// (src/pipeline.py:260-272): beer_lambert (src/optics.py:71-94) →
// code_densities (src/stain_sep.py:168-201) → normalize_block
// (src/normalize.py:115-151) → inverse_beer_lambert (src/optics.py:97-110).
//
// Kernels:
//   k_xform_warp<MODE>  persistent; every warp owns a ring of shared-memory
//                       slots fed and drained by 1-D TMA bulk copies
//                       (cp.async.bulk G2S / S2G, mbarrier completion) and
//                       recolours 16 px per lane per 512-px sub-slice in place:
//                       fp32 path two pixels at a time (FFMA2/FMUL2), OD from a
//                       replicated shared-memory table addressed with one PRMT
//                       per channel, output bytes packed with PRMT.  MODE: 0 =
//                       EXACT with the analytic per-pixel bound, 1 = FAST, 2 =
//                       EXACT with a calibrated constant bound, 3 = identity
//                       (memory-path ceiling).  EXACT appends uncertified pixels
//                       to a repair list.
//   k_xform_repair      fp64 reference-order recompute of the listed pixels (or
//                       of every pixel if the list overflowed).
//   k_xform_strict      fp64 reference-order path for every pixel (STRICT mode,
//                       head/tail pixels, unaligned buffers).
//   k_calibrate         runs the fast path and the fp64 path on all 2^24 RGB
//                       colours and returns the largest relative error of the
//                       fast path: a certification bound valid by exhaustion.
#include "launch_count.h"
#include "params.cuh"
#include "spcn.h"
#include "recolor.cuh"
#include "spcn_device.cuh"
#include "xform.h"

#include <cstdio>
#include <cstdlib>

namespace spcn {

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

struct SmemLut {
  const double* t;
  __device__ double operator()(int c, uint32_t i) const { return t[c * 256 + i]; }
};

// ---------------------------------------------------------------------------
// k_xform_warp: the same per-thread pipeline, but every warp owns its own
// ring of NSW slots of NSUB x 512 px and is its own producer: lane 0 issues the
// 1-D TMA bulk load of the warp's next slices, the warp recolours a slice in
// place in shared memory (each lane: 16 px of each 512-px sub-slice, so the
// 48-byte lane blocks stay bank-conflict-free), and lane 0 issues the TMA bulk
// store from the same slot; the slot is refilled as soon as that store has
// finished reading it.  No CTA-wide stage coupling: a slow warp never holds
// back the others' refills.  Work: slices grid-strided over all warps; NSUB
// amortises the per-slice bookkeeping (bulk ops, barrier waits) over more px.
// The OD table is placed at the ABSOLUTE shared address kXAbs (the dynamic
// window starts at a small driver-reserved offset; up to kXAbs bytes of
// padding are allocated in front), so its lookups are LDS [addr + kXAbs].
constexpr uint32_t kXAbs = 4096;

template <int CW, int REP, int NSW, int BLK, int NSUB>
struct WCfg {
  static constexpr int kThreads = 32 * CW;
  static constexpr int kSlicePx = 512 * NSUB;
  static constexpr int kSlotBytes = 3 * kSlicePx;
  static constexpr int kLutBytes = LutLayout<REP>::kBytes;
  static constexpr size_t kSmem =
      kXAbs + kLutBytes + (size_t)CW * NSW * kSlotBytes + CW * NSW * 8;
  static_assert(kSmem <= (BLK == 1 ? 227 * 1024 : 113 * 1024), "shared memory budget");
};

// fp: the kernel's __grid_constant__ parameter block, or a __constant__ slot
// of a device-built recolouring — both constant-bank operands after inlining.
template <int MODE, int CW, int REP, int NSW, int BLK, int NSUB>
__device__ __forceinline__ void xform_warp_body(const uint8_t* __restrict__ src,
                                                uint8_t* __restrict__ dst, int64_t npix,
                                                const FastP& fp, RepairList rl) {
  using C = WCfg<CW, REP, NSW, BLK, NSUB>;
  constexpr int kSlicePx = C::kSlicePx, kSlotBytes = C::kSlotBytes;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  if (base > kXAbs) __trap();   // layout assumption (window base <= 4 KB)
  uint8_t* smem = smem_raw + (kXAbs - base);   // the table at absolute kXAbs
  const uint8_t* lut = smem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* myslots = smem + C::kLutBytes + (size_t)warp * NSW * kSlotBytes;
  uint64_t* mybar =
      reinterpret_cast<uint64_t*>(smem + C::kLutBytes + (size_t)CW * NSW * kSlotBytes) + warp * NSW;

  LutLayout<REP>::fill(smem, &fp.lut[0][0], tid, C::kThreads);
  if (lane == 0) {
    for (int s = 0; s < NSW; ++s) mbar_init(&mybar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();

  uint32_t lc[3];
  LutLayout<REP>::lane_consts(lane, lc);
  float2 I[3];   // calibrated interval: from the host, or from the on-device calibration
#pragma unroll
  for (int c = 0; c < 3; ++c)
    I[c] = (MODE == 2 && rl.alpha_bits) ? calibrated_interval(fp.i0t[c], __uint_as_float(*rl.alpha_bits))
                                        : fp.I[c];
  const int64_t nslices = (npix + kSlicePx - 1) / kSlicePx;
  const int64_t gw = (int64_t)blockIdx.x * CW + warp, GW = (int64_t)gridDim.x * CW;
  uint64_t pol = 0;
  // slot indices as running counters (no 64-bit modulo per slice)
  int ls = 0;                            // lane 0: slot of the next load
  int64_t lj = gw;                       // lane 0: slice of the next load
  auto issue_load = [&]() {   // lane 0 only: next slice into slot ls
    if (lj < nslices) {
      const uint32_t bytes = static_cast<uint32_t>(3 * min64(kSlicePx, npix - lj * kSlicePx));
      mbar_expect_tx(&mybar[ls], bytes);
      bulk_g2s(myslots + ls * kSlotBytes, src + 3 * lj * kSlicePx, bytes, &mybar[ls], pol);
    }
    lj += GW;
    ls = ls + 1 == NSW ? 0 : ls + 1;
  };
  if (lane == 0) {
    pol = policy_evict_first();
    for (int k = 0; k < NSW; ++k) issue_load();
  }

  int s = 0;
  uint32_t phase = 0;
  for (int64_t j = gw, k = 0; j < nslices; j += GW, ++k) {
    mbar_wait(&mybar[s], phase);
    const int n = (int)min64(kSlicePx, npix - j * kSlicePx);
    uint8_t* sbase = myslots + s * kSlotBytes;
#pragma unroll
    for (int u = 0; u < NSUB; ++u)
      recolor_block<MODE, kXAbs>(fp, lut, lc, sbase + u * 1536 + 48 * lane, u * 512 + 16 * lane < n,
                          j * kSlicePx + u * 512 + 16 * lane, rl, lane, I);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      bulk_s2g(dst + 3 * j * kSlicePx, sbase, static_cast<uint32_t>(3 * n));
      bulk_commit();
      if (k >= 1) {
        bulk_wait_read<1>();          // the store of slice k-1 has read its slot
        issue_load();                 // refill that slot (load number k-1+NSW)
      }
    }
    if (++s == NSW) {
      s = 0;
      phase ^= 1u;
    }
  }
  if (lane == 0) bulk_wait_all();
}

template <int MODE, int CW, int REP, int NSW, int BLK, int NSUB>
__global__ void __launch_bounds__(32 * CW, BLK)
    k_xform_warp(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t npix,
                 const __grid_constant__ FastP fp, RepairList rl) {
  xform_warp_body<MODE, CW, REP, NSW, BLK, NSUB>(src, dst, npix, fp, rl);
}

// fp64 recompute of the listed pixels; if the list overflowed (count > cap)
// every pixel of the body is recomputed instead.  The fp64 table is staged in
// shared memory (per-thread table indices differ, so reading it from the
// kernel-parameter bank would serialise).
__device__ __forceinline__ void repair_body(const uint8_t* __restrict__ src,
                                            uint8_t* __restrict__ dst, int64_t npix,
                                            const StrictP& sp, const double* lut,
                                            const NnlsGram& G, RepairList rl,
                                            unsigned long long n) {
  if (n > rl.cap) {
    for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < npix; i += 256ll * gridDim.x) {
      const uint32_t out =
          strict_pixel(sp, G, SmemLut{lut}, src[3 * i], src[3 * i + 1], src[3 * i + 2]);
      dst[3 * i] = out & 255u;
      dst[3 * i + 1] = (out >> 8) & 255u;
      dst[3 * i + 2] = (out >> 16) & 255u;
    }
    return;
  }
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n;
       i += 256ull * gridDim.x) {
    const unsigned long long it = rl.items[i];
    const uint32_t rgb = static_cast<uint32_t>(it & 0xffffffu);
    const int64_t gp = static_cast<int64_t>(it >> 24);
    const uint32_t out =
        strict_pixel(sp, G, SmemLut{lut}, rgb & 255u, (rgb >> 8) & 255u, rgb >> 16);
    dst[3 * gp] = out & 255u;
    dst[3 * gp + 1] = (out >> 8) & 255u;
    dst[3 * gp + 2] = (out >> 16) & 255u;
  }
}

__global__ void __launch_bounds__(256) k_xform_repair(const uint8_t* __restrict__ src,
                                                      uint8_t* __restrict__ dst, int64_t npix,
                                                      const __grid_constant__ StrictP sp,
                                                      RepairList rl) {
  const unsigned long long n = *rl.count;
  if (n == 0) return;
  __shared__ double lut[3 * 256];
  for (int i = threadIdx.x; i < 3 * 256; i += 256) lut[i] = sp.lut[i >> 8][i & 255];
  __syncthreads();
  repair_body(src, dst, npix, sp, lut, gram_of(sp), rl, n);
}

__global__ void __launch_bounds__(256) k_xform_strict(const uint8_t* __restrict__ src,
                                                      uint8_t* __restrict__ dst, int64_t npix,
                                                      const __grid_constant__ StrictP sp) {
  __shared__ double lut[3 * 256];
  for (int i = threadIdx.x; i < 3 * 256; i += 256) lut[i] = sp.lut[i >> 8][i & 255];
  __syncthreads();
  const NnlsGram G = gram_of(sp);
  for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < npix; i += 256ll * gridDim.x) {
    const uint32_t r = src[3 * i], g = src[3 * i + 1], b = src[3 * i + 2];
    const uint32_t out = strict_pixel(sp, G, SmemLut{lut}, r, g, b);
    dst[3 * i] = out & 255u;
    dst[3 * i + 1] = (out >> 8) & 255u;
    dst[3 * i + 2] = (out >> 16) & 255u;
  }
}

// Exhaustive calibration: for every RGB colour (two per thread-iteration,
// through the same fast_pair as the transform) compare y_fast = i0 * 2^e
// (the exact product the certification scales) with the fp64 reference
// value y_ref = i0 * exp(-v') computed in the reference's operation order;
// record max |y_ref - y_fast| / y_fast over colours with y_fast > 0.
__device__ __forceinline__ void calibrate_body(const FastP& fp, const StrictP& sp,
                                               unsigned int* __restrict__ max_bits, uint32_t q0,
                                               uint32_t q1) {
  __shared__ double lut[3 * 256];
  __shared__ float flut[3 * 256];
  for (int i = threadIdx.x; i < 3 * 256; i += 256) {
    lut[i] = sp.lut[i >> 8][i & 255];
    flut[i] = fp.lut[i >> 8][i & 255];
  }
  __syncthreads();
  // the worst relative error as a (numerator, denominator) pair compared by
  // cross-multiplication (no fp64 division per colour); divided once at the
  // end.  A pair within fp64 rounding of the true maximum may be kept instead
  // of it — well inside the 2^-20 margin spcn_xform_calibrate adds.
  double wnum = 0.0, wden = 1.0;
  float worst = 0.f;
  const NnlsGram G = gram_of(sp);
  for (uint32_t q = q0 + blockIdx.x * 256u + threadIdx.x; q < q1; q += 256u * gridDim.x) {
    const uint32_t ca = 2u * q, cb = 2u * q + 1u;   // colours: r | g<<8 | b<<16
    const float2 v0 = make_float2(flut[ca & 255], flut[cb & 255]);
    const float2 v1 = make_float2(flut[256 + ((ca >> 8) & 255)], flut[256 + ((cb >> 8) & 255)]);
    const float2 v2 = make_float2(flut[512 + (ca >> 16)], flut[512 + (cb >> 16)]);
    const FastPair fq = fast_pair(fp, v0, v1, v2);
    const float e[3][2] = {{fq.e0.x, fq.e0.y}, {fq.e1.x, fq.e1.y}, {fq.e2.x, fq.e2.y}};
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const uint32_t col = side ? cb : ca;
      const double d0 = lut[col & 255], d1 = lut[256 + ((col >> 8) & 255)], d2 = lut[512 + (col >> 16)];
      const double b0 = strict_dot3(sp.ws[0][0], sp.ws[1][0], sp.ws[2][0], d0, d1, d2);
      const double b1 = strict_dot3(sp.ws[0][1], sp.ws[1][1], sp.ws[2][1], d0, d1, d2);
      double h0, h1;
      strict_nnls(b0, b1, G, sp.lam, sp.max_sweeps, sp.tol, h0, h1);
      const double s0 = __dmul_rn(sp.f[0], h0), s1 = __dmul_rn(sp.f[1], h1);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double od = __dadd_rn(__dmul_rn(sp.wt[c][0], s0), __dmul_rn(sp.wt[c][1], s1));
        const double yref = __dmul_rn(sp.i0t[c], exp(-od));
        const double yfast = (double)fp.i0t[c] * (double)ex2_approx(e[c][side]);
        if (yfast > 0.0) {
          const double num = fabs(yref - yfast);
          if (num * wden > wnum * yfast) {
            wnum = num;
            wden = yfast;
          }
        } else if (yref >= 0.25) {
          worst = 1.0f;  // cannot happen for finite inputs; forces the analytic path
        }
      }
    }
  }
  worst = fmaxf(worst, (float)(wnum / wden));
  for (int off = 16; off; off >>= 1) worst = fmaxf(worst, __shfl_xor_sync(0xffffffffu, worst, off));
  if ((threadIdx.x & 31) == 0) atomicMax(max_bits, __float_as_uint(worst));
}

__global__ void __launch_bounds__(256) k_calibrate(const __grid_constant__ FastP fp,
                                                   const __grid_constant__ StrictP sp,
                                                   unsigned int* __restrict__ max_bits,
                                                   uint32_t q0, uint32_t q1) {
  calibrate_body(fp, sp, max_bits, q0, q1);
}

// ---------------------------------------------------------------------------
// Device-built recolouring: fit -> transform with no host round trip.
// k_build_xform forms StrictP / FastP of one recolouring on the device from
// the fit's arena (basis, p99, absent flags) and the source OD table already
// resident for the SNMF, with the same params.cuh code the host runs; the
// block is copied into a __constant__ slot, and the slot-templated kernels
// read it exactly as the host path reads its __grid_constant__ block (both
// are constant-bank operands, so the main kernel's SASS is unchanged).  A
// recolouring the fast path cannot take (status != 0: invalid fit, degenerate
// p99, ill-conditioned basis) leaves the output untouched; the caller then
// runs the host-checked path, which raises the reference's error or takes
// the strict path.
__constant__ DevParams c_dp[kDpSlots];

__global__ void __launch_bounds__(256) k_build_xform(const __grid_constant__ XformBuildIn in,
                                                     const double* __restrict__ lut,
                                                     const double* __restrict__ fit,
                                                     DevParams* __restrict__ out,
                                                     unsigned int* __restrict__ ws_hdr) {
  StrictP& sp = out->sp;
  for (int i = threadIdx.x; i < 3 * 256; i += 256) {
    (&sp.lut[0][0])[i] = lut[i];
    (&out->fp.lut[0][0])[i] = static_cast<float>(lut[i]);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // arena B: basis f64[6] | p99 f64[2] | info i32[4] | absent i32[2]
  auto absent_of = [](const double* a) { return reinterpret_cast<const int32_t*>(a + 10); };
  auto basis_ok = [](const double* w) {                                 // api.cu check_basis
    for (int k = 0; k < 6; ++k)
      if (!isfinite(w[k]) || w[k] < 0) return false;
    for (int j = 0; j < 2; ++j) {
      const double nrm = sqrt(p_add(p_add(p_mul(w[j], w[j]), p_mul(w[2 + j], w[2 + j])),
                                    p_mul(w[4 + j], w[4 + j])));
      if (fabs(nrm - 1.0) > 1e-9) return false;
    }
    return true;
  };
  const double* basis = fit;
  const double* p99 = fit + 6;
  const double* tgt = in.tgt_fit_dev;               // a target fitted on the device, or null
  const double* tbasis = tgt ? tgt : in.tgt_basis;
  const double* tp99 = tgt ? tgt + 6 : in.tgt_p99;
  const double* ti0v = tgt ? in.tgt_i0_dev : in.tgt_i0;
  int32_t st = 0;
  if (absent_of(fit)[0] || absent_of(fit)[1]) st = -SPCN_ESTAIN_ABSENT;
  if (tgt && st == 0) {                             // the host checked a host-side target
    if (absent_of(tgt)[0] || absent_of(tgt)[1]) st = -SPCN_ESTAIN_ABSENT;
    for (int j = 0; j < 2 && st == 0; ++j)
      if (!(tp99[j] > 0.0) || !isfinite(tp99[j])) st = -SPCN_EDEGENERATE;
    if (st == 0 && !basis_ok(tbasis)) st = -SPCN_EINVAL;
    for (int c = 0; c < 3 && st == 0; ++c)
      if (!isfinite(ti0v[c])) st = -SPCN_EINVAL;
  }
  double f[2] = {1.0, 1.0};
  for (int j = 0; j < 2 && st == 0; ++j) {
    if (!(p99[j] > 0.0) || !isfinite(p99[j])) st = -SPCN_EDEGENERATE;   // scale_factors
    else f[j] = __ddiv_rn(tp99[j], p99[j]);
    if (st == 0 && (!(f[j] > 0.0) || !isfinite(f[j]))) st = -SPCN_EDEGENERATE;
  }
  if (st == 0 && !basis_ok(basis)) st = -SPCN_EINVAL;
  fill_strict_scalars(sp, basis, tbasis, f, ti0v, in.code_lam, in.max_sweeps);
  if (st == 0 && !fill_fast_scalars(out->fp, sp, true, nullptr)) st = 1;   // strict path only
  out->status = st;
  ws_hdr[0] = ws_hdr[1] = 0u;   // repair count
  ws_hdr[2] = 0u;               // calibration word
}

template <int SLOT>
__global__ void __launch_bounds__(256) k_calibrate_c(unsigned int* __restrict__ max_bits,
                                                     uint32_t q0, uint32_t q1) {
  if (c_dp[SLOT].status != 0) return;
  calibrate_body(c_dp[SLOT].fp, c_dp[SLOT].sp, max_bits, q0, q1);
}

// MODE 2: the calibrated bound (calibration word in the workspace); MODE 0:
// the analytic per-pixel bound (images too small to amortise a calibration)
template <int SLOT, int MODE, int CW, int REP, int NSW, int BLK, int NSUB>
__global__ void __launch_bounds__(32 * CW, BLK)
    k_xform_warp_c(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t npix,
                   RepairList rl) {
  // a declined recolouring runs zero slices (an early exit here would make
  // the compiler keep the shared-memory window base out of uniform registers)
  xform_warp_body<MODE, CW, REP, NSW, BLK, NSUB>(src, dst, c_dp[SLOT].status == 0 ? npix : 0,
                                                 c_dp[SLOT].fp, rl);
}

// The repair list of the vector body [head, head + body), plus the (< 16 px)
// unaligned head and tail of the buffer, all on the fp64 path.
template <int SLOT>
__global__ void __launch_bounds__(256) k_xform_repair_c(const uint8_t* __restrict__ src,
                                                        uint8_t* __restrict__ dst, int64_t npix,
                                                        int64_t head, int64_t body,
                                                        RepairList rl) {
  const StrictP& sp = c_dp[SLOT].sp;
  if (c_dp[SLOT].status != 0) return;
  const unsigned long long n = *rl.count;
  const bool edges = blockIdx.x == 0 && (head > 0 || head + body < npix);
  if (n == 0 && !edges) return;
  __shared__ double lut[3 * 256];
  for (int i = threadIdx.x; i < 3 * 256; i += 256) lut[i] = sp.lut[i >> 8][i & 255];
  __syncthreads();
  const NnlsGram G = gram_of(sp);
  if (edges) {
    const int64_t tail = npix - head - body;
    for (int64_t k = threadIdx.x; k < head + tail; k += 256) {
      const int64_t i = k < head ? k : head + body + (k - head);
      const uint32_t out = strict_pixel(sp, G, SmemLut{lut}, src[3 * i], src[3 * i + 1], src[3 * i + 2]);
      dst[3 * i] = out & 255u;
      dst[3 * i + 1] = (out >> 8) & 255u;
      dst[3 * i + 2] = (out >> 16) & 255u;
    }
  }
  if (n > 0) repair_body(src + 3 * head, dst + 3 * head, body, sp, lut, G, rl, n);
}

// ------------------------------------------------------------------ launchers
static int g_sm_count = 0;

using XformFn = void (*)(const uint8_t*, uint8_t*, int64_t, FastP, RepairList);

using XformCFn = void (*)(const uint8_t*, uint8_t*, int64_t, RepairList);

struct Shape {
  int cw, rep, nsub, blk, nsw, threads, tile_px, blocks_per_sm;
  size_t smem;
  XformFn fn[4];
  XformCFn cfn[kDpSlots][2];   // device-built slots x {calibrated, analytic} (production only)
};

template <int CW, int REP, int NSW, int BLK, int NSUB, bool SLOTS = false>
Shape make_wshape() {
  using C = WCfg<CW, REP, NSW, BLK, NSUB>;
  Shape s{CW, REP, NSUB, BLK, NSW, C::kThreads, CW * C::kSlicePx, 0, C::kSmem,
          {k_xform_warp<0, CW, REP, NSW, BLK, NSUB>, k_xform_warp<1, CW, REP, NSW, BLK, NSUB>,
           k_xform_warp<2, CW, REP, NSW, BLK, NSUB>, k_xform_warp<3, CW, REP, NSW, BLK, NSUB>},
          {{nullptr, nullptr}, {nullptr, nullptr}}};
  static_assert(kDpSlots == 2, "slot table");
  if constexpr (SLOTS) {
    s.cfn[0][0] = k_xform_warp_c<0, 2, CW, REP, NSW, BLK, NSUB>;
    s.cfn[0][1] = k_xform_warp_c<0, 0, CW, REP, NSW, BLK, NSUB>;
    s.cfn[1][0] = k_xform_warp_c<1, 2, CW, REP, NSW, BLK, NSUB>;
    s.cfn[1][1] = k_xform_warp_c<1, 0, CW, REP, NSW, BLK, NSUB>;
  }
  return s;
}

// Compiled shapes; SPCN_XFORM_SHAPE="CWxREPxNSUBxBLK" selects one
// (experiments); the first entry is the production shape.
// SPCN_XFORM_IDENTITY=1 makes the kernel copy input to output (memory-path
// ceiling measurement only).
static Shape g_shapes[] = {
    make_wshape<16, 24, 3, 1, 2, true>(),   // production: per-warp rings of 2x512-px slots, mixed table
    make_wshape<16, 16, 3, 1, 2>(), make_wshape<16, 16, 2, 1, 3>(), make_wshape<16, 16, 4, 1, 1>(),
    make_wshape<8, 16, 3, 2, 1>(), make_wshape<20, 16, 2, 1, 2>(), make_wshape<20, 24, 2, 1, 2>(),
    make_wshape<16, 24, 4, 1, 1>()};
static Shape* g_shape = nullptr;
static int g_slot_bps = 1;   // resident CTAs/SM of the slot kernels
static bool g_identity = false;

cudaError_t xform_setup_device() {
  if (g_shape) return cudaSuccess;
  int dev;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  Shape* pick = &g_shapes[0];
  if (const char* env = getenv("SPCN_XFORM_SHAPE")) {
    int cw = 0, rep = 0, nsub = 0, blk = 0, nsw = 0;   // CWxREPxNSUBxBLK[xNSW]
    const int nf = sscanf(env, "%dx%dx%dx%dx%d", &cw, &rep, &nsub, &blk, &nsw);
    if (nf >= 4)
      for (auto& s : g_shapes)
        if (s.cw == cw && s.rep == rep && s.nsub == nsub && s.blk == blk &&
            (nf == 4 || s.nsw == nsw)) {
          pick = &s;
          break;
        }
  }
  if (const char* env = getenv("SPCN_XFORM_IDENTITY")) g_identity = env[0] == '1';
  for (auto fn : pick->fn) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pick->smem);
    if (e != cudaSuccess) return e;
  }
  // the device-built path always runs the production shape
  for (auto& pair : g_shapes[0].cfn)
    for (auto fn : pair) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)g_shapes[0].smem);
      if (e != cudaSuccess) return e;
    }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_slot_bps, g_shapes[0].cfn[0][0],
                                                    g_shapes[0].threads, g_shapes[0].smem);
  if (e != cudaSuccess) return e;
  if (g_slot_bps < 1) g_slot_bps = 1;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pick->blocks_per_sm, pick->fn[2],
                                                    pick->threads, pick->smem);
  if (e != cudaSuccess) return e;
  if (pick->blocks_per_sm < 1) pick->blocks_per_sm = 1;
  g_shape = pick;
  return cudaSuccess;
}

cudaError_t launch_xform_main(int mode, const uint8_t* src, uint8_t* dst, int64_t npix,
                             const FastP& fp, const StrictP& sp, unsigned long long* count,
                             unsigned long long* items, unsigned long long cap,
                             const unsigned int* alpha_bits, cudaStream_t st) {
  cudaError_t e = xform_setup_device();
  if (e != cudaSuccess) return e;
  const Shape& s = *g_shape;
  const int64_t ntiles = (npix + s.tile_px - 1) / s.tile_px;
  const int grid = static_cast<int>(min64(ntiles, (int64_t)g_sm_count * s.blocks_per_sm));
  RepairList rl{count, items, cap, alpha_bits};
  s.fn[g_identity ? 3 : mode]<<<grid, s.threads, s.smem, st>>>(src, dst, npix, fp, rl);
  return launched();
}

cudaError_t launch_xform_build(int slot, const XformBuildIn& in, const double* lut,
                               const double* fit, DevParams* staging, void* ws,
                               int32_t* status_host, cudaEvent_t built, uint32_t q0, uint32_t q1,
                               cudaStream_t st) {
  cudaError_t e = xform_setup_device();
  if (e != cudaSuccess) return e;
  unsigned int* hdr = static_cast<unsigned int*>(ws);
  k_build_xform<<<1, 256, 0, st>>>(in, lut, fit, staging, hdr);
  if ((e = launched()) != cudaSuccess) return e;
  e = cudaMemcpyToSymbolAsync(c_dp, staging, sizeof(DevParams), slot * sizeof(DevParams),
                              cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  if (status_host &&
      (e = cudaMemcpyAsync(status_host, &staging->status, sizeof(int32_t), cudaMemcpyDeviceToHost,
                           st)) != cudaSuccess)
    return e;
  if (built && (e = cudaEventRecord(built, st)) != cudaSuccess) return e;
  if (q1 <= q0) return cudaSuccess;
  // colour pairs [q0, q1) with launch_calibrate's proportional grid
  const int64_t full = (int64_t)g_sm_count * 16;
  int64_t grid = (full * (int64_t)(q1 - q0) + (1 << 23) - 1) >> 23;
  if (grid < 1) grid = 1;
  if (slot == 0) k_calibrate_c<0><<<(int)grid, 256, 0, st>>>(hdr + 2, q0, q1);
  else k_calibrate_c<1><<<(int)grid, 256, 0, st>>>(hdr + 2, q0, q1);
  return launched();
}

cudaError_t launch_xform_main_c(int slot, bool analytic, const uint8_t* src, uint8_t* dst,
                                int64_t npix, unsigned long long* count,
                                unsigned long long* items, unsigned long long cap,
                                const unsigned int* alpha_bits, cudaStream_t st) {
  cudaError_t e = xform_setup_device();
  if (e != cudaSuccess) return e;
  if (npix <= 0) return cudaSuccess;
  const Shape& s = g_shapes[0];
  const int64_t ntiles = (npix + s.tile_px - 1) / s.tile_px;
  const int grid = static_cast<int>(min64(ntiles, (int64_t)g_sm_count * g_slot_bps));
  RepairList rl{count, items, cap, analytic ? nullptr : alpha_bits};
  s.cfn[slot][analytic ? 1 : 0]<<<grid, s.threads, s.smem, st>>>(src, dst, npix, rl);
  return launched();
}

cudaError_t launch_xform_repair_c(int slot, const uint8_t* src, uint8_t* dst, int64_t npix,
                                  int64_t head, int64_t body, unsigned long long* count,
                                  unsigned long long* items, unsigned long long cap,
                                  cudaStream_t st) {
  cudaError_t e = xform_setup_device();
  if (e != cudaSuccess) return e;
  RepairList rl{count, items, cap};
  if (slot == 0) k_xform_repair_c<0><<<g_sm_count * 4, 256, 0, st>>>(src, dst, npix, head, body, rl);
  else k_xform_repair_c<1><<<g_sm_count * 4, 256, 0, st>>>(src, dst, npix, head, body, rl);
  return launched();
}

const char* xform_shape_name() {
  static char buf[96];
  if (xform_setup_device() != cudaSuccess || !g_shape) return "unavailable";
  snprintf(buf, sizeof(buf), "k_xform_warp: %d warps/CTA, LUT x%d, %d x 512-px sub-slices/slot, "
           "%d CTA/SM", g_shape->cw, g_shape->rep, g_shape->nsub, g_shape->blocks_per_sm);
  return buf;
}

cudaError_t launch_xform_repair(const uint8_t* src, uint8_t* dst, int64_t npix, const StrictP& sp,
                                unsigned long long* count, unsigned long long* items,
                                unsigned long long cap, cudaStream_t st) {
  cudaError_t e = xform_setup_device();
  if (e != cudaSuccess) return e;
  RepairList rl{count, items, cap};
  k_xform_repair<<<g_sm_count * 4, 256, 0, st>>>(src, dst, npix, sp, rl);
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

cudaError_t launch_calibrate(const FastP& fp, const StrictP& sp, unsigned int* max_bits,
                             cudaStream_t st, uint32_t q0, uint32_t q1) {
  cudaError_t e = xform_setup_device();
  if (e != cudaSuccess) return e;
  if (q1 <= q0) return cudaSuccess;
  // colour pairs [q0, q1); a share of the 2^23 pairs gets a proportional grid
  const int64_t full = (int64_t)g_sm_count * 16;
  int64_t grid = (full * (int64_t)(q1 - q0) + (1 << 23) - 1) >> 23;
  if (grid < 1) grid = 1;
  k_calibrate<<<(int)grid, 256, 0, st>>>(fp, sp, max_bits, q0, q1);
  return launched();
}

int xform_tile_pixels() { return g_shape ? g_shape->tile_px : 16 * 512 * 2; }

}  // namespace spcn
