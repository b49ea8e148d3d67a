// batch.cu — many independent recolourings in one launch (configs[1]: 4096
// patches of 512^2, each with its own source FitParams, one fixed target).
//
// Reference semantics per item: `_normalize_one` (src/cli.py:220-244) =
// fit(source) then transform against the target, errors collected per item
// as in `cmd_batch` (src/cli.py:270-301).  The fits come from the batched fit
// kernels (sample.cu, snmf.cu, select.cu); this file turns the per-item fit
// results into parameter blocks on the device and recolours all items with
// one CTA per item per launch:
//   k_build_params     per item: factors + degeneracy checks (src/normalize.py:103-112,
//                      src/pipeline.py:291-297), StrictP, fp32 table, FastS
//                      (params.cuh, identical to the single-item host path);
//   k_xform_batch      per-warp TMA rings over the item's 512-px slices, the
//                      item's FastS read from the kernel-parameter block
//                      (uniform across the CTA), its table from global memory;
//   k_repair_batch     fp64 reference-order recompute of uncertified pixels,
//                      item located by binary search over the pixel offsets.
#include "batch.h"
#include "launch_count.h"
#include "params.cuh"
#include "spcn_device.cuh"

namespace spcn {

constexpr int kBW = 16;         // warps per CTA
constexpr int kBNSW = 4;        // slots per warp
constexpr int kBLut = 2 * 65536;
constexpr size_t kBSmem = kBLut + (size_t)kBW * kBNSW * 1536 + kBW * kBNSW * 8;

__device__ __forceinline__ int64_t bmin64(int64_t a, int64_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------- parameter build
__global__ void __launch_bounds__(128) k_build_params(
    int nitems, const double* __restrict__ i0, const double* __restrict__ luts,
    const double* __restrict__ bases, const double* __restrict__ p99,
    const __grid_constant__ BatchTarget tgt, double code_lam, int max_sweeps, int exact,
    FastS* __restrict__ fs, float* __restrict__ flut, StrictP* __restrict__ sps,
    int32_t* __restrict__ status) {
  const int p = blockIdx.x;
  if (p >= nitems) return;
  StrictP& sp = sps[p];
  for (int i = threadIdx.x; i < 768; i += 128) (&sp.lut[0][0])[i] = luts[(int64_t)p * 768 + i];
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t st = status[p];
    double f[2] = {1.0, 1.0};
    if (st == 0) {
      const double s0 = p99[2 * p], s1 = p99[2 * p + 1];
      if (!(s0 > 0.0) || !(s1 > 0.0)) {
        st = -SPCN_EDEGENERATE;                       // scale_factors: source p99 zero
      } else {
        f[0] = __ddiv_rn(tgt.p99[0], s0);
        f[1] = __ddiv_rn(tgt.p99[1], s1);
        if (!(f[0] > 0.0) || !(f[1] > 0.0)) st = -SPCN_EDEGENERATE;   // target p99 zero
      }
    }
    fill_strict_scalars(sp, bases + 6 * (int64_t)p, tgt.basis, f, tgt.i0, code_lam, max_sweeps);
    FastS s;
    const bool ok = st == 0 && fill_fast_scalars(s, sp, exact != 0, nullptr);
    fs[p] = s;
    if (st == 0 && !ok) st = 1;                       // valid, but strict path only
    status[p] = st;
  }
  for (int i = threadIdx.x; i < 768; i += 128)
    flut[(int64_t)p * 768 + i] = static_cast<float>(luts[(int64_t)p * 768 + i]);
}

// ---------------------------------------------------------------- batched recolour
struct GlobalLut {
  const StrictP* p;
  __device__ double operator()(int c, uint32_t x) const { return p->lut[c][x]; }
};
__device__ __noinline__ uint32_t b_strict_rgb(const StrictP* sp, uint32_t rgb) {
  return strict_pixel(*sp, GlobalLut{sp}, rgb & 255u, (rgb >> 8) & 255u, rgb >> 16);
}

__device__ __forceinline__ uint32_t b_lop3_xor_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xBE;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ float b_od(const uint8_t* lut, const uint32_t* w, int idx, uint32_t lc) {
  const uint32_t sel = 0x7604u | ((uint32_t)(idx & 3) << 4);
  return *reinterpret_cast<const float*>(lut + __byte_perm(w[idx >> 2], lc, sel));
}
__device__ __forceinline__ uint32_t b_pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
__device__ __forceinline__ uint32_t b_byte(const uint32_t* w, int idx) {
  return (w[idx >> 2] >> (8 * (idx & 3))) & 0xffu;
}

template <int MODE>
__device__ __forceinline__ uint32_t b_recolor_pair(const FastS& fp, const uint8_t* lut,
                                                   const uint32_t* w, int k, const uint32_t* lc,
                                                   uint32_t* ob) {
  const int a = 3 * k, b = 3 * k + 3;
  const float2 v0 = make_float2(b_od(lut, w, a, lc[0]), b_od(lut, w, b, lc[0]));
  const float2 v1 = make_float2(b_od(lut, w, a + 1, lc[1]), b_od(lut, w, b + 1, lc[1]));
  const float2 v2 = make_float2(b_od(lut, w, a + 2, lc[2]), b_od(lut, w, b + 2, lc[2]));
  const FastPair fq = fast_pair(fp, v0, v1, v2);
  const float e[3][2] = {{fq.e0.x, fq.e0.y}, {fq.e1.x, fq.e1.y}, {fq.e2.x, fq.e2.y}};
  if (MODE == 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float2 pw = make_float2(ex2_approx(e[c][0]), ex2_approx(e[c][1]));
      const float2 r = __ffma2_rn(bc2(fp.i0t[c]), pw, bc2(kMagic));
      ob[a + c] = __float_as_uint(r.x);
      ob[b + c] = __float_as_uint(r.y);
    }
    return 0u;
  }
  const float2 alpha = __ffma2_rn(bc2(fp.a1), fq.T, bc2(fp.a0));
  uint32_t bad = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float pa = ex2_approx(e[c][0]), pb = ex2_approx(e[c][1]);
    const float2 Ia = cert_interval(fp.i0t[c], alpha.x), Ib = cert_interval(fp.i0t[c], alpha.y);
    const float2 ra = __ffma2_rn(Ia, bc2(pa), bc2(kMagic));
    const float2 rb = __ffma2_rn(Ib, bc2(pb), bc2(kMagic));
    ob[a + c] = __float_as_uint(ra.y);
    ob[b + c] = __float_as_uint(rb.y);
    bad = b_lop3_xor_or(__float_as_uint(ra.y), __float_as_uint(ra.x), bad);
    bad = b_lop3_xor_or(__float_as_uint(rb.y), __float_as_uint(rb.x), bad);
  }
  return bad;
}

// MODE 0 = EXACT (analytic certification + repair list), 1 = FAST.
template <int MODE>
__global__ void __launch_bounds__(32 * kBW, 1)
    k_xform_batch(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                  const float* __restrict__ flut, const StrictP* __restrict__ sps,
                  const __grid_constant__ BatchArgs args, unsigned long long* __restrict__ rcount,
                  unsigned long long* __restrict__ ritems, unsigned long long rcap) {
  const int item = blockIdx.x;
  if (item >= args.n || args.strict[item]) return;     // strict items run elsewhere
  const FastS& fp = args.s[item];
  const int64_t px0 = args.off[item], npix = args.off[item + 1] - px0;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint8_t* lut = smem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* myslots = smem + kBLut + (size_t)warp * kBNSW * 1536;
  uint64_t* mybar = reinterpret_cast<uint64_t*>(smem + kBLut + (size_t)kBW * kBNSW * 1536) +
                    warp * kBNSW;
  const float* tl = flut + (int64_t)(args.item0 + item) * 768;
  for (int i = tid; i < 256 * 96; i += 32 * kBW) {
    const int x = i / 96, rem = i - 96 * (i / 96), c = rem >> 5, r = rem & 31;
    const int off = (c == 2 ? 65536 : 0) + x * 256 + (c == 1 ? 128 : 0) + r * 4;
    *reinterpret_cast<float*>(smem + off) = tl[c * 256 + x];
  }
  if (lane == 0) {
    for (int s = 0; s < kBNSW; ++s) mbar_init(&mybar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const uint32_t lrep = (uint32_t)lane * 4;
  const uint32_t lc[3] = {lrep, 128u + lrep, 0x10000u | lrep};
  const uint8_t* isrc = src + 3 * px0;
  uint8_t* idst = dst + 3 * px0;
  const int64_t nslices = (npix + 511) / 512;
  uint64_t pol = 0;
  auto issue_load = [&](int64_t k) {
    const int64_t j = warp + k * kBW;
    if (j >= nslices) return;
    const int s = (int)(k % kBNSW);
    const uint32_t bytes = static_cast<uint32_t>(3 * bmin64(512, npix - j * 512));
    mbar_expect_tx(&mybar[s], bytes);
    bulk_g2s(myslots + s * 1536, isrc + 3 * j * 512, bytes, &mybar[s], pol);
  };
  if (lane == 0) {
    pol = policy_evict_first();
    for (int k = 0; k < kBNSW; ++k) issue_load(k);
  }
  for (int64_t k = 0;; ++k) {
    const int64_t j = warp + k * kBW;
    if (j >= nslices) break;
    const int s = (int)(k % kBNSW);
    mbar_wait(&mybar[s], (uint32_t)((k / kBNSW) & 1));
    const int64_t n = bmin64(512, npix - j * 512);
    const bool valid = 16 * lane < n;
    uint8_t* slot = myslots + s * 1536 + 48 * lane;
    uint32_t w[12], ob[48], o[12];
    uint32_t badpairs = 0;
    if (valid) {
      const uint4* q = reinterpret_cast<const uint4*>(slot);
      const uint4 q0 = q[0], q1 = q[1], q2 = q[2];
      w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w;
      w[4] = q1.x; w[5] = q1.y; w[6] = q1.z; w[7] = q1.w;
      w[8] = q2.x; w[9] = q2.y; w[10] = q2.z; w[11] = q2.w;
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) {
        const uint32_t bad = b_recolor_pair<MODE>(fp, lut, w, 2 * qq, lc, ob);
        if (MODE == 0) badpairs |= (bad != 0u ? 1u : 0u) << qq;
#pragma unroll
        for (int t = 0; t < 12; ++t)
          if (4 * t + 3 >= 6 * qq && 4 * t + 3 < 6 * qq + 6)
            o[t] = b_pack4(ob[4 * t], ob[4 * t + 1], ob[4 * t + 2], ob[4 * t + 3]);
      }
      uint4* d = reinterpret_cast<uint4*>(slot);
      d[0] = make_uint4(o[0], o[1], o[2], o[3]);
      d[1] = make_uint4(o[4], o[5], o[6], o[7]);
      d[2] = make_uint4(o[8], o[9], o[10], o[11]);
    }
    if (MODE == 0 && __any_sync(0xffffffffu, badpairs != 0u)) {
      uint32_t badmask = 0;
#pragma unroll
      for (int qq = 0; qq < 8; ++qq) badmask |= ((badpairs >> qq) & 1u) * (3u << (2 * qq));
      const uint32_t cnt = __popc(badmask);
      uint32_t incl = cnt;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      unsigned long long base = 0;
      if (lane == 31) base = atomicAdd(rcount, (unsigned long long)total);
      base = __shfl_sync(0xffffffffu, base, 31);
      unsigned long long it = base + incl - cnt;
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        if (!((badmask >> kk) & 1u)) continue;
        const uint32_t rgb = b_byte(w, 3 * kk) | (b_byte(w, 3 * kk + 1) << 8) |
                             (b_byte(w, 3 * kk + 2) << 16);
        const int64_t gp = px0 + j * 512 + 16 * lane + kk;   // pixel index in the batch
        if (it < rcap) {
          ritems[it] = (static_cast<unsigned long long>(gp) << 24) | rgb;
        } else {  // list overflow: fp64 recompute patched into the slot before the store
          const uint32_t px = b_strict_rgb(sps + args.item0 + item, rgb);
          slot[3 * kk] = px & 255u;
          slot[3 * kk + 1] = (px >> 8) & 255u;
          slot[3 * kk + 2] = (px >> 16) & 255u;
        }
        ++it;
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      bulk_s2g(idst + 3 * j * 512, myslots + s * 1536, static_cast<uint32_t>(3 * n));
      bulk_commit();
      if (k >= 1) {
        bulk_wait_read<1>();
        issue_load(k - 1 + kBNSW);
      }
    }
  }
  if (lane == 0) bulk_wait_all();
}

// fp64 repair of the listed pixels; the item is found by binary search.
__global__ void __launch_bounds__(256) k_repair_batch(uint8_t* __restrict__ dst,
                                                      const StrictP* __restrict__ sps,
                                                      const int64_t* __restrict__ off, int nitems,
                                                      const unsigned long long* __restrict__ rcount,
                                                      const unsigned long long* __restrict__ ritems,
                                                      unsigned long long rcap) {
  const unsigned long long n = min(*rcount, rcap);
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n; i += 256ull * gridDim.x) {
    const unsigned long long v = ritems[i];
    const uint32_t rgb = static_cast<uint32_t>(v & 0xffffffu);
    const int64_t gp = static_cast<int64_t>(v >> 24);
    int lo = 0, hi = nitems;          // find item: off[lo] <= gp < off[lo+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (off[mid] <= gp) lo = mid; else hi = mid;
    }
    const uint32_t out = strict_pixel(sps[lo], GlobalLut{sps + lo}, rgb & 255u, (rgb >> 8) & 255u,
                                      rgb >> 16);
    dst[3 * gp] = out & 255u;
    dst[3 * gp + 1] = (out >> 8) & 255u;
    dst[3 * gp + 2] = (out >> 16) & 255u;
  }
}

// strict fp64 recolour of whole items (items whose fast path is not applicable)
__global__ void __launch_bounds__(256) k_strict_batch(const uint8_t* __restrict__ src,
                                                      uint8_t* __restrict__ dst,
                                                      const StrictP* __restrict__ sps,
                                                      const int64_t* __restrict__ off,
                                                      const int32_t* __restrict__ status,
                                                      int nitems) {
  const int item = blockIdx.y;
  if (item >= nitems || status[item] != 1) return;
  const StrictP& sp = sps[item];
  const GlobalLut gl{sps + item};
  for (int64_t i = off[item] + blockIdx.x * 256ll + threadIdx.x; i < off[item + 1];
       i += 256ll * gridDim.x) {
    const uint32_t out = strict_pixel(sp, gl, src[3 * i], src[3 * i + 1], src[3 * i + 2]);
    dst[3 * i] = out & 255u;
    dst[3 * i + 1] = (out >> 8) & 255u;
    dst[3 * i + 2] = (out >> 16) & 255u;
  }
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_build_params(int nitems, const double* i0, const double* luts,
                                const double* bases, const double* p99, const BatchTarget& tgt,
                                double code_lam, int max_sweeps, int exact, FastS* fs, float* flut,
                                StrictP* sps, int32_t* status, cudaStream_t st) {
  if (nitems <= 0) return cudaSuccess;
  k_build_params<<<nitems, 128, 0, st>>>(nitems, i0, luts, bases, p99, tgt, code_lam, max_sweeps,
                                         exact, fs, flut, sps, status);
  return launched();
}

cudaError_t launch_xform_batch(int mode, const uint8_t* src, uint8_t* dst, const float* flut,
                               const StrictP* sps, const BatchArgs& args, unsigned long long* rcount,
                               unsigned long long* ritems, unsigned long long rcap,
                               cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_xform_batch<0>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_xform_batch<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kBSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (args.n <= 0) return cudaSuccess;
  if (mode == 1)
    k_xform_batch<1><<<args.n, 32 * kBW, kBSmem, st>>>(src, dst, flut, sps, args, rcount, ritems,
                                                        rcap);
  else
    k_xform_batch<0><<<args.n, 32 * kBW, kBSmem, st>>>(src, dst, flut, sps, args, rcount, ritems,
                                                        rcap);
  return launched();
}

cudaError_t launch_repair_batch(uint8_t* dst, const StrictP* sps, const int64_t* off, int nitems,
                                unsigned long long* rcount, unsigned long long* ritems,
                                unsigned long long rcap, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_repair_batch<<<sms * 4, 256, 0, st>>>(dst, sps, off, nitems, rcount, ritems, rcap);
  return launched();
}

cudaError_t launch_strict_batch(const uint8_t* src, uint8_t* dst, const StrictP* sps,
                                const int64_t* off, const int32_t* status, int nitems,
                                int64_t max_pix, cudaStream_t st) {
  if (nitems <= 0) return cudaSuccess;
  int64_t gx = (max_pix + 255) / 256;
  if (gx > 64) gx = 64;
  k_strict_batch<<<dim3((unsigned)gx, nitems), 256, 0, st>>>(src, dst, sps, off, status, nitems);
  return launched();
}

}  // namespace spcn
