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
//   k_repair_items     fp64 reference-order recompute of uncertified pixels,
//                      one CTA per item over its segment of the per-CTA
//                      repair lists k_xform_batch wrote.
#include "batch.h"
#include "launch_count.h"
#include "params.cuh"
#include "recolor.cuh"
#include "spcn_device.cuh"

namespace spcn {

constexpr int kBW = 16;                      // warps per CTA
constexpr int kBNSW = 3;                     // ring slots per warp
constexpr int kBNSub = 2;                    // 512-px sub-slices per slot
constexpr int kBRep = 24;                    // OD table replicas (mixed layout, recolor.cuh)
constexpr uint32_t kBAbs = 4096;             // absolute shared address of the OD table
constexpr int kBSlicePx = 512 * kBNSub;
constexpr int kBSlotBytes = 3 * kBSlicePx;
constexpr int kBLut = LutLayout<kBRep>::kBytes;
constexpr size_t kBSmem = kBAbs + kBLut + (size_t)kBW * kBNSW * kBSlotBytes + kBW * kBNSW * 8;
static_assert(kBSmem <= 227 * 1024, "shared memory budget");

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
struct SmemLut {
  const double* t;
  __device__ double operator()(int c, uint32_t i) const { return t[c * 256 + i]; }
};

struct GlobalLut {
  const StrictP* p;
  __device__ double operator()(int c, uint32_t x) const { return p->lut[c][x]; }
};

// Persistent: CTA b recolours items b, b + grid, ... (fast-path items only,
// status 0).  Per item the CTA rebuilds the replicated OD table from the
// item's fp32 table and loads the item's FastS into registers; every warp
// then runs its TMA ring over the item's slices j = warp, warp + kBW, ...
// Lane 0's producer cursor walks the same (item, slice) sequence ahead of the
// consumer, so the ring keeps streaming across item boundaries.
template <int MODE>
__global__ void __launch_bounds__(32 * kBW, 1)
    k_xform_batch(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int nitems,
                  const int64_t* __restrict__ off, const int32_t* __restrict__ status,
                  const FastS* __restrict__ fs, const float* __restrict__ flut,
                  BatchRepair br) {
  // EXACT: this CTA's own repair list (no contention with other CTAs); the
  // items it recolours leave contiguous segments of it, recorded per item
  // for k_repair_items
  RepairList rl{br.counts + blockIdx.x, br.items + (size_t)blockIdx.x * br.cap_cta, br.cap_cta};
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const uint32_t wbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  if (wbase > kBAbs) __trap();                 // layout assumption (window base <= 4 KB)
  uint8_t* smem = smem_raw + (kBAbs - wbase);  // the OD table at absolute kBAbs
  const uint8_t* lut = smem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* myslots = smem + kBLut + (size_t)warp * kBNSW * kBSlotBytes;
  uint64_t* mybar = reinterpret_cast<uint64_t*>(smem + kBLut + (size_t)kBW * kBNSW * kBSlotBytes) +
                    warp * kBNSW;
  const int G = gridDim.x;
  auto next_item = [&](int it) {
    while (it < nitems && status[it] != 0) it += G;
    return it;
  };
  auto nslices = [&](int it) { return (off[it + 1] - off[it] + kBSlicePx - 1) / kBSlicePx; };
  if (lane == 0) {
    for (int q = 0; q < kBNSW; ++q) mbar_init(&mybar[q], 1);
    mbar_fence_init();
  }
  uint32_t lc[3];
  LutLayout<kBRep>::lane_consts(lane, lc);

  // producer cursor (lane 0): next (item, slice) to load and loads issued so far
  int p_item = next_item(blockIdx.x);
  int64_t p_j = warp, p_loads = 0;
  uint64_t pol = 0;
  auto settle = [&]() {
    while (p_item < nitems && p_j >= nslices(p_item)) {
      p_item = next_item(p_item + G);
      p_j = warp;
    }
  };
  auto issue_load = [&]() {   // lane 0 only
    settle();
    if (p_item >= nitems) return;
    const int q = (int)(p_loads % kBNSW);
    const int64_t base = off[p_item], npx = off[p_item + 1] - base;
    const uint32_t bytes = static_cast<uint32_t>(3 * bmin64(kBSlicePx, npx - p_j * kBSlicePx));
    mbar_expect_tx(&mybar[q], bytes);
    bulk_g2s(myslots + q * kBSlotBytes, src + 3 * (base + p_j * kBSlicePx), bytes, &mybar[q], pol);
    ++p_loads;
    p_j += kBW;
  };
  __syncthreads();   // barriers initialised
  if (lane == 0) {
    pol = policy_evict_first();
    for (int q = 0; q < kBNSW; ++q) issue_load();
  }

  int64_t k = 0;   // this warp's consumed-slice sequence number
  int prev = -1;
  for (int it = next_item(blockIdx.x); it < nitems; it = next_item(it + G)) {
    __syncthreads();                                   // previous item's table no longer read
    if (MODE == 0 && tid == 0) {                       // segment bookkeeping (EXACT)
      const unsigned long long c = *(volatile unsigned long long*)rl.count;
      if (prev >= 0) br.seg[3 * prev + 1] = c;
      br.seg[3 * it] = c;
      br.seg[3 * it + 2] = blockIdx.x;
      prev = it;
    }
    LutLayout<kBRep>::fill(smem, flut + (int64_t)it * 768, tid, 32 * kBW);
    const FastS fp = fs[it];
    __syncthreads();
    const int64_t base = off[it], npx = off[it + 1] - base;
    const int64_t nsl = (npx + kBSlicePx - 1) / kBSlicePx;
    for (int64_t j = warp; j < nsl; j += kBW, ++k) {
      const int q = (int)(k % kBNSW);
      mbar_wait(&mybar[q], (uint32_t)((k / kBNSW) & 1));
      const int64_t n = bmin64(kBSlicePx, npx - j * kBSlicePx);
      uint8_t* sbase = myslots + q * kBSlotBytes;
#pragma unroll
      for (int u = 0; u < kBNSub; ++u)
        recolor_block<MODE, kBAbs>(fp, lut, lc, sbase + u * 1536 + 48 * lane, u * 512 + 16 * lane < n,
                            base + j * kBSlicePx + u * 512 + 16 * lane, rl, lane, fp.I);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        bulk_s2g(dst + 3 * (base + j * kBSlicePx), sbase, static_cast<uint32_t>(3 * n));
        bulk_commit();
        if (k >= 1) {
          bulk_wait_read<1>();     // the store of slice k-1 has read its slot
          issue_load();            // refill it (load number k-1+kBNSW)
        }
      }
    }
  }
  if (MODE == 0) {
    __syncthreads();
    if (tid == 0 && prev >= 0) br.seg[3 * prev + 1] = *(volatile unsigned long long*)rl.count;
  }
  if (lane == 0) bulk_wait_all();
}

// fp64 repair, one CTA per item: the item's segment of its CTA's list (the
// pixels k_xform_batch could not certify), with the item's fp64 OD table in
// shared memory and its Gram factors formed once; if the segment overflowed
// the CTA's list, every pixel of the item is recomputed instead.  Exact
// either way (strict_pixel = the reference's operation order).
// Per item, the uncertified pixels' colours are deduplicated first: the
// certification outcome is a function of the colour, so a colour that fails
// fails for every pixel that has it, and the list repeats colours about as
// often as the item does (~10x).  Phase 1 inserts the list's colours into a
// shared-memory table, phase 2 evaluates each distinct colour once in fp64,
// phase 3 writes every listed pixel from the table (colours that did not fit
// in the table are evaluated directly) — the same bytes, a fraction of the
// fp64 work.
constexpr int kRepThreads = 1024;
constexpr int kRepBits = 13, kRepSlots = 1 << kRepBits;
constexpr uint32_t kRepEmpty = 0xffffffffu;

__device__ __forceinline__ uint32_t rep_slot(uint32_t rgb) {
  return (rgb * 2654435761u) >> (32 - kRepBits);
}

__global__ void __launch_bounds__(kRepThreads) k_repair_items(const uint8_t* __restrict__ src,
                                                              uint8_t* __restrict__ dst,
                                                              const StrictP* __restrict__ sps,
                                                              const int64_t* __restrict__ off,
                                                              const int32_t* __restrict__ status,
                                                              int nitems, BatchRepair br) {
  const int it = blockIdx.x;
  if (it >= nitems || status[it] != 0) return;
  const unsigned long long s0 = br.seg[3 * it], s1 = br.seg[3 * it + 1];
  if (s1 <= s0) return;                               // nothing to repair

  __shared__ double lut[3 * 256];
  extern __shared__ uint32_t rtab[];                  // keys [kRepSlots] | outputs [kRepSlots]
  uint32_t* rkey = rtab;
  uint32_t* rout = rtab + kRepSlots;
  const StrictP& sp = sps[it];
  for (int i = threadIdx.x; i < 3 * 256; i += kRepThreads) lut[i] = sp.lut[i >> 8][i & 255];
  const NnlsGram G = gram_of(sp);
  if (s1 > br.cap_cta) {                              // the list overflowed: whole item
    __syncthreads();
    for (int64_t i = off[it] + threadIdx.x; i < off[it + 1]; i += kRepThreads) {
      const uint32_t out = strict_pixel(sp, G, SmemLut{lut}, src[3 * i], src[3 * i + 1],
                                        src[3 * i + 2]);
      dst[3 * i] = out & 255u;
      dst[3 * i + 1] = (out >> 8) & 255u;
      dst[3 * i + 2] = (out >> 16) & 255u;
    }
    return;
  }
  for (int i = threadIdx.x; i < kRepSlots; i += kRepThreads) rkey[i] = kRepEmpty;
  __syncthreads();
  const unsigned long long* items = br.items + (size_t)br.seg[3 * it + 2] * br.cap_cta;
  // phase 1: distinct colours of the list (a colour that finds no slot within
  // 32 probes is evaluated directly in phase 3)
  for (unsigned long long i = s0 + threadIdx.x; i < s1; i += kRepThreads) {
    const uint32_t rgb = static_cast<uint32_t>(items[i] & 0xffffffu);
    uint32_t sl = rep_slot(rgb);
    for (int probe = 0; probe < 32; ++probe, sl = (sl + 1) & (kRepSlots - 1)) {
      const uint32_t k = atomicCAS(&rkey[sl], kRepEmpty, rgb);
      if (k == kRepEmpty || k == rgb) break;
    }
  }
  __syncthreads();
  // phase 2: one fp64 evaluation per distinct colour
  for (int i = threadIdx.x; i < kRepSlots; i += kRepThreads) {
    const uint32_t rgb = rkey[i];
    if (rgb != kRepEmpty)
      rout[i] = strict_pixel(sp, G, SmemLut{lut}, rgb & 255u, (rgb >> 8) & 255u, rgb >> 16);
  }
  __syncthreads();
  // phase 3: every listed pixel from the table
  for (unsigned long long i = s0 + threadIdx.x; i < s1; i += kRepThreads) {
    const unsigned long long v = items[i];
    const uint32_t rgb = static_cast<uint32_t>(v & 0xffffffu);
    const int64_t gp = static_cast<int64_t>(v >> 24);
    uint32_t sl = rep_slot(rgb), out = 0;
    bool hit = false;
    for (int probe = 0; probe < 32; ++probe, sl = (sl + 1) & (kRepSlots - 1)) {
      const uint32_t k = rkey[sl];
      if (k == rgb) {
        out = rout[sl];
        hit = true;
        break;
      }
      if (k == kRepEmpty) break;
    }
    if (!hit) out = strict_pixel(sp, G, SmemLut{lut}, rgb & 255u, (rgb >> 8) & 255u, rgb >> 16);
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
  const NnlsGram G = gram_of(sp);
  for (int64_t i = off[item] + blockIdx.x * 256ll + threadIdx.x; i < off[item + 1];
       i += 256ll * gridDim.x) {
    const uint32_t out = strict_pixel(sp, G, gl, src[3 * i], src[3 * i + 1], src[3 * i + 2]);
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

int batch_grid(int nitems) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
  }
  return nitems < sms ? nitems : sms;
}

cudaError_t launch_xform_batch(int mode, const uint8_t* src, uint8_t* dst, int nitems,
                               const int64_t* off, const int32_t* status, const FastS* fs,
                               const float* flut, const BatchRepair& br, cudaStream_t st) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_xform_batch<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kBSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_xform_batch<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kBSmem);
    if (e != cudaSuccess) {
      sms = 0;
      return e;
    }
  }
  if (nitems <= 0) return cudaSuccess;
  const int grid = batch_grid(nitems);
  if (mode == 1)
    k_xform_batch<1><<<grid, 32 * kBW, kBSmem, st>>>(src, dst, nitems, off, status, fs, flut, br);
  else
    k_xform_batch<0><<<grid, 32 * kBW, kBSmem, st>>>(src, dst, nitems, off, status, fs, flut, br);
  return launched();
}

cudaError_t launch_repair_items(const uint8_t* src, uint8_t* dst, const StrictP* sps,
                                const int64_t* off, const int32_t* status, int nitems,
                                const BatchRepair& br, cudaStream_t st) {
  if (nitems <= 0) return cudaSuccess;
  constexpr int kSmem = 2 * kRepSlots * sizeof(uint32_t);
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(k_repair_items,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  k_repair_items<<<nitems, kRepThreads, kSmem, st>>>(src, dst, sps, off, status, nitems, br);
  return launched();
}

cudaError_t launch_strict_batch(const uint8_t* src, uint8_t* dst, const StrictP* sps,
                                const int64_t* off, const int32_t* status, int nitems,
                                int64_t max_pix, cudaStream_t st) {
  if (nitems <= 0) return cudaSuccess;
  int64_t gx = (max_pix + 255) / 256;
  if (gx > 64) gx = 64;
  for (int i0 = 0; i0 < nitems; i0 += kMaxGridY) {   // gridDim.y <= 65535
    const int ni = nitems - i0 < kMaxGridY ? nitems - i0 : kMaxGridY;
    k_strict_batch<<<dim3((unsigned)gx, ni), 256, 0, st>>>(src, dst, sps + i0, off + i0,
                                                           status + i0, ni);
    const cudaError_t e = launched();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace spcn
