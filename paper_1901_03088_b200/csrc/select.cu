// select.cu — exact order statistics on the device (K3/K7b).
//
// Reference: percentile src/order_stats.py:11-36 (sorted[lo] + (sorted[hi] -
// sorted[lo]) * frac, rank = p/100*(n-1)) as used by stain_stats
// src/normalize.py:83-100.  A sort is not needed: each query is an MSD radix
// select over the fp64 bit patterns (mapped to order-preserving uint64),
// 11-bit digits, shared-memory histograms, one CTA per query.  Exact by
// construction (integer counting), so percentile-histogram counts are
// bit-exact given identical densities.
#include "select.h"

#include <cooperative_groups.h>
#include "launch_count.h"
#include "spcn_device.cuh"

namespace spcn {

constexpr int kSelThreads = 512;
constexpr int kDigit = 11;
constexpr int kBins = 1 << kDigit;

__device__ __forceinline__ uint64_t key_of(double x) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double val_of(uint64_t k) {
  const uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

// keys: values[stride*j + i] for i in [begin, end) — j = component (stain) picked per query.
// Once the keys sharing the selected prefix fit in shared memory (kSelCand),
// one more pass gathers them there and the remaining digits are resolved on
// the copy — two or three passes over the segment instead of six.
constexpr int kSelCand = 4096;
constexpr int kSelQThreads = 1024;   // k_select: one CTA per query, as wide as it goes

__global__ void __launch_bounds__(kSelQThreads) k_select(const double* __restrict__ values,
                                                       const SelQuery* __restrict__ qs,
                                                       double* __restrict__ out) {
  const SelQuery q = qs[blockIdx.x];
  __shared__ uint32_t hist[kBins];
  __shared__ uint32_t s_scan[kSelQThreads];
  __shared__ uint64_t s_prefix;
  __shared__ int64_t s_k;
  __shared__ uint32_t s_binc;       // keys with the selected prefix
  __shared__ uint32_t s_ncand;
  __shared__ uint64_t cand[kSelCand];
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_k = q.k;
    s_binc = 0xffffffffu;
  }
  const double* v = values + q.offset;
  int used = 0;  // bits of the prefix fixed so far
  bool in_smem = false;
  uint32_t ncand = 0;
  while (used < 64) {
    const int dbits = (64 - used) < kDigit ? (64 - used) : kDigit;
    const int shift = 64 - used - dbits;
    for (int i = threadIdx.x; i < kBins; i += kSelQThreads) hist[i] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    if (!in_smem && used > 0 && s_binc <= (uint32_t)kSelCand) {
      // gather the keys with this prefix into shared memory (any order: the
      // histograms below only count)
      if (threadIdx.x == 0) s_ncand = 0;
      __syncthreads();
      for (int64_t i = q.begin + threadIdx.x; i < q.end; i += kSelQThreads) {
        const uint64_t key = key_of(v[i]);
        if ((key >> (64 - used)) == prefix) cand[atomicAdd(&s_ncand, 1u)] = key;
      }
      __syncthreads();
      ncand = s_ncand;
      in_smem = true;
    }
    if (in_smem) {
      for (uint32_t i = threadIdx.x; i < ncand; i += kSelQThreads) {
        const uint64_t key = cand[i];
        if ((key >> (64 - used)) == prefix)
          atomicAdd(&hist[(uint32_t)((key >> shift) & ((1u << dbits) - 1u))], 1u);
      }
    } else {
      for (int64_t i = q.begin + threadIdx.x; i < q.end; i += kSelQThreads) {
        const uint64_t key = key_of(v[i]);
        if (used == 0 || (key >> (64 - used)) == prefix)
          hist_add_agg(hist, (uint32_t)((key >> shift) & ((1u << dbits) - 1u)));
      }
    }
    __syncthreads();
    // locate the digit holding rank k: per-thread chunk sums + block scan
    constexpr int kPer = kBins / kSelQThreads;  // bins per thread
    uint32_t loc = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) loc += hist[threadIdx.x * kPer + j];
    s_scan[threadIdx.x] = loc;
    __syncthreads();
    for (int off = 1; off < kSelQThreads; off <<= 1) {
      const uint32_t y = threadIdx.x >= off ? s_scan[threadIdx.x - off] : 0u;
      __syncthreads();
      s_scan[threadIdx.x] += y;
      __syncthreads();
    }
    const int64_t k = s_k;
    const int64_t incl = s_scan[threadIdx.x];
    const int64_t excl = incl - loc;
    __syncthreads();
    if (k >= excl && k < incl) {
      int64_t c = excl;
      for (int j = 0; j < kPer; ++j) {
        const int bin = threadIdx.x * kPer + j;
        if (k < c + hist[bin]) {
          s_prefix = (prefix << dbits) | (uint64_t)bin;
          s_k = k - c;
          s_binc = hist[bin];
          break;
        }
        c += hist[bin];
      }
    }
    __syncthreads();
    used += dbits;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = val_of(s_prefix);
}

// Queries for per-segment percentiles of both stains: for segment s and
// stain j, ranks lo, hi (p/100*(n-1)) and n-1 (the max).
__global__ void k_p99_queries(const int64_t* __restrict__ seg, int nseg, int64_t total, double p,
                              SelQuery* __restrict__ qs) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nseg * 2) return;
  const int s = idx >> 1, j = idx & 1;
  const int64_t b = seg[s], e = seg[s + 1], n = e - b;
  const double rank = __dmul_rn(p / 100.0, (double)(n > 0 ? n - 1 : 0));
  const int64_t lo = (int64_t)floor(rank), hi = (int64_t)ceil(rank);
  SelQuery* q = qs + 3 * idx;
  for (int t = 0; t < 3; ++t) {
    q[t].offset = j * total;
    q[t].begin = b;
    q[t].end = e;
  }
  q[0].k = lo;
  q[1].k = hi;
  q[2].k = n > 0 ? n - 1 : 0;
}

// ---------------------------------------------------------------------------
// k_p99_seg: one CTA per (segment, stain) producing the three order
// statistics k_p99_combine needs (ranks lo, hi and the max).  The 99th
// percentile sits just below the maximum, so: pass 1 finds the max key; pass 2
// histograms only the keys within a window below it (bin = (max - key) >>
// kWinShift, i.e. 2^-12-relative bins over two octaves — few values, spread
// over many bins, so the shared-memory atomics do not collide); pass 3
// gathers the keys of the bins holding ranks lo..hi into shared memory, where
// an MSD radix select resolves them exactly.  If the window or the candidate
// list is too small/large for a pathological distribution, the CTA falls back
// to the all-global radix select.  Exact integer counting throughout: the
// same order statistics as a sort.
constexpr int kTop = 13;
constexpr int kTopBins = 1 << kTop;
constexpr int kCand = 8192;
constexpr int kWinShift = 40;   // 2^52 key units per octave -> 2^12 bins per octave

struct SegShared {
  uint32_t hist[kTopBins];
  unsigned long long cand[kCand];
  uint32_t scan[kSelThreads];
  unsigned long long red[kSelThreads / 32];
  int loc_bin;
  long long loc_rank;
  uint32_t ncand;
};

// Block-wide: the bin of hist[0..nb) holding rank k -> sh.loc_bin, and k's
// rank inside that bin -> sh.loc_rank.
__device__ void hist_locate(SegShared& sh, int nb, int64_t k) {
  const int per = nb / kSelThreads;
  uint32_t loc = 0;
  for (int j = 0; j < per; ++j) loc += sh.hist[threadIdx.x * per + j];
  sh.scan[threadIdx.x] = loc;
  __syncthreads();
  for (int off = 1; off < kSelThreads; off <<= 1) {
    const uint32_t y = threadIdx.x >= off ? sh.scan[threadIdx.x - off] : 0u;
    __syncthreads();
    sh.scan[threadIdx.x] += y;
    __syncthreads();
  }
  const int64_t incl = sh.scan[threadIdx.x], excl = incl - loc;
  if (k >= excl && k < incl) {
    int64_t c = excl;
    for (int j = 0; j < per; ++j) {
      const int bin = threadIdx.x * per + j;
      if (k < c + sh.hist[bin]) {
        sh.loc_bin = bin;
        sh.loc_rank = k - c;
        break;
      }
      c += sh.hist[bin];
    }
  }
  __syncthreads();
}

// MSD radix select of rank k among cnt keys src(i), i in [0, cnt).
template <class Src>
__device__ uint64_t radix_select(SegShared& sh, const Src& src, int64_t cnt, int64_t k) {
  uint64_t prefix = 0;
  int used = 0;
  while (used < 64) {
    const int dbits = (64 - used) < kDigit ? (64 - used) : kDigit;
    const int shift = 64 - used - dbits;
    for (int i = threadIdx.x; i < kBins; i += kSelThreads) sh.hist[i] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < cnt; i += kSelThreads) {
      const uint64_t key = src(i);
      if (used == 0 || (key >> (64 - used)) == prefix)
        hist_add_agg(sh.hist, (uint32_t)((key >> shift) & ((1u << dbits) - 1u)));
    }
    __syncthreads();
    hist_locate(sh, kBins, k);
    prefix = (prefix << dbits) | (uint64_t)sh.loc_bin;
    k = sh.loc_rank;
    used += dbits;
    __syncthreads();
  }
  return prefix;
}

__global__ void __launch_bounds__(kSelThreads) k_p99_seg(const double* __restrict__ h,
                                                        int64_t total,
                                                        const int64_t* __restrict__ seg,
                                                        double p, double* __restrict__ sel) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SegShared& sh = *reinterpret_cast<SegShared*>(smem_raw);
  const int idx = blockIdx.x, s = idx >> 1, j = idx & 1;
  const int64_t b = seg[s], e = seg[s + 1], n = e - b;
  if (n <= 0) {
    if (threadIdx.x < 3) sel[3 * idx + threadIdx.x] = 0.0;
    return;
  }
  const double rank = __dmul_rn(p / 100.0, (double)(n - 1));
  const int64_t klo = (int64_t)floor(rank), khi = (int64_t)ceil(rank);
  const double* v = h + j * total + b;
  // pass 1: the max key
  uint64_t mx = 0;
  for (int64_t i = threadIdx.x; i < n; i += kSelThreads) {
    const uint64_t key = key_of(v[i]);
    mx = key > mx ? key : mx;
  }
  for (int off = 16; off; off >>= 1) {
    const uint64_t o = __shfl_xor_sync(0xffffffffu, mx, off);
    mx = o > mx ? o : mx;
  }
  if ((threadIdx.x & 31) == 0) sh.red[threadIdx.x >> 5] = mx;
  for (int i = threadIdx.x; i < kTopBins; i += kSelThreads) sh.hist[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kSelThreads / 32; ++w) mx = sh.red[w] > mx ? sh.red[w] : mx;
    sh.red[0] = mx;
  }
  __syncthreads();
  mx = sh.red[0];
  // pass 2: histogram of the window below the max (bin 0 = the largest keys)
  constexpr uint64_t kWin = (uint64_t)(kTopBins - 1) << kWinShift;
  for (int64_t i = threadIdx.x; i < n; i += kSelThreads) {
    const uint64_t d = mx - key_of(v[i]);
    if (d < kWin) hist_add_agg(sh.hist, (uint32_t)(d >> kWinShift));
  }
  __syncthreads();
  // ranks counted from the top: rt = n - 1 - k
  const int64_t rt_hi = n - 1 - khi, rt_lo = n - 1 - klo;   // rt_hi <= rt_lo
  uint32_t inwin = 0;
  for (int i = threadIdx.x; i < kTopBins; i += kSelThreads) inwin += sh.hist[i];
  for (int off = 16; off; off >>= 1) inwin += __shfl_xor_sync(0xffffffffu, inwin, off);
  if ((threadIdx.x & 31) == 0) sh.scan[threadIdx.x >> 5] = inwin;
  __syncthreads();
  inwin = 0;
  for (int w = 0; w < kSelThreads / 32; ++w) inwin += sh.scan[w];
  __syncthreads();
  uint64_t klo_key = 0, khi_key = 0;
  bool done = false;
  if ((int64_t)inwin > rt_lo) {
    hist_locate(sh, kTopBins, rt_hi);
    const int b1 = sh.loc_bin;
    const int64_t r1 = sh.loc_rank;
    __syncthreads();
    hist_locate(sh, kTopBins, rt_lo);
    const int b2 = sh.loc_bin;
    const int64_t r2 = sh.loc_rank;
    int64_t ncand = 0, before2 = 0;
    for (int t = b1; t <= b2; ++t) {
      if (t == b2) before2 = ncand;
      ncand += sh.hist[t];
    }
    if (ncand <= kCand) {
      // pass 3: gather the keys of bins b1..b2
      if (threadIdx.x == 0) sh.ncand = 0;
      __syncthreads();
      const uint64_t dlo = (uint64_t)b1 << kWinShift, dhi = ((uint64_t)(b2 + 1) << kWinShift);
      for (int64_t i = threadIdx.x; i < n; i += kSelThreads) {
        const uint64_t key = key_of(v[i]);
        const uint64_t d = mx - key;
        if (d >= dlo && d < dhi) sh.cand[atomicAdd(&sh.ncand, 1u)] = key;
      }
      __syncthreads();
      const auto src = [&](int64_t i) -> uint64_t { return sh.cand[i]; };
      // top-rank r within the candidates -> bottom rank ncand - 1 - r
      khi_key = radix_select(sh, src, ncand, ncand - 1 - r1);
      klo_key = radix_select(sh, src, ncand, ncand - 1 - (before2 + r2));
      done = true;
    }
  }
  if (!done) {
    const auto src = [&](int64_t i) -> uint64_t { return key_of(v[i]); };
    __syncthreads();
    klo_key = radix_select(sh, src, n, klo);
    khi_key = radix_select(sh, src, n, khi);
  }
  if (threadIdx.x == 0) {
    sel[3 * idx] = val_of(klo_key);
    sel[3 * idx + 1] = val_of(khi_key);
    sel[3 * idx + 2] = val_of(mx);
  }
}

// k_p99_seg_cluster: the same three passes for ONE large segment (the
// single-slide fit's 100 k samples) on a cluster of kCl CTAs per stain: every
// CTA streams 1/kCl of the values; the max, the window histogram (each CTA
// sums 1/kCl of the bins across the cluster through distributed shared
// memory) and the candidate list are combined in CTA 0's shared memory, which
// then runs the radix select.  Same bins, same candidates, same select as
// k_p99_seg — with kCl times the streaming parallelism.
constexpr int kCl = 8;

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kSelThreads)
    k_p99_seg_cluster(const double* __restrict__ h, int64_t total,
                      const int64_t* __restrict__ seg, double p, double* __restrict__ sel) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SegShared& sh = *reinterpret_cast<SegShared*>(smem_raw);
  __shared__ unsigned long long s_mx;
  __shared__ int s_go, s_b1, s_b2;
  __shared__ long long s_r1, s_r2;
  const int cr = (int)cl.block_rank();
  const int idx = blockIdx.x / kCl, s = idx >> 1, j = idx & 1;
  const int64_t b = seg[s], e = seg[s + 1], n = e - b;
  if (n <= 0) {                                    // uniform over the cluster
    if (cr == 0 && threadIdx.x < 3) sel[3 * idx + threadIdx.x] = 0.0;
    return;
  }
  const double* v = h + j * total + b;
  SegShared& sh0 = *cl.map_shared_rank(&sh, 0);
  const int64_t i0 = (int64_t)cr * kSelThreads + threadIdx.x, step = (int64_t)kCl * kSelThreads;
  // pass 1: the max key (per CTA, then across the cluster)
  uint64_t mx = 0;
  for (int64_t i = i0; i < n; i += step) {
    const uint64_t key = key_of(v[i]);
    mx = key > mx ? key : mx;
  }
  for (int off = 16; off; off >>= 1) {
    const uint64_t o = __shfl_xor_sync(0xffffffffu, mx, off);
    mx = o > mx ? o : mx;
  }
  if ((threadIdx.x & 31) == 0) sh.red[threadIdx.x >> 5] = mx;
  for (int i = threadIdx.x; i < kTopBins; i += kSelThreads) sh.hist[i] = 0;
  if (threadIdx.x == 0) sh.ncand = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kSelThreads / 32; ++w) mx = sh.red[w] > mx ? sh.red[w] : mx;
    s_mx = mx;
  }
  cl.sync();
  mx = 0;
  for (int r = 0; r < kCl; ++r) {
    const uint64_t o = *cl.map_shared_rank(&s_mx, r);
    mx = o > mx ? o : mx;
  }
  // pass 2: window histogram, per CTA, then summed bin-slice by bin-slice into
  // CTA 0's candidate area (free until pass 3) and copied to its histogram
  constexpr uint64_t kWin = (uint64_t)(kTopBins - 1) << kWinShift;
  for (int64_t i = i0; i < n; i += step) {
    const uint64_t d = mx - key_of(v[i]);
    if (d < kWin) atomicAdd(&sh.hist[(uint32_t)(d >> kWinShift)], 1u);
  }
  cl.sync();
  uint32_t* sum0 = reinterpret_cast<uint32_t*>(sh0.cand);
  for (int bin = cr * kSelThreads + threadIdx.x; bin < kTopBins; bin += kCl * kSelThreads) {
    uint32_t c = 0;
    for (int r = 0; r < kCl; ++r) c += cl.map_shared_rank(sh.hist, r)[bin];
    sum0[bin] = c;
  }
  cl.sync();
  const double rank = __dmul_rn(p / 100.0, (double)(n - 1));
  const int64_t klo = (int64_t)floor(rank), khi = (int64_t)ceil(rank);
  const int64_t rt_hi = n - 1 - khi, rt_lo = n - 1 - klo;   // ranks from the top
  if (cr == 0) {
    const uint32_t* sum = reinterpret_cast<const uint32_t*>(sh.cand);
    uint32_t inwin = 0;
    for (int i = threadIdx.x; i < kTopBins; i += kSelThreads) {
      sh.hist[i] = sum[i];
      inwin += sum[i];
    }
    for (int off = 16; off; off >>= 1) inwin += __shfl_xor_sync(0xffffffffu, inwin, off);
    if ((threadIdx.x & 31) == 0) sh.scan[threadIdx.x >> 5] = inwin;
    __syncthreads();
    inwin = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) inwin += sh.scan[w];
    __syncthreads();
    int go = 0;
    if ((int64_t)inwin > rt_lo) {
      hist_locate(sh, kTopBins, rt_hi);
      const int b1 = sh.loc_bin;
      const int64_t r1 = sh.loc_rank;
      __syncthreads();
      hist_locate(sh, kTopBins, rt_lo);
      const int b2 = sh.loc_bin;
      const int64_t r2 = sh.loc_rank;
      int64_t ncand = 0, before2 = 0;
      for (int t = b1; t <= b2; ++t) {
        if (t == b2) before2 = ncand;
        ncand += sh.hist[t];
      }
      if (ncand <= kCand) {
        go = 1;
        if (threadIdx.x == 0) {
          s_b1 = b1;
          s_b2 = b2;
          s_r1 = r1;
          s_r2 = before2 + r2;
          sh.ncand = 0;
        }
      }
    }
    if (threadIdx.x == 0) s_go = go;
  }
  cl.sync();
  const int go = *cl.map_shared_rank(&s_go, 0);
  if (go) {
    // pass 3: every CTA appends the keys of bins b1..b2 to CTA 0's list
    const int b1 = *cl.map_shared_rank(&s_b1, 0), b2 = *cl.map_shared_rank(&s_b2, 0);
    const uint64_t dlo = (uint64_t)b1 << kWinShift, dhi = ((uint64_t)(b2 + 1) << kWinShift);
    for (int64_t i = i0; i < n; i += step) {
      const uint64_t key = key_of(v[i]);
      const uint64_t d = mx - key;
      if (d >= dlo && d < dhi) sh0.cand[atomicAdd(&sh0.ncand, 1u)] = key;
    }
  }
  cl.sync();
  if (cr != 0) return;
  uint64_t klo_key, khi_key;
  if (go) {
    const int64_t ncand = sh.ncand;
    const auto src = [&](int64_t i) -> uint64_t { return sh.cand[i]; };
    khi_key = radix_select(sh, src, ncand, ncand - 1 - s_r1);
    klo_key = radix_select(sh, src, ncand, ncand - 1 - s_r2);
  } else {
    const auto src = [&](int64_t i) -> uint64_t { return key_of(v[i]); };
    klo_key = radix_select(sh, src, n, klo);
    khi_key = radix_select(sh, src, n, khi);
  }
  if (threadIdx.x == 0) {
    sel[3 * idx] = val_of(klo_key);
    sel[3 * idx + 1] = val_of(khi_key);
    sel[3 * idx + 2] = val_of(mx);
  }
}

__global__ void k_p99_combine(const int64_t* __restrict__ seg, int nseg, double p,
                              const double* __restrict__ sel, double* __restrict__ p99,
                              int32_t* __restrict__ absent) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nseg * 2) return;
  const int s = idx >> 1;
  const int64_t n = seg[s + 1] - seg[s];
  if (n <= 0) {
    p99[idx] = 0.0;
    absent[idx] = 1;
    return;
  }
  const double a = sel[3 * idx], b = sel[3 * idx + 1], mx = sel[3 * idx + 2];
  const double rank = __dmul_rn(p / 100.0, (double)(n - 1));
  const double frac = __dsub_rn(rank, floor(rank));
  p99[idx] = __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), frac));
  absent[idx] = (mx <= 0.0) ? 1 : 0;   // s.max(initial=0) <= 0 (src/normalize.py:91)
}

__global__ void k_build_queries(const int64_t* __restrict__ b, const int64_t* __restrict__ e,
                                const int64_t* __restrict__ k, int nq, SelQuery* __restrict__ qs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq) return;
  qs[i].offset = 0;
  qs[i].begin = b[i];
  qs[i].end = e[i];
  qs[i].k = k[i];
}

cudaError_t launch_build_queries(const int64_t* b, const int64_t* e, const int64_t* k, int nq,
                                 SelQuery* qs, cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  k_build_queries<<<(nq + 127) / 128, 128, 0, st>>>(b, e, k, nq, qs);
  return launched();
}

cudaError_t launch_select(const double* values, const SelQuery* qs, int nq, double* out,
                          cudaStream_t st) {
  if (nq <= 0) return cudaSuccess;
  k_select<<<nq, kSelQThreads, 0, st>>>(values, qs, out);
  return launched();
}

cudaError_t launch_p99(const double* h, int64_t total, const int64_t* seg, int nseg, double p,
                       SelQuery* qbuf, double* selbuf, double* p99, int32_t* absent,
                       cudaStream_t st) {
  if (nseg <= 0) return cudaSuccess;
  const int n2 = nseg * 2;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e0 = cudaFuncSetAttribute(k_p99_seg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)sizeof(SegShared));
    if (e0 != cudaSuccess) return e0;
    attr = true;
  }
  (void)qbuf;
  static bool attr_cl = false;
  if (!attr_cl) {
    const cudaError_t e0 = cudaFuncSetAttribute(k_p99_seg_cluster,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)sizeof(SegShared));
    if (e0 != cudaSuccess) return e0;
    attr_cl = true;
  }
  // a single large segment (one slide's sample) is latency-bound on one CTA
  // per stain: spread it over a cluster; many segments keep one CTA each
  if (nseg == 1) {
    k_p99_seg_cluster<<<n2 * kCl, kSelThreads, sizeof(SegShared), st>>>(h, total, seg, p, selbuf);
  } else {
    k_p99_seg<<<n2, kSelThreads, sizeof(SegShared), st>>>(h, total, seg, p, selbuf);
  }
  cudaError_t e = launched();
  if (e != cudaSuccess) return e;
  k_p99_combine<<<(n2 + 127) / 128, 128, 0, st>>>(seg, nseg, p, selbuf, p99, absent);
  return launched();
}

// ---------------------------------------------------------------------------
// Weighted per-segment percentile over colour-table entries: segment s holds
// ucount[s] entries at seg[s] with densities h[j*total + i] and pixel counts
// w[i] (summing to n = seg[s+1] - seg[s] samples).  The order statistics of
// the expanded multiset are found by an MSD radix select over the fp64 bit
// patterns (non-negative doubles order like their bits) with the counts as
// weights — exact, the same values a sort of the n samples gives — staged in
// shared memory when the segment fits.  Interpolation and the absent rule as
// k_p99_combine.
constexpr int kWThreads = 512;
constexpr int kWCap = 12288;   // entries staged in shared memory (k_colour_table's fill limit)
constexpr bool kWStage = false;   // with the candidate gather, 3-4 passes read L2 directly

__device__ __forceinline__ unsigned long long wkey(double x) {
  const unsigned long long b = __double_as_longlong(x);
  return b == 0x8000000000000000ull ? 0ull : b;   // -0 sorts as +0
}

__global__ void __launch_bounds__(kWThreads) k_p99_weighted(
    const double* __restrict__ h, int64_t total, const uint32_t* __restrict__ w,
    const int32_t* __restrict__ ucount, const int64_t* __restrict__ seg, int nseg, double p,
    double* __restrict__ p99, int32_t* __restrict__ absent) {
  extern __shared__ __align__(16) unsigned long long s_key[];   // [kWCap]
  uint32_t* s_w = reinterpret_cast<uint32_t*>(s_key + kWCap);    // [kWCap]
  __shared__ uint32_t hist[256];
  __shared__ unsigned long long s_red[kWThreads / 32];
  __shared__ unsigned long long s_bc[2];   // chosen prefix, remaining rank
  __shared__ uint32_t s_binw;
  // entries sharing the first two digits with the selected rank: after two
  // passes they are gathered here and the last six digits only visit them
  constexpr int kWCand = 1024;
  __shared__ unsigned long long c_key[kWCand];
  __shared__ uint32_t c_w[kWCand];
  __shared__ int s_nc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
    const int64_t o0 = seg[sg], n = seg[sg + 1] - o0;
    const int ne = ucount[sg];
    for (int j = 0; j < 2; ++j) {
      const int idx = 2 * sg + j;
      if (n <= 0 || ne <= 0) {
        if (tid == 0) {
          p99[idx] = 0.0;
          absent[idx] = 1;
        }
        continue;
      }
      const double* hv = h + (int64_t)j * total + o0;
      const uint32_t* wv = w + o0;
      const bool staged = kWStage && ne <= kWCap;
      if (staged)
        for (int i = tid; i < ne; i += kWThreads) {
          s_key[i] = wkey(hv[i]);
          s_w[i] = wv[i];
        }
      __syncthreads();
      auto key_at = [&](int i) { return staged ? s_key[i] : wkey(hv[i]); };
      auto w_at = [&](int i) { return staged ? s_w[i] : wv[i]; };
      // block max / min-above reduction helpers
      auto block_max = [&](unsigned long long v) {
        for (int off = 16; off; off >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (lane == 0) s_red[warp] = v;
        __syncthreads();
        unsigned long long r = 0;
        for (int k = 0; k < kWThreads / 32; ++k) r = max(r, s_red[k]);
        __syncthreads();
        return r;
      };
      auto block_min = [&](unsigned long long v) {
        for (int off = 16; off; off >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, off));
        if (lane == 0) s_red[warp] = v;
        __syncthreads();
        unsigned long long r = ~0ull;
        for (int k = 0; k < kWThreads / 32; ++k) r = min(r, s_red[k]);
        __syncthreads();
        return r;
      };
      // weighted MSD radix select of rank k: returns the key; s_binw = the
      // weight of entries equal to it, s_bc[1] = k's rank among them
      auto select = [&](int64_t k) {
        unsigned long long prefix = 0;
        bool cand = false;
        int nc = 0;
        for (int shift = 56; shift >= 0; shift -= 8) {
          if (tid < 256) hist[tid] = 0;
          __syncthreads();
          const unsigned long long mask = shift == 56 ? 0ull : (~0ull << (shift + 8));
          if (cand) {
            for (int i = tid; i < nc; i += kWThreads) {
              const unsigned long long kk = c_key[i];
              if ((kk & mask) == prefix) atomicAdd(&hist[(kk >> shift) & 255u], c_w[i]);
            }
          } else {
            for (int i = tid; i < ne; i += kWThreads) {
              const unsigned long long kk = key_at(i);
              if ((kk & mask) == prefix) atomicAdd(&hist[(kk >> shift) & 255u], w_at(i));
            }
          }
          __syncthreads();
          if (warp == 0) {   // warp scan of 256 bins (8 per lane)
            uint32_t loc[8], sum = 0;
            for (int b = 0; b < 8; ++b) {
              loc[b] = hist[lane * 8 + b];
              sum += loc[b];
            }
            uint32_t incl = sum;
            for (int off = 1; off < 32; off <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
              if (lane >= off) incl += y;
            }
            uint32_t before = incl - sum;
            for (int b = 0; b < 8; ++b) {
              if (k >= (int64_t)before && k < (int64_t)(before + loc[b])) {
                s_bc[0] = prefix | ((unsigned long long)(lane * 8 + b) << shift);
                s_bc[1] = (unsigned long long)(k - before);
                s_binw = loc[b];
              }
              before += loc[b];
            }
          }
          __syncthreads();
          prefix = s_bc[0];
          k = (int64_t)s_bc[1];
          __syncthreads();
          if (!cand && shift == 48) {   // gather the entries with this 16-bit prefix
            if (tid == 0) s_nc = 0;
            __syncthreads();
            for (int i = tid; i < ne; i += kWThreads) {
              const unsigned long long kk = key_at(i);
              if ((kk & (~0ull << 48)) == prefix) {
                const int j = atomicAdd(&s_nc, 1);
                if (j < kWCand) {
                  c_key[j] = kk;
                  c_w[j] = w_at(i);
                }
              }
            }
            __syncthreads();
            nc = s_nc;
            cand = nc <= kWCand;      // (more: keep scanning every entry)
            __syncthreads();
          }
        }
        return prefix;
      };
      const double rank = __dmul_rn(p / 100.0, (double)(n - 1));
      const int64_t klo = (int64_t)floor(rank), khi = (int64_t)ceil(rank);
      unsigned long long mx = 0;
      for (int i = tid; i < ne; i += kWThreads) mx = max(mx, key_at(i));
      mx = block_max(mx);
      const unsigned long long klo_key = select(klo);
      const unsigned long long rem = s_bc[1];
      const uint32_t binw = s_binw;
      unsigned long long khi_key = klo_key;
      if (khi != klo && rem + 1 >= binw) {   // the next distinct value
        unsigned long long nx = ~0ull;
        for (int i = tid; i < ne; i += kWThreads) {
          const unsigned long long kk = key_at(i);
          if (kk > klo_key) nx = min(nx, kk);
        }
        khi_key = block_min(nx);
      }
      if (tid == 0) {
        const double a = __longlong_as_double(klo_key), b = __longlong_as_double(khi_key);
        const double frac = __dsub_rn(rank, floor(rank));
        p99[idx] = __dadd_rn(a, __dmul_rn(__dsub_rn(b, a), frac));
        absent[idx] = mx == 0ull ? 1 : 0;   // s.max(initial=0) <= 0 (src/normalize.py:91)
      }
      __syncthreads();
    }
  }
}

cudaError_t launch_p99_weighted(const double* h, int64_t total, const uint32_t* w,
                                const int32_t* ucount, const int64_t* seg, int nseg, double p,
                                double* p99, int32_t* absent, cudaStream_t st) {
  if (nseg <= 0) return cudaSuccess;
  constexpr int smem = kWStage ? kWCap * (8 + 4) : 0;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e =
        cudaFuncSetAttribute(k_p99_weighted, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int g = nseg < 4 * sms ? nseg : 4 * sms;
  k_p99_weighted<<<g, kWThreads, smem, st>>>(h, total, w, ucount, seg, nseg, p, p99, absent);
  return launched();
}

}  // namespace spcn
