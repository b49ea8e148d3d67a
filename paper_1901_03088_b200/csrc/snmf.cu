// snmf.cu — batched sparse-NMF stain-basis fit (K6) and batched density
// coding of the fit samples (K7a).
//
// Reference: fit_basis src/stain_sep.py:239-336 (+ _w_step :210-236,
// snmf_objective :204-207, order_stains :104-116) and code_densities
// src/stain_sep.py:168-201 as used by fit src/pipeline.py:225-226.
//
// One thread-block CLUSTER per problem (cluster size 1 for the 4096-patch
// batch, 8 for a single whole-slide fit).  Each CTA owns a contiguous slice
// of the problem's sampled pixels; OD values are re-read through the
// problem's 256-entry table from the 3-byte RGB sample (24 B/px of fp64 OD
// never touch HBM); stain densities H live in a global scratch array.
// Every reduction (objective, V H^T, H H^T, sum H) is a fixed-order
// warp-shuffle → CTA → DSMEM cluster tree, and every CTA of the cluster
// combines the partials in the same rank order, so all CTAs hold bitwise
// identical totals and take identical control decisions (W-step accept,
// convergence) without a broadcast.  Scalar arithmetic that numpy routes
// through BLAS (3-vector dots, the K=2 matmul element) uses the same FMA
// chain numpy/OpenBLAS uses; long reductions differ from BLAS only in
// summation order (basis within cosine 1e-3, measured
// ~1e-15).
#include <cooperative_groups.h>
#include <cstdlib>
#include <cstring>

#include "launch_count.h"
#include "ctable.cuh"
#include "snmf.h"
#include "spcn_device.cuh"

namespace cg = cooperative_groups;

namespace spcn {

constexpr int kSnMaxThreads = 512;
constexpr int kNStat = 12;  // rr, s0, s1, vht[3][2], hht00, hht01, hht11

__device__ __forceinline__ double fma_dot3(double a0, double a1, double a2, double b0, double b1,
                                           double b2) {
  // numpy 1-D @ 1-D of length 3 on OpenBLAS: fma(a2,b2, fma(a1,b1, a0*b0))
  return __fma_rn(a2, b2, __fma_rn(a1, b1, __dmul_rn(a0, b0)));
}

template <int NT, int N>
__device__ __forceinline__ void cta_reduce(double (&v)[N], double* warp_part,
                                           double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < N; ++q)
#pragma unroll
    for (int off = 16; off; off >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], off);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < N; ++q) warp_part[warp * N + q] = v[q];
  __syncthreads();
  if (threadIdx.x < N) {
    double s = 0.0;
    for (int w = 0; w < NT / 32; ++w) s += warp_part[w * N + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

struct SnmfShared {
  double lut[3 * 256];
  double w[6];            // current basis, row-major [c][j]
  double cand[6];
  double part[2][kNStat]; // double-buffered CTA partials (read by the cluster)
  double tot[kNStat];     // cluster totals (identical in every CTA)
  double warp_part[kSnMaxThreads / 32][kNStat];
  double g[4];            // g00, g01, g11, det
  int flag;
};

// NT threads per CTA, MINB CTAs per SM (512 x 1 for the cluster fit of one
// slide; 128 x 4 for the one-CTA-per-problem batch, see launch_snmf).
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_snmf(
    const uint8_t* __restrict__ samples, const double* __restrict__ od,
    const int64_t* __restrict__ offsets, int nprob, const double* __restrict__ luts,
    const __grid_constant__ SnmfArgs a, int* __restrict__ ticket,
    int64_t total, double* __restrict__ basis_out, double* __restrict__ hist_out,
    int32_t* __restrict__ info_out, const uint32_t* __restrict__ ukey,
    const uint32_t* __restrict__ ucnt, const int32_t* __restrict__ ucount) {
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int ncl = gridDim.x / cs;
  const int cid = blockIdx.x / cs;
  __shared__ SnmfShared sh;
  const int tid = threadIdx.x;
  int phase = 0;

  // cluster-wide sum of a CTA partial: every CTA reads all ranks in order
  auto cluster_total = [&](int nstat) {
    cluster.sync();
    if (tid < nstat) {
      double s = 0.0;
      for (int r = 0; r < cs; ++r) {
        const double* rp = cluster.map_shared_rank(&sh.part[phase & 1][0], r);
        s += rp[tid];
      }
      sh.tot[tid] = s;
    }
    ++phase;
    __syncthreads();
  };

  // problem scheduling: clusters take p = cid, cid + ncl, ...; single CTAs
  // pull problems from a global ticket counter (problems differ a lot in
  // outer-iteration count, so static assignment leaves SMs idle)
  __shared__ int s_ticket;
  auto next_problem = [&](int p) {
    if (cs > 1 || !ticket) return p < 0 ? cid : p + ncl;
    __syncthreads();   // everyone has read the previous ticket
    if (tid == 0) s_ticket = atomicAdd(ticket, 1);
    __syncthreads();
    return s_ticket;
  };
  for (int p = next_problem(-1); p < nprob; p = next_problem(p)) {
    const int64_t o0 = offsets[p], m = offsets[p + 1] - offsets[p];
    // with the colour table: entries [o0, o0 + ucount[p]) of (rgb, pixel count)
    const int64_t me = ukey ? (int64_t)ucount[p] : m;
    const int64_t lo = o0 + (me * rank) / cs, hi = o0 + (me * (rank + 1)) / cs;
    if (!od)
      for (int i = tid; i < 3 * 256; i += NT) sh.lut[i] = luts[(int64_t)p * 768 + i];
    if (tid < 6) sh.w[tid] = a.w_init[tid];
    __syncthreads();
    const double lam = a.lam, code_lam = a.lam / 2.0;
    // OD of entry i and its weight (pixels of that colour; 1 without the table)
    auto load_od = [&](int64_t i, double& v0, double& v1, double& v2) -> double {
      if (od) {
        v0 = od[i]; v1 = od[total + i]; v2 = od[2 * total + i];
        return 1.0;
      }
      if (ukey) {
        const uint32_t rgb = ukey[i];
        v0 = sh.lut[rgb & 255u]; v1 = sh.lut[256 + ((rgb >> 8) & 255u)];
        v2 = sh.lut[512 + (rgb >> 16)];
        return (double)ucnt[i];
      }
      const uint8_t* px = samples + 3 * i;
      v0 = sh.lut[px[0]]; v1 = sh.lut[256 + px[1]]; v2 = sh.lut[512 + px[2]];
      return 1.0;
    };
    double* hist = hist_out + (int64_t)p * (a.max_outer + 1);

    // --- H-step + objective + sufficient statistics (one fused pass)
    auto hstep = [&]() {
      if (tid == 0) {
        const double* w = sh.w;
        const double g00 = fma_dot3(w[0], w[2], w[4], w[0], w[2], w[4]);
        const double g11 = fma_dot3(w[1], w[3], w[5], w[1], w[3], w[5]);
        const double g01 = fma_dot3(w[0], w[2], w[4], w[1], w[3], w[5]);
        sh.g[0] = g00; sh.g[1] = g01; sh.g[2] = g11;
        sh.g[3] = __dsub_rn(__dmul_rn(g00, g11), __dmul_rn(g01, g01));
      }
      __syncthreads();
      const double w00 = sh.w[0], w01 = sh.w[1], w10 = sh.w[2], w11 = sh.w[3], w20 = sh.w[4],
                   w21 = sh.w[5];
      const NnlsGram G = make_nnls_gram(sh.g[0], sh.g[1], sh.g[2], sh.g[3]);
      double st[kNStat];
#pragma unroll
      for (int q = 0; q < kNStat; ++q) st[q] = 0.0;
      // weighted sums over colours; with weight 1 every update is the same
      // single-rounding fma as the unweighted per-pixel sum
      auto accumulate = [&](double wt, double v0, double v1, double v2, double h0, double h1) {
        const double r0 = v0 - __fma_rn(w01, h1, __dmul_rn(w00, h0));
        const double r1 = v1 - __fma_rn(w11, h1, __dmul_rn(w10, h0));
        const double r2 = v2 - __fma_rn(w21, h1, __dmul_rn(w20, h0));
        st[0] = __fma_rn(wt, __fma_rn(r2, r2, __fma_rn(r1, r1, __dmul_rn(r0, r0))), st[0]);
        st[1] = __fma_rn(wt, h0, st[1]);
        st[2] = __fma_rn(wt, h1, st[2]);
        const double wh0 = __dmul_rn(wt, h0), wh1 = __dmul_rn(wt, h1);
        st[3] = __fma_rn(v0, wh0, st[3]); st[4] = __fma_rn(v0, wh1, st[4]);
        st[5] = __fma_rn(v1, wh0, st[5]); st[6] = __fma_rn(v1, wh1, st[6]);
        st[7] = __fma_rn(v2, wh0, st[7]); st[8] = __fma_rn(v2, wh1, st[8]);
        st[9] = __fma_rn(h0, wh0, st[9]); st[10] = __fma_rn(h0, wh1, st[10]);
        st[11] = __fma_rn(h1, wh1, st[11]);
      };
      // two independent pixels per thread per step: their division chains
      // interleave (the fp64 pipe is latency-bound with one)
      for (int64_t i = lo + tid; i < hi; i += 2 * NT) {
        const bool two = i + NT < hi;
        const int64_t i2 = two ? i + NT : i;
        double a0, a1, a2, c0, c1, c2;
        const double wa = load_od(i, a0, a1, a2);
        const double wc = load_od(i2, c0, c1, c2);
        NnlsState sa = nnls_seed(strict_dot3(w00, w10, w20, a0, a1, a2),
                                 strict_dot3(w01, w11, w21, a0, a1, a2), G, code_lam, 1e-9);
        NnlsState sc = nnls_seed(strict_dot3(w00, w10, w20, c0, c1, c2),
                                 strict_dot3(w01, w11, w21, c0, c1, c2), G, code_lam, 1e-9);
        nnls_finish(sa, G, 500, 1e-9);
        nnls_finish(sc, G, 500, 1e-9);
        accumulate(wa, a0, a1, a2, sa.x0, sa.x1);
        if (two) accumulate(wc, c0, c1, c2, sc.x0, sc.x1);
      }
      cta_reduce<NT, kNStat>(st, &sh.warp_part[0][0], sh.part[phase & 1]);
      cluster_total(kNStat);
      return sh.tot[0] + lam * (sh.tot[1] + sh.tot[2]);
    };

    double f = hstep();
    double row0 = sh.tot[1], row1 = sh.tot[2];
    double vht[3][2], hht[2][2];
    auto grab_stats = [&]() {
      for (int c = 0; c < 3; ++c) {
        vht[c][0] = sh.tot[3 + 2 * c];
        vht[c][1] = sh.tot[4 + 2 * c];
      }
      hht[0][0] = sh.tot[9]; hht[0][1] = hht[1][0] = sh.tot[10]; hht[1][1] = sh.tot[11];
    };
    grab_stats();
    if (rank == 0 && tid == 0) hist[0] = f;
    int it = 0, converged = 0;
    double f_rec = f;
    const double floor_f = 1e-12 * (double)m;
    for (it = 1; it <= a.max_outer; ++it) {
      // _w_step (src/stain_sep.py:210-236).  The candidate's objective with H
      // fixed follows from the sufficient statistics of the H-step pass:
      // replacing column j by c = w_j + d changes ||V - WH||^2 by
      // -2 d.(VH^T_j - W HH^T_j) + |d|^2 HH^T_jj (lam*sum(H) is unchanged),
      // so no pass over the samples is needed.  f is the explicit objective of
      // the current (W, H); each accepted candidate's value carries over to the
      // next column's test, as in the reference.
      if (tid == 0) {
        double* w = sh.w;
        for (int j = 0; j < 2; ++j) {
          const int k = 1 - j;
          if (hht[j][j] <= 0.0) continue;
          double u[3];
          for (int c = 0; c < 3; ++c) {
            u[c] = __dsub_rn(vht[c][j], __dmul_rn(w[c * 2 + k], hht[k][j]));
            u[c] = u[c] < 0.0 ? 0.0 : u[c];   // np.maximum(u, 0.0)
          }
          const double nrm = sqrt(fma_dot3(u[0], u[1], u[2], u[0], u[1], u[2]));
          if (nrm <= 1e-15) continue;
          double cand[3], dg = 0.0, dd = 0.0;
          for (int c = 0; c < 3; ++c) {
            cand[c] = __ddiv_rn(u[c], nrm);
            const double d = cand[c] - w[c * 2 + j];
            const double g = vht[c][j] - (w[c * 2] * hht[0][j] + w[c * 2 + 1] * hht[1][j]);
            dg += d * g;
            dd += d * d;
          }
          const double ft = f + (dd * hht[j][j] - 2.0 * dg);
          if (ft <= f) {
            for (int c = 0; c < 3; ++c) w[c * 2 + j] = cand[c];
            f = ft;
          }
        }
      }
      __syncthreads();
      f = hstep();
      row0 = sh.tot[1];
      row1 = sh.tot[2];
      grab_stats();
      if (rank == 0 && tid == 0) hist[it] = f;
      const double last = f_rec;   // history[-2]
      f_rec = f;
      if (fabs(last - f) <= a.rel_tol * fmax(fabs(last), 1e-12)) { converged = 1; break; }
      if (f <= floor_f) { converged = 1; break; }
    }
    if (it > a.max_outer) it = a.max_outer;
    // flags and ordering (src/stain_sep.py:315-336)
    if (rank == 0 && tid == 0) {
      int flags = 0;
      if (!converged) flags |= 1;
      const double tot = row0 + row1;
      if (tot > 0 && fmin(row0, row1) <= 1e-9 * tot) flags |= 2;
      const double* w = sh.w;
      const double rb0 = w[0] - w[4], rb1 = w[1] - w[5];
      double* bo = basis_out + (int64_t)p * 6;
      if (rb1 > rb0) {
        for (int c = 0; c < 3; ++c) { bo[2 * c] = w[2 * c + 1]; bo[2 * c + 1] = w[2 * c]; }
      } else {
        for (int c = 0; c < 6; ++c) bo[c] = w[c];
      }
      int32_t* inf = info_out + (int64_t)p * 4;
      inf[0] = it;
      inf[1] = converged;
      inf[2] = flags;
      inf[3] = it + 1;  // history length
    }
    cluster.sync();   // before the next problem reuses shared state
  }
}

// Batched code_densities over the fit samples: problem p's pixels
// [off[p], off[p+1]) through its own OD table and basis.
__global__ void __launch_bounds__(256) k_code_samples(
    const uint8_t* __restrict__ samples, const int64_t* __restrict__ offsets, int nprob,
    const double* __restrict__ luts, const double* __restrict__ bases, double lam, int max_sweeps,
    double* __restrict__ h, int64_t total) {
  const int p = blockIdx.y;
  const int64_t o0 = offsets[p], o1 = offsets[p + 1];
  __shared__ double lut[768];
  __shared__ double w[6], g[4];
  for (int i = threadIdx.x; i < 768; i += 256) lut[i] = luts[(int64_t)p * 768 + i];
  if (threadIdx.x < 6) w[threadIdx.x] = bases[(int64_t)p * 6 + threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    // code_densities' scalar Gram order (src/stain_sep.py:197-199): plain mul/add
    g[0] = __dadd_rn(__dadd_rn(__dmul_rn(w[0], w[0]), __dmul_rn(w[2], w[2])), __dmul_rn(w[4], w[4]));
    g[2] = __dadd_rn(__dadd_rn(__dmul_rn(w[1], w[1]), __dmul_rn(w[3], w[3])), __dmul_rn(w[5], w[5]));
    g[1] = __dadd_rn(__dadd_rn(__dmul_rn(w[0], w[1]), __dmul_rn(w[2], w[3])), __dmul_rn(w[4], w[5]));
    g[3] = __dsub_rn(__dmul_rn(g[0], g[2]), __dmul_rn(g[1], g[1]));
  }
  __syncthreads();
  const NnlsGram G = make_nnls_gram(g[0], g[1], g[2], g[3]);
  for (int64_t i = o0 + blockIdx.x * 256ll + threadIdx.x; i < o1; i += 256ll * gridDim.x) {
    const uint8_t* px = samples + 3 * i;
    const double v0 = lut[px[0]], v1 = lut[256 + px[1]], v2 = lut[512 + px[2]];
    const double b0 = strict_dot3(w[0], w[2], w[4], v0, v1, v2);
    const double b1 = strict_dot3(w[1], w[3], w[5], v0, v1, v2);
    double h0, h1;
    strict_nnls(b0, b1, G, lam, max_sweeps, 0.0, h0, h1);
    h[i] = h0;
    h[total + i] = h1;
  }
}

// The same coding over the colour table of the samples (k_colour_table's
// entries: problem p's first ucount[p] entries at off[p] are (rgb, count)):
// one fp64 evaluation per distinct colour, written at the entry's position.
__global__ void __launch_bounds__(256) k_code_table(
    const uint32_t* __restrict__ ukey, const int32_t* __restrict__ ucount,
    const int64_t* __restrict__ offsets, int nprob, const double* __restrict__ luts,
    const double* __restrict__ bases, double lam, int max_sweeps, double* __restrict__ h,
    int64_t total) {
  const int p = blockIdx.y;
  const int64_t o0 = offsets[p], o1 = o0 + ucount[p];
  __shared__ double lut[768];
  __shared__ double w[6], g[4];
  for (int i = threadIdx.x; i < 768; i += 256) lut[i] = luts[(int64_t)p * 768 + i];
  if (threadIdx.x < 6) w[threadIdx.x] = bases[(int64_t)p * 6 + threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    g[0] = __dadd_rn(__dadd_rn(__dmul_rn(w[0], w[0]), __dmul_rn(w[2], w[2])), __dmul_rn(w[4], w[4]));
    g[2] = __dadd_rn(__dadd_rn(__dmul_rn(w[1], w[1]), __dmul_rn(w[3], w[3])), __dmul_rn(w[5], w[5]));
    g[1] = __dadd_rn(__dadd_rn(__dmul_rn(w[0], w[1]), __dmul_rn(w[2], w[3])), __dmul_rn(w[4], w[5]));
    g[3] = __dsub_rn(__dmul_rn(g[0], g[2]), __dmul_rn(g[1], g[1]));
  }
  __syncthreads();
  const NnlsGram G = make_nnls_gram(g[0], g[1], g[2], g[3]);
  for (int64_t i = o0 + blockIdx.x * 256ll + threadIdx.x; i < o1; i += 256ll * gridDim.x) {
    const uint32_t rgb = ukey[i];
    const double v0 = lut[rgb & 255u], v1 = lut[256 + ((rgb >> 8) & 255u)], v2 = lut[512 + (rgb >> 16)];
    const double b0 = strict_dot3(w[0], w[2], w[4], v0, v1, v2);
    const double b1 = strict_dot3(w[1], w[3], w[5], v0, v1, v2);
    double h0, h1;
    strict_nnls(b0, b1, G, lam, max_sweeps, 0.0, h0, h1);
    h[i] = h0;
    h[total + i] = h1;
  }
}

cudaError_t launch_code_table(const uint32_t* ukey, const int32_t* ucount, const int64_t* offsets,
                              int nprob, int64_t max_m, const double* luts, const double* bases,
                              double lam, int max_sweeps, double* h, int64_t total,
                              cudaStream_t st) {
  if (nprob <= 0) return cudaSuccess;
  // CTAs per problem: each loads the problem's 6 KB OD table first, so few
  // CTAs with more colours each (C2, ~10 k colours per problem: 16 -> 0.73
  // ms, 4 -> 0.54, 2 -> 0.52); SPCN_CODE_TABLE_GX overrides (A/B)
  static const int gx_cap = [] {
    const char* e = std::getenv("SPCN_CODE_TABLE_GX");
    return e && std::atoi(e) > 0 ? std::atoi(e) : 2;
  }();
  int64_t gx = (max_m + 255) / 256;
  if (gx > gx_cap) gx = gx_cap;
  if (gx < 1) gx = 1;
  for (int p0 = 0; p0 < nprob; p0 += kMaxGridY) {   // gridDim.y <= 65535
    const int np = nprob - p0 < kMaxGridY ? nprob - p0 : kMaxGridY;
    k_code_table<<<dim3((unsigned)gx, np), 256, 0, st>>>(ukey, ucount + p0, offsets + p0, np,
                                                         luts + (int64_t)p0 * 768,
                                                         bases + (int64_t)p0 * 6, lam, max_sweeps,
                                                         h, total);
    const cudaError_t e = launched();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// k_colour_table: the fit samples are 8-bit RGB and repeat heavily (a 100 k
// sample of an H&E patch holds ~10 k distinct colours), while every SNMF
// quantity is a function of the colour.  One CTA per problem counts the
// distinct colours of the problem's samples in a shared-memory hash table and
// writes them as (rgb, pixel count) entries at the problem's sample offset;
// the SNMF passes then iterate over ~10x fewer entries with weights.  If the
// table fills up, the problem's samples are listed one by one with count 1.

constexpr int kCT = 1024;   // threads of k_colour_table

__global__ void __launch_bounds__(kCT) k_colour_table(const uint8_t* __restrict__ samples,
                                                      const int64_t* __restrict__ offsets,
                                                      int nprob, uint32_t* __restrict__ ukey,
                                                      uint32_t* __restrict__ ucnt,
                                                      int32_t* __restrict__ ucount) {
  extern __shared__ __align__(16) uint32_t tab[];   // keys [kTabSlots], counts [kTabSlots]
  uint32_t* key = tab;
  uint32_t* cnt = tab + kTabSlots;
  __shared__ int s_full, s_used;   // table too full (or a probe failed) -> list the samples
  __shared__ uint32_t s_scan[kCT];
  const int tid = threadIdx.x;
  for (int p = blockIdx.x; p < nprob; p += gridDim.x) {
    const int64_t o0 = offsets[p], m = offsets[p + 1] - o0;
    for (int i = tid; i < kTabSlots; i += kCT) {
      key[i] = kTabEmpty;
      cnt[i] = 0;
    }
    if (tid == 0) s_full = s_used = 0;
    __syncthreads();
    // samples [a, a + 16 nb) in 16-sample groups at 16-byte-aligned addresses
    // (three vector loads each); the few before and after one by one
    const int64_t a0 = (16 - (o0 & 15)) & 15, a = m < a0 ? m : a0;
    const int64_t nb = (m - a) / 16, rest0 = a + 16 * nb;
    const int64_t rounds = (nb + kCT - 1) / kCT;
    for (int64_t r = 0; r < rounds; ++r) {
      const int64_t g = r * kCT + tid;
      uint32_t rgb[16];
      if (g < nb) {
        const uint4* v = reinterpret_cast<const uint4*>(samples + 3 * (o0 + a + 16 * g));
        const uint4 q0 = __ldg(v), q1 = __ldg(v + 1), q2 = __ldg(v + 2);
        const uint32_t w[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int i = 3 * j;
          const uint64_t pr = ((uint64_t)w[(i >> 2) + ((i >> 2) < 11 ? 1 : 0)] << 32) | w[i >> 2];
          rgb[j] = (uint32_t)(pr >> (8 * (i & 3))) & 0xffffffu;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) rgb[j] = kNoColour;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) ct_insert(key, cnt, &s_full, rgb[j]);
    }
    // head [0, a) and tail [rest0, m): < 32 samples, one warp
    if (tid < 32) {
      const int64_t i = tid < a ? tid : rest0 + (tid - a);
      uint32_t rgb = kNoColour;
      if ((tid < a) || (tid >= a && i < m)) {
        const uint8_t* px = samples + 3 * (o0 + i);
        rgb = px[0] | (px[1] << 8) | (px[2] << 16);
      }
      ct_insert(key, cnt, &s_full, rgb);
    }
    __syncthreads();
    ct_overfull<kCT>(key, &s_used, &s_full);
    if (!s_full) {
      ct_finish_par<kCT>(key, cnt, s_scan, reinterpret_cast<uint16_t*>(tab + 2 * kTabSlots),
                         ukey, ucnt, o0, &ucount[p]);
    } else {
      for (int64_t i = tid; i < m; i += kCT) {
        const uint8_t* px = samples + 3 * (o0 + i);
        ukey[o0 + i] = px[0] | (px[1] << 8) | (px[2] << 16);
        ucnt[o0 + i] = 1u;
      }
      if (tid == 0) ucount[p] = (int32_t)m;
      __syncthreads();
    }
  }
}

cudaError_t launch_snmf(const uint8_t* samples, const double* od, const int64_t* offsets, int nprob,
                        const double* luts, const SnmfArgs& a, double* hbuf, int64_t total,
                        double* basis_out, double* hist_out, int32_t* info_out, int cluster,
                        cudaStream_t st) {
  if (nprob <= 0) return cudaSuccess;
  static int sms = 0, occ1 = 0;
  if (!sms) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, k_snmf<512, 1>, 512, 0);
    // clusters of up to 16 CTAs (non-portable size) for one slide's fit
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_snmf<512, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) {
      sms = 0;
      return e;
    }
    if (occ1 < 1) occ1 = 1;
  }
  const bool single = cluster == 1;
  // colour table in the caller's scratch: keys | counts (total each) | per-problem sizes
  uint32_t* ukey = nullptr;
  uint32_t* ucnt = nullptr;
  int32_t* ucount = nullptr;
  // (batches only: a single slide's fit runs on a cluster of CTAs, while the
  // table of one problem is built by one CTA and would cost more than it saves)
  if (hbuf && !od && samples && single) {
    static bool attr = false;
    constexpr int kTabSmem = 2 * kTabSlots * sizeof(uint32_t) + kTabSlots * sizeof(uint16_t);
    if (!attr) {
      const cudaError_t e0 = cudaFuncSetAttribute(k_colour_table,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  kTabSmem);
      if (e0 != cudaSuccess) return e0;
      attr = true;
    }
    ukey = reinterpret_cast<uint32_t*>(hbuf);
    ucnt = ukey + total;
    ucount = reinterpret_cast<int32_t*>(ucnt + total);
    int g = nprob < 4 * sms ? nprob : 4 * sms;
    k_colour_table<<<g, kCT, kTabSmem, st>>>(samples, offsets, nprob, ukey, ucnt, ucount);
    const cudaError_t e1 = launched();
    if (e1 != cudaSuccess) return e1;
  }
  // work ticket of the dynamic problem queue: in the caller's scratch right
  // after the table (no stream-ordered allocation per call: a pool that
  // returns memory to the driver makes every call re-map it)
  int* ticket = nullptr;
  bool own_ticket = false;
  if (single && nprob > 1) {
    cudaError_t e = cudaSuccess;
    if (hbuf) {
      ticket = reinterpret_cast<int*>(reinterpret_cast<uint32_t*>(hbuf) + 2 * total + nprob);
    } else {
      e = cudaMallocAsync(reinterpret_cast<void**>(&ticket), sizeof(int), st);
      own_ticket = true;
    }
    if (e == cudaSuccess) e = cudaMemsetAsync(ticket, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
  }
  // one-CTA-per-problem batches: 128 threads x 4 CTAs per SM (each problem's
  // serial W-step and barriers overlap other CTAs' H-step passes: 9.3 ms vs
  // 11.5 ms for 512 x 1 on the 4096-patch batch).  SPCN_SNMF_BATCH = "512x1" |
  // "256x2" | "128x4" | "64x8" | "32x16" selects another shape (experiments).
  static int bshape = -1, occ_b = 1;
  if (bshape < 0) {
    bshape = 2;
    if (const char* env = getenv("SPCN_SNMF_BATCH")) {
      if (!strcmp(env, "512x1")) bshape = 0;
      if (!strcmp(env, "256x2")) bshape = 1;
      if (!strcmp(env, "128x4")) bshape = 2;
      if (!strcmp(env, "64x8")) bshape = 3;
      if (!strcmp(env, "32x16")) bshape = 4;
    }
    const void* fns[5] = {nullptr, (const void*)k_snmf<256, 2>, (const void*)k_snmf<128, 4>,
                          (const void*)k_snmf<64, 8>, (const void*)k_snmf<32, 16>};
    const void* fn = fns[bshape];
    const int nt = 512 >> bshape;
    if (bshape) {
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_b, fn, nt, 0);
      if (e != cudaSuccess) return e;
      if (occ_b < 1) occ_b = 1;
    }
  }
  // (fewer problems than 4 per SM: 512 threads each finish sooner)
  const bool alt = single && bshape != 0 && nprob >= 4 * sms;
  int nclusters = nprob;
  const int max_clusters = alt ? sms * occ_b : single ? sms * occ1 : (sms * 2) / cluster;
  if (nclusters > max_clusters) nclusters = max_clusters;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclusters * cluster);
  cfg.blockDim = dim3(alt ? (512 >> bshape) : 512);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const uint32_t* ck = ukey;
  const uint32_t* cc = ucnt;
  const int32_t* cu = ucount;
  cudaError_t e =
      !alt ? cudaLaunchKernelEx(&cfg, k_snmf<512, 1>, samples, od, offsets, nprob, luts, a, ticket,
                                total, basis_out, hist_out, info_out, ck, cc, cu)
      : bshape == 1
          ? cudaLaunchKernelEx(&cfg, k_snmf<256, 2>, samples, od, offsets, nprob, luts, a, ticket,
                               total, basis_out, hist_out, info_out, ck, cc, cu)
      : bshape == 2
          ? cudaLaunchKernelEx(&cfg, k_snmf<128, 4>, samples, od, offsets, nprob, luts, a, ticket,
                               total, basis_out, hist_out, info_out, ck, cc, cu)
      : bshape == 3
          ? cudaLaunchKernelEx(&cfg, k_snmf<64, 8>, samples, od, offsets, nprob, luts, a, ticket,
                               total, basis_out, hist_out, info_out, ck, cc, cu)
          : cudaLaunchKernelEx(&cfg, k_snmf<32, 16>, samples, od, offsets, nprob, luts, a, ticket,
                               total, basis_out, hist_out, info_out, ck, cc, cu);
  if (own_ticket) {
    const cudaError_t e2 = cudaFreeAsync(ticket, st);
    if (e == cudaSuccess) e = e2;
  }
  return e != cudaSuccess ? e : launched();
}

cudaError_t launch_code_samples(const uint8_t* samples, const int64_t* offsets, int nprob,
                                int64_t max_m, const double* luts, const double* bases,
                                double lam, int max_sweeps, double* h, int64_t total,
                                cudaStream_t st) {
  if (nprob <= 0 || max_m <= 0) return cudaSuccess;
  int64_t gx = (max_m + 255) / 256;
  if (gx > 64) gx = 64;
  for (int p0 = 0; p0 < nprob; p0 += kMaxGridY) {   // gridDim.y <= 65535
    const int np = nprob - p0 < kMaxGridY ? nprob - p0 : kMaxGridY;
    k_code_samples<<<dim3((unsigned)gx, np), 256, 0, st>>>(samples, offsets + p0, np,
                                                           luts + (int64_t)p0 * 768,
                                                           bases + (int64_t)p0 * 6, lam,
                                                           max_sweeps, h, total);
    const cudaError_t e = launched();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace spcn
