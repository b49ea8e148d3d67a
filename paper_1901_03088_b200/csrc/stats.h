// stats.h — whole-slide percentile passes (internal launch interface).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "spcn_device.cuh"

namespace spcn {
struct StatsArgs {
  FastS fs;                 // density coefficients of the source basis
  float lut[3][256];        // fp32 OD table
  float coef[2];            // density error bound per unit T (params.cuh density_error_coeffs)
  uint32_t white;           // white threshold: non-white = not all channels > white
  uint32_t white_by_od;     // 1: channel > white  <=>  lut[c][x] < lut[c][white] (see stats.cu)
  float nwod[3];            // -lut[c][white]
  uint32_t base[2];         // histogram window start (fp32 key) per stain
  uint32_t shift[2];        // bin = (key - base) >> shift
  int32_t nbins;            // <= 8192
  double a[2], b[2];        // refine window [a, b) per stain
  float lf[4][4];           // table pass: linear upper-bound forms k.v + b (see stats.cu)
};
cudaError_t launch_stats_hist(const uint8_t* src, int64_t npix, const StatsArgs& a,
                              unsigned long long* hist, unsigned long long* counts,
                              cudaStream_t st);
cudaError_t launch_stats_refine(const uint8_t* src, int64_t npix, const StatsArgs& a,
                                const StrictP& sp, unsigned long long* counts, double* cand,
                                unsigned long long* wcnt, unsigned long long cap,
                                cudaStream_t st);
cudaError_t launch_stats_table(const uint8_t* src, int64_t npix, const StatsArgs& a,
                               unsigned long long* table, unsigned long long* counts,
                               cudaStream_t st);
cudaError_t launch_cube_class(const StatsArgs& a, uint8_t* cls, cudaStream_t st);
cudaError_t launch_stats_cube(const uint8_t* src, int64_t npix, const StatsArgs& a,
                              const uint8_t* cls, unsigned long long* table,
                              unsigned long long* counts, cudaStream_t st);
cudaError_t launch_entries_hist(const double* x, const unsigned long long* w, int64_t m,
                                const double* lo, const double* scale, int nbins,
                                unsigned long long* hist, cudaStream_t st);
cudaError_t launch_entries_collect(const double* x, const unsigned long long* w, int64_t m,
                                   const double* lo, const double* scale, int nbins,
                                   const int32_t* bins, double* vals, unsigned long long* wts,
                                   unsigned long long cap, unsigned long long* nsel,
                                   cudaStream_t st);
cudaError_t launch_table_scan(const unsigned long long* table, const StrictP& sp, double* x,
                              unsigned long long* w, unsigned long long cap,
                              unsigned long long* n_out, cudaStream_t st);
}  // namespace spcn
