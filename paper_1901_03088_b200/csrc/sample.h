// sample.h — launch interface of the sampling / i0 kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "spcn.h"

namespace spcn {
cudaError_t launch_visit_single(const int32_t* counts, int n, int chunks, double used_min,
                                int64_t target, int64_t cap, spcn_patch_take* takes,
                                int64_t* take_nw, cudaStream_t st);
cudaError_t launch_sample_count(const uint8_t* img, const spcn_patch* patches, int npatches,
                                int max_chunks, int thr, int32_t* counts, cudaStream_t st);
cudaError_t launch_sample_compact(const uint8_t* img, const spcn_patch* patches, int npatches,
                                  int max_chunks, int thr, const int32_t* counts,
                                  const spcn_patch_take* takes, uint8_t* out_px,
                                  int32_t* bright_hist, cudaStream_t st);
cudaError_t launch_i0_from_hist(const int32_t* hist, int nprob, double* i0, int32_t* empty,
                                cudaStream_t st);
cudaError_t launch_od_tables(const double* i0, int nprob, double* lut, cudaStream_t st);
cudaError_t launch_visit(const int32_t* counts, int n, int max_chunks, int k0, const int32_t* dims,
                         const spcn_visit_plan& plan, int64_t* state, spcn_patch_take* takes,
                         int64_t* offsets, cudaStream_t st);
}  // namespace spcn
