// snmf.h — launch interface of the batched SNMF / sample-coding kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spcn {
struct SnmfArgs {
  double lam;
  double rel_tol;
  double w_init[6];   // row-major 3x2 initial basis (host: reference init, src/stain_sep.py:271-274)
  int32_t max_outer;
  int32_t pad_;
};
cudaError_t launch_snmf(const uint8_t* samples, const double* od, const int64_t* offsets, int nprob,
                        const double* luts, const SnmfArgs& a, double* hbuf, int64_t total,
                        double* basis_out, double* hist_out, int32_t* info_out, int cluster,
                        cudaStream_t st);
cudaError_t launch_code_samples(const uint8_t* samples, const int64_t* offsets, int nprob,
                                int64_t max_m, const double* luts, const double* bases,
                                double lam, int max_sweeps, double* h, int64_t total,
                                cudaStream_t st);
cudaError_t launch_code_table(const uint32_t* ukey, const int32_t* ucount, const int64_t* offsets,
                              int nprob, int64_t max_m, const double* luts, const double* bases,
                              double lam, int max_sweeps, double* h, int64_t total,
                              cudaStream_t st);
}  // namespace spcn
