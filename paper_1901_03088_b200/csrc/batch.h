// batch.h — batched recolouring (internal launch interface).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "spcn.h"
#include "spcn_device.cuh"

namespace spcn {
constexpr int kMaxBatch = 148;   // items per launch (kernel-parameter block ~20 KB)

struct BatchTarget {
  double i0[3];
  double basis[6];
  double p99[2];
};

struct BatchArgs {
  int32_t n, item0;                 // items in this launch, index of the first item
  int64_t off[kMaxBatch + 1];       // absolute pixel offsets of items item0.. (into src/dst)
  int8_t strict[kMaxBatch];         // 1 = fast path not applicable (strict kernel)
  FastS s[kMaxBatch];
};

cudaError_t launch_build_params(int nitems, const double* i0, const double* luts,
                                const double* bases, const double* p99, const BatchTarget& tgt,
                                double code_lam, int max_sweeps, int exact, FastS* fs, float* flut,
                                StrictP* sps, int32_t* status, cudaStream_t st);
cudaError_t launch_xform_batch(int mode, const uint8_t* src, uint8_t* dst, const float* flut,
                               const StrictP* sps, const BatchArgs& args,
                               unsigned long long* rcount, unsigned long long* ritems,
                               unsigned long long rcap, cudaStream_t st);
cudaError_t launch_repair_batch(uint8_t* dst, const StrictP* sps, const int64_t* off, int nitems,
                                unsigned long long* rcount, unsigned long long* ritems,
                                unsigned long long rcap, cudaStream_t st);
cudaError_t launch_strict_batch(const uint8_t* src, uint8_t* dst, const StrictP* sps,
                                const int64_t* off, const int32_t* status, int nitems,
                                int64_t max_pix, cudaStream_t st);
}  // namespace spcn
