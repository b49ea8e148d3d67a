// batch.h — batched recolouring (internal launch interface).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "spcn.h"
#include "spcn_device.cuh"

namespace spcn {
struct BatchTarget {
  double i0[3];
  double basis[6];
  double p99[2];
};

cudaError_t launch_build_params(int nitems, const double* i0, const double* luts,
                                const double* bases, const double* p99, const BatchTarget& tgt,
                                double code_lam, int max_sweeps, int exact, FastS* fs, float* flut,
                                StrictP* sps, int32_t* status, cudaStream_t st);
// EXACT batches: one repair list per CTA of k_xform_batch (counts[cta],
// items[cta * cap_cta ...]) and per item its segment (seg[3i] = start,
// seg[3i+1] = end, seg[3i+2] = the CTA) — see k_repair_items.
struct BatchRepair {
  unsigned long long* counts;
  unsigned long long* items;
  unsigned long long cap_cta;
  unsigned long long* seg;
};

int batch_grid(int nitems);
cudaError_t launch_xform_batch(int mode, const uint8_t* src, uint8_t* dst, int nitems,
                               const int64_t* off, const int32_t* status, const FastS* fs,
                               const float* flut, const BatchRepair& br, cudaStream_t st);
cudaError_t launch_repair_items(const uint8_t* src, uint8_t* dst, const StrictP* sps,
                                const int64_t* off, const int32_t* status, int nitems,
                                const BatchRepair& br, cudaStream_t st);
cudaError_t launch_strict_batch(const uint8_t* src, uint8_t* dst, const StrictP* sps,
                                const int64_t* off, const int32_t* status, int nitems,
                                int64_t max_pix, cudaStream_t st);
}  // namespace spcn
