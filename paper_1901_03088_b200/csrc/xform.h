// xform.h — host-side launch interface of the recolor kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "spcn.h"
#include "spcn_device.cuh"

namespace spcn {
cudaError_t xform_setup_device();
cudaError_t launch_xform_main(int mode, const uint8_t* src, uint8_t* dst, int64_t npix,
                              const FastP& fp, const StrictP& sp, unsigned long long* count,
                              unsigned long long* items, unsigned long long cap,
                              const unsigned int* alpha_bits, cudaStream_t st);
cudaError_t launch_xform_repair(const uint8_t* src, uint8_t* dst, int64_t npix, const StrictP& sp,
                                unsigned long long* count, unsigned long long* items,
                                unsigned long long cap, cudaStream_t st);
cudaError_t launch_xform_strict(const uint8_t* src, uint8_t* dst, int64_t npix,
                                const StrictP& sp, cudaStream_t st);
cudaError_t launch_code_densities(const double* od, double* h, int64_t n, const StrictP& sp,
                                  cudaStream_t st);
cudaError_t launch_normalize_block(const double* h, uint8_t* out, int64_t n, const StrictP& sp,
                                   cudaStream_t st);
cudaError_t launch_beer_lambert(const uint8_t* px, double* od, int64_t n, const StrictP& sp,
                                cudaStream_t st);
cudaError_t launch_inverse_bl(const double* od, uint8_t* out, int64_t n, const StrictP& sp,
                              cudaStream_t st);
// ---- device-built recolouring (xform.cu k_build_xform) -------------------
constexpr int kDpSlots = SPCN_FITTED_SLOTS;   // __constant__ parameter slots (ring; see api.cu)
// fp sits at 8 mod 16, as the kernel-parameter copy does (after src, dst,
// npix): the compiler then forms the same constant-operand / uniform-register
// mix for both (at 0 mod 16 it batches the fields into LDCU.128 loads, and the
// extra uniform registers push the shared-memory base out of the uniform file)
struct alignas(16) DevParams {
  int32_t status;   // 0 fast path; 1 strict only; < 0 invalid (-SPCN_E* code)
  int32_t pad_;
  FastP fp;
  StrictP sp;
};
struct XformBuildIn {   // the host-known half: target profile and options
  double tgt_basis[6];
  double tgt_p99[2];
  double tgt_i0[3];
  double code_lam;
  int32_t max_sweeps;
  int32_t pad_;
  const double* tgt_fit_dev;   // device (optional): the target's arena B, read instead of the above
  const double* tgt_i0_dev;    // device: the target's i0 (with tgt_fit_dev)
};
// build (1 CTA) -> copy into __constant__ slot `slot` -> optional status
// read-back into pinned host memory (then `built` is recorded) -> exhaustive
// calibration of colour pairs [q0, q1) into ws+8
cudaError_t launch_xform_build(int slot, const XformBuildIn& in, const double* lut,
                               const double* fit, DevParams* staging, void* ws,
                               int32_t* status_host, cudaEvent_t built, uint32_t q0, uint32_t q1,
                               cudaStream_t st);
cudaError_t launch_xform_main_c(int slot, bool analytic, const uint8_t* src, uint8_t* dst,
                                int64_t npix, unsigned long long* count,
                                unsigned long long* items, unsigned long long cap,
                                const unsigned int* alpha_bits, cudaStream_t st);
cudaError_t launch_xform_repair_c(int slot, const uint8_t* src, uint8_t* dst, int64_t npix,
                                  int64_t head, int64_t body, unsigned long long* count,
                                  unsigned long long* items, unsigned long long cap,
                                  cudaStream_t st);
cudaError_t launch_calibrate(const FastP& fp, const StrictP& sp, unsigned int* max_bits,
                             cudaStream_t st, uint32_t q0 = 0, uint32_t q1 = 1u << 23);
int xform_tile_pixels();
const char* xform_shape_name();
}  // namespace spcn
