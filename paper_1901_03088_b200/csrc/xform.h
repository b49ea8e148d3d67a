// xform.h — host-side launch interface of the recolor kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
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
cudaError_t launch_calibrate(const FastP& fp, const StrictP& sp, unsigned int* max_bits,
                             cudaStream_t st, uint32_t q0 = 0, uint32_t q1 = 1u << 23);
int xform_tile_pixels();
const char* xform_shape_name();
}  // namespace spcn
