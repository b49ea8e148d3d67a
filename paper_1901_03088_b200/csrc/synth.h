// synth.h — launch interface of the synthetic slide generator (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "spcn.h"

namespace spcn {
cudaError_t launch_render(uint8_t* out, int64_t width, int64_t row0, int64_t rows, int64_t height,
                          uint64_t seed, const spcn_synth_params& p, cudaStream_t st);
}
