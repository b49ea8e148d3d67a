// launch_count.h — process-wide count of libspcn kernel launches (diagnostics:
// bench.py reports how many of our kernels ran inside its timed region).
#pragma once
#include <atomic>
#include <cuda_runtime.h>

namespace spcn {
constexpr int kMaxGridY = 65535;   // launches with items on gridDim.y are split at this size
extern std::atomic<unsigned long long> g_launches;
inline cudaError_t launched(unsigned n = 1) {
  g_launches.fetch_add(n, std::memory_order_relaxed);
  return cudaGetLastError();
}
}  // namespace spcn
