// select.h — launch interface of the order-statistic kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spcn {
struct SelQuery {
  int64_t offset;      // element offset of the value array the query reads
  int64_t begin, end;  // segment [begin, end) relative to offset
  int64_t k;           // zero-based rank
};
cudaError_t launch_select(const double* values, const SelQuery* qs, int nq, double* out,
                          cudaStream_t st);
cudaError_t launch_p99(const double* h, int64_t total, const int64_t* seg, int nseg, double p,
                       SelQuery* qbuf, double* selbuf, double* p99, int32_t* absent,
                       cudaStream_t st);
cudaError_t launch_p99_weighted(const double* h, int64_t total, const uint32_t* w,
                                const int32_t* ucount, const int64_t* seg, int nseg, double p,
                                double* p99, int32_t* absent, cudaStream_t st);
}  // namespace spcn
namespace spcn {
cudaError_t launch_build_queries(const int64_t* b, const int64_t* e, const int64_t* k, int nq,
                                 SelQuery* qs, cudaStream_t st);
}
