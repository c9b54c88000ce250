// pearson_gemm.cu -- placeholder until the tcgen05 block GEMM lands.
#include "corr_internal.cuh"
namespace corr {
cudaError_t launch_pearson_block(const corr_field*, const corr_field*, const RegionDev*, const RegionDev*, int64_t,
                                 int, unsigned long long*, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace corr
