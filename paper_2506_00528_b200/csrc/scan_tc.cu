// scan_tc.cu -- int8 tcgen05 Delta GEMM with fused top-k (placeholder: not yet built).
#include "common.cuh"
#include "internal.h"

namespace uq {

TcPlan plan_tc(int64_t, int64_t, int32_t, int32_t, int) {
  TcPlan p{};
  p.ok = false;
  return p;
}

cudaError_t launch_scan_tc(const uint8_t*, int64_t, const uint8_t*, int64_t, int32_t, int32_t,
                           const TcPlan&, uint32_t*, uint64_t*, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace uq
