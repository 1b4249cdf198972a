// tcgen05/TMEM bf16 fused region kernel (placeholder until the kernel lands).
#include "common.cuh"

namespace smlrt {

int tc_pack_model(smlrt_model_s& m) {
  (void)m;
  return SMLRT_OK;
}

int launch_region_tc(const smlrt_model_s&, const DevPlan&, const void* const*, const int32_t*, int,
                     const DevPlan&, void* const*, const int32_t*, int, int64_t, int64_t, float*,
                     cudaStream_t, uint32_t*, bool) {
  return SMLRT_E_UNSUPPORTED;
}

}  // namespace smlrt
