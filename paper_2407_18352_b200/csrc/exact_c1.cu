// C1 Binomial Options surrogate 5-64-32-1 (exact fp32 fused region)
#include "exact_region.cuh"

namespace smlrt {

int exact_try_c1(const smlrt_model_s& m, const DevPlan& in, const Ptrs& src, const DevPlan& out, const Ptrs& dst,
                 bool all_f32, int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status, bool probe_only,
                 bool* done) {
  int rc = SMLRT_OK;
  if ((rc = try_fused<5, 64, 32, 1>(m, in, src, out, dst, all_f32, r0, r1, staged, s, status, probe_only, done)) !=
      SMLRT_OK || *done)  // C1
    return rc;
  return SMLRT_OK;
}

}  // namespace smlrt
