// Small analytic models: jacobi / "price = strike" 5->1, identity 5->5, C4 conv1 as a patch MLP 64->8
#include "exact_region.cuh"

namespace smlrt {

int exact_try_small(const smlrt_model_s& m, const DevPlan& in, const Ptrs& src, const DevPlan& out, const Ptrs& dst,
                    bool all_f32, int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status, bool probe_only,
                    bool* done) {
  int rc = SMLRT_OK;
  if ((rc = try_fused<5, 1>(m, in, src, out, dst, all_f32, r0, r1, staged, s, status, probe_only, done)) !=
      SMLRT_OK || *done)  // jacobi_model / price = strike
    return rc;
  if ((rc = try_fused<5, 5>(m, in, src, out, dst, all_f32, r0, r1, staged, s, status, probe_only, done)) !=
      SMLRT_OK || *done)  // model_identity5 fixture
    return rc;
  if ((rc = try_fused<64, 8>(m, in, src, out, dst, all_f32, r0, r1, staged, s, status, probe_only, done)) !=
      SMLRT_OK || *done)  // C4 conv1 as a patch MLP
    return rc;
  return SMLRT_OK;
}

}  // namespace smlrt
