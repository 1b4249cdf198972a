// C5 MiniWeather 3x3x4 halo surrogate 36-8-4 (exact fp32 fused region)
// 5 resident CTAs per SM (96 registers, a few bytes of spill): the 36 gathered
// inputs per thread are loads in flight, and 20 warps per SM hide the gather
// latency better than 16 warps without spills (0.260 -> 0.237 ms)
#ifndef SMLRT_EXACT_MINB
#define SMLRT_EXACT_MINB 5
#endif
#include "exact_region.cuh"

namespace smlrt {

int exact_try_c5(const smlrt_model_s& m, const DevPlan& in, const Ptrs& src, const DevPlan& out, const Ptrs& dst,
                 bool all_f32, int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status, bool probe_only,
                 bool* done) {
  int rc = SMLRT_OK;
  if ((rc = try_fused<36, 8, 4>(m, in, src, out, dst, all_f32, r0, r1, staged, s, status, probe_only, done)) !=
      SMLRT_OK || *done)  // C5
    return rc;
  return SMLRT_OK;
}

}  // namespace smlrt
