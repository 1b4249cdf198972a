// Shared helpers of the SIMT kernels (kernels_simt.cu) and the exact fused
// region kernels (exact_region.cuh, instantiated per model shape in
// exact_*.cu so the heavily unrolled instantiations compile in parallel).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace smlrt {

// array pointers + dtypes of one plan's arrays (kernel parameter)
struct Ptrs {
  const void* p[8];
  int32_t dt[8];
};

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float load_as_f32(const void* base, int dtype, int64_t i) {
  return dtype == SMLRT_F32 ? __ldg(reinterpret_cast<const float*>(base) + i)
                            : __double2float_rn(__ldg(reinterpret_cast<const double*>(base) + i));
}

__device__ __forceinline__ double load_as_f64(const void* base, int dtype, int64_t i) {
  return dtype == SMLRT_F32 ? (double)__ldg(reinterpret_cast<const float*>(base) + i)
                            : __ldg(reinterpret_cast<const double*>(base) + i);
}

__device__ __forceinline__ void store_f32(void* base, int dtype, int64_t i, float v) {
  if (dtype == SMLRT_F32)
    reinterpret_cast<float*>(base)[i] = v;
  else
    reinterpret_cast<double*>(base)[i] = (double)v;
}

__device__ __forceinline__ void store_f64(void* base, int dtype, int64_t i, double v) {
  if (dtype == SMLRT_F32)
    reinterpret_cast<float*>(base)[i] = __double2float_rn(v);
  else
    reinterpret_cast<double*>(base)[i] = v;
}

__device__ __forceinline__ bool nonfinite(float v) {
  return (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
}

// np.maximum(y, 0): NaN wins, -0 -> +0 (numpy returns +0 for maximum(-0., 0.)).
__device__ __forceinline__ float relu_exact(float y) { return (y > 0.0f || y != y) ? y : 0.0f; }

__device__ __forceinline__ float activate(float y, int act) {
  if (act == SMLRT_RELU) return relu_exact(y);
  if (act == SMLRT_TANH) return tanhf(y);
  return y;
}


__device__ __forceinline__ int64_t element_address(const DevPlan& P, uint32_t r, int c) {
  if (P.uniform) return P.col_off[c] + row_offset_uniform(P, r);
  uint32_t idx[SMLRT_MAX_SWEEP];
  unravel(P, r, idx);
  return col_address(P, c, idx);
}


}  // namespace
}  // namespace smlrt
