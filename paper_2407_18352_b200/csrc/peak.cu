// FP32 CUDA-core peak microbenchmark (the roofline denominator of the exact
// fp32 path: "measure it with an FMA loop the same way").
//
// Three instruction mixes, each thread running 8 independent chains so the
// pipes, not dependency latency, set the rate:
//   mode 0  FFMA          fma.rn.f32                      2 flop / instruction
//   mode 1  FMUL + FADD   mul.rn.f32 then add.rn.f32      1 flop / instruction
//   mode 2  packed pairs  mul.rn.f32x2 then fma.rn.f32x2(p, 1, acc)
//                         (the exact kernels' ordered mul-then-add sequence on
//                         f32x2 pairs)                     2 flop / instruction
// The result is flop/s over the whole device (one launch, CUDA events).
#include "common.cuh"

namespace smlrt {
namespace {

constexpr int kChains = 8;

template <int MODE>
__global__ void __launch_bounds__(256) fp32_peak_kernel(float* out, int iters, float w, float one_f) {
  if constexpr (MODE == 2) {
    uint64_t acc[kChains], wp, one;
    asm("mov.b64 %0, {%1, %1};" : "=l"(wp) : "f"(w));
    // `one` arrives as a kernel parameter: a literal 1 would let ptxas fold
    // fma(p, 1, acc) into an add and contract the pair into one FFMA2
    asm("mov.b64 %0, {%1, %1};" : "=l"(one) : "f"(one_f));
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      const float v = (float)(threadIdx.x + c) * 1e-7f;
      asm("mov.b64 %0, {%1, %1};" : "=l"(acc[c]) : "f"(v));
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) {
        uint64_t p;
        asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(acc[c]), "l"(wp));
        asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[c]) : "l"(p), "l"(one));
      }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[c]));
      s += lo + hi;
    }
    if (s == 12345.0f) out[threadIdx.x] = s;  // keeps the chains live
  } else {
    float acc[kChains], x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      x[c] = (float)(threadIdx.x + c) * 1e-7f;
      acc[c] = x[c];
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) {
        if constexpr (MODE == 0) {
          asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[c]) : "f"(x[c]), "f"(w));
        } else {
          float p;
          asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(p) : "f"(acc[c]), "f"(w));
          asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(acc[c]) : "f"(p));
        }
      }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += acc[c];
    if (s == 12345.0f) out[threadIdx.x] = s;
  }
}

}  // namespace
}  // namespace smlrt

using namespace smlrt;

extern "C" int smlrt_fp32_peak(int32_t mode, double* flops_per_s) {
  if (!flops_per_s || mode < 0 || mode > 2) return fail(SMLRT_E_INVALID, "fp32_peak: bad argument");
  int dev = 0, sms = 0;
  SMLRT_CUDA(cudaGetDevice(&dev));
  SMLRT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  float* out = nullptr;
  SMLRT_CUDA(cudaMalloc(&out, 256 * sizeof(float)));
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  auto launch = [&](int it) {
    if (mode == 0) fp32_peak_kernel<0><<<blocks, threads>>>(out, it, 0.5f, 1.0f);
    else if (mode == 1) fp32_peak_kernel<1><<<blocks, threads>>>(out, it, 0.5f, 1.0f);
    else fp32_peak_kernel<2><<<blocks, threads>>>(out, it, 0.5f, 1.0f);
  };
  cudaEvent_t e0, e1;
  SMLRT_CUDA(cudaEventCreate(&e0));
  SMLRT_CUDA(cudaEventCreate(&e1));
  launch(256);  // warm-up (clocks up, module loaded)
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    SMLRT_CUDA(cudaEventRecord(e0));
    launch(iters);
    SMLRT_CUDA(cudaEventRecord(e1));
    SMLRT_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    SMLRT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  SMLRT_CUDA(cudaGetLastError());
  const double per_iter = mode == 0 ? 2.0 * kChains : (mode == 1 ? 2.0 * kChains : 4.0 * kChains);
  *flops_per_s = (double)blocks * threads * iters * per_iter / (best * 1e-3);
  return SMLRT_OK;
}
