// Microbenchmarks of TMEM -> RF reads (tcgen05.ld) on sm_100a, and a probe of
// the TMEM layout of an f16 accumulator.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2407_18352_b200/csrc tmem_bench.cu -o tmem_bench
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"
using namespace smlrt::ptx;

__device__ __forceinline__ void ld16(uint32_t a, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(a));
}

template <int MODE>
__global__ void tmem_read_bench(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t col = ((i * 64) + (warp >> 2) * 32) & 511;
    if constexpr (MODE == 0) {  // x32, wait each
      uint32_t v[32];
      tmem_ld32(base + col, v);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) acc ^= v[e];
    } else if constexpr (MODE == 1) {  // 2 x32 then one wait
      uint32_t v[32], w[32];
      tmem_ld32(base + col, v);
      tmem_ld32(base + ((col + 256) & 511), w);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) acc ^= v[e] + w[e];
    } else {  // x16, wait each
      uint32_t v[16];
      ld16(base + col, v);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 16; ++e) acc ^= v[e];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(slot, 512);
  }
}

// D[128 x 64] = A[128 x 16] * B[64 x 16]^T in f16 inputs; accumulator format
// `cf` (0 = f16, 1 = f32); dumps the raw 32-bit TMEM words of lane 0..127, cols 0..63
__global__ void f16acc_probe(int cf, uint32_t* out) {
  __shared__ __align__(1024) uint8_t sa[128 * 32];
  __shared__ __align__(1024) uint8_t sb[64 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 128 * 16; i += 128) {
    const int r = i / 16, k = i % 16;
    *reinterpret_cast<__half*>(sa + sw32_offset(r, k)) = __float2half(k == 0 ? 1.0f : 0.0f);
  }
  for (int i = threadIdx.x; i < 64 * 16; i += 128) {
    const int n = i / 16, k = i % 16;
    *reinterpret_cast<__half*>(sb + sw32_offset(n, k)) = __float2half(k == 0 ? (float)n + 0.5f : 0.0f);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(&slot, 128);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = ((uint32_t)cf << 4) | ((64 >> 3) << 17) | ((128 >> 4) << 24);
    mma_bf16(t, smem_desc(smem_u32(sa), 256, kSwizzle32), smem_desc(smem_u32(sb), 256, kSwizzle32), idesc, 0);
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < 64; c += 32) {
    uint32_t v[32];
    tmem_ld32(t + ((uint32_t)(warp * 32) << 16) + c, v);
    tmem_wait_ld();
    for (int e = 0; e < 32; ++e) out[(warp * 32 + lane) * 64 + c + e] = v[e];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(t, 128);
  }
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 4096);
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16}) {
      auto k = mode == 0 ? tmem_read_bench<0> : mode == 1 ? tmem_read_bench<1> : tmem_read_bench<2>;
      k<<<148, warps * 32>>>(iters, cyc, sink);
      k<<<148, warps * 32>>>(iters, cyc, sink);
      cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
      const double bytes = (double)iters * warps * 32 * 4 * (mode == 0 ? 32 : mode == 1 ? 64 : 16);
      printf("mode %d (%s) warps %2d: %.1f B/clk/SM  (%.0f cycles)\n", mode,
             mode == 0 ? "x32+wait" : mode == 1 ? "2x32+wait" : "x16+wait", warps, bytes / avg, avg);
    }
  uint32_t* d;
  cudaMalloc(&d, 128 * 64 * 4);
  static uint32_t hbuf[128 * 64];
  for (int cf = 0; cf < 2; ++cf) {
    cudaMemset(d, 0xff, 128 * 64 * 4);
    f16acc_probe<<<1, 128>>>(cf, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hbuf, d, sizeof(hbuf), cudaMemcpyDeviceToHost);
    printf("acc %s (%s): lane0 cols0-7:", cf ? "f32" : "f16", cudaGetErrorString(e));
    for (int c = 0; c < 8; ++c) printf(" %08x", hbuf[c]);
    printf("\n  lane5 cols 30-35:");
    for (int c = 30; c < 36; ++c) printf(" %08x", hbuf[5 * 64 + c]);
    printf("\n");
  }
  return 0;
}
