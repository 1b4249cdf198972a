// Cycles per K=16 bf16 MMA in a 16-step accumulation chain (M=128, N=64/128/256)
// with the A/B descriptors advancing through SW128 K-major operands as a real
// GEMM K loop does (not the same operand every time).  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2407_18352_b200/csrc mma_chain.cu -o mma_chain
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"
using namespace smlrt::ptx;

__global__ void k(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (192 * 1024) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot;
  if (warp == 0) {
    // A: 128 rows x 256 K (4 SW128 chunks of 16 KB) at sm; B: up to 256 rows x 256 K (4 chunks of 32 KB) at sm+64K
    const uint64_t a0 = smem_desc(smem_u32(sm), 1024, kSwizzle128);
    const uint64_t b0 = smem_desc(smem_u32(sm + 65536), 1024, kSwizzle128);
    uint32_t ph = 0;
    const int Ns[3] = {64, 128, 256};
    for (int ni = 0; ni < 3; ++ni) {
      const int N = Ns[ni];
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128 >> 4) << 24);
      for (int alt = 0; alt < 2; ++alt) {
        unsigned long long sum = 0;
        for (int rep = 0; rep < 20; ++rep) {
          __syncwarp();
          const unsigned long long t0 = clock64();
#pragma unroll
          for (int ks = 0; ks < 16; ++ks) {
            const int kc = ks >> 2, k = ks & 3;
            mma_ss_elect(t + (alt ? (ks & 1) * 256 : 0), a0 + ((kc * 16384 + k * 32) >> 4),
                         b0 + ((kc * N * 128 + k * 32) >> 4), idesc, alt ? ks > 1 : ks > 0);
          }
          mma_commit_elect(&bar);
          mbar_wait(&bar, ph);
          ph ^= 1;
          tc_fence_after();
          const unsigned long long dt = clock64() - t0;
          if (rep >= 4) sum += dt;
        }
        if (threadIdx.x == 0) out[ni * 2 + alt] = sum / 16;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(t, 512); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 16 * 8); cudaMemset(d, 0, 128);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<1, 128, 200 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[16]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("status %s\n", cudaGetErrorString(e));
  const int Ns[3] = {64, 128, 256};
  for (int ni = 0; ni < 3; ++ni)
    printf("N=%3d: 16 K-steps (advancing operands) one accumulator %llu cyc (%.0f/MMA), two alternating %llu (%.0f/MMA)\n",
           Ns[ni], h[ni * 2], h[ni * 2] / 16.0, h[ni * 2 + 1], h[ni * 2 + 1] / 16.0);
  return 0;
}
