// TMEM read bandwidth of tcgen05.ld (epilogue-style drains) while one thread
// keeps the tensor core busy with M=128 N=256 K=16 MMAs into other TMEM
// columns.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2407_18352_b200/csrc tmem_contention.cu -o tmem_contention
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"
using namespace smlrt::ptx;

template <int MMA_ON, int LDW>
__global__ void bench(int iters, unsigned long long* cyc, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;                 // A [128 x 16] SW32 (junk)
  uint8_t* sb = sm + 4096;          // B [256 x 16] SW32 (junk)
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 3072; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); stop = 0; }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  unsigned long long t0 = clock64();
  if (warp == 0) {
    if (MMA_ON) {
      const uint64_t ad = smem_desc(smem_u32(sa), 256, kSwizzle32), bd = smem_desc(smem_u32(sb), 256, kSwizzle32);
      int n = 0;
      while (!stop) {  // D = cols [256, 512)
        for (int k = 0; k < 8; ++k) mma_ss_elect(tbase + 256, ad, bd, (1u << 4) | (1u << 7) | (1u << 10) | ((256 >> 3) << 17) | ((128 >> 4) << 24), 1);
        ++n;
        if ((n & 3) == 0) { mma_commit_elect(&bar); mbar_wait(&bar, ((n >> 2) - 1) & 1); }
      }
    }
  } else if (warp > 0 && warp <= LDW) {
    const uint32_t base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
      uint32_t v[32];
      tmem_ld32(base + ((i * 32) & 255), v);  // cols [0, 256)
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) acc ^= v[e];
    }
    if (acc == 0x12345u) sink[threadIdx.x] = acc;
  }
  // ld warps finish -> stop the MMA warp
  if (warp > 0) {
    asm volatile("bar.sync 1, %0;" :: "r"(LDW * 32));
    if (warp == 1 && lane == 0) { cyc[blockIdx.x] = clock64() - t0; stop = 1; }
  }
  __syncthreads();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int MMA, int LDW>
void run(const char* name, int iters) {
  unsigned long long* cyc; uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 4096);
  auto k = bench<MMA, LDW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  k<<<148, 32 * (LDW + 1), 16384>>>(iters, cyc, sink);
  k<<<148, 32 * (LDW + 1), 16384>>>(iters, cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
  const double bytes = (double)iters * LDW * 32 * 4 * 32;
  printf("%-28s ld warps %2d: %6.1f B/clk/SM  (%.0f cycles, %s)\n", name, LDW, bytes / avg, avg, cudaGetErrorString(e));
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  run<0, 4>("no MMA", 2048);
  run<1, 4>("MMA N=256 running", 2048);
  run<0, 8>("no MMA", 2048);
  run<1, 8>("MMA N=256 running", 2048);
  run<0, 12>("no MMA", 2048);
  run<1, 12>("MMA N=256 running", 2048);
  return 0;
}
