// How many CTAs per SM hold TMEM at once: 8 x 148 CTAs of 128 threads each
// allocate `ncols` TMEM columns (or none), spin ~20 us, free them.  The
// kernel time shows the real concurrency (20 us = all resident).  Not part
// of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2407_18352_b200/csrc tmem_occupancy.cu -o tmem_occupancy
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"
using namespace smlrt::ptx;

__global__ void __launch_bounds__(128, 8) k(int ncols, int use, unsigned spin_ns, unsigned* maxc, unsigned* cur) {
  __shared__ uint32_t slot;
  __shared__ __align__(16) uint8_t pad[10 * 1024];
  if (use && threadIdx.x < 32) tmem_alloc(&slot, ncols);
  pad[threadIdx.x] = 1;
  __syncthreads();
  uint32_t sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (threadIdx.x == 0) {
    unsigned c = atomicAdd(&cur[sm], 1) + 1;
    atomicMax(&maxc[sm], c);
  }
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(200);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  } while (t1 - t0 < spin_ns);
  if (threadIdx.x == 0) atomicSub(&cur[sm], 1);
  __syncthreads();
  if (use && threadIdx.x < 32) tmem_dealloc(slot, ncols);
  if (pad[threadIdx.x + 1] == 7) maxc[200] = 1;
}

int main() {
  unsigned *maxc, *cur;
  cudaMalloc(&maxc, 256 * 4);
  cudaMalloc(&cur, 256 * 4);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, 0);
  printf("occupancy API: %d CTAs per SM\n", occ);
  const int cases[][2] = {{0, 0}, {1, 32}, {1, 64}, {1, 128}, {1, 256}};
  for (auto& c : cases) {
    cudaMemset(maxc, 0, 256 * 4);
    cudaMemset(cur, 0, 256 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<sms * 8, 128>>>(c[1], c[0], 20000, maxc, cur);  // warm
    cudaMemset(maxc, 0, 256 * 4);
    cudaEventRecord(e0);
    k<<<sms * 8, 128>>>(c[1], c[0], 20000, maxc, cur);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned h[256];
    cudaMemcpy(h, maxc, sizeof h, cudaMemcpyDeviceToHost);
    unsigned mx = 0, mn = 1000;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx, mn = h[i] < mn ? h[i] : mn;
    printf("tmem %s %3d cols: %.1f us for 8 x %d CTAs of 20 us; concurrent CTAs per SM %u..%u (%s)\n",
           c[0] ? "alloc" : "none ", c[1], ms * 1000, sms, mn, mx, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
