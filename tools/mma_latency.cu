// Round-trip latency of one tcgen05.mma (M=128, K=16, N = 64/128/256) ->
// tcgen05.commit -> mbarrier wait, and of tcgen05.ld x16 -> wait::ld, measured
// by one CTA with clock64.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2407_18352_b200/csrc mma_latency.cu -o mma_latency
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"
using namespace smlrt::ptx;

template <int ALT>
__global__ void k(unsigned long long* out) {
  __shared__ __align__(1024) uint8_t sm[16384];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot;
  if (warp == 0) {
    const uint64_t ad = smem_desc(smem_u32(sm), 256, kSwizzle32), bd = smem_desc(smem_u32(sm + 4096), 256, kSwizzle32);
    uint32_t ph = 0;
    const int Ns[3] = {64, 128, 256};
    for (int ni = 0; ni < 3; ++ni) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(Ns[ni] >> 3) << 17) | ((128 >> 4) << 24);
      for (int nm = 1; nm <= 16; nm *= 4) {
        unsigned long long best = ~0ull, sum = 0;
        for (int rep = 0; rep < 20; ++rep) {
          __syncwarp();
          const unsigned long long t0 = clock64();
          for (int j = 0; j < nm; ++j) mma_ss_elect(t + (ALT ? (j & 1) * 256 : 0), ad, bd, idesc, j > 1 || (!ALT && j > 0));
          mma_commit_elect(&bar);
          mbar_wait(&bar, ph);
          ph ^= 1;
          tc_fence_after();
          const unsigned long long dt = clock64() - t0;
          if (rep >= 4) { sum += dt; if (dt < best) best = dt; }
        }
        if (threadIdx.x == 0) { out[ni * 3 + (nm == 1 ? 0 : nm == 4 ? 1 : 2)] = sum / 16; }
      }
    }
    // tcgen05.ld x16 -> wait round trip
    unsigned long long s2 = 0;
    for (int rep = 0; rep < 20; ++rep) {
      uint32_t v[16];
      const unsigned long long t0 = clock64();
      tmem_ld16(t, v);
      tmem_wait_ld16(v);
      const unsigned long long dt = clock64() - t0;
      if (rep >= 4) s2 += dt;
      if (v[0] == 12345u) out[15] = v[1];
    }
    if (threadIdx.x == 0) out[9] = s2 / 16;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(t, 512); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 16 * 8); cudaMemset(d, 0, 128);
  for (int alt = 0; alt < 2; ++alt) {
  if (alt) k<1><<<1, 128>>>(d); else k<0><<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[16]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s accumulators: status %s\n", alt ? "two alternating" : "one", cudaGetErrorString(e));
  const int Ns[3] = {64, 128, 256};
  for (int ni = 0; ni < 3; ++ni)
    printf("N=%3d: 1 MMA + commit + wait %llu cyc, 4 MMAs %llu, 16 MMAs %llu\n", Ns[ni], h[ni * 3], h[ni * 3 + 1], h[ni * 3 + 2]);
  printf("tcgen05.ld x16 + wait::ld: %llu cyc\n", h[9]);
  }
  return 0;
}
