// Latency and throughput of the warp-level mma.sync shapes the small-MLP and
// stencil kernels use (m16n8k16 bf16, m16n8k8 tf32) on sm_100a, by clock64.
// Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_sync_bench.cu -o mma_sync_bench
#include <cstdio>
#include <cstdint>

template <int CH, bool TF32>
__global__ void k(unsigned long long* out, float* sink, int iters) {
  float d[CH][4];
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0.f;
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (TF32)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  float s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

template <int CH, bool TF32>
void run(const char* name, int warps, unsigned long long* d_out, float* sink) {
  const int iters = 4096;
  k<CH, TF32><<<1, 32 * warps>>>(d_out, sink, iters);
  cudaDeviceSynchronize();
  unsigned long long c;
  cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / iters;  // cycles per loop iteration (CH mma per warp)
  printf("%s chains=%d warps/SM=%d: %.2f cycles per iteration -> %.2f cycles per mma per warp, SM rate %.3f mma/cycle\n",
         name, CH, warps, per, per / CH, CH * warps / per);
}

int main() {
  unsigned long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 8);
  cudaMalloc(&sink, 1 << 20);
  for (int w : {1, 4, 8, 16, 32}) {
    run<1, false>("bf16 m16n8k16", w, d_out, sink);
    run<4, false>("bf16 m16n8k16", w, d_out, sink);
    run<8, false>("bf16 m16n8k16", w, d_out, sink);
  }
  for (int w : {1, 4, 16}) {
    run<1, true>("tf32 m16n8k8", w, d_out, sink);
    run<8, true>("tf32 m16n8k8", w, d_out, sink);
  }
  return 0;
}
