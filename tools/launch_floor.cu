// Host round-trip floor of a synchronous call on this box: one empty kernel
// launched directly or as a 1-node CUDA graph, then cudaStreamSynchronize or
// a spin on a mapped host word the kernel writes.  Compare with the prepared
// region's per-call cost (tools/overhead.py).  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 launch_floor.cu -o launch_floor
#include <chrono>
#include <cstdio>

__global__ void empty_kernel(volatile unsigned* flag, unsigned v) {
  if (flag && threadIdx.x == 0) *flag = v;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  unsigned* h;
  cudaHostAlloc(&h, 4, cudaHostAllocMapped);
  unsigned* d;
  cudaHostGetDevicePointer(&d, h, 0);
  *h = 0;
  const int N = 2000;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  for (int i = 0; i < 200; ++i) empty_kernel<<<1, 32, 0, s>>>(nullptr, 0);
  cudaStreamSynchronize(s);
  auto t0 = now();
  for (int i = 0; i < N; ++i) {
    empty_kernel<<<1, 32, 0, s>>>(nullptr, 0);
    cudaStreamSynchronize(s);
  }
  printf("direct launch + stream sync: %.2f us\n", us(t0, now()) / N);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  empty_kernel<<<1, 32, 0, s>>>(nullptr, 0);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int i = 0; i < 200; ++i) cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  t0 = now();
  for (int i = 0; i < N; ++i) {
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
  }
  printf("1-node graph launch + stream sync: %.2f us\n", us(t0, now()) / N);
  t0 = now();
  for (int i = 0; i < N; ++i) cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  printf("1-node graph launch alone (async): %.2f us\n", us(t0, now()) / N);
  t0 = now();
  for (unsigned i = 1; i <= (unsigned)N; ++i) {
    empty_kernel<<<1, 32, 0, s>>>(d, i);
    while (*(volatile unsigned*)h != i) {
    }
  }
  printf("direct launch + spin on mapped flag: %.2f us\n", us(t0, now()) / N);
  cudaStreamSynchronize(s);
  return 0;
}
