// Exact-fp32 CUDA-core kernels for the CNN surrogates and wide dense layers.
//
//   conv_front_kernel  : window gather (through the in-plan, or a dense batch)
//                        -> non-overlapping conv2d -> act -> optional maxpool2d,
//                        one CTA per sweep row (frame); the conv is the
//                        reference's patch functor + dense layer, so every
//                        output accumulates over (c, dy, dx) in row-major
//                        order with separate RN multiply and add (bitwise
//                        equal to _matmul_rowwise, models.py:188-194).
//   dense_tiled_kernel : Y = act(X W^T + b), 64x64 output tile per CTA, K
//                        staged through shared memory in chunks of 32; each
//                        output still accumulates over the input index in
//                        ascending order with separate multiply and add.
// The C4 ParticleFilter config (conv 8x8/8 1->8, relu, maxpool 2, 512->128
// relu, 128->2) runs as front kernel + two tiled dense layers + scatter.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include <cstring>

#include <cuda.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace smlrt {



namespace {

__device__ __forceinline__ float act_exact(float y, int act) {
  if (act == SMLRT_RELU) return (y > 0.0f || y != y) ? y : 0.0f;  // np.maximum(y, 0): NaN wins, -0 -> +0
  if (act == SMLRT_TANH) return tanhf(y);
  return y;
}

__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

struct FrontArgs {
  // input addressing: either a dense batch (x != nullptr, row pitch in_feat)
  // or the in-plan (uniform 2-D window fast path when win_w > 0)
  const float* x;
  int64_t r0, r1;
  int C, H, W, K, OC, OH, OW;  // conv geometry
  int act;
  int pool;                    // maxpool kernel (1 = none)
  int out_w;                   // floats per output row
  const float* w;              // [OC][C*K*K]
  const float* b;              // [OC]
  float* out;                  // [rows][out_w]
  const void* src;             // plan array base (window path)
  int src_dt;
  // bf16 tail (the CNN bf16 path): features as bf16 rows of out_pitch
  // elements instead of f32 rows in `out`
  __nv_bfloat16* out_bf;
  int out_pitch;
};

// feature i of the front's output row (row - r0)
__device__ __forceinline__ void put_feat(const FrontArgs& a, int64_t r, int i, float v) {
  if (a.out_bf != nullptr)
    a.out_bf[r * a.out_pitch + i] = __float2bfloat16_rn(v);
  else
    a.out[r * a.out_w + i] = v;
}

constexpr int kMaxOC = 16;

__global__ void __launch_bounds__(256) conv_front_kernel(const __grid_constant__ FrontArgs a,
                                                         const __grid_constant__ DevPlan P) {
  extern __shared__ float sm[];
  const int KK = a.C * a.K * a.K;
  float* ws = sm;                          // [KK][OC] (transposed: o fastest)
  float* conv = sm + KK * a.OC;            // [OC][OH][OW]
  for (int i = threadIdx.x; i < KK * a.OC; i += blockDim.x) {
    const int f = i / a.OC, o = i % a.OC;
    ws[i] = a.w[o * KK + f];
  }
  __syncthreads();
  const int64_t row = a.r0 + blockIdx.x;
  int64_t base = 0;
  if (a.x == nullptr) base = P.col_off0 + row_offset_uniform(P, (uint32_t)row);
  const int npos = a.OH * a.OW;
  for (int p = threadIdx.x; p < npos; p += blockDim.x) {
    const int py = p / a.OW, px = p % a.OW;
    float acc[kMaxOC];
#pragma unroll
    for (int o = 0; o < kMaxOC; ++o) acc[o] = 0.0f;
    int f = 0;
    for (int c = 0; c < a.C; ++c)
      for (int dy = 0; dy < a.K; ++dy) {
        const int y = py * a.K + dy;
        for (int dx = 0; dx < a.K; ++dx, ++f) {
          const int xx = px * a.K + dx;
          const int64_t col = ((int64_t)c * a.H + y) * a.W + xx;  // flattened image index
          float v;
          if (a.x != nullptr) {
            v = __ldg(a.x + (row - a.r0) * (int64_t)a.C * a.H * a.W + col);
          } else if (P.win_w > 0 && a.C == 1) {
            const int64_t addr = base + (int64_t)y * P.win_pitch + xx;
            v = a.src_dt == SMLRT_F32 ? __ldg(reinterpret_cast<const float*>(a.src) + addr)
                                      : __double2float_rn(__ldg(reinterpret_cast<const double*>(a.src) + addr));
          } else {
            const int64_t addr = __ldg(P.col_off + col) - P.col_off0 + base;
            v = a.src_dt == SMLRT_F32 ? __ldg(reinterpret_cast<const float*>(a.src) + addr)
                                      : __double2float_rn(__ldg(reinterpret_cast<const double*>(a.src) + addr));
          }
          const float* wf = ws + f * a.OC;
#pragma unroll
          for (int o = 0; o < kMaxOC; ++o)
            if (o < a.OC) acc[o] = __fadd_rn(acc[o], __fmul_rn(v, wf[o]));
        }
      }
#pragma unroll
    for (int o = 0; o < kMaxOC; ++o)
      if (o < a.OC) conv[o * npos + p] = act_exact(__fadd_rn(acc[o], __ldg(a.b + o)), a.act);
  }
  __syncthreads();
  const int64_t orr = row - a.r0;
  if (a.pool <= 1) {
    for (int i = threadIdx.x; i < a.OC * npos; i += blockDim.x) put_feat(a, orr, i, conv[i]);
    return;
  }
  const int PH = a.OH / a.pool, PW = a.OW / a.pool;
  for (int i = threadIdx.x; i < a.OC * PH * PW; i += blockDim.x) {
    const int o = i / (PH * PW), q = i % (PH * PW), qy = q / PW, qx = q % PW;
    float m = conv[o * npos + (qy * a.pool) * a.OW + qx * a.pool];
    for (int dy = 0; dy < a.pool; ++dy)
      for (int dx = 0; dx < a.pool; ++dx)
        m = max_nan(m, conv[o * npos + (qy * a.pool + dy) * a.OW + qx * a.pool + dx]);
    put_feat(a, orr, i, m);
  }
}

// Compile-time geometry (C = 1, K = 8, OC = 8: the C4 model): one thread per
// conv position, each patch row fetched as two float4, weights as float4
// broadcasts from shared memory; same (dy, dx) accumulation order.
template <int K, int OC>
__global__ void __launch_bounds__(256) conv_front_fixed_kernel(const __grid_constant__ FrontArgs a,
                                                               const __grid_constant__ DevPlan P) {
  static_assert(K % 4 == 0 && OC % 4 == 0, "vector widths");
  extern __shared__ float sm[];
  float* ws = sm;                 // [K*K][OC]
  float* conv = sm + K * K * OC;  // [OC][OH][OW]
  for (int i = threadIdx.x; i < K * K * OC; i += blockDim.x) ws[i] = a.w[(i % OC) * K * K + i / OC];
  __syncthreads();
  const int64_t row = a.r0 + blockIdx.x;
  const float* img;
  int64_t pitch;
  if (a.x != nullptr) {
    img = a.x + (row - a.r0) * (int64_t)a.H * a.W;
    pitch = a.W;
  } else {
    img = reinterpret_cast<const float*>(a.src) + P.col_off0 + row_offset_uniform(P, (uint32_t)row);
    pitch = P.win_pitch;
  }
  const int npos = a.OH * a.OW;
  for (int p = threadIdx.x; p < npos; p += blockDim.x) {
    const int py = p / a.OW, px = p % a.OW;
    float acc[OC];
#pragma unroll
    for (int o = 0; o < OC; ++o) acc[o] = 0.0f;
    const float* prow = img + (int64_t)(py * K) * pitch + px * K;
#pragma unroll
    for (int dy = 0; dy < K; ++dy) {
      float v[K];
#pragma unroll
      for (int q = 0; q < K / 4; ++q) {
        const float4 u = __ldg(reinterpret_cast<const float4*>(prow + dy * pitch) + q);
        v[4 * q] = u.x;
        v[4 * q + 1] = u.y;
        v[4 * q + 2] = u.z;
        v[4 * q + 3] = u.w;
      }
#pragma unroll
      for (int dx = 0; dx < K; ++dx) {
        const float* wf = ws + (dy * K + dx) * OC;
#pragma unroll
        for (int o4 = 0; o4 < OC / 4; ++o4) {
          const float4 w4 = *reinterpret_cast<const float4*>(wf + 4 * o4);
          acc[4 * o4] = __fadd_rn(acc[4 * o4], __fmul_rn(v[dx], w4.x));
          acc[4 * o4 + 1] = __fadd_rn(acc[4 * o4 + 1], __fmul_rn(v[dx], w4.y));
          acc[4 * o4 + 2] = __fadd_rn(acc[4 * o4 + 2], __fmul_rn(v[dx], w4.z));
          acc[4 * o4 + 3] = __fadd_rn(acc[4 * o4 + 3], __fmul_rn(v[dx], w4.w));
        }
      }
    }
#pragma unroll
    for (int o = 0; o < OC; ++o) conv[o * npos + p] = act_exact(__fadd_rn(acc[o], __ldg(a.b + o)), a.act);
  }
  __syncthreads();
  const int64_t orr = row - a.r0;
  if (a.pool <= 1) {
    for (int i = threadIdx.x; i < OC * npos; i += blockDim.x) put_feat(a, orr, i, conv[i]);
    return;
  }
  const int PH = a.OH / a.pool, PW = a.OW / a.pool;
  for (int i = threadIdx.x; i < OC * PH * PW; i += blockDim.x) {
    const int o = i / (PH * PW), q = i % (PH * PW), qy = q / PW, qx = q % PW;
    float m = conv[o * npos + (qy * a.pool) * a.OW + qx * a.pool];
    for (int dy = 0; dy < a.pool; ++dy)
      for (int dx = 0; dx < a.pool; ++dx)
        m = max_nan(m, conv[o * npos + (qy * a.pool + dy) * a.OW + qx * a.pool + dx]);
    put_feat(a, orr, i, m);
  }
}

// C4 front, specialised for one 1-channel frame per CTA with a 16 x 16
// position grid (K = 8, OC = 8 over a 128 x 128 window), conv + act + 2x2
// max-pool in registers: warp w owns conv rows 2w, 2w+1 (lane = 16 * row +
// column), the pool is two butterfly shuffles.  Weights and bias ride in the
// parameter bank (uniform LDCU into FMUL2 operands); output pairs (o, o+1)
// accumulate with packed mul.rn.f32x2 + fma.rn.f32x2(p, 1, acc), the same
// ordered multiply-then-add as the reference's _matmul_rowwise over the
// (dy, dx) patch features -- bitwise equal, half the FP32 issue slots.
struct ConvW8 {
  float w[64 * 8];  // [(dy*8 + dx)][o]
  float b[8];
  uint64_t one2;    // (1.0f, 1.0f), opaque to ptxas (see kernels_simt.cu add2)
};

__device__ __forceinline__ uint64_t cpk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void cupk2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t cmul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t cadd2(uint64_t acc, uint64_t p, uint64_t one) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(p), "l"(one), "l"(acc));
  return r;
}

// Window loads with a 64-B L2 prefetch-size hint.  A 512-B window row starts
// 64 B into a 128-B line; with the default fetch size the L2 reads whole
// 128-B lines from DRAM (1.342 GB for 1.074 GB of windows on C4, measured, the
// same through TMA with or without L2 promotion); `.L2::64B` fetches only the
// touched 64-B halves: DRAM reads = the window bytes (1.08 GB), C4's conv
// front 195 -> 158 us.
__device__ __forceinline__ float4 ld_window(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L2::64B.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__global__ void __launch_bounds__(256) conv_pool_k8oc8_kernel(const __grid_constant__ FrontArgs a,
                                                              const __grid_constant__ DevPlan P,
                                                              const __grid_constant__ ConvW8 cw) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int py = 2 * warp + (lane >> 4), px = lane & 15;
  const int64_t row = a.r0 + blockIdx.x;
  const float* img;
  int64_t pitch;
  if (a.x != nullptr) {
    img = a.x + (row - a.r0) * (int64_t)a.H * a.W;
    pitch = a.W;
  } else {
    img = reinterpret_cast<const float*>(a.src) + P.col_off0 + row_offset_uniform(P, (uint32_t)row);
    pitch = P.win_pitch;
  }
  const float* prow = img + (int64_t)(py * 8) * pitch + px * 8;
  float4 u[8][2];
#pragma unroll
  for (int dy = 0; dy < 8; ++dy) {  // all 16 loads in flight before the math
    u[dy][0] = ld_window(reinterpret_cast<const float4*>(prow + dy * pitch));
    u[dy][1] = ld_window(reinterpret_cast<const float4*>(prow + dy * pitch) + 1);
  }
  uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
  for (int dy = 0; dy < 8; ++dy) {
    const float v[8] = {u[dy][0].x, u[dy][0].y, u[dy][0].z, u[dy][0].w,
                        u[dy][1].x, u[dy][1].y, u[dy][1].z, u[dy][1].w};
#pragma unroll
    for (int dx = 0; dx < 8; ++dx) {
      const uint64_t vv = cpk2(v[dx], v[dx]);
      const float* wf = cw.w + (dy * 8 + dx) * 8;
#pragma unroll
      for (int op = 0; op < 4; ++op)
        acc[op] = cadd2(acc[op], cmul2(vv, *reinterpret_cast<const uint64_t*>(wf + 2 * op)), cw.one2);
    }
  }
  float y[8];
#pragma unroll
  for (int op = 0; op < 4; ++op) {
    cupk2(cadd2(acc[op], *reinterpret_cast<const uint64_t*>(cw.b + 2 * op), cw.one2), y[2 * op], y[2 * op + 1]);
    y[2 * op] = act_exact(y[2 * op], a.act);
    y[2 * op + 1] = act_exact(y[2 * op + 1], a.act);
  }
  const int64_t orr = row - a.r0;
  if (a.pool == 2) {
    // 2x2 window = lanes {l, l^1, l^16, l^17}; NaN propagates like np.max
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      float m = max_nan(y[o], __shfl_xor_sync(0xffffffffu, y[o], 1));
      m = max_nan(m, __shfl_xor_sync(0xffffffffu, m, 16));
      y[o] = m;
    }
    if (lane < 16 && (lane & 1) == 0) {
#pragma unroll
      for (int o = 0; o < 8; ++o) put_feat(a, orr, o * 64 + warp * 8 + (lane >> 1), y[o]);
    }
  } else {
#pragma unroll
    for (int o = 0; o < 8; ++o) put_feat(a, orr, o * 256 + py * 16 + px, y[o]);
  }
}

// ------------------------------------------------------------ tiled dense --
// Exact dense layer on output pairs: thread = 4 rows x 4 columns (2 column
// pairs), each multiply-accumulate a packed mul.rn.f32x2 + fma.rn.f32x2(p, 1,
// acc) in ascending k -- the reference's ordered rowwise product, bitwise,
// with half the FP32 issue slots of the scalar kernel above.  FUSE2 (out <=
// 128, one column block): the layer's activations stay in shared memory and
// the next dense layer (out2 <= 4 units, e.g. C4's 128 -> 2) runs in the
// same CTA, one ordered dot product per (row, unit).
#ifndef SMLRT_PF_TC
#define SMLRT_PF_TC 8
#endif
// TC = output columns per thread: 4 (32 rows x 128 columns per CTA) or 8 (64
// rows: three LDS.128 per 32 packed FP instructions instead of two per 16);
// with TC = 8 a thread's columns are two groups of four, [4 tj, +4) and
// [64 + 4 tj, +4), so each group's float4 reads are contiguous across threads
constexpr int PJ = 128, PK = 32, TC = SMLRT_PF_TC;
// PT threads per CTA (8 warps: 64-row tiles).  Measured on C4: 7 warps
// (56-row tiles, 293 CTAs for the 296 slots of 2 per SM instead of 256 CTAs)
// is equal (0.2763 vs 0.2771 ms region), so the CTA count is not the limiter
#ifndef SMLRT_PF_PT
#define SMLRT_PF_PT 256
#endif
constexpr int PT = SMLRT_PF_PT;
constexpr int PR = 4 * (PT / (PJ / TC));

template <bool FUSE2>
__global__ void __launch_bounds__(PT) dense_pair_kernel(const float* __restrict__ x, int64_t rows, int in, int out,
                                                         const float* __restrict__ W, const float* __restrict__ b,
                                                         int act, float* __restrict__ y, uint32_t* status,
                                                         const float* __restrict__ W2, const float* __restrict__ b2,
                                                         int out2, int act2, uint64_t one) {
  constexpr int CG = PJ / TC, NG = TC / 4;  // column groups per CTA, float4 groups per thread
  // hs (the fused tail's activations) reuses the K tiles' space after the K loop
  constexpr int XB = PK * (PR + 4), WB = PK * (PJ + 4), HB = FUSE2 ? PR * (PJ + 1) : 1;
  __shared__ __align__(16) float smem[XB + WB > HB ? XB + WB : HB];
  auto xs = reinterpret_cast<float(*)[PR + 4]>(smem);
  auto wsh = reinterpret_cast<float(*)[PJ + 4]>(smem + XB);
  auto hs = reinterpret_cast<float(*)[FUSE2 ? PJ + 1 : 1]>(smem);
  const int tr = threadIdx.x / CG, tj = threadIdx.x % CG;  // rows 4 tr .. +3
  const int64_t row0 = (int64_t)blockIdx.x * PR;
  const int j0 = blockIdx.y * PJ;
  auto col_of = [&](int g, int c) { return g * (PJ / NG) + 4 * tj + c; };  // group g, column c < 4
  uint64_t acc[4][TC / 2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int p = 0; p < TC / 2; ++p) acc[i][p] = 0ull;
  // the next K tile is fetched into registers while the current one is consumed
  constexpr int NX = (PR * PK + PT - 1) / PT, NW = (PJ * PK + PT - 1) / PT;
  float px[NX], pw[NW];
  auto fetch = [&](int k0) {
    const int kn = min(PK, in - k0);
#pragma unroll
    for (int u = 0; u < NX; ++u) {
      const int i = threadIdx.x + PT * u, r = i / PK, k = i % PK;
      const int64_t gr = row0 + r;
      px[u] = (i < PR * PK && gr < rows && k < kn) ? x[gr * in + k0 + k] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < NW; ++u) {
      const int i = threadIdx.x + PT * u, j = i / PK, k = i % PK;
      pw[u] = (i < PJ * PK && j0 + j < out && k < kn) ? __ldg(W + (int64_t)(j0 + j) * in + k0 + k) : 0.0f;
    }
  };
  fetch(0);
  for (int k0 = 0; k0 < in; k0 += PK) {
    const int kn = min(PK, in - k0);
#pragma unroll
    for (int u = 0; u < NX; ++u) {
      const int i = threadIdx.x + PT * u;
      if (i < PR * PK) xs[i % PK][i / PK] = px[u];
    }
#pragma unroll
    for (int u = 0; u < NW; ++u) {
      const int i = threadIdx.x + PT * u;
      if (i < PJ * PK) wsh[i % PK][i / PK] = pw[u];
    }
    __syncthreads();
    if (k0 + PK < in) fetch(k0 + PK);
    for (int k = 0; k < kn; ++k) {
      const float4 xv = *reinterpret_cast<const float4*>(&xs[k][tr * 4]);
      uint64_t w[TC / 2];
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        const float4 wv = *reinterpret_cast<const float4*>(&wsh[k][col_of(g, 0)]);
        w[2 * g] = cpk2(wv.x, wv.y);
        w[2 * g + 1] = cpk2(wv.z, wv.w);
      }
      const float xr[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t xx = cpk2(xr[i], xr[i]);
#pragma unroll
        for (int p = 0; p < TC / 2; ++p) acc[i][p] = cadd2(acc[i][p], cmul2(xx, w[p]), one);
      }
    }
    __syncthreads();
  }
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rl = tr * 4 + i;
    const int64_t r = row0 + rl;
#pragma unroll
    for (int p = 0; p < TC / 2; ++p) {
      float v[2];
      cupk2(acc[i][p], v[0], v[1]);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cl = col_of(p / 2, 2 * (p % 2) + e), c = j0 + cl;
        if (c < out) {
          const float hv = act_exact(__fadd_rn(v[e], __ldg(b + c)), act);
          if constexpr (FUSE2) {
            hs[rl][cl] = hv;
          } else if (r < rows) {
            y[r * out + c] = hv;
            bad |= (__float_as_uint(hv) & 0x7f800000u) == 0x7f800000u;
          }
        }
      }
    }
  }
  if constexpr (FUSE2) {
    __syncthreads();
    if ((int)threadIdx.x < PR * out2) {
      const int rl = threadIdx.x / out2, o = threadIdx.x % out2;
      const int64_t r = row0 + rl;
      float a2 = 0.0f;
      for (int f = 0; f < out; ++f) a2 = __fadd_rn(a2, __fmul_rn(hs[rl][f], __ldg(W2 + o * out + f)));
      const float yv = act_exact(__fadd_rn(a2, __ldg(b2 + o)), act2);
      if (r < rows) {
        y[r * out2 + o] = yv;
        bad = (__float_as_uint(yv) & 0x7f800000u) == 0x7f800000u;
      }
    }
  }
  if (status != nullptr && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    flag_nonfinite(status);
}

int launch_front(const smlrt_model_s& m, const float* x, const DevPlan* P, const void* src, int src_dt,
                 int64_t r0, int64_t r1, float* out, int* out_w, int* next_layer, cudaStream_t s,
                 __nv_bfloat16* out_bf = nullptr, int out_pitch = 0) {
  const DevLayer& c = m.layers[0];
  FrontArgs a{};
  a.x = x;
  a.r0 = r0;
  a.r1 = r1;
  a.C = c.in_c;
  a.H = c.in_h;
  a.W = c.in_w;
  a.K = c.kernel;
  a.OC = c.out_c;
  a.OH = c.in_h / c.kernel;
  a.OW = c.in_w / c.kernel;
  a.act = c.act;
  a.w = c.w;
  a.b = c.b;
  a.out = out;
  a.src = src;
  a.src_dt = src_dt;
  a.pool = 1;
  a.out_bf = out_bf;
  a.out_pitch = out_pitch;
  *next_layer = 1;
  if (m.n_layers > 1 && m.layers[1].kind == SMLRT_MAXPOOL2D) {
    a.pool = m.layers[1].kernel;
    *next_layer = 2;
  }
  a.out_w = m.layers[*next_layer - 1].out;
  *out_w = a.out_w;
  if (a.OC > kMaxOC) return fail(SMLRT_E_UNSUPPORTED, "conv2d with more than 16 output channels");
  const size_t smem = ((size_t)a.C * a.K * a.K * a.OC + (size_t)a.OC * a.OH * a.OW) * 4;
  if (smem > 200 * 1024) return fail(SMLRT_E_UNSUPPORTED, "conv2d front does not fit shared memory");
  static int configured = 0;
  if (!configured) {
    SMLRT_CUDA(cudaFuncSetAttribute(conv_front_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured = 1;
  }
  DevPlan dummy{};
  const bool aligned = (a.x != nullptr && a.W % 4 == 0) ||
                       (P != nullptr && src_dt == SMLRT_F32 && P->win_w == a.W && P->win_pitch % 4 == 0 &&
                        ((P->col_off0 + P->ustride[0]) % 4 == 0) && P->n_sweep == 1 && P->col_off0 % 4 == 0 &&
                        (reinterpret_cast<uintptr_t>(src) & 15) == 0);
  if (a.C == 1 && a.K == 8 && a.OC == 8 && aligned && a.OH == 16 && a.OW == 16 && (a.pool == 1 || a.pool == 2) &&
      m.host_params.size() >= 64 * 8 + 8) {
    ConvW8 cw{};
    const float* hw = m.host_params.data();  // conv layer first: W [OC][K*K], then b [OC]
    for (int o = 0; o < 8; ++o)
      for (int k = 0; k < 64; ++k) cw.w[k * 8 + o] = hw[o * 64 + k];
    for (int o = 0; o < 8; ++o) cw.b[o] = hw[64 * 8 + o];
    const float one[2] = {1.0f, 1.0f};
    std::memcpy(&cw.one2, one, sizeof(one));
    conv_pool_k8oc8_kernel<<<(unsigned)(r1 - r0), 256, 0, s>>>(a, P ? *P : dummy, cw);
    count_launch();
  } else if (a.C == 1 && a.K == 8 && a.OC == 8 && aligned) {
    conv_front_fixed_kernel<8, 8><<<(unsigned)(r1 - r0), 256, smem, s>>>(a, P ? *P : dummy);
    count_launch();
  } else {
    conv_front_kernel<<<(unsigned)(r1 - r0), 256, smem, s>>>(a, P ? *P : dummy);
    count_launch();
  }
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

// dense tail (layers [first, n)) over front output; ping-pong through t0/t1
uint64_t one2() {
  const float one[2] = {1.0f, 1.0f};
  uint64_t v;
  std::memcpy(&v, one, sizeof(v));
  return v;
}

int dense_tail(const smlrt_model_s& m, int first, const float* cur, int64_t rows, float* y, float* t0, float* t1,
               cudaStream_t s, uint32_t* status) {
  if (rows <= 0) return SMLRT_OK;
  // common CNN tail: dense (<= 128 units) -> dense (<= 4 units), fused in one launch
  if (m.n_layers - first == 2 && m.layers[first].kind == SMLRT_DENSE && m.layers[first + 1].kind == SMLRT_DENSE &&
      m.layers[first].out <= PJ && m.layers[first + 1].out <= 4) {
    const DevLayer &L1 = m.layers[first], &L2 = m.layers[first + 1];
    dim3 grid((unsigned)((rows + PR - 1) / PR), 1);
    dense_pair_kernel<true><<<grid, PT, 0, s>>>(cur, rows, L1.in, L1.out, L1.w, L1.b, L1.act, y, status, L2.w, L2.b,
                                                  L2.out, L2.act, one2());
    count_launch();
    SMLRT_CUDA(cudaGetLastError());
    return SMLRT_OK;
  }
  for (int l = first; l < m.n_layers; ++l) {
    const bool last = l == m.n_layers - 1;
    float* dst = last ? y : ((l - first) % 2 ? t1 : t0);
    if (int rc = launch_dense_exact_tiled(cur, rows, m.layers[l], dst, s, last ? status : nullptr)) return rc;
    cur = dst;
  }
  return SMLRT_OK;
}

}  // namespace

bool cnn_model(const smlrt_model_s& m) {
  if (m.n_layers < 1 || m.layers[0].kind != SMLRT_CONV2D) return false;
  int l = (m.n_layers > 1 && m.layers[1].kind == SMLRT_MAXPOOL2D) ? 2 : 1;
  for (; l < m.n_layers; ++l)
    if (m.layers[l].kind != SMLRT_DENSE) return false;
  return true;
}

int launch_dense_exact_tiled(const float* x, int64_t rows, const DevLayer& L, float* y, cudaStream_t s,
                             uint32_t* status) {
  if (rows <= 0) return SMLRT_OK;
  if (L.kind != SMLRT_DENSE) return fail(SMLRT_E_UNSUPPORTED, "layer order not supported by the exact path");
  dim3 grid((unsigned)((rows + PR - 1) / PR), (unsigned)((L.out + PJ - 1) / PJ));
  dense_pair_kernel<false><<<grid, PT, 0, s>>>(x, rows, L.in, L.out, L.w, L.b, L.act, y, status, nullptr, nullptr, 0,
                                                SMLRT_IDENTITY, one2());
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

int infer_cnn_dense(const smlrt_model_s& m, const float* x, int64_t rows, float* y, cudaStream_t s,
                    uint32_t* status) {
  if (!cnn_model(m)) return fail(SMLRT_E_UNSUPPORTED, "model is not conv2d(+maxpool) + dense");
  float *f, *t0, *t1;
  size_t per = 1;
  for (int l = 1; l < m.n_layers; ++l) per = std::max(per, (size_t)m.layers[l].out);
  SMLRT_CUDA(cudaMallocAsync(&f, per * rows * 4 * 3, s));
  t0 = f + per * rows;
  t1 = t0 + per * rows;
  int ow, nl;
  int rc = launch_front(m, x, nullptr, nullptr, SMLRT_F32, 0, rows, f, &ow, &nl, s);
  if (!rc) rc = (nl < m.n_layers) ? dense_tail(m, nl, f, rows, y, t0, t1, s, status)
                                  : fail(SMLRT_E_UNSUPPORTED, "CNN without a dense head");
  cudaFreeAsync(f, s);
  return rc;
}

// bf16 CNN region (precision "bf16"): the conv(+pool) front is the exact
// CUDA-core kernel (it is HBM-bound: its FP32 work fits under the window
// reads), writing its features as bf16 rows padded to the chain's K; the
// dense tail (512 -> 128 -> 2 on C4) is the generic tcgen05 layer chain
// (TMA-fed GEMMs, bias/act/bf16 fused), the f32 outputs go through the
// out-plan scatter or the checked commit's staging.  The exact path's dense
// tail was a third of the region on CUDA cores (FP32-bound); on the tensor
// core it is a few microseconds.
int launch_region_cnn_bf16(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs,
                           const int32_t* in_dt, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt,
                           int n_out, int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  if (m.chain_blob == nullptr || m.chain.empty() || m.chain_first < 1)
    return fail(SMLRT_E_UNSUPPORTED, "bf16 CNN: the dense tail has a layer wider than 4096");
  const int64_t rows = r1 - r0;
  if (rows <= 0) return SMLRT_OK;
  const int k0 = m.chain[0].k_pad, maxw = chain_max_width(m), G = m.out_features;
  const int64_t ch = std::min<int64_t>(rows, 1 << 16);
  const size_t act_bytes = (size_t)ch * maxw * 2;
  uint8_t* buf;
  SMLRT_CUDA(cudaMallocAsync(&buf, 2 * act_bytes + (size_t)ch * G * 4, s));
  auto* act0 = reinterpret_cast<__nv_bfloat16*>(buf);
  auto* act1 = reinterpret_cast<__nv_bfloat16*>(buf + act_bytes);
  auto* y = reinterpret_cast<float*>(buf + 2 * act_bytes);
  int rc = SMLRT_OK;
  for (int64_t r = r0; r < r1 && !rc; r += ch) {
    const int64_t n = std::min(ch, r1 - r);
    // K padding columns must read as zero: the front never writes them and
    // the chain's ping-pong reuses act0 at another pitch
    if (m.layers[m.chain_first - 1].out < k0) SMLRT_CUDA(cudaMemsetAsync(act0, 0, (size_t)n * k0 * 2, s));
    int ow = 0, nl = 0;
    rc = launch_front(m, nullptr, &in, in_ptrs[in.uarray], in_dt[in.uarray], r, r + n, nullptr, &ow, &nl, s, act0,
                      k0);
    if (rc) break;
    if (nl != m.chain_first) {
      rc = fail(SMLRT_E_UNSUPPORTED, "bf16 CNN: front and chain disagree on the first dense layer");
      break;
    }
    float* ydst = staged ? staged + (r - r0) * G : y;
    rc = chain_forward(m, act0, act1, n, ydst, status, s);
    if (!rc && !staged) rc = launch_scatter(out, ydst, SMLRT_F32, out_ptrs, out_dt, n_out, r, r + n, s, nullptr);
  }
  cudaFreeAsync(buf, s);
  return rc;
}

// Rows are processed in chunks of <= 16384 on the caller's stream: conv
// front, dense tail, scatter.  (Round 2 measured an overlapped variant --
// fronts on a low-priority stream, each chunk's tail on a high-priority one --
// at 0.354 / 0.402 / 0.640 ms for 2 / 4 / 8 chunks vs 0.324 ms in one chunk:
// a chunk's tail grid is too small to fill the SMs the fronts leave; removed.)
int launch_region_cnn(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs, const int32_t* in_dt,
                      int n_in, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt, int n_out,
                      int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  if (!in.uniform) return fail(SMLRT_E_UNSUPPORTED, "CNN region needs a single-array input map");
  if (m.precision == SMLRT_BF16)
    return launch_region_cnn_bf16(m, in, in_ptrs, in_dt, out, out_ptrs, out_dt, n_out, r0, r1, staged, s, status);
  const int64_t rows = r1 - r0;
  if (rows <= 0) return SMLRT_OK;
  const int64_t ch = std::min<int64_t>(16384, rows);
  size_t per = 1;  // widest activation after the conv front
  for (int l = 1; l < m.n_layers; ++l) per = std::max(per, (size_t)m.layers[l].out);
  float* buf;
  SMLRT_CUDA(cudaMallocAsync(&buf, (per * 3 + m.out_features) * ch * 4, s));
  float* f = buf;  // front output, two ping-pong activations, outputs
  float* t0 = f + per * ch;
  float* t1 = t0 + per * ch;
  float* yo = t1 + per * ch;
  int rc = SMLRT_OK;
  for (int64_t r = r0; r < r1 && !rc; r += ch) {
    const int64_t n = std::min(ch, r1 - r);
    int ow, nl;
    rc = launch_front(m, nullptr, &in, in_ptrs[in.uarray], in_dt[in.uarray], r, r + n, f, &ow, &nl, s);
    if (rc) break;
    float* ydst = staged ? staged + (r - r0) * m.out_features : yo;
    rc = dense_tail(m, nl, f, n, ydst, t0, t1, s, status);
    if (!rc && !staged) rc = launch_scatter(out, ydst, SMLRT_F32, out_ptrs, out_dt, n_out, r, r + n, s, nullptr);
  }
  cudaFreeAsync(buf, s);
  (void)n_in;
  return rc;
}

}  // namespace smlrt
