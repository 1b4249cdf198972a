// fp32-exact halo-stencil region (C5 MiniWeather, 36 -> 8 -> 4): bitwise the
// reference's ordered multiply-then-add forward pass (models.py:188-224), fed
// by the same TMA row ring as the bf16 stencil kernel.
//
// The per-point kernel (exact_region.cuh, one point per thread) spends most
// of its issue slots outside the FP pipe: 36 gathered loads with their
// address arithmetic and ~120 uniform weight loads per point (0.233 ms, 0.62
// of the FP32 roofline).  Here (0.200 ms, 0.72):
//   * a CTA owns 128 sweep columns x a block of rows; thread 0 streams each
//     stage (4 planes x (4 + 2) rows x 132 columns) through TMA;
//   * a thread computes 2 adjacent columns x 2 rows = 4 points; each feature
//     is a scalar from an 8-B shared load, broadcast into a packed
//     multiply with a hidden-unit weight pair from the parameter bank
//     (FMUL2 R, R.F32, UR.F32x2): every weight pair is fetched once for the
//     thread's 4 points;
//   * per (point, hidden unit) the accumulation runs over the 36 features in
//     the functor's order with separate RN multiply and add (mul.rn.f32x2,
//     then fma.rn.f32x2(p, 1, acc) with an opaque one: RN(p + acc) exactly,
//     no contraction), + b1, act; layer 2 likewise over the 8 hidden units in
//     order -- the same operation sequence per output as the reference.
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "simt_common.cuh"
#include "stencil_common.cuh"

namespace smlrt {

int make_map_f32_3d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                    uint64_t s2, uint32_t b0, uint32_t b1, uint32_t b2, int promote);

namespace {

using namespace stencil;

constexpr int SX_TW = 128;                 // output columns per CTA (64 threads x 2)
constexpr int SX_BOX = 132;                // TMA box width (16-B aligned start, <= 2 columns left of the halo)
#ifndef SX_RPT_
#define SX_RPT_ 2
#endif
constexpr int SX_RPT = SX_RPT_;            // output rows per thread
constexpr int SX_BR = 2 * SX_RPT;          // output rows per stage (2 thread rows x RPT)
constexpr int SX_NS = 2;                   // ring stages
constexpr int SX_VROWS = SX_BR + 2;        // staged input rows per variable
constexpr int SX_VF = SX_VROWS * SX_BOX;   // floats per variable in a stage
constexpr int SX_STAGE = 4 * SX_VF;        // floats per stage
constexpr int SX_SMEM = 1024 + SX_NS * SX_STAGE * 4 + 64;
static_assert(SX_STAGE % 32 == 0, "stages stay 128-B aligned");

struct SxArgs {
  int32_t c0, r0v, p0v, al;
  int64_t nj, i_begin, i_end, rb;
  float* dst;
  int64_t ocol[4];
  int64_t o0, o1, r0;
  float* staged;
  uint32_t* status;
  int act1, act2;
  // weights as output-unit pairs, in use order: layer 1 [f][hidden pair],
  // layer 2 [hidden][output pair]; biases as pairs
  uint64_t w1[36][4];
  uint64_t b1[4];
  uint64_t w2[8][2];
  uint64_t b2[2];
  uint64_t one;  // (1, 1): opaque to ptxas, keeps mul and add separate
};

template <int ACT>
__device__ __forceinline__ float sx_act(float y) {
  if constexpr (ACT == SMLRT_RELU) return relu_exact(y);  // np.maximum(y, 0): NaN wins, -0 -> +0
  else if constexpr (ACT == SMLRT_TANH) return tanhf(y);
  else return y;
}

__device__ __forceinline__ uint64_t sx_mul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// RN(acc + p): fma(p, 1, acc) with the opaque one
__device__ __forceinline__ uint64_t sx_add2(uint64_t acc, uint64_t p, uint64_t one) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(p), "l"(one), "l"(acc));
  return r;
}
__device__ __forceinline__ uint64_t sx_pk(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void sx_upk(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

#ifndef SX_MINB
#define SX_MINB 4
#endif
template <int ACT1>
__global__ void __launch_bounds__(128, SX_MINB) stencil_exact_kernel(const __grid_constant__ CUtensorMap tm,
                                                            const __grid_constant__ SxArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  float* ring = reinterpret_cast<float*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + SX_NS * SX_STAGE);
  const int tid = threadIdx.x, cp = tid & 63, rh = tid >> 6;  // column pair, row half
  const int64_t jb = (int64_t)blockIdx.x * SX_TW;
  const int64_t i0 = a.i_begin + (int64_t)blockIdx.y * a.rb;
  const int64_t i1 = min(i0 + a.rb, a.i_end);
  const int nblk = (int)((i1 - i0 + SX_BR - 1) / SX_BR);
  auto issue = [&](int b) {
    const int st = b % SX_NS;
    sm_expect_tx(full + st, SX_STAGE * 4);
    sm_tma(smem_u32(ring + st * SX_STAGE), &tm, full + st, a.c0 + (int)jb, (int)(a.r0v + i0 + b * SX_BR), a.p0v);
  };
  if (tid == 0) {
    for (int k = 0; k < SX_NS; ++k) mbar_init(full + k, 1);
    mbar_fence_init();
    for (int b = 0; b < min(nblk, SX_NS); ++b) issue(b);
  }
  __syncthreads();
  const uint64_t one = a.one;
  const int64_t js0 = jb + 2 * cp;  // this thread's first column
  const bool v0 = js0 < a.nj, v1 = js0 + 1 < a.nj;
  const bool stg = a.staged != nullptr;
  bool bad = false;

  for (int b = 0; b < nblk; ++b) {
    const int st = b % SX_NS;
    sm_wait(full + st, (uint32_t)(b / SX_NS) & 1u);
    const float* sb = ring + st * SX_STAGE + a.al + 2 * cp + rh * SX_RPT * SX_BOX;
    // points (r, c): rows rh*RPT + r, columns 2cp + c; accumulators over hidden pairs
    uint64_t acc[SX_RPT][2][4];
#pragma unroll
    for (int r = 0; r < SX_RPT; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int hp = 0; hp < 4; ++hp) acc[r][c][hp] = 0ull;
#pragma unroll 1
    for (int v = 0; v < 4; ++v) {  // not unrolled: the weights stream per variable (registers)
      // rows r .. r + RPT + 1 of variable v, columns 2cp .. 2cp + 3 (relative to the halo)
      float xv[SX_RPT + 2][4];
#pragma unroll
      for (int k = 0; k < SX_RPT + 2; ++k) {
        const float* row = sb + v * SX_VF + k * SX_BOX;
        const float2 p = *reinterpret_cast<const float2*>(row);
        const float2 q = *reinterpret_cast<const float2*>(row + 2);
        xv[k][0] = p.x, xv[k][1] = p.y, xv[k][2] = q.x, xv[k][3] = q.y;
      }
#pragma unroll
      for (int di = 0; di < 3; ++di)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
          const int f = v * 9 + di * 3 + dj;
#pragma unroll
          for (int hp = 0; hp < 4; ++hp) {
            const uint64_t w = a.w1[f][hp];
#pragma unroll
            for (int r = 0; r < SX_RPT; ++r)
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                const float x = xv[r + di][c + dj];
                acc[r][c][hp] = sx_add2(acc[r][c][hp], sx_mul2(sx_pk(x, x), w), one);
              }
          }
        }
    }
    __syncthreads();  // every thread has read stage st
    if (tid == 0 && b + SX_NS < nblk) issue(b + SX_NS);
    // layer 1 bias + act, layer 2 in hidden order, + b2, act, store
#pragma unroll
    for (int r = 0; r < SX_RPT; ++r) {
      const int64_t i = i0 + (int64_t)b * SX_BR + rh * SX_RPT + r;
      if (i >= i1) break;
      float out[2][4];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint64_t y[2] = {0ull, 0ull};
#pragma unroll
        for (int hp = 0; hp < 4; ++hp) {
          float h0, h1;
          sx_upk(sx_add2(acc[r][c][hp], a.b1[hp], one), h0, h1);
          h0 = sx_act<ACT1>(h0);
          h1 = sx_act<ACT1>(h1);
#pragma unroll
          for (int op = 0; op < 2; ++op) y[op] = sx_add2(y[op], sx_mul2(sx_pk(h0, h0), a.w2[2 * hp][op]), one);
#pragma unroll
          for (int op = 0; op < 2; ++op) y[op] = sx_add2(y[op], sx_mul2(sx_pk(h1, h1), a.w2[2 * hp + 1][op]), one);
        }
#pragma unroll
        for (int op = 0; op < 2; ++op) {
          sx_upk(sx_add2(y[op], a.b2[op], one), out[c][2 * op], out[c][2 * op + 1]);
          out[c][2 * op] = activate(out[c][2 * op], a.act2);
          out[c][2 * op + 1] = activate(out[c][2 * op + 1], a.act2);
        }
      }
      if (stg) {
        float* sg = a.staged + (i * a.nj + js0 - a.r0) * 4;
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          if (v0) sg[o] = out[0][o];
          if (v1) sg[4 + o] = out[1][o];
        }
      } else {
        float* op = a.dst + i * a.o0 + js0 * a.o1;
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          if (v0) op[a.ocol[o]] = out[0][o];
          if (v1) op[a.o1 + a.ocol[o]] = out[1][o];
        }
      }
#pragma unroll
      for (int o = 0; o < 4; ++o) bad |= (v0 && nonfinite(out[0][o])) || (v1 && nonfinite(out[1][o]));
    }
  }
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) atomicOr(a.status, SMLRT_STATUS_NONFINITE);
}

template <int ACT1>
int launch_sx(const smlrt_model_s& m, const DevPlan& in, const void* src, const DevPlan& out, void* dst,
              int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  SxArgs a{};
  StencilGeom geo;
  if (!stencil_geom(in, SX_BOX - SX_TW - 2, &geo)) return SMLRT_E_UNSUPPORTED;
  const int64_t nj = (int64_t)in.sdiv[1].d, s0 = in.ustride[0], P = geo.plane;
  if (r0 % nj != 0 || (r1 % nj != 0 && r1 != in.n_rows)) return SMLRT_E_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(src) & 15) != 0) return SMLRT_E_UNSUPPORTED;
  CUtensorMap tm;
  if (make_map_f32_3d(&tm, src, (uint64_t)s0, (uint64_t)(P / s0), (uint64_t)(in.uarray_numel / P),
                      (uint64_t)s0 * 4, (uint64_t)P * 4, SX_BOX, SX_VROWS, 4, 0) != SMLRT_OK)
    return SMLRT_E_UNSUPPORTED;
  a.c0 = geo.c0;
  a.r0v = geo.r0v;
  a.p0v = geo.p0v;
  a.al = geo.al;
  a.nj = nj;
  a.i_begin = r0 / nj;
  a.i_end = (r1 + nj - 1) / nj;
  a.dst = static_cast<float*>(dst);
  for (int o = 0; o < 4; ++o) a.ocol[o] = out.col_inl[o];
  a.o0 = out.ustride[0];
  a.o1 = out.ustride[1];
  a.r0 = r0;
  a.staged = staged;
  a.status = status;
  a.act1 = m.layers[0].act;
  a.act2 = m.layers[1].act;
  const float* p = m.host_params.data();  // [W1 8x36][b1 8][W2 4x8][b2 4]
  auto pair = [](float lo, float hi) {
    uint64_t r;
    const float v[2] = {lo, hi};
    std::memcpy(&r, v, 8);
    return r;
  };
  for (int f = 0; f < 36; ++f)
    for (int hp = 0; hp < 4; ++hp) a.w1[f][hp] = pair(p[(2 * hp) * 36 + f], p[(2 * hp + 1) * 36 + f]);
  for (int hp = 0; hp < 4; ++hp) a.b1[hp] = pair(p[288 + 2 * hp], p[288 + 2 * hp + 1]);
  for (int h = 0; h < 8; ++h)
    for (int op = 0; op < 2; ++op) a.w2[h][op] = pair(p[296 + (2 * op) * 8 + h], p[296 + (2 * op + 1) * 8 + h]);
  for (int op = 0; op < 2; ++op) a.b2[op] = pair(p[328 + 2 * op], p[328 + 2 * op + 1]);
  a.one = pair(1.0f, 1.0f);
  static int slots = 0;
  if (!slots) {
    int dev = 0, sms = 148, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    SMLRT_CUDA(cudaFuncSetAttribute(stencil_exact_kernel<ACT1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SX_SMEM));
    SMLRT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stencil_exact_kernel<ACT1>, 128, SX_SMEM));
    slots = std::max(1, per_sm) * sms;
  }
  const int64_t rows = a.i_end - a.i_begin;
  const int64_t ncb = (nj + SX_TW - 1) / SX_TW;
  const int64_t ny = std::max<int64_t>(1, slots / ncb);
  int64_t rb = (rows + ny - 1) / ny;
  rb = std::max<int64_t>(SX_BR, (rb + SX_BR - 1) / SX_BR * SX_BR);
  a.rb = rb;
  dim3 grid((unsigned)ncb, (unsigned)((rows + rb - 1) / rb));
  stencil_exact_kernel<ACT1><<<grid, 128, SX_SMEM, s>>>(tm, a);
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

}  // namespace


// fp32-exact region through the stencil kernel, or SMLRT_E_UNSUPPORTED when
// the model / plans do not have its shape (36 -> 8 -> 4 dense, f32 arrays,
// the 4-variable 3x3 halo in-plan, a uniform out-plan over the same sweep)
int launch_region_stencil_exact(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs,
                                const int32_t* in_dt, const DevPlan& out, void* const* out_ptrs,
                                const int32_t* out_dt, int64_t r0, int64_t r1, float* staged, cudaStream_t s,
                                uint32_t* status) {
  if (m.n_layers != 2 || m.layers[0].kind != SMLRT_DENSE || m.layers[1].kind != SMLRT_DENSE) return SMLRT_E_UNSUPPORTED;
  if (m.layers[0].in != 36 || m.layers[0].out != 8 || m.layers[1].out != 4) return SMLRT_E_UNSUPPORTED;
  if (!in.uniform || !out.uniform || in.n_sweep != 2 || out.n_sweep != 2 || out.n_cols != 4) return SMLRT_E_UNSUPPORTED;
  if (in_dt[in.uarray] != SMLRT_F32 || out_dt[out.uarray] != SMLRT_F32) return SMLRT_E_UNSUPPORTED;
  if (out.sdiv[0].d != in.sdiv[0].d || out.sdiv[1].d != in.sdiv[1].d) return SMLRT_E_UNSUPPORTED;
  if (r1 <= r0) return SMLRT_OK;
  const void* src = in_ptrs[in.uarray];
  void* dst = out_ptrs[out.uarray];
  const int act = m.layers[0].act;
  if (act == SMLRT_RELU) return launch_sx<SMLRT_RELU>(m, in, src, out, dst, r0, r1, staged, s, status);
  if (act == SMLRT_TANH) return launch_sx<SMLRT_TANH>(m, in, src, out, dst, r0, r1, staged, s, status);
  return launch_sx<SMLRT_IDENTITY>(m, in, src, out, dst, r0, r1, staged, s, status);
}

}  // namespace smlrt
