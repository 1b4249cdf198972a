// Persistent warp-specialised tcgen05 GEMM with TMA operand streaming, the
// building block of the wide-MLP path (C3 MiniBUDE 6-1024-512-256-1):
//
//   D[M x N] = A[M x K] * B[N x K]^T   (bf16 operands, fp32 accumulation in TMEM)
//
// warp 0: TMA producer (one thread) -- A box [128 rows x BK], B box [BN x BK]
//         into a STAGES-deep SMEM ring (SW128 for BK = 64, SW32 for BK = 16)
// warp 1: MMA issuer (one thread) -- BK/16 tcgen05.mma per stage into one of
//         two TMEM accumulators (2 x BN <= 512 columns)
// warps 2-5: epilogue (one TMEM lane quarter each, thread = row):
//   EPI_BF16: out = bf16(act(acc + bias)) row-major (next layer's A operand)
//   EPI_DOT : y = act3(sum_n act(acc + bias[n]) * w_next[n] + b_next), then the
//             region's out-plan scatter (fused final dense layer, N == BN)
// Rows beyond M read as zeros (TMA OOB fill) and are not stored.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "simt_common.cuh"
#include "tc_ptx.cuh"

namespace smlrt {
namespace {

using namespace ptx;

constexpr int GBM = 128;
constexpr int GTHREADS = 192;
enum { EPI_BF16 = 0, EPI_DOT = 1, EPI_F32 = 2, EPI_DOTG = 3 };
constexpr int DOTG_MAX = 4;  // EPI_DOTG: outputs of the fused last layer

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

template <int ACT>
__device__ __forceinline__ float act_g(float y) {
  if constexpr (ACT == SMLRT_RELU) {
    float r;
    asm("max.NaN.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(y));
    return r;
  } else if constexpr (ACT == SMLRT_TANH) {
    return tanhf(y);
  } else {
    return y;
  }
}

struct GemmArgs {
  int M, N, K;
  int act;                 // activation of this layer
  const float* bias;       // [N]
  // EPI_BF16
  __nv_bfloat16* out;      // [M][ldo]
  int64_t ldo;
  // EPI_F32: act(acc + bias) as f32 for columns n < n_valid, row stride ldo
  float* out_f32;
  int n_valid;
  // EPI_DOT
  const float* w_next;     // [N]
  float b_next;
  int act_next;
  int64_t r0;              // sweep row of A row 0
  float* staged;           // checked commit: staged[row - r_stage0]
  int64_t r_stage0;
  uint32_t* status;
  // EPI_DOTG (generic chain, last layer fused into the one before it):
  // y[m][o] = act_last(sum_n bf16(act(acc + bias[n])) * w_last[o][n] + b_last[o]),
  // f32 rows of g_out into out_f32 (row stride ldo)
  const __nv_bfloat16* w_last;  // [>= g_out][k_last] bf16 (the chain blob's layer)
  const float* b_last;
  int g_out, k_last, act_last;
};

struct OutPtrs {
  void* p[8];
  int32_t dt[8];
};

template <int BN, int BK, int STAGES>
struct GemmLay {
  static constexpr int A_BYTES = GBM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int OFF_BIAS = STAGES * STAGE;
  static constexpr int OFF_WN = OFF_BIAS + 4096 * 4;
  static constexpr int OFF_BAR = OFF_WN + 256 * 4;
  static constexpr int N_BAR = 2 * STAGES + 4;
  static constexpr int OFF_TMEM = OFF_BAR + N_BAR * 8;
  static constexpr int ALLOC = OFF_TMEM + 16 + 1024;
  static constexpr uint32_t SW = BK == 64 ? kSwizzle128 : kSwizzle32;
  static constexpr uint32_t SBO = BK == 64 ? 1024 : 256;
  static_assert(BK == 64 || BK == 16, "BK is 64 (SW128) or 16 (SW32)");
  static_assert(2 * BN <= 512 && BN % 16 == 0 && BN <= 256, "BN");
};

#ifndef SMLRT_GEMM_EPI_PACKED
#define SMLRT_GEMM_EPI_PACKED 1
#endif
// packed f32x2 helpers for the EPI_DOT epilogue (bias add, relu, dot with w_next)
__device__ __forceinline__ uint64_t gpk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t gadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t gfma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
template <int ACT>
__device__ __forceinline__ uint64_t gact2(uint64_t h) {
  if constexpr (ACT == SMLRT_RELU) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(h));
    return gpk2(act_g<ACT>(lo), act_g<ACT>(hi));
  } else {
    return h;
  }
}

template <int ACT, int BN, int EPI>
__device__ __forceinline__ void gemm_epilogue(uint32_t tbase, uint64_t* tfull, uint64_t* tempty, int n_my,
                                              int n_tiles_n, const GemmArgs& g, const float* bias_s,
                                              const float* wn_s, const DevPlan& Pout, const OutPtrs& dst,
                                              int q, int lane) {
  const int r = q * 32 + lane;
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  for (int i = 0; i < n_my; ++i) {
    const int t = blockIdx.x + i * gridDim.x;
    const int mb = t / n_tiles_n, nb = t % n_tiles_n;
    const int ab = i & 1;
    mbar_wait(tfull + ab, (i >> 1) & 1);
    tc_fence_after();
    const int64_t m = (int64_t)mb * GBM + r;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};  // packed partial sums (SMLRT_GEMM_EPI_PACKED)
    // 32 columns at a time; with BN a multiple of 64 each TMEM request
    // fetches 64 columns (half the wait points)
    auto consume = [&](const uint32_t* v, int c0) {
      const int n0 = nb * BN + c0;
      if constexpr (EPI == EPI_F32) {
        bool bad = false;
        if (m < g.M) {
          float* o = g.out_f32 + m * g.ldo;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int n = n0 + e;
            if (n < g.n_valid) {
              const float y = act_g<ACT>(__uint_as_float(v[e]) + bias_s[n]);
              bad |= (__float_as_uint(y) & 0x7f800000u) == 0x7f800000u;
              o[n] = y;
            }
          }
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) flag_nonfinite(g.status);
      } else if constexpr (EPI == EPI_BF16) {
        uint32_t p[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float lo = act_g<ACT>(__uint_as_float(v[2 * e]) + bias_s[n0 + 2 * e]);
          const float hi = act_g<ACT>(__uint_as_float(v[2 * e + 1]) + bias_s[n0 + 2 * e + 1]);
          p[e] = pack_bf16(lo, hi);
        }
        if (m < g.M) {
          uint4* o = reinterpret_cast<uint4*>(g.out + m * g.ldo + n0);
#pragma unroll
          for (int j = 0; j < 4; ++j) o[j] = make_uint4(p[4 * j], p[4 * j + 1], p[4 * j + 2], p[4 * j + 3]);
        }
      } else if constexpr (EPI == EPI_DOTG) {
        // the hidden activations rounded to bf16 (the chain's quantisation
        // point between layers), dotted with the last layer's bf16 weights
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int n = n0 + e;
          const float h = __bfloat162float(__float2bfloat16_rn(act_g<ACT>(__uint_as_float(v[e]) + bias_s[n])));
#pragma unroll
          for (int o = 0; o < DOTG_MAX; ++o)
            if (o < g.g_out) acc[o] = fmaf(h, __bfloat162float(g.w_last[(int64_t)o * g.k_last + n]), acc[o]);
        }
      } else {
#if SMLRT_GEMM_EPI_PACKED
        if constexpr (ACT != SMLRT_TANH) {
          // add.f32x2 + relu + fma.f32x2 per pair, bias / w_next as LDS.128
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 bb = *reinterpret_cast<const float4*>(bias_s + c0 + e);
            const float4 ww = *reinterpret_cast<const float4*>(wn_s + c0 + e);
            const uint64_t h0 = gact2<ACT>(gadd2(gpk2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])), gpk2(bb.x, bb.y)));
            const uint64_t h1 =
                gact2<ACT>(gadd2(gpk2(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3])), gpk2(bb.z, bb.w)));
            acc2[(e >> 1) & 3] = gfma2(h0, gpk2(ww.x, ww.y), acc2[(e >> 1) & 3]);
            acc2[((e >> 1) + 1) & 3] = gfma2(h1, gpk2(ww.z, ww.w), acc2[((e >> 1) + 1) & 3]);
          }
          return;
        }
#endif
#pragma unroll
        for (int e = 0; e < 32; ++e)
          acc[e & 7] = fmaf(act_g<ACT>(__uint_as_float(v[e]) + bias_s[c0 + e]), wn_s[c0 + e], acc[e & 7]);
      }
    };
    if constexpr (BN % 64 == 0 && EPI == EPI_BF16) {  // (EPI_DOT measured slower with x64: 226 vs 201 us per 1M rows)
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 64) {
        uint32_t v[64];
        tmem_ld64(tbase + lane_off + ab * BN + c0, v);
        tmem_wait_ld();
        if (c0 + 64 == BN) {
          tc_fence_before();
          mbar_arrive(tempty + ab);
        }
        consume(v, c0);
        consume(v + 32, c0 + 32);
      }
    } else {
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tbase + lane_off + ab * BN + c0, v);
        tmem_wait_ld();
        if (c0 + 32 == BN) {
          tc_fence_before();
          mbar_arrive(tempty + ab);
        }
        consume(v, c0);
      }
    }
    if constexpr (EPI == EPI_DOTG) {
      bool bad = false;
      if (m < g.M) {
        float* o = g.out_f32 + m * g.ldo;
#pragma unroll
        for (int k = 0; k < DOTG_MAX; ++k)
          if (k < g.g_out) {
            float y = acc[k] + g.b_last[k];
            if (g.act_last == SMLRT_RELU) y = act_g<SMLRT_RELU>(y);
            else if (g.act_last == SMLRT_TANH) y = tanhf(y);
            bad |= (__float_as_uint(y) & 0x7f800000u) == 0x7f800000u;
            o[k] = y;
          }
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) flag_nonfinite(g.status);
    }
    if constexpr (EPI == EPI_DOT) {
      for (int p = 0; p < 4; ++p) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc2[p]));
        acc[2 * p] += lo;
        acc[2 * p + 1] += hi;
      }
      float y = ((acc[0] + acc[4]) + (acc[1] + acc[5])) + ((acc[2] + acc[6]) + (acc[3] + acc[7])) + g.b_next;
      if (g.act_next == SMLRT_RELU) y = act_g<SMLRT_RELU>(y);
      else if (g.act_next == SMLRT_TANH) y = tanhf(y);
      bool bad = false;
      if (m < g.M) {
        const int64_t row = g.r0 + m;
        bad = (__float_as_uint(y) & 0x7f800000u) == 0x7f800000u;
        if (g.staged != nullptr) {
          g.staged[row - g.r_stage0] = y;
        } else {
          int64_t addr;
          int arr;
          if (Pout.uniform) {
            addr = Pout.col_off0 + row_offset_uniform(Pout, (uint32_t)row);
            arr = Pout.uarray;
          } else {
            uint32_t idx[SMLRT_MAX_SWEEP];
            unravel(Pout, (uint32_t)row, idx);
            addr = col_address(Pout, 0, idx);
            arr = __ldg(Pout.col_arr);
          }
          if (dst.dt[arr] == SMLRT_F32)
            reinterpret_cast<float*>(dst.p[arr])[addr] = y;
          else
            reinterpret_cast<double*>(dst.p[arr])[addr] = (double)y;
        }
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) flag_nonfinite(g.status);
    }
  }
}

template <int BN, int BK, int STAGES, int EPI>
__global__ void __launch_bounds__(GTHREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                   const __grid_constant__ GemmArgs g, const __grid_constant__ DevPlan Pout,
                   const __grid_constant__ OutPtrs dst) {
  using L = GemmLay<BN, BK, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;  // warp-uniform to the compiler
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* full = bar;
  uint64_t* empty = bar + STAGES;
  uint64_t* tfull = bar + 2 * STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);
  float* bias_s = reinterpret_cast<float*>(smem + L::OFF_BIAS);
  float* wn_s = reinterpret_cast<float*>(smem + L::OFF_WN);

  const int n_tiles_n = (g.N + BN - 1) / BN;
  const int n_tiles = ((g.M + GBM - 1) / GBM) * n_tiles_n;
  const int n_my = blockIdx.x < n_tiles ? (n_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const int ksteps = g.K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, 128);
    }
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  for (int i = threadIdx.x; i < g.N && i < 4096; i += GTHREADS) bias_s[i] = g.bias[i];
  if (EPI == EPI_DOT)
    for (int i = threadIdx.x; i < g.N && i < 256; i += GTHREADS) wn_s[i] = g.w_next[i];
  if (warp == 1) tmem_alloc(tmem_slot, 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512))));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0, ph = 0;
      for (int i = 0; i < n_my; ++i) {
        const int t = blockIdx.x + i * gridDim.x;
        const int mb = t / n_tiles_n, nb = t % n_tiles_n;
        for (int kb = 0; kb < ksteps; ++kb) {
          mbar_wait(empty + s, ph ^ 1);
          mbar_expect_tx(full + s, L::STAGE);
          const uint32_t sa = smem_u32(smem + s * L::STAGE);
          tma_load_2d(sa, &ta, full + s, kb * BK, mb * GBM);
          tma_load_2d(sa + L::A_BYTES, &tb, full + s, kb * BK, nb * BN);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(GBM, BN);
      const uint64_t d0 = smem_desc(smem_u32(smem), L::SBO, L::SW);
      int s = 0, ph = 0;
      for (int i = 0; i < n_my; ++i) {
        const int ab = i & 1;
        mbar_wait(tempty + ab, ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + ab * BN;
        for (int kb = 0; kb < ksteps; ++kb) {
          mbar_wait(full + s, ph);
          tc_fence_after();
          const uint64_t ad = d0 + ((s * L::STAGE) >> 4);
          const uint64_t bd = d0 + ((s * L::STAGE + L::A_BYTES) >> 4);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) mma_bf16(d, ad + k * 2, bd + k * 2, idesc, (kb | k) != 0);
          mma_commit(empty + s);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(tfull + ab);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    if (g.act == SMLRT_RELU)
      gemm_epilogue<SMLRT_RELU, BN, EPI>(tbase, tfull, tempty, n_my, n_tiles_n, g, bias_s, wn_s, Pout, dst, q, lane);
    else if (g.act == SMLRT_TANH)
      gemm_epilogue<SMLRT_TANH, BN, EPI>(tbase, tfull, tempty, n_my, n_tiles_n, g, bias_s, wn_s, Pout, dst, q, lane);
    else
      gemm_epilogue<SMLRT_IDENTITY, BN, EPI>(tbase, tfull, tempty, n_my, n_tiles_n, g, bias_s, wn_s, Pout, dst, q,
                                             lane);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512))));
  }
}

// ------------------------------------------------ fused layers 1 + 2 (C3)
// D2[128 x NH*256] = act1(X W1^T + b1) W2^T for a 128-row tile, the layer-1
// activations never leaving the SM: four producer warps gather the tile's rows
// through the in-plan and compute layer 1 on the CUDA cores (packed FFMA2,
// bf16-valued x and W1, fp32 sums) one 64-wide K chunk at a time, writing it
// in the SW128 K-major A layout straight into the A ring; the MMA thread
// consumes it against TMA-streamed W2 chunks.  Replaces the materialised
// [rows x H1] layer-1 output, which made layer 1 an HBM-write-bound kernel.
//
// warp 0: TMA (W2 [256 x 64] boxes)     warp 1: MMA issuer
// warps 2..: epilogue, 4 per 256-column half (thread = row)
// last 8 warps: layer-1 producer (thread = row; warps 0-3 / 4-7 of them take
//   the low / high 32 columns of each 64-wide chunk)
// warp 0 TMA, warp 1 MMA, warps 2 .. 2+4NH-1 epilogue (4 per N-half), then 4 producer warps
constexpr int L12_PW = 8;  // producer warps: 2 per SM sub-partition (latency hiding)
template <int NH>
constexpr int l12_threads() { return 32 * (2 + 4 * NH + L12_PW); }
#ifndef SMLRT_L12_SA
#define SMLRT_L12_SA 3
#endif
#ifndef SMLRT_L12_SB
#define SMLRT_L12_SB 4
#endif
constexpr int L12_SA = SMLRT_L12_SA, L12_SB = SMLRT_L12_SB;  // A ring (on-chip layer 1), B ring (TMA W2 boxes)
constexpr int L12_H1MAX = 1024;

template <int NH>
struct L12Lay {
  static constexpr int SA = L12_SA;
  static constexpr int A_BYTES = GBM * 64 * 2;
  static constexpr int B_BYTES = 256 * 64 * 2;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + L12_SA * A_BYTES;
  static constexpr int OFF_W1 = OFF_B + L12_SB * B_BYTES;  // per k pair: 8 float2 (7 weight slots, bias)
  static constexpr int OFF_B2 = OFF_W1 + L12_H1MAX / 2 * 64;
  static constexpr int OFF_BAR = OFF_B2 + NH * 256 * 4;
  enum { AFULL = 0, AEMPTY = L12_SA, BFULL = 2 * L12_SA, BEMPTY = BFULL + L12_SB, TFULL = BEMPTY + L12_SB,
         TEMPTY = TFULL + 1, NBAR = TEMPTY + NH };
  static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
  static constexpr int ALLOC = OFF_TMEM + 16 + 1024;
  static_assert(ALLOC <= 232448, "shared memory budget");
};

struct L12Args {
  int M, H1, F;
  int act1, act2;
  int64_t r0;               // sweep row of tile row 0
  const float* w1p;         // [H1/2][16] f32: slot f < 7 = (W1[2p][f], W1[2p+1][f]) (bf16-valued), slot 7 = (b1[2p], b1[2p+1])
  const float* b2;          // [NH*256]
  const void* src;          // in-plan's array
  int src_dt;
  __nv_bfloat16* out;       // [M][NH*256]
};

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2pk(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}

template <int ACT>
__device__ __forceinline__ uint32_t act_pack2(uint64_t v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  if constexpr (ACT == SMLRT_RELU) return pack_relu_bf16(lo, hi);
  else if constexpr (ACT == SMLRT_TANH) return pack_bf16(tanhf(lo), tanhf(hi));
  else return pack_bf16(lo, hi);
}

// Thread (rq, cq) of the 256 producer threads computes rows rq and rq + 64 of
// the tile for k pairs [8 cq, 8 cq + 8) of each 64-wide chunk: every
// broadcast weight load (LDS.128) serves two rows, halving the producer's
// share of the SMEM port the tensor core reads its operands through.
// Tile rows of a persistent CTA: tile i of this CTA starts at row
// (first + i * stride) * rows + off (a CTA pair: 256-row pair tiles, rank r
// owning rows [128 r, 128 r + 128)).
struct TileRows {
  int first, stride, rows, off;
  __device__ __forceinline__ int64_t row0(int i) const { return (int64_t)(first + i * stride) * rows + off; }
};
// waits of the TMA and epilogue roles: plain try_wait polling by default
// (SMLRT_W4_SLEEP=1: suspend-hinted try_wait)
#ifndef SMLRT_W4_SLEEP
#define SMLRT_W4_SLEEP 0
#endif
__device__ __forceinline__ void w4_wait(uint64_t* bar, uint32_t parity) {
#if SMLRT_W4_SLEEP
  mbar_wait_sleep(bar, parity);
#else
  mbar_wait(bar, parity);
#endif
}
// AFULL arrival: 0 = every thread on the local barrier, 1 = one elected lane
// per warp on the local barrier, 2 = one lane per warp on the pair leader's
// (rank 0) barrier through the cluster window
template <int ARR>
__device__ __forceinline__ void producer_arrive(uint64_t* bar) {
  if constexpr (ARR == 0) {
    mbar_arrive(bar);
  } else {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      if constexpr (ARR == 1)
        mbar_arrive(bar);
      else
        mbar_arrive_remote(mapa(bar, 0));
    }
  }
}

template <int ACT1, int F, class L, class Args, int ARR = 0>
__device__ __forceinline__ void l12_producer(uint8_t* smem, uint64_t* bar, int n_my, const Args& a,
                                             const DevPlan& Pin, int tid, TileRows tr) {
  const int KB = a.H1 / 64;
  const int rq = tid & 63, cq = tid >> 6;
  const uint32_t w1s = smem_u32(smem + L::OFF_W1);  // explicit ld.shared (a generic load stalls on long scoreboard)
  // the next tile's inputs are loaded one tile ahead (DRAM latency off the A ring's critical path)
  auto load_x = [&](int i, float (&x)[2][F]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t m = tr.row0(i) + rq + 64 * h;
      const int64_t ro = m < a.M ? row_offset_uniform(Pin, (uint32_t)(a.r0 + m)) : 0;
#pragma unroll
      for (int f = 0; f < F; ++f) {
        x[h][f] = 0.0f;
        if (m < a.M && f < a.F && i < n_my) {
          const int64_t addr = Pin.col_inl[f] + ro;
          x[h][f] = a.src_dt == SMLRT_F32 ? __ldg(reinterpret_cast<const float*>(a.src) + addr)
                                          : __double2float_rn(__ldg(reinterpret_cast<const double*>(a.src) + addr));
        }
      }
    }
  };
  float xn[2][F];
  load_x(0, xn);
  int s = 0, ph = 0;
  for (int i = 0; i < n_my; ++i) {
    uint64_t xd[2][F];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const float x = __bfloat162float(__float2bfloat16_rn(xn[h][f]));  // the tensor-core operand precision
        xd[h][f] = f2pk(x, x);
      }
    load_x(i + 1, xn);
    for (int kb = 0; kb < KB; ++kb) {
      if constexpr (ARR == 0)
        mbar_wait_sleep(bar + L::AEMPTY + s, ph ^ 1);
      else
        w4_wait(bar + L::AEMPTY + s, ph ^ 1);
      const uint32_t ab = smem_u32(smem + L::OFF_A) + s * L::A_BYTES;
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {  // 16-byte chunk j = k pairs 4j..4j+3
        const int j = 2 * cq + jj;
        uint32_t pk[2][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t w = w1s + (uint32_t)(kb * 32 + 4 * j + q) * 64;
          const float4 w0 = ld_shared_f4(w), w1 = ld_shared_f4(w + 16), w2 = ld_shared_f4(w + 32),
                       w3 = ld_shared_f4(w + 48);
          const float wv[14] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w, w2.x, w2.y, w2.z, w2.w, w3.x, w3.y};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint64_t acc = f2pk(w3.z, w3.w);  // (b1[k], b1[k+1])
#pragma unroll
            for (int f = 0; f < F; ++f) acc = ffma2(xd[h][f], f2pk(wv[2 * f], wv[2 * f + 1]), acc);
            pk[h][q] = act_pack2<ACT1>(acc);
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = rq + 64 * h;
          st_shared_v4(ab + r * 128 + ((j ^ (r & 7)) << 4), pk[h][0], pk[h][1], pk[h][2], pk[h][3]);  // SW128
        }
      }
      fence_async_smem();
      producer_arrive<ARR>(bar + L::AFULL + s);
      if (++s == L::SA) {
        s = 0;
        ph ^= 1;
      }
    }
  }
}

// thread = row of this warp's lane quarter; this warp group drains N-half h
// with the next 16-column TMEM load in flight while the current one is
// converted and stored
template <int ACT2, int NH>
__device__ __forceinline__ void l12_epilogue(uint8_t* smem, uint64_t* bar, uint32_t tbase, int n_my,
                                             const L12Args& a, int q, int h, int lane) {
  using L = L12Lay<NH>;
  const int r = q * 32 + lane;
  const uint32_t taddr = tbase + ((uint32_t)(q * 32) << 16) + h * 256;
  const uint32_t b2s = smem_u32(smem + L::OFF_B2) + h * 256 * 4;
  for (int i = 0; i < n_my; ++i) {
    const int64_t m = (int64_t)(blockIdx.x + i * gridDim.x) * GBM + r;
    mbar_wait_sleep(bar + L::TFULL, i & 1);
    tc_fence_after();
    uint4* o = reinterpret_cast<uint4*>(a.out + m * (NH * 256) + h * 256);
    // 64-column TMEM requests: 4 wait points per tile instead of 16 (the
    // accumulator is single-buffered, so the drain time stalls the MMA)
#pragma unroll 1
    for (int c4 = 0; c4 < 4; ++c4) {
      uint32_t v[64];
      tmem_ld64(taddr + c4 * 64, v);
      tmem_wait_ld();
      if (c4 == 3) {
        tc_fence_before();
        mbar_arrive(bar + L::TEMPTY + h);
      }
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int c = c4 * 4 + cc;
        uint32_t p[8];
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          const float4 bb = ld_shared_f4(b2s + (c * 16 + 4 * e4) * 4);
          const uint32_t* vv = v + cc * 16 + 4 * e4;
#if SMLRT_GEMM_EPI_PACKED
          if constexpr (ACT2 != SMLRT_TANH) {
            // add.f32x2 + one cvt(.relu).bf16x2 per pair: 2 instructions instead of 5
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const uint64_t hsum = gadd2(gpk2(__uint_as_float(vv[2 * u]), __uint_as_float(vv[2 * u + 1])),
                                          gpk2(u ? bb.z : bb.x, u ? bb.w : bb.y));
              float lo, hi;
              asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(hsum));
              p[2 * e4 + u] = ACT2 == SMLRT_RELU ? pack_relu_bf16(lo, hi) : pack_bf16(lo, hi);
            }
            continue;
          }
#endif
          p[2 * e4] = pack_bf16(act_g<ACT2>(__uint_as_float(vv[0]) + bb.x), act_g<ACT2>(__uint_as_float(vv[1]) + bb.y));
          p[2 * e4 + 1] =
              pack_bf16(act_g<ACT2>(__uint_as_float(vv[2]) + bb.z), act_g<ACT2>(__uint_as_float(vv[3]) + bb.w));
        }
        if (m < a.M) {
          o[2 * c] = make_uint4(p[0], p[1], p[2], p[3]);
          o[2 * c + 1] = make_uint4(p[4], p[5], p[6], p[7]);
        }
      }
    }
  }
}

template <int NH, int F>
__global__ void __launch_bounds__(l12_threads<NH>(), 1)
    l12_fused_kernel(const __grid_constant__ CUtensorMap tb, const __grid_constant__ L12Args a,
                     const __grid_constant__ DevPlan Pin) {
  using L = L12Lay<NH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;  // warp-uniform to the compiler
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);
  const int n_tiles = (a.M + GBM - 1) / GBM;
  const int n_my = (int)blockIdx.x < n_tiles ? (n_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const int KB = a.H1 / 64;

  if (threadIdx.x == 0) {
    for (int i = 0; i < L12_SA; ++i) {
      mbar_init(bar + L::AFULL + i, 32 * L12_PW);
      mbar_init(bar + L::AEMPTY + i, 1);
    }
    for (int i = 0; i < L12_SB; ++i) {
      mbar_init(bar + L::BFULL + i, 1);
      mbar_init(bar + L::BEMPTY + i, 1);
    }
    mbar_init(bar + L::TFULL, 1);
    for (int h = 0; h < NH; ++h) mbar_init(bar + L::TEMPTY + h, 128);  // one warp group per half
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  {
    const float4* g = reinterpret_cast<const float4*>(a.w1p);
    float4* w = reinterpret_cast<float4*>(smem + L::OFF_W1);
    for (int i = threadIdx.x; i < a.H1 / 2 * 4; i += l12_threads<NH>()) w[i] = g[i];
    float* b2s = reinterpret_cast<float*>(smem + L::OFF_B2);
    for (int i = threadIdx.x; i < NH * 256; i += l12_threads<NH>()) b2s[i] = a.b2[i];
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0, ph = 0;
      for (int i = 0; i < n_my; ++i)
        for (int kb = 0; kb < KB; ++kb)
          for (int h = 0; h < NH; ++h) {
            mbar_wait_sleep(bar + L::BEMPTY + s, ph ^ 1);
            mbar_expect_tx(bar + L::BFULL + s, L::B_BYTES);
            tma_load_2d(smem_u32(smem + L::OFF_B + s * L::B_BYTES), &tb, bar + L::BFULL + s, kb * 64, h * 256);
            if (++s == L12_SB) {
              s = 0;
              ph ^= 1;
            }
          }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(GBM, 256);
      const uint64_t a0 = smem_desc(smem_u32(smem + L::OFF_A), 1024, kSwizzle128);
      const uint64_t b0 = smem_desc(smem_u32(smem + L::OFF_B), 1024, kSwizzle128);
      int sa = 0, pa = 0, sb = 0, pb = 0;
      for (int i = 0; i < n_my; ++i) {
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(bar + L::AFULL + sa, pa);
          tc_fence_after();
          for (int h = 0; h < NH; ++h) {
            mbar_wait(bar + L::BFULL + sb, pb);
            if (kb == 0) mbar_wait(bar + L::TEMPTY + h, (i & 1) ^ 1);
            tc_fence_after();
            const uint64_t ad = a0 + ((sa * L::A_BYTES) >> 4);
            const uint64_t bd = b0 + ((sb * L::B_BYTES) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_bf16(tbase + h * 256, ad + k * 2, bd + k * 2, idesc, (kb | k) != 0);
            mma_commit(bar + L::BEMPTY + sb);
            if (++sb == L12_SB) {
              sb = 0;
              pb ^= 1;
            }
          }
          mma_commit(bar + L::AEMPTY + sa);
          if (++sa == L12_SA) {
            sa = 0;
            pa ^= 1;
          }
        }
        mma_commit(bar + L::TFULL);
      }
    }
    __syncwarp();
  } else if (warp < 2 + 4 * NH) {
    const int q = warp & 3, h = (warp - 2) >> 2;
    if (a.act2 == SMLRT_RELU)
      l12_epilogue<SMLRT_RELU, NH>(smem, bar, tbase, n_my, a, q, h, lane);
    else if (a.act2 == SMLRT_TANH)
      l12_epilogue<SMLRT_TANH, NH>(smem, bar, tbase, n_my, a, q, h, lane);
    else
      l12_epilogue<SMLRT_IDENTITY, NH>(smem, bar, tbase, n_my, a, q, h, lane);
  } else {
    const int t = threadIdx.x - 32 * (2 + 4 * NH);
    if (a.act1 == SMLRT_RELU)
      l12_producer<SMLRT_RELU, F, L12Lay<1>>(smem, bar, n_my, a, Pin, t, TileRows{(int)blockIdx.x, (int)gridDim.x, GBM, 0});
    else if (a.act1 == SMLRT_TANH)
      l12_producer<SMLRT_TANH, F, L12Lay<1>>(smem, bar, n_my, a, Pin, t, TileRows{(int)blockIdx.x, (int)gridDim.x, GBM, 0});
    else
      l12_producer<SMLRT_IDENTITY, F, L12Lay<1>>(smem, bar, n_my, a, Pin, t, TileRows{(int)blockIdx.x, (int)gridDim.x, GBM, 0});
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// ------------------------------------- fused layers 1-4 (C3, no HBM round trip)
// The whole 6-1024-512-256-1 forward pass of a 128-row tile on one SM:
//   layer 1  CUDA cores (producer warps, as in l12_fused_kernel) -> A1 ring
//   layer 2  tcgen05, N = 512 as two 256-column TMEM regions R1 | R2, K = H1
//            streamed in 64-wide A1 chunks against TMA W2 boxes [256 x 32]
//   layer 3  the epilogue drains R1 then R2 (+b2, act, bf16) into a 4-slot
//            ring of 64-wide K chunks (A3, SW128); tcgen05 multiplies them
//            against TMA W3 boxes into R1 (free once drained): N = H3 = 256
//   layer 4  the epilogue drains R1 (+b3, act, . w4, +b4, act) and scatters
//            through the out plan (or stages for a checked commit)
// so layer 2's [rows x 512] activations never leave the SM (the two-kernel
// chain wrote and re-read 1 KB per row of HBM).  Per tile the tensor pipe
// runs layer 2 (16,384 cycles at N = 256) then layer 3 (4,096); it waits
// only for the R1 drain between them and the layer-4 drain before the next
// tile's R1 writes.
//
// warp 0: TMA (W2 / W3 boxes)   warp 1: MMA issuer (warp-uniform, elect)
// warps 2-9: epilogue, 2 per TMEM lane quarter (column halves)
// warps 10-17: layer-1 producers (thread = two rows x 8 k pairs)
constexpr int W4_EPI = 8, W4_PW = 8;

constexpr int W4_THREADS = 32 * (2 + W4_EPI + W4_PW);
// NS = 2: CTA pair (cta_group::2).  Rank 0 issues M = 256 MMAs over both
// CTAs' A1 / A3 rings and TMEM; every W box is split along N, each CTA
// loading its 128-row half (half the L2 -> SMEM weight traffic per SM, and
// twice the ring depth in the same shared memory).
template <int NS>
struct W4Lay {
  static constexpr int SA = 3;                        // A1 ring (128 x 64 bf16, SW128)
  static constexpr int SB = 4 * NS;                   // B ring (this CTA's part of a [256 x 32] box, SW64)
  static constexpr int A_BYTES = GBM * 64 * 2;
  static constexpr int B_BYTES = 256 / NS * 32 * 2;
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + SA * A_BYTES;
  static constexpr int OFF_A3 = OFF_B + SB * B_BYTES;  // 4 slots, same layout as A1
  static constexpr int OFF_W1 = OFF_A3 + 4 * A_BYTES;
  static constexpr int OFF_B2 = OFF_W1 + L12_H1MAX / 2 * 64;
  static constexpr int OFF_B3 = OFF_B2 + 512 * 4;
  static constexpr int OFF_W4 = OFF_B3 + 256 * 4;
  static constexpr int OFF_RED = OFF_W4 + 256 * 4;     // 128 partial dot products
  static constexpr int OFF_BAR = OFF_RED + 128 * 4;
  enum { AFULL = 0, AEMPTY = SA, BFULL = 2 * SA, BEMPTY = BFULL + SB, TFULL = BEMPTY + SB, TFULL1, R1FREE, R2FREE,
         A3FULL, A3EMPTY = A3FULL + 4, L3FULL = A3EMPTY + 4, L3FREE, NBAR };
  static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
  static constexpr int ALLOC = OFF_TMEM + 16 + 1024;
  static_assert(ALLOC <= 232448, "shared memory budget");
};

struct W4Args {
  int M, H1, F;
  int act1, act2, act3, act4;
  int64_t r0;               // sweep row of tile row 0
  const float* w1p;         // layer-1 pair table (see l12_producer)
  const float* b2;          // [512]
  const float* b3;          // [256]
  const float* w4;          // [256]
  float b4;
  const void* src;          // in-plan's array
  int src_dt;
  float* staged;            // checked commit: staged[row - r_stage0]
  int64_t r_stage0;
  uint32_t* status;
};

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// one arrival per warp on the MMA issuer's barrier (the pair leader's)
template <int NS>
__device__ __forceinline__ void warp_arrive_mma(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    if constexpr (NS == 2)
      mbar_arrive_remote(mapa(bar, 0));
    else
      mbar_arrive(bar);
  }
}
// waits of the MMA issuer (also on barriers the peer CTA arrives on): a
// cta-scope acquire -- the cluster-scope form costs an L1 invalidate
// (CCTL.IVALL) per wait, and the MMA issuer reads no global memory
template <int NS>
__device__ __forceinline__ void mma_wait(uint64_t* bar, uint32_t parity) {
  mbar_wait(bar, parity);
}
template <int NS>
__device__ __forceinline__ void w4_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (NS == 2)
    mma2_ss_elect(d, a, b, idesc, acc);
  else
    mma_ss_elect(d, a, b, idesc, acc);
}
template <int NS>
__device__ __forceinline__ void w4_commit(uint64_t* bar) {
  if constexpr (NS == 2)
    mma2_commit_mc_elect(bar, 0x3);
  else
    mma_commit_elect(bar);
}
// this CTA's half of a W box; the bytes complete on the leader's BFULL
template <int NS>
__device__ __forceinline__ void w4_tma(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  if constexpr (NS == 2) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mapa(bar, 0))
        : "memory");
  } else {
    tma_load_2d(dst, map, bar, c0, c1);
  }
}

template <int ACT>
__device__ __forceinline__ uint64_t w4_act2(uint64_t h) {
  if constexpr (ACT == SMLRT_TANH) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(h));
    return gpk2(tanhf(lo), tanhf(hi));
  } else {
    return gact2<ACT>(h);
  }
}

// drain 64 accumulator columns of this thread's row (+bias, act, bf16) into
// one A3 chunk (SW128 K-major, row r)
template <int ACT>
__device__ __forceinline__ void w4_drain_chunk(uint32_t taddr, uint32_t bias_s, uint32_t dst, int r) {
  uint32_t v[64];
  tmem_ld64(taddr, v);
  tmem_wait_ld();
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // 16-byte chunk j = columns 8j .. 8j+7
    uint32_t p[4];
#pragma unroll
    for (int e2 = 0; e2 < 2; ++e2) {
      const float4 bb = ld_shared_f4(bias_s + (8 * j + 4 * e2) * 4);
      const uint32_t* vv = v + 8 * j + 4 * e2;
      if constexpr (ACT != SMLRT_TANH) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint64_t hsum = gadd2(gpk2(__uint_as_float(vv[2 * u]), __uint_as_float(vv[2 * u + 1])),
                                      gpk2(u ? bb.z : bb.x, u ? bb.w : bb.y));
          float lo, hi;
          asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(hsum));
          p[2 * e2 + u] = ACT == SMLRT_RELU ? pack_relu_bf16(lo, hi) : pack_bf16(lo, hi);
        }
      } else {
        p[2 * e2] = pack_bf16(tanhf(__uint_as_float(vv[0]) + bb.x), tanhf(__uint_as_float(vv[1]) + bb.y));
        p[2 * e2 + 1] = pack_bf16(tanhf(__uint_as_float(vv[2]) + bb.z), tanhf(__uint_as_float(vv[3]) + bb.w));
      }
    }
    st_shared_v4(dst + r * 128 + ((j ^ (r & 7)) << 4), p[0], p[1], p[2], p[3]);
  }
}

template <int ACT2, int ACT3, int NS>
__device__ __forceinline__ void w4_epilogue(uint8_t* smem, uint64_t* bar, uint32_t tbase, int n_my, const W4Args& a,
                                            const DevPlan& Pout, const OutPtrs& dst, int q, int half, int lane,
                                            TileRows tr) {
  using L = W4Lay<NS>;
  const int r = q * 32 + lane;
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  const uint32_t b2s = smem_u32(smem + L::OFF_B2), b3s = smem_u32(smem + L::OFF_B3), w4s = smem_u32(smem + L::OFF_W4);
  const uint32_t a3 = smem_u32(smem + L::OFF_A3);
  float* red = reinterpret_cast<float*>(smem + L::OFF_RED);
  for (int i = 0; i < n_my; ++i) {
    const int64_t m = tr.row0(i) + r;
    // layer-2 activations: R1 -> A3 chunks 0-3 (this half: 2 of them), then R2 -> chunks 4-7;
    // R1's last MMAs are issued before R2's (TFULL1), so its drain overlaps them
#pragma unroll 1
    for (int reg = 0; reg < 2; ++reg) {
      w4_wait(bar + (reg ? L::TFULL : L::TFULL1), i & 1);
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < 2; ++cc) {
        const int slot = half * 2 + cc;                 // chunk c = 4 reg + slot
        mbar_wait(bar + L::A3EMPTY + slot, reg ^ 1);    // slot use 2i + reg waits for use 2i + reg - 1
        w4_drain_chunk<ACT2>(tbase + lane_off + reg * 256 + slot * 64, b2s + (reg * 256 + slot * 64) * 4,
                             a3 + slot * L::A_BYTES, r);
        fence_async_smem();
        warp_arrive_mma<NS>(bar + L::A3FULL + slot);
      }
      tc_fence_before();
      warp_arrive_mma<NS>(bar + (reg ? L::R2FREE : L::R1FREE));
    }
    // layer 3 accumulator (R1) -> +b3, act, . w4 over this half's 128 columns
    w4_wait(bar + L::L3FULL, i & 1);
    tc_fence_after();
    uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll 1
    for (int c4 = 0; c4 < 2; ++c4) {
      const int c0 = half * 128 + c4 * 64;
      uint32_t v[64];
      tmem_ld64(tbase + lane_off + c0, v);
      tmem_wait_ld();
      if (c4 == 1) {
        tc_fence_before();
        warp_arrive_mma<NS>(bar + L::L3FREE);
      }
#pragma unroll
      for (int e = 0; e < 64; e += 4) {
        const float4 bb = ld_shared_f4(b3s + (c0 + e) * 4);
        const float4 ww = ld_shared_f4(w4s + (c0 + e) * 4);
        const uint64_t h0 = w4_act2<ACT3>(gadd2(gpk2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])), gpk2(bb.x, bb.y)));
        const uint64_t h1 = w4_act2<ACT3>(gadd2(gpk2(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3])), gpk2(bb.z, bb.w)));
        acc2[(e >> 1) & 3] = gfma2(h0, gpk2(ww.x, ww.y), acc2[(e >> 1) & 3]);
        acc2[((e >> 1) + 1) & 3] = gfma2(h1, gpk2(ww.z, ww.w), acc2[((e >> 1) + 1) & 3]);
      }
    }
    float part = 0.f;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc2[p]));
      part += lo + hi;
    }
    if (half == 1) red[r] = part;
    named_sync(1 + q, 64);
    if (half == 0) {
      float y = part + red[r] + a.b4;
      if (a.act4 == SMLRT_RELU) y = act_g<SMLRT_RELU>(y);
      else if (a.act4 == SMLRT_TANH) y = tanhf(y);
      bool bad = false;
      if (m < a.M) {
        const int64_t row = a.r0 + m;
        bad = (__float_as_uint(y) & 0x7f800000u) == 0x7f800000u;
        if (a.staged != nullptr) {
          a.staged[row - a.r_stage0] = y;
        } else {
          int64_t addr;
          int arr;
          if (Pout.uniform) {
            addr = Pout.col_off0 + row_offset_uniform(Pout, (uint32_t)row);
            arr = Pout.uarray;
          } else {
            uint32_t idx[SMLRT_MAX_SWEEP];
            unravel(Pout, (uint32_t)row, idx);
            addr = col_address(Pout, 0, idx);
            arr = __ldg(Pout.col_arr);
          }
          if (dst.dt[arr] == SMLRT_F32)
            reinterpret_cast<float*>(dst.p[arr])[addr] = y;
          else
            reinterpret_cast<double*>(dst.p[arr])[addr] = (double)y;
        }
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) flag_nonfinite(a.status);
    }
  }
}

template <int F, int NS>
__global__ void __launch_bounds__(W4_THREADS, 1)
    w4_fused_kernel(const __grid_constant__ CUtensorMap tw2, const __grid_constant__ CUtensorMap tw3,
                    const __grid_constant__ W4Args a, const __grid_constant__ DevPlan Pin,
                    const __grid_constant__ DevPlan Pout, const __grid_constant__ OutPtrs dst) {
  using L = W4Lay<NS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;  // warp-uniform to the compiler
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);
  const int rank = NS == 2 ? (int)cluster_rank() : 0;
  // tiles of GBM * NS rows; this CTA owns rows [rank * GBM, rank * GBM + GBM) of each
  const int n_tiles = (a.M + GBM * NS - 1) / (GBM * NS);
  const int unit = (int)blockIdx.x / NS, units = (int)gridDim.x / NS;
  const int n_my = unit < n_tiles ? (n_tiles - unit + units - 1) / units : 0;
  const TileRows tr{unit, units, GBM * NS, rank * GBM};
  const int KB = a.H1 / 64;

  if (threadIdx.x == 0) {
    for (int i = 0; i < L::SA; ++i) {
      mbar_init(bar + L::AFULL + i, W4_PW * NS);
      mbar_init(bar + L::AEMPTY + i, 1);
    }
    for (int i = 0; i < L::SB; ++i) {
      mbar_init(bar + L::BFULL + i, 1);
      mbar_init(bar + L::BEMPTY + i, 1);
    }
    mbar_init(bar + L::TFULL, 1);
    mbar_init(bar + L::TFULL1, 1);
    mbar_init(bar + L::R1FREE, W4_EPI * NS);
    mbar_init(bar + L::R2FREE, W4_EPI * NS);
    for (int i = 0; i < 4; ++i) {
      mbar_init(bar + L::A3FULL + i, 4 * NS);
      mbar_init(bar + L::A3EMPTY + i, 1);
    }
    mbar_init(bar + L::L3FULL, 1);
    mbar_init(bar + L::L3FREE, W4_EPI * NS);
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tw2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tw3)) : "memory");
  }
  {
    const float4* g = reinterpret_cast<const float4*>(a.w1p);
    float4* w = reinterpret_cast<float4*>(smem + L::OFF_W1);
    for (int i = threadIdx.x; i < a.H1 / 2 * 4; i += W4_THREADS) w[i] = g[i];
    float* b2s = reinterpret_cast<float*>(smem + L::OFF_B2);
    for (int i = threadIdx.x; i < 512; i += W4_THREADS) b2s[i] = a.b2[i];
    float* b3s = reinterpret_cast<float*>(smem + L::OFF_B3);
    float* w4s = reinterpret_cast<float*>(smem + L::OFF_W4);
    for (int i = threadIdx.x; i < 256; i += W4_THREADS) {
      b3s[i] = a.b3[i];
      w4s[i] = a.w4[i];
    }
  }
  if (warp == 1) {
    if constexpr (NS == 2)
      tmem_alloc2(tmem_slot, 512);
    else
      tmem_alloc(tmem_slot, 512);
  }
  tc_fence_before();
  if constexpr (NS == 2)
    cluster_sync();  // peer barriers initialised and TMEM allocated before any remote arrive / MMA
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0, ph = 0;
      auto load = [&](const CUtensorMap* map, int k0, int n0) {
        w4_wait(bar + L::BEMPTY + s, ph ^ 1);
        if (rank == 0) mbar_expect_tx(bar + L::BFULL + s, L::B_BYTES * NS);
        w4_tma<NS>(smem_u32(smem + L::OFF_B + s * L::B_BYTES), map, bar + L::BFULL + s, k0, n0);
        if (++s == L::SB) {
          s = 0;
          ph ^= 1;
        }
      };
      const int nh = rank * (256 / NS);  // this CTA's rows of each box
      for (int i = 0; i < n_my; ++i) {
        for (int kb = 0; kb < KB; ++kb)
          for (int hh = 0; hh < 2; ++hh) {
            const int h = kb == 0 ? 1 - hh : hh;  // the MMA issuer's region order
            for (int kh = 0; kh < 2; ++kh) load(&tw2, kb * 64 + kh * 32, h * 256 + nh);
          }
        for (int c = 0; c < 8; ++c)
          for (int kh = 0; kh < 2; ++kh) load(&tw3, c * 64 + kh * 32, nh);
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_bf16(GBM * NS, 256);
      const uint64_t a0 = smem_desc(smem_u32(smem + L::OFF_A), 1024, kSwizzle128);
      const uint64_t a30 = smem_desc(smem_u32(smem + L::OFF_A3), 1024, kSwizzle128);
      const uint64_t b0 = smem_desc(smem_u32(smem + L::OFF_B), 512, kSwizzle64);
      int sa = 0, pa = 0, sb = 0, pb = 0;
      for (int i = 0; i < n_my; ++i) {
        // ---- layer 2: R1 | R2 += A1 chunk x W2 boxes
        // the first chunk goes to R2 first (drained during the previous
        // tile's layer 3) while the layer-4 drain still reads R1; the last
        // chunk finishes R1 first so its drain overlaps R2's last MMAs
        for (int kb = 0; kb < KB; ++kb) {
          mma_wait<NS>(bar + L::AFULL + sa, pa);
          tc_fence_after();
          const uint64_t ad = a0 + ((sa * L::A_BYTES) >> 4);
#pragma unroll 1
          for (int hh = 0; hh < 2; ++hh) {
            const int h = kb == 0 ? 1 - hh : hh;
            if (kb == 0) {
              mma_wait<NS>(bar + (h ? L::R2FREE : L::L3FREE), (i & 1) ^ 1);
              tc_fence_after();
            }
#pragma unroll 1
            for (int kh = 0; kh < 2; ++kh) {
              mma_wait<NS>(bar + L::BFULL + sb, pb);
              tc_fence_after();
              const uint64_t bd = b0 + ((sb * L::B_BYTES) >> 4);
#pragma unroll
              for (int k = 0; k < 2; ++k)
                w4_mma<NS>(tbase + h * 256, ad + (kh * 2 + k) * 2, bd + k * 2, idesc, (kb | kh | k) != 0);
              w4_commit<NS>(bar + L::BEMPTY + sb);
              if (++sb == L::SB) {
                sb = 0;
                pb ^= 1;
              }
            }
            if (kb == KB - 1 && h == 0) w4_commit<NS>(bar + L::TFULL1);
          }
          w4_commit<NS>(bar + L::AEMPTY + sa);
          if (++sa == L::SA) {
            sa = 0;
            pa ^= 1;
          }
        }
        w4_commit<NS>(bar + L::TFULL);
        // ---- layer 3: R1 = A3 chunks x W3 boxes (R1 drained first)
        mma_wait<NS>(bar + L::R1FREE, i & 1);
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          const int slot = c & 3;
          mma_wait<NS>(bar + L::A3FULL + slot, c >> 2);
          tc_fence_after();
          const uint64_t ad = a30 + ((slot * L::A_BYTES) >> 4);
#pragma unroll 1
          for (int kh = 0; kh < 2; ++kh) {
            mma_wait<NS>(bar + L::BFULL + sb, pb);
            tc_fence_after();
            const uint64_t bd = b0 + ((sb * L::B_BYTES) >> 4);
#pragma unroll
            for (int k = 0; k < 2; ++k)
              w4_mma<NS>(tbase, ad + (kh * 2 + k) * 2, bd + k * 2, idesc, (c | kh | k) != 0);
            w4_commit<NS>(bar + L::BEMPTY + sb);
            if (++sb == L::SB) {
              sb = 0;
              pb ^= 1;
            }
          }
          w4_commit<NS>(bar + L::A3EMPTY + slot);
        }
        w4_commit<NS>(bar + L::L3FULL);
      }
    }
    __syncwarp();
  } else if (warp < 2 + W4_EPI) {
    const int q = warp & 3, half = (warp - 2) >> 2;
    if (a.act2 == SMLRT_RELU && a.act3 == SMLRT_RELU)
      w4_epilogue<SMLRT_RELU, SMLRT_RELU, NS>(smem, bar, tbase, n_my, a, Pout, dst, q, half, lane, tr);
    else if (a.act2 == SMLRT_TANH && a.act3 == SMLRT_TANH)
      w4_epilogue<SMLRT_TANH, SMLRT_TANH, NS>(smem, bar, tbase, n_my, a, Pout, dst, q, half, lane, tr);
    else
      w4_epilogue<SMLRT_IDENTITY, SMLRT_IDENTITY, NS>(smem, bar, tbase, n_my, a, Pout, dst, q, half, lane, tr);
  } else {
    const int t = threadIdx.x - 32 * (2 + W4_EPI);
    constexpr int ARR = NS == 2 ? 2 : 1;
    if (a.act1 == SMLRT_RELU)
      l12_producer<SMLRT_RELU, F, L, W4Args, ARR>(smem, bar, n_my, a, Pin, t, tr);
    else if (a.act1 == SMLRT_TANH)
      l12_producer<SMLRT_TANH, F, L, W4Args, ARR>(smem, bar, n_my, a, Pin, t, tr);
    else
      l12_producer<SMLRT_IDENTITY, F, L, W4Args, ARR>(smem, bar, n_my, a, Pin, t, tr);
  }
  tc_fence_before();
  if constexpr (NS == 2)
    cluster_sync();
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (NS == 2)
      tmem_dealloc2(tbase, 512);
    else
      tmem_dealloc(tbase, 512);
  }
}


// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// bf16 row-major [rows][cols] (row pitch ld elements), box [box_rows][bk]
int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows, int bk) {
  EncodeFn enc = encoder();
  if (!enc) return fail(SMLRT_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)bk, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   bk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : (bk == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SMLRT_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return SMLRT_OK;
}

int sm_count() {
  int d = 0, n = 148;
  cudaGetDevice(&d);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
  return n;
}

template <int BN, int BK, int STAGES, int EPI>
int gemm_launch(const void* A, int64_t lda, const void* B, int64_t ldb, const GemmArgs& g, const DevPlan& Pout,
                const OutPtrs& dst, cudaStream_t s) {
  using L = GemmLay<BN, BK, STAGES>;
  CUtensorMap ta, tb;
  if (int rc = make_map(&ta, A, g.M, g.K, lda, GBM, BK)) return rc;
  if (int rc = make_map(&tb, B, g.N, g.K, ldb, BN, BK)) return rc;
  static int configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured & (1 << dev))) {
    SMLRT_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, BK, STAGES, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    L::ALLOC));
    configured |= 1 << dev;
  }
  const int tiles = ((g.M + GBM - 1) / GBM) * ((g.N + BN - 1) / BN);
  const int grid = std::max(1, std::min(tiles, sm_count()));
  gemm_tc_kernel<BN, BK, STAGES, EPI><<<grid, GTHREADS, L::ALLOC, s>>>(ta, tb, g, Pout, dst);
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

// gather through the in-plan into bf16 [rows][16] (features >= F are zero)
__global__ void gather_bf16_kernel(const __grid_constant__ DevPlan P, const void* src, int dt, int F, int64_t r0,
                                   int64_t rows, __nv_bfloat16* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  const int64_t row = r0 + i;
  const int64_t ro = row_offset_uniform(P, (uint32_t)row);
  uint32_t p[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    float v[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int f = 2 * e + h;
      v[h] = 0.0f;
      if (f < F) {
        const int64_t a = __ldg(P.col_off + f) + ro;
        v[h] = dt == SMLRT_F32 ? __ldg(reinterpret_cast<const float*>(src) + a)
                               : __double2float_rn(__ldg(reinterpret_cast<const double*>(src) + a));
      }
    }
    p[e] = pack_bf16(v[0], v[1]);
  }
  uint4* o = reinterpret_cast<uint4*>(out + i * 16);
  o[0] = make_uint4(p[0], p[1], p[2], p[3]);
  o[1] = make_uint4(p[4], p[5], p[6], p[7]);
}

uint16_t bf16_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

}  // namespace

// --------------------------------------------------------- wide MLP models
// dense 4-layer models F(<=16) -> H1 (multiple of 256) -> H2 (multiple of 64,
// <=1024) -> H3 (<= 256, multiple of 32) -> 1
// SMLRT_WIDE_UNFUSED=1: materialise layer 1 (A/B measurements, parity tests of both paths)
bool l12_disabled() {
  static const int v = [] {
    const char* e = std::getenv("SMLRT_WIDE_UNFUSED");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

bool wide_shape(const smlrt_model_s& m) {
  if (m.n_layers != 4) return false;
  for (const auto& L : m.layers)
    if (L.kind != SMLRT_DENSE) return false;
  const int h1 = m.layers[0].out, h2 = m.layers[1].out, h3 = m.layers[2].out;
  return m.in_features <= 16 && h1 % 256 == 0 && h1 <= 4096 && h2 % 64 == 0 && h2 <= 1024 && h2 % 256 == 0 &&
         h3 % 32 == 0 && h3 <= 256 && m.layers[3].out == 1 && h1 % 64 == 0;
}

// layers 1+2 fused on chip (l12_fused_kernel): F <= 7, H1 <= 1024, H2 in {256, 512}
bool l12_shape(const smlrt_model_s& m) {
  const int h1 = m.layers[0].out, h2 = m.layers[1].out;
  return m.in_features <= 7 && h1 <= L12_H1MAX && h1 % 64 == 0 && (h2 == 256 || h2 == 512);
}

size_t wide_w1p_off(const smlrt_model_s& m) {  // byte offset of the f32 layer-1 pair table in tc_blob
  const int h1 = m.layers[0].out, h2 = m.layers[1].out, h3 = m.layers[2].out;
  const size_t bf = ((size_t)h1 * 16 + (size_t)h2 * h1 + (size_t)h3 * h2) * 2;
  return (bf + 255) & ~size_t(255);
}

int wide_pack(smlrt_model_s& m) {
  // bf16 weights: W1p [H1][16] (K padded), W2 [H2][H1], W3 [H3][H2]; then (l12
  // shapes) the f32 layer-1 pair table of l12_fused_kernel
  const int F = m.in_features, h1 = m.layers[0].out, h2 = m.layers[1].out, h3 = m.layers[2].out;
  std::vector<uint16_t> w((size_t)h1 * 16 + (size_t)h2 * h1 + (size_t)h3 * h2, 0);
  const float* p = m.host_params.data();
  const float* W1 = p;
  const float* W2 = W1 + (size_t)h1 * F + h1;
  const float* W3 = W2 + (size_t)h2 * h1 + h2;
  size_t o = 0;
  for (int n = 0; n < h1; ++n)
    for (int k = 0; k < 16; ++k) w[o++] = k < F ? bf16_bits(W1[(size_t)n * F + k]) : 0;
  for (size_t i = 0; i < (size_t)h2 * h1; ++i) w[o++] = bf16_bits(W2[i]);
  for (size_t i = 0; i < (size_t)h3 * h2; ++i) w[o++] = bf16_bits(W3[i]);
  const size_t off = wide_w1p_off(m);
  std::vector<float> pairs;
  if (l12_shape(m)) {
    const float* b1 = W1 + (size_t)h1 * F;
    auto bfv = [](float v) {  // value of the bf16 rounding of v
      uint32_t u = (uint32_t)bf16_bits(v) << 16;
      float r;
      std::memcpy(&r, &u, 4);
      return r;
    };
    pairs.assign((size_t)h1 / 2 * 16, 0.0f);
    for (int p = 0; p < h1 / 2; ++p) {
      for (int f = 0; f < F; ++f) {
        pairs[(size_t)p * 16 + 2 * f] = bfv(W1[(size_t)(2 * p) * F + f]);
        pairs[(size_t)p * 16 + 2 * f + 1] = bfv(W1[(size_t)(2 * p + 1) * F + f]);
      }
      pairs[(size_t)p * 16 + 14] = b1[2 * p];
      pairs[(size_t)p * 16 + 15] = b1[2 * p + 1];
    }
  }
  const size_t bytes = pairs.empty() ? w.size() * 2 : off + pairs.size() * 4;
  SMLRT_CUDA(cudaMalloc(&m.tc_blob, bytes));
  SMLRT_CUDA(cudaMemcpy(m.tc_blob, w.data(), w.size() * 2, cudaMemcpyHostToDevice));
  if (!pairs.empty())
    SMLRT_CUDA(cudaMemcpy(reinterpret_cast<uint8_t*>(m.tc_blob) + off, pairs.data(), pairs.size() * 4,
                          cudaMemcpyHostToDevice));
  m.tc_bytes = bytes;
  return SMLRT_OK;
}

template <int NH, int F>
int l12_launch(const CUtensorMap& tb, const L12Args& a, const DevPlan& in, cudaStream_t s) {
  using L = L12Lay<NH>;
  static int configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured & (1 << dev))) {
    SMLRT_CUDA(cudaFuncSetAttribute(l12_fused_kernel<NH, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::ALLOC));
    configured |= 1 << dev;
  }
  const int tiles = (a.M + GBM - 1) / GBM;
  const int grid = std::max(1, std::min(tiles, sm_count()));
  l12_fused_kernel<NH, F><<<grid, l12_threads<NH>(), L::ALLOC, s>>>(tb, a, in);
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

// the fully fused kernel: l12 shapes with H2 = 512, H3 = 256 and one
// activation for layers 2 and 3 (SMLRT_WIDE_W4=0 selects the two-kernel chain)
bool w4_shape(const smlrt_model_s& m) {
  static const int off = [] {
    const char* e = std::getenv("SMLRT_WIDE_W4");
    return e && std::atoi(e) == 0;
  }();
  return !off && l12_shape(m) && m.layers[1].out == 512 && m.layers[2].out == 256 &&
         m.layers[1].act == m.layers[2].act;
}

// CTA pairs (cta_group::2: half of every W box per SM, half the L2 -> SMEM
// weight traffic) by default; SMLRT_W4_PAIR=0 runs one CTA per 128-row tile.
// C3 step, power-capped: pair 75.2 ms at ~1.72 GHz, single 78.6 ms at
// ~1.61 GHz -- per clock they are even, the pair draws less power
bool w4_pair() {
  static const int v = [] {
    const char* e = std::getenv("SMLRT_W4_PAIR");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

template <int F, int NS>
int w4_launch(const CUtensorMap& tw2, const CUtensorMap& tw3, const W4Args& a, const DevPlan& in, const DevPlan& out,
              const OutPtrs& dst, cudaStream_t s) {
  using L = W4Lay<NS>;
  static int configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured & (1 << dev))) {
    SMLRT_CUDA(cudaFuncSetAttribute(w4_fused_kernel<F, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::ALLOC));
    configured |= 1 << dev;
  }
  const int tiles = (a.M + GBM * NS - 1) / (GBM * NS);
  const int grid = NS * std::max(1, std::min(tiles, sm_count() / NS));
  if constexpr (NS == 1) {
    w4_fused_kernel<F, 1><<<grid, W4_THREADS, L::ALLOC, s>>>(tw2, tw3, a, in, out, dst);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(W4_THREADS);
    cfg.dynamicSmemBytes = L::ALLOC;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SMLRT_CUDA(cudaLaunchKernelEx(&cfg, w4_fused_kernel<F, 2>, tw2, tw3, a, in, out, dst));
  }
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

int launch_region_wide(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs, const int32_t* in_dt,
                       const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt, int n_out, int64_t r0,
                       int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  if (!in.uniform) return fail(SMLRT_E_UNSUPPORTED, "wide path needs a single-array input map");
  if (w4_shape(m) && in.n_cols == m.in_features && m.in_features <= SMLRT_INLINE_COLS && !l12_disabled()) {
    const int h1 = m.layers[0].out;
    const __nv_bfloat16* W2 = reinterpret_cast<const __nv_bfloat16*>(m.tc_blob) + (size_t)h1 * 16;
    const __nv_bfloat16* W3 = W2 + (size_t)512 * h1;
    const bool pair = w4_pair();
    CUtensorMap tw2, tw3;
    if (int rc = make_map(&tw2, W2, 512, h1, h1, pair ? 128 : 256, 32)) return rc;
    if (int rc = make_map(&tw3, W3, 256, 512, 512, pair ? 128 : 256, 32)) return rc;
    OutPtrs dst{};
    for (int i = 0; i < n_out && i < 8; ++i) {
      dst.p[i] = out_ptrs[i];
      dst.dt[i] = out_dt[i];
    }
    W4Args a{};
    a.M = (int)(r1 - r0);
    a.H1 = h1;
    a.F = m.in_features;
    a.act1 = m.layers[0].act;
    a.act2 = m.layers[1].act;
    a.act3 = m.layers[2].act;
    a.act4 = m.layers[3].act;
    a.r0 = r0;
    a.w1p = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(m.tc_blob) + wide_w1p_off(m));
    a.b2 = m.layers[1].b;
    a.b3 = m.layers[2].b;
    a.w4 = m.layers[3].w;
    a.b4 = m.host_params.back();
    a.src = in_ptrs[in.uarray];
    a.src_dt = in_dt[in.uarray];
    a.staged = staged;
    a.r_stage0 = r0;
    a.status = status;
    if (pair)
      return m.in_features <= 6 ? w4_launch<6, 2>(tw2, tw3, a, in, out, dst, s)
                                : w4_launch<7, 2>(tw2, tw3, a, in, out, dst, s);
    return m.in_features <= 6 ? w4_launch<6, 1>(tw2, tw3, a, in, out, dst, s)
                              : w4_launch<7, 1>(tw2, tw3, a, in, out, dst, s);
  }
  const int F = m.in_features, h1 = m.layers[0].out, h2 = m.layers[1].out, h3 = m.layers[2].out;
  const __nv_bfloat16* W1p = reinterpret_cast<const __nv_bfloat16*>(m.tc_blob);
  const __nv_bfloat16* W2 = W1p + (size_t)h1 * 16;
  const __nv_bfloat16* W3 = W2 + (size_t)h2 * h1;
  const int64_t rows = r1 - r0;
  // rows per block: the layer-2 activations of a block round-trip HBM
  // ([rows x H2] bf16); SMLRT_WIDE_BLOCK overrides the default 2^22 (measured: 2^19 / 2^20 / 2^21 / 2^22 rows -> 94.4 / 93.0 / 92.2 / 91.1 ms per C3 step)
  static const int64_t block_rows = [] {
    const char* e = std::getenv("SMLRT_WIDE_BLOCK");
    const long long v = e ? std::atoll(e) : 0;
    return v > 0 ? (int64_t)v : (int64_t)(1 << 22);
  }();
  const int64_t ch = std::min<int64_t>(rows, block_rows);
  const bool fused12 = l12_shape(m) && in.n_cols == F && F <= SMLRT_INLINE_COLS && !l12_disabled();
  __nv_bfloat16* buf;
  SMLRT_CUDA(cudaMallocAsync(&buf, (size_t)ch * (fused12 ? h2 : 16 + h1 + h2) * 2, s));
  __nv_bfloat16* x16 = buf;
  __nv_bfloat16* a1 = x16 + ch * 16;
  __nv_bfloat16* a2 = fused12 ? buf : a1 + ch * h1;
  CUtensorMap tw2;
  if (fused12)
    if (int rc = make_map(&tw2, W2, h2, h1, h1, 256, 64)) {
      cudaFreeAsync(buf, s);
      return rc;
    }
  OutPtrs dst{};
  for (int i = 0; i < n_out && i < 8; ++i) {
    dst.p[i] = out_ptrs[i];
    dst.dt[i] = out_dt[i];
  }
  DevPlan none{};
  int rc = SMLRT_OK;
  for (int64_t r = r0; r < r1 && !rc; r += ch) {
    const int n = (int)std::min(ch, r1 - r);
    GemmArgs g{};
    g.M = n;
    g.status = status;
    if (fused12) {
      // layers 1 + 2 in one kernel, layer 1 produced on chip -> a2 [n x h2]
      L12Args la{};
      la.M = n;
      la.H1 = h1;
      la.F = F;
      la.act1 = m.layers[0].act;
      la.act2 = m.layers[1].act;
      la.r0 = r;
      la.w1p = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(m.tc_blob) + wide_w1p_off(m));
      la.b2 = m.layers[1].b;
      la.src = in_ptrs[in.uarray];
      la.src_dt = in_dt[in.uarray];
      la.out = a2;
      if (h2 == 512)
        rc = F <= 6 ? l12_launch<2, 6>(tw2, la, in, s) : l12_launch<2, 7>(tw2, la, in, s);
      else
        rc = F <= 6 ? l12_launch<1, 6>(tw2, la, in, s) : l12_launch<1, 7>(tw2, la, in, s);
      if (rc) break;
    } else {
      gather_bf16_kernel<<<(n + 255) / 256, 256, 0, s>>>(in, in_ptrs[in.uarray], in_dt[in.uarray], F, r, n, x16);
      count_launch();
      if (cudaGetLastError() != cudaSuccess) return fail(SMLRT_E_CUDA, "gather_bf16 launch failed");
      // layer 1: [n x 16] * W1p^T -> a1 [n x h1]
      g.N = h1;
      g.K = 16;
      g.act = m.layers[0].act;
      g.bias = m.layers[0].b;
      g.out = a1;
      g.ldo = h1;
      rc = gemm_launch<256, 16, 8, EPI_BF16>(x16, 16, W1p, 16, g, none, dst, s);
      if (rc) break;
      // layer 2: a1 * W2^T -> a2 [n x h2]
      g.N = h2;
      g.K = h1;
      g.act = m.layers[1].act;
      g.bias = m.layers[1].b;
      g.out = a2;
      g.ldo = h2;
      rc = gemm_launch<256, 64, 4, EPI_BF16>(a1, h1, W2, h1, g, none, dst, s);
      if (rc) break;
    }
    // layer 3 + fused layer 4 (dot) + scatter
    g.N = h3;
    g.K = h2;
    g.act = m.layers[2].act;
    g.bias = m.layers[2].b;
    g.w_next = m.layers[3].w;
    g.act_next = m.layers[3].act;
    g.b_next = m.host_params.back();
    g.r0 = r;
    g.staged = staged;
    g.r_stage0 = r0;
    if (h3 == 256)
      rc = gemm_launch<256, 64, 4, EPI_DOT>(a2, h2, W3, h2, g, out, dst, s);
    else if (h3 == 128)
      rc = gemm_launch<128, 64, 4, EPI_DOT>(a2, h2, W3, h2, g, out, dst, s);
    else
      rc = fail(SMLRT_E_UNSUPPORTED, "wide path: H3 must be 128 or 256");
  }
  cudaFreeAsync(buf, s);
  return rc;
}

// ------------------------------------------------ generic tcgen05 layer chain
// Any dense model at bf16 (models.py:40-64 has no shape restrictions; neither
// does this path): per block of rows, the in-plan gather writes bf16 rows
// padded to K0 (16, or a multiple of 64), every hidden layer is one
// persistent TMA/tcgen05 GEMM with bias + activation + bf16 fused in the
// epilogue (EPI_BF16, widths padded to multiples of 64 with zero weights, so
// padded activations are act(0) = 0), and the last layer writes f32 rows
// (EPI_F32) that the out-plan scatter (or the checked commit's staging)
// consumes.  The shape-specialised fused kernels (bonds, MiniBUDE) stay the
// fast path; this is the fallback that keeps every bf16 model runnable.
namespace {

int chain_k0(int f) { return f <= 16 ? 16 : (f + 63) / 64 * 64; }
int chain_pad(int n) { return (n + 63) / 64 * 64; }

// gather through any plan into bf16 [rows][k0] (columns >= n_cols are zero)
__global__ void __launch_bounds__(256) chain_gather_kernel(const __grid_constant__ DevPlan P,
                                                           const __grid_constant__ Ptrs src, int64_t r0,
                                                           int64_t rows, int k0, __nv_bfloat16* out) {
  const int64_t n = rows * k0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = e / k0;
    const int c = (int)(e - rr * k0);
    float v = 0.0f;
    if (c < P.n_cols) {
      const int a = P.uniform ? P.uarray : __ldg(P.col_arr + c);
      v = load_as_f32(src.p[a], src.dt[a], element_address(P, (uint32_t)(r0 + rr), c));
    }
    out[e] = __float2bfloat16_rn(v);
  }
}

template <int EPI>
int chain_gemm(const void* A, int64_t lda, const void* B, int k_pad, int n_pad, GemmArgs& g, const DevPlan& none,
               const OutPtrs& dst, cudaStream_t s) {
  g.K = k_pad;
  g.N = n_pad;
  const bool k16 = k_pad == 16;
  if (n_pad % 256 == 0)
    return k16 ? gemm_launch<256, 16, 8, EPI>(A, lda, B, k_pad, g, none, dst, s)
               : gemm_launch<256, 64, 4, EPI>(A, lda, B, k_pad, g, none, dst, s);
  if (n_pad % 128 == 0)
    return k16 ? gemm_launch<128, 16, 8, EPI>(A, lda, B, k_pad, g, none, dst, s)
               : gemm_launch<128, 64, 4, EPI>(A, lda, B, k_pad, g, none, dst, s);
  return k16 ? gemm_launch<64, 16, 8, EPI>(A, lda, B, k_pad, g, none, dst, s)
             : gemm_launch<64, 64, 4, EPI>(A, lda, B, k_pad, g, none, dst, s);
}

}  // namespace

// first layer of the chain: 0 for a dense model; for a conv2d(+maxpool2d)
// model the first dense layer after the front (the CNN bf16 path runs the
// front on CUDA cores and its dense tail as this chain); -1 if none fits
int chain_first_layer(const smlrt_model_s& m) {
  int l = 0;
  if (cnn_model(m)) l = (m.n_layers > 1 && m.layers[1].kind == SMLRT_MAXPOOL2D) ? 2 : 1;
  if (l >= m.n_layers) return -1;
  for (int k = l; k < m.n_layers; ++k)
    if (m.layers[k].kind != SMLRT_DENSE || m.layers[k].out > 4096) return -1;
  return l;
}

bool chain_ok(const smlrt_model_s& m) { return !cnn_model(m) && chain_first_layer(m) == 0; }

int chain_pack(smlrt_model_s& m) {
  const int first = chain_first_layer(m);
  if (first < 0) return SMLRT_OK;
  std::vector<uint8_t> blob;
  const float* p = m.host_params.data();
  for (int l = 0; l < first; ++l) {  // skip the front's parameters (conv W, b; pooling has none)
    const auto& L = m.layers[l];
    if (L.kind == SMLRT_CONV2D) p += (size_t)L.out_c * L.in_c * L.kernel * L.kernel + L.out_c;
  }
  int k = chain_k0(m.layers[first].in);
  m.chain.clear();
  m.chain_first = first;
  for (int l = first; l < m.n_layers; ++l) {
    const auto& L = m.layers[l];
    smlrt_model_s::ChainLayer c{};
    c.k_pad = k;
    c.n_pad = chain_pad(L.out);
    c.n = L.out;
    c.act = L.act;
    c.w_off = (blob.size() + 1023) & ~size_t(1023);
    c.b_off = (c.w_off + (size_t)c.n_pad * c.k_pad * 2 + 255) & ~size_t(255);
    blob.resize(c.b_off + (size_t)c.n_pad * 4, 0);
    auto* w = reinterpret_cast<uint16_t*>(blob.data() + c.w_off);
    for (int n = 0; n < L.out; ++n)
      for (int kk = 0; kk < L.in; ++kk) w[(size_t)n * c.k_pad + kk] = bf16_bits(p[(size_t)n * L.in + kk]);
    std::memcpy(blob.data() + c.b_off, p + (size_t)L.out * L.in, (size_t)L.out * 4);
    p += (size_t)L.out * L.in + L.out;
    m.chain.push_back(c);
    k = c.n_pad;
  }
  SMLRT_CUDA(cudaMalloc(&m.chain_blob, blob.size()));
  SMLRT_CUDA(cudaMemcpy(m.chain_blob, blob.data(), blob.size(), cudaMemcpyHostToDevice));
  return SMLRT_OK;
}

int chain_max_width(const smlrt_model_s& m) {
  int w = m.chain.empty() ? 0 : m.chain[0].k_pad;
  for (const auto& c : m.chain) w = std::max(w, c.n_pad);
  return w;
}

// SMLRT_CHAIN_FUSE_LAST=0: the last layer as its own GEMM (A/B switch)
bool chain_fuse_last() {
  static const int v = [] {
    const char* e = std::getenv("SMLRT_CHAIN_FUSE_LAST");
    return (e && std::atoi(e) == 0) ? 0 : 1;
  }();
  return v != 0;
}

// the chain's GEMMs over n rows whose bf16 layer-0 activations are in act0
// ([n][k_pad0]); act1 is a second [n][max_width] buffer; the last layer
// writes f32 [n][G] rows into y
int chain_forward(const smlrt_model_s& m, __nv_bfloat16* act0, __nv_bfloat16* act1, int64_t n, float* y,
                  uint32_t* status, cudaStream_t s) {
  const uint8_t* wb = reinterpret_cast<const uint8_t*>(m.chain_blob);
  const int G = m.out_features;
  DevPlan none{};
  OutPtrs dst{};
  __nv_bfloat16* cur = act0;
  __nv_bfloat16* nxt = act1;
  const int nl = (int)m.chain.size();
  // a last layer of <= 4 outputs rides in the previous layer's epilogue when
  // that layer is one N tile (no f32 round trip, one GEMM launch less)
  const bool fuse_last = chain_fuse_last() && nl >= 2 && m.chain[nl - 1].n <= DOTG_MAX &&
                         (m.chain[nl - 2].n_pad == 64 || m.chain[nl - 2].n_pad == 128 || m.chain[nl - 2].n_pad == 256);
  for (int l = 0; l < nl; ++l) {
    const auto& c = m.chain[l];
    if (fuse_last && l == nl - 2) {
      const auto& c2 = m.chain[nl - 1];
      GemmArgs g{};
      g.M = (int)n;
      g.act = c.act;
      g.bias = reinterpret_cast<const float*>(wb + c.b_off);
      g.status = status;
      g.out_f32 = y;
      g.ldo = G;
      g.w_last = reinterpret_cast<const __nv_bfloat16*>(wb + c2.w_off);
      g.b_last = reinterpret_cast<const float*>(wb + c2.b_off);
      g.g_out = c2.n;
      g.k_last = c2.k_pad;
      g.act_last = c2.act;
      return chain_gemm<EPI_DOTG>(cur, c.k_pad, wb + c.w_off, c.k_pad, c.n_pad, g, none, dst, s);
    }
    GemmArgs g{};
    g.M = (int)n;
    g.act = c.act;
    g.bias = reinterpret_cast<const float*>(wb + c.b_off);
    g.status = status;
    const void* W = wb + c.w_off;
    int rc;
    if (l + 1 < nl) {
      g.out = nxt;
      g.ldo = c.n_pad;
      rc = chain_gemm<EPI_BF16>(cur, c.k_pad, W, c.k_pad, c.n_pad, g, none, dst, s);
      std::swap(cur, nxt);
    } else {
      g.out_f32 = y;
      g.ldo = G;
      g.n_valid = G;
      rc = chain_gemm<EPI_F32>(cur, c.k_pad, W, c.k_pad, c.n_pad, g, none, dst, s);
    }
    if (rc) return rc;
  }
  return SMLRT_OK;
}

int launch_region_chain(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs, const int32_t* in_dt,
                        int n_in, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt, int n_out,
                        int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  if (m.chain_blob == nullptr || m.chain.empty() || m.chain_first != 0)
    return fail(SMLRT_E_UNSUPPORTED, "bf16 layer chain: model has non-dense or > 4096-wide layers");
  if (n_in > 8 || n_out > 8) return fail(SMLRT_E_UNSUPPORTED, "bf16 layer chain: more than 8 arrays per plan");
  Ptrs src{};
  for (int i = 0; i < n_in; ++i) {
    src.p[i] = in_ptrs[i];
    src.dt[i] = in_dt[i];
  }
  const int maxw = chain_max_width(m);
  const int G = m.out_features;
  // rows per block: two bf16 activation buffers + the f32 output stay within 256 MB
  const int64_t rows = r1 - r0;
  const int64_t per_row = (int64_t)maxw * 2 * 2 + (int64_t)G * 4;
  const int64_t ch = std::min<int64_t>(rows, std::max<int64_t>(GBM, ((256ll << 20) / per_row) / GBM * GBM));
  uint8_t* buf;
  SMLRT_CUDA(cudaMallocAsync(&buf, (size_t)ch * per_row, s));
  auto* act0 = reinterpret_cast<__nv_bfloat16*>(buf);
  auto* act1 = act0 + ch * maxw;
  auto* y = reinterpret_cast<float*>(act1 + ch * maxw);
  int rc = SMLRT_OK;
  for (int64_t r = r0; r < r1 && !rc; r += ch) {
    const int64_t n = std::min(ch, r1 - r);
    const int k0 = m.chain[0].k_pad;
    const int blocks = (int)std::min<int64_t>((n * k0 + 255) / 256, 148 * 16);
    chain_gather_kernel<<<blocks, 256, 0, s>>>(in, src, r, n, k0, act0);
    count_launch();
    if (cudaGetLastError() != cudaSuccess) {
      rc = fail(SMLRT_E_CUDA, "chain gather launch failed");
      break;
    }
    // f32 rows: straight into the checked commit's staging, else a scratch block for the scatter
    rc = chain_forward(m, act0, act1, n, staged != nullptr ? staged + (r - r0) * G : y, status, s);
    if (!rc && staged == nullptr)
      rc = launch_scatter(out, y, SMLRT_F32, out_ptrs, out_dt, n_out, r, r + n, s, nullptr);
  }
  cudaFreeAsync(buf, s);
  return rc;
}

// f32 3-D tensor map (the C4 frame windows): dims {d0 (contiguous), d1, d2},
// byte strides of dims 1 and 2, box {b0, b1, b2}; no swizzle, no L2 promotion
// (a window's partial 128-B lines are fetched as sectors, not whole lines)
int make_map_f32_3d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                    uint64_t s2, uint32_t b0, uint32_t b1, uint32_t b2, int promote) {
  EncodeFn enc = encoder();
  if (!enc) return fail(SMLRT_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  const CUtensorMapL2promotion pr = promote == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                  : promote == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                  : promote == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                   : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SMLRT_E_CUDA, "cuTensorMapEncodeTiled (3-D f32) failed: " + std::to_string((int)r));
  return SMLRT_OK;
}

}  // namespace smlrt
