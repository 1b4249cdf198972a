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
#include <cstring>
#include <vector>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace smlrt {
namespace {

using namespace ptx;

constexpr int GBM = 128;
constexpr int GTHREADS = 192;
enum { EPI_BF16 = 0, EPI_DOT = 1 };

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
  // EPI_DOT
  const float* w_next;     // [N]
  float b_next;
  int act_next;
  int64_t r0;              // sweep row of A row 0
  float* staged;           // checked commit: staged[row - r_stage0]
  int64_t r_stage0;
  uint32_t* status;
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
  static constexpr int OFF_WN = OFF_BIAS + 1024 * 4;
  static constexpr int OFF_BAR = OFF_WN + 256 * 4;
  static constexpr int N_BAR = 2 * STAGES + 4;
  static constexpr int OFF_TMEM = OFF_BAR + N_BAR * 8;
  static constexpr int ALLOC = OFF_TMEM + 16 + 1024;
  static constexpr uint32_t SW = BK == 64 ? kSwizzle128 : kSwizzle32;
  static constexpr uint32_t SBO = BK == 64 ? 1024 : 256;
  static_assert(BK == 64 || BK == 16, "BK is 64 (SW128) or 16 (SW32)");
  static_assert(2 * BN <= 512 && BN % 16 == 0 && BN <= 256, "BN");
};

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
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t v[32];
      tmem_ld32(tbase + lane_off + ab * BN + c0, v);
      tmem_wait_ld();
      if (c0 + 32 == BN) {
        tc_fence_before();
        mbar_arrive(tempty + ab);
      }
      const int n0 = nb * BN + c0;
      if constexpr (EPI == EPI_BF16) {
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
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e)
          acc[e & 7] = fmaf(act_g<ACT>(__uint_as_float(v[e]) + bias_s[c0 + e]), wn_s[c0 + e], acc[e & 7]);
      }
    }
    if constexpr (EPI == EPI_DOT) {
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
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(g.status, SMLRT_STATUS_NONFINITE);
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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
  for (int i = threadIdx.x; i < g.N && i < 1024; i += GTHREADS) bias_s[i] = g.bias[i];
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
                   bk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B,
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
bool wide_shape(const smlrt_model_s& m) {
  if (m.n_layers != 4) return false;
  for (const auto& L : m.layers)
    if (L.kind != SMLRT_DENSE) return false;
  const int h1 = m.layers[0].out, h2 = m.layers[1].out, h3 = m.layers[2].out;
  return m.in_features <= 16 && h1 % 256 == 0 && h1 <= 4096 && h2 % 64 == 0 && h2 <= 1024 && h2 % 256 == 0 &&
         h3 % 32 == 0 && h3 <= 256 && m.layers[3].out == 1 && h1 % 64 == 0;
}

int wide_pack(smlrt_model_s& m) {
  // bf16 weights: W1p [H1][16] (K padded), W2 [H2][H1], W3 [H3][H2]
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
  SMLRT_CUDA(cudaMalloc(&m.tc_blob, w.size() * 2));
  SMLRT_CUDA(cudaMemcpy(m.tc_blob, w.data(), w.size() * 2, cudaMemcpyHostToDevice));
  m.tc_bytes = w.size() * 2;
  return SMLRT_OK;
}

int launch_region_wide(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs, const int32_t* in_dt,
                       const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt, int n_out, int64_t r0,
                       int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  if (!in.uniform) return fail(SMLRT_E_UNSUPPORTED, "wide path needs a single-array input map");
  const int F = m.in_features, h1 = m.layers[0].out, h2 = m.layers[1].out, h3 = m.layers[2].out;
  const __nv_bfloat16* W1p = reinterpret_cast<const __nv_bfloat16*>(m.tc_blob);
  const __nv_bfloat16* W2 = W1p + (size_t)h1 * 16;
  const __nv_bfloat16* W3 = W2 + (size_t)h2 * h1;
  const int64_t rows = r1 - r0;
  const int64_t ch = std::min<int64_t>(rows, 1 << 20);
  __nv_bfloat16* buf;
  SMLRT_CUDA(cudaMallocAsync(&buf, (size_t)ch * (16 + h1 + h2) * 2, s));
  __nv_bfloat16* x16 = buf;
  __nv_bfloat16* a1 = x16 + ch * 16;
  __nv_bfloat16* a2 = a1 + ch * h1;
  OutPtrs dst{};
  for (int i = 0; i < n_out && i < 8; ++i) {
    dst.p[i] = out_ptrs[i];
    dst.dt[i] = out_dt[i];
  }
  DevPlan none{};
  int rc = SMLRT_OK;
  for (int64_t r = r0; r < r1 && !rc; r += ch) {
    const int n = (int)std::min(ch, r1 - r);
    gather_bf16_kernel<<<(n + 255) / 256, 256, 0, s>>>(in, in_ptrs[in.uarray], in_dt[in.uarray], F, r, n, x16);
    if (cudaGetLastError() != cudaSuccess) return fail(SMLRT_E_CUDA, "gather_bf16 launch failed");
    GemmArgs g{};
    g.M = n;
    g.status = status;
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

}  // namespace smlrt
