// Fused gather -> 3-layer MLP -> scatter on the 5th-generation tensor cores
// (tcgen05 / TMEM), bf16 operands, fp32 accumulation.  Models [F<=16] -> H1 ->
// H2 -> 1 (C2 "bonds": 16-256-128-1).
//
// One persistent CTA per SM, 17 warps, warp-specialised:
//   warps 12-15  loader   : gather 128 rows x F through the plan, f32->bf16,
//                           st.shared into a 4-stage SW32 ring (X)
//   warp  16     MMA      : one thread issues  L1: X[128x16] * W1^T -> TMEM[0,H1)
//                           and                L2: A2[128xH1] * W2^T -> TMEM[H1 + b*H2]
//                           (b = tile parity), commits to mbarriers
//   warps 4-11   epilogue1: TMEM L1 acc -> +b1, act -> bf16 -> A2[b] (SW128),
//                           two warpgroups split H1
//   warps 0-3    epilogue2: TMEM L2 acc[b] -> +b2, act, dot w3 (CUDA cores),
//                           +b3, act -> scatter through the out plan
// TMEM: H1 + 2*H2 <= 512 columns, so L2 of tile i overlaps epilogue-1 of
// tile i+1 and epilogue-2 of tile i-1.  Weights stay resident in SMEM.
//
// Reference semantics replaced: runtime.py:308-370 (gather_batch -> infer ->
// scatter_from) at the bf16 tolerance of SURVEY.md section 8(d).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace smlrt {
namespace {

using namespace ptx;

constexpr int BM = 128;
constexpr int KX = 16;
constexpr int XSTAGES = 4;
constexpr int WARP_EPI2 = 0, WARP_EPI1 = 4, WARP_LOAD = 12, WARP_MMA = 16;
constexpr int NTHREADS = 17 * 32;

template <int H1, int H2>
struct Lay {
  static_assert(H1 % 64 == 0 && H1 >= 64 && H1 <= 256, "H1: multiple of 64, <= 256");
  static_assert(H2 % 32 == 0 && H2 >= 32 && H2 <= 256, "H2: multiple of 32, <= 256");
  static_assert(H1 + 2 * H2 <= 512, "TMEM columns");
  static constexpr int KC = H1 / 64;          // layer-2 K chunks of 64
  static constexpr int W2_CHUNK = H2 * 128;   // [H2][64] bf16, SW128
  static constexpr int A2_CHUNK = BM * 128;   // [128][64] bf16, SW128
  static constexpr int A2_BUF = KC * A2_CHUNK;
  static constexpr int X_STAGE = BM * 32;     // [128][16] bf16, SW32
  static constexpr int OFF_W2 = 0;
  static constexpr int OFF_A2 = OFF_W2 + KC * W2_CHUNK;
  static constexpr int OFF_W1 = OFF_A2 + 2 * A2_BUF;
  static constexpr int OFF_X = OFF_W1 + H1 * 32;
  static constexpr int OFF_B1 = OFF_X + XSTAGES * X_STAGE;
  static constexpr int OFF_B2 = OFF_B1 + H1 * 4;
  static constexpr int OFF_W3 = OFF_B2 + H2 * 4;
  static constexpr int OFF_B3 = OFF_W3 + H2 * 4;
  static constexpr int OFF_BAR = OFF_B3 + 16;
  enum {
    B_XFULL = 0,
    B_XEMPTY = XSTAGES,
    B_L1FULL = 2 * XSTAGES,
    B_L1EMPTY,
    B_A2FULL,
    B_A2EMPTY = B_A2FULL + 2,
    B_L2FULL = B_A2EMPTY + 2,
    B_L2EMPTY = B_L2FULL + 2,
    N_BAR = B_L2EMPTY + 2
  };
  static constexpr int OFF_TMEM = OFF_BAR + N_BAR * 8;
  static constexpr int BYTES = OFF_TMEM + 16;
  static constexpr int ALLOC = BYTES + 1024;  // 1 KB alignment slack (SW128 atoms)
  // global blob produced by tc_pack_model: W2 img | W1 img | b1 | b2 | w3 | b3
  static constexpr int BLOB_W1 = KC * W2_CHUNK;
  static constexpr int BLOB_TAIL = BLOB_W1 + H1 * 32;
  static constexpr int TAIL = H1 * 4 + 2 * H2 * 4 + 16;
  static constexpr int BLOB = BLOB_TAIL + TAIL;
  static constexpr int T_L1 = 0, T_L2 = H1;  // TMEM column bases
};

struct TcArgs {
  const uint8_t* blob;
  const float* x_fast;  // dense f32 rows of 16 (fast gather path) or nullptr
  int64_t x_pitch;      // elements between rows on the fast path
  int F;
  int act1, act2, act3;
  int64_t r0, r1;
  int n_tiles;
  float* staged;
  uint32_t* status;
};

struct Ptrs8 {
  const void* p[8];
  int32_t dt[8];
};

__device__ __forceinline__ float act_f(float y, int act) {
  if (act == SMLRT_RELU) return relu_nan(y);
  if (act == SMLRT_TANH) return tanhf(y);
  return y;
}

template <int ACT>
__device__ __forceinline__ float act_t(float y) {
  if constexpr (ACT == SMLRT_RELU) return relu_nan(y);
  else if constexpr (ACT == SMLRT_TANH) return tanhf(y);
  else return y;
}

template <int ACT>
__device__ __forceinline__ uint32_t act_pack(float lo, float hi) {
  if constexpr (ACT == SMLRT_RELU) return pack_relu_bf16(lo, hi);
  else return pack_bf16(act_t<ACT>(lo), act_t<ACT>(hi));
}

// epilogue 1 for one 32-column slab: +b1, activation, bf16, SW128 st.shared
template <int ACT>
__device__ __forceinline__ void epi1_slab(const uint32_t (&v)[32], const float* b1, int c0, uint32_t a2,
                                          int a2_chunk, int r) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = c0 + 8 * j;
    const float4 bl = *reinterpret_cast<const float4*>(b1 + c);
    const float4 bh = *reinterpret_cast<const float4*>(b1 + c + 4);
    const float* x = reinterpret_cast<const float*>(v) + 8 * j;
    st_shared_v4(a2 + (c >> 6) * a2_chunk + sw128_offset(r, c & 63),
                 act_pack<ACT>(x[0] + bl.x, x[1] + bl.y), act_pack<ACT>(x[2] + bl.z, x[3] + bl.w),
                 act_pack<ACT>(x[4] + bh.x, x[5] + bh.y), act_pack<ACT>(x[6] + bh.z, x[7] + bh.w));
  }
}

// epilogue 2 for one 32-column slab: acc += act(v + b2) * w3
template <int ACT>
__device__ __forceinline__ void epi2_slab(const uint32_t (&v)[32], const float* b2, const float* w3, int c0,
                                          float (&acc)[4]) {
#pragma unroll
  for (int e = 0; e < 32; e += 4) {
    const float4 bb = *reinterpret_cast<const float4*>(b2 + c0 + e);
    const float4 ww = *reinterpret_cast<const float4*>(w3 + c0 + e);
    acc[0] = fmaf(act_t<ACT>(__uint_as_float(v[e]) + bb.x), ww.x, acc[0]);
    acc[1] = fmaf(act_t<ACT>(__uint_as_float(v[e + 1]) + bb.y), ww.y, acc[1]);
    acc[2] = fmaf(act_t<ACT>(__uint_as_float(v[e + 2]) + bb.z), ww.z, acc[2]);
    acc[3] = fmaf(act_t<ACT>(__uint_as_float(v[e + 3]) + bb.w), ww.w, acc[3]);
  }
}

__device__ __forceinline__ float ld_elem(const void* base, int dt, int64_t i) {
  return dt == SMLRT_F32 ? __ldg(reinterpret_cast<const float*>(base) + i)
                         : __double2float_rn(__ldg(reinterpret_cast<const double*>(base) + i));
}

template <int H1, int H2>
__global__ void __launch_bounds__(NTHREADS, 1)
    mlp3_tc_kernel(const __grid_constant__ TcArgs a, const __grid_constant__ DevPlan Pin,
                   const __grid_constant__ Ptrs8 src, const __grid_constant__ DevPlan Pout,
                   const __grid_constant__ Ptrs8 dst) {
  using L = Lay<H1, H2>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  // ---------------------------------------------------------------- setup
  if (threadIdx.x == 0) {
    for (int s = 0; s < XSTAGES; ++s) {
      mbar_init(bar + L::B_XFULL + s, 128);
      mbar_init(bar + L::B_XEMPTY + s, 1);
    }
    mbar_init(bar + L::B_L1FULL, 1);
    mbar_init(bar + L::B_L1EMPTY, 256);
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar + L::B_A2FULL + b, 256);
      mbar_init(bar + L::B_A2EMPTY + b, 1);
      mbar_init(bar + L::B_L2FULL + b, 1);
      mbar_init(bar + L::B_L2EMPTY + b, 128);
    }
    mbar_fence_init();
  }
  if (warp == WARP_MMA) tmem_alloc(tmem_slot, 512);
  {  // resident weights: blob -> smem (16-byte vectors)
    const int4* g = reinterpret_cast<const int4*>(a.blob);
    for (int i = threadIdx.x; i < L::BLOB_W1 / 16; i += NTHREADS)
      reinterpret_cast<int4*>(smem + L::OFF_W2)[i] = g[i];
    for (int i = threadIdx.x; i < H1 * 32 / 16; i += NTHREADS)
      reinterpret_cast<int4*>(smem + L::OFF_W1)[i] = g[L::BLOB_W1 / 16 + i];
    for (int i = threadIdx.x; i < L::TAIL / 16; i += NTHREADS)
      reinterpret_cast<int4*>(smem + L::OFF_B1)[i] = g[L::BLOB_TAIL / 16 + i];
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int n_my = (a.n_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;

  if (warp >= WARP_LOAD && warp < WARP_MMA) {
    // ============================================================ loader
    const int t = threadIdx.x - WARP_LOAD * 32;  // tile row
    float cur[16], nxt[16];
    auto load_row = [&](int it, float(&v)[16]) {
      const int64_t tile = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
      const int64_t row = a.r0 + tile * BM + t;
#pragma unroll
      for (int f = 0; f < 16; ++f) v[f] = 0.0f;
      if (row >= a.r1) return;
      if (a.x_fast != nullptr) {
        const float4* p = reinterpret_cast<const float4*>(a.x_fast + row * a.x_pitch);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float4 u = __ldg(p + q);
          v[4 * q] = u.x;
          v[4 * q + 1] = u.y;
          v[4 * q + 2] = u.z;
          v[4 * q + 3] = u.w;
        }
      } else if (Pin.uniform) {
        const int64_t ro = row_offset_uniform(Pin, (uint32_t)row);
        const void* base = src.p[Pin.uarray];
        const int dt = src.dt[Pin.uarray];
#pragma unroll
        for (int f = 0; f < 16; ++f)
          if (f < a.F) v[f] = ld_elem(base, dt, __ldg(Pin.col_off + f) + ro);
      } else {
        uint32_t idx[SMLRT_MAX_SWEEP];
        unravel(Pin, (uint32_t)row, idx);
#pragma unroll
        for (int f = 0; f < 16; ++f)
          if (f < a.F) {
            const int arr = __ldg(Pin.col_arr + f);
            v[f] = ld_elem(src.p[arr], src.dt[arr], col_address(Pin, f, idx));
          }
      }
    };
    if (n_my > 0) load_row(0, cur);
    for (int it = 0; it < n_my; ++it) {
      if (it + 1 < n_my) load_row(it + 1, nxt);
      const int s = it % XSTAGES;
      mbar_wait(bar + L::B_XEMPTY + s, ((it / XSTAGES) & 1) ^ 1);
      const uint32_t xs = smem_u32(smem + L::OFF_X + s * L::X_STAGE);
      st_shared_v4(xs + sw32_offset(t, 0), pack_bf16(cur[0], cur[1]), pack_bf16(cur[2], cur[3]),
                   pack_bf16(cur[4], cur[5]), pack_bf16(cur[6], cur[7]));
      st_shared_v4(xs + sw32_offset(t, 8), pack_bf16(cur[8], cur[9]), pack_bf16(cur[10], cur[11]),
                   pack_bf16(cur[12], cur[13]), pack_bf16(cur[14], cur[15]));
      fence_async_smem();
      mbar_arrive(bar + L::B_XFULL + s);
#pragma unroll
      for (int f = 0; f < 16; ++f) cur[f] = nxt[f];
    }
  } else if (warp == WARP_MMA) {
    // ========================================================= MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc1 = idesc_bf16(BM, H1);
      constexpr uint32_t idesc2 = idesc_bf16(BM, H2);
      const uint32_t w1 = smem_u32(smem + L::OFF_W1);
      const uint32_t w2 = smem_u32(smem + L::OFF_W2);
      const uint32_t x0 = smem_u32(smem + L::OFF_X);
      const uint32_t a20 = smem_u32(smem + L::OFF_A2);
      auto issue_l2 = [&](int j) {
        const int b = j & 1;
        mbar_wait(bar + L::B_A2FULL + b, (j >> 1) & 1);
        mbar_wait(bar + L::B_L2EMPTY + b, ((j >> 1) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kc = 0; kc < L::KC; ++kc)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = smem_desc(a20 + b * L::A2_BUF + kc * L::A2_CHUNK + k * 32, 1024, kSwizzle128);
            const uint64_t bd = smem_desc(w2 + kc * L::W2_CHUNK + k * 32, 1024, kSwizzle128);
            mma_bf16(tbase + L::T_L2 + b * H2, ad, bd, idesc2, (kc | k) != 0);
          }
        mma_commit(bar + L::B_A2EMPTY + b);
        mma_commit(bar + L::B_L2FULL + b);
      };
      const uint64_t w1d = smem_desc(w1, 256, kSwizzle32);
      for (int it = 0; it < n_my; ++it) {
        const int s = it % XSTAGES;
        mbar_wait(bar + L::B_XFULL + s, (it / XSTAGES) & 1);
        mbar_wait(bar + L::B_L1EMPTY, (it & 1) ^ 1);
        tc_fence_after();
        mma_bf16(tbase + L::T_L1, smem_desc(x0 + s * L::X_STAGE, 256, kSwizzle32), w1d, idesc1, 0);
        mma_commit(bar + L::B_XEMPTY + s);
        mma_commit(bar + L::B_L1FULL);
        if (it > 0) issue_l2(it - 1);
      }
      if (n_my > 0) issue_l2(n_my - 1);
    }
    __syncwarp();
  } else if (warp >= WARP_EPI1) {
    // ======================================================== epilogue 1
    const int half = (warp - WARP_EPI1) >> 2;
    const int q = warp & 3;
    const int r = q * 32 + lane;
    constexpr int HC = H1 / 2;
    const float* b1 = reinterpret_cast<const float*>(smem + L::OFF_B1);
    const uint32_t lane_addr = tbase + ((uint32_t)(q * 32) << 16);
    for (int it = 0; it < n_my; ++it) {
      const int b = it & 1;
      mbar_wait(bar + L::B_L1FULL, it & 1);
      mbar_wait(bar + L::B_A2EMPTY + b, ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t a2 = smem_u32(smem + L::OFF_A2 + b * L::A2_BUF);
#pragma unroll 1
      for (int cc = 0; cc < HC / 32; ++cc) {
        const int c0 = half * HC + cc * 32;
        uint32_t v[32];
        tmem_ld32(lane_addr + L::T_L1 + c0, v);
        tmem_wait_ld();
        if (cc == HC / 32 - 1) {
          tc_fence_before();
          mbar_arrive(bar + L::B_L1EMPTY);
        }
        if (a.act1 == SMLRT_RELU)
          epi1_slab<SMLRT_RELU>(v, b1, c0, a2, L::A2_CHUNK, r);
        else if (a.act1 == SMLRT_TANH)
          epi1_slab<SMLRT_TANH>(v, b1, c0, a2, L::A2_CHUNK, r);
        else
          epi1_slab<SMLRT_IDENTITY>(v, b1, c0, a2, L::A2_CHUNK, r);
      }
      fence_async_smem();
      mbar_arrive(bar + L::B_A2FULL + b);
    }
  } else {
    // ======================================================== epilogue 2
    const int q = warp;  // warps 0-3
    const int r = q * 32 + lane;
    const float* b2 = reinterpret_cast<const float*>(smem + L::OFF_B2);
    const float* w3 = reinterpret_cast<const float*>(smem + L::OFF_W3);
    const float b3 = *reinterpret_cast<const float*>(smem + L::OFF_B3);
    const uint32_t lane_addr = tbase + ((uint32_t)(q * 32) << 16);
    for (int it = 0; it < n_my; ++it) {
      const int b = it & 1;
      mbar_wait(bar + L::B_L2FULL + b, (it >> 1) & 1);
      tc_fence_after();
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
      for (int cc = 0; cc < H2 / 32; ++cc) {
        uint32_t v[32];
        tmem_ld32(lane_addr + L::T_L2 + b * H2 + cc * 32, v);
        tmem_wait_ld();
        if (a.act2 == SMLRT_RELU)
          epi2_slab<SMLRT_RELU>(v, b2, w3, cc * 32, acc);
        else if (a.act2 == SMLRT_TANH)
          epi2_slab<SMLRT_TANH>(v, b2, w3, cc * 32, acc);
        else
          epi2_slab<SMLRT_IDENTITY>(v, b2, w3, cc * 32, acc);
      }
      tc_fence_before();
      mbar_arrive(bar + L::B_L2EMPTY + b);
      const float y = act_f((acc[0] + acc[1]) + (acc[2] + acc[3]) + b3, a.act3);
      const int64_t tile = (int64_t)blockIdx.x + (int64_t)it * gridDim.x;
      const int64_t row = a.r0 + tile * BM + r;
      bool bad = false;
      if (row < a.r1) {
        bad = (__float_as_uint(y) & 0x7f800000u) == 0x7f800000u;
        if (a.staged != nullptr) {
          a.staged[row - a.r0] = y;
        } else {
          int64_t addr;
          int arr;
          if (Pout.uniform) {
            addr = __ldg(Pout.col_off) + row_offset_uniform(Pout, (uint32_t)row);
            arr = Pout.uarray;
          } else {
            uint32_t idx[SMLRT_MAX_SWEEP];
            unravel(Pout, (uint32_t)row, idx);
            addr = col_address(Pout, 0, idx);
            arr = __ldg(Pout.col_arr);
          }
          void* base = const_cast<void*>(dst.p[arr]);
          if (dst.dt[arr] == SMLRT_F32)
            reinterpret_cast<float*>(base)[addr] = y;
          else
            reinterpret_cast<double*>(base)[addr] = (double)y;
        }
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.status, SMLRT_STATUS_NONFINITE);
    }
  }

  // -------------------------------------------------------------- teardown
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// ---------------------------------------------------------- host helpers --
uint16_t f2bf(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

template <int H1, int H2>
std::vector<uint8_t> pack(const smlrt_model_s& m) {
  using L = Lay<H1, H2>;
  std::vector<uint8_t> blob(L::BLOB, 0);
  const int F = m.in_features;
  const float* W1 = m.host_params.data();
  const float* b1 = W1 + (size_t)H1 * F;
  const float* W2 = b1 + H1;
  const float* b2 = W2 + (size_t)H2 * H1;
  const float* W3 = b2 + H2;
  const float* b3 = W3 + H2;
  auto put = [&](size_t off, float v) {
    uint16_t h = f2bf(v);
    std::memcpy(blob.data() + off, &h, 2);
  };
  for (int kc = 0; kc < L::KC; ++kc)
    for (int n = 0; n < H2; ++n)
      for (int k = 0; k < 64; ++k) put(kc * L::W2_CHUNK + sw128_offset(n, k), W2[(size_t)n * H1 + kc * 64 + k]);
  for (int n = 0; n < H1; ++n)
    for (int k = 0; k < KX; ++k) put(L::BLOB_W1 + sw32_offset(n, k), k < F ? W1[(size_t)n * F + k] : 0.0f);
  float* tail = reinterpret_cast<float*>(blob.data() + L::BLOB_TAIL);
  std::memcpy(tail, b1, H1 * 4);
  std::memcpy(tail + H1, b2, H2 * 4);
  std::memcpy(tail + H1 + H2, W3, H2 * 4);
  tail[H1 + 2 * H2] = b3[0];
  return blob;
}

bool shape_is(const smlrt_model_s& m, int h1, int h2) {
  return m.n_layers == 3 && m.in_features <= KX && m.layers[0].out == h1 && m.layers[1].out == h2 &&
         m.layers[2].out == 1;
}

int num_sms() {
  int d = 0, n = 148;
  cudaGetDevice(&d);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
  return n;
}

template <int H1, int H2>
int launch(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs, const int32_t* in_dt,
           int n_in, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt, int n_out, int64_t r0,
           int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  using L = Lay<H1, H2>;
  if (n_in > 8 || n_out > 8) return SMLRT_E_UNSUPPORTED;
  static int configured_mask = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured_mask & (1 << dev))) {
    SMLRT_CUDA(cudaFuncSetAttribute(mlp3_tc_kernel<H1, H2>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::ALLOC));
    configured_mask |= 1 << dev;
  }
  TcArgs a{};
  a.blob = reinterpret_cast<const uint8_t*>(m.tc_blob);
  a.F = m.in_features;
  a.act1 = m.layers[0].act;
  a.act2 = m.layers[1].act;
  a.act3 = m.layers[2].act;
  a.r0 = r0;
  a.r1 = r1;
  a.n_tiles = (int)((r1 - r0 + BM - 1) / BM);
  a.staged = staged;
  a.status = status;
  Ptrs8 src{}, dst{};
  for (int i = 0; i < n_in; ++i) {
    src.p[i] = in_ptrs[i];
    src.dt[i] = in_dt[i];
  }
  for (int i = 0; i < n_out; ++i) {
    dst.p[i] = out_ptrs[i];
    dst.dt[i] = out_dt[i];
  }
  // fast gather: one f32 array, 16 contiguous features per row, 16-B aligned
  if (in.dense_rows && in.n_cols == 16 && m.in_features == 16 && in_dt[in.uarray] == SMLRT_F32) {
    const float* base = reinterpret_cast<const float*>(in_ptrs[in.uarray]) + in.col_off0;
    if (in.ustride[0] % 4 == 0 && (reinterpret_cast<uintptr_t>(base) & 15) == 0) {
      a.x_fast = base;
      a.x_pitch = in.ustride[0];
    }
  }
  const int grid = std::max(1, std::min(a.n_tiles, num_sms()));
  mlp3_tc_kernel<H1, H2><<<grid, NTHREADS, L::ALLOC, s>>>(a, in, src, out, dst);
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

// ------------------------------------------------------ descriptor self-test
// One CTA: D[128 x N] = A[128 x K] * B[N x K]^T with A/B staged exactly like
// the fused kernel stages them (SW32 when K == 16, SW128 chunks otherwise).
template <int N>
__global__ void __launch_bounds__(128, 1) tc_selftest_kernel(const float* A, const float* B, int K, float* D) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const bool sw32 = (K == 16);
  const int a_bytes = 128 * K * 2;
  uint8_t* sa = smem;
  uint8_t* sb = smem + a_bytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sb + N * K * 2);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 128 * K; i += 128) {
    const int r = i / K, k = i % K;
    const uint32_t off = sw32 ? sw32_offset(r, k) : (k / 64) * (128 * 128) + sw128_offset(r, k & 63);
    *reinterpret_cast<__nv_bfloat16*>(sa + off) = __float2bfloat16_rn(A[i]);
  }
  for (int i = threadIdx.x; i < N * K; i += 128) {
    const int r = i / K, k = i % K;
    const uint32_t off = sw32 ? sw32_offset(r, k) : (k / 64) * (N * 128) + sw128_offset(r, k & 63);
    *reinterpret_cast<__nv_bfloat16*>(sb + off) = __float2bfloat16_rn(B[i]);
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(slot, 256);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *slot;
  if (threadIdx.x == 0) {
    const uint32_t ia = smem_u32(sa), ib = smem_u32(sb);
    const uint32_t idesc = idesc_bf16(128, N);
    if (sw32) {
      mma_bf16(tbase, smem_desc(ia, 256, kSwizzle32), smem_desc(ib, 256, kSwizzle32), idesc, 0);
    } else {
      for (int kc = 0; kc < K / 64; ++kc)
        for (int k = 0; k < 4; ++k)
          mma_bf16(tbase, smem_desc(ia + kc * 128 * 128 + k * 32, 1024, kSwizzle128),
                   smem_desc(ib + kc * N * 128 + k * 32, 1024, kSwizzle128), idesc, (kc | k) != 0);
    }
    mma_commit(bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  tc_fence_after();
  const int r = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + c0, v);
    tmem_wait_ld();
    for (int e = 0; e < 32; ++e) D[r * N + c0 + e] = __uint_as_float(v[e]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 256);
  }
}

}  // namespace

int tc_pack_model(smlrt_model_s& m) {
  std::vector<uint8_t> blob;
  if (shape_is(m, 256, 128))
    blob = pack<256, 128>(m);
  else if (shape_is(m, 128, 64))
    blob = pack<128, 64>(m);
  else
    return SMLRT_OK;  // no tcgen05 kernel for this shape; region_infer reports it
  SMLRT_CUDA(cudaMalloc(&m.tc_blob, blob.size()));
  SMLRT_CUDA(cudaMemcpy(m.tc_blob, blob.data(), blob.size(), cudaMemcpyHostToDevice));
  m.tc_bytes = blob.size();
  return SMLRT_OK;
}

int launch_region_tc(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs, const int32_t* in_dt,
                     int n_in, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt, int n_out,
                     int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status, bool probe_only) {
  if (m.tc_blob == nullptr && !(probe_only && m.precision == SMLRT_BF16 &&
                                (shape_is(m, 256, 128) || shape_is(m, 128, 64))))
    return SMLRT_E_UNSUPPORTED;
  if (probe_only) return SMLRT_OK;
  if (shape_is(m, 256, 128))
    return launch<256, 128>(m, in, in_ptrs, in_dt, n_in, out, out_ptrs, out_dt, n_out, r0, r1, staged, s, status);
  if (shape_is(m, 128, 64))
    return launch<128, 64>(m, in, in_ptrs, in_dt, n_in, out, out_ptrs, out_dt, n_out, r0, r1, staged, s, status);
  return SMLRT_E_UNSUPPORTED;
}

}  // namespace smlrt

extern "C" int smlrt_tc_selftest(int K, int N, const float* A, const float* B, float* D) {
  using namespace smlrt;
  if (!(K == 16 || (K % 64 == 0 && K <= 256)) || !(N == 128 || N == 256))
    return fail(SMLRT_E_INVALID, "tc_selftest: K in {16, 64, 128, 192, 256}, N in {128, 256}");
  float *dA, *dB, *dD;
  SMLRT_CUDA(cudaMalloc(&dA, 128 * K * 4));
  SMLRT_CUDA(cudaMalloc(&dB, N * K * 4));
  SMLRT_CUDA(cudaMalloc(&dD, 128 * N * 4));
  SMLRT_CUDA(cudaMemcpy(dA, A, 128 * K * 4, cudaMemcpyHostToDevice));
  SMLRT_CUDA(cudaMemcpy(dB, B, N * K * 4, cudaMemcpyHostToDevice));
  const int smem = 128 * K * 2 + N * K * 2 + 64 + 1024;
  if (N == 128) {
    SMLRT_CUDA(cudaFuncSetAttribute(tc_selftest_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc_selftest_kernel<128><<<1, 128, smem>>>(dA, dB, K, dD);
  } else {
    SMLRT_CUDA(cudaFuncSetAttribute(tc_selftest_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc_selftest_kernel<256><<<1, 128, smem>>>(dA, dB, K, dD);
  }
  SMLRT_CUDA(cudaGetLastError());
  SMLRT_CUDA(cudaDeviceSynchronize());
  SMLRT_CUDA(cudaMemcpy(D, dD, 128 * N * 4, cudaMemcpyDeviceToHost));
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return SMLRT_OK;
}
