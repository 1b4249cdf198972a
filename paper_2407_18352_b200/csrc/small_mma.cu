// bf16 fused region for small dense MLPs (C1 options at bf16, and any
// 3-layer model F <= 8 -> H1 <= 64 -> H2 <= 64 -> G <= 8): gather ->
// forward -> scatter in one kernel, every layer on warp-level tensor-core
// MMAs with the activations kept in registers.
//
// At bf16 such a model is 0.1 % of the tensor peak per byte it reads, so the
// region is HBM- and latency-bound: a warp owns 16-row tiles whose rows
// arrive through a ring of bulk copies (packed AoS rows) or per-lane loads
// through the in-plan (tf32 m16n8k8 for layer 1: the f32 features are
// the operands), the bias is each accumulator's initial value, and act +
// bf16 packing of layer l's accumulators IS layer l+1's A fragment (the m16n8
// C and A fragment layouts coincide), so no activation ever leaves the
// registers.  Weights are B fragments loaded once per thread (shared memory
// -> registers).  Layer 3's N = 8 columns hold the G outputs.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "simt_common.cuh"
#include "tc_ptx.cuh"

namespace smlrt {
namespace {

using namespace ptx;

constexpr int SMM_G = 8, SMM_F = 8;

template <int N1, int N2>
struct SmmArgs {
  int64_t r0, r1;                 // sweep rows of the call
  const float* src;               // the in-plan's array (uniform, f32)
  float* dst;                     // the out-plan's array (uniform, f32)
  float* staged;                  // checked commit: [rows][G]
  uint32_t* status;
  int g, act1, act2, act3;
};

// per-lane B fragments and biases, laid out [what][lane] in global memory and
// staged through shared memory at kernel start.  Each bias is its
// accumulator's initial value (f32, the lane's output columns 2q, 2q + 1 of
// an n8 tile -- the m16n8 C fragment holds them for rows g and g + 8).
template <int N1, int N2>
struct SmmFrags {
  static constexpr int T1 = N1 / 8, T2 = N2 / 8, K2 = N1 / 16, K3 = N2 / 16;
  uint32_t w1[T1][32][2];      // tf32 (k = q, q + 4; n = 8t + g)
  float4 b1[T1][32];           // C quad (n = 8t + 2q, 8t + 2q + 1) x rows g, g + 8
  uint32_t w2[T2][K2][32][2];  // bf16 pairs
  float4 b2[T2][32];
  uint32_t w3[K3][32][2];
  float4 b3[32];
};

// dense input rows stream through a ring of shared-memory stages filled by
// 1-D bulk copies: a chunk is SMM_TPW tiles per warp (the CTA's 4 warps), so
// SMM_S - 1 chunks of every resident CTA are in flight while it computes --
// per-lane loads one tile ahead keep too few bytes in flight to cover DRAM
// latency at this little compute per byte
#ifndef SMM_TPW
#define SMM_TPW 4  // tiles per warp per chunk
#endif
#ifndef SMM_S
#define SMM_S 4  // ring stages
#endif
#ifndef SMM_MINB
#define SMM_MINB 1
#endif
constexpr int SMM_CH = 4 * SMM_TPW * 16;  // rows per chunk
__host__ __device__ constexpr int smm_stage_floats(int F) { return (SMM_CH * F + 8 + 31) / 32 * 32; }

// not volatile: the two tiles a warp holds interleave their MMA chains
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                         const float4& c) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c.x), "f"(c.y), "f"(c.z), "f"(c.w));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// first k step of a chain: the accumulator starts at the bias quad
__device__ __forceinline__ void mma_bf16_c(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                           const float4& c) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%11,%12,%13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c.x), "f"(c.y), "f"(c.z), "f"(c.w));
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// bounded wait: a copy that never lands traps instead of hanging the device
__device__ __forceinline__ void smm_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  for (uint32_t n = 0;; ++n) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    if (n > (1u << 26)) __trap();
  }
}

template <int ACT>
__device__ __forceinline__ uint32_t act_pack(float lo, float hi) {
  if constexpr (ACT == SMLRT_RELU) return pack_relu_bf16(lo, hi);
  else if constexpr (ACT == SMLRT_TANH) return pack_bf16(tanhf(lo), tanhf(hi));
  else return pack_bf16(lo, hi);
}
__device__ __forceinline__ float act_f(float y, int act) {
  if (act == SMLRT_RELU) return relu_nan(y);
  if (act == SMLRT_TANH) return tanhf(y);
  return y;
}

// DENSE: packed AoS input rows (row pitch == F, columns contiguous) stream
// through the bulk-copy ring and each lane picks its fragment elements out of
// the staged rows; the rows past the last whole chunk (and every non-dense
// plan) load per lane through the plan, one tile ahead
template <int N1, int N2, int ACT1, int ACT2, bool ONE_D, bool DENSE>
__global__ void __launch_bounds__(128, SMM_MINB) small_mma_kernel(const __grid_constant__ SmmArgs<N1, N2> a,
                                                        const __grid_constant__ DevPlan P,
                                                        const __grid_constant__ DevPlan Q,
                                                        const SmmFrags<N1, N2>* __restrict__ fr) {
  using Fr = SmmFrags<N1, N2>;
  constexpr int T1 = Fr::T1, T2 = Fr::T2, K2 = Fr::K2, K3 = Fr::K3;
  __shared__ __align__(16) Fr sf;
  __shared__ __align__(8) uint64_t full[SMM_S];
  extern __shared__ __align__(128) float ring[];
  const int F = P.n_cols;
  if constexpr (DENSE) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < SMM_S; ++s) mbar_init(&full[s], 1);
      mbar_fence_init();
    }
  }
  {
    const uint4* s4 = reinterpret_cast<const uint4*>(fr);
    uint4* d4 = reinterpret_cast<uint4*>(&sf);
    for (int i = threadIdx.x; i < (int)(sizeof(Fr) / 16); i += blockDim.x) d4[i] = __ldg(s4 + i);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3, warp = threadIdx.x >> 5;
  uint32_t w1[T1][2], w3[K3][2];
#pragma unroll
  for (int t = 0; t < T1; ++t) w1[t][0] = sf.w1[t][lane][0], w1[t][1] = sf.w1[t][lane][1];
#ifndef SMM_W2_SMEM
  uint32_t w2[T2][K2][2];
#pragma unroll
  for (int t = 0; t < T2; ++t)
#pragma unroll
    for (int k = 0; k < K2; ++k) w2[t][k][0] = sf.w2[t][k][lane][0], w2[t][k][1] = sf.w2[t][k][lane][1];
#define SMM_W2(t, k, i) w2[t][k][i]
#else
  // layer-2 fragments read from shared memory per use (fewer registers, more warps)
#define SMM_W2(t, k, i) sf.w2[t][k][lane][i]
#endif
#pragma unroll
  for (int k = 0; k < K3; ++k) w3[k][0] = sf.w3[k][lane][0], w3[k][1] = sf.w3[k][lane][1];
  // this lane's feature columns (k = q and q + 4 of the padded 8) and the
  // outputs it holds (2q, 2q + 1)
  const bool k0ok = q < F, k1ok = q + 4 < F;
  const int64_t c0 = k0ok ? P.col_inl[q] : 0, c1 = k1ok ? P.col_inl[q + 4] : 0;
  const int o0 = 2 * q, o1 = 2 * q + 1;
  const bool h0 = o0 < a.g, h1 = o1 < a.g;
  const bool stg = a.staged != nullptr;
  const int64_t ntiles = (a.r1 - a.r0 + 15) / 16;
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x / 32) + warp;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  const int64_t ip = ONE_D ? P.ustride[0] : 0;  // input element step per row
  const int64_t op = stg ? a.g : (ONE_D ? Q.ustride[0] : 0);
  const int64_t oc0 = stg ? o0 : (h0 ? Q.col_inl[o0] : 0), oc1 = stg ? o1 : (h1 ? Q.col_inl[o1] : 0);
  float* const obase = stg ? a.staged - a.r0 * a.g : a.dst;
  const int64_t nfull = (a.r1 - a.r0) / 16;  // tiles with all 16 rows in the call
  float chk = 0.0f;                          // y * 0 accumulates NaN iff an output is non-finite

  auto in_off = [&](int64_t r) { return ONE_D ? r * ip : row_offset_uniform(P, (uint32_t)r); };
  auto out_off = [&](int64_t r) { return stg || ONE_D ? r * op : row_offset_uniform(Q, (uint32_t)r); };
  auto load = [&](int64_t tile, uint32_t (&a1)[4]) {
    const int64_t ra = a.r0 + tile * 16 + g, rb = ra + 8;
    const bool va = tile < ntiles && ra < a.r1, vb = tile < ntiles && rb < a.r1;
    const float* pa = a.src + (va ? in_off(ra) : 0);
    const float* pb = a.src + (vb ? in_off(rb) : 0);
    // layer 1 (tf32, K = 8): a0 = (row g, k = q), a1 = (row g+8, q), a2/a3 = k + 4
    a1[0] = va && k0ok ? __float_as_uint(__ldg(pa + c0)) : 0u;
    a1[1] = vb && k0ok ? __float_as_uint(__ldg(pb + c0)) : 0u;
    a1[2] = va && k1ok ? __float_as_uint(__ldg(pa + c1)) : 0u;
    a1[3] = vb && k1ok ? __float_as_uint(__ldg(pb + c1)) : 0u;
  };
  // one 16-row tile: forward pass on the MMAs, outputs to the out-plan
  auto tile_body = [&](const uint32_t (&a1)[4], int64_t tile) {
    float d1[T1][4];
#pragma unroll
    for (int t = 0; t < T1; ++t) mma_tf32(d1[t], a1, w1[t][0], w1[t][1], sf.b1[t][lane]);
    // layer 2 (bf16): k16 step k = n8 tiles 2k, 2k + 1 of layer 1
    float d2[T2][4];
#pragma unroll
    for (int k = 0; k < K2; ++k) {
      const uint32_t af[4] = {act_pack<ACT1>(d1[2 * k][0], d1[2 * k][1]), act_pack<ACT1>(d1[2 * k][2], d1[2 * k][3]),
                              act_pack<ACT1>(d1[2 * k + 1][0], d1[2 * k + 1][1]),
                              act_pack<ACT1>(d1[2 * k + 1][2], d1[2 * k + 1][3])};
#pragma unroll
      for (int t = 0; t < T2; ++t) {
        if (k == 0) mma_bf16_c(d2[t], af, SMM_W2(t, 0, 0), SMM_W2(t, 0, 1), sf.b2[t][lane]);
        else mma_bf16(d2[t], af, SMM_W2(t, k, 0), SMM_W2(t, k, 1));
      }
    }
    // layer 3 (bf16, N = 8 holds the outputs)
    float y[4];
#pragma unroll
    for (int k = 0; k < K3; ++k) {
      const uint32_t af[4] = {act_pack<ACT2>(d2[2 * k][0], d2[2 * k][1]), act_pack<ACT2>(d2[2 * k][2], d2[2 * k][3]),
                              act_pack<ACT2>(d2[2 * k + 1][0], d2[2 * k + 1][1]),
                              act_pack<ACT2>(d2[2 * k + 1][2], d2[2 * k + 1][3])};
      if (k == 0) mma_bf16_c(y, af, w3[0][0], w3[0][1], sf.b3[lane]);
      else mma_bf16(y, af, w3[k][0], w3[k][1]);
    }
    if (a.act3 != SMLRT_IDENTITY) {
#pragma unroll
      for (int e = 0; e < 4; ++e) y[e] = act_f(y[e], a.act3);
    }
    // y = (row g: outputs o0, o1), (row g + 8: o0, o1); unused columns and
    // rows past the end are finite (zero inputs, zero weights)
    const int64_t ra = a.r0 + tile * 16 + g, rb = ra + 8;
    if ((stg || ONE_D) && tile < nfull) {
      float* pa = obase + ra * op;
      float* pb = pa + 8 * op;
      if (h0) pa[oc0] = y[0], pb[oc0] = y[2];
      if (h1) pa[oc1] = y[1], pb[oc1] = y[3];
    } else {
      const bool va = ra < a.r1, vb = rb < a.r1;
      float* pa = obase + out_off(va ? ra : a.r0);
      float* pb = obase + out_off(vb ? rb : a.r0);
      if (va && h0) pa[oc0] = y[0];
      if (va && h1) pa[oc1] = y[1];
      if (vb && h0) pb[oc0] = y[2];
      if (vb && h1) pb[oc1] = y[3];
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) chk = fmaf(y[e], 0.0f, chk);
  };

  int64_t t0 = 0;  // first tile of the per-lane path
  if constexpr (DENSE) {
    const int64_t nch = (a.r1 - a.r0) / SMM_CH;
    const int64_t mine = nch > (int64_t)blockIdx.x ? (nch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int sb = smm_stage_floats(F);
    // chunk c's rows start at gsrc + c * SMM_CH * F; a chunk is a multiple of
    // 16 B, so every chunk has the same misalignment `al` (floats) and copies
    // from the 16-B boundary below to the one above -- both inside the
    // 16-B granules of the array's own first and last bytes
    const float* gsrc = a.src + P.col_inl[0] + a.r0 * F;
    const int al = (int)((reinterpret_cast<uintptr_t>(gsrc) & 15) >> 2);
    const uint32_t bytes = (uint32_t)(((SMM_CH * F + al) * 4 + 15) & ~15);
    auto issue = [&](int64_t k) {
      const int s = (int)(k % SMM_S);
      const float* src = gsrc + (blockIdx.x + k * gridDim.x) * (int64_t)SMM_CH * F - al;
      expect_tx(&full[s], bytes);
      bulk_g2s(smem_u32(ring + s * sb), src, bytes, &full[s]);
    };
    if (threadIdx.x == 0)
      for (int64_t k = 0; k < SMM_S && k < mine; ++k) issue(k);
    for (int64_t k = 0; k < mine; ++k) {
      const int s = (int)(k % SMM_S);
      smm_wait(&full[s], (uint32_t)((k / SMM_S) & 1));
      const float* xs = ring + s * sb + al + warp * (SMM_TPW * 16) * F;
      uint32_t af[SMM_TPW][4];
#pragma unroll
      for (int j = 0; j < SMM_TPW; ++j) {
        const float* xa = xs + (j * 16 + g) * F;
        af[j][0] = k0ok ? __float_as_uint(xa[q]) : 0u;
        af[j][1] = k0ok ? __float_as_uint(xa[8 * F + q]) : 0u;
        af[j][2] = k1ok ? __float_as_uint(xa[q + 4]) : 0u;
        af[j][3] = k1ok ? __float_as_uint(xa[8 * F + q + 4]) : 0u;
      }
      __syncthreads();  // every warp has its fragments: the stage is free
      if (threadIdx.x == 0 && k + SMM_S < mine) {
        fence_async_smem();
        issue(k + SMM_S);
      }
      const int64_t tile0 = (blockIdx.x + k * gridDim.x) * (SMM_CH / 16) + warp * SMM_TPW;
#pragma unroll
      for (int j = 0; j < SMM_TPW; ++j) tile_body(af[j], tile0 + j);
    }
    t0 = nch * (SMM_CH / 16);
  }
  uint32_t nxt[4];
  load(t0 + wid, nxt);
  for (int64_t tile = t0 + wid; tile < ntiles; tile += nw) {
    const uint32_t a1[4] = {nxt[0], nxt[1], nxt[2], nxt[3]};
    load(tile + nw, nxt);
    tile_body(a1, tile);
  }
  if (__any_sync(0xffffffffu, chk != chk) && lane == 0) atomicOr(a.status, SMLRT_STATUS_NONFINITE);
}
#undef SMM_W2

uint32_t smm_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}
uint32_t smm_bf16(float f) {
  uint32_t u = smm_bits(f);
  u += 0x7fffu + ((u >> 16) & 1u);
  return u >> 16;
}
uint32_t smm_tf32(float f) {
  uint32_t u = smm_bits(f);
  u += 0xfffu + ((u >> 13) & 1u);
  return u & ~0x1fffu;
}

template <int N1, int N2>
int build_smm(smlrt_model_s& m) {
  using Fr = SmmFrags<N1, N2>;
  const DevLayer &L1 = m.layers[0], &L2 = m.layers[1], &L3 = m.layers[2];
  const int F = L1.in, H1 = L1.out, H2 = L2.out, G = L3.out;
  Fr h{};
  const float* p = m.host_params.data();  // [W1][b1][W2][b2][W3][b3]
  const float *W1 = p, *b1 = W1 + (size_t)H1 * F, *W2 = b1 + H1, *b2 = W2 + (size_t)H2 * H1,
              *W3 = b2 + H2, *b3 = W3 + (size_t)G * H2;
  auto w1 = [&](int n, int k) { return n < H1 && k < F ? W1[(size_t)n * F + k] : 0.0f; };
  auto w2 = [&](int n, int k) { return n < H2 && k < H1 ? W2[(size_t)n * H1 + k] : 0.0f; };
  auto w3 = [&](int n, int k) { return n < G && k < H2 ? W3[(size_t)n * H2 + k] : 0.0f; };
  auto bias = [&](const float* b, int n, int nmax) { return n < nmax ? b[n] : 0.0f; };
  // the C quad of columns (n, n + 1) for rows g and g + 8
  auto quad = [&](const float* b, int n, int nmax) {
    return float4{bias(b, n, nmax), bias(b, n + 1, nmax), bias(b, n, nmax), bias(b, n + 1, nmax)};
  };
  for (int l = 0; l < 32; ++l) {
    const int gg = l >> 2, qq = l & 3;
    for (int t = 0; t < Fr::T1; ++t) {
      h.w1[t][l][0] = smm_tf32(w1(8 * t + gg, qq));
      h.w1[t][l][1] = smm_tf32(w1(8 * t + gg, qq + 4));
      h.b1[t][l] = quad(b1, 8 * t + 2 * qq, H1);
    }
    for (int t = 0; t < Fr::T2; ++t) {
      const int n = 8 * t + gg;
      for (int k = 0; k < Fr::K2; ++k) {
        const int kk = 16 * k + 2 * qq;
        h.w2[t][k][l][0] = smm_bf16(w2(n, kk)) | (smm_bf16(w2(n, kk + 1)) << 16);
        h.w2[t][k][l][1] = smm_bf16(w2(n, kk + 8)) | (smm_bf16(w2(n, kk + 9)) << 16);
      }
      h.b2[t][l] = quad(b2, 8 * t + 2 * qq, H2);
    }
    for (int k = 0; k < Fr::K3; ++k) {
      const int kk = 16 * k + 2 * qq;
      h.w3[k][l][0] = smm_bf16(w3(gg, kk)) | (smm_bf16(w3(gg, kk + 1)) << 16);
      h.w3[k][l][1] = smm_bf16(w3(gg, kk + 8)) | (smm_bf16(w3(gg, kk + 9)) << 16);
    }
    h.b3[l] = quad(b3, 2 * qq, G);
  }
  SMLRT_CUDA(cudaMalloc(&m.smm_blob, sizeof(Fr)));
  SMLRT_CUDA(cudaMemcpy(m.smm_blob, &h, sizeof(Fr), cudaMemcpyHostToDevice));
  return SMLRT_OK;
}

// the padded widths of a model the kernel takes, or false
bool smm_shape(const smlrt_model_s& m, int* n1, int* n2) {
  if (m.n_layers != 3) return false;
  for (int l = 0; l < 3; ++l)
    if (m.layers[l].kind != SMLRT_DENSE) return false;
  const int F = m.layers[0].in, H1 = m.layers[0].out, H2 = m.layers[1].out, G = m.layers[2].out;
  if (F > SMM_F || H1 > 64 || H2 > 64 || G > SMM_G) return false;
  const int a1 = m.layers[0].act, a2 = m.layers[1].act;
  if (a1 != a2) return false;
  auto r16 = [](int n) { return n <= 16 ? 16 : n <= 32 ? 32 : 64; };
  *n1 = r16(H1);
  *n2 = r16(H2);
  return true;
}

template <int N1, int N2, int ACT1, int ACT2>
int launch_smm(const smlrt_model_s& m, const DevPlan& in, const void* src, const DevPlan& out, void* dst,
               int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  using Fr = SmmFrags<N1, N2>;
  const DevLayer &L1 = m.layers[0], &L2 = m.layers[1], &L3 = m.layers[2];
  const int G = L3.out;
  const void* dev = m.smm_blob;
  if (dev == nullptr) return SMLRT_E_UNSUPPORTED;
  SmmArgs<N1, N2> a{};
  a.r0 = r0;
  a.r1 = r1;
  a.src = static_cast<const float*>(src);
  a.dst = static_cast<float*>(dst);
  a.staged = staged;
  a.status = status;
  a.g = G;
  a.act1 = L1.act;
  a.act2 = L2.act;
  a.act3 = L3.act;
  // persistent grid: one wave of resident CTAs, each warp striding over
  // tiles (dense rows: over ring chunks); occupancy per feature count, as
  // the ring's stage size depends on it
  const int64_t tiles = (r1 - r0 + 15) / 16;
  const int F = in.n_cols;
  const bool dense = in.n_sweep == 1 && out.n_sweep == 1 && in.dense_rows && in.ustride[0] == in.n_cols;
  const size_t ring = dense ? (size_t)SMM_S * smm_stage_floats(F) * sizeof(float) : 0;
  static int slots[2][SMM_F + 1] = {};
  int& sl = slots[dense][F];
  if (!sl) {
    if (dense)  // the ring of 8-feature rows exceeds the 48 KB default
      SMLRT_CUDA(cudaFuncSetAttribute(small_mma_kernel<N1, N2, ACT1, ACT2, true, true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMM_S * smm_stage_floats(SMM_F) * (int)sizeof(float)));
    int dev_id = 0, sms = 148, per_sm = 0;
    cudaGetDevice(&dev_id);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev_id);
    if (dense)
      SMLRT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, small_mma_kernel<N1, N2, ACT1, ACT2, true, true>,
                                                               128, ring));
    else
      SMLRT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, small_mma_kernel<N1, N2, ACT1, ACT2, true, false>, 128, 0));
    sl = std::max(1, per_sm) * sms;
  }
  const int64_t blocks = std::min<int64_t>((tiles + 3) / 4, sl);
  const unsigned grid = (unsigned)std::max<int64_t>(1, blocks);
  if (dense)
    small_mma_kernel<N1, N2, ACT1, ACT2, true, true><<<grid, 128, ring, s>>>(a, in, out, static_cast<const Fr*>(dev));
  else if (in.n_sweep == 1 && out.n_sweep == 1)
    small_mma_kernel<N1, N2, ACT1, ACT2, true, false><<<grid, 128, 0, s>>>(a, in, out, static_cast<const Fr*>(dev));
  else
    small_mma_kernel<N1, N2, ACT1, ACT2, false, false><<<grid, 128, 0, s>>>(a, in, out, static_cast<const Fr*>(dev));
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

template <int N1, int N2>
int launch_smm_act(const smlrt_model_s& m, const DevPlan& in, const void* src, const DevPlan& out, void* dst,
                   int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  const int a1 = m.layers[0].act, a2 = m.layers[1].act;
  if (a1 == SMLRT_RELU && a2 == SMLRT_RELU)
    return launch_smm<N1, N2, SMLRT_RELU, SMLRT_RELU>(m, in, src, out, dst, r0, r1, staged, s, status);
  if (a1 == SMLRT_TANH && a2 == SMLRT_TANH)
    return launch_smm<N1, N2, SMLRT_TANH, SMLRT_TANH>(m, in, src, out, dst, r0, r1, staged, s, status);
  if (a1 == SMLRT_IDENTITY && a2 == SMLRT_IDENTITY)
    return launch_smm<N1, N2, SMLRT_IDENTITY, SMLRT_IDENTITY>(m, in, src, out, dst, r0, r1, staged, s, status);
  return SMLRT_E_UNSUPPORTED;
}

}  // namespace

// bf16 region through the small-MLP warp-MMA kernel, or SMLRT_E_UNSUPPORTED
// when the model / plans do not fit it (3 dense layers F <= 8, H1 and H2 in
// {16, 32, 64} after rounding up to 16 -- the zero padding is exact --, G <=
// 8, matching hidden activations; f32 arrays, uniform plans)
int launch_region_small_mma(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs,
                            const int32_t* in_dt, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt,
                            int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  int n1 = 0, n2 = 0;
  if (m.smm_blob == nullptr || !smm_shape(m, &n1, &n2)) return SMLRT_E_UNSUPPORTED;
  if (!in.uniform || !out.uniform || in.n_cols != m.layers[0].in || out.n_cols != m.layers[2].out)
    return SMLRT_E_UNSUPPORTED;
  if (in_dt[in.uarray] != SMLRT_F32 || out_dt[out.uarray] != SMLRT_F32) return SMLRT_E_UNSUPPORTED;
  if (r1 <= r0) return SMLRT_OK;
  const void* src = in_ptrs[in.uarray];
  void* dst = out_ptrs[out.uarray];
  // 1-D sweeps: the tcgen05 kernel (small_tc.cu); other sweeps and
  // SMLRT_SMALL_TC=0 take the warp-MMA kernel below
  const int rc = launch_region_small_tc(m, in, src, out, dst, r0, r1, staged, s, status);
  if (rc != SMLRT_E_UNSUPPORTED) return rc;
#define SMM_GO(A, B)                                                                      \
  if (n1 == A && n2 == B) return launch_smm_act<A, B>(m, in, src, out, dst, r0, r1, staged, s, status)
  SMM_GO(64, 32);
  SMM_GO(64, 64);
  SMM_GO(32, 32);
  SMM_GO(32, 16);
  SMM_GO(16, 16);
  SMM_GO(64, 16);
  SMM_GO(32, 64);
  SMM_GO(16, 32);
  SMM_GO(16, 64);
#undef SMM_GO
  return SMLRT_E_UNSUPPORTED;
}

// at upload (bf16 models): the kernel's B-fragment blob when the shape fits
int small_mma_pack(smlrt_model_s& m) {
  int n1 = 0, n2 = 0;
  if (!smm_shape(m, &n1, &n2)) return SMLRT_OK;
  if (int rc = small_tc_pack(m, n1, n2)) return rc;
#define SMM_B(A, B) \
  if (n1 == A && n2 == B) return build_smm<A, B>(m)
  SMM_B(64, 32);
  SMM_B(64, 64);
  SMM_B(32, 32);
  SMM_B(32, 16);
  SMM_B(16, 16);
  SMM_B(64, 16);
  SMM_B(32, 64);
  SMM_B(16, 32);
  SMM_B(16, 64);
#undef SMM_B
  return SMLRT_OK;
}

}  // namespace smlrt
