// bf16 fused region for small dense MLPs (C1 options at bf16, and any
// 3-layer model F <= 8 -> H1 <= 64 -> H2 <= 64 -> G <= 8): gather ->
// forward -> scatter in one kernel, every layer on warp-level tensor-core
// MMAs with the activations kept in registers.
//
// At bf16 such a model is 0.1 % of the tensor peak per byte it reads, so the
// region is HBM- and latency-bound: a warp owns 16-row tiles, its lanes load
// their A-fragment elements of the tile's rows straight from the application
// array through the in-plan (tf32 m16n8k8 for layer 1: the f32 features are
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

constexpr int SMM_G = 8;

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
// staged through shared memory at kernel start
// Biases ride in the MMAs: layer 1's input column F (< 8) is the constant 1
// with b1 as its weights; layers 2 and 3 get one more k16 step whose A
// fragment is the constant (1, 0, ...) and whose B fragment is the bias.
template <int N1, int N2>
struct SmmFrags {
  static constexpr int T1 = N1 / 8, T2 = N2 / 8, K2 = N1 / 16 + 1, K3 = N2 / 16 + 1;
  uint32_t w1[T1][32][2];      // tf32 (k = q, q + 4; n = 8t + g), row F = b1
  uint32_t w2[T2][K2][32][2];  // bf16 pairs; step K2-1 = b2
  uint32_t w3[K3][32][2];      // step K3-1 = b3
};

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
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

// row offset of sweep row r: the 1-D sweep (AoS / SoA records) is one multiply
template <bool ONE_D>
__device__ __forceinline__ int64_t smm_row(const DevPlan& P, int64_t r) {
  if constexpr (ONE_D) return r * P.ustride[0];
  else return row_offset_uniform(P, (uint32_t)r);
}

// DENSE: packed AoS input rows (row pitch == F, columns contiguous): a warp
// reads its tile's 16 x F floats as one coalesced run into shared memory and
// each lane picks its fragment elements there -- no per-element addressing
template <int N1, int N2, int ACT1, int ACT2, bool ONE_D, bool DENSE>
__global__ void __launch_bounds__(128) small_mma_kernel(const __grid_constant__ SmmArgs<N1, N2> a,
                                                        const __grid_constant__ DevPlan P,
                                                        const __grid_constant__ DevPlan Q,
                                                        const SmmFrags<N1, N2>* __restrict__ fr) {
  using Fr = SmmFrags<N1, N2>;
  constexpr int T1 = Fr::T1, T2 = Fr::T2, K2 = Fr::K2, K3 = Fr::K3;
  __shared__ __align__(16) Fr sf;
  {
    const uint4* s4 = reinterpret_cast<const uint4*>(fr);
    uint4* d4 = reinterpret_cast<uint4*>(&sf);
    for (int i = threadIdx.x; i < (int)(sizeof(Fr) / 16); i += blockDim.x) d4[i] = __ldg(s4 + i);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
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
  // A of the bias steps: (1, 0) at k = 0 of the step for quad member 0
  const uint32_t one_lo = q == 0 ? 0x3f80u : 0u;  // bf16 1.0 in the low half
  const uint32_t abias[4] = {one_lo, one_lo, 0u, 0u};
  // this lane's feature columns (k = q and q + 4 of the padded 8; column F is
  // the constant 1 of layer 1's bias) and the outputs it holds (2q, 2q + 1)
  const int F = P.n_cols;
  const bool k0ok = q < F, k1ok = q + 4 < F;
  const uint32_t c0v = q == F ? 0x3f800000u : 0u, c1v = q + 4 == F ? 0x3f800000u : 0u;
  const int64_t c0 = k0ok ? P.col_inl[q] : 0, c1 = k1ok ? P.col_inl[q + 4] : 0;
  const int o0 = 2 * q, o1 = 2 * q + 1;
  const bool h0 = o0 < a.g, h1 = o1 < a.g;
  const bool stg = a.staged != nullptr;
  // per-lane pointers of the first tile's rows g and g + 8 (ONE_D: advanced by
  // a constant per tile; otherwise recomputed through the plan)
  const int64_t ntiles = (a.r1 - a.r0 + 15) / 16;
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  const int64_t ip = ONE_D ? P.ustride[0] : 0;  // input element step per row
  const int64_t op = stg ? a.g : (ONE_D ? Q.ustride[0] : 0);
  const int64_t oc0 = stg ? o0 : (h0 ? Q.col_inl[o0] : 0), oc1 = stg ? o1 : (h1 ? Q.col_inl[o1] : 0);
  float* const obase = stg ? a.staged - a.r0 * a.g : a.dst;
  float chk = 0.0f;  // y * 0 accumulates NaN iff an output is non-finite

  auto in_off = [&](int64_t r) { return ONE_D ? r * ip : row_offset_uniform(P, (uint32_t)r); };
  auto out_off = [&](int64_t r) { return stg || ONE_D ? r * op : row_offset_uniform(Q, (uint32_t)r); };
  __shared__ float xt[4][16 * 8];  // per-warp tile staging (DENSE)
  float* xw = xt[threadIdx.x >> 5];
  const float* dsrc = a.src + (DENSE ? P.col_inl[0] : 0);
  // full tiles (all 16 rows in the call) load and store without predicates
  const int64_t nfull = (a.r1 - a.r0) / 16;
  auto load_dense = [&](int64_t tile, float (&v)[4]) {
    const float* base = dsrc + (a.r0 + tile * 16) * F + lane;
    if (tile < nfull) {
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = (32 * u < 16 * 7 && lane + 32 * u < 16 * F) ? __ldg(base + 32 * u) : 0.0f;
    } else {
      const int64_t left = tile < ntiles ? (a.r1 - a.r0 - tile * 16) * F : 0;  // elements in the tail tile
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = (lane + 32 * u < 16 * F && lane + 32 * u < left) ? __ldg(base + 32 * u) : 0.0f;
    }
  };
  auto frag_dense = [&](const float (&v)[4], uint32_t (&a1)[4]) {
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (lane + 32 * u < 16 * F) xw[lane + 32 * u] = v[u];
    __syncwarp();
    a1[0] = k0ok ? __float_as_uint(xw[g * F + q]) : c0v;
    a1[1] = k0ok ? __float_as_uint(xw[(g + 8) * F + q]) : c0v;
    a1[2] = k1ok ? __float_as_uint(xw[g * F + q + 4]) : c1v;
    a1[3] = k1ok ? __float_as_uint(xw[(g + 8) * F + q + 4]) : c1v;
  };
  auto load = [&](int64_t tile, uint32_t (&a1)[4]) {
    const int64_t ra = a.r0 + tile * 16 + g, rb = ra + 8;
    const bool va = tile < ntiles && ra < a.r1, vb = tile < ntiles && rb < a.r1;
    const float* pa = a.src + (va ? in_off(ra) : 0);
    const float* pb = a.src + (vb ? in_off(rb) : 0);
    // layer 1 (tf32, K = 8): a0 = (row g, k = q), a1 = (row g+8, q), a2/a3 = k + 4
    a1[0] = va && k0ok ? __float_as_uint(__ldg(pa + c0)) : c0v;
    a1[1] = vb && k0ok ? __float_as_uint(__ldg(pb + c0)) : c0v;
    a1[2] = va && k1ok ? __float_as_uint(__ldg(pa + c1)) : c1v;
    a1[3] = vb && k1ok ? __float_as_uint(__ldg(pb + c1)) : c1v;
  };
  uint32_t nxt[4];
  float nxv[4];
  if constexpr (DENSE) load_dense(wid, nxv);
  else load(wid, nxt);
  for (int64_t tile = wid; tile < ntiles; tile += nw) {
    uint32_t a1[4];
    if constexpr (DENSE) {
      frag_dense(nxv, a1);
      load_dense(tile + nw, nxv);
    } else {
      a1[0] = nxt[0], a1[1] = nxt[1], a1[2] = nxt[2], a1[3] = nxt[3];
      load(tile + nw, nxt);
    }
    float d1[T1][4];
#pragma unroll
    for (int t = 0; t < T1; ++t) {
      d1[t][0] = d1[t][1] = d1[t][2] = d1[t][3] = 0.0f;
      mma_tf32(d1[t], a1, w1[t][0], w1[t][1]);
    }
    // layer 2 (bf16): k16 step k = n8 tiles 2k, 2k + 1 of layer 1; last = bias
    float d2[T2][4];
#pragma unroll
    for (int t = 0; t < T2; ++t) {
      d2[t][0] = d2[t][1] = d2[t][2] = d2[t][3] = 0.0f;
      mma_bf16(d2[t], abias, SMM_W2(t, K2 - 1, 0), SMM_W2(t, K2 - 1, 1));
    }
#pragma unroll
    for (int k = 0; k < K2 - 1; ++k) {
      const uint32_t af[4] = {act_pack<ACT1>(d1[2 * k][0], d1[2 * k][1]), act_pack<ACT1>(d1[2 * k][2], d1[2 * k][3]),
                              act_pack<ACT1>(d1[2 * k + 1][0], d1[2 * k + 1][1]),
                              act_pack<ACT1>(d1[2 * k + 1][2], d1[2 * k + 1][3])};
#pragma unroll
      for (int t = 0; t < T2; ++t) mma_bf16(d2[t], af, SMM_W2(t, k, 0), SMM_W2(t, k, 1));
    }
    // layer 3 (bf16, N = 8 holds the outputs)
    float y[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    mma_bf16(y, abias, w3[K3 - 1][0], w3[K3 - 1][1]);
#pragma unroll
    for (int k = 0; k < K3 - 1; ++k) {
      const uint32_t af[4] = {act_pack<ACT2>(d2[2 * k][0], d2[2 * k][1]), act_pack<ACT2>(d2[2 * k][2], d2[2 * k][3]),
                              act_pack<ACT2>(d2[2 * k + 1][0], d2[2 * k + 1][1]),
                              act_pack<ACT2>(d2[2 * k + 1][2], d2[2 * k + 1][3])};
      mma_bf16(y, af, w3[k][0], w3[k][1]);
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
  // layer 1's column F carries b1; layers 2/3 have a bias k step
  auto w1b = [&](int n, int k) { return k == F ? (n < H1 ? b1[n] : 0.0f) : w1(n, k); };
  for (int l = 0; l < 32; ++l) {
    const int gg = l >> 2, qq = l & 3;
    for (int t = 0; t < Fr::T1; ++t) {
      h.w1[t][l][0] = smm_tf32(w1b(8 * t + gg, qq));
      h.w1[t][l][1] = smm_tf32(w1b(8 * t + gg, qq + 4));
    }
    for (int t = 0; t < Fr::T2; ++t) {
      const int n = 8 * t + gg;
      for (int k = 0; k < Fr::K2 - 1; ++k) {
        const int kk = 16 * k + 2 * qq;
        h.w2[t][k][l][0] = smm_bf16(w2(n, kk)) | (smm_bf16(w2(n, kk + 1)) << 16);
        h.w2[t][k][l][1] = smm_bf16(w2(n, kk + 8)) | (smm_bf16(w2(n, kk + 9)) << 16);
      }
      h.w2[t][Fr::K2 - 1][l][0] = qq == 0 && n < H2 ? smm_bf16(b2[n]) : 0u;  // k = 0 of the bias step
      h.w2[t][Fr::K2 - 1][l][1] = 0u;
    }
    for (int k = 0; k < Fr::K3 - 1; ++k) {
      const int kk = 16 * k + 2 * qq;
      h.w3[k][l][0] = smm_bf16(w3(gg, kk)) | (smm_bf16(w3(gg, kk + 1)) << 16);
      h.w3[k][l][1] = smm_bf16(w3(gg, kk + 8)) | (smm_bf16(w3(gg, kk + 9)) << 16);
    }
    h.w3[Fr::K3 - 1][l][0] = qq == 0 && gg < G ? smm_bf16(b3[gg]) : 0u;
    h.w3[Fr::K3 - 1][l][1] = 0u;
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
  if (F > 7 || H1 > 64 || H2 > 64 || G > SMM_G) return false;  // column F carries b1
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
  // persistent grid: one wave of resident CTAs, each warp striding over tiles
  const int64_t tiles = (r1 - r0 + 15) / 16;
  static int slots = 0;
  if (!slots) {
    int dev_id = 0, sms = 148, per_sm = 0;
    cudaGetDevice(&dev_id);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev_id);
    SMLRT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, small_mma_kernel<N1, N2, ACT1, ACT2, true, false>, 128, 0));
    slots = std::max(1, per_sm) * sms;
  }
  const int64_t blocks = std::min<int64_t>((tiles + 3) / 4, slots);
  const unsigned grid = (unsigned)std::max<int64_t>(1, blocks);
  const bool dense = in.n_sweep == 1 && in.dense_rows && in.ustride[0] == in.n_cols;
  if (in.n_sweep == 1 && out.n_sweep == 1 && dense)
    small_mma_kernel<N1, N2, ACT1, ACT2, true, true><<<grid, 128, 0, s>>>(a, in, out, static_cast<const Fr*>(dev));
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
