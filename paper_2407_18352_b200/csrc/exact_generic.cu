// Fused exact region for any small dense MLP (runtime dimensions): the
// fallback of the templated instantiations (exact_c1/c5/small.cu) for shapes
// that have none -- gather -> every layer -> scatter in one persistent
// kernel, bitwise equal to the reference's ordered f32 arithmetic
// (_matmul_rowwise, models.py:188-194: acc = acc + x_f * w[j, f] in feature
// order, separate multiply and add, then + b[j], then the activation).
//
// A CTA owns T rows at a time (thread = row).  All layers' weights sit in
// shared memory transposed to [in][out8] (out padded to 8) so eight
// consecutive outputs of one input feature are two LDS.128 broadcasts; each
// row's activations live in two shared ping-pong buffers laid out [feature][T]
// (thread-contiguous, conflict-free).  Eight outputs are accumulated at once
// as four packed f32x2 pairs: mul.rn.f32x2 then fma.rn.f32x2(p, one, acc)
// with `one` from the parameter bank (RN(p*1 + acc) = RN(p + acc) exactly,
// and ptxas cannot contract it into an FFMA2 -- the templated kernels' trick).
#include "simt_common.cuh"
#include "exact_region.cuh"

namespace smlrt {
namespace {

constexpr int GX_MAX_LAYERS = 8;
constexpr int GX_MAX_WIDTH = 256;

struct GxLayer {
  const float* w;  // [out][in] f32 (device copy of the model)
  const float* b;  // [out]
  int in, out, out8, act;
  int wt_off;      // float offset of this layer's transposed weights in shared memory
  int b_off;       // float offset of its bias
};

struct GxArgs {
  GxLayer L[GX_MAX_LAYERS];
  int n_layers, maxw, act_floats;  // act_floats = 2 * maxw * T
  float one2[2];                   // (1, 1) for the packed add
};

__device__ __forceinline__ uint64_t gx_pk(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void gx_unpk(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

template <int T>
__global__ void __launch_bounds__(T) region_generic_exact_kernel(const __grid_constant__ GxArgs a,
                                                                   const __grid_constant__ DevPlan Pin,
                                                                   const __grid_constant__ Ptrs src,
                                                                   const __grid_constant__ DevPlan Pout,
                                                                   const __grid_constant__ Ptrs dst, int64_t r0,
                                                                   int64_t r1, float* __restrict__ staged,
                                                                   uint32_t* status) {
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  const int t = threadIdx.x;
  // transposed weights + biases, once per (persistent) CTA
  for (int l = 0; l < a.n_layers; ++l) {
    const GxLayer& L = a.L[l];
    for (int i = t; i < L.in * L.out8; i += T) {
      const int f = i / L.out8, j = i - f * L.out8;
      sm[L.wt_off + i] = j < L.out ? __ldg(L.w + (int64_t)j * L.in + f) : 0.0f;
    }
    for (int j = t; j < L.out; j += T) sm[L.b_off + j] = __ldg(L.b + j);
  }
  __syncthreads();
  float* buf0 = sm;                 // [maxw][T]
  float* buf1 = sm + a.maxw * T;
  uint64_t one;
  asm("mov.b64 %0, {%1, %2};" : "=l"(one) : "f"(a.one2[0]), "f"(a.one2[1]));
  const int G = a.L[a.n_layers - 1].out;
  bool bad = false;
  for (int64_t blk = r0 + (int64_t)blockIdx.x * T; blk < r1; blk += (int64_t)gridDim.x * T) {
    const int64_t row = blk + t;
    const bool live = row < r1;
    // gather (compose_tensor order: plan columns)
    for (int c = 0; c < Pin.n_cols; ++c) {
      float v = 0.0f;
      if (live) {
        const int arr = Pin.uniform ? Pin.uarray : __ldg(Pin.col_arr + c);
        v = load_as_f32(src.p[arr], src.dt[arr], element_address(Pin, (uint32_t)row, c));
      }
      buf0[c * T + t] = v;
    }
    float* in = buf0;
    float* out = buf1;
    for (int l = 0; l < a.n_layers; ++l) {
      const GxLayer& L = a.L[l];
      const float* wt = sm + L.wt_off;
      for (int j0 = 0; j0 < L.out; j0 += 8) {
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
        for (int f = 0; f < L.in; ++f) {
          const float x = in[f * T + t];
          const uint64_t xx = gx_pk(x, x);
          const float4 w0 = *reinterpret_cast<const float4*>(wt + f * L.out8 + j0);
          const float4 w1 = *reinterpret_cast<const float4*>(wt + f * L.out8 + j0 + 4);
          const uint64_t wp[4] = {gx_pk(w0.x, w0.y), gx_pk(w0.z, w0.w), gx_pk(w1.x, w1.y), gx_pk(w1.z, w1.w)};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint64_t p;
            asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(xx), "l"(wp[k]));
            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[k]) : "l"(p), "l"(one));
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float lo, hi;
          gx_unpk(acc[k], lo, hi);
          const int j = j0 + 2 * k;
          if (j < L.out) out[j * T + t] = activate(__fadd_rn(lo, sm[L.b_off + j]), L.act);
          if (j + 1 < L.out) out[(j + 1) * T + t] = activate(__fadd_rn(hi, sm[L.b_off + j + 1]), L.act);
        }
      }
      float* tmp = in;
      in = out;
      out = tmp;
    }
    if (!live) continue;
    for (int g = 0; g < G; ++g) bad |= nonfinite(in[g * T + t]);
    if (staged != nullptr) {
      for (int g = 0; g < G; ++g) staged[(row - r0) * G + g] = in[g * T + t];
    } else {
      for (int g = 0; g < G; ++g) {
        const int arr = Pout.uniform ? Pout.uarray : __ldg(Pout.col_arr + g);
        store_f32(const_cast<void*>(dst.p[arr]), dst.dt[arr], element_address(Pout, (uint32_t)row, g),
                  in[g * T + t]);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && (t & 31) == 0) flag_nonfinite(status);
}

template <int T>
int gx_launch(const GxArgs& a, size_t smem, const DevPlan& in, const Ptrs& src, const DevPlan& out, const Ptrs& dst,
              int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  static int configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured & (1 << dev))) {
    SMLRT_CUDA(cudaFuncSetAttribute(region_generic_exact_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    227 * 1024));
    configured |= 1 << dev;
  }
  int sms = 148, per_sm = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  SMLRT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, region_generic_exact_kernel<T>, T, smem));
  const int64_t blocks = (r1 - r0 + T - 1) / T;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sms * std::max(1, per_sm)));
  region_generic_exact_kernel<T><<<grid, T, smem, s>>>(a, in, src, out, dst, r0, r1, staged, status);
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

}  // namespace

// the layout the kernel needs, or false (too many layers, too wide, or the
// weights + activation buffers exceed shared memory)
static bool gx_layout(const smlrt_model_s& m, int T, GxArgs* a, size_t* smem) {
  if (m.n_layers > GX_MAX_LAYERS) return false;
  int maxw = m.in_features;
  for (const auto& L : m.layers) {
    if (L.kind != SMLRT_DENSE) return false;
    maxw = std::max(maxw, L.out);
  }
  if (maxw > GX_MAX_WIDTH) return false;
  int off = 2 * maxw * T;
  for (int l = 0; l < m.n_layers; ++l) {
    const auto& L = m.layers[l];
    GxLayer& g = a->L[l];
    g.w = L.w;
    g.b = L.b;
    g.in = L.in;
    g.out = L.out;
    g.out8 = (L.out + 7) / 8 * 8;
    g.act = L.act;
    g.wt_off = (off + 3) / 4 * 4;
    g.b_off = g.wt_off + g.in * g.out8;
    off = g.b_off + L.out;
  }
  a->n_layers = m.n_layers;
  a->maxw = maxw;
  a->act_floats = 2 * maxw * T;
  a->one2[0] = a->one2[1] = 1.0f;
  *smem = (size_t)off * 4;
  return *smem <= 200 * 1024;
}

int exact_try_generic(const smlrt_model_s& m, const DevPlan& in, const Ptrs& src, const DevPlan& out, const Ptrs& dst,
                      bool /*all_f32*/, int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status,
                      bool probe_only, bool* done) {
  if (*done) return SMLRT_OK;
  GxArgs a{};
  size_t smem = 0;
  // 128 rows per CTA when it leaves room for two CTAs per SM, else 64
  int T = 0;
  if (gx_layout(m, 128, &a, &smem) && smem <= 100 * 1024)
    T = 128;
  else if (gx_layout(m, 64, &a, &smem))
    T = 64;
  if (T == 0) return SMLRT_OK;  // not handled: the unfused path runs
  *done = true;
  if (probe_only) return SMLRT_OK;
  return T == 128 ? gx_launch<128>(a, smem, in, src, out, dst, r0, r1, staged, s, status)
                  : gx_launch<64>(a, smem, in, src, out, dst, r0, r1, staged, s, status);
}

}  // namespace smlrt
