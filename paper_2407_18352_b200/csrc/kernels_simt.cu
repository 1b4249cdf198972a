// CUDA-core kernels of the region runtime (sm_100a):
//
//   gather_kernel       K1  compose_tensor / concretize_to (bridge.py:351-395)
//   scatter_kernel      K2  scatter_from's strided write + astype (bridge.py:450-454)
//   dense_exact_kernel  K3a one dense layer, reference accumulation order
//                           (_matmul_rowwise, models.py:188-194)
//   region_exact_kernel K1+K3a+K2 fused: gather -> MLP in registers -> scatter
//
// Exactness.  numpy's _matmul_rowwise computes, per output element,
//   acc = 0; for f in 0..in-1: acc = acc + (x[f] * w[j,f])    (f32, RN, no FMA)
// then y = acc + b[j], then relu = np.maximum(y, 0) (NaN propagates).  The
// kernels below use __fmul_rn/__fadd_rn in exactly that order, so relu and
// identity models are bitwise identical to the reference; tanh uses CUDA's
// tanhf (within 2 ulp, checked at tolerance, as the reference's own tests do).
#include <cuda_runtime.h>

#include "common.cuh"

namespace smlrt {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float load_as_f32(const void* base, int dtype, int64_t i) {
  return dtype == SMLRT_F32 ? __ldg(reinterpret_cast<const float*>(base) + i)
                            : __double2float_rn(__ldg(reinterpret_cast<const double*>(base) + i));
}

__device__ __forceinline__ double load_as_f64(const void* base, int dtype, int64_t i) {
  return dtype == SMLRT_F32 ? (double)__ldg(reinterpret_cast<const float*>(base) + i)
                            : __ldg(reinterpret_cast<const double*>(base) + i);
}

__device__ __forceinline__ void store_f32(void* base, int dtype, int64_t i, float v) {
  if (dtype == SMLRT_F32)
    reinterpret_cast<float*>(base)[i] = v;
  else
    reinterpret_cast<double*>(base)[i] = (double)v;
}

__device__ __forceinline__ void store_f64(void* base, int dtype, int64_t i, double v) {
  if (dtype == SMLRT_F32)
    reinterpret_cast<float*>(base)[i] = __double2float_rn(v);
  else
    reinterpret_cast<double*>(base)[i] = v;
}

__device__ __forceinline__ bool nonfinite(float v) {
  return (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
}

// np.maximum(y, 0): NaN wins; relu of a finite value is max(y, +0).
__device__ __forceinline__ float activate(float y, int act) {
  if (act == SMLRT_RELU) return (y < 0.0f) ? 0.0f : y;
  if (act == SMLRT_TANH) return tanhf(y);
  return y;
}

struct Ptrs {
  const void* p[8];
  int32_t dt[8];
};

__device__ __forceinline__ int64_t element_address(const DevPlan& P, uint32_t r, int c) {
  if (P.uniform) return P.col_off[c] + row_offset_uniform(P, r);
  uint32_t idx[SMLRT_MAX_SWEEP];
  unravel(P, r, idx);
  return col_address(P, c, idx);
}

// ---------------------------------------------------------------- gather --
// One thread per dense output element, linear over [rows x cols] so the
// stores are fully coalesced; reads follow the plan.
template <typename OutT>
__global__ void __launch_bounds__(kThreads) gather_kernel(const __grid_constant__ DevPlan P,
                                                          const __grid_constant__ Ptrs src, OutT* __restrict__ out,
                                                          int64_t r0, int64_t n_elem) {
  const FastDiv cdiv = P.cdiv;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_elem;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint32_t rr, c;
    if (n_elem < (1ll << 32)) {
      rr = cdiv.div((uint32_t)e);
      c = (uint32_t)e - rr * P.n_cols;
    } else {
      rr = (uint32_t)(e / P.n_cols);
      c = (uint32_t)(e - (int64_t)rr * P.n_cols);
    }
    uint32_t r = (uint32_t)(r0 + rr);
    int a = P.uniform ? P.uarray : P.col_arr[c];
    int64_t addr = element_address(P, r, c);
    if constexpr (sizeof(OutT) == 4)
      out[e] = load_as_f32(src.p[a], src.dt[a], addr);
    else
      out[e] = load_as_f64(src.p[a], src.dt[a], addr);
  }
}

// --------------------------------------------------------------- scatter --
template <typename InT>
__global__ void __launch_bounds__(kThreads) scatter_kernel(const __grid_constant__ DevPlan P,
                                                           const InT* __restrict__ in,
                                                           const __grid_constant__ Ptrs dst, int64_t r0, int64_t n_elem,
                                                           const uint32_t* gate) {
  if (gate != nullptr && *gate != 0u) return;  // COMMIT_CHECKED: nothing written on error
  const FastDiv cdiv = P.cdiv;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_elem;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint32_t rr, c;
    if (n_elem < (1ll << 32)) {
      rr = cdiv.div((uint32_t)e);
      c = (uint32_t)e - rr * P.n_cols;
    } else {
      rr = (uint32_t)(e / P.n_cols);
      c = (uint32_t)(e - (int64_t)rr * P.n_cols);
    }
    uint32_t r = (uint32_t)(r0 + rr);
    int a = P.uniform ? P.uarray : P.col_arr[c];
    int64_t addr = element_address(P, r, c);
    void* base = const_cast<void*>(dst.p[a]);
    if constexpr (sizeof(InT) == 4)
      store_f32(base, dst.dt[a], addr, in[e]);
    else
      store_f64(base, dst.dt[a], addr, in[e]);
  }
}

// ------------------------------------------------------ dense layer (exact) --
// Thread per (row, block of TJ outputs); weights are warp-uniform loads.
template <int TJ>
__global__ void __launch_bounds__(kThreads) dense_exact_kernel(const float* __restrict__ x, int64_t rows,
                                                               int in, int out,
                                                               const float* __restrict__ W,
                                                               const float* __restrict__ b, int act,
                                                               float* __restrict__ y,
                                                               uint32_t* status) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int j0 = blockIdx.y * TJ;
  bool bad = false;
  if (r < rows) {
    float acc[TJ];
#pragma unroll
    for (int u = 0; u < TJ; ++u) acc[u] = 0.0f;
    const float* xr = x + r * in;
    for (int f = 0; f < in; ++f) {
      float xf = xr[f];
#pragma unroll
      for (int u = 0; u < TJ; ++u)
        if (j0 + u < out) acc[u] = __fadd_rn(acc[u], __fmul_rn(xf, __ldg(W + (int64_t)(j0 + u) * in + f)));
    }
#pragma unroll
    for (int u = 0; u < TJ; ++u) {
      if (j0 + u < out) {
        float v = activate(__fadd_rn(acc[u], __ldg(b + j0 + u)), act);
        y[r * out + j0 + u] = v;
        bad |= nonfinite(v);
      }
    }
  }
  if (status != nullptr && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    atomicOr(status, SMLRT_STATUS_NONFINITE);
}

template <typename S, typename D>
__global__ void convert_kernel(const S* __restrict__ s, D* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (sizeof(S) == 8 && sizeof(D) == 4)
      d[i] = __double2float_rn(s[i]);
    else
      d[i] = (D)s[i];
  }
}

int grid_for(int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  int64_t cap = 148 * 16;  // 16 resident 256-thread CTAs' worth per SM, grid-stride beyond
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

Ptrs pack(const void* const* ptrs, const int32_t* dts, int n) {
  Ptrs p{};
  for (int i = 0; i < n && i < 8; ++i) {
    p.p[i] = ptrs[i];
    p.dt[i] = dts[i];
  }
  return p;
}

// ========================== fused exact region kernel ==========================
// The model's parameters travel in the kernel parameter bank (constant bank
// 0, <= 32 KB since CUDA 12.1), so every multiply reads its weight as a
// constant operand: 1 FMUL + 1 FADD per multiply-accumulate and no loads.
template <int... D>
struct Shape;

template <int A, int B>
struct Shape<A, B> {
  static constexpr int L = 1, IN = A, OUT = B, MAXW = (A > B ? A : B);
  static constexpr int NPARAM = A * B + B;
};
template <int A, int B, int C>
struct Shape<A, B, C> {
  static constexpr int L = 2, IN = A, OUT = C, MAXW = (A > B ? (A > C ? A : C) : (B > C ? B : C));
  static constexpr int NPARAM = A * B + B + B * C + C;
};
template <int A, int B, int C, int E>
struct Shape<A, B, C, E> {
  static constexpr int L = 3, IN = A, OUT = E;
  static constexpr int NPARAM = A * B + B + B * C + C + C * E + E;
};

template <int NP, int NL>
struct ModelParams {
  int act[NL];
  float w[NP];
};

template <int IN, int OUT>
__device__ __forceinline__ void layer_exact(const float (&x)[IN], float (&y)[OUT], const float* W,
                                            const float* b, int act) {
#pragma unroll
  for (int j = 0; j < OUT; ++j) {
    float acc = 0.0f;
#pragma unroll
    for (int f = 0; f < IN; ++f) acc = __fadd_rn(acc, __fmul_rn(x[f], W[j * IN + f]));
    y[j] = __fadd_rn(acc, b[j]);
  }
  // activation under one warp-uniform branch, so the matvec above exists once
  if (act == SMLRT_RELU) {
#pragma unroll
    for (int j = 0; j < OUT; ++j) y[j] = (y[j] < 0.0f) ? 0.0f : y[j];
  } else if (act == SMLRT_TANH) {
#pragma unroll
    for (int j = 0; j < OUT; ++j) y[j] = tanhf(y[j]);
  }
}

template <int A, int B>
__device__ __forceinline__ void forward(const ModelParams<Shape<A, B>::NPARAM, 1>& mp,
                                        const float (&x)[A], float (&y)[B]) {
  layer_exact<A, B>(x, y, mp.w, mp.w + A * B, mp.act[0]);
}
template <int A, int B, int C>
__device__ __forceinline__ void forward(const ModelParams<Shape<A, B, C>::NPARAM, 2>& mp,
                                        const float (&x)[A], float (&y)[C]) {
  float h[B];
  layer_exact<A, B>(x, h, mp.w, mp.w + A * B, mp.act[0]);
  constexpr int o = A * B + B;
  layer_exact<B, C>(h, y, mp.w + o, mp.w + o + B * C, mp.act[1]);
}
template <int A, int B, int C, int E>
__device__ __forceinline__ void forward(const ModelParams<Shape<A, B, C, E>::NPARAM, 3>& mp,
                                        const float (&x)[A], float (&y)[E]) {
  float h1[B], h2[C];
  layer_exact<A, B>(x, h1, mp.w, mp.w + A * B, mp.act[0]);
  constexpr int o1 = A * B + B;
  layer_exact<B, C>(h1, h2, mp.w + o1, mp.w + o1 + B * C, mp.act[1]);
  constexpr int o2 = o1 + B * C + C;
  layer_exact<C, E>(h2, y, mp.w + o2, mp.w + o2 + C * E, mp.act[2]);
}

template <bool F32, int IN>
__device__ __forceinline__ void load_row(const DevPlan& P, const Ptrs& src, uint32_t r, float (&x)[IN]) {
  if (P.uniform) {
    int64_t ro = row_offset_uniform(P, r);
    const void* base = src.p[P.uarray];
    int dt = src.dt[P.uarray];
#pragma unroll
    for (int f = 0; f < IN; ++f) {
      int64_t a = __ldg(P.col_off + f) + ro;
      x[f] = F32 ? __ldg(reinterpret_cast<const float*>(base) + a) : load_as_f32(base, dt, a);
    }
  } else {
    uint32_t idx[SMLRT_MAX_SWEEP];
    unravel(P, r, idx);
#pragma unroll
    for (int f = 0; f < IN; ++f) {
      int arr = __ldg(P.col_arr + f);
      x[f] = load_as_f32(src.p[arr], src.dt[arr], col_address(P, f, idx));
    }
  }
}

template <bool F32, class S, int... D>
__global__ void __launch_bounds__(128) region_exact_kernel(
    const ModelParams<S::NPARAM, S::L> mp, const __grid_constant__ DevPlan Pin,
    const __grid_constant__ Ptrs src, const __grid_constant__ DevPlan Pout,
    const __grid_constant__ Ptrs dst, int64_t r0, int64_t r1, float* __restrict__ staged, uint32_t* status) {
  int64_t row = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool bad = false;
  if (row < r1) {
    float x[S::IN], y[S::OUT];
    load_row<F32>(Pin, src, (uint32_t)row, x);
    forward<D...>(mp, x, y);
#pragma unroll
    for (int g = 0; g < S::OUT; ++g) bad |= nonfinite(y[g]);
    if (staged != nullptr) {
#pragma unroll
      for (int g = 0; g < S::OUT; ++g) staged[(row - r0) * S::OUT + g] = y[g];
    } else if (Pout.uniform) {
      int64_t ro = row_offset_uniform(Pout, (uint32_t)row);
      void* base = const_cast<void*>(dst.p[Pout.uarray]);
      int dt = dst.dt[Pout.uarray];
#pragma unroll
      for (int g = 0; g < S::OUT; ++g) {
        int64_t a = __ldg(Pout.col_off + g) + ro;
        if (F32)
          reinterpret_cast<float*>(base)[a] = y[g];
        else
          store_f32(base, dt, a, y[g]);
      }
    } else {
      uint32_t idx[SMLRT_MAX_SWEEP];
      unravel(Pout, (uint32_t)row, idx);
#pragma unroll
      for (int g = 0; g < S::OUT; ++g) {
        int arr = __ldg(Pout.col_arr + g);
        store_f32(const_cast<void*>(dst.p[arr]), dst.dt[arr], col_address(Pout, g, idx), y[g]);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(status, SMLRT_STATUS_NONFINITE);
}

template <int... D>
bool dims_match(const smlrt_model_s& m) {
  const int d[] = {D...};
  constexpr int n = sizeof...(D);
  if (m.n_layers != n - 1) return false;
  for (int l = 0; l < m.n_layers; ++l)
    if (m.layers[l].kind != SMLRT_DENSE || m.layers[l].in != d[l] || m.layers[l].out != d[l + 1]) return false;
  return true;
}

template <int... D>
int try_fused(const smlrt_model_s& m, const DevPlan& in, const Ptrs& src, const DevPlan& out,
              const Ptrs& dst, bool all_f32, int64_t r0, int64_t r1, float* staged, cudaStream_t s,
              uint32_t* status, bool probe_only, bool* done) {
  using S = Shape<D...>;
  if (*done || !dims_match<D...>(m)) return SMLRT_OK;
  *done = true;
  if (probe_only) return SMLRT_OK;
  ModelParams<S::NPARAM, S::L> mp;
  for (int l = 0; l < S::L; ++l) mp.act[l] = m.layers[l].act;
  for (int i = 0; i < S::NPARAM; ++i) mp.w[i] = m.host_params[i];
  int64_t n = r1 - r0;
  dim3 grid((unsigned)((n + 127) / 128));
  if (all_f32)
    region_exact_kernel<true, S, D...><<<grid, 128, 0, s>>>(mp, in, src, out, dst, r0, r1, staged, status);
  else
    region_exact_kernel<false, S, D...><<<grid, 128, 0, s>>>(mp, in, src, out, dst, r0, r1, staged, status);
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

}  // namespace

// ================================ launchers ================================

int launch_gather(const DevPlan& p, const void* const* ptrs, const int32_t* dtypes, int n_arrays,
                  void* out, int out_dtype, int64_t r0, int64_t r1, cudaStream_t s) {
  int64_t n = (r1 - r0) * (int64_t)p.n_cols;
  if (n <= 0) return SMLRT_OK;
  Ptrs src = pack(ptrs, dtypes, n_arrays);
  if (out_dtype == SMLRT_F32)
    gather_kernel<float><<<grid_for(n), kThreads, 0, s>>>(p, src, (float*)out, r0, n);
  else
    gather_kernel<double><<<grid_for(n), kThreads, 0, s>>>(p, src, (double*)out, r0, n);
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

int launch_scatter(const DevPlan& p, const void* in, int in_dtype, void* const* ptrs,
                   const int32_t* dtypes, int n_arrays, int64_t r0, int64_t r1, cudaStream_t s,
                   const uint32_t* gate) {
  int64_t n = (r1 - r0) * (int64_t)p.n_cols;
  if (n <= 0) return SMLRT_OK;
  Ptrs dst = pack((const void* const*)ptrs, dtypes, n_arrays);
  if (in_dtype == SMLRT_F32)
    scatter_kernel<float><<<grid_for(n), kThreads, 0, s>>>(p, (const float*)in, dst, r0, n, gate);
  else
    scatter_kernel<double><<<grid_for(n), kThreads, 0, s>>>(p, (const double*)in, dst, r0, n, gate);
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

int launch_dense_exact(const float* x, int64_t rows, const DevLayer& L, float* y, cudaStream_t s,
                       uint32_t* status) {
  if (rows <= 0) return SMLRT_OK;
  constexpr int TJ = 8;
  dim3 grid((unsigned)((rows + kThreads - 1) / kThreads), (unsigned)((L.out + TJ - 1) / TJ));
  dense_exact_kernel<TJ><<<grid, kThreads, 0, s>>>(x, rows, L.in, L.out, L.w, L.b, L.act, y, status);
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

int launch_convert(const void* src, int sdt, void* dst, int ddt, int64_t n, cudaStream_t s) {
  if (n <= 0) return SMLRT_OK;
  if (sdt == ddt) {
    SMLRT_CUDA(cudaMemcpyAsync(dst, src, n * (sdt == SMLRT_F32 ? 4 : 8), cudaMemcpyDeviceToDevice, s));
    return SMLRT_OK;
  }
  if (sdt == SMLRT_F64)
    convert_kernel<double, float><<<grid_for(n), kThreads, 0, s>>>((const double*)src, (float*)dst, n);
  else
    convert_kernel<float, double><<<grid_for(n), kThreads, 0, s>>>((const float*)src, (double*)dst, n);
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

int launch_region_exact_fused(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs,
                              const int32_t* in_dt, int n_in, const DevPlan& out,
                              void* const* out_ptrs, const int32_t* out_dt, int n_out, int64_t r0,
                              int64_t r1, float* staged, cudaStream_t s, uint32_t* status,
                              bool probe_only) {
  if (n_in > 8 || n_out > 8) return SMLRT_E_UNSUPPORTED;
  Ptrs src = pack(in_ptrs, in_dt, n_in);
  Ptrs dst = pack((const void* const*)out_ptrs, out_dt, n_out);
  bool all_f32 = true;
  for (int i = 0; i < n_in; ++i) all_f32 &= in_dt[i] == SMLRT_F32;
  for (int i = 0; i < n_out; ++i) all_f32 &= out_dt[i] == SMLRT_F32;
  bool done = false;
  int rc = SMLRT_OK;
#define SMLRT_TRY(...)                                                                          \
  if ((rc = try_fused<__VA_ARGS__>(m, in, src, out, dst, all_f32, r0, r1, staged, s, status, \
                                   probe_only, &done)) != SMLRT_OK)                            \
    return rc;
  // Instantiated shapes: the frozen configs' exact-fp32 models and the
  // reference's analytic models (jacobi/strike 5->1, identity 5->5).
  SMLRT_TRY(5, 64, 32, 1)   // C1 Binomial Options
  SMLRT_TRY(36, 8, 4)       // C5 MiniWeather 3x3x4 halo -> 8 -> 4
  SMLRT_TRY(5, 1)           // jacobi_model / "price = strike"
  SMLRT_TRY(5, 5)           // model_identity5 fixture
  SMLRT_TRY(64, 8)          // C4 conv1 as a patch MLP
#undef SMLRT_TRY
  return done ? SMLRT_OK : SMLRT_E_UNSUPPORTED;
}

}  // namespace smlrt
