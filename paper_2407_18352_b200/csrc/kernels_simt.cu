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

#include <cstring>
#include <type_traits>

#include "exact_region.cuh"


namespace smlrt {
namespace {

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

// Uniform plans: one thread per row -- one row offset per row instead of one
// unravel per element, column offsets from the parameter bank; the staged
// row is read contiguously and every column's stores are coalesced across
// the warp (the checked commit's scatter of C5's 4-plane output).
template <typename InT>
__global__ void __launch_bounds__(kThreads) scatter_rows_kernel(const __grid_constant__ DevPlan P,
                                                                const InT* __restrict__ in,
                                                                const __grid_constant__ Ptrs dst, int64_t r0,
                                                                int64_t rows, const uint32_t* gate) {
  if (gate != nullptr && *gate != 0u) return;
  const int G = P.n_cols;
  void* base = const_cast<void*>(dst.p[P.uarray]);
  const int dt = dst.dt[P.uarray];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ro = row_offset_uniform(P, (uint32_t)(r0 + i));
    const InT* v = in + i * G;
    for (int c = 0; c < G; ++c) {
      if constexpr (sizeof(InT) == 4)
        store_f32(base, dt, P.col_inl[c] + ro, v[c]);
      else
        store_f64(base, dt, P.col_inl[c] + ro, v[c]);
    }
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
    flag_nonfinite(status);
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
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

int launch_scatter(const DevPlan& p, const void* in, int in_dtype, void* const* ptrs,
                   const int32_t* dtypes, int n_arrays, int64_t r0, int64_t r1, cudaStream_t s,
                   const uint32_t* gate) {
  int64_t n = (r1 - r0) * (int64_t)p.n_cols;
  if (n <= 0) return SMLRT_OK;
  Ptrs dst = pack((const void* const*)ptrs, dtypes, n_arrays);
  if (p.uniform && p.n_cols <= SMLRT_INLINE_COLS) {
    const int64_t rows = r1 - r0;
    if (in_dtype == SMLRT_F32)
      scatter_rows_kernel<float><<<grid_for(rows), kThreads, 0, s>>>(p, (const float*)in, dst, r0, rows, gate);
    else
      scatter_rows_kernel<double><<<grid_for(rows), kThreads, 0, s>>>(p, (const double*)in, dst, r0, rows, gate);
  } else if (in_dtype == SMLRT_F32)
    scatter_kernel<float><<<grid_for(n), kThreads, 0, s>>>(p, (const float*)in, dst, r0, n, gate);
  else
    scatter_kernel<double><<<grid_for(n), kThreads, 0, s>>>(p, (const double*)in, dst, r0, n, gate);
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

int launch_dense_exact(const float* x, int64_t rows, const DevLayer& L, float* y, cudaStream_t s,
                       uint32_t* status) {
  if (rows <= 0) return SMLRT_OK;
  constexpr int TJ = 8;
  dim3 grid((unsigned)((rows + kThreads - 1) / kThreads), (unsigned)((L.out + TJ - 1) / TJ));
  dense_exact_kernel<TJ><<<grid, kThreads, 0, s>>>(x, rows, L.in, L.out, L.w, L.b, L.act, y, status);
  count_launch();
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
  count_launch();
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
  // Instantiated shapes (one translation unit each): the frozen configs'
  // exact-fp32 models and the reference's analytic models.
  for (ExactTryFn fn : {exact_try_c1, exact_try_c5, exact_try_small, exact_try_generic})
    if ((rc = fn(m, in, src, out, dst, all_f32, r0, r1, staged, s, status, probe_only, &done)) != SMLRT_OK || done)
      return rc;
  return done ? SMLRT_OK : SMLRT_E_UNSUPPORTED;
}

int exact_fused_kind(const smlrt_model_s& m) {
  DevPlan d{};
  Ptrs p{};
  bool done = false;
  for (ExactTryFn fn : {exact_try_c1, exact_try_c5, exact_try_small})
    if (fn(m, d, p, d, p, true, 0, 0, nullptr, nullptr, nullptr, true, &done) == SMLRT_OK && done) return 1;
  if (exact_try_generic(m, d, p, d, p, true, 0, 0, nullptr, nullptr, nullptr, true, &done) == SMLRT_OK && done)
    return 6;
  return 0;
}

}  // namespace smlrt
