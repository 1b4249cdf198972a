// Shared definitions of libsmlrt_b200: host plan/model objects, the device
// plan descriptor passed by value to every kernel, fast integer division for
// sweep unravelling, and error plumbing.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/smlrt_b200.h"

namespace smlrt {

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
#define SMLRT_CUDA(call)                                                     \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                   \
      return ::smlrt::fail(SMLRT_E_CUDA, std::string(#call) + ": " +         \
                                             cudaGetErrorString(e_));        \
  } while (0)

// ------------------------------------------------------- fast division --
// Unsigned 32-bit division by a runtime-invariant divisor (Granlund-Montgomery
// round-up variant): q = (umulhi(n, m) + n) >> s, exact for every n < 2^32.
struct FastDiv {
  uint32_t d, m, s;
  __host__ __device__ FastDiv() : d(1), m(0), s(0) {}
  __host__ __device__ explicit FastDiv(uint32_t div) : d(div) {
    s = 0;
    while ((1ull << s) < div) ++s;
    m = (uint32_t)((((1ull << s) - div) << 32) / div + 1);
  }
  __host__ __device__ __forceinline__ uint32_t div(uint32_t n) const {
#ifdef __CUDA_ARCH__
    uint32_t hi = __umulhi(n, m);
#else
    uint32_t hi = (uint32_t)(((uint64_t)n * m) >> 32);
#endif
    return (uint32_t)(((uint64_t)hi + n) >> s);
  }
};

// -------------------------------------------------- device plan (by value) --
// Address of (row r, column c) = col_off[c] + sum_k idx_k(r) * stride(c, k),
// idx = row-major unravel of r over the sweep shape.  For "uniform" plans all
// columns share `ustride`, so the row part is computed once per row.
constexpr int SMLRT_INLINE_COLS = 64;

struct DevPlan {
  int32_t n_sweep;
  int32_t n_cols;
  int32_t uniform;
  int32_t all_f32;          // filled at launch from the dtypes
  int64_t n_rows;
  int64_t ustride[SMLRT_MAX_SWEEP];
  FastDiv sdiv[SMLRT_MAX_SWEEP];  // sweep extents
  FastDiv cdiv;                   // n_cols
  const int64_t* col_off;   // [n_cols]
  const int32_t* col_arr;   // [n_cols] array index
  const int64_t* col_str;   // [n_cols * n_sweep] (non-uniform plans)
  int32_t uarray;           // uniform: the single array index
  int32_t dense_rows;       // uniform, 1-D sweep, columns one contiguous run
  int64_t col_off0;         // col_off[0] (host copy, for launch-time decisions)
  int32_t win_w;            // >0: columns form a 2-D window of rows of win_w
  int64_t win_pitch;        //     elements at this pitch (uniform plans)
  int64_t uarray_numel;     // uniform: elements of the single array (plan-time extent)
  int64_t col_inl[SMLRT_INLINE_COLS];  // col_off copy in the parameter bank (n_cols <= SMLRT_INLINE_COLS)
};

__host__ __device__ __forceinline__ int64_t row_offset_uniform(const DevPlan& p, uint32_t r) {
  int64_t off = 0;
#pragma unroll
  for (int k = SMLRT_MAX_SWEEP - 1; k >= 0; --k) {
    if (k < p.n_sweep) {
      uint32_t q = p.sdiv[k].div(r);
      uint32_t i = r - q * p.sdiv[k].d;
      off += (int64_t)i * p.ustride[k];
      r = q;
    }
  }
  return off;
}

// per-row multi-index (non-uniform plans combine it with each column's strides)
__device__ __forceinline__ void unravel(const DevPlan& p, uint32_t r, uint32_t* idx) {
#pragma unroll
  for (int k = SMLRT_MAX_SWEEP - 1; k >= 0; --k) {
    if (k < p.n_sweep) {
      uint32_t q = p.sdiv[k].div(r);
      idx[k] = r - q * p.sdiv[k].d;
      r = q;
    } else {
      idx[k] = 0;
    }
  }
}

__device__ __forceinline__ int64_t col_address(const DevPlan& p, int c, const uint32_t* idx) {
  int64_t a = p.col_off[c];
  const int64_t* s = p.col_str + (int64_t)c * p.n_sweep;
  for (int k = 0; k < p.n_sweep; ++k) a += (int64_t)idx[k] * s[k];
  return a;
}

// ------------------------------------------------------------ host plan --
struct DeviceTables {
  int64_t* col_off = nullptr;
  int32_t* col_arr = nullptr;
  int64_t* col_str = nullptr;
};

}  // namespace smlrt

struct smlrt_plan_s {
  int direction = 0;
  int n_sweep = 0;
  int64_t sweep[SMLRT_MAX_SWEEP] = {0};
  int64_t n_rows = 0;
  int n_arrays = 0;
  int n_cols = 0;
  std::vector<smlrt_view_t> views;
  std::vector<int64_t> array_numel;  // storage extents the plan was validated against
  std::vector<int64_t> col_off;
  std::vector<int32_t> col_arr;
  std::vector<int64_t> col_str;  // n_cols * n_sweep
  bool uniform = false;
  int uarray = 0;
  int64_t ustride[SMLRT_MAX_SWEEP] = {0};
  bool dense_rows = false;
  int64_t row_pitch = 0;
  bool injective = false;
  int win_w = 0;
  int64_t win_pitch = 0;
  std::mutex mu;
  std::map<int, smlrt::DeviceTables> dev;
  ~smlrt_plan_s();
  // device tables for the current device (uploads once)
  int tables(smlrt::DevPlan* out);
};

namespace smlrt {

// Raise the non-finite bit of a status word: a plain store (every writer
// stores the same bit, no read-modify-write needed), so the word may also live
// in mapped host memory (the synchronous call's zero-copy status flag).
__device__ __forceinline__ void flag_nonfinite(uint32_t* status) {
  *reinterpret_cast<volatile uint32_t*>(status) = SMLRT_STATUS_NONFINITE;
}

// kernels launched by this library since load (smlrt_launch_count): the bench
// reports how many of its own launches a timed region made
extern std::atomic<unsigned long long> g_launches;
inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// one dense layer on the device
struct DevLayer {
  int kind = SMLRT_DENSE;
  int in, out, act;
  int kernel = 0, stride = 0, in_c = 0, in_h = 0, in_w = 0, out_c = 0;
  float* w = nullptr;       // f32 [out][in]
  float* b = nullptr;       // f32 [out]
  void* w_bf16 = nullptr;   // bf16 weights in the tcgen05 operand layout
};

}  // namespace smlrt

struct smlrt_model_s {
  int precision = 0;
  int device = 0;
  int n_layers = 0;
  int in_features = 0, out_features = 0, max_width = 0;
  std::vector<smlrt::DevLayer> layers;
  std::vector<float> host_params;  // packed [W0,b0,W1,b1,...] for the templated path
  void* tc_blob = nullptr;          // tcgen05 path: packed bf16 weights + f32 bias
  size_t tc_bytes = 0;
  // generic tcgen05 layer chain (any dense model): per layer the bf16 weights
  // [n_pad x k_pad] (K-major, zero padded) and f32 bias [n_pad] in chain_blob
  struct ChainLayer {
    int k_pad, n_pad, n, act;
    size_t w_off, b_off;  // byte offsets in chain_blob
  };
  std::vector<ChainLayer> chain;
  void* chain_blob = nullptr;
  int chain_first = -1;  // model layer the chain starts at (CNN: the first dense layer)
  // small-MLP warp-MMA kernel (small_mma.cu): per-lane B fragments + biases
  void* smm_blob = nullptr;
  // small-MLP tcgen05 kernel (small_tc.cu): swizzled tf32 W1 / bf16 W2, W3 images
  void* stc_blob = nullptr;
  std::vector<float> stc_epi;  // [b2 (64) | b3 (8)] for the kernel parameters
  ~smlrt_model_s();
};

namespace smlrt {

// kernel entry points (kernels_simt.cu / mlp_tc.cu)
int launch_gather(const DevPlan& p, const void* const* ptrs, const int32_t* dtypes, int n_arrays,
                  void* out, int out_dtype, int64_t r0, int64_t r1, cudaStream_t s);
int launch_scatter(const DevPlan& p, const void* in, int in_dtype, void* const* ptrs,
                   const int32_t* dtypes, int n_arrays, int64_t r0, int64_t r1, cudaStream_t s,
                   const uint32_t* gate_status);
int launch_dense_exact(const float* x, int64_t rows, const DevLayer& L, float* y,
                       cudaStream_t s, uint32_t* status_if_last);
int launch_convert(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n,
                   cudaStream_t s);
// fused exact region: returns SMLRT_E_UNSUPPORTED if no instantiation fits
int launch_region_exact_fused(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs,
                              const int32_t* in_dt, int n_in, const DevPlan& out,
                              void* const* out_ptrs, const int32_t* out_dt, int n_out,
                              int64_t r0, int64_t r1, float* staged, cudaStream_t s,
                              uint32_t* status, bool probe_only);
// 1: a templated fused instantiation, 6: the runtime-dims fused kernel, 0: unfused
int exact_fused_kind(const smlrt_model_s& m);
// conv2d(+maxpool2d) front + exact dense tail (cnn_exact.cu)
bool cnn_model(const smlrt_model_s& m);
int launch_region_cnn(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs, const int32_t* in_dt,
                      int n_in, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt, int n_out,
                      int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status);
int infer_cnn_dense(const smlrt_model_s& m, const float* x, int64_t rows, float* y, cudaStream_t s,
                    uint32_t* status);
int launch_dense_exact_tiled(const float* x, int64_t rows, const DevLayer& L, float* y, cudaStream_t s,
                             uint32_t* status);
int launch_region_tc(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs,
                     const int32_t* in_dt, int n_in, const DevPlan& out, void* const* out_ptrs,
                     const int32_t* out_dt, int n_out, int64_t r0, int64_t r1, float* staged,
                     cudaStream_t s, uint32_t* status, bool probe_only);
int tc_pack_model(smlrt_model_s& m);
// wide 4-layer MLPs (gemm_tc.cu): TMA-fed tcgen05 GEMM chain
bool wide_shape(const smlrt_model_s& m);
int wide_pack(smlrt_model_s& m);
int launch_region_wide(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs, const int32_t* in_dt,
                       const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt, int n_out, int64_t r0,
                       int64_t r1, float* staged, cudaStream_t s, uint32_t* status);
// bf16 halo-stencil regions on tcgen05 (stencil_tc.cu); SMLRT_E_UNSUPPORTED if not that shape
int small_mma_pack(smlrt_model_s& m);
int small_tc_pack(smlrt_model_s& m, int n1, int n2);
int launch_region_small_tc(const smlrt_model_s& m, const DevPlan& in, const void* src, const DevPlan& out, void* dst,
                           int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status);
int launch_region_small_mma(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs,
                            const int32_t* in_dt, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt,
                            int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status);
int launch_region_stencil_exact(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs,
                                const int32_t* in_dt, const DevPlan& out, void* const* out_ptrs,
                                const int32_t* out_dt, int64_t r0, int64_t r1, float* staged, cudaStream_t s,
                                uint32_t* status);
int launch_region_stencil_tc(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs,
                             const int32_t* in_dt, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt,
                             int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status);
// generic tcgen05 layer chain (gemm_tc.cu): any dense model, any plans
bool chain_ok(const smlrt_model_s& m);
int chain_first_layer(const smlrt_model_s& m);
int chain_pack(smlrt_model_s& m);
int chain_max_width(const smlrt_model_s& m);
int chain_forward(const smlrt_model_s& m, __nv_bfloat16* act0, __nv_bfloat16* act1, int64_t n, float* y,
                  uint32_t* status, cudaStream_t s);
int launch_region_chain(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs, const int32_t* in_dt,
                        int n_in, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt, int n_out,
                        int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status);

}  // namespace smlrt
