// Fused exact-fp32 region kernel (gather -> MLP -> scatter), templated on
// the model shape; see kernels_simt.cu's header comment for the exactness
// argument.  Included by exact_c1.cu / exact_c5.cu / exact_small.cu.
#pragma once

#include <cstring>
#include <type_traits>

#include "simt_common.cuh"

#ifndef SMLRT_OPT_UNR
#define SMLRT_OPT_UNR 8
#endif

namespace smlrt {
namespace {

// ========================== fused exact region kernel ==========================
// The model's parameters travel in the kernel parameter bank (constant bank
// 0, <= 32 KB since CUDA 12.1), packed on the host in the order the unrolled
// forward pass consumes them and 16-byte aligned, so the compiler fetches
// four weights per LDCU.128 into uniform registers (one per warp) and every
// multiply-accumulate is 1 FMUL + 1 FADD with a uniform-register operand.
// Scalar (unaligned, strided) weight fetches cost one LDCU per multiply and
// made the kernel MIO-bound (short-scoreboard stalls).
constexpr int r4(int n) { return (n + 3) & ~3; }

template <int... D>
struct Shape;

// 1 layer: W [B][r4(A)] row-major (rows padded), b [r4(B)]
template <int A, int B>
struct Shape<A, B> {
  static constexpr int L = 1, IN = A, OUT = B;
  static constexpr int SW = r4(A), OB = B * SW;
  static constexpr int NPARAM = OB + r4(B);
};
// 2 layers, streamed over a row pair: P1[f/2] = {(W1[f][i], W1[f+1][i]) for
// i < A, (b1[f], b1[f+1])} -- hidden-unit pairs for output-paired f32x2 ops --
// padded to S1 = r4(2(A+1));
// P2[f] = {W2[0..C)[f]} (a column of W2, output-paired) padded to S2 = r4(C);
// b2 [r4(C)]
template <int A, int B, int C>
struct Shape<A, B, C> {
  static constexpr int L = 2, IN = A, OUT = C;
  static constexpr int S1 = r4(2 * (A + 1)), S2 = r4(C);
  static constexpr int O2 = (B / 2) * S1, OB2 = O2 + B * S2;
  static constexpr int NPARAM = OB2 + r4(C);
};
// 3 layers: as above, then W3 [E][r4(C)] row-major, b3 [r4(E)]
template <int A, int B, int C, int E>
struct Shape<A, B, C, E> {
  static constexpr int L = 3, IN = A, OUT = E;
  static constexpr int S1 = r4(2 * (A + 1)), S2 = r4(C), S3 = r4(C);
  static constexpr int O2 = (B / 2) * S1, OB2 = O2 + B * S2, O3 = OB2 + r4(C), OB3 = O3 + E * S3;
  static constexpr int NPARAM = OB3 + r4(E);
};

template <int NP, int NL>
struct alignas(16) ModelParams {
  float w[NP];
  uint64_t one2;  // (1.0f, 1.0f): opaque to ptxas, see add2()
  int act[NL];
};

// ---- packed f32x2 arithmetic (sm_100 FMUL2 / FFMA2), bitwise IEEE RN ----
// ptxas contracts mul.rn.f32x2 followed by add.rn.f32x2 into FFMA2 (even with
// --fmad=false), which would change the rounding.  The add is therefore
// written as fma(p, one, acc) with `one` = (1, 1) read from the parameter
// bank: RN(p*1 + acc) == RN(p + acc) exactly (also for signed zeros, NaN and
// infinities), and ptxas cannot fold a multiply into it.
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t add2(uint64_t acc, uint64_t p, uint64_t one) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(p), "l"(one), "l"(acc));
  return r;
}
__device__ __forceinline__ uint64_t ldw2(const float* w) { return *reinterpret_cast<const uint64_t*>(w); }
__device__ __forceinline__ ulonglong2 ldw4(const float* w) { return *reinterpret_cast<const ulonglong2*>(w); }

// y[j] = act(ordered dot(x, W[j, :]) + b[j]); W rows at stride SW
template <int IN, int OUT, int SW>
__device__ __forceinline__ void layer_exact(const float (&x)[IN], float (&y)[OUT], const float* W,
                                            const float* b, int act) {
#pragma unroll
  for (int j = 0; j < OUT; ++j) {
    float acc = 0.0f;
#pragma unroll
    for (int f = 0; f < IN; ++f) acc = __fadd_rn(acc, __fmul_rn(x[f], W[j * SW + f]));
    y[j] = __fadd_rn(acc, b[j]);
  }
  // activation under one warp-uniform branch, so the matvec above exists once
  if (act == SMLRT_RELU) {
#pragma unroll
    for (int j = 0; j < OUT; ++j) y[j] = relu_exact(y[j]);
  } else if (act == SMLRT_TANH) {
#pragma unroll
    for (int j = 0; j < OUT; ++j) y[j] = tanhf(y[j]);
  }
}

template <int ACT>
__device__ __forceinline__ float act_c(float y) {
  if constexpr (ACT == SMLRT_RELU) return relu_exact(y);
  else if constexpr (ACT == SMLRT_TANH) return tanhf(y);
  else return y;
}

// Layers 1 and 2 streamed: hidden unit f of layer 1 is finished (ordered dot,
// + b1[f], act1) and immediately folded into every layer-2 accumulator,
// acc[j] = acc[j] + h_f * W2[j, f] in ascending f -- the same operation
// sequence per output as _matmul_rowwise (models.py:188-194), so bitwise equal,
// but only the C accumulators (not all B hidden values) are live: ~4x fewer
// registers than materialising h1, hence 4x the resident warps.
//
// Two rows (a, b) per thread share every instruction: layer 1 runs on row
// pairs (x_a[i], x_b[i]) x (w, w) with duplicated weights; layer 2 on output
// pairs (h, h) x (W2[j, f], W2[j+1, f]).  Each FMUL2/FFMA2 does the work of
// two FMUL/FADD, halving the issue slots of the (issue-bound) kernel.
template <int ACT1, int A, int B, int C, int S1, int S2, int UNR, int R>
__device__ __forceinline__ void layers12_streamed(const float* P1, const float* P2, const float* b2, int act2,
                                                  uint64_t one, const float (&x)[R][A], float (&y)[R][C]) {
  static_assert(C % 2 == 0 && B % 2 == 0, "output-paired layers need even widths");
  uint64_t acc[R][C / 2];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < C / 2; ++j) acc[r][j] = 0ull;
  // partial unroll keeps the loop body inside the instruction cache (a fully
  // unrolled 5-64-32 body stalls on instruction fetch); fp stays warp-uniform,
  // so the weights are still fetched as uniform LDCU.128s
#pragma unroll (UNR / 2 > 0 ? UNR / 2 : 1)
  for (int fp = 0; fp < B / 2; ++fp) {
    // layer 1 for hidden units (2fp, 2fp+1): (x, x) * (W1[2fp][i], W1[2fp+1][i]);
    // explicit 16-byte weight fetches (the compiler cannot prove the alignment
    // of P1 + fp * S1 under the partial unroll and would issue 8-byte LDCUs)
    uint64_t w1[S1 / 2];
#pragma unroll
    for (int i = 0; i < S1 / 4; ++i) {
      const ulonglong2 q = ldw4(P1 + fp * S1 + 4 * i);
      w1[2 * i] = q.x;
      w1[2 * i + 1] = q.y;
    }
    float h[R][2];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      uint64_t hp = 0ull;
#pragma unroll
      for (int i = 0; i < A; ++i) hp = add2(hp, mul2(pk2(x[r][i], x[r][i]), w1[i]), one);
      hp = add2(hp, w1[A], one);  // + (b1[2fp], b1[2fp+1])
      upk2(hp, h[r][0], h[r][1]);
      h[r][0] = act_c<ACT1>(h[r][0]);
      h[r][1] = act_c<ACT1>(h[r][1]);
    }
    // layer 2, output pairs, hidden units in ascending order
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int f = 2 * fp + u;
#pragma unroll
      for (int j = 0; j < C / 2; ++j) {
        const ulonglong2 q = ldw4(P2 + f * S2 + 4 * (j / 2));
        const uint64_t w = (j & 1) ? q.y : q.x;
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r][j] = add2(acc[r][j], mul2(pk2(h[r][u], h[r][u]), w), one);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < C / 2; ++j) {
      float lo, hi;
      upk2(add2(acc[r][j], ldw2(b2 + 2 * j), one), lo, hi);  // acc + b2
      y[r][2 * j] = activate(lo, act2);
      y[r][2 * j + 1] = activate(hi, act2);
    }
}

// Input-outer order for narrow hidden layers (C5: 36-8-4): for each input i
// the B/2 hidden-pair accumulators advance together, so only x and B/2 packed
// accumulators are live (not a hidden pair's whole weight row) -- fewer
// registers, more resident warps.  Per hidden unit the operation sequence is
// unchanged (i ascending, bias last; layer 2 f ascending): bitwise identical
// to layers12_streamed.
template <int ACT1, int A, int B, int C, int S1, int S2, int R>
__device__ __forceinline__ void layers12_io(const float* P1, const float* P2, const float* b2, int act2,
                                            uint64_t one, const float (&x)[R][A], float (&y)[R][C]) {
  static_assert(C % 2 == 0 && B % 2 == 0, "output-paired layers need even widths");
  uint64_t hp[R][B / 2];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int p = 0; p < B / 2; ++p) hp[r][p] = 0ull;
#pragma unroll
  for (int i = 0; i < A; ++i)
#pragma unroll
    for (int p = 0; p < B / 2; ++p) {
      const uint64_t w = ldw2(P1 + p * S1 + 2 * i);
#pragma unroll
      for (int r = 0; r < R; ++r) hp[r][p] = add2(hp[r][p], mul2(pk2(x[r][i], x[r][i]), w), one);
    }
  float h[R][B];
#pragma unroll
  for (int p = 0; p < B / 2; ++p) {
    const uint64_t bb = ldw2(P1 + p * S1 + 2 * A);  // (b1[2p], b1[2p+1])
#pragma unroll
    for (int r = 0; r < R; ++r) {
      upk2(add2(hp[r][p], bb, one), h[r][2 * p], h[r][2 * p + 1]);
      h[r][2 * p] = act_c<ACT1>(h[r][2 * p]);
      h[r][2 * p + 1] = act_c<ACT1>(h[r][2 * p + 1]);
    }
  }
  uint64_t acc[R][C / 2];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < C / 2; ++j) acc[r][j] = 0ull;
#pragma unroll
  for (int f = 0; f < B; ++f)
#pragma unroll
    for (int j = 0; j < C / 2; ++j) {
      const uint64_t w = ldw2(P2 + f * S2 + 2 * j);
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r][j] = add2(acc[r][j], mul2(pk2(h[r][f], h[r][f]), w), one);
    }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < C / 2; ++j) {
      float lo, hi;
      upk2(add2(acc[r][j], ldw2(b2 + 2 * j), one), lo, hi);
      y[r][2 * j] = activate(lo, act2);
      y[r][2 * j + 1] = activate(hi, act2);
    }
}

template <int A, int B, int C>
constexpr bool io_order();

template <int ACT1, int R, int UNR, int A, int B>
__device__ __forceinline__ void forward(const ModelParams<Shape<A, B>::NPARAM, 1>& mp,
                                        const float (&x)[R][A], float (&y)[R][B]) {
  using S = Shape<A, B>;
#pragma unroll
  for (int r = 0; r < R; ++r) layer_exact<A, B, S::SW>(x[r], y[r], mp.w, mp.w + S::OB, mp.act[0]);
}
template <int ACT1, int R, int UNR, int A, int B, int C>
__device__ __forceinline__ void forward(const ModelParams<Shape<A, B, C>::NPARAM, 2>& mp,
                                        const float (&x)[R][A], float (&y)[R][C]) {
  using S = Shape<A, B, C>;
  if constexpr (io_order<A, B, C>())
    layers12_io<ACT1, A, B, C, S::S1, S::S2, R>(mp.w, mp.w + S::O2, mp.w + S::OB2, mp.act[1], mp.one2, x, y);
  else
    layers12_streamed<ACT1, A, B, C, S::S1, S::S2, UNR, R>(mp.w, mp.w + S::O2, mp.w + S::OB2, mp.act[1], mp.one2, x,
                                                           y);
}
template <int ACT1, int R, int UNR, int A, int B, int C, int E>
__device__ __forceinline__ void forward(const ModelParams<Shape<A, B, C, E>::NPARAM, 3>& mp,
                                        const float (&x)[R][A], float (&y)[R][E]) {
  using S = Shape<A, B, C, E>;
  float h2[R][C];
  layers12_streamed<ACT1, A, B, C, S::S1, S::S2, UNR, R>(mp.w, mp.w + S::O2, mp.w + S::OB2, mp.act[1], mp.one2, x,
                                                         h2);
#pragma unroll
  for (int r = 0; r < R; ++r) layer_exact<C, E, S::S3>(h2[r], y[r], mp.w + S::O3, mp.w + S::OB3, mp.act[2]);
}

// host: model.host_params ([W (out x in), b] per layer, row-major) -> the
// packed use-order layout above
template <int A, int B>
void pack_params(const float* hp, float* w, Shape<A, B>*) {
  using S = Shape<A, B>;
  for (int j = 0; j < B; ++j)
    for (int f = 0; f < A; ++f) w[j * S::SW + f] = hp[j * A + f];
  for (int j = 0; j < B; ++j) w[S::OB + j] = hp[A * B + j];
}
template <int A, int B, int C>
void pack12(const float* hp, float* w, int S1, int S2, int O2, int OB2) {
  const float *W1 = hp, *b1 = W1 + A * B, *W2 = b1 + B, *b2 = W2 + B * C;
  for (int f = 0; f < B; ++f) {
    const int fp = f / 2, u = f % 2;  // hidden-unit pair, slot within the pair
    for (int i = 0; i < A; ++i) w[fp * S1 + 2 * i + u] = W1[f * A + i];
    w[fp * S1 + 2 * A + u] = b1[f];
    for (int j = 0; j < C; ++j) w[O2 + f * S2 + j] = W2[j * B + f];
  }
  for (int j = 0; j < C; ++j) w[OB2 + j] = b2[j];
}
template <int A, int B, int C>
void pack_params(const float* hp, float* w, Shape<A, B, C>*) {
  using S = Shape<A, B, C>;
  pack12<A, B, C>(hp, w, S::S1, S::S2, S::O2, S::OB2);
}
template <int A, int B, int C, int E>
void pack_params(const float* hp, float* w, Shape<A, B, C, E>*) {
  using S = Shape<A, B, C, E>;
  pack12<A, B, C>(hp, w, S::S1, S::S2, S::O2, S::OB2);
  const float *W3 = hp + A * B + B + B * C + C, *b3 = W3 + C * E;
  for (int j = 0; j < E; ++j)
    for (int f = 0; f < C; ++f) w[S::O3 + j * S::S3 + f] = W3[j * C + f];
  for (int j = 0; j < E; ++j) w[S::OB3 + j] = b3[j];
}

// RUN > 1 (f32 uniform plans whose columns come in contiguous runs of RUN
// elements, checked at launch): one 64-bit address per run, the run's
// elements at immediate offsets -- the halo gather's address arithmetic
// otherwise outweighs its loads.
template <bool F32, int RUN, int IN>
__device__ __forceinline__ void load_row(const DevPlan& P, const Ptrs& src, uint32_t r, float (&x)[IN]) {
  if (P.uniform) {
    int64_t ro = row_offset_uniform(P, r);
    const void* base = src.p[P.uarray];
    if constexpr (F32 && RUN > 1 && IN <= SMLRT_INLINE_COLS && IN % RUN == 0) {
      const float* pr = reinterpret_cast<const float*>(base) + ro;
#pragma unroll
      for (int g = 0; g < IN / RUN; ++g) {
        const float* q = pr + P.col_inl[g * RUN];
#pragma unroll
        for (int k = 0; k < RUN; ++k) x[g * RUN + k] = __ldg(q + k);
      }
      return;
    }
    int dt = src.dt[P.uarray];
#pragma unroll
    for (int f = 0; f < IN; ++f) {
      int64_t a = (IN <= SMLRT_INLINE_COLS ? P.col_inl[f] : __ldg(P.col_off + f)) + ro;
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

// columns of a uniform plan form contiguous runs of `run` elements
inline bool plan_runs(const DevPlan& P, int run) {
  if (!P.uniform || P.n_cols > SMLRT_INLINE_COLS || P.n_cols % run != 0) return false;
  for (int c = 0; c < P.n_cols; ++c)
    if (P.col_inl[c] != P.col_inl[c - c % run] + c % run) return false;
  return true;
}

template <int... D>
struct Tune {
  static constexpr int R = 1, UNR = 64, RUN = 1;
};
template <int A, int B, int C>
struct Tune<A, B, C> {
  static constexpr int R = 2, UNR = B, RUN = 1;
  static constexpr bool IO = false;
};
template <int A, int B, int C, int E>
struct Tune<A, B, C, E> {
  static constexpr int R = 2, UNR = B, RUN = 1;
};
template <>
#ifndef SMLRT_OPT_R
#define SMLRT_OPT_R 2
#endif
struct Tune<5, 64, 32, 1> {  // C1: [k, 0:5] rows
  static constexpr int R = SMLRT_OPT_R, UNR = SMLRT_OPT_UNR, RUN = 5;
};
template <>
#ifndef SMLRT_MW_R
#define SMLRT_MW_R 1
#endif
#ifndef SMLRT_MW_IO
#define SMLRT_MW_IO 1
#endif
struct Tune<36, 8, 4> {  // C5: 3x3x4 halo = 12 runs of 3
  static constexpr int R = SMLRT_MW_R, UNR = 8, RUN = 3;
  static constexpr bool IO = SMLRT_MW_IO;
};
template <int A, int B, int C>
constexpr bool io_order() { return Tune<A, B, C>::IO; }

// R rows per thread (rows blockIdx*128*R + threadIdx + 128 r: coalesced per r)
// a translation unit may set SMLRT_EXACT_MINB (resident CTAs per SM) to cap
// the register allocation of its instantiations
#ifdef SMLRT_EXACT_MINB
#define SMLRT_EXACT_LB __launch_bounds__(128, SMLRT_EXACT_MINB)
#else
#define SMLRT_EXACT_LB __launch_bounds__(128)
#endif
template <bool F32, int ACT1, int R, int UNR, int RUN, class S, int... D>
__global__ void SMLRT_EXACT_LB region_exact_kernel(
    const ModelParams<S::NPARAM, S::L> mp, const __grid_constant__ DevPlan Pin,
    const __grid_constant__ Ptrs src, const __grid_constant__ DevPlan Pout,
    const __grid_constant__ Ptrs dst, int64_t r0, int64_t r1, float* __restrict__ staged, uint32_t* status) {
  const int64_t row0 = r0 + blockIdx.x * (int64_t)(128 * R) + threadIdx.x;
  bool bad = false;
  float x[R][S::IN], y[R][S::OUT];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t row = row0 + 128 * r;
    if (row < r1) {
      load_row<F32, RUN>(Pin, src, (uint32_t)row, x[r]);
    } else {
#pragma unroll
      for (int f = 0; f < S::IN; ++f) x[r][f] = 0.0f;
    }
  }
  forward<ACT1, R, UNR, D...>(mp, x, y);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t row = row0 + 128 * r;
    if (row >= r1) continue;
#pragma unroll
    for (int g = 0; g < S::OUT; ++g) bad |= nonfinite(y[r][g]);
    if (staged != nullptr) {
#pragma unroll
      for (int g = 0; g < S::OUT; ++g) staged[(row - r0) * S::OUT + g] = y[r][g];
    } else if (Pout.uniform) {
      int64_t ro = row_offset_uniform(Pout, (uint32_t)row);
      void* base = const_cast<void*>(dst.p[Pout.uarray]);
      int dt = dst.dt[Pout.uarray];
      float* pr = reinterpret_cast<float*>(base) + ro;  // one row address, column offsets added
#pragma unroll
      for (int g = 0; g < S::OUT; ++g) {
        const int64_t c = S::OUT <= SMLRT_INLINE_COLS ? Pout.col_inl[g] : __ldg(Pout.col_off + g);
        if (F32)
          pr[c] = y[r][g];
        else
          store_f32(base, dt, c + ro, y[r][g]);
      }
    } else {
      uint32_t idx[SMLRT_MAX_SWEEP];
      unravel(Pout, (uint32_t)row, idx);
#pragma unroll
      for (int g = 0; g < S::OUT; ++g) {
        int arr = __ldg(Pout.col_arr + g);
        store_f32(const_cast<void*>(dst.p[arr]), dst.dt[arr], col_address(Pout, g, idx), y[r][g]);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flag_nonfinite(status);
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

// rows per thread / layer-1 loop unroll per shape (measured on B200)
// RUN: contiguous input-column run the gather exploits when the plan has it
template <int... D>
int try_fused(const smlrt_model_s& m, const DevPlan& in, const Ptrs& src, const DevPlan& out,
              const Ptrs& dst, bool all_f32, int64_t r0, int64_t r1, float* staged, cudaStream_t s,
              uint32_t* status, bool probe_only, bool* done) {
  using S = Shape<D...>;
  if (*done || !dims_match<D...>(m)) return SMLRT_OK;
  *done = true;
  if (probe_only) return SMLRT_OK;
  ModelParams<S::NPARAM, S::L> mp{};
  for (int l = 0; l < S::L; ++l) mp.act[l] = m.layers[l].act;
  pack_params(m.host_params.data(), mp.w, static_cast<S*>(nullptr));
  const float one[2] = {1.0f, 1.0f};
  std::memcpy(&mp.one2, one, sizeof(one));
  int64_t n = r1 - r0;
  constexpr int R = Tune<D...>::R, UNR = Tune<D...>::UNR;
  dim3 grid((unsigned)((n + 128 * R - 1) / (128 * R)));
  // layer-1 activation is a template argument (it sits inside the streamed loop)
  constexpr int RUN = Tune<D...>::RUN;
  const bool runs = RUN > 1 && plan_runs(in, RUN);
  auto go = [&](auto act1) {
    constexpr int A1 = decltype(act1)::value;
    if (all_f32 && runs)
      region_exact_kernel<true, A1, R, UNR, RUN, S, D...><<<grid, 128, 0, s>>>(mp, in, src, out, dst, r0, r1,
                                                                               staged, status);
    else if (all_f32)
      region_exact_kernel<true, A1, R, UNR, 1, S, D...><<<grid, 128, 0, s>>>(mp, in, src, out, dst, r0, r1, staged,
                                                                             status);
    else
      region_exact_kernel<false, A1, R, UNR, 1, S, D...><<<grid, 128, 0, s>>>(mp, in, src, out, dst, r0, r1,
                                                                              staged, status);
  };
  if (S::L == 1 || m.layers[0].act == SMLRT_IDENTITY)
    go(std::integral_constant<int, SMLRT_IDENTITY>{});
  else if (m.layers[0].act == SMLRT_RELU)
    go(std::integral_constant<int, SMLRT_RELU>{});
  else
    go(std::integral_constant<int, SMLRT_TANH>{});
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

}  // namespace

// tries one shape instantiation set; *done = true when the model matched
using ExactTryFn = int (*)(const smlrt_model_s&, const DevPlan&, const Ptrs&, const DevPlan&, const Ptrs&, bool,
                           int64_t, int64_t, float*, cudaStream_t, uint32_t*, bool, bool*);
int exact_try_c1(const smlrt_model_s&, const DevPlan&, const Ptrs&, const DevPlan&, const Ptrs&, bool, int64_t,
                 int64_t, float*, cudaStream_t, uint32_t*, bool, bool*);
int exact_try_c5(const smlrt_model_s&, const DevPlan&, const Ptrs&, const DevPlan&, const Ptrs&, bool, int64_t,
                 int64_t, float*, cudaStream_t, uint32_t*, bool, bool*);
int exact_try_small(const smlrt_model_s&, const DevPlan&, const Ptrs&, const DevPlan&, const Ptrs&, bool, int64_t,
                    int64_t, float*, cudaStream_t, uint32_t*, bool, bool*);
// any small dense MLP, runtime dimensions (exact_generic.cu)
int exact_try_generic(const smlrt_model_s&, const DevPlan&, const Ptrs&, const DevPlan&, const Ptrs&, bool, int64_t,
                      int64_t, float*, cudaStream_t, uint32_t*, bool, bool*);

}  // namespace smlrt
