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
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "tc_ptx.cuh"

// SMLRT_SLEEPWAIT=1: every mbarrier wait in this file carries a suspend-time
// hint, so waiting warps (the MMA issuer above all) stop re-polling and leave
// their sub-partition's issue slots to the epilogue warps sharing it
#ifndef SMLRT_LDX64
#define SMLRT_LDX64 1
#endif
#ifndef SMLRT_SLEEPWAIT
#define SMLRT_SLEEPWAIT 0
#endif
#if SMLRT_SLEEPWAIT
#define mbar_wait mbar_wait_sleep
#endif

namespace smlrt {
namespace {

using namespace ptx;

constexpr int BM = 128;
constexpr int KX = 16;
#ifndef SMLRT_XSTAGES
#define SMLRT_XSTAGES 2
#endif
constexpr int XSTAGES = SMLRT_XSTAGES;
#ifndef SMLRT_EPI1_PARTS
#define SMLRT_EPI1_PARTS 2
#endif
// epilogue-1 warps per TMEM lane quarter: each drains H1/NP columns
constexpr int NP = SMLRT_EPI1_PARTS;
constexpr int WARP_EPI2 = 0, WARP_EPI1 = 4, WARP_LOAD = 4 + 4 * NP, WARP_MMA = WARP_LOAD + 4;
constexpr int NTHREADS = (WARP_MMA + 1) * 32;
#ifndef SMLRT_MMA2W
#define SMLRT_MMA2W 1
#endif
// SMLRT_MMA2W=1 (single-CTA SS kernel): layer 1 and layer 2 are issued by two
// different warps, so the next tile's layer-1 MMA does not queue behind the
// MMA warp's waits for the current tile's A2 buffer.
constexpr int MMA2W = SMLRT_MMA2W;
template <bool PAIR>
constexpr int ss_threads() { return PAIR ? NTHREADS : NTHREADS + 32 * MMA2W; }
#ifndef SMLRT_LDEPTH
#define SMLRT_LDEPTH 1
#endif
constexpr int LDEPTH = SMLRT_LDEPTH;  // X tiles of global loads in flight per loader thread
#ifndef SMLRT_L2DUAL
#define SMLRT_L2DUAL 0
#endif
// SMLRT_L2DUAL=1 (single-CTA kernel): layer 2's 16 K-steps alternate between
// two TMEM accumulators summed in epilogue 2.  In isolation consecutive M=128
// N=128 MMAs into one accumulator cost ~108 cycles each and ~64 when two
// accumulators alternate (tools/mma_latency.cu, same operands every MMA); in
// the kernel it measured 1.21 ms vs 1.14 ms: the two accumulators take the
// columns of layer 2's double buffer, and the single-buffered accumulator
// stalls the MMA warp on epilogue 2 (~500 cycles per tile).  Off by default.
constexpr bool L2DUAL = SMLRT_L2DUAL != 0;

// Biases ride on the tensor cores: a constant "ones" tile [128 x 16] (columns
// 0 and 1 = 1.0) times a bias tile [N x 16] holding bf16(b) in k=0 and
// bf16(b - bf16(b)) in k=1 adds b (to ~16 mantissa bits) to every row of the
// accumulator, so the epilogues never touch the biases.
template <int H1, int H2, int NS = 1>
struct Lay {
  // NS = 2: CTA-pair (cta_group::2) kernel -- every B operand (W1, W2 and the
  // bias tiles) is split along N, each CTA holding rows [rank N/2, (rank+1) N/2)
  static_assert(H1 % 64 == 0 && H1 >= 64 && H1 <= 256, "H1: multiple of 64, <= 256");
  static_assert(H2 % 32 == 0 && H2 >= 32 && H2 <= 256, "H2: multiple of 32, <= 256");
  static_assert(H1 + 2 * H2 <= 512, "TMEM columns");
  static constexpr int KC = H1 / 64;          // layer-2 K chunks of 64
  static constexpr int N1 = H1 / NS, N2 = H2 / NS;  // B rows held by this CTA
  static constexpr int W2_CHUNK = N2 * 128;   // [N2][64] bf16, SW128
  static constexpr int A2_CHUNK = BM * 128;   // [128][64] bf16, SW128
  static constexpr int A2_BUF = KC * A2_CHUNK;
  static constexpr int X_STAGE = BM * 32;     // [128][16] bf16, SW32
  static constexpr int OFF_W2 = 0;
  static constexpr int OFF_A2 = OFF_W2 + KC * W2_CHUNK;
  static constexpr int OFF_W1 = OFF_A2 + 2 * A2_BUF;   // [N1][16] SW32
  static constexpr int OFF_W1B = OFF_W1 + N1 * 32;     // [N1][16] SW32 bias tile
  static constexpr int OFF_W2B = OFF_W1B + N1 * 32;    // [N2][16] SW32 bias tile
  static constexpr int OFF_ONES = OFF_W2B + N2 * 32;   // [128][16] SW32
  static constexpr int OFF_X = OFF_ONES + BM * 32;
  static constexpr int OFF_W3 = OFF_X + XSTAGES * X_STAGE;
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
    B_L1FULL2 = B_L2EMPTY + 2,  // single-CTA kernel: layer 1 as two N = H1/2 halves
    B_L1EMPTY2,
    N_BAR
  };
  static constexpr int OFF_TMEM = OFF_BAR + N_BAR * 8;
  static constexpr int BYTES = OFF_TMEM + 16;
  static constexpr int ALLOC = BYTES + 1024;  // 1 KB alignment slack (SW128 atoms)
  static_assert(ALLOC <= 232448, "shared memory budget");
  // global blob produced by tc_pack_model: W2 | W1 | W1B | W2B | w3 | b3 (same order as smem)
  static constexpr int BLOB_W1 = KC * W2_CHUNK;
  static constexpr int BLOB_TAIL = BLOB_W1 + 2 * N1 * 32 + N2 * 32;
  static constexpr int TAIL = H2 * 4 + 16;
  static constexpr int BLOB = BLOB_TAIL + TAIL;  // per CTA rank; NS of them back to back
  static constexpr int T_L1 = 0, T_L2 = H1;  // TMEM column bases
};

struct TcArgs {
  const uint8_t* blob;
  const float* x_fast;  // dense contiguous f32 rows of 16 (fast gather path) or nullptr
  int F;
  int act1, act2, act3;
  int64_t r0, r1;
  int n_tiles;
  float* staged;
  uint32_t* status;
  // biases and the last layer's weights in the parameter bank (uniform LDCU
  // in the epilogues; the single-CTA kernel adds the biases there instead of
  // spending tensor-core K slices and shared-memory bandwidth on them)
  alignas(16) float b1[256];
  float b2[256];
  float w3[256];
  float b3;
};

__device__ __forceinline__ uint64_t add2f(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ uint64_t fma2f(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
#ifndef SMLRT_EPI2_PACKED
#define SMLRT_EPI2_PACKED 1
#endif

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

__device__ __forceinline__ float ld_elem(const void* base, int dt, int64_t i) {
  return dt == SMLRT_F32 ? __ldg(reinterpret_cast<const float*>(base) + i)
                         : __double2float_rn(__ldg(reinterpret_cast<const double*>(base) + i));
}

// Debug-only pipeline trace (build with -DSMLRT_TC_TRACE; `make trace`):
// clock64 stamps of each role's events for the first TR_TILES tiles of CTAs 0/1.
#ifdef SMLRT_TC_TRACE
constexpr int TR_TILES = 1024, TR_EV = 16;
__device__ unsigned long long g_tc_trace[2][TR_TILES][TR_EV];
#define TR(ev, it)                                                   \
  do {                                                               \
    if (blockIdx.x < 2 && (it) < TR_TILES)                           \
      g_tc_trace[blockIdx.x][(it)][(ev)] = clock64();                \
  } while (0)
#else
#define TR(ev, it) \
  do {             \
  } while (0)
#endif

// Tile schedule: single CTAs take 128-row tiles blockIdx + i*grid; a CTA pair
// takes 256-row pair tiles (cluster + i*clusters), rank r owning rows [128 r, 128 r + 128).
struct Sched {
  int first, stride, rank, pair;
  __device__ __forceinline__ int64_t tile(int it) const {
    const int64_t t = (int64_t)first + (int64_t)it * stride;
    return pair ? 2 * t + rank : t;
  }
};

// producers/consumers arrive on the MMA-issuing CTA's barrier (rank 0 of a pair)
template <bool PAIR>
__device__ __forceinline__ void arrive_mma(uint64_t* bar) {
  if constexpr (PAIR)
    mbar_arrive_remote(mapa(bar, 0));
  else
    mbar_arrive(bar);
}

// ------------------------------------------------------------ epilogue 1
// TMEM L1 accumulator (bias already added by the MMA) -> act -> bf16 ->
// A2[b] in the SW128 K-major layout layer 2 consumes.  Thread = row r; this
// warpgroup covers columns [half*H1/2, (half+1)*H1/2).
template <int ACT, int H1, int H2, class L, bool PAIR>
__device__ __forceinline__ void epilogue1(uint8_t* smem, uint64_t* bar, uint32_t tbase, int n_my, int half,
                                          int q, int lane, const TcArgs& a) {
  constexpr int HC = H1 / NP;  // columns this warp drains (`half` = part index)
  const int r = q * 32 + lane;
  const uint32_t lane_addr = tbase + ((uint32_t)(q * 32) << 16) + L::T_L1 + half * HC;
  // swizzled 16-B chunk j of row r lives at rowbase + ((j ^ (r&7)) << 4)
  const uint32_t rowbase = smem_u32(smem + L::OFF_A2) + r * 128 + (half * HC / 64) * L::A2_CHUNK;
  uint32_t xo[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) xo[j] = rowbase + ((j ^ (r & 7)) << 4);
  for (int it = 0; it < n_my; ++it) {
    const int b = it & 1;
    mbar_wait(bar + L::B_L1FULL, it & 1);
    if (q == 0 && half == 0 && lane == 0) TR(2, it);
    tc_fence_after();
    // x16 loads with the next one in flight while the current one is
    // activated, packed and stored; the L1 buffer is released after the last load
    mbar_wait(bar + L::B_A2EMPTY + b, ((it >> 1) & 1) ^ 1);
    if (q == 0 && half == 0 && lane == 0) TR(3, it);
    const uint32_t boff = b * L::A2_BUF;
    uint32_t v[2][16];
    tmem_ld16(lane_addr, v[0]);
#pragma unroll
    for (int c = 0; c < HC / 16; ++c) {
      tmem_wait_ld16(v[c & 1]);
      if (c + 1 < HC / 16) {
        tmem_ld16(lane_addr + (c + 1) * 16, v[(c + 1) & 1]);
      } else {
        tc_fence_before();
        arrive_mma<PAIR>(bar + L::B_L1EMPTY);
        if (q == 0 && half == 0 && lane == 0) TR(4, it);
      }
      const float* f = reinterpret_cast<const float*>(v[c & 1]);
      float fb[16];
      if constexpr (!PAIR) {  // + b1 (packed adds, bias pairs from the parameter bank)
        const uint64_t* bp = reinterpret_cast<const uint64_t*>(a.b1 + half * HC + c * 16);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint64_t sum = add2f(*reinterpret_cast<const uint64_t*>(&v[c & 1][2 * e]), bp[e]);
          asm("mov.b64 {%0, %1}, %2;" : "=f"(fb[2 * e]), "=f"(fb[2 * e + 1]) : "l"(sum));
        }
        f = fb;
      }
      const uint32_t coff = boff + (c >> 2) * L::A2_CHUNK;
#if defined(SMLRT_ABLATE) && SMLRT_ABLATE == 1  // timing experiment only: no A2 stores
      if (f[0] == 12345.0f)
#endif
#pragma unroll
      for (int j = 0; j < 2; ++j)
        st_shared_v4(xo[((c >> 1) & 1) * 4 + (c & 1) * 2 + j] + coff, act_pack<ACT>(f[8 * j], f[8 * j + 1]),
                     act_pack<ACT>(f[8 * j + 2], f[8 * j + 3]), act_pack<ACT>(f[8 * j + 4], f[8 * j + 5]),
                     act_pack<ACT>(f[8 * j + 6], f[8 * j + 7]));
    }
    fence_async_smem();
    arrive_mma<PAIR>(bar + L::B_A2FULL + b);
    if (q == 0 && half == 0 && lane == 0) TR(5, it);
  }
}

// Single-CTA epilogue 1 over layer 1 split in two N = H1/2 halves, each with
// its own TMEM columns and full/empty barriers: the MMA warp issues half a of
// tile i+1 as soon as half a of tile i is drained, so the drain of one half
// overlaps the layer-1 MMA (and its commit latency) of the other instead of
// serialising behind a single-buffered accumulator.  Warp (q, part) drains
// columns [part*H1/4, +H1/4) of each half for its 32 rows.
template <int ACT, int H1, int H2, class L, int PART>
__device__ __forceinline__ void epilogue1_split(uint8_t* smem, uint64_t* bar, uint32_t tbase, int n_my, int q,
                                                int lane, const TcArgs& a) {
  static_assert(NP == 2, "two epilogue-1 warps per lane quarter");
  constexpr int HH = H1 / 2, HC = HH / 2;
  static_assert(HC % 16 == 0 && HC <= 64, "x16 loads, <= 64 registers per half");
  const int r = q * 32 + lane;
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  const uint32_t a2row = smem_u32(smem + L::OFF_A2) + r * 128;
  for (int it = 0; it < n_my; ++it) {
    const int b = it & 1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mbar_wait(bar + (h == 0 ? L::B_L1FULL : L::B_L1FULL2), it & 1);
      if (q == 0 && PART == 0 && lane == 0) TR(h == 0 ? 2 : 12, it);
      tc_fence_after();
      const int col0 = h * HH + PART * HC;  // first hidden unit of this warp's columns (compile-time)
      // drain the whole half into registers first and release its TMEM
      // columns at once; only then wait for the A2 buffer (which frees when
      // layer 2 of tile it-2 completes)
      uint32_t v[HC];
#if SMLRT_LDX64
      if constexpr (HC == 64)
        tmem_ld64(tbase + lane_off + L::T_L1 + col0, v);
      else
#endif
#pragma unroll
        for (int c = 0; c < HC / 16; ++c)
          tmem_ld16(tbase + lane_off + L::T_L1 + col0 + c * 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16 * c));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar + (h == 0 ? L::B_L1EMPTY : L::B_L1EMPTY2));
      if (h == 0) mbar_wait(bar + L::B_A2EMPTY + b, ((it >> 1) & 1) ^ 1);
#pragma unroll
      for (int c = 0; c < HC / 16; ++c) {
        const int col = col0 + c * 16;
        float f[16];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint64_t bb = *reinterpret_cast<const uint64_t*>(a.b1 + col + 2 * e);  // uniform LDCU
          const uint64_t sum = add2f(*reinterpret_cast<const uint64_t*>(&v[16 * c + 2 * e]), bb);
          asm("mov.b64 {%0, %1}, %2;" : "=f"(f[2 * e]), "=f"(f[2 * e + 1]) : "l"(sum));
        }
        // SW128 K-major: hidden unit `col` -> chunk col/64, 16-B slot (col%64)/8 ^ (r&7)
        const uint32_t base = a2row + b * L::A2_BUF + (col >> 6) * L::A2_CHUNK;
        const int j0 = (col & 63) >> 3;
#pragma unroll
        for (int j = 0; j < 2; ++j)
          st_shared_v4(base + (((j0 + j) ^ (r & 7)) << 4), act_pack<ACT>(f[8 * j], f[8 * j + 1]),
                       act_pack<ACT>(f[8 * j + 2], f[8 * j + 3]), act_pack<ACT>(f[8 * j + 4], f[8 * j + 5]),
                       act_pack<ACT>(f[8 * j + 6], f[8 * j + 7]));
      }
    }
    fence_async_smem();
    mbar_arrive(bar + L::B_A2FULL + b);
#ifndef SMLRT_TRACE_ALT
#define SMLRT_TRACE_ALT 0
#endif
    if (q == 0 && PART == SMLRT_TRACE_ALT && lane == 0) TR(5, it);
    if (q == 3 && PART == (1 ^ SMLRT_TRACE_ALT) && lane == 0) TR(3, it);
    if (q == 1 && PART == (1 ^ SMLRT_TRACE_ALT) && lane == 0) TR(4, it);
    if (q == 2 && PART == (0 ^ SMLRT_TRACE_ALT) && lane == 0) TR(10, it);
  }
}

template <int ACT, int H1, int H2, class L>
__device__ __forceinline__ void epilogue1_split_dispatch(uint8_t* smem, uint64_t* bar, uint32_t tbase, int n_my,
                                                         int part, int q, int lane, const TcArgs& a) {
  if (part == 0)
    epilogue1_split<ACT, H1, H2, L, 0>(smem, bar, tbase, n_my, q, lane, a);
  else
    epilogue1_split<ACT, H1, H2, L, 1>(smem, bar, tbase, n_my, q, lane, a);
}

// ------------------------------------------------------------ epilogue 2
// TMEM L2 accumulator (+b2 from the MMA) -> act -> dot w3 -> +b3 -> act3 ->
// scatter.  Thread = row.
template <int ACT, int H1, int H2, class L, bool PAIR>
__device__ __forceinline__ void epilogue2(uint8_t* smem, uint64_t* bar, uint32_t tbase, int n_my, int q, int lane,
                                          const TcArgs& a, const DevPlan& Pout, const Ptrs8& dst, Sched sc) {
  const int r = q * 32 + lane;
  const uint32_t w3 = smem_u32(smem + L::OFF_W3);
  const float b3 = PAIR ? *reinterpret_cast<const float*>(smem + L::OFF_B3) : a.b3;
  const uint32_t lane_addr = tbase + ((uint32_t)(q * 32) << 16) + L::T_L2;
  const bool out_fast = Pout.uniform && Pout.n_sweep == 1 && dst.dt[Pout.uarray] == SMLRT_F32 && a.staged == nullptr;
  float* out_base = out_fast ? reinterpret_cast<float*>(const_cast<void*>(dst.p[Pout.uarray])) + Pout.col_off0
                             : nullptr;
  constexpr bool DA = !PAIR && L2DUAL;
  for (int it = 0; it < n_my; ++it) {
    const int b = DA ? 0 : (it & 1);
    mbar_wait(bar + L::B_L2FULL + b, DA ? (it & 1) : ((it >> 1) & 1));
    if (q == 0 && lane == 0) TR(6, it);
    tc_fence_after();
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};  // packed-pair partial sums (SMLRT_EPI2_PACKED)
#if SMLRT_LDX64
    if constexpr (!PAIR && !DA && H2 % 64 == 0) {
      // 64 columns per TMEM request, half the wait points of the x32 loop
#pragma unroll
      for (int c2 = 0; c2 < H2 / 64; ++c2) {
        uint32_t v[64];
        tmem_ld64(lane_addr + b * H2 + c2 * 64, v);
        tmem_wait_ld();
        if (c2 == H2 / 64 - 1) {
          tc_fence_before();
          mbar_arrive(bar + L::B_L2EMPTY + b);
        }
#if SMLRT_EPI2_PACKED
        if constexpr (ACT != SMLRT_TANH) {
          // packed pairs: add.f32x2 (b2), two max.NaN (relu), fma.f32x2 (w3):
          // 2 instructions per hidden unit instead of 3
#pragma unroll
          for (int e = 0; e < 64; e += 2) {
            const uint64_t bb = *reinterpret_cast<const uint64_t*>(a.b2 + c2 * 64 + e);
            const uint64_t ww = *reinterpret_cast<const uint64_t*>(a.w3 + c2 * 64 + e);
            uint64_t h = add2f((uint64_t)v[e] | ((uint64_t)v[e + 1] << 32), bb);
            if constexpr (ACT == SMLRT_RELU) {
              float lo, hi;
              asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(h));
              asm("mov.b64 %0, {%1, %2};" : "=l"(h) : "f"(relu_nan(lo)), "f"(relu_nan(hi)));
            }
            acc2[(e >> 1) & 3] = fma2f(h, ww, acc2[(e >> 1) & 3]);
          }
          continue;
        }
#endif
#pragma unroll
        for (int e = 0; e < 64; e += 4) {
          const float4 ww = *reinterpret_cast<const float4*>(a.w3 + c2 * 64 + e);
          const float4 bb = *reinterpret_cast<const float4*>(a.b2 + c2 * 64 + e);
          acc[((e >> 2) & 1) * 4 + 0] = fmaf(act_t<ACT>(__uint_as_float(v[e]) + bb.x), ww.x, acc[((e >> 2) & 1) * 4 + 0]);
          acc[((e >> 2) & 1) * 4 + 1] = fmaf(act_t<ACT>(__uint_as_float(v[e + 1]) + bb.y), ww.y, acc[((e >> 2) & 1) * 4 + 1]);
          acc[((e >> 2) & 1) * 4 + 2] = fmaf(act_t<ACT>(__uint_as_float(v[e + 2]) + bb.z), ww.z, acc[((e >> 2) & 1) * 4 + 2]);
          acc[((e >> 2) & 1) * 4 + 3] = fmaf(act_t<ACT>(__uint_as_float(v[e + 3]) + bb.w), ww.w, acc[((e >> 2) & 1) * 4 + 3]);
        }
      }
    } else
#endif
#pragma unroll
    for (int cc = 0; cc < H2 / 32; ++cc) {
      uint32_t v[32];
      tmem_ld32(lane_addr + b * H2 + cc * 32, v);
      if constexpr (DA) {
        uint32_t w[32];
        tmem_ld32(lane_addr + H2 + cc * 32, w);  // odd K-steps' accumulator
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) + __uint_as_float(w[e]));
      } else {
        tmem_wait_ld();
      }
      if (cc == H2 / 32 - 1) {
        tc_fence_before();
        arrive_mma<PAIR>(bar + L::B_L2EMPTY + b);
      }
#pragma unroll
      for (int e = 0; e < 32; e += 4) {
        if constexpr (!PAIR) {
          const float4 ww = *reinterpret_cast<const float4*>(a.w3 + cc * 32 + e);
          const float4 bb = *reinterpret_cast<const float4*>(a.b2 + cc * 32 + e);
          acc[((e >> 2) & 1) * 4 + 0] = fmaf(act_t<ACT>(__uint_as_float(v[e]) + bb.x), ww.x, acc[((e >> 2) & 1) * 4 + 0]);
          acc[((e >> 2) & 1) * 4 + 1] = fmaf(act_t<ACT>(__uint_as_float(v[e + 1]) + bb.y), ww.y, acc[((e >> 2) & 1) * 4 + 1]);
          acc[((e >> 2) & 1) * 4 + 2] = fmaf(act_t<ACT>(__uint_as_float(v[e + 2]) + bb.z), ww.z, acc[((e >> 2) & 1) * 4 + 2]);
          acc[((e >> 2) & 1) * 4 + 3] = fmaf(act_t<ACT>(__uint_as_float(v[e + 3]) + bb.w), ww.w, acc[((e >> 2) & 1) * 4 + 3]);
          continue;
        }
        const float4 ww = ld_shared_f4(w3 + (cc * 32 + e) * 4);
        acc[((e >> 2) & 1) * 4 + 0] = fmaf(act_t<ACT>(__uint_as_float(v[e])), ww.x, acc[((e >> 2) & 1) * 4 + 0]);
        acc[((e >> 2) & 1) * 4 + 1] = fmaf(act_t<ACT>(__uint_as_float(v[e + 1])), ww.y, acc[((e >> 2) & 1) * 4 + 1]);
        acc[((e >> 2) & 1) * 4 + 2] = fmaf(act_t<ACT>(__uint_as_float(v[e + 2])), ww.z, acc[((e >> 2) & 1) * 4 + 2]);
        acc[((e >> 2) & 1) * 4 + 3] = fmaf(act_t<ACT>(__uint_as_float(v[e + 3])), ww.w, acc[((e >> 2) & 1) * 4 + 3]);
      }
    }
    for (int p = 0; p < 4; ++p) {
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc2[p]));
      acc[2 * p] += lo;
      acc[2 * p + 1] += hi;
    }
    const float y = act_f(((acc[0] + acc[4]) + (acc[1] + acc[5])) + ((acc[2] + acc[6]) + (acc[3] + acc[7])) + b3,
                          a.act3);
    const int64_t row = a.r0 + sc.tile(it) * BM + r;
    bool bad = false;
    if (row < a.r1) {
      bad = (__float_as_uint(y) & 0x7f800000u) == 0x7f800000u;
      if (out_fast) {
        out_base[row * Pout.ustride[0]] = y;
      } else if (a.staged != nullptr) {
        a.staged[row - a.r0] = y;
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
        void* base = const_cast<void*>(dst.p[arr]);
        if (dst.dt[arr] == SMLRT_F32)
          reinterpret_cast<float*>(base)[addr] = y;
        else
          reinterpret_cast<double*>(base)[addr] = (double)y;
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) flag_nonfinite(a.status);
    if (q == 0 && lane == 0) TR(7, it);
  }
}

template <int H1, int H2, bool PAIR>
__global__ void __launch_bounds__(ss_threads<PAIR>(), 1)
    mlp3_tc_kernel(const __grid_constant__ TcArgs a, const __grid_constant__ DevPlan Pin,
                   const __grid_constant__ Ptrs8 src, const __grid_constant__ DevPlan Pout,
                   const __grid_constant__ Ptrs8 dst) {
  constexpr int NS = PAIR ? 2 : 1;
  using L = Lay<H1, H2, NS>;
  const uint32_t rank = PAIR ? cluster_rank() : 0;
  const Sched sc = PAIR ? Sched{(int)blockIdx.x / 2, (int)gridDim.x / 2, (int)rank, 1}
                        : Sched{(int)blockIdx.x, (int)gridDim.x, 0, 0};
  const bool leader = rank == 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  // ---------------------------------------------------------------- setup
  if (threadIdx.x == 0) {
    for (int s = 0; s < XSTAGES; ++s) {
      mbar_init(bar + L::B_XFULL + s, 128 * NS);
      mbar_init(bar + L::B_XEMPTY + s, 1);
    }
    mbar_init(bar + L::B_L1FULL, 1);
    mbar_init(bar + L::B_L1EMPTY, 128 * NP * NS);
    mbar_init(bar + L::B_L1FULL2, 1);
    mbar_init(bar + L::B_L1EMPTY2, 128 * NP * NS);
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar + L::B_A2FULL + b, 128 * NP * NS);
      mbar_init(bar + L::B_A2EMPTY + b, 1);
      mbar_init(bar + L::B_L2FULL + b, 1);
      mbar_init(bar + L::B_L2EMPTY + b, 128 * NS);
    }
    mbar_fence_init();
  }
  if (warp == WARP_MMA) {
    if constexpr (PAIR)
      tmem_alloc2(tmem_slot, 512);
    else
      tmem_alloc(tmem_slot, 512);
  }
  {  // resident weights: this rank's blob -> smem (16-byte vectors); ones tile built here
    const int4* g = reinterpret_cast<const int4*>(a.blob + rank * L::BLOB);
    for (int i = threadIdx.x; i < L::BLOB_W1 / 16; i += ss_threads<PAIR>())
      reinterpret_cast<int4*>(smem + L::OFF_W2)[i] = g[i];
    for (int i = threadIdx.x; i < (L::BLOB_TAIL - L::BLOB_W1) / 16; i += ss_threads<PAIR>())
      reinterpret_cast<int4*>(smem + L::OFF_W1)[i] = g[L::BLOB_W1 / 16 + i];
    for (int i = threadIdx.x; i < L::TAIL / 16; i += ss_threads<PAIR>())
      reinterpret_cast<int4*>(smem + L::OFF_W3)[i] = g[L::BLOB_TAIL / 16 + i];
    for (int i = threadIdx.x; i < BM * KX; i += ss_threads<PAIR>()) {
      const int row = i / KX, k = i % KX;
      *reinterpret_cast<__nv_bfloat16*>(smem + L::OFF_ONES + sw32_offset(row, k)) =
          __float2bfloat16_rn(k < 2 ? 1.0f : 0.0f);
    }
  }
  fence_async_smem();
  tc_fence_before();
  if constexpr (PAIR)
    cluster_sync();  // peer barriers, weights and TMEM ready before any MMA
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int n_units = PAIR ? (a.n_tiles + 1) / 2 : a.n_tiles;
  const int n_my = (n_units - sc.first + sc.stride - 1) / sc.stride;

  if (warp >= WARP_LOAD && warp < WARP_MMA) {
    // ============================================================ loader
    const int t = threadIdx.x - WARP_LOAD * 32;
    const uint32_t xbase = smem_u32(smem + L::OFF_X);
    if (a.x_fast != nullptr) {
      // tile = 2048 contiguous floats: thread t moves float4 #(t + 128 i), i < 4.
      // Loads run LDEPTH tiles ahead in registers (the next tile's loads are
      // issued as soon as the current one is stored).  A first loader that
      // issued them only after the XEMPTY wait capped the kernel at ~0.9 TB/s;
      // with the split MMA issuers one tile ahead is enough and the fastest
      // (LDEPTH 1 / 2 / 3: 0.966 / 1.005 / 1.008 ms).
      float4 buf[LDEPTH][4];
      auto load_tile = [&](int it, float4(&v)[4]) {
        const int64_t row0 = a.r0 + sc.tile(it) * BM;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int idx = t + 128 * i;
          const int64_t row = row0 + (idx >> 2);
          v[i] = (it < n_my && row < a.r1)
                     ? __ldg(reinterpret_cast<const float4*>(a.x_fast + row * 16) + (idx & 3))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
#pragma unroll
      for (int d = 0; d < LDEPTH; ++d) load_tile(d, buf[d]);
      for (int it0 = 0; it0 < n_my; it0 += LDEPTH) {
#pragma unroll
        for (int d = 0; d < LDEPTH; ++d) {
          const int it = it0 + d;
          if (it >= n_my) break;
          const int s = it % XSTAGES;
          mbar_wait(bar + L::B_XEMPTY + s, ((it / XSTAGES) & 1) ^ 1);
          const uint32_t xs = xbase + s * L::X_STAGE;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int idx = t + 128 * i;
            st_shared_v2(xs + sw32_offset(idx >> 2, (idx & 3) * 4), pack_bf16(buf[d][i].x, buf[d][i].y),
                         pack_bf16(buf[d][i].z, buf[d][i].w));
          }
          fence_async_smem();
          arrive_mma<PAIR>(bar + L::B_XFULL + s);
          if (t == 0) TR(8, it);
          load_tile(it + LDEPTH, buf[d]);
        }
      }
    } else {
      // general plan-driven gather: thread = tile row
      float cur[16], nxt[16];
      auto load_row = [&](int it, float(&v)[16]) {
        const int64_t row = a.r0 + sc.tile(it) * BM + t;
#pragma unroll
        for (int f = 0; f < 16; ++f) v[f] = 0.0f;
        if (row >= a.r1) return;
        if (Pin.uniform) {
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
        const uint32_t xs = xbase + s * L::X_STAGE;
        st_shared_v4(xs + sw32_offset(t, 0), pack_bf16(cur[0], cur[1]), pack_bf16(cur[2], cur[3]),
                     pack_bf16(cur[4], cur[5]), pack_bf16(cur[6], cur[7]));
        st_shared_v4(xs + sw32_offset(t, 8), pack_bf16(cur[8], cur[9]), pack_bf16(cur[10], cur[11]),
                     pack_bf16(cur[12], cur[13]), pack_bf16(cur[14], cur[15]));
        fence_async_smem();
        arrive_mma<PAIR>(bar + L::B_XFULL + s);
#pragma unroll
        for (int f = 0; f < 16; ++f) cur[f] = nxt[f];
      }
    }
  } else if ((warp == WARP_MMA || (MMA2W && warp == WARP_MMA + 1)) && !PAIR) {
    // ========================================================= MMA issuer
    // Whole warp runs the loop (warp-uniform control flow, descriptors in
    // uniform registers), elect.sync inside the asm picks the issuing lane:
    // ~3 instructions per MMA.  A lane-0 branch costs ~14 (R2UR / ELECT /
    // BRA.U.ANY per MMA), ~110 cycles of single-warp issue latency -- more
    // than the 64 tensor cycles of an M=128 N=128 K=16 MMA, which made the
    // issuer the bottleneck.
    constexpr uint32_t idesc1 = idesc_bf16(BM, H1);
    constexpr uint32_t idesc2 = idesc_bf16(BM, H2);
    const uint64_t w1d = smem_desc(smem_u32(smem + L::OFF_W1), 256, kSwizzle32);
    const uint64_t x0d = smem_desc(smem_u32(smem + L::OFF_X), 256, kSwizzle32);
    const uint64_t a20d = smem_desc(smem_u32(smem + L::OFF_A2), 1024, kSwizzle128);
    const uint64_t w20d = smem_desc(smem_u32(smem + L::OFF_W2), 1024, kSwizzle128);
    auto issue_l2 = [&](int j) {
      const int b = j & 1;
      mbar_wait(bar + L::B_A2FULL + b, (j >> 1) & 1);
      if (lane == 0) TR(11, j);
      if constexpr (L2DUAL)
        mbar_wait(bar + L::B_L2EMPTY, (j & 1) ^ 1);
      else
        mbar_wait(bar + L::B_L2EMPTY + b, ((j >> 1) & 1) ^ 1);
      if (lane == 0) TR(1, j);
      tc_fence_after();
      const uint64_t ab = a20d + ((b * L::A2_BUF) >> 4);
      if constexpr (L2DUAL) {
#pragma unroll
        for (int ks = 0; ks < 4 * L::KC; ++ks)  // even K-steps -> accumulator 0, odd -> accumulator 1
          mma_ss_elect(tbase + L::T_L2 + (ks & 1) * H2, ab + (((ks >> 2) * L::A2_CHUNK + (ks & 3) * 32) >> 4),
                       w20d + (((ks >> 2) * L::W2_CHUNK + (ks & 3) * 32) >> 4), idesc2, ks >= 2);
        mma_commit_elect(bar + L::B_A2EMPTY + b);
        mma_commit_elect(bar + L::B_L2FULL);
        return;
      }
      const uint32_t d = tbase + L::T_L2 + b * H2;
#if defined(SMLRT_ABLATE) && SMLRT_ABLATE == 2  // timing experiment only: one L2 MMA per tile
      mma_ss_elect(d, ab, w20d, idesc2, 0);
#else
#pragma unroll
      for (int kc = 0; kc < L::KC; ++kc)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_ss_elect(d, ab + ((kc * L::A2_CHUNK + k * 32) >> 4), w20d + ((kc * L::W2_CHUNK + k * 32) >> 4), idesc2,
                       (kc | k) != 0);
#endif
      mma_commit_elect(bar + L::B_A2EMPTY + b);
      mma_commit_elect(bar + L::B_L2FULL + b);
    };
    constexpr uint32_t idesc1h = idesc_bf16(BM, H1 / 2);
    if (MMA2W && warp == WARP_MMA + 1) {
      for (int j = 0; j < n_my; ++j) issue_l2(j);
      __syncwarp();
    } else {
    for (int it = 0; it < n_my; ++it) {
      const int s = it % XSTAGES;
      mbar_wait(bar + L::B_XFULL + s, (it / XSTAGES) & 1);
      if (lane == 0) TR(9, it);
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // layer 1 in two halves with separate TMEM columns / barriers
        mbar_wait(bar + (h == 0 ? L::B_L1EMPTY : L::B_L1EMPTY2), (it & 1) ^ 1);
        if (lane == 0 && h == 0) TR(0, it);
#ifdef SMLRT_TC_TRACE
        if (lane == 0 && h == 0 && blockIdx.x < 2 && it < TR_TILES) {
          unsigned long long ns;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
          g_tc_trace[blockIdx.x][it][15] = ns;
        }
#endif
        tc_fence_after();
        mma_ss_elect(tbase + L::T_L1 + h * (H1 / 2), x0d + ((s * L::X_STAGE) >> 4),
                     w1d + ((h * (H1 / 2) * 32) >> 4), idesc1h, 0);
        mma_commit_elect(bar + (h == 0 ? L::B_L1FULL : L::B_L1FULL2));
        if (lane == 0 && h == 0) TR(14, it);
      }
      mma_commit_elect(bar + L::B_XEMPTY + s);
      if (lane == 0) TR(13, it);
      if (!MMA2W && it > 0) issue_l2(it - 1);
    }
    (void)idesc1;
    if (!MMA2W && n_my > 0) issue_l2(n_my - 1);
    __syncwarp();
    }
  } else if (warp == WARP_MMA && PAIR && leader) {
    // ================================================ MMA issuer (CTA pair)
    // rank 0's whole warp runs the loop, elect.sync issues M = 256 MMAs over
    // both CTAs' SMEM and TMEM (same reasoning as the single-CTA issuer)
    constexpr uint32_t idesc1 = idesc_bf16(BM * NS, H1);
    constexpr uint32_t idesc2 = idesc_bf16(BM * NS, H2);
    const uint64_t w1d = smem_desc(smem_u32(smem + L::OFF_W1), 256, kSwizzle32);
    const uint64_t w1bd = smem_desc(smem_u32(smem + L::OFF_W1B), 256, kSwizzle32);
    const uint64_t w2bd = smem_desc(smem_u32(smem + L::OFF_W2B), 256, kSwizzle32);
    const uint64_t onesd = smem_desc(smem_u32(smem + L::OFF_ONES), 256, kSwizzle32);
    const uint64_t x0d = smem_desc(smem_u32(smem + L::OFF_X), 256, kSwizzle32);
    const uint64_t a20d = smem_desc(smem_u32(smem + L::OFF_A2), 1024, kSwizzle128);
    const uint64_t w20d = smem_desc(smem_u32(smem + L::OFF_W2), 1024, kSwizzle128);
    auto issue_l2 = [&](int j) {
      const int b = j & 1;
      mbar_wait(bar + L::B_A2FULL + b, (j >> 1) & 1);
      mbar_wait(bar + L::B_L2EMPTY + b, ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tbase + L::T_L2 + b * H2;
      const uint64_t ab = a20d + ((b * L::A2_BUF) >> 4);
      mma2_ss_elect(d, onesd, w2bd, idesc2, 0);  // D = b2
#pragma unroll
      for (int kc = 0; kc < L::KC; ++kc)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma2_ss_elect(d, ab + ((kc * L::A2_CHUNK + k * 32) >> 4), w20d + ((kc * L::W2_CHUNK + k * 32) >> 4), idesc2,
                        1);
      mma2_commit_mc_elect(bar + L::B_A2EMPTY + b, 0x3);
      mma2_commit_mc_elect(bar + L::B_L2FULL + b, 0x3);
    };
    for (int it = 0; it < n_my; ++it) {
      const int s = it % XSTAGES;
      mbar_wait(bar + L::B_XFULL + s, (it / XSTAGES) & 1);
      mbar_wait(bar + L::B_L1EMPTY, (it & 1) ^ 1);
      tc_fence_after();
      mma2_ss_elect(tbase + L::T_L1, onesd, w1bd, idesc1, 0);  // D = b1
      mma2_ss_elect(tbase + L::T_L1, x0d + ((s * L::X_STAGE) >> 4), w1d, idesc1, 1);
      mma2_commit_mc_elect(bar + L::B_XEMPTY + s, 0x3);
      mma2_commit_mc_elect(bar + L::B_L1FULL, 0x3);
      if (it > 0) issue_l2(it - 1);
    }
    if (n_my > 0) issue_l2(n_my - 1);
    __syncwarp();
  } else if (warp == WARP_MMA) {
    // pair rank 1: its MMA warp idles (rank 0 issues for both CTAs)
  } else if (warp >= WARP_EPI1 && !PAIR) {
    const int part = (warp - WARP_EPI1) >> 2;
    if (a.act1 == SMLRT_RELU)
      epilogue1_split_dispatch<SMLRT_RELU, H1, H2, L>(smem, bar, tbase, n_my, part, warp & 3, lane, a);
    else if (a.act1 == SMLRT_TANH)
      epilogue1_split_dispatch<SMLRT_TANH, H1, H2, L>(smem, bar, tbase, n_my, part, warp & 3, lane, a);
    else
      epilogue1_split_dispatch<SMLRT_IDENTITY, H1, H2, L>(smem, bar, tbase, n_my, part, warp & 3, lane, a);
  } else if (warp >= WARP_EPI1) {
    const int half = (warp - WARP_EPI1) >> 2;  // part index in [0, NP)
    if (a.act1 == SMLRT_RELU)
      epilogue1<SMLRT_RELU, H1, H2, L, PAIR>(smem, bar, tbase, n_my, half, warp & 3, lane, a);
    else if (a.act1 == SMLRT_TANH)
      epilogue1<SMLRT_TANH, H1, H2, L, PAIR>(smem, bar, tbase, n_my, half, warp & 3, lane, a);
    else
      epilogue1<SMLRT_IDENTITY, H1, H2, L, PAIR>(smem, bar, tbase, n_my, half, warp & 3, lane, a);
  } else {
    if (a.act2 == SMLRT_RELU)
      epilogue2<SMLRT_RELU, H1, H2, L, PAIR>(smem, bar, tbase, n_my, warp, lane, a, Pout, dst, sc);
    else if (a.act2 == SMLRT_TANH)
      epilogue2<SMLRT_TANH, H1, H2, L, PAIR>(smem, bar, tbase, n_my, warp, lane, a, Pout, dst, sc);
    else
      epilogue2<SMLRT_IDENTITY, H1, H2, L, PAIR>(smem, bar, tbase, n_my, warp, lane, a, Pout, dst, sc);
  }

  // -------------------------------------------------------------- teardown
  tc_fence_before();
  if constexpr (PAIR)
    cluster_sync();
  else
    __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    if constexpr (PAIR)
      tmem_dealloc2(tbase, 512);
    else
      tmem_dealloc(tbase, 512);
  }
}

// TS self-test: D[128 x N] = A[128 x K] * B[N x K]^T with A staged in TMEM by
// tcgen05.st (bf16 pairs): validates the TMEM A-operand (TS) layout.
template <int N>
__global__ void __launch_bounds__(128, 1) tc_selftest_ts_kernel(const float* A, const float* B, int K, float* D) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sb = smem;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sb + N * K * 2);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < N * K; i += 128) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sb + (k / 64) * (N * 128) + sw128_offset(r, k & 63)) = __float2bfloat16_rn(B[i]);
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *slot;
  const int r = warp * 32 + lane;
  const uint32_t a_col = 256;  // A at columns [256, 256 + K/2), D at [0, N)
  for (int k0 = 0; k0 < K; k0 += 32) {
    uint32_t p[16];
    for (int e = 0; e < 16; ++e) p[e] = pack_bf16(A[r * K + k0 + 2 * e], A[r * K + k0 + 2 * e + 1]);
    tmem_st16(tbase + ((uint32_t)(warp * 32) << 16) + a_col + k0 / 2, p);
  }
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint64_t bd = smem_desc(smem_u32(sb), 1024, kSwizzle128);
    for (int kc = 0; kc < K / 64; ++kc)
      for (int k = 0; k < 4; ++k)
        mma_bf16_ts(tbase, tbase + a_col + kc * 32 + k * 8, bd + ((kc * N * 128 + k * 32) >> 4),
                    idesc_bf16(128, N), (kc | k) != 0);
    mma_commit(bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  tc_fence_after();
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

template <int H1, int H2, int NS>
std::vector<uint8_t> pack(const smlrt_model_s& m) {
  using L = Lay<H1, H2, NS>;
  std::vector<uint8_t> blob((size_t)L::BLOB * NS, 0);
  const int F = m.in_features;
  const float* W1 = m.host_params.data();
  const float* b1 = W1 + (size_t)H1 * F;
  const float* W2 = b1 + H1;
  const float* b2 = W2 + (size_t)H2 * H1;
  const float* W3 = b2 + H2;
  const float* b3 = W3 + H2;
  auto bf = [](float v) {  // value of the bf16 rounding of v
    uint32_t u = (uint32_t)f2bf(v) << 16;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
  };
  for (int rk = 0; rk < NS; ++rk) {
    uint8_t* base = blob.data() + (size_t)rk * L::BLOB;
    auto put = [&](size_t off, float v) {
      uint16_t h = f2bf(v);
      std::memcpy(base + off, &h, 2);
    };
    // B operands: this rank's N rows (rk * N/NS ...)
    for (int kc = 0; kc < L::KC; ++kc)
      for (int n = 0; n < L::N2; ++n)
        for (int k = 0; k < 64; ++k)
          put(kc * L::W2_CHUNK + sw128_offset(n, k), W2[(size_t)(rk * L::N2 + n) * H1 + kc * 64 + k]);
    const size_t o_w1 = L::BLOB_W1, o_w1b = o_w1 + L::N1 * 32, o_w2b = o_w1b + L::N1 * 32;
    for (int n = 0; n < L::N1; ++n) {
      const int gn = rk * L::N1 + n;
      for (int k = 0; k < KX; ++k) put(o_w1 + sw32_offset(n, k), k < F ? W1[(size_t)gn * F + k] : 0.0f);
      put(o_w1b + sw32_offset(n, 0), b1[gn]);
      put(o_w1b + sw32_offset(n, 1), b1[gn] - bf(b1[gn]));
    }
    for (int n = 0; n < L::N2; ++n) {
      const int gn = rk * L::N2 + n;
      put(o_w2b + sw32_offset(n, 0), b2[gn]);
      put(o_w2b + sw32_offset(n, 1), b2[gn] - bf(b2[gn]));
    }
    float* tail = reinterpret_cast<float*>(base + L::BLOB_TAIL);
    std::memcpy(tail, W3, H2 * 4);
    tail[H2] = b3[0];
  }
  return blob;
}

bool shape_is(const smlrt_model_s& m, int h1, int h2) {
  for (const auto& L : m.layers)
    if (L.kind != SMLRT_DENSE) return false;
  return m.n_layers == 3 && m.in_features <= KX && m.layers[0].out == h1 && m.layers[1].out == h2 &&
         m.layers[2].out == 1;
}

int num_sms() {
  int d = 0, n = 148;
  cudaGetDevice(&d);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
  return n;
}

// CTA-pair kernel (SMLRT_TC_PAIR=1); off by default: measured slower than the
// single-CTA kernel on bonds (1.24 ms vs 1.14 ms with the elect.sync issuer)
bool use_pair() {
  static const int v = [] {
    const char* e = std::getenv("SMLRT_TC_PAIR");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0;
}

template <int H1, int H2>
constexpr size_t pair_blob_off() {
  return ((size_t)Lay<H1, H2, 1>::BLOB + 1023) & ~size_t(1023);
}

template <int H1, int H2>
int launch(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs, const int32_t* in_dt,
           int n_in, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt, int n_out, int64_t r0,
           int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  if (n_in > 8 || n_out > 8) return SMLRT_E_UNSUPPORTED;
  const bool pair = use_pair();
  static int configured_mask = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured_mask & (1 << dev))) {
    SMLRT_CUDA(cudaFuncSetAttribute(mlp3_tc_kernel<H1, H2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    Lay<H1, H2, 1>::ALLOC));
    SMLRT_CUDA(cudaFuncSetAttribute(mlp3_tc_kernel<H1, H2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    Lay<H1, H2, 2>::ALLOC));
    configured_mask |= 1 << dev;
  }
  TcArgs a{};
  a.blob = reinterpret_cast<const uint8_t*>(m.tc_blob) + (pair ? pair_blob_off<H1, H2>() : 0);
  {
    const int F = m.in_features;
    const float* b1 = m.host_params.data() + (size_t)H1 * F;
    const float* b2 = b1 + H1 + (size_t)H2 * H1;
    const float* w3 = b2 + H2;
    std::memcpy(a.b1, b1, H1 * 4);
    std::memcpy(a.b2, b2, H2 * 4);
    std::memcpy(a.w3, w3, H2 * 4);
    a.b3 = w3[H2];
  }
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
  // fast gather: one f32 array of dense 16-float rows (a contiguous tile), 16-B aligned
  if (in.dense_rows && in.n_cols == 16 && in.ustride[0] == 16 && m.in_features == 16 &&
      in_dt[in.uarray] == SMLRT_F32) {
    const float* base = reinterpret_cast<const float*>(in_ptrs[in.uarray]) + in.col_off0;
    if ((reinterpret_cast<uintptr_t>(base) & 15) == 0) a.x_fast = base;
  }
  if (!pair) {
    const int grid = std::max(1, std::min(a.n_tiles, num_sms()));
    mlp3_tc_kernel<H1, H2, false><<<grid, ss_threads<false>(), Lay<H1, H2, 1>::ALLOC, s>>>(a, in, src, out, dst);
    count_launch();
  } else {
    const int pairs = (a.n_tiles + 1) / 2;
    const int grid = 2 * std::max(1, std::min(pairs, num_sms() / 2));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = Lay<H1, H2, 2>::ALLOC;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SMLRT_CUDA(cudaLaunchKernelEx(&cfg, mlp3_tc_kernel<H1, H2, true>, a, in, src, out, dst));
    count_launch();
  }
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
  if (int rc = chain_pack(m)) return rc;  // the generic fallback of every dense model
  if (int rc = small_mma_pack(m)) return rc;  // small 3-layer MLPs (warp-MMA kernel)
  if (wide_shape(m)) return wide_pack(m);
  // [single-CTA blob][pad to 1 KB][rank-0 blob][rank-1 blob]
  std::vector<uint8_t> blob, pair;
  size_t off = 0;
  if (shape_is(m, 256, 128)) {
    blob = pack<256, 128, 1>(m);
    pair = pack<256, 128, 2>(m);
    off = pair_blob_off<256, 128>();
  } else if (shape_is(m, 128, 64)) {
    blob = pack<128, 64, 1>(m);
    pair = pack<128, 64, 2>(m);
    off = pair_blob_off<128, 64>();

  } else {
    return SMLRT_OK;  // no tcgen05 kernel for this shape; region_infer reports it
  }
  blob.resize(off, 0);
  blob.insert(blob.end(), pair.begin(), pair.end());
  SMLRT_CUDA(cudaMalloc(&m.tc_blob, blob.size()));
  SMLRT_CUDA(cudaMemcpy(m.tc_blob, blob.data(), blob.size(), cudaMemcpyHostToDevice));
  m.tc_bytes = blob.size();
  return SMLRT_OK;
}

int launch_region_tc(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs, const int32_t* in_dt,
                     int n_in, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt, int n_out,
                     int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status, bool probe_only) {
  // probe_only: is there a shape-specialised fused kernel (the generic chain
  // is probed with chain_ok)
  if (probe_only)
    return m.precision == SMLRT_BF16 && (shape_is(m, 256, 128) || shape_is(m, 128, 64) || wide_shape(m))
               ? SMLRT_OK
               : SMLRT_E_UNSUPPORTED;
  // halo stencils over a 2-D sweep (C5 shape): the plan decides, not the model alone
  int rc = launch_region_stencil_tc(m, in, in_ptrs, in_dt, out, out_ptrs, out_dt, r0, r1, staged, s, status);
  if (rc != SMLRT_E_UNSUPPORTED) return rc;
  // small 3-layer MLPs (C1's 5-64-32-1 at bf16): one warp-MMA kernel with the
  // activations in registers (the bonds-family tcgen05 kernel instantiated at
  // 64-32 measured 63 us on C1 vs 36.5 us: its per-tile handshakes dominate)
  rc = launch_region_small_mma(m, in, in_ptrs, in_dt, out, out_ptrs, out_dt, r0, r1, staged, s, status);
  if (rc != SMLRT_E_UNSUPPORTED) return rc;
  if (m.tc_blob != nullptr) {
    if (wide_shape(m))
      rc = launch_region_wide(m, in, in_ptrs, in_dt, out, out_ptrs, out_dt, n_out, r0, r1, staged, s, status);
    else if (shape_is(m, 256, 128))
      rc = launch<256, 128>(m, in, in_ptrs, in_dt, n_in, out, out_ptrs, out_dt, n_out, r0, r1, staged, s, status);
    else if (shape_is(m, 128, 64))
      rc = launch<128, 64>(m, in, in_ptrs, in_dt, n_in, out, out_ptrs, out_dt, n_out, r0, r1, staged, s, status);
  }
  if (rc != SMLRT_E_UNSUPPORTED) return rc;
  // any other dense model (or plans the specialised kernels do not take)
  return launch_region_chain(m, in, in_ptrs, in_dt, n_in, out, out_ptrs, out_dt, n_out, r0, r1, staged, s, status);
}

}  // namespace smlrt

#ifdef SMLRT_TC_TRACE
extern "C" int smlrt_tc_trace_dump(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, smlrt::g_tc_trace, sizeof(smlrt::g_tc_trace)) == cudaSuccess ? 0 : -1;
}
#endif

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

extern "C" int smlrt_tc_selftest_ts(int K, int N, const float* A, const float* B, float* D) {
  using namespace smlrt;
  if (!(K % 64 == 0 && K <= 256) || !(N == 64 || N == 128 || N == 256))
    return fail(SMLRT_E_INVALID, "tc_selftest_ts: K in {64,128,192,256}, N in {64,128,256}");
  float *dA, *dB, *dD;
  SMLRT_CUDA(cudaMalloc(&dA, 128 * K * 4));
  SMLRT_CUDA(cudaMalloc(&dB, N * K * 4));
  SMLRT_CUDA(cudaMalloc(&dD, 128 * N * 4));
  SMLRT_CUDA(cudaMemcpy(dA, A, 128 * K * 4, cudaMemcpyHostToDevice));
  SMLRT_CUDA(cudaMemcpy(dB, B, N * K * 4, cudaMemcpyHostToDevice));
  const int smem = N * K * 2 + 64 + 1024;
  if (N == 64) {
    SMLRT_CUDA(cudaFuncSetAttribute(tc_selftest_ts_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc_selftest_ts_kernel<64><<<1, 128, smem>>>(dA, dB, K, dD);
  } else if (N == 128) {
    SMLRT_CUDA(cudaFuncSetAttribute(tc_selftest_ts_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc_selftest_ts_kernel<128><<<1, 128, smem>>>(dA, dB, K, dD);
  } else {
    SMLRT_CUDA(cudaFuncSetAttribute(tc_selftest_ts_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc_selftest_ts_kernel<256><<<1, 128, smem>>>(dA, dB, K, dD);
  }
  SMLRT_CUDA(cudaGetLastError());
  SMLRT_CUDA(cudaDeviceSynchronize());
  SMLRT_CUDA(cudaMemcpy(D, dD, 128 * N * 4, cudaMemcpyDeviceToHost));
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return SMLRT_OK;
}
