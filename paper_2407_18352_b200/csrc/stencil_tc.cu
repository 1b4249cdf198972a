// bf16 halo-stencil region on the tensor cores (C5 MiniWeather at bf16, and
// any region of the same shape): a 2-D sweep with unit inner stride whose
// in-functor gathers, per point (i, j), V variables x NDI rows x 3 columns
// around it -- [i, j, 0:V, 0:NDI, 0:3] = ([0:V, i-a:i-a+NDI, j-b:j-b+3]),
// `wrap_tensors` of bridge.py:288-344 -- into a 2-layer MLP (hidden <= 16,
// outputs <= 8) whose outputs the out-functor scatters per point.
//
// The fp32-exact kernel for this shape is bound by the FP32 pipe (ordered
// mul-then-add, 640 flop per point); at bf16 the work is 0.2 % of the tensor
// peak and the bound is HBM (16 B read + 16 B written per point) -- so the
// design minimises instructions and latency per point:
//   * thread 0 streams the input through a TMA ring: a stage holds, per
//     variable, one box of (BR + 2) input rows x 136 columns around the
//     CTA's 128-column tile (the 2 halo rows are re-read from L2, not HBM);
//     the next stage lands while the current one is consumed;
//   * each warp owns 32 columns = two m16 point tiles per row; the point
//     features go straight from shared memory into the A fragments of
//     warp-level MMAs: layer 1 on tf32 m16n8k8 (f32 operands unconverted,
//     K permuted so each lane reads one variable's rows with 8-B loads,
//     conflict-free), the bias as the accumulator's initial value; act +
//     bf16 packing of the accumulator IS the A fragment of layer 2 (the C and
//     A fragment layouts coincide), layer 2 one bf16 m16n8k16;
//   * the accumulators hold (point, output) pairs: stores go through the
//     out-plan (coalesced per output plane) or to the checked commit's
//     staging; for 4 outputs layer 2's columns 4..7 repeat 0..3 so every lane
//     stores two values with no predicate.
// Why not tcgen05 here: with one point per TMEM lane every 128 points need a
// tcgen05.st -> barrier -> MMA -> commit -> mbarrier wait -> tcgen05.ld
// round trip; measured on C5 that round trip bound the kernel at 0.2-0.4 ms
// whatever the staging (docs: DESIGN.md "C5 at bf16").  Warp-level MMAs keep
// operands and results in registers with no cross-warp handshake.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "simt_common.cuh"
#include "tc_ptx.cuh"
#include "stencil_common.cuh"

namespace smlrt {

int make_map_f32_3d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                    uint64_t s2, uint32_t b0, uint32_t b1, uint32_t b2, int promote);

namespace {

using namespace ptx;
using namespace stencil;

#ifndef SM_BR_
#define SM_BR_ 4
#endif
#ifndef SM_NS_
#define SM_NS_ 2
#endif
#ifndef SM_RB_
#define SM_RB_ 0
#endif
constexpr int SM_TW = 128;   // output columns per CTA: 4 warps x 2 m16 tiles
constexpr int SM_BOX = 132;  // TMA box width: the tile's 130 columns from a 16-B aligned start
constexpr int SM_BR = SM_BR_;  // output rows per stage
constexpr int SM_NS = SM_NS_;  // ring stages
constexpr int SM_RB = SM_RB_;  // output rows per CTA (0: sized for one wave of resident CTAs)
constexpr int SM_G = 8;        // max outputs (one n8 tile)
constexpr int SM_V = 4;        // variables (one per lane of a quad)
constexpr int SM_VROWS = SM_BR + 2;                 // staged input rows per variable
constexpr int SM_VF = SM_VROWS * SM_BOX;            // floats per variable in a stage
constexpr int SM_STAGE = SM_V * SM_VF;              // floats per stage (multiple of 32: 128-B aligned)
constexpr int SM_SMEM = 1024 + SM_NS * SM_STAGE * 4 + 64 + 256 + 2 * 5 * 256 + 96;
static_assert(SM_STAGE % 32 == 0, "stages stay 128-B aligned");
static_assert((SM_VF % 32) == 24 || (SM_VF % 32) == 8, "variables land on distinct bank octets");

struct SmArgs {
  int32_t c0, r0v, p0v;  // box origin: column (16-B aligned), row of var 0's first input row, plane of var 0
  int32_t al;            // tile point 0's left halo column within the box
  int64_t nj;            // sweep columns
  int64_t i_begin, i_end;
  int64_t rb;            // output rows per CTA
  float* dst;            // out-plan's array (uniform, f32)
  int64_t ocol[SM_G];
  int64_t o0, o1;        // out-plan sweep strides
  int64_t r0;            // first sweep row of the call (staged index base)
  float* staged;         // checked commit: [rows][G] f32
  uint32_t* status;
  int act2, g;
  uint32_t w1f[2][5][32][2];  // layer-1 tf32 B fragments per n8 tile, k8 step, lane (permuted K)
  uint32_t w2f[32][2];        // layer-2 B fragment per lane
  float b1[16];               // layer-1 bias (accumulator init), zero padded
  float b2[SM_G];
};

#ifdef SM_MMA_VOLATILE
#define SM_MMA_ASM asm volatile
#else
#define SM_MMA_ASM asm
#endif
__device__ __forceinline__ void mma_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                          const float (&c)[4]) {
  SM_MMA_ASM(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%11,%12,%13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c[0]), "f"(c[1]), "f"(c[2]),
        "f"(c[3]));
}

__device__ __forceinline__ float sm_act(float y, int act) {
  if (act == SMLRT_RELU) return relu_nan(y);
  if (act == SMLRT_TANH) return tanhf(y);
  return y;
}
template <int ACT>
__device__ __forceinline__ uint32_t sm_act_pack(float lo, float hi) {
  if constexpr (ACT == SMLRT_RELU) return pack_relu_bf16(lo, hi);
  else if constexpr (ACT == SMLRT_TANH) return pack_bf16(tanhf(lo), tanhf(hi));
  else return pack_bf16(lo, hi);
}
// predicated global store (no branch around a lane-divergent condition)
__device__ __forceinline__ void stg_if(bool p, float* addr, float v) {
  asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %0, 0;\n@q st.global.f32 [%1], %2;\n}\n" ::"r"((int)p), "l"(addr),
               "f"(v)
               : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// Layer 1 runs on tf32 MMAs (m16n8k8): the f32 features go from shared
// memory into the A fragments unconverted (tf32 keeps 10 mantissa bits, more
// than bf16's 7).  Quad member q = v holds its variable's 9 features; a
// lane's two 8-B loads of a (variable, di) row give columns 2g .. 2g+3 =
// (dj0, dj1, dj2) of point 2g and of point 2g+1.  K is permuted so those
// registers ARE the fragments: k8 step di (0..2) = (dj0, dj2) of row di --
// a0 a1 = first load, a2 a3 = second load; steps 3 and 4 = the dj1 columns
// of rows (0, 1) and (2, padding).  K = 40.  One LDS reads one row of four
// variables for 8 point pairs -- four planes 24 banks apart: conflict-free.
constexpr int SM_KS = 5;
// MMA k of feature (v, di, dj)
__host__ __device__ constexpr int sm_kpos(int v, int di, int dj) {
  return dj != 1 ? 8 * di + v + (dj == 2 ? 4 : 0) : 8 * (3 + di / 2) + v + 4 * (di % 2);
}

__device__ __forceinline__ void mma_1688_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                              const float (&c)[4]) {
  SM_MMA_ASM(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%11,%12,%13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c[0]), "f"(c[1]), "f"(c[2]),
        "f"(c[3]));
}

#ifndef SM_MINB
#define SM_MINB 4
#endif
template <int NT1, int ACT1, bool G4>
__global__ void __launch_bounds__(128, SM_MINB) stencil_mma_kernel(const __grid_constant__ CUtensorMap tm,
                                                             const __grid_constant__ SmArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // (indexing the __shared__ array keeps the loads in the shared window: LDS, ordered after the waits)
  float* ring = reinterpret_cast<float*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + SM_NS * SM_STAGE);
  // per-lane MMA B fragments go through shared memory: kernel-parameter
  // reads indexed by lane serialise (one constant-bank address per lane)
  uint32_t* w2s = reinterpret_cast<uint32_t*>(full + SM_NS);  // layer-2 [32][2]
  uint32_t* w1s = w2s + 64;                                    // layer-1 [NT1][KS][32][2]
  float* bs = reinterpret_cast<float*>(w1s + 2 * SM_KS * 64);  // b1 [16], b2 [8]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  if (tid < 64) w2s[tid] = a.w2f[tid >> 1][tid & 1];
  for (int k = tid; k < NT1 * SM_KS * 64; k += 128) w1s[k] = (&a.w1f[0][0][0][0])[k];
  if (tid < 16) bs[tid] = a.b1[tid];
  if (tid < SM_G) bs[16 + tid] = a.b2[tid];

  const int64_t jb = (int64_t)blockIdx.x * SM_TW;  // sweep column of the tile's first point
  const int64_t i0 = a.i_begin + (int64_t)blockIdx.y * a.rb;
  const int64_t i1 = min(i0 + a.rb, a.i_end);
  const int nblk = (int)((i1 - i0 + SM_BR - 1) / SM_BR);
  auto issue = [&](int b) {  // thread 0: output-row block b's input rows (+2 halo) of all variables
    const int st = b % SM_NS;
    sm_expect_tx(full + st, SM_STAGE * 4);
    sm_tma(smem_u32(ring + st * SM_STAGE), &tm, full + st, a.c0 + (int)jb, (int)(a.r0v + i0 + b * SM_BR), a.p0v);
  };
  if (tid == 0) {
    for (int k = 0; k < SM_NS; ++k) mbar_init(full + k, 1);
    mbar_fence_init();
    for (int b = 0; b < min(nblk, SM_NS); ++b) issue(b);
  }

  // MMA rows g and g + 8 of a 16-point tile are the points 2g and 2g + 1
  // (a row permutation of A and D): this lane's four input columns 2g .. 2g+3
  // of a (variable, di) row are two 8-B aligned LDS.64 for both points.
  // Lane quad member q reads variable q, whose planes sit 24 banks apart.
  // layer 2's accumulator columns (2q, 2q+1); with G4 columns 4..7 repeat
  // outputs 0..3 so that every lane stores: quad member q writes outputs
  // 2(q&1), 2(q&1)+1 of point 2g + (q>>1)
  const int o_lo = G4 ? 2 * (q & 1) : 2 * q, o_hi = o_lo + 1;
  const bool has_lo = o_lo < a.g, has_hi = o_hi < a.g;
  // outputs: element (row i, column js, output o) at out + i*RI + js*RJ + oc[o]
  // -- the out-plan's array, or the checked commit's [rows][G] staging
  const bool stg = a.staged != nullptr;
  const int64_t RI = stg ? a.nj * a.g : a.o0, RJ = stg ? a.g : a.o1;
  const int64_t oc_lo = has_lo ? (stg ? o_lo : a.ocol[o_lo]) : 0, oc_hi = has_hi ? (stg ? o_hi : a.ocol[o_hi]) : 0;
  const int64_t js_lane = jb + warp * 32 + 2 * g + (G4 ? (q >> 1) : 0);  // this lane's (first) point, tile 0
  float* const olane = (stg ? a.staged - a.r0 * a.g : a.dst) + js_lane * RJ;
  float* const plo = olane + oc_lo;  // output o_lo of the lane's point, row 0 (rows add i * RI)
  const int64_t dhi = oc_hi - oc_lo;
  const int64_t t16 = 16 * RJ;
  const int64_t nj = a.nj;
  const bool full_cols = jb + SM_TW <= nj;  // every point of the CTA tile is in the sweep
  const int act2 = a.act2;
  __syncthreads();  // barrier init and the fragment tables visible before use
  float c1[NT1][4];
#pragma unroll
  for (int t = 0; t < NT1; ++t) {
    c1[t][0] = c1[t][2] = bs[8 * t + 2 * q];
    c1[t][1] = c1[t][3] = bs[8 * t + 2 * q + 1];
  }
  const float c2[4] = {has_lo ? bs[16 + o_lo] : 0.0f, has_hi ? bs[16 + o_hi] : 0.0f, has_lo ? bs[16 + o_lo] : 0.0f,
                       has_hi ? bs[16 + o_hi] : 0.0f};
  uint32_t w1[NT1][SM_KS][2];
#pragma unroll
  for (int t = 0; t < NT1; ++t)
#pragma unroll
    for (int s = 0; s < SM_KS; ++s) {
      w1[t][s][0] = w1s[((t * SM_KS + s) * 32 + lane) * 2];
      w1[t][s][1] = w1s[((t * SM_KS + s) * 32 + lane) * 2 + 1];
    }

  float chk = 0.0f;  // y * 0 accumulates NaN iff some stored output is non-finite
  const float* lane_ring = ring + q * SM_VF + a.al + 2 * g + warp * 32;
  // one m16 tile: points 2g, 2g+1 (+16 t2) of input-stage row r; orow = the
  // lane's output pointer for this row
  auto tile = [&](auto full_tile, const float* sb, int r, int t2, float* orow, uint32_t w2a, uint32_t w2b) {
    float d1[NT1][4];
#pragma unroll
    for (int t = 0; t < NT1; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) d1[t][e] = c1[t][e];
    float2 u[3], w[3];  // row di: (dj0, dj1 | dj1, dj2) of point 2g = u.x, u.y, w.x; of 2g+1 = u.y, w.x, w.y
#pragma unroll
    for (int di = 0; di < 3; ++di) {
      const float* ra = sb + (r + di) * SM_BOX + t2 * 16;
      u[di] = *reinterpret_cast<const float2*>(ra);
      w[di] = *reinterpret_cast<const float2*>(ra + 2);
    }
#pragma unroll
    for (int s2 = 0; s2 < SM_KS; ++s2) {
      uint32_t af[4];
      if (s2 < 3) {  // (dj0, dj2) of row s2
        af[0] = __float_as_uint(u[s2].x), af[1] = __float_as_uint(u[s2].y);
        af[2] = __float_as_uint(w[s2].x), af[3] = __float_as_uint(w[s2].y);
      } else {  // dj1 of rows 2(s2-3), 2(s2-3)+1
        const int da = 2 * (s2 - 3), db = da + 1;
        af[0] = __float_as_uint(u[da].y), af[1] = __float_as_uint(w[da].x);
        af[2] = db < 3 ? __float_as_uint(u[db].y) : 0u;
        af[3] = db < 3 ? __float_as_uint(w[db].x) : 0u;
      }
#pragma unroll
      for (int t = 0; t < NT1; ++t) mma_1688_tf32(d1[t], af, w1[t][s2][0], w1[t][s2][1], d1[t]);
    }
    // act1 + bf16: the layer-1 accumulators are layer 2's A fragment
    const uint32_t a2[4] = {sm_act_pack<ACT1>(d1[0][0], d1[0][1]), sm_act_pack<ACT1>(d1[0][2], d1[0][3]),
                            NT1 > 1 ? sm_act_pack<ACT1>(d1[NT1 - 1][0], d1[NT1 - 1][1]) : 0u,
                            NT1 > 1 ? sm_act_pack<ACT1>(d1[NT1 - 1][2], d1[NT1 - 1][3]) : 0u};
    float y[4];
    mma_16816(y, a2, w2a, w2b, c2);
    if (act2 != SMLRT_IDENTITY) {
#pragma unroll
      for (int e = 0; e < 4; ++e) y[e] = sm_act(y[e], act2);
    }
    float* op = orow + t2 * t16;
    constexpr bool FULL = decltype(full_tile)::value;
    if constexpr (G4) {
      // y = (point 2g: col 2q, 2q+1), (point 2g+1: ...); this lane stores point 2g + (q>>1)
      const float ya = q < 2 ? y[0] : y[2], yb = q < 2 ? y[1] : y[3];
      if (FULL || js_lane + t2 * 16 < nj) {
        op[0] = ya;
        op[dhi] = yb;
        chk = fmaf(ya, 0.0f, chk);
        chk = fmaf(yb, 0.0f, chk);
      }
    } else {
      // y = (point 2g: o_lo, o_hi), (point 2g+1: o_lo, o_hi)
      bool v0 = has_lo, v1 = has_lo, w0 = has_hi, w1v = has_hi;
      if (!FULL) {
        const int64_t js0 = js_lane + t2 * 16;
        v0 &= js0 < nj, w0 &= js0 < nj, v1 &= js0 + 1 < nj, w1v &= js0 + 1 < nj;
      }
      stg_if(v0, op, y[0]);
      stg_if(v1, op + RJ, y[2]);
      stg_if(w0, op + dhi, y[1]);
      stg_if(w1v, op + dhi + RJ, y[3]);
      chk = fmaf(v0 ? y[0] : 0.0f, 0.0f, chk);
      chk = fmaf(v1 ? y[2] : 0.0f, 0.0f, chk);
      chk = fmaf(w0 ? y[1] : 0.0f, 0.0f, chk);
      chk = fmaf(w1v ? y[3] : 0.0f, 0.0f, chk);
    }
  };
  using full_t = std::integral_constant<bool, true>;
  using part_t = std::integral_constant<bool, false>;
  for (int b = 0; b < nblk; ++b) {
    const int st = b % SM_NS;
    sm_wait(full + st, (uint32_t)(b / SM_NS) & 1u);
    const uint32_t w2a = w2s[2 * lane], w2b = w2s[2 * lane + 1];
    const int64_t ib = i0 + (int64_t)b * SM_BR;
    const float* sb = lane_ring + st * SM_STAGE;
    if (ib + SM_BR <= i1 && full_cols) {  // whole stage, every column in the sweep: no guards
#pragma unroll
      for (int r = 0; r < SM_BR; ++r) {
        float* orow = plo + (ib + r) * RI;
#pragma unroll
        for (int t2 = 0; t2 < 2; ++t2) tile(full_t{}, sb, r, t2, orow, w2a, w2b);
      }
    } else {
      const int nr = i1 - ib < SM_BR ? (int)(i1 - ib) : SM_BR;
#pragma unroll 1
      for (int r = 0; r < nr; ++r) {
        float* orow = plo + (ib + r) * RI;
#pragma unroll
        for (int t2 = 0; t2 < 2; ++t2) tile(part_t{}, sb, r, t2, orow, w2a, w2b);
      }
    }
    __syncthreads();  // every warp is done with stage st
    if (tid == 0 && b + SM_NS < nblk) issue(b + SM_NS);
  }
  const bool bad = chk != chk;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.status, SMLRT_STATUS_NONFINITE);
}

// round-to-nearest-even bf16 bits of a finite f32 (weights are checked finite at load)
uint32_t sm_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return u >> 16;
}
uint32_t sm_pair(float lo, float hi) { return sm_bf16(lo) | (sm_bf16(hi) << 16); }

// tf32 (round to nearest even, 10 mantissa bits) bits of a finite f32
uint32_t sm_tf32(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0xfffu + ((u >> 13) & 1u);
  return u & ~0x1fffu;
}

template <int NT1, int ACT1, bool G4>
int launch_sm(const smlrt_model_s& m, const DevPlan& in, const void* src, const DevPlan& out, void* dst,
              int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  SmArgs a{};
  StencilGeom geo;
  if (!stencil_geom(in, SM_BOX - SM_TW - 2, &geo)) return SMLRT_E_UNSUPPORTED;
  const int64_t P = geo.plane;
  a.c0 = geo.c0;
  a.r0v = geo.r0v;
  a.p0v = geo.p0v;
  a.al = geo.al;
  const int64_t nj = (int64_t)in.sdiv[1].d, s0 = in.ustride[0];
  if (r0 % nj != 0 || (r1 % nj != 0 && r1 != in.n_rows)) return SMLRT_E_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(src) & 15) != 0) return SMLRT_E_UNSUPPORTED;
  CUtensorMap tm;
  if (make_map_f32_3d(&tm, src, (uint64_t)s0, (uint64_t)(P / s0), (uint64_t)(in.uarray_numel / P),
                      (uint64_t)s0 * 4, (uint64_t)P * 4, SM_BOX, SM_VROWS, SM_V, 0) != SMLRT_OK)
    return SMLRT_E_UNSUPPORTED;
  const DevLayer &L1 = m.layers[0], &L2 = m.layers[1];
  const int H = L1.out, G = L2.out, Fi = L1.in;
  a.nj = nj;
  a.i_begin = r0 / nj;
  a.i_end = (r1 + nj - 1) / nj;
  a.dst = static_cast<float*>(dst);
  for (int o = 0; o < G; ++o) a.ocol[o] = out.col_inl[o];
  a.o0 = out.ustride[0];
  a.o1 = out.ustride[1];
  a.r0 = r0;
  a.staged = staged;
  a.status = status;
  a.act2 = L2.act;
  a.g = G;
  const float* p = m.host_params.data();  // [W1][b1][W2][b2]
  const float* W1 = p;
  const float* b1 = W1 + (size_t)H * Fi;
  const float* W2 = b1 + H;
  const float* b2 = W2 + (size_t)G * H;
  // W1 over the permuted K: kfeat[k] = the feature at MMA position k (-1: padding)
  int kfeat[8 * SM_KS];
  for (int k = 0; k < 8 * SM_KS; ++k) kfeat[k] = -1;
  for (int v = 0; v < 4; ++v)
    for (int mm = 0; mm < 9; ++mm) kfeat[sm_kpos(v, mm / 3, mm % 3)] = v * 9 + mm;
  auto w1 = [&](int n, int k) { return n < H && kfeat[k] >= 0 ? W1[(size_t)n * Fi + kfeat[k]] : 0.0f; };
  // with G4 the layer-2 columns 4..7 repeat outputs 0..3
  auto w2 = [&](int o, int h) {
    const int oo = G4 ? (o & 3) : o;
    return oo < G && h < H ? W2[(size_t)oo * H + h] : 0.0f;
  };
  for (int l = 0; l < 32; ++l) {
    const int gg = l >> 2, qq = l & 3;
    for (int t = 0; t < NT1; ++t)
      for (int st = 0; st < SM_KS; ++st) {
        const int k = 8 * st + qq, n = 8 * t + gg;  // tf32 B fragment: (k, n), (k + 4, n) of col-major W1^T
        a.w1f[t][st][l][0] = sm_tf32(w1(n, k));
        a.w1f[t][st][l][1] = sm_tf32(w1(n, k + 4));
      }
    a.w2f[l][0] = sm_pair(w2(gg, 2 * qq), w2(gg, 2 * qq + 1));
    a.w2f[l][1] = sm_pair(w2(gg, 2 * qq + 8), w2(gg, 2 * qq + 9));
  }
  for (int k = 0; k < H; ++k) a.b1[k] = b1[k];
  for (int o = 0; o < G; ++o) a.b2[o] = b2[o];
  static bool configured = false;
  if (!configured) {
    SMLRT_CUDA(cudaFuncSetAttribute(stencil_mma_kernel<NT1, ACT1, G4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    SM_SMEM));
    configured = true;
  }
  const int64_t rows = a.i_end - a.i_begin;
  // rows per CTA: one wave of resident CTAs (each streams its rows through
  // the TMA ring without a second prologue), at least 2 stages
  const int64_t ncb = (nj + SM_TW - 1) / SM_TW;
  static int slots = 0;
  if (!slots) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    SMLRT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stencil_mma_kernel<NT1, ACT1, G4>, 128, SM_SMEM));
    slots = std::max(1, per_sm) * sms;
  }
  int64_t rb = SM_RB;
  if (rb <= 0) {
    const int64_t ny = std::max<int64_t>(1, slots / ncb);
    rb = (rows + ny - 1) / ny;
    rb = std::max<int64_t>(2 * SM_BR, (rb + SM_BR - 1) / SM_BR * SM_BR);
  }
  a.rb = rb;
  dim3 grid((unsigned)ncb, (unsigned)((rows + rb - 1) / rb));
  stencil_mma_kernel<NT1, ACT1, G4><<<grid, 128, SM_SMEM, s>>>(tm, a);
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

}  // namespace

// bf16 region through the stencil kernel, or SMLRT_E_UNSUPPORTED when the
// model / plans do not have its shape (2 dense layers 36 -> <= 16 -> <= 8,
// f32 arrays, the 4-variable 3x3 halo in-plan, a uniform out-plan over the
// same 2-D sweep)
int launch_region_stencil_tc(const smlrt_model_s& m, const DevPlan& in, const void* const* in_ptrs,
                             const int32_t* in_dt, const DevPlan& out, void* const* out_ptrs, const int32_t* out_dt,
                             int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  if (m.n_layers != 2 || m.layers[0].kind != SMLRT_DENSE || m.layers[1].kind != SMLRT_DENSE) return SMLRT_E_UNSUPPORTED;
  if (m.layers[0].in != 36 || m.layers[0].out > 16 || m.layers[1].out > SM_G) return SMLRT_E_UNSUPPORTED;
  if (!in.uniform || !out.uniform || in.n_sweep != 2 || out.n_sweep != 2) return SMLRT_E_UNSUPPORTED;
  if (in_dt[in.uarray] != SMLRT_F32 || out_dt[out.uarray] != SMLRT_F32) return SMLRT_E_UNSUPPORTED;
  if (out.sdiv[0].d != in.sdiv[0].d || out.sdiv[1].d != in.sdiv[1].d || out.n_cols > SMLRT_INLINE_COLS)
    return SMLRT_E_UNSUPPORTED;
  if (r1 <= r0) return SMLRT_OK;
  const void* src = in_ptrs[in.uarray];
  void* dst = out_ptrs[out.uarray];
  const int act = m.layers[0].act;
  const bool g4 = m.layers[1].out == 4;
#define SM_GO(NT, A)                                                                                    \
  return g4 ? launch_sm<NT, A, true>(m, in, src, out, dst, r0, r1, staged, s, status)                  \
            : launch_sm<NT, A, false>(m, in, src, out, dst, r0, r1, staged, s, status)
  if (m.layers[0].out <= 8) {
    if (act == SMLRT_RELU) SM_GO(1, SMLRT_RELU);
    if (act == SMLRT_TANH) SM_GO(1, SMLRT_TANH);
    SM_GO(1, SMLRT_IDENTITY);
  }
  if (act == SMLRT_RELU) SM_GO(2, SMLRT_RELU);
  if (act == SMLRT_TANH) SM_GO(2, SMLRT_TANH);
  SM_GO(2, SMLRT_IDENTITY);
#undef SM_GO
}

}  // namespace smlrt
