// bf16 fused region for small dense MLPs on the 5th-generation tensor cores
// (C1 options at bf16, and any 3-layer model F <= 8 -> H1 <= 64 -> H2 <= 64
// -> G <= 8 over a 1-D sweep): gather -> forward -> scatter in one kernel.
//
// The reference's forward pass per row (models.py:197-224, _matmul_rowwise
// models.py:188-194) is three dense layers; at these widths a 128-row tile
// is ~1 us of tensor work split into two tiny MMAs, so the kernel is built
// around latency, not tensor throughput:
//   * one CTA = one 128-row chain: thread t owns row t = TMEM lane t.  Its
//     packed row of F <= 6 features goes straight from global memory
//     (prefetched one tile ahead in registers) into a 32-B-per-row SW32 tile
//     of tf32 values; K columns 6 and 7 hold 1.0 and their weights are
//     tf32(b1) and tf32(b1 - tf32(b1)), so layer 1's bias rides in the MMA
//     at ~f32 precision;
//   * layer 1: one kind::tf32 MMA M=128 N=H1 K=8 -> TMEM;
//   * each thread drains its lane (tcgen05.ld), act + bf16 pack, and stores
//     the packed pairs back into the SAME lane's TMEM columns (tcgen05.st):
//     they are layer 2's A operand (TS form), no shared-memory round trip;
//   * layer 2: H1/16 kind::f16 TS MMAs M=128 N=H2 into the columns after A2;
//   * layer 3 (G <= 8 outputs): act(acc2 + b2) as bf16 pairs back into the
//     lane's TMEM, one more TS MMA chain M=128 N=16 (measured equal to
//     packed f32x2 FMAs on the FP32 pipe, with 40 fewer instructions per 32
//     rows);
//   * 8 chains per SM (4 for H2 = 64: 64 / 128 TMEM columns each), one per
//     CTA by default (STC_CPS), interleave with no cross-chain handshakes.
// Quantisation points are those of the warp-MMA kernel (small_mma.cu), so
// both are checked against one emulation (tests/test_gpu_small_mma.py).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "simt_common.cuh"
#include "tc_ptx.cuh"

namespace smlrt {
namespace {

using namespace ptx;

constexpr int STC_G = 8, STC_F = 6, STC_H = 64;  // F <= 6: K = 8 holds the features and two bias columns

struct StcArgs {
  int64_t r0, r1;
  const float* src;     // row 0's first feature: packed rows of F floats
  float* obase;  // out-plan array, or the checked commit's staging shifted by -r0 * g
  uint32_t* status;
  const uint8_t* blob;  // [W1 (K = 8 tf32)][W2 K16-blocks][W3 K16-blocks] (bf16), SW32 images
  int64_t op;           // output element step per sweep row
  int64_t ocol[STC_G];  // output column offsets (out-plan, or 0..g-1 staged)
  int F, g, act3;
  alignas(8) float b2[STC_H];
  float b3[STC_G];
};

__host__ __device__ constexpr int stc_cols(int n1, int n2) {
  const int need = n1 > n1 / 2 + n2 ? n1 : n1 / 2 + n2;
  return need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : 256;
}
// 128-row chains per SM (all of TMEM, at most 8) and per CTA (STC_CPS)
#ifndef STC_CPS
#define STC_CPS 1  // C1 bf16: 1 / 2 / 8 chains per CTA equal (18.5 us); before the uniform warp index 1 was fastest
#endif
__host__ __device__ constexpr int stc_sm_chains(int n1, int n2) {
  return 512 / stc_cols(n1, n2) < 8 ? 512 / stc_cols(n1, n2) : 8;
}
__host__ __device__ constexpr int stc_chains(int n1, int n2) {
  return stc_sm_chains(n1, n2) < STC_CPS ? stc_sm_chains(n1, n2) : STC_CPS;
}

template <int ACT>
__device__ __forceinline__ uint32_t stc_pack(float lo, float hi) {
  if constexpr (ACT == SMLRT_RELU) return pack_relu_bf16(lo, hi);
  else if constexpr (ACT == SMLRT_TANH) return pack_bf16(tanhf(lo), tanhf(hi));
  else return pack_bf16(lo, hi);
}
__device__ __forceinline__ float stc_act(float y, int act) {
  if (act == SMLRT_RELU) return relu_nan(y);
  if (act == SMLRT_TANH) return tanhf(y);
  return y;
}
__device__ __forceinline__ uint64_t stc_pair(float lo, float hi) {
  return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ uint64_t stc_add2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// SW32 K-major: 32-B rows, 16-B chunk c of row r at chunk c ^ ((r >> 2) & 1)
__device__ __forceinline__ uint32_t sw32_chunk(uint32_t row, uint32_t c) {
  return row * 32u + ((c ^ ((row >> 2) & 1u)) << 4);
}

template <int NCH>
__device__ __forceinline__ void stc_chain_sync(int chain) {  // the chain's 4 warps (named barrier 1 + chain)
  if constexpr (NCH == 1)
    __syncthreads();  // a constant barrier id: a runtime one reserves all 16 and caps CTAs per SM
  else
    asm volatile("bar.sync %0, 128;" ::"r"(chain + 1) : "memory");
}

// NCH chains per CTA (STC_CPS), 8 / NCH CTAs per SM.  A kernel that may
// allocate TMEM gets a new CTA on an SM only after the resident ones have
// released their allocation permit (tools/tmem_occupancy.cu: 8 x 20-us CTAs
// per SM holding 64 columns each take 47 us, not 20), so the allocation is
// the kernel's first instruction; one 8-chain CTA per SM has no launch ramp
// at all but runs each tile slower (named barriers of one CTA, its MMAs in
// one issue order): 1 chain per CTA is the fastest on C1 (22.2 vs 24.6 us)
template <int N1, int N2, int ACT, int GP>
__global__ void __launch_bounds__(128 * stc_chains(N1, N2), stc_sm_chains(N1, N2) / stc_chains(N1, N2)) small_tc_kernel(const __grid_constant__ StcArgs a) {
  constexpr int TC = stc_cols(N1, N2), NCH = stc_chains(N1, N2);
  constexpr int W1B = N1 * 32, W2B = N2 * 32, K2 = N1 / 16;
  constexpr int A2C = 0, D2C = N1 / 2;  // TMEM columns: A2 over acc1's drained half, acc2 after it
  // layer 3: A3 = the packed bf16 layer-2 activations over the
  // dead A2 columns [0, N2/2), acc3 (16 columns, G <= 8 used) after A3
  constexpr int A3C = 0, D3C = N2 / 2, K3 = N2 / 16, W3B = 16 * 32;
  static_assert(D3C + 16 <= TC, "acc3 fits the allocation");
  __shared__ __align__(1024) uint8_t sA1[NCH][128 * 32];
  __shared__ __align__(1024) uint8_t sW[W1B + K2 * W2B + K3 * W3B];
  __shared__ __align__(8) uint64_t bar[NCH][3];
  __shared__ uint32_t slot;
  // the warp index through a shuffle from lane 0 is warp-uniform to the
  // compiler: the TMEM addresses below live in uniform registers (no R2UR
  // per tcgen05.ld/st) and the issuing-warp branches are uniform
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int ch = warp >> 2, ct = tid & 127, wq = warp & 3;  // chain, row in the tile, TMEM lane quarter
  if (warp == 0) tmem_alloc(&slot, TC * NCH);  // first: releases the allocation permit early
  const uint32_t a1s = smem_u32(sA1[ch]), ws = smem_u32(sW);
  const uint64_t a1d = smem_desc(a1s, 256, kSwizzle32);
  const uint64_t w1d = smem_desc(ws, 256, kSwizzle32);
  const uint64_t w2d = smem_desc(ws + W1B, 256, kSwizzle32);
  const uint64_t w3d = smem_desc(ws + W1B + K2 * W2B, 256, kSwizzle32);
  constexpr uint32_t id3 = idesc_bf16(128, 16);
  constexpr uint32_t id1 = idesc_tf32(128, N1), id2 = idesc_bf16(128, N2);

  const int64_t ntiles = (a.r1 - a.r0 + 127) / 128;
  const int F = a.F;
  float chk = 0.0f;  // y * 0 accumulates NaN iff an output is non-finite
  // this thread's row and pointers, advanced by the grid stride per tile;
  // rows past the end re-read the last row (their outputs are not stored)
  const int64_t tile0 = (int64_t)blockIdx.x * NCH + ch, tstep = (int64_t)gridDim.x * NCH;
  int64_t row = a.r0 + tile0 * 128 + ct;
  const int64_t step = tstep * 128;
  const float* const plast = a.src + (a.r1 - 1) * F;
  const float* pi = a.src + row * F;
  float* po = a.obase + row * a.op;
  const int64_t ostep = step * a.op;
  float x[STC_F];
  auto load = [&](const float* p) {
    p = p < plast ? p : plast;
#pragma unroll
    for (int f = 0; f < STC_F; ++f) x[f] = f < F ? __ldg(p + f) : 0.0f;
  };
  load(pi);  // the first tile's features in flight during the prologue below
  {  // weights -> shared memory (once per SM): every load in flight before the first store
    constexpr int NV = (W1B + K2 * W2B + K3 * W3B) / 16, NT = 128 * NCH, PER = (NV + NT - 1) / NT;
    const int4* g = reinterpret_cast<const int4*>(a.blob);
    int4* d = reinterpret_cast<int4*>(sW);
    int4 t[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j)
      if (tid + NT * j < NV) t[j] = __ldg(g + tid + NT * j);
#pragma unroll
    for (int j = 0; j < PER; ++j)
      if (tid + NT * j < NV) d[tid + NT * j] = t[j];
  }
  if (ct == 0) {
    mbar_init(&bar[ch][0], 1);
    mbar_init(&bar[ch][1], 1);
    mbar_init(&bar[ch][2], 1);
    mbar_fence_init();
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot + ch * TC;                   // this chain's columns
  const uint32_t my = tb + ((uint32_t)(wq * 32) << 16);  // this warp's 32 lanes of them
  int it = 0;
  for (int64_t tile = tile0; tile < ntiles; tile += tstep, ++it) {
    // ---- layer-1 A tile: tf32 features (truncated as the MMA reads them) in
    // K columns 0..F-1, zeros up to 5, 1.0 in the bias columns 6 and 7
    constexpr uint32_t kOne = 0x3F800000u, kT = 0xFFFFE000u;
    st_shared_v4(a1s + sw32_chunk(ct, 0), __float_as_uint(x[0]) & kT, __float_as_uint(x[1]) & kT,
                 __float_as_uint(x[2]) & kT, __float_as_uint(x[3]) & kT);
    st_shared_v4(a1s + sw32_chunk(ct, 1), __float_as_uint(x[4]) & kT, __float_as_uint(x[5]) & kT, kOne, kOne);
    pi += step * F;
    load(pi);  // next tile's features in flight during this tile's chain
    fence_async_smem();
    tc_fence_before();
    stc_chain_sync<NCH>(ch);
    if (wq == 0) {
      tc_fence_after();
      mma_tf32_ss_elect(tb, a1d, w1d, id1, 0);
      mma_commit_elect(&bar[ch][0]);
      mbar_wait_sleep(&bar[ch][0], it & 1);  // the issuing warp waits; the others sleep in the barrier
    }
    stc_chain_sync<NCH>(ch);
    tc_fence_after();
    // ---- layer-1 epilogue: act + bf16 pairs back into this lane's columns (layer 2's A)
#pragma unroll
    for (int c = 0; c < N1; c += 16) {
      uint32_t r[16], p[8];
      tmem_ld16(my + c, r);
      tmem_wait_ld16(r);
#pragma unroll
      for (int e = 0; e < 8; ++e) p[e] = stc_pack<ACT>(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
      tmem_st8(my + A2C + c / 2, p);  // columns [c/2, c/2 + 8) of acc1 were drained by this or an earlier chunk
    }
    tmem_wait_st();
    tc_fence_before();
    stc_chain_sync<NCH>(ch);
    if (wq == 0) {
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < K2; ++k) mma_ts_elect(tb + D2C, tb + A2C + 8 * k, w2d + ((k * W2B) >> 4), id2, k > 0);
      mma_commit_elect(&bar[ch][1]);
      mbar_wait_sleep(&bar[ch][1], it & 1);
    }
    stc_chain_sync<NCH>(ch);
    tc_fence_after();
    // ---- layer-2 epilogue: act(acc2 + b2) as bf16 pairs into this lane's
    // A3 columns, then one N = 16 TS MMA chain (K = N2) gives the G outputs
    const uint64_t* b2p = reinterpret_cast<const uint64_t*>(a.b2);
#pragma unroll
    for (int c = 0; c < N2; c += 16) {
      uint32_t r[16], h[8];
      tmem_ld16(my + D2C + c, r);
      tmem_wait_ld16(r);
#pragma unroll
      for (int e = 0; e < 16; e += 2) {
        const uint64_t z = stc_add2(stc_pair(__uint_as_float(r[e]), __uint_as_float(r[e + 1])), b2p[(c + e) / 2]);
        h[e / 2] = stc_pack<ACT>(__uint_as_float((uint32_t)z), __uint_as_float((uint32_t)(z >> 32)));
      }
      tmem_st8(my + A3C + c / 2, h);  // columns below D2C + c: already drained
    }
    tmem_wait_st();
    tc_fence_before();
    stc_chain_sync<NCH>(ch);
    if (wq == 0) {
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < K3; ++k) mma_ts_elect(tb + D3C, tb + A3C + 8 * k, w3d + ((k * W3B) >> 4), id3, k > 0);
      mma_commit_elect(&bar[ch][2]);
      mbar_wait_sleep(&bar[ch][2], it & 1);
    }
    stc_chain_sync<NCH>(ch);
    tc_fence_after();
    float y[GP];
    {
      uint32_t r[16];
      tmem_ld16(my + D3C, r);
      tmem_wait_ld16(r);
#pragma unroll
      for (int o = 0; o < GP; ++o) y[o] = __uint_as_float(r[o]) + a.b3[o];
    }
    if (row < a.r1) {
#pragma unroll
      for (int o = 0; o < GP; ++o)
        if (GP == 1 || o < a.g) {
          const float yo = a.act3 == SMLRT_IDENTITY ? y[o] : stc_act(y[o], a.act3);
          po[a.ocol[o]] = yo;
          chk = fmaf(yo, 0.0f, chk);
        }
    }
    row += step;
    po += ostep;
  }
  if (__any_sync(0xffffffffu, chk != chk) && (tid & 31) == 0) atomicOr(a.status, SMLRT_STATUS_NONFINITE);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(slot, TC * NCH);
  }
}

uint32_t stc_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}
float stc_float(uint32_t u) {
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
float stc_tf32(float f) {  // round to nearest even at tf32 (10 mantissa bits)
  uint32_t u = stc_bits(f);
  u += 0xfffu + ((u >> 13) & 1u);
  return stc_float(u & ~0x1fffu);
}
uint16_t stc_bf16(float f) {
  uint32_t u = stc_bits(f);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
uint32_t sw32_byte(uint32_t row, uint32_t byte) {
  return row * 32u + ((((byte >> 4) & 1u) ^ ((row >> 2) & 1u)) << 4) + (byte & 15u);
}

template <int N1, int N2, int ACT, int GP>
int launch_act(const StcArgs& a, int64_t r0, int64_t r1, cudaStream_t s) {
  constexpr int NCH = stc_chains(N1, N2), CPS = stc_sm_chains(N1, N2) / NCH;  // CTAs per SM
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // one CTA (NCH chains) per SM at most; fewer when the call has fewer tiles
  const int64_t tiles = (r1 - r0 + 127) / 128;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((tiles + NCH - 1) / NCH, (int64_t)sms * CPS));
  small_tc_kernel<N1, N2, ACT, GP><<<grid, 128 * NCH, 0, s>>>(a);
  count_launch();
  SMLRT_CUDA(cudaGetLastError());
  return SMLRT_OK;
}

template <int N1, int N2, int ACT>
int launch_g(const StcArgs& a, int64_t r0, int64_t r1, cudaStream_t s) {
  // outputs rounded up to 1 / 2 / 4 / 8 (the padded ones have zero weights and are not stored)
  if (a.g == 1) return launch_act<N1, N2, ACT, 1>(a, r0, r1, s);
  if (a.g == 2) return launch_act<N1, N2, ACT, 2>(a, r0, r1, s);
  if (a.g <= 4) return launch_act<N1, N2, ACT, 4>(a, r0, r1, s);
  return launch_act<N1, N2, ACT, 8>(a, r0, r1, s);
}
template <int N1, int N2>
int launch_shape(const StcArgs& a, int act, int64_t r0, int64_t r1, cudaStream_t s) {
  if (act == SMLRT_RELU) return launch_g<N1, N2, SMLRT_RELU>(a, r0, r1, s);
  if (act == SMLRT_TANH) return launch_g<N1, N2, SMLRT_TANH>(a, r0, r1, s);
  if (act == SMLRT_IDENTITY) return launch_g<N1, N2, SMLRT_IDENTITY>(a, r0, r1, s);
  return SMLRT_E_UNSUPPORTED;
}

int pad16(int n) { return n <= 16 ? 16 : n <= 32 ? 32 : 64; }

bool stc_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("SMLRT_SMALL_TC");
    on = (e == nullptr || std::atoi(e) != 0) ? 1 : 0;
  }
  return on == 1;
}

}  // namespace

// at upload (bf16 models whose shape the warp-MMA kernel takes): the SW32
// operand images of W1 (tf32, bias as two extra K columns) and W2 (bf16), and
// the epilogue constants
int small_tc_pack(smlrt_model_s& m, int n1, int n2) {
  const DevLayer &L1 = m.layers[0], &L2 = m.layers[1], &L3 = m.layers[2];
  const int F = L1.in, H1 = L1.out, H2 = L2.out, G = L3.out;
  if (F > STC_F || G > STC_G || n1 > STC_H || n2 > STC_H) return SMLRT_OK;
  const float* p = m.host_params.data();  // [W1][b1][W2][b2][W3][b3]
  const float *W1 = p, *b1 = W1 + (size_t)H1 * F, *W2 = b1 + H1, *b2 = W2 + (size_t)H2 * H1, *W3 = b2 + H2,
              *b3 = W3 + (size_t)G * H2;
  const size_t w1b = (size_t)n1 * 32, w2b = (size_t)n2 * 32;
  // [W1][W2 K16-blocks][W3 K16-blocks: 16 rows (outputs, zero past G) x 32 B]
  std::vector<uint8_t> img(w1b + (size_t)(n1 / 16) * w2b + (size_t)(n2 / 16) * 512, 0);
  for (int n = 0; n < H1; ++n)
    for (int k = 0; k < 8; ++k) {  // features 0..F-1, zeros, the bias as tf32 hi + lo at 6, 7
      float w = 0.0f;
      if (k < F) w = stc_tf32(W1[(size_t)n * F + k]);
      else if (k == 6) w = stc_tf32(b1[n]);
      else if (k == 7) w = stc_tf32(b1[n] - stc_tf32(b1[n]));
      const uint32_t u = stc_bits(w);
      std::memcpy(img.data() + sw32_byte(n, k * 4), &u, 4);
    }
  for (int n = 0; n < H2; ++n)
    for (int k = 0; k < H1; ++k) {
      const uint16_t h = stc_bf16(W2[(size_t)n * H1 + k]);
      std::memcpy(img.data() + w1b + (k / 16) * w2b + sw32_byte(n, (k % 16) * 2), &h, 2);
    }
  for (int o = 0; o < G; ++o)
    for (int k = 0; k < H2; ++k) {
      const uint16_t h = stc_bf16(W3[(size_t)o * H2 + k]);
      std::memcpy(img.data() + w1b + (size_t)(n1 / 16) * w2b + (k / 16) * 512 + sw32_byte(o, (k % 16) * 2), &h, 2);
    }
  m.stc_epi.assign(STC_H + STC_G, 0.0f);  // [b2 | b3]
  for (int n = 0; n < H2; ++n) m.stc_epi[n] = b2[n];
  for (int o = 0; o < G; ++o) m.stc_epi[STC_H + o] = b3[o];
  SMLRT_CUDA(cudaMalloc(&m.stc_blob, img.size()));
  SMLRT_CUDA(cudaMemcpy(m.stc_blob, img.data(), img.size(), cudaMemcpyHostToDevice));
  return SMLRT_OK;
}

// bf16 region through the small-MLP tcgen05 kernel, or SMLRT_E_UNSUPPORTED
// (no blob, a sweep of more than one axis, or SMLRT_SMALL_TC=0): the caller
// has checked the model shape, uniform f32 plans and the column counts
int launch_region_small_tc(const smlrt_model_s& m, const DevPlan& in, const void* src, const DevPlan& out, void* dst,
                           int64_t r0, int64_t r1, float* staged, cudaStream_t s, uint32_t* status) {
  // packed rows only (row pitch == F, columns one contiguous run): other
  // plans keep the warp-MMA kernel's per-lane plan loads
  if (m.stc_blob == nullptr || !stc_enabled() || in.n_sweep != 1 || out.n_sweep != 1 || !in.dense_rows ||
      in.ustride[0] != in.n_cols)
    return SMLRT_E_UNSUPPORTED;
  const DevLayer &L1 = m.layers[0], &L2 = m.layers[1], &L3 = m.layers[2];
  const int n1 = pad16(L1.out), n2 = pad16(L2.out), G = L3.out;
  StcArgs a{};
  a.r0 = r0;
  a.r1 = r1;
  a.src = static_cast<const float*>(src) + in.col_inl[0];
  a.status = status;
  a.blob = static_cast<const uint8_t*>(m.stc_blob);
  a.F = L1.in;
  a.g = G;
  a.act3 = L3.act;
  if (staged != nullptr) {
    a.obase = staged - r0 * G;
    a.op = G;
    for (int o = 0; o < G; ++o) a.ocol[o] = o;
  } else {
    a.obase = static_cast<float*>(dst);
    a.op = out.ustride[0];
    for (int o = 0; o < G; ++o) a.ocol[o] = out.col_inl[o];
  }
  std::memcpy(a.b2, m.stc_epi.data(), sizeof(a.b2));
  std::memcpy(a.b3, m.stc_epi.data() + STC_H, sizeof(a.b3));
  const int act = L1.act;
#define STC_GO(A, B) \
  if (n1 == A && n2 == B) return launch_shape<A, B>(a, act, r0, r1, s)
  STC_GO(64, 32);
  STC_GO(64, 64);
  STC_GO(32, 32);
  STC_GO(32, 16);
  STC_GO(16, 16);
  STC_GO(64, 16);
  STC_GO(32, 64);
  STC_GO(16, 32);
  STC_GO(16, 64);
#undef STC_GO
  return SMLRT_E_UNSUPPORTED;
}

}  // namespace smlrt
