// Shared pieces of the halo-stencil region kernels (stencil_tc.cu: bf16
// warp-MMA; stencil_exact.cu: fp32-exact): the TMA row ring's PTX wrappers.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace smlrt {
namespace stencil {

using namespace ptx;

// one box of the 3-D tensor map (columns, rows of a plane, planes)
__device__ __forceinline__ void sm_tma(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void sm_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// mbarrier wait that traps after ~2^26 polls (seconds): a TMA that never
// lands fails the launch instead of hanging the device
__device__ __forceinline__ void sm_wait(uint64_t* bar, uint32_t parity) {
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


// Host: the geometry of a 4-variable 3x3 halo in-plan over a 2-D sweep with
// unit inner stride -- run (v, d) starts at col_inl[(v*3 + d)*3] = first_v +
// d*s0, the variables' planes equally spaced by a multiple of s0 -- such that
// every element read lies inside the s0-pitched rows (no wrap).  The TMA box
// starts at the 16-B aligned column c0 at or left of the halo column; al =
// the halo column's offset in the box (even, <= max_al).
struct StencilGeom {
  int32_t c0, r0v, p0v, al;  // box origin column, first input row (plane-local), plane of variable 0
  int64_t plane;             // elements between the variables' planes
};

inline bool stencil_geom(const DevPlan& in, int max_al, StencilGeom* g) {
  if (!in.uniform || in.n_sweep != 2 || in.ustride[1] != 1 || in.n_cols != 36) return false;
  const int64_t s0 = in.ustride[0], nj = in.sdiv[1].d, numel = in.uarray_numel;
  if (s0 <= 0 || s0 % 4 != 0 || numel % s0 != 0) return false;
  for (int v = 0; v < 4; ++v)
    for (int d = 0; d < 3; ++d)
      for (int k = 0; k < 3; ++k)
        if (in.col_inl[(v * 3 + d) * 3 + k] != in.col_inl[v * 9] + d * s0 + k) return false;
  const int64_t f0 = in.col_inl[0], P = in.col_inl[9] - f0;
  if (f0 < 0 || P <= 0 || P % s0 != 0 || numel % P != 0) return false;
  for (int v = 1; v < 4; ++v)
    if (in.col_inl[v * 9] - f0 != v * P) return false;
  const int64_t col = f0 % s0, row = (f0 % P) / s0, pl = f0 / P;  // halo column / first row / plane of var 0
  if (col + nj + 1 >= s0 || pl + 4 > numel / P || P / s0 >= (1ll << 31) || numel / P >= (1ll << 31)) return false;
  const int64_t c0 = col & ~int64_t(3);
  g->al = (int32_t)(col - c0);
  if (g->al > max_al || g->al % 2 != 0) return false;  // the tile's columns in the box, 8-B shared loads
  g->c0 = (int32_t)c0;
  g->r0v = (int32_t)row;
  g->p0v = (int32_t)pl;
  g->plane = P;
  return true;
}

}  // namespace stencil
}  // namespace smlrt
