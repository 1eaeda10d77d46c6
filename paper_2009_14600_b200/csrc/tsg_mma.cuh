// tsg_mma.cuh -- warp-level tile-product helpers shared by the numeric
// kernels (tsg_numeric.cu, tsg_panel.cu): mma.sync wrappers, the 0/1
// indicator operands of the fused counting pass, lane-dense chunk loads and
// the accumulator layout.
#pragma once
#include "tsg_common.cuh"

namespace tsg {
namespace {

__device__ __forceinline__ void mma16816(float (&d)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// fp16 accumulate (two .f16x2 registers per m16n8 tile)
__device__ __forceinline__ void mma16816_h(uint32_t (&d)[2], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 "
      "{%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};\n"
      : "+r"(d[0]), "+r"(d[1])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// 1.0 where the binary16 slot is nonzero, 0.0 where it is zero (per half)
__device__ __forceinline__ uint32_t nz_h2(uint32_t x) {
  uint32_t r;
  asm("set.ne.f16x2.f16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(0u));
  return r;
}
__device__ __forceinline__ uint4 nz_h2(const uint4& v) {
  return make_uint4(nz_h2(v.x), nz_h2(v.y), nz_h2(v.z), nz_h2(v.w));
}

// nonzero halves of a .f16x2 register (0, 1 or 2)
__device__ __forceinline__ uint32_t count_nz_h2(uint32_t x) {
  return ((x & 0x7fffu) != 0u) + ((x & 0x7fff0000u) != 0u);
}

// nonzero halves of four .f16x2 registers holding non-negative counts (the
// 0/1-indicator accumulators: bit 15 of each half is clear): adding 0x7fff
// to a half sets its bit 15 exactly when it is nonzero, without a carry
// into the next half
__device__ __forceinline__ uint32_t count_nz_counts(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  constexpr uint32_t M = 0x7fff7fffu, H = 0x80008000u;
  return __popc((a + M) & H) + __popc((b + M) & H) + __popc((c + M) & H) + __popc((d + M) & H);
}

// chunk index of this lane for a tile with meta {lane mask, base}; 0 = zeros
__device__ __forceinline__ uint32_t chunk_index(uint32_t lm, uint32_t base, int lane) {
  return ((lm >> lane) & 1u) ? base + __popc(lm & lanemask_lt()) : 0u;
}

// Unconditional load: absent lanes read the shared zero chunk 0 (one
// broadcast sector), so no zero-fill and no branch on the hot path.
__device__ __forceinline__ uint4 load_chunk(const uint4* __restrict__ base, uint32_t lm,
                                            uint32_t first, unsigned lt, unsigned bit) {
  const uint32_t idx = (lm & bit) ? first + __popc(lm & lt) : 0u;
  return __ldg(base + idx);
}

// Per-lane constants of the accumulator layout: acc[h][i] holds
// (row g + 8*(i>>1), col 2t + (i&1) + 8h); cm[h] masks the columns of a
// row left of col 2t + 8h.
struct LaneLayout {
  int g, t;
  uint32_t cm[2];
  __device__ __forceinline__ explicit LaneLayout(int lane) {
    g = lane >> 2;
    t = lane & 3;
    cm[0] = (1u << (2 * t)) - 1u;
    cm[1] = (1u << (2 * t + 8)) - 1u;
  }
};

// Realised row masks of an m16n16 accumulator tile, computed inside the
// lane group that holds the rows: returns (row g mask) | (row g+8 mask) << 16
// (bit c = column c nonzero), identical in the four lanes 4g .. 4g+3.
__device__ __forceinline__ uint32_t group_row_masks(const float (&acc)[2][4], int t) {
  uint32_t x = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (acc[h][i] != 0.0f) x |= 1u << ((i & 1) + 8 * h + 16 * (i >> 1));
  x <<= 2 * t;
  x |= __shfl_xor_sync(kFull, x, 1);
  x |= __shfl_xor_sync(kFull, x, 2);
  return x;
}

}  // namespace
}  // namespace tsg
