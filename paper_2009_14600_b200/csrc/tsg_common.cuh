// tsg_common.cuh -- device data layout of the B200 tSparse path.
//
// Tile size is 16x16 (the reference hard-wires 8x8,
// proj/include/tilemul/tile_format.hpp:12).  A tiled matrix lives in HBM as
// a CSR-of-tiles (struct of arrays), tiles sorted by (tile_row, tile_col)
// exactly like TiledMatrix.tiles (tile_format.hpp:43-55):
//
//   trp   u32[tile_rows+1]  first tile of each tile row
//   tcol  u32[T]            tile column
//   rmask u16[T*16]         row r bit c  <=> slot (r,c) nonzero  (the 256-bit
//                           occupancy mask; reference bit 8r+c, tile_format.hpp:20-23)
//   occ   u32[T]            lo16 = column occupancy (OR of rows), hi16 = row
//                           occupancy: the O(1) zero-product filter inputs
//                           (tile_product_nonzero, pipeline.cpp:23-35)
//   voff  u32[T]            first value of the tile
//   fhdr  u16[T*32]         per mma lane: (slot byte | prefix << 8), see below
//   vals  f16[nnz]          values, packed per tile in *fragment order*
//
// Fragment order (our layout, not the reference's ascending-bit order): the
// 256 slots of a tile are numbered by (mma lane L, slot j) where lane L of an
// m16n8k16 warp holds slot j of its operand registers.  A tile that will be
// the A operand is packed in "A order", a B operand in "B order" (A order of
// the transpose).  Lane L's nonzeros are then one contiguous run starting
// at prefix(L); fhdr[L] says which of its 8 slots are present.  Building an
// operand fragment is one coalesced 64-byte header load plus popc(byte)
// (usually 0-2) two-byte loads per lane -- no per-element index search.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

namespace tsg {

constexpr int kTile = 16;
constexpr unsigned kFull = 0xffffffffu;

enum Role : int { kRoleA = 0, kRoleB = 1 };

struct TileMat {
  int64_t rows = 0, cols = 0;
  uint32_t tile_rows = 0, tile_cols = 0;
  uint64_t cap_tiles = 0, cap_vals = 0;  // allocated capacity (upper bounds)
  uint32_t* trp = nullptr;
  uint32_t* tcol = nullptr;
  uint16_t* rmask = nullptr;
  uint32_t* occ = nullptr;
  uint32_t* voff = nullptr;
  uint16_t* fhdr[2] = {nullptr, nullptr};  // per role
  __half* vals[2] = {nullptr, nullptr};    // per role
};

// Slot (r, c) of a tile used as operand `role` -> (lane, j).
//   A operand (row-major 16x16, PTX m16n8k16 .f16 A fragment):
//     reg0={(g,2t),(g,2t+1)} reg1={(g+8,2t),(g+8,2t+1)}
//     reg2={(g,2t+8),(g,2t+9)} reg3={(g+8,2t+8),(g+8,2t+9)}
//   B operand (k x n = the A layout of B^T; regs 0,2 feed the n0..7 mma as
//   {b0,b1}, regs 1,3 the n8..15 mma):
//     reg0={(2t,g),(2t+1,g)} reg1={(2t,g+8),(2t+1,g+8)}
//     reg2={(2t+8,g),(2t+9,g)} reg3={(2t+8,g+8),(2t+9,g+8)}
//   with g = L>>2, t = L&3, slot j = 2*reg + half.
__host__ __device__ inline void slot_of(int role, int r, int c, int& lane, int& j) {
  if (role == kRoleB) { int tmp = r; r = c; c = tmp; }
  const int g = r & 7, t = (c & 7) >> 1;
  const int reg = (r >> 3) | ((c >> 3) << 1);
  lane = 4 * g + t;
  j = 2 * reg + (c & 1);
}

__host__ __device__ inline void rc_of(int role, int lane, int j, int& r, int& c) {
  const int g = lane >> 2, t = lane & 3;
  const int reg = j >> 1, h = j & 1;
  r = g + 8 * (reg & 1);
  c = 2 * t + h + 8 * (reg >> 1);
  if (role == kRoleB) { int tmp = r; r = c; c = tmp; }
}

// Accumulator (C/D fragment, two n8 halves: acc0 = cols 0..7, acc1 = 8..15):
//   acc[h][i]: row g + 8*(i>>1), col 2t + (i&1) + 8*h.
// That is exactly A-order slot j = 2*(i>>1 | h<<1) + (i&1), so a C tile
// written in A order can feed the next stage of a chain directly.

// Device error flags (OR-ed), mapped to tsg_status by the host.
enum ErrBits : unsigned {
  kErrInvariant = 1u,  // unsorted / duplicate / out-of-range CSR
  kErrOverflow = 2u,   // |x| > 65504 or non-finite input
  kErrPrecision = 4u,  // non-finite accumulator
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace tsg
