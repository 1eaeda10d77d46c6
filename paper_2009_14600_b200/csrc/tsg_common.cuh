// tsg_common.cuh -- device data layout of the B200 tSparse path.
//
// Tile size is 16x16 (the reference hard-wires 8x8,
// proj/include/tilemul/tile_format.hpp:12).  A tiled matrix lives in HBM as
// a CSR-of-tiles (struct of arrays), tiles sorted by (tile_row, tile_col)
// exactly like TiledMatrix.tiles (tile_format.hpp:43-55):
//
//   trp   u32[tile_rows+1]  first tile of each tile row
//   tco   uint2[T]          {tile column, occupancy}; occupancy lo16 = column
//                           occupancy (OR of rows), hi16 = row occupancy: the
//                           O(1) zero-product filter (pipeline.cpp:23-35)
//   rm2   u32[T*8]          the 256-bit occupancy mask as interleaved row
//                           masks: word g = row g | row g+8 << 16 (bit c of
//                           row r <=> slot (r,c) nonzero; reference bit 8r+c,
//                           tile_format.hpp:20-23)
//   meta  uint2[T]  (per operand role)  {lane mask, first chunk}
//   chunk uint4[]   (per operand role)  16-byte lane chunks, chunk 0 = zeros
//   rec   uint4[T]  (per operand role)  {lane mask, first chunk, occupancy, tile col}
//                   -- meta and tco in one 16-byte record for random gathers
//
// Lane-dense operand chunks (our layout, not the reference's ascending-bit
// order): mma.m16n8k16 lane L holds 8 fp16 slots of a 16x16 operand in four
// .f16x2 registers.  A tile stores, for every lane with at least one nonzero
// slot, those 16 bytes verbatim ("chunk"); lane mask bit L says the chunk
// exists, and it lives at meta.y + popc(lane mask below L).  Loading an
// operand fragment is therefore one LDG.128 per lane (absent lanes read the
// zero chunk 0) -- no per-element index arithmetic on the hot path.  A tile
// that will be the A operand is stored in "A order", a B operand in "B order"
// (the A order of its transpose, chunk registers stored {reg0, reg2, reg1,
// reg3} so each n8 MMA's {b0, b1} is one register pair); A.A stores both.
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
  uint64_t cap = 0;  // allocated tiles/chunks capacity (upper bound: nnz)
  uint32_t* trp = nullptr;
  uint2* tco = nullptr;
  uint32_t* rm2 = nullptr;
  // (B-role conversions) per input CSR entry: its tile's rank within its
  // tile row (add trp[tile row]), | kDupEntry unless it
  // is the first kept entry of that tile in its row, kNoTile if dropped; and
  // the input row pointers -- single-column A tiles enumerate through them
  uint32_t* etile = nullptr;
  const int64_t* csr_rp = nullptr;
  // per input CSR entry: its rounded binary16 value (0 when dropped) -- the
  // general path multiplies straight from the CSR
  uint16_t* h16 = nullptr;
  // (a B summary, tsg_bsum) per tile: its row occupancy, in place of tco
  const uint16_t* ro16 = nullptr;
  uint2* meta[2] = {nullptr, nullptr};
  uint4* rec[2] = {nullptr, nullptr};  // {lane mask, first chunk, occupancy, tile column}: one gather per tile
  uint4* chunk[2] = {nullptr, nullptr};
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

// Accumulator (C/D fragment, two n8 halves: acc[0] = cols 0..7, acc[1] = 8..15):
//   acc[h][i]: row g + 8*(i>>1), col 2t + (i&1) + 8*h.

constexpr uint32_t kNoTile = 0xffffffffu;
constexpr uint32_t kDupEntry = 0x80000000u;

// Device error flags (OR-ed), mapped to tsg_status by the host.
enum ErrBits : unsigned {
  kErrInvariant = 1u,  // unsorted / duplicate / out-of-range CSR
  kErrOverflow = 2u,   // |x| > 65504 or non-finite input
  kErrPrecision = 4u,  // non-finite accumulator
  kCancelled = 8u,     // an output slot cancelled to exactly 0 (compaction needed)
  kErrPool = 16u,      // general path: the overflow-piece pool was too small (the host reruns)
  kErrRowPtr = 32u,    // row_ptr[0] != 0, row_ptr[rows] != nnz or decreasing: no kernel reads the
                       // entries (an InvariantError, like validate_coo, tile_format.cpp:34-51)
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned spread4(unsigned n) {  // bit t -> bit 2t
  return (n & 1u) | ((n & 2u) << 1) | ((n & 4u) << 2) | ((n & 8u) << 3);
}

// 16 row masks of an m16n16 accumulator held as acc[h][i] (see above):
// from the 8 ballots B[h][i] (bit L = lane L's acc[h][i] nonzero), row r's
// mask.  Returned in lane r (r < 16); other lanes get row r & 15.
__device__ __forceinline__ unsigned row_mask_from_ballots(const unsigned (&B)[2][4], int lane) {
  const int r = lane & 15, sh = 4 * (r & 7);
  const bool lo = r < 8;  // selects, not a runtime index: keeps B in registers
  const unsigned n0 = ((lo ? B[0][0] : B[0][2]) >> sh) & 0xfu;
  const unsigned n1 = ((lo ? B[0][1] : B[0][3]) >> sh) & 0xfu;
  const unsigned n2 = ((lo ? B[1][0] : B[1][2]) >> sh) & 0xfu;
  const unsigned n3 = ((lo ? B[1][1] : B[1][3]) >> sh) & 0xfu;
  return spread4(n0) | (spread4(n1) << 1) | (spread4(n2) << 8) | (spread4(n3) << 9);
}

}  // namespace tsg
