// tsg_tiles8.cu -- the reference's 8x8 TiledMatrix layout on the GPU (SURVEY
// 8(f) row 2, "GPU 8x8 <-> 16x16 re-tiling"): the C++ drop-in's
// spgemm_square takes and returns 8x8 tiles, and these kernels move them to
// and from the CSR the 16x16 pipeline consumes and produces.
//
//   tiles8_to_csr   8x8 tiles -> CSR: warp per 8-row tile row, lane r < 8
//                   walks row r through the tile row's tiles (ascending
//                   columns), so every CSR row comes out sorted -- the
//                   to_element_coo order (tile_format.cpp:131-154) without
//                   its global sort
//   csr_to_tiles8   CSR -> 8x8 tiles, from_element_coo(Fp32Stored) of the
//                   CSR (tile_format.cpp:61-129): warp per 8-row group, lanes
//                   r < 8 merge their rows by tile column (REDUX min); each
//                   step is one tile: its 64-bit bitmap (bit 8r + c) is the OR
//                   of the lanes' row bytes and its elements are row-major,
//                   i.e. in bit order.  A count pass sizes the output, a scan
//                   gives each group its tile and element offsets, the write
//                   pass fills them.  Zeros are dropped (as from_element_coo).
#include <cstdint>

#include "tsg_kernels.cuh"

namespace tsg {

namespace {

constexpr uint32_t kNone = 0xffffffffu;

// ---- 8x8 tiles -> CSR -----------------------------------------------------------
__global__ void tiles8_rowcount_kernel(Tiles8View t, const uint32_t* __restrict__ trp, int64_t rows,
                                       int64_t* __restrict__ rowcnt, unsigned* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t T = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t r = T * 8 + lane;
  if (T * 8 >= rows || lane >= 8 || r >= rows) return;
  uint32_t n = 0;
  for (uint32_t i = trp[T]; i < trp[T + 1]; ++i) n += __popcll((t.bitmap[i] >> (8 * lane)) & 0xffull);
  rowcnt[r] = n;
  (void)err;
}

__global__ void tiles8_to_csr_kernel(Tiles8View t, const uint32_t* __restrict__ trp, int64_t rows,
                                     const int64_t* __restrict__ rp, int32_t* __restrict__ col,
                                     float* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const int64_t T = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t r = T * 8 + lane;
  if (T * 8 >= rows || lane >= 8 || r >= rows) return;
  int64_t p = rp[r];
  for (uint32_t i = trp[T]; i < trp[T + 1]; ++i) {
    const unsigned long long bm = t.bitmap[i];
    uint32_t row_bits = uint32_t(bm >> (8 * lane)) & 0xffu;
    if (!row_bits) continue;
    // the row's elements follow the earlier rows' in the tile's run (bit order)
    uint64_t e = t.elem_index[i] + uint64_t(__popcll(bm & ((1ull << (8 * lane)) - 1ull)));
    for (; row_bits; row_bits &= row_bits - 1u, ++e, ++p) {
      col[p] = int32_t(t.tile_col[i] * 8u + uint32_t(__ffs(row_bits) - 1));
      val[p] = t.val[e];
    }
  }
}

// tile-row pointers of the (row, col)-sorted tiles: trp[T] = first tile of tile row T
__global__ void tiles8_trp_kernel(const uint32_t* __restrict__ tile_row, int64_t ntiles, int64_t tile_rows,
                                  uint32_t* __restrict__ trp, unsigned* __restrict__ err) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= ntiles; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t cur = i < ntiles ? int64_t(tile_row[i]) : tile_rows;
    const int64_t prev = i > 0 ? int64_t(tile_row[i - 1]) : -1;
    if (cur < prev || cur > tile_rows) {
      atomicOr(err, unsigned(kErrInvariant));
      continue;
    }
    for (int64_t T = prev + 1; T <= cur; ++T) trp[T] = uint32_t(i);
  }
}

// ---- CSR -> 8x8 tiles -----------------------------------------------------------
// One 8-row group, one warp.  kWrite: fill the tiles at (tile0, elem0); else
// count them.  Lanes r < 8 hold row r's cursor; a step takes the smallest
// pending tile column J and every lane consumes its entries in J.
template <bool kWrite>
__device__ __forceinline__ void group_walk(const CsrView& C, const float* val, int64_t g, int lane, uint32_t& ntiles,
                                           uint32_t& nelem, Tiles8Out o, uint64_t tile0, uint64_t elem0,
                                           unsigned& err) {
  const int64_t r = g * 8 + lane;
  const bool has = lane < 8 && r < C.rows;
  int64_t p = has ? C.row_ptr[r] : 0;
  const int64_t end = has ? C.row_ptr[r + 1] : 0;
  int32_t prev = -1;
  ntiles = 0;
  nelem = 0;
  while (true) {
    // skip zeros: from_element_coo drops them
    while (p < end && val[p] == 0.0f) ++p;
    const uint32_t mine = p < end ? uint32_t(C.col[p]) >> 3 : kNone;
    const uint32_t J = __reduce_min_sync(kFull, mine);
    if (J == kNone) break;
    uint32_t bits = 0, cnt = 0;
    const int64_t first = p;
    while (p < end && (uint32_t(C.col[p]) >> 3) == J) {
      const int32_t c = C.col[p];
      const float v = val[p];
      if (c <= prev || c >= C.cols) err |= kErrInvariant;
      if (!isfinite(v)) err |= kErrOverflow;
      prev = c;
      if (v != 0.0f) {
        bits |= 1u << (c & 7);
        ++cnt;
      }
      ++p;
    }
    // elements before this lane's in the tile: the earlier rows' counts
    uint32_t inc = cnt;
#pragma unroll
    for (int o2 = 1; o2 < 8; o2 <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, inc, o2);
      if (lane >= o2) inc += y;
    }
    const uint32_t tile_n = __shfl_sync(kFull, inc, 7);
    if (kWrite) {
      const uint32_t lo = __reduce_or_sync(kFull, lane < 4 ? bits << (8 * lane) : 0u);
      const uint32_t hi = __reduce_or_sync(kFull, lane >= 4 && lane < 8 ? bits << (8 * (lane - 4)) : 0u);
      if (lane == 0) {
        const uint64_t t = tile0 + ntiles;
        o.tile_row[t] = uint32_t(g);
        o.tile_col[t] = J;
        o.bitmap[t] = (unsigned long long)lo | ((unsigned long long)hi << 32);
        o.elem_index[t] = elem0 + nelem;
      }
      uint64_t e = elem0 + nelem + (inc - cnt);
      for (int64_t q = first; q < p; ++q)
        if (val[q] != 0.0f) o.val[e++] = val[q];
    }
    ++ntiles;
    nelem += tile_n;
  }
}

__global__ void csr_tiles8_count_kernel(CsrView C, const float* __restrict__ val, int64_t groups,
                                        uint32_t* __restrict__ gt, uint32_t* __restrict__ ge,
                                        unsigned* __restrict__ err_flag) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  if (g >= groups) return;
  uint32_t nt, ne;
  unsigned err = 0;
  group_walk<false>(C, val, g, lane, nt, ne, Tiles8Out{}, 0, 0, err);
  err = __reduce_or_sync(kFull, err);
  if (lane == 0) {
    gt[g] = nt;
    ge[g] = ne;
    if (err) atomicOr(err_flag, err);
  }
}

__global__ void csr_tiles8_write_kernel(CsrView C, const float* __restrict__ val, int64_t groups,
                                        const unsigned long long* __restrict__ toff,
                                        const unsigned long long* __restrict__ eoff, Tiles8Out o) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  if (g >= groups) return;
  uint32_t nt, ne;
  unsigned err = 0;
  group_walk<true>(C, val, g, lane, nt, ne, o, toff[g], eoff[g], err);
}

}  // namespace

void launch_tiles8_to_csr(const Tiles8View& t, const uint32_t* trp, int64_t rows, int64_t* rowcnt, const int64_t* rp,
                          int32_t* col, float* val, unsigned* err, bool count, cudaStream_t st) {
  const int64_t tile_rows = (rows + 7) / 8;
  if (tile_rows == 0) return;
  const unsigned blocks = unsigned((tile_rows * 32 + 255) / 256);
  if (count)
    tiles8_rowcount_kernel<<<blocks, 256, 0, st>>>(t, trp, rows, rowcnt, err);
  else
    tiles8_to_csr_kernel<<<blocks, 256, 0, st>>>(t, trp, rows, rp, col, val);
}

void launch_tiles8_trp(const uint32_t* tile_row, int64_t ntiles, int64_t tile_rows, uint32_t* trp, unsigned* err,
                       cudaStream_t st) {
  const unsigned blocks = unsigned(std::min<int64_t>((ntiles + 256) / 256, 2368));
  tiles8_trp_kernel<<<blocks, 256, 0, st>>>(tile_row, ntiles, tile_rows, trp, err);
}

void launch_csr_tiles8_count(const CsrView& C, const float* val, uint32_t* gt, uint32_t* ge, unsigned* err,
                             cudaStream_t st) {
  const int64_t groups = (C.rows + 7) / 8;
  if (groups == 0) return;
  csr_tiles8_count_kernel<<<unsigned((groups * 32 + 255) / 256), 256, 0, st>>>(C, val, groups, gt, ge, err);
}

void launch_csr_tiles8_write(const CsrView& C, const float* val, const unsigned long long* toff,
                             const unsigned long long* eoff, const Tiles8Out& o, cudaStream_t st) {
  const int64_t groups = (C.rows + 7) / 8;
  if (groups == 0) return;
  csr_tiles8_write_kernel<<<unsigned((groups * 32 + 255) / 256), 256, 0, st>>>(C, val, groups, toff, eoff, o);
}

}  // namespace tsg
