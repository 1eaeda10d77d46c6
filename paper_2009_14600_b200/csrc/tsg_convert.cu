// tsg_convert.cu -- subsystem (1): CSR -> 16x16 tiled bitmap format.
//
// GPU restatement of from_element_coo(m, Fp16Stored)
// (proj/src/tile_format.cpp:61-129) at T = 16:
//   * validation of the COO/CSR invariant        tile_format.cpp:34-51
//   * non-finite -> OverflowError (or dropped)   tile_format.cpp:82-86
//   * exact zero dropped                         tile_format.cpp:87
//   * round_to_half (RNE, |x| > 65504 throws)    tile_format.cpp:89-90, half.cpp:12-36
//   * values that round to zero dropped          tile_format.cpp:98
//   * tiles keyed (tile_row, tile_col), slots in-tile, tiles sorted
//     (the std::sort at tile_format.cpp:106-110 is replaced by a 16-way
//      merge across the rows of a tile row: CSR rows are already sorted).
//
// One warp per tile row (16 CSR rows, lane r<16 owns row r).  Each step the
// warp takes the minimum pending tile column (REDUX), every row lane
// consumes its entries in that tile, and the tile is emitted.  Two passes
// (count, fill) with a prefix sum between them; the fill pass stages each
// tile densely in shared memory and cuts the lane-dense operand chunks of
// one or both roles (A order and/or B order, see tsg_common.cuh), plus the
// tile's 256-bit occupancy mask and row/column occupancy words.
#include "tsg_kernels.cuh"

namespace tsg {

namespace {

// Single-step RNE double -> binary16 (no double rounding through float).
__device__ __forceinline__ unsigned short f64_to_half_bits(double x) {
  unsigned short h;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(x));
  return h;
}

// Loads value p as binary16 bits (kDtype: 0 f16 bits, 1 f32, 2 f64).  Sets
// kErrOverflow on |x| > 65504 or non-finite input (unless dropped); `keep`
// is false when the entry is dropped (zero, underflow, dropped non-finite).
template <int kDtype>
__device__ __forceinline__ unsigned short load_half(const void* val, int64_t p,
                                                    bool drop_nonfinite, unsigned& err,
                                                    bool& keep) {
  unsigned short h = 0;
  keep = false;
  if (kDtype == 1) {
    const float x = __ldg(static_cast<const float*>(val) + p);
    if (!isfinite(x)) {
      if (!drop_nonfinite) err |= kErrOverflow;
      return 0;
    }
    if (fabsf(x) > 65504.0f) {
      err |= kErrOverflow;
      return 0;
    }
    h = __half_as_ushort(__float2half_rn(x));
  } else if (kDtype == 2) {
    const double x = __ldg(static_cast<const double*>(val) + p);
    if (!isfinite(x)) {
      if (!drop_nonfinite) err |= kErrOverflow;
      return 0;
    }
    if (fabs(x) > 65504.0) {
      err |= kErrOverflow;
      return 0;
    }
    h = f64_to_half_bits(x);
  } else {
    h = __ldg(static_cast<const unsigned short*>(val) + p);
    if ((h & 0x7c00u) == 0x7c00u) {  // inf / nan
      if (!drop_nonfinite) err |= kErrOverflow;
      return 0;
    }
  }
  keep = (h & 0x7fffu) != 0;  // exact zero or underflow-to-(+-)0 dropped
  return h;
}

constexpr int kBitW = 256;  // count-pass bitmap words per warp (8192 tile columns)

template <bool kFill, int kDtype>
__global__ void __launch_bounds__(256) convert_kernel(CsrView in, TileMat out, int roles,
                                                     const uint32_t* __restrict__ tile_base,
                                                     const uint32_t* __restrict__ val_base,
                                                     uint32_t* __restrict__ row_ntiles,
                                                     uint32_t* __restrict__ row_nvals,
                                                     unsigned* __restrict__ err_flag,
                                                     int drop_nonfinite,
                                                     const uint8_t* __restrict__ needed) {
  // per warp: the tile staged densely (row-major) and transposed, as fp16 bits
  __shared__ __align__(16) uint16_t s_tile[8][2][256];
  __shared__ uint32_t s_bits[kFill ? 1 : 8][kBitW];  // count pass: tile-column bitmap
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint32_t I = blockIdx.x * 8 + wib;
  if (I >= out.tile_rows) return;
  uint16_t* st = s_tile[wib][0];
  uint16_t* stT = s_tile[wib][1];

  const int64_t row = int64_t(I) * kTile + lane;
  const bool has_row = lane < kTile && row < in.rows;
  int64_t p = has_row ? in.row_ptr[row] : 0;
  const int64_t end = has_row ? in.row_ptr[row + 1] : 0;
  unsigned err = 0;
  int32_t prev_col = -1;
  if (!kFill && has_row && end < p) err |= kErrInvariant;

  // A tile row no tile of the other operand refers to is only validated (the
  // reference validates the whole input, tile_format.cpp:34-51): no tiles.
  if (needed && !needed[I]) {
    if (kFill) {
      if (out.etile)
        for (; p < end; ++p) out.etile[p] = kNoTile;
      return;
    }
    for (; p < end; ++p) {
      const int32_t c = __ldg(in.col + p);
      if (c <= prev_col || c >= in.cols || c < 0) err |= kErrInvariant;
      prev_col = c;
      bool keep;
      load_half<kDtype>(in.val, p, drop_nonfinite, err, keep);
    }
    const unsigned e = __reduce_or_sync(kFull, err);
    if (lane == 0) {
      row_ntiles[I] = 0;
      row_nvals[I] = 0;
      if (e) atomicOr(err_flag, e);
    }
    return;
  }
  if (!kFill) {
    // Count pass over a panel whose tile columns span at most kBitW*32 tiles
    // (banded matrices: FEM27, Poisson): no merge -- lanes take the panel's
    // entries (contiguous in the CSR) 32 at a time, validate them
    // (tile_format.cpp:34-51, 82-96) and mark each kept entry's tile column
    // in a bitmap; tiles = popcount.  Wider panels take the merge below.
    const int64_t r0 = int64_t(I) * kTile, r1 = r0 + kTile < in.rows ? r0 + kTile : in.rows;
    const int64_t E0 = in.row_ptr[r0], E1 = in.row_ptr[r1];
    const bool rows_ok = __all_sync(kFull, !has_row || end >= p);
    uint32_t jlo = 0xffffffffu, jhi = 0;
    if (has_row && end > p) {
      jlo = uint32_t(__ldg(in.col + p)) >> 4;
      jhi = uint32_t(__ldg(in.col + end - 1)) >> 4;
    }
    jlo = __reduce_min_sync(kFull, jlo);
    jhi = __reduce_max_sync(kFull, jhi);
    if (rows_ok && E1 >= E0 && (jlo == 0xffffffffu || jhi - jlo < uint32_t(kBitW) * 32u)) {
      uint32_t* bm = s_bits[wib];
      for (int i = lane; i < kBitW; i += 32) bm[i] = 0;
      __syncwarp();
      // lane r < 16: first entry of row r (rows past the panel: E1)
      const int64_t rstart = lane < kTile && row < in.rows ? p : E1;
      uint32_t nv = 0;
      for (int64_t q0 = E0; q0 < E1; q0 += 32) {
        const int64_t q = q0 + lane;
        int r = 0;  // last row whose start is <= q
#pragma unroll
        for (int b = 8; b > 0; b >>= 1) {
          const int64_t v = __shfl_sync(kFull, rstart, r + b);
          if (v <= q) r += b;
        }
        const int64_t first = __shfl_sync(kFull, rstart, r);
        if (q < E1) {
          const int32_t c = __ldg(in.col + q);
          if (c >= in.cols || c < 0 || (q > first && c <= __ldg(in.col + q - 1))) err |= kErrInvariant;
          bool keep;
          load_half<kDtype>(in.val, q, drop_nonfinite, err, keep);
          const uint32_t j = (uint32_t(c) >> 4) - jlo;
          if (keep && c >= 0 && j < uint32_t(kBitW) * 32u) {
            atomicOr(bm + (j >> 5), 1u << (j & 31));
            ++nv;
          }
        }
      }
      __syncwarp();
      uint32_t nt = 0;
      for (int i = lane; i < kBitW; i += 32) nt += __popc(bm[i]);
      nt = __reduce_add_sync(kFull, nt);
      nv = __reduce_add_sync(kFull, nv);
      const unsigned e = __reduce_or_sync(kFull, err);
      if (lane == 0) {
        row_ntiles[I] = nt;
        row_nvals[I] = nv;
        if (e) atomicOr(err_flag, e);
      }
      return;
    }
  }
  uint32_t ntiles = 0, nvals = 0;
  uint32_t tbase = 0;
  uint32_t cbase[2] = {0, 0};
  if (kFill) {
    tbase = tile_base[I];
    // chunk capacity of a tile row = its kept nnz (every present lane holds >= 1)
    cbase[0] = cbase[1] = 1u + val_base[I];
  }
  // column of the lane's next entry, loaded one entry ahead so the row walk
  // below is not a chain of dependent global loads
  int32_t c_cur = p < end ? __ldg(in.col + p) : 0;
  while (true) {
    const uint32_t my_tc = (p < end) ? uint32_t(c_cur) >> 4 : 0xffffffffu;
    const uint32_t J = __reduce_min_sync(kFull, my_tc);
    if (J == 0xffffffffu) break;
    if (kFill) {
      reinterpret_cast<uint4*>(st)[lane] = make_uint4(0, 0, 0, 0);
      reinterpret_cast<uint4*>(stT)[lane] = make_uint4(0, 0, 0, 0);
      __syncwarp();
    }
    uint32_t rm = 0;
    bool first = true;  // first kept entry of this tile in this row
    while (p < end) {
      const int32_t c = c_cur;
      if ((uint32_t(c) >> 4) != J) break;
      const int32_t c_next = p + 1 < end ? __ldg(in.col + p + 1) : 0;
      if (!kFill) {
        if (c <= prev_col || c >= in.cols || c < 0) err |= kErrInvariant;
        prev_col = c;
      }
      bool keep;
      const unsigned short h = load_half<kDtype>(in.val, p, drop_nonfinite, err, keep);
      if (keep) {
        rm |= 1u << (c & 15);
        if (kFill) {
          st[lane * 16 + (c & 15)] = h;
          stT[(c & 15) * 16 + lane] = h;
        }
      }
      if (kFill && out.etile) {
        out.etile[p] = keep ? ((tbase + ntiles) | (first ? 0u : kDupEntry)) : kNoTile;
        first &= !keep;
      }
      ++p;
      c_cur = c_next;
    }
    // Termination holds for any input: the lane holding the minimum tile
    // column always consumes at least one entry.  Invalid input only sets
    // the flag; the host discards the results.
    const unsigned any = __ballot_sync(kFull, rm != 0);
    if (any == 0) continue;  // every value of this tile dropped
    const uint32_t tile_nnz = __reduce_add_sync(kFull, __popc(rm));
    if (kFill) {
      __syncwarp();
      const uint32_t t = tbase + ntiles;
      const uint32_t colocc = __reduce_or_sync(kFull, rm) & 0xffffu;
      if (lane == 0) {
        out.tco[t] = make_uint2(J, colocc | ((any & 0xffffu) << 16));
        out.trow[t] = I;
      }
      // the 256-bit mask as interleaved row masks: word g = row g | row g+8 << 16
      const uint32_t rm_hi = __shfl_sync(kFull, rm, (lane & 7) + 8);
      if (lane < 8) out.rm2[size_t(t) * 8 + lane] = rm | (rm_hi << 16);
      // cut the lane chunks: A order reads row pairs (r, 2t..2t+1) of the
      // staged tile, B order the same pairs of the transposed tile
#pragma unroll
      for (int role = 0; role < 2; ++role) {
        if (!(roles & (1 << role))) continue;
        const uint16_t* src = role == kRoleA ? st : stT;
        const int g = lane >> 2, tq = lane & 3;
        uint32_t reg[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)  // reg i = rows g + 8(i&1), cols 2t + 8(i>>1) .. +1
          reg[i] = *reinterpret_cast<const uint32_t*>(src + (g + 8 * (i & 1)) * 16 + 2 * tq + 8 * (i >> 1));
        const bool present = (reg[0] | reg[1] | reg[2] | reg[3]) != 0u;
        const unsigned lm = __ballot_sync(kFull, present);
        // B chunks are stored {reg0, reg2, reg1, reg3}: the {b0, b1} operand
        // pair of each n8 MMA is then one aligned register pair
        if (present)
          out.chunk[role][cbase[role] + __popc(lm & lanemask_lt())] =
              role == kRoleA ? make_uint4(reg[0], reg[1], reg[2], reg[3])
                             : make_uint4(reg[0], reg[2], reg[1], reg[3]);
        if (lane == 0) {
          out.meta[role][t] = make_uint2(lm, cbase[role]);
          if (out.rec[role]) out.rec[role][t] = make_uint4(lm, cbase[role], colocc | ((any & 0xffffu) << 16), J);
        }
        cbase[role] += __popc(lm);
      }
      __syncwarp();
    }
    ++ntiles;
    nvals += tile_nnz;
  }
  if (!kFill) {
    const unsigned e = __reduce_or_sync(kFull, err);
    if (lane == 0) {
      row_ntiles[I] = ntiles;
      row_nvals[I] = nvals;
      if (e) atomicOr(err_flag, e);
    }
  }
}

// B tile rows that some A tile refers to (A's tile columns).
__global__ void mark_needed_kernel(const TileMat A, uint8_t* __restrict__ needed) {
  const uint32_t nt = A.trp[A.tile_rows];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x)
    needed[__ldg(&A.tco[t].x)] = 1;
}

__global__ void row_stats_kernel(const uint32_t* __restrict__ trp, uint32_t tile_rows,
                                 unsigned* __restrict__ max_row_tiles) {
  unsigned m = 0;
  for (uint32_t I = blockIdx.x * blockDim.x + threadIdx.x; I < tile_rows;
       I += gridDim.x * blockDim.x)
    m = max(m, trp[I + 1] - trp[I]);
  m = __reduce_max_sync(kFull, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(max_row_tiles, m);
}

// Column counts of A (histogram) for C-bar.
__global__ void col_hist_kernel(const int32_t* __restrict__ col, int64_t nnz, int64_t ncols,
                                unsigned* __restrict__ hist) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nnz;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t c = __ldg(col + i);
    if (c >= 0 && c < ncols) atomicAdd(hist + c, 1u);
  }
}

__global__ void cbar_dot_kernel(const unsigned* __restrict__ hist, const int64_t* __restrict__ rpB,
                                int64_t n, unsigned long long* __restrict__ out) {
  unsigned long long acc = 0;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x)
    acc += (unsigned long long)hist[k] * (unsigned long long)(rpB[k + 1] - rpB[k]);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(kFull, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

}  // namespace

void launch_convert_count(const CsrView& in, TileMat& out, uint32_t* row_ntiles,
                          uint32_t* row_nvals, unsigned* err_flag, int drop_nonfinite,
                          const uint8_t* needed, cudaStream_t st) {
  const unsigned blocks = (out.tile_rows + 7) / 8;
  if (blocks == 0) return;
  auto k = in.dtype == 0 ? convert_kernel<false, 0> : in.dtype == 2 ? convert_kernel<false, 2>
                                                                    : convert_kernel<false, 1>;
  k<<<blocks, 256, 0, st>>>(in, out, 0, nullptr, nullptr, row_ntiles, row_nvals, err_flag,
                            drop_nonfinite, needed);
}

void launch_convert_fill(const CsrView& in, TileMat& out, int roles, const uint32_t* tile_base,
                         const uint32_t* val_base, int drop_nonfinite, const uint8_t* needed,
                         cudaStream_t st) {
  const unsigned blocks = (out.tile_rows + 7) / 8;
  if (blocks == 0) return;
  auto k = in.dtype == 0 ? convert_kernel<true, 0> : in.dtype == 2 ? convert_kernel<true, 2>
                                                                   : convert_kernel<true, 1>;
  k<<<blocks, 256, 0, st>>>(in, out, roles, tile_base, val_base, nullptr, nullptr, nullptr,
                            drop_nonfinite, needed);
}

void launch_mark_needed(const TileMat& A, uint8_t* needed, cudaStream_t st) {
  if (A.cap == 0) return;
  unsigned blocks = unsigned((A.cap + 255) / 256);
  if (blocks > 2368) blocks = 2368;
  mark_needed_kernel<<<blocks, 256, 0, st>>>(A, needed);
}

void launch_row_stats(const TileMat& A, unsigned* max_row_tiles, cudaStream_t st) {
  if (A.tile_rows == 0) return;
  unsigned blocks = (A.tile_rows + 255) / 256;
  if (blocks > 592) blocks = 592;
  row_stats_kernel<<<blocks, 256, 0, st>>>(A.trp, A.tile_rows, max_row_tiles);
}

void launch_cbar(const int32_t* colA, int64_t nnzA, int64_t inner, const int64_t* rpB,
                 unsigned* hist, unsigned long long* out, cudaStream_t st) {
  if (nnzA > 0) col_hist_kernel<<<1184, 256, 0, st>>>(colA, nnzA, inner, hist);
  if (inner > 0) cbar_dot_kernel<<<592, 256, 0, st>>>(hist, rpB, inner, out);
}

}  // namespace tsg
