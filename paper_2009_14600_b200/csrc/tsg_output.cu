// tsg_output.cu -- subsystem (4): tiled -> CSR, with compaction fused in.
//
// GPU restatement of compact (proj/src/kernels.cpp:205-220: drop empty
// tiles, keep popcount(bitmap) values per tile) followed by to_element_coo
// (proj/src/tile_format.cpp:131-154: countr_zero walk + global (row, col)
// sort).  The sort disappears: tiles of a tile row are already in column
// order, so row r of the output is the concatenation over the row's tiles
// of each tile's row-r run.  One warp per output tile row: lanes 0-15 own
// rows, lanes 16-31 take every other tile and hand their offsets over.
#include "tsg_kernels.cuh"

namespace tsg {

namespace {

__global__ void __launch_bounds__(256) out_rowcount_kernel(uint32_t tile_rows, int64_t rows,
                                                          const uint32_t* __restrict__ seg_row_ptr,
                                                          const uint16_t* __restrict__ cmask,
                                                          int64_t* __restrict__ rowcnt) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows) return;
  const uint32_t s0 = seg_row_ptr[I], s1 = seg_row_ptr[I + 1];
  const int r = lane & 15;
  uint32_t n = 0;
  for (uint32_t s = s0 + (lane >> 4); s < s1; s += 2) n += __popc(__ldg(cmask + size_t(s) * 16 + r));
  n += __shfl_xor_sync(kFull, n, 16);
  const int64_t row = int64_t(I) * 16 + r;
  if (lane < 16 && row < rows) rowcnt[row] = n;
}

__global__ void __launch_bounds__(256) out_fill_kernel(uint32_t tile_rows, int64_t rows,
                                                      const uint32_t* __restrict__ seg_row_ptr,
                                                      const uint32_t* __restrict__ seg_col,
                                                      const uint16_t* __restrict__ cmask,
                                                      const uint32_t* __restrict__ elem_off,
                                                      const float* __restrict__ cvals,
                                                      const int64_t* __restrict__ row_ptr,
                                                      int32_t* __restrict__ col,
                                                      float* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows) return;
  const uint32_t s0 = seg_row_ptr[I], s1 = seg_row_ptr[I + 1];
  const int r = lane & 15;
  const int hi = lane >> 4;
  const int64_t row = int64_t(I) * 16 + r;
  int64_t cur = (row < rows) ? row_ptr[row] : 0;
  for (uint32_t sb = s0; sb < s1; sb += 2) {
    const uint32_t s = sb + hi;
    const bool act = s < s1;
    const unsigned m = act ? __ldg(cmask + size_t(s) * 16 + r) : 0u;
    const unsigned n = __popc(m);
    // row-major prefix inside the tile: rows < r of the same tile
    unsigned incl = n;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const unsigned v = __shfl_up_sync(kFull, incl, o, 16);
      if (r >= o) incl += v;
    }
    const unsigned pre = incl - n;
    // lanes 16-31 (second tile) start after lane r's first-tile run
    const unsigned n_first = __shfl_sync(kFull, n, r);
    const int64_t my_cur = cur + (hi ? n_first : 0);
    if (act && n) {
      const uint32_t J = __ldg(seg_col + s);
      const float* src = cvals + __ldg(elem_off + s) + pre;
      unsigned mm = m;
      int64_t d = my_cur;
      int q = 0;
      while (mm) {
        const int c = __ffs(mm) - 1;
        mm &= mm - 1;
        col[d] = int32_t(J * 16 + c);
        val[d] = __ldg(src + q);
        ++q;
        ++d;
      }
    }
    const unsigned n_second = __shfl_sync(kFull, n, r + 16);
    cur += n_first + n_second;
  }
}

}  // namespace

void launch_out_rowcount(const TileMat& A, int64_t rows, const TaskList& tl, const OutTiles& ot,
                         int64_t* rowcnt, cudaStream_t st) {
  const unsigned blocks = (A.tile_rows + 7) / 8;
  if (blocks == 0) return;
  out_rowcount_kernel<<<blocks, 256, 0, st>>>(A.tile_rows, rows, tl.seg_row_ptr, ot.cmask, rowcnt);
}

void launch_out_fill(const TileMat& A, int64_t rows, const TaskList& tl, const OutTiles& ot,
                     const int64_t* row_ptr, int32_t* col, float* val, cudaStream_t st) {
  const unsigned blocks = (A.tile_rows + 7) / 8;
  if (blocks == 0) return;
  out_fill_kernel<<<blocks, 256, 0, st>>>(A.tile_rows, rows, tl.seg_row_ptr, tl.seg_col, ot.cmask,
                                          ot.elem_off, ot.vals, row_ptr, col, val);
}

}  // namespace tsg
