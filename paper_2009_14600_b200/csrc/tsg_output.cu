// tsg_output.cu -- subsystem (4): tiled -> CSR and the compaction fix-up.
//
// The tiled -> CSR conversion of the reference (to_element_coo,
// proj/src/tile_format.cpp:131-154: countr_zero walk + global (row, col)
// sort) is folded into the numeric phase: tiles of a tile row are already
// in column order, so the counting pass's transposed prefix gives every
// output slot its final CSR position and the numeric kernel stores there
// (tsg_numeric.cu).  What remains here is compact() (kernels.cpp:205-220)
// for the case the reference's counting pass exists for: an output slot
// that the boolean product counted but whose value cancelled to exactly 0.
// The numeric kernel marks those slots col = -1; these kernels squeeze them
// out of each row in order (one warp per row, ballot compaction), keeping
// the output deterministic.  Skipped entirely when nothing cancelled.
#include "tsg_kernels.cuh"

namespace tsg {

namespace {

__global__ void __launch_bounds__(256) compact_count_kernel(int64_t rows,
                                                           const int64_t* __restrict__ rp,
                                                           const int32_t* __restrict__ col,
                                                           int64_t* __restrict__ rowcnt) {
  const int lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int64_t lo = rp[row], hi = rp[row + 1];
  int64_t n = 0;
  for (int64_t i = lo + lane; i < hi; i += 32) n += __ldg(col + i) >= 0;
  n = __reduce_add_sync(kFull, unsigned(n));
  if (lane == 0) rowcnt[row] = n;
}

__global__ void __launch_bounds__(256) compact_fill_kernel(int64_t rows,
                                                          const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ col_in,
                                                          const float* __restrict__ val_in,
                                                          const int64_t* __restrict__ new_rp,
                                                          int32_t* __restrict__ col,
                                                          float* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int64_t lo = rp[row], hi = rp[row + 1];
  int64_t dst = new_rp[row];
  for (int64_t i0 = lo; i0 < hi; i0 += 32) {
    const int64_t i = i0 + lane;
    const int32_t c = i < hi ? __ldg(col_in + i) : -1;
    const bool keep = c >= 0;
    const unsigned kb = __ballot_sync(kFull, keep);
    if (keep) {
      const int64_t d = dst + __popc(kb & lanemask_lt());
      col[d] = c;
      val[d] = __ldg(val_in + i);
    }
    dst += __popc(kb);
  }
}

}  // namespace

void launch_compact_count(int64_t rows, const OutPlan& op, int64_t* rowcnt, cudaStream_t st) {
  const uint64_t blocks = (uint64_t(rows) + 7) / 8;
  if (blocks == 0) return;
  compact_count_kernel<<<unsigned(blocks), 256, 0, st>>>(rows, op.row_ptr, op.col, rowcnt);
}

void launch_compact_fill(int64_t rows, const OutPlan& op, const int64_t* new_rp, int32_t* col,
                         float* val, cudaStream_t st) {
  const uint64_t blocks = (uint64_t(rows) + 7) / 8;
  if (blocks == 0) return;
  compact_fill_kernel<<<unsigned(blocks), 256, 0, st>>>(rows, op.row_ptr, op.col, op.val, new_rp,
                                                        col, val);
}

}  // namespace tsg
