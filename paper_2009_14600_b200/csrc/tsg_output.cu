// tsg_output.cu -- subsystem (4): tiled -> CSR.
//
// The numeric kernel leaves every output tile's realised entries packed
// row-major at its staging offset and its realised bitmap as 16 row
// masks -- the reference's
// MulResult after compact() (kernels.cpp:205-220; zero accumulators are
// already gone).  This file is to_element_coo (tile_format.cpp:131-154):
// instead of a countr_zero walk plus a global (row, col) sort, the CSR
// position of every entry follows from counts alone, because a tile row's
// segments are already in column order:
//
//   row_count_kernel   counted entries per CSR row        (warp per tile row)
//   CUB exclusive scan -> row_ptr                          (tsg_api.cu)
//   assemble_kernel    a batch of segments' staged values into shared
//                      memory, then per row of the tile row a warp-wide
//                      scan of the batch's run lengths and a flattened copy
//                      in CSR order (lanes over output positions: each
//                      store is contiguous, and 1-entry tiles do not idle
//                      the warp); columns come from the row masks.
#include "tsg_kernels.cuh"

namespace tsg {

namespace {

// Realised entries per CSR row: warp per tile row, lanes over its segments
// (32-byte row-mask record per segment), one sum per row r.
__global__ void __launch_bounds__(256) row_count_kernel(int64_t rows, uint32_t tile_rows,
                                                       const uint32_t* __restrict__ srp,
                                                       const uint16_t* __restrict__ rmask,
                                                       int64_t* __restrict__ rowcnt) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows) return;
  const uint32_t s0 = srp[I], s1 = srp[I + 1];
  uint32_t sum[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) sum[r] = 0;
  const uint4* rec = reinterpret_cast<const uint4*>(rmask);
  for (uint32_t s = s0 + lane; s < s1; s += 32) {
    const uint4 lo = __ldg(rec + 2 * uint64_t(s)), hi = __ldg(rec + 2 * uint64_t(s) + 1);
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
    for (int r = 0; r < 16; ++r) sum[r] += __popc((w[r >> 1] >> (16 * (r & 1))) & 0xffffu);
  }
  uint32_t mine = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t t = __reduce_add_sync(kFull, sum[r]);
    if (lane == r) mine = t;
  }
  const int64_t row = int64_t(I) * 16 + lane;
  if (lane < 16 && row < rows) rowcnt[row] = mine;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// lane owning flattened index q: the number of lanes whose inclusive end is <= q
__device__ __forceinline__ int owner_of(uint32_t incl, uint32_t q) {
  int j = 0;
#pragma unroll
  for (int b = 16; b > 0; b >>= 1) {
    const uint32_t e = __shfl_sync(kFull, incl, j + b - 1);
    if (e <= q) j += b;
  }
  return j & 31;
}

// column of the k-th (0-based) set bit of a 16-bit row mask
__device__ __forceinline__ uint32_t kth_bit(uint32_t m, uint32_t k) {
  uint32_t c = 0;
#pragma unroll
  for (int b = 8; b > 0; b >>= 1)
    if (__popc(m & ((1u << (c + b)) - 1u)) <= k) c += b;
  return c;
}

constexpr uint32_t kAsmW = 1024;  // staged values per warp batch (shared memory)

// Warp per tile row.  Segments are taken in batches of up to 32 whose
// staged values fit kAsmW: (1) the batch's staged runs are copied into
// shared memory (flattened over the segments, contiguous per segment);
// (2) for each row r of the tile row, the runs of row r of the batch's
// segments are consecutive in the CSR (segments are in column order), so
// the copy is flattened over them: lane q of an iteration writes CSR
// position base_r + q -- every store instruction is one contiguous,
// coalesced range -- taking its value from shared memory and its column
// from the owning segment's row mask.  Non-finite values raise
// kErrPrecision here (finalize_segment's check, kernels.cpp:115-127).
__global__ void __launch_bounds__(256) assemble_kernel(int64_t rows, uint32_t tile_rows, TaskList tl,
                                                      Staged sg, const int64_t* __restrict__ row_ptr,
                                                      int32_t* __restrict__ col,
                                                      float* __restrict__ val,
                                                      unsigned* __restrict__ err_flag) {
  __shared__ float s_val[8][kAsmW];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const uint32_t I = blockIdx.x * 8 + w;
  if (I >= tile_rows) return;
  float* sv = s_val[w];
  const uint32_t s0 = tl.seg_row_ptr[I], s1 = tl.seg_row_ptr[I + 1];
  const int64_t row = int64_t(I) * 16 + (lane & 15);
  uint32_t carry = (lane < 16 && row < rows) ? uint32_t(row_ptr[row]) : 0u;  // lane r: row r
  const uint4* rec = reinterpret_cast<const uint4*>(sg.rmask);
  bool bad = false;
  for (uint32_t sb = s0; sb < s1;) {
    const uint32_t s = sb + lane;
    uint4 lo = make_uint4(0, 0, 0, 0), hi = lo;
    if (s < s1) {
      lo = __ldg(rec + 2 * uint64_t(s));
      hi = __ldg(rec + 2 * uint64_t(s) + 1);
    }
    uint32_t m2[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};  // rows 2i | 2i+1 << 16
    uint32_t tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) tot += __popc(m2[i]);
    uint32_t incl = warp_incl_scan(tot, lane);
    // batch = the longest prefix of segments whose values fit (>= 1: tot <= 256)
    const unsigned fit = __ballot_sync(kFull, s < s1 && incl <= kAsmW);
    const uint32_t nb = __popc(fit);
    const uint32_t T = __shfl_sync(kFull, incl, nb - 1);
    if (uint32_t(lane) >= nb) {  // not in this batch
#pragma unroll
      for (int i = 0; i < 8; ++i) m2[i] = 0;
      tot = 0;
      incl = T;
    }
    const uint32_t so = (uint32_t(lane) < nb) ? __ldg(tl.stage_off + s) : 0u;
    const uint32_t cbase = (uint32_t(lane) < nb) ? __ldg(tl.seg_col + s) * 16u : 0u;
    // (1) staged runs -> shared memory
    {
      const uint32_t from = so - (incl - tot);
      for (uint32_t q0 = 0; q0 < T; q0 += 32) {
        const uint32_t q = q0 + lane;
        const int j = owner_of(incl, q);
        const uint32_t f = __shfl_sync(kFull, from, j);
        if (q < T) sv[q] = __ldg(sg.val + f + q);
      }
    }
    __syncwarp();
    // (2) row by row, CSR order
    uint32_t src = incl - tot;  // shared-memory start of this segment's row r
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t m = (m2[r >> 1] >> (16 * (r & 1))) & 0xffffu;
      const uint32_t v = __popc(m);
      const uint32_t ri = warp_incl_scan(v, lane);
      const uint32_t rt = __shfl_sync(kFull, ri, 31);
      if (rt) {
        const uint32_t base = __shfl_sync(kFull, carry, r);
        const uint32_t from = src - (ri - v);
        for (uint32_t q0 = 0; q0 < rt; q0 += 32) {
          const uint32_t q = q0 + lane;
          const int j = owner_of(ri, q);
          const uint32_t f = __shfl_sync(kFull, from, j);
          const uint32_t mj = __shfl_sync(kFull, m, j);
          const uint32_t ej = __shfl_sync(kFull, ri - v, j);
          const uint32_t cb = __shfl_sync(kFull, cbase, j);
          if (q < rt) {
            const float x = sv[f + q];
            bad |= !isfinite(x);
            col[base + q] = int32_t(cb + kth_bit(mj, q - ej));
            val[base + q] = x;
          }
        }
        if (lane == r) carry += rt;
      }
      src += v;
    }
    __syncwarp();
    sb += nb;
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(err_flag, unsigned(kErrPrecision));
}

}  // namespace

void launch_row_counts(int64_t rows, uint32_t tile_rows, const TaskList& tl, const Staged& sg,
                       int64_t* rowcnt, cudaStream_t st) {
  const unsigned blocks = (tile_rows + 7) / 8;
  if (blocks == 0) return;
  row_count_kernel<<<blocks, 256, 0, st>>>(rows, tile_rows, tl.seg_row_ptr, sg.rmask, rowcnt);
}

void launch_assemble(int64_t rows, uint32_t tile_rows, const TaskList& tl, const Staged& sg,
                     const int64_t* row_ptr, int32_t* col, float* val, unsigned* err_flag,
                     cudaStream_t st) {
  const unsigned blocks = (tile_rows + 7) / 8;
  if (blocks == 0) return;
  assemble_kernel<<<blocks, 256, 0, st>>>(rows, tile_rows, tl, sg, row_ptr, col, val, err_flag);
}

}  // namespace tsg
