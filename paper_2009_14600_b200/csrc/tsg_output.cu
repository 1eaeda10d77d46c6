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

// Segment chunks: a tile row's segments in runs of at most kChunkSegs, so
// hub tile rows (R-MAT) are spread over many warps.  Thread per tile row.
__global__ void chunk_fill_kernel(uint32_t tile_rows, const uint32_t* __restrict__ srp,
                                  const uint32_t* __restrict__ chunk_base, AsmChunks ch) {
  const uint32_t I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I > tile_rows) return;
  if (I == tile_rows) {
    *ch.n = chunk_base[tile_rows];
    return;
  }
  const uint32_t s0 = srp[I], s1 = srp[I + 1];
  uint32_t c = chunk_base[I];
  for (uint32_t s = s0; s < s1; s += kChunkSegs, ++c) {
    ch.tile_row[c] = I;
    ch.seg_begin[c] = s;
    ch.seg_end[c] = min(s1, s + kChunkSegs);
  }
}

__global__ void chunk_count_kernel(uint32_t tile_rows, const uint32_t* __restrict__ srp,
                                   uint32_t* __restrict__ nchunks) {
  const uint32_t I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I < tile_rows) nchunks[I] = (srp[I + 1] - srp[I] + kChunkSegs - 1) / kChunkSegs;
}

// Realised entries per (chunk, CSR row): warp per chunk, lanes over its
// segments (32-byte row-mask record per segment); row totals by atomics.
__global__ void __launch_bounds__(256) row_count_kernel(int64_t rows, AsmChunks ch,
                                                       const uint16_t* __restrict__ rmask,
                                                       unsigned long long* __restrict__ rowcnt) {
  const int lane = threadIdx.x & 31;
  const uint32_t c = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (c >= *ch.n) return;
  const uint32_t s0 = ch.seg_begin[c], s1 = ch.seg_end[c], I = ch.tile_row[c];
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
  if (lane < 16) {
    ch.off[size_t(c) * 16 + lane] = mine;  // count for now; offsets after the scan
    if (row < rows && mine) atomicAdd(rowcnt + row, (unsigned long long)mine);
  }
}

// Counts -> CSR offsets of each chunk's rows: warp per tile row walks its
// chunks in order (lane r carries row r).
__global__ void __launch_bounds__(256) chunk_offset_kernel(int64_t rows, uint32_t tile_rows,
                                                          const uint32_t* __restrict__ chunk_base,
                                                          const int64_t* __restrict__ row_ptr, AsmChunks ch) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows || lane >= 16) return;
  const int64_t row = int64_t(I) * 16 + lane;
  uint32_t carry = row < rows ? uint32_t(row_ptr[row]) : 0u;
  for (uint32_t c = chunk_base[I]; c < chunk_base[I + 1]; ++c) {
    const uint32_t n = ch.off[size_t(c) * 16 + lane];
    ch.off[size_t(c) * 16 + lane] = carry;
    carry += n;
  }
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

constexpr uint32_t kAsmW = 512;  // staged values per warp batch (shared memory)

// Warp per tile row.  Segments are taken in batches of up to 32 (lane j =
// segment j of the batch) whose staged values fit kAsmW.  Every entry of a
// batch goes to row r's CSR range at an offset = entries of row r in
// earlier segments of the tile row (segments are in column order) -- a
// stable partition of the batch's entries by r:
//   (1) scatter: lanes over the batch's staged entries (contiguous per
//       segment, so the global reads coalesce); entry e of segment j finds
//       its row from the segment's 16 row-prefix bytes and its column from
//       the row mask, ranks itself among the lanes holding the same row
//       (match.any) and lands in shared memory at the batch's row-r offset;
//   (2) copy out: lanes over the batch's entries in row order; each store
//       instruction covers at most a few contiguous CSR ranges.
// Non-finite values raise kErrPrecision here (finalize_segment's check,
// kernels.cpp:115-127).
__global__ void __launch_bounds__(256) assemble_kernel(int64_t rows, AsmChunks ch, TaskList tl, Staged sg,
                                                      int32_t* __restrict__ col,
                                                      float* __restrict__ val,
                                                      unsigned* __restrict__ err_flag) {
  __shared__ float s_val[8][kAsmW];
  __shared__ int32_t s_col[8][kAsmW];
  __shared__ uint4 s_pre[8][32];   // per batch segment: 16 exclusive row-prefix bytes
  __shared__ uint4 s_msk[8][64];   // per batch segment: 16 row masks (two uint4)
  __shared__ uint32_t s_ctr[8][16];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const uint32_t c = blockIdx.x * 8 + w;
  if (c >= *ch.n) return;
  float* sv = s_val[w];
  int32_t* sc = s_col[w];
  const uint32_t s0 = ch.seg_begin[c], s1 = ch.seg_end[c];
  // lane r: CSR position of row r's first entry in this chunk
  uint32_t carry = lane < 16 ? ch.off[size_t(c) * 16 + lane] : 0u;
  const uint4* rec = reinterpret_cast<const uint4*>(sg.rmask);
  const unsigned lt = lanemask_lt();
  bool bad = false;
  for (uint32_t sb = s0; sb < s1;) {
    const uint32_t s = sb + lane;
    uint4 lo = make_uint4(0, 0, 0, 0), hi = lo;
    if (s < s1) {
      lo = __ldg(rec + 2 * uint64_t(s));
      hi = __ldg(rec + 2 * uint64_t(s) + 1);
    }
    const uint32_t m2[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};  // rows 2i | 2i+1 << 16
    uint32_t pc[16];
    uint32_t tot = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      pc[r] = __popc((m2[r >> 1] >> (16 * (r & 1))) & 0xffffu);
      tot += pc[r];
    }
    uint32_t incl = warp_incl_scan(tot, lane);
    // batch = the longest prefix of segments whose values fit (>= 1: tot <= 256)
    const uint32_t nb = __popc(__ballot_sync(kFull, s < s1 && incl <= kAsmW));
    const uint32_t T = __shfl_sync(kFull, incl, nb - 1);
    const bool in = uint32_t(lane) < nb;
    if (!in) {
#pragma unroll
      for (int r = 0; r < 16; ++r) pc[r] = 0;
      tot = 0;
      incl = T;
    }
    const uint32_t so = in ? __ldg(tl.stage_off + s) : 0u;
    const uint32_t cbase = in ? __ldg(tl.seg_col + s) * 16u : 0u;
    // per-segment row prefixes (bytes: <= 240 before row 15) and masks
    uint32_t pw[4] = {0, 0, 0, 0}, run = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      pw[r >> 2] |= run << (8 * (r & 3));
      run += pc[r];
    }
    s_pre[w][lane] = make_uint4(pw[0], pw[1], pw[2], pw[3]);
    s_msk[w][2 * lane] = in ? lo : make_uint4(0, 0, 0, 0);
    s_msk[w][2 * lane + 1] = in ? hi : make_uint4(0, 0, 0, 0);
    // batch row totals -> row offsets in shared memory (lane r holds row r)
    uint32_t ro = 0, rt_mine = 0, acc = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t t = __reduce_add_sync(kFull, pc[r]);
      if (lane == r) {
        ro = acc;
        rt_mine = t;
      }
      acc += t;
    }
    if (lane < 16) s_ctr[w][lane] = 0;
    __syncwarp();
    // (1) scatter into row order
    const uint32_t excl = incl - tot;
    for (uint32_t q0 = 0; q0 < T; q0 += 32) {
      const uint32_t q = q0 + lane;
      const int j = owner_of(incl, q);
      const uint32_t ej = __shfl_sync(kFull, excl, j);
      const uint32_t soj = __shfl_sync(kFull, so, j);
      const uint32_t cbj = __shfl_sync(kFull, cbase, j);
      const bool act = q < T;
      const uint32_t e = q - ej;
      uint32_t r = 16;  // sentinel for inactive lanes
      float x = 0.0f;
      int32_t c = 0;
      if (act) {
        x = __ldg(sg.val + soj + e);
        const uint4 pv = s_pre[w][j];
        const uint32_t pb[4] = {pv.x, pv.y, pv.z, pv.w};
        r = 0;  // last row whose prefix is <= e (prefixes are non-decreasing)
#pragma unroll
        for (int b = 8; b > 0; b >>= 1) {
          const uint32_t rr = r + b;
          const uint32_t pre = (pb[rr >> 2] >> (8 * (rr & 3))) & 0xffu;
          if (pre <= e) r = rr;
        }
        const uint32_t pre_r = (pb[r >> 2] >> (8 * (r & 3))) & 0xffu;
        const uint32_t m = reinterpret_cast<const uint16_t*>(&s_msk[w][2 * j])[r];
        c = int32_t(cbj + kth_bit(m, e - pre_r));
      }
      const unsigned grp = __match_any_sync(kFull, r);
      const uint32_t ro_r = __shfl_sync(kFull, ro, r & 15);
      if (act) {
        const uint32_t d = ro_r + s_ctr[w][r] + __popc(grp & lt);
        sv[d] = x;
        sc[d] = c;
      }
      __syncwarp();
      if (act && (grp >> lane) == 1u) s_ctr[w][r] += __popc(grp);  // highest lane of the group
      __syncwarp();
    }
    // (2) copy out in row order: position q -> row r (lane r holds ro, rt)
    for (uint32_t q0 = 0; q0 < T; q0 += 32) {
      const uint32_t q = q0 + lane;
      int r = 0;
#pragma unroll
      for (int b = 8; b > 0; b >>= 1) {
        const uint32_t v = __shfl_sync(kFull, ro, r + b);
        if (v <= q) r += b;
      }
      // rows with no entries share their offset with the next row: the search
      // lands on the last such row, whose offset is still ro_r <= q
      const uint32_t ro_r = __shfl_sync(kFull, ro, r), base = __shfl_sync(kFull, carry, r);
      if (q < T) {
        const float x = sv[q];
        bad |= !isfinite(x);
        const uint32_t dst = base + (q - ro_r);
        col[dst] = sc[q];
        val[dst] = x;
      }
    }
    if (lane < 16) carry += rt_mine;
    __syncwarp();
    sb += nb;
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(err_flag, unsigned(kErrPrecision));
}

}  // namespace

void launch_asm_chunks(uint32_t tile_rows, const uint32_t* seg_row_ptr, uint32_t* nchunks, cudaStream_t st) {
  if (tile_rows == 0) return;
  chunk_count_kernel<<<(tile_rows + 255) / 256, 256, 0, st>>>(tile_rows, seg_row_ptr, nchunks);
}

void launch_asm_chunk_fill(uint32_t tile_rows, const uint32_t* seg_row_ptr, const uint32_t* chunk_base,
                           AsmChunks& ch, cudaStream_t st) {
  chunk_fill_kernel<<<(tile_rows + 1 + 255) / 256, 256, 0, st>>>(tile_rows, seg_row_ptr, chunk_base, ch);
}

void launch_row_counts(int64_t rows, const AsmChunks& ch, uint64_t max_chunks, const Staged& sg,
                       int64_t* rowcnt, cudaStream_t st) {
  const uint64_t blocks = (max_chunks + 7) / 8;
  if (blocks == 0) return;
  row_count_kernel<<<unsigned(blocks), 256, 0, st>>>(rows, ch, sg.rmask,
                                                      reinterpret_cast<unsigned long long*>(rowcnt));
}

void launch_chunk_offsets(int64_t rows, uint32_t tile_rows, const uint32_t* chunk_base, const int64_t* row_ptr,
                          AsmChunks& ch, cudaStream_t st) {
  const unsigned blocks = (tile_rows + 7) / 8;
  if (blocks == 0) return;
  chunk_offset_kernel<<<blocks, 256, 0, st>>>(rows, tile_rows, chunk_base, row_ptr, ch);
}

void launch_assemble(int64_t rows, const AsmChunks& ch, uint64_t max_chunks, const TaskList& tl,
                     const Staged& sg, int32_t* col, float* val, unsigned* err_flag, cudaStream_t st) {
  const uint64_t blocks = (max_chunks + 7) / 8;
  if (blocks == 0) return;
  assemble_kernel<<<unsigned(blocks), 256, 0, st>>>(rows, ch, tl, sg, col, val, err_flag);
}

}  // namespace tsg
