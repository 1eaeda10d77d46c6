// tsg_symbolic.cu -- subsystem (2): tile-pair task list and boolean sizing.
//
// GPU restatement at T = 16 of
//   enumerate_pairs       proj/src/pipeline.cpp:37-60
//   filter_zero_products  proj/src/pipeline.cpp:62-70  (tile_product_nonzero :23-35)
//   sort_and_segment      proj/src/pipeline.cpp:72-109 (segment part; the sort
//                         itself is a stable segmented radix sort, tsg_api.cu)
//   counting_pass         proj/src/kernels.cpp:79-103  (boolean_tile_mm pipeline.cpp:11-21)
//
// Enumeration and filtering are fused (raw 16x16 pair counts
// are 12-16x the filtered ones on the sparse configs), count-then-fill, so
// raw pairs are never materialised.  Work unit: one warp per 32 consecutive
// A tiles; the warp flattens their raw pairs (sum of B tile-row lengths) and
// load-balances them across lanes with a shuffle binary search, so skewed
// B tile rows (R-MAT) keep all lanes busy.  Pairs of one A tile are written
// in ascending B-tile order at the A tile's prefix-sum offset, i.e. the
// reference's enumeration order (A tiles in (row, col) order, then B tiles).
#include "tsg_kernels.cuh"

namespace tsg {

namespace {

template <bool kFill>
__global__ void __launch_bounds__(256) enum_kernel(TileMat A, TileMat B, uint64_t tA,
                                                  uint32_t* __restrict__ tile_cnt,
                                                  const uint32_t* __restrict__ tile_off,
                                                  uint64_t* __restrict__ pairs,
                                                  uint32_t* __restrict__ keys,
                                                  unsigned long long* __restrict__ raw_total) {
  __shared__ uint32_t s_cnt[8][33];
  __shared__ unsigned long long s_raw[8];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t a0 = (uint64_t(blockIdx.x) * 8 + wib) * 32;
  unsigned long long raw = 0;
  if (a0 < tA) {
    const uint64_t a = a0 + lane;
    const bool valid = a < tA;
    uint32_t bs = 0, bl = 0, colocc = 0, base_off = 0;
    if (valid) {
      const uint32_t k = __ldg(A.tcol + a);
      bs = __ldg(B.trp + k);
      bl = __ldg(B.trp + k + 1) - bs;
      colocc = __ldg(A.occ + a) & 0xffffu;
      if (kFill) base_off = __ldg(tile_off + a);
    }
    uint32_t incl = bl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    const uint32_t excl = incl - bl;
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    raw = total;
    s_cnt[wib][lane] = 0;
    __syncwarp();
    for (uint32_t q0 = 0; q0 < total; q0 += 32) {
      const uint32_t q = q0 + lane;
      const bool active = q < total;
      // owner lane = number of lanes whose inclusive end is <= q
      int s = 0;
#pragma unroll
      for (int b = 16; b > 0; b >>= 1) {
        const uint32_t v = __shfl_sync(kFull, incl, s + b - 1);
        if (v <= q) s += b;
      }
      if (!active) s = 32;
      const uint32_t bs_s = __shfl_sync(kFull, bs, s & 31);
      const uint32_t ex_s = __shfl_sync(kFull, excl, s & 31);
      const uint32_t co_s = __shfl_sync(kFull, colocc, s & 31);
      const uint32_t off_s = __shfl_sync(kFull, base_off, s & 31);
      const uint32_t b = bs_s + (q - ex_s);
      bool pass = false;
      if (active) pass = (co_s & (__ldg(B.occ + b) >> 16)) != 0;
      const unsigned grp = __match_any_sync(kFull, s);
      const unsigned pb = __ballot_sync(kFull, pass);
      const uint32_t before = s_cnt[wib][s];
      if (kFill && pass) {
        const uint32_t pos = off_s + before + __popc(pb & grp & lanemask_lt());
        pairs[pos] = (a0 + uint64_t(s)) | (uint64_t(b) << 32);
        keys[pos] = __ldg(B.tcol + b);
      }
      __syncwarp();
      if (active && lane == __ffs(grp) - 1) s_cnt[wib][s] = before + __popc(pb & grp);
      __syncwarp();
    }
    if (!kFill && valid) tile_cnt[a] = s_cnt[wib][lane];
  }
  if (!kFill) {
    if (lane == 0) s_raw[wib] = raw;  // warp-uniform
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < 8; ++w) t += s_raw[w];
      if (t) atomicAdd(raw_total, t);
    }
  }
}

__global__ void row_pair_off_kernel(const uint32_t* __restrict__ trp, uint32_t tile_rows,
                                    const uint32_t* __restrict__ tile_off,
                                    uint32_t* __restrict__ row_pair_off) {
  const uint32_t I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I <= tile_rows) row_pair_off[I] = tile_off[trp[I]];
}

// Segment heads after the per-row sort: a new segment starts at each row
// start and wherever the output tile column changes (pipeline.cpp:94-107).
template <bool kFill>
__global__ void __launch_bounds__(256) seg_kernel(uint32_t tile_rows,
                                                 const uint32_t* __restrict__ row_pair_off,
                                                 const uint32_t* __restrict__ keys,
                                                 uint32_t* __restrict__ row_nseg,
                                                 const uint32_t* __restrict__ seg_row_ptr,
                                                 uint32_t* __restrict__ seg_off,
                                                 uint32_t* __restrict__ seg_col) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows) return;
  const uint32_t lo = row_pair_off[I], hi = row_pair_off[I + 1];
  uint32_t carry = 0xffffffffu;
  uint32_t nseg = 0;
  const uint32_t base = kFill ? seg_row_ptr[I] : 0;
  for (uint32_t i0 = lo; i0 < hi; i0 += 32) {
    const uint32_t i = i0 + lane;
    const bool active = i < hi;
    const uint32_t key = active ? __ldg(keys + i) : 0xfffffffeu;
    uint32_t prev = __shfl_up_sync(kFull, key, 1);
    if (lane == 0) prev = carry;
    const bool head = active && key != prev;
    const unsigned hb = __ballot_sync(kFull, head);
    if (kFill && head) {
      const uint32_t s = base + nseg + __popc(hb & lanemask_lt());
      seg_off[s] = i;
      seg_col[s] = key;
    }
    nseg += __popc(hb);
    carry = __shfl_sync(kFull, key, 31);
  }
  if (!kFill && lane == 0) row_nseg[I] = nseg;
}

// counting_pass: per segment OR of boolean 16x16 products, popcount.
// Lanes 0-15 / 16-31 take alternating pairs; lane r&15 owns output row r.
__global__ void __launch_bounds__(256) counting_kernel(TileMat A, TileMat B, TaskList tl,
                                                      uint32_t* __restrict__ counted) {
  const int lane = threadIdx.x & 31;
  const uint64_t s = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (s >= tl.nseg) return;
  const uint32_t p0 = tl.seg_off[s], p1 = tl.seg_off[s + 1];
  const int r = lane & 15;
  uint32_t acc = 0;
  for (uint32_t p = p0 + (lane >> 4); p < p1; p += 2) {
    const uint64_t pr = __ldg(reinterpret_cast<const unsigned long long*>(tl.pairs) + p);
    const uint32_t a = uint32_t(pr), b = uint32_t(pr >> 32);
    const uint32_t ra = __ldg(A.rmask + size_t(a) * 16 + r);
    const uint4* bm = reinterpret_cast<const uint4*>(B.rmask + size_t(b) * 16);
    const uint4 b0 = __ldg(bm), b1 = __ldg(bm + 1);
    const uint32_t w[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    uint32_t out = 0;
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const uint32_t brow = (w[kk >> 1] >> (16 * (kk & 1))) & 0xffffu;
      out |= (0u - ((ra >> kk) & 1u)) & brow;
    }
    acc |= out;
  }
  acc |= __shfl_xor_sync(kFull, acc, 16);
  const uint32_t cnt = __reduce_add_sync(kFull, lane < 16 ? __popc(acc) : 0u);
  if (lane == 0) counted[s] = cnt;
}

}  // namespace

void launch_enum_count(const TileMat& A, const TileMat& B, uint64_t tA, uint32_t* tile_cnt,
                       unsigned long long* raw_total, cudaStream_t st) {
  const uint64_t warps = (tA + 31) / 32;
  const uint64_t blocks = (warps + 7) / 8;
  if (blocks == 0) return;
  enum_kernel<false><<<unsigned(blocks), 256, 0, st>>>(A, B, tA, tile_cnt, nullptr, nullptr,
                                                        nullptr, raw_total);
}

void launch_enum_fill(const TileMat& A, const TileMat& B, uint64_t tA, const uint32_t* tile_off,
                      uint64_t* pairs, uint32_t* keys, cudaStream_t st) {
  const uint64_t warps = (tA + 31) / 32;
  const uint64_t blocks = (warps + 7) / 8;
  if (blocks == 0) return;
  enum_kernel<true><<<unsigned(blocks), 256, 0, st>>>(A, B, tA, nullptr, tile_off, pairs, keys,
                                                       nullptr);
}

void launch_row_pair_off(const TileMat& A, const uint32_t* tile_off, uint32_t* row_pair_off,
                         cudaStream_t st) {
  const uint32_t n = A.tile_rows + 1;
  row_pair_off_kernel<<<(n + 255) / 256, 256, 0, st>>>(A.trp, A.tile_rows, tile_off,
                                                       row_pair_off);
}

void launch_seg_count(const TileMat& A, const uint32_t* row_pair_off, const uint32_t* keys,
                      uint32_t* row_nseg, cudaStream_t st) {
  const unsigned blocks = (A.tile_rows + 7) / 8;
  if (blocks == 0) return;
  seg_kernel<false><<<blocks, 256, 0, st>>>(A.tile_rows, row_pair_off, keys, row_nseg, nullptr,
                                            nullptr, nullptr);
}

void launch_seg_fill(const TileMat& A, const uint32_t* row_pair_off, const uint32_t* keys,
                     const uint32_t* seg_row_ptr, uint32_t* seg_off, uint32_t* seg_col,
                     cudaStream_t st) {
  const unsigned blocks = (A.tile_rows + 7) / 8;
  if (blocks == 0) return;
  seg_kernel<true><<<blocks, 256, 0, st>>>(A.tile_rows, row_pair_off, keys, nullptr, seg_row_ptr,
                                           seg_off, seg_col);
}

void launch_counting(const TileMat& A, const TileMat& B, const TaskList& tl, uint32_t* counted,
                     cudaStream_t st) {
  const uint64_t blocks = (tl.nseg + 7) / 8;
  if (blocks == 0) return;
  counting_kernel<<<unsigned(blocks), 256, 0, st>>>(A, B, tl, counted);
}

}  // namespace tsg
