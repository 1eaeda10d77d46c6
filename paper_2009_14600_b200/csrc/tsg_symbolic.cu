// tsg_symbolic.cu -- subsystem (2): tile-pair task list and boolean sizing.
//
// GPU restatement at T = 16 of
//   enumerate_pairs       proj/src/pipeline.cpp:37-60
//   filter_zero_products  proj/src/pipeline.cpp:62-70  (tile_product_nonzero :23-35)
//   sort_and_segment      proj/src/pipeline.cpp:72-109
//   counting_pass         proj/src/kernels.cpp:79-103  (boolean_tile_mm pipeline.cpp:11-21)
//
// Two ways to build the task list; both yield the identical TaskList (pairs
// sorted by (out row, out col, k), one segment per output tile):
//
//  * light rows (every A tile row has <= 32 tiles -- FEM27, Poisson, AMG):
//    one warp per tile row, lane l owns A tile (I, k_l) and walks B tile row
//    k_l (sorted by J).  Each step takes the minimum pending J (REDUX): the
//    lanes holding it are exactly that output tile's pairs, already in
//    ascending k (lane order).  This is a 32-way merge -- the sort the
//    reference does with std::sort on (row, col, k) keys happens in
//    registers, and segments fall out directly.  Count pass + prefix sums +
//    fill pass; the zero-product filter is applied per pair on the fly.
//
//  * general rows: fused enumerate+filter (count, scan, fill; raw pairs are
//    never materialised), a stable segmented radix sort by
//    output tile column per tile row (tsg_api.cu), then segment heads.
//    One warp per 32 consecutive A tiles flattens their raw pairs and
//    load-balances them across lanes with a shuffle binary search, so
//    skewed B tile rows (R-MAT) keep all lanes busy.
//
// counting_pass: boolean 16x16 tile products OR-accumulated per segment run
// on the u8 tensor cores: mma.m16n8k32 u8 multiplies two tile pairs per
// instruction (k = 16 inner slots of pair 2m, then 16 of pair 2m+1), 0/1
// operands expanded from the row / column bit masks (two instructions per
// register, see kbytes_lo).  A nonzero count is exactly a structurally
// nonzero output slot.
#include "tsg_kernels.cuh"

namespace tsg {

namespace {

constexpr uint32_t kInf = 0xffffffffu;

// ---------------------------------------------------------------- light rows
template <bool kFill>
__global__ void __launch_bounds__(256) merge_kernel(TileMat A, TileMat B,
                                                   uint32_t* __restrict__ row_np,
                                                   uint32_t* __restrict__ row_ns,
                                                   uint32_t* __restrict__ row_raw,
                                                   const uint32_t* __restrict__ row_pair_off,
                                                   TaskList tl) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= A.tile_rows) return;
  const uint32_t a0 = A.trp[I];
  const uint32_t na = A.trp[I + 1] - a0;  // <= 32 on this path
  uint32_t a = 0, colocc = 0, cur = 0, end = 0;
  uint2 am = make_uint2(0, 0);
  if (lane < na) {
    a = a0 + lane;
    const uint2 ac = __ldg(A.tco + a);
    colocc = ac.y & 0xffffu;
    cur = __ldg(B.trp + ac.x);
    end = __ldg(B.trp + ac.x + 1);
    if (kFill) am = __ldg(A.meta[kRoleA] + a);
  }
  const uint32_t raw_len = end - cur;  // raw pairs of this A tile (pipeline.cpp:52-58)
  uint2 bt = cur < end ? __ldg(B.tco + cur) : make_uint2(kInf, 0);
  uint2 bn = cur + 1 < end ? __ldg(B.tco + cur + 1) : make_uint2(kInf, 0);
  uint32_t np = 0, ns = 0;
  uint32_t pair_base = 0, seg_base = 0;
  if (kFill) {
    pair_base = row_pair_off[I];
    seg_base = tl.seg_row_ptr[I];
  }
  while (true) {
    const uint32_t J = __reduce_min_sync(kFull, bt.x);
    if (J == kInf) break;
    const bool take = bt.x == J;
    const bool pass = take && (colocc & (bt.y >> 16)) != 0u;
    const unsigned pb = __ballot_sync(kFull, pass);
    if (pb) {
      if (kFill) {
        if (pass) {
          const uint32_t pos = pair_base + np + __popc(pb & lanemask_lt());
          tl.pairs[pos] = uint64_t(a) | (uint64_t(cur) << 32);
          const uint2 bm = __ldg(B.meta[kRoleB] + cur);
          tl.pmeta[pos] = make_uint4(am.x, am.y, bm.x, bm.y);
        }
        if (lane == 0) {
          const uint32_t s = seg_base + ns;
          tl.seg_off[s] = pair_base + np;
          tl.seg_col[s] = J;
          tl.seg_row[s] = I;
        }
      }
      np += __popc(pb);
      ++ns;
    }
    if (take) {
      ++cur;
      bt = bn;
      bn = cur + 1 < end ? __ldg(B.tco + cur + 1) : make_uint2(kInf, 0);
    }
  }
  if (!kFill) {
    const uint32_t rw = __reduce_add_sync(kFull, raw_len);
    if (lane == 0) {
      row_np[I] = np;
      row_ns[I] = ns;
      row_raw[I] = rw;
    }
  }
}

// ------------------------------------------------------------- general rows
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
      const uint2 ac = __ldg(A.tco + a);
      bs = __ldg(B.trp + ac.x);
      bl = __ldg(B.trp + ac.x + 1) - bs;
      colocc = ac.y & 0xffffu;
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
      uint2 bt = make_uint2(0, 0);
      if (active) {
        bt = __ldg(B.tco + b);
        pass = (co_s & (bt.y >> 16)) != 0;
      }
      const unsigned grp = __match_any_sync(kFull, s);
      const unsigned pbal = __ballot_sync(kFull, pass);
      const uint32_t before = s_cnt[wib][s];
      if (kFill && pass) {
        const uint32_t pos = off_s + before + __popc(pbal & grp & lanemask_lt());
        pairs[pos] = (a0 + uint64_t(s)) | (uint64_t(b) << 32);
        keys[pos] = bt.x;
      }
      __syncwarp();
      if (active && lane == __ffs(grp) - 1) s_cnt[wib][s] = before + __popc(pbal & grp);
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
                                                 uint32_t* __restrict__ row_nseg, TaskList tl) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows) return;
  const uint32_t lo = row_pair_off[I], hi = row_pair_off[I + 1];
  uint32_t carry = kInf;
  uint32_t nseg = 0;
  const uint32_t base = kFill ? tl.seg_row_ptr[I] : 0;
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
      tl.seg_off[s] = i;
      tl.seg_col[s] = key;
      tl.seg_row[s] = I;
    }
    nseg += __popc(hb);
    carry = __shfl_sync(kFull, key, 31);
  }
  if (!kFill && lane == 0) row_nseg[I] = nseg;
}

// operand metas per sorted pair (general path)
__global__ void pair_meta_kernel(TileMat A, TileMat B, TaskList tl) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= tl.npairs) return;
  const uint64_t pr = tl.pairs[i];
  const uint2 am = __ldg(A.meta[kRoleA] + uint32_t(pr));
  const uint2 bm = __ldg(B.meta[kRoleB] + uint32_t(pr >> 32));
  tl.pmeta[i] = make_uint4(am.x, am.y, bm.x, bm.y);
}

// ------------------------------------------------------------ counting pass
__device__ __forceinline__ void imma_u8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                        uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// 0/1 operand bytes for the u8 MMA.  Any permutation of the inner index k
// is valid as long as A and B agree, so lane t owns the k = t, t+4, t+8,
// t+12 bits of a 16-bit row/column mask: byte i of the register is nonzero
// iff bit t+4i is set.  PRMT duplicates the two mask bytes ({b0,b0,b1,b1},
// or {b2,b2,b3,b3} for the high 16 bits) and one AND with the per-lane mask
// (bits t, 12+t, 16+t, 28+t) isolates the four bits.  Byte values need only
// be zero / nonzero: the MMA sums products, and any positive sum means the
// output slot is structurally nonzero.
__device__ __forceinline__ uint32_t kbytes_lo(uint32_t m, uint32_t tmask) {
  return __byte_perm(m, 0, 0x1100) & tmask;
}
__device__ __forceinline__ uint32_t kbytes_hi(uint32_t m, uint32_t tmask) {
  return __byte_perm(m, 0, 0x3322) & tmask;
}


// One warp per segment.  Lane j loads pair j of the segment (one coalesced
// round per 32 pairs) together with the epilogue's indices; per batch of 8
// pairs the warp broadcasts the tile ids and each lane loads the
// interleaved row word (rows g, g+8) of each A tile and column word (cols
// g, g+8) of each B tile.  Lanes past the segment end hold the pad pair
// {capA, capB}, whose masks are zero.
template <int kCntPairs>  // tile pairs per batch (kCntPairs / 2 IMMA pairs)
__global__ void __launch_bounds__(256) counting_kernel(TileMat A, TileMat B, TaskList tl,
                                                      OutPlan op) {
  const int lane = threadIdx.x & 31;
  const uint64_t s = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (s >= tl.nseg) return;
  const int g = lane >> 2, t = lane & 3;
  const uint32_t p0 = tl.seg_off[s], p1 = tl.seg_off[s + 1];
  int d[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
  const uint2* pairs = reinterpret_cast<const uint2*>(tl.pairs);
  const uint2 pad = pairs[tl.npairs];
  const uint32_t tmask = (1u << t) | (1u << (12 + t)) | (1u << (16 + t)) | (1u << (28 + t));
  for (uint32_t pb = p0; pb < p1; pb += 32) {
    const uint32_t n = min(32u, p1 - pb);
    const uint2 pl = lane < n ? __ldg(pairs + pb + lane) : pad;
    for (uint32_t u0 = 0; u0 < n; u0 += kCntPairs) {
      uint32_t ra[kCntPairs], cb[kCntPairs];
#pragma unroll
      for (int u = 0; u < kCntPairs; ++u) {
        const int q = int(u0) + u;
        const uint32_t a = __shfl_sync(kFull, pl.x, q & 31);
        const uint32_t b = __shfl_sync(kFull, pl.y, q & 31);
        const bool in = u0 + u < 32;  // q wraps past lane 31 only in the last batch
        ra[u] = __ldg(A.rm2 + ((in ? a : pad.x) * 8 + g));  // rows g | g+8 << 16
        cb[u] = __ldg(B.cm2 + ((in ? b : pad.y) * 8 + g));  // cols g | g+8 << 16
      }
#pragma unroll
      for (int u = 0; u < kCntPairs; u += 2) {
        if (u0 + u < n) {
          // k 0..15 = inner slots of pair u, k 16..31 = pair u+1
          const uint32_t a0 = kbytes_lo(ra[u], tmask), a1 = kbytes_hi(ra[u], tmask);
          const uint32_t a2 = kbytes_lo(ra[u + 1], tmask), a3 = kbytes_hi(ra[u + 1], tmask);
          imma_u8(d[0], a0, a1, a2, a3, kbytes_lo(cb[u], tmask), kbytes_lo(cb[u + 1], tmask));
          imma_u8(d[1], a0, a1, a2, a3, kbytes_hi(cb[u], tmask), kbytes_hi(cb[u + 1], tmask));
        }
      }
    }
  }
  unsigned bal[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < 4; ++i) bal[h][i] = __ballot_sync(kFull, d[h][i] != 0);
  const unsigned rmask = row_mask_from_ballots(bal, lane);  // row lane & 15
  const unsigned hi = __shfl_sync(kFull, rmask, (lane & 7) + 8);
  // 64-bit: segments * 16 passes 2^32 on R-MAT (403M segments)
  if (lane < 8) op.bm2[s * 8 + lane] = rmask | (hi << 16);
  if (lane < 16) op.cnt[s * 16 + lane] = uint8_t(__popc(rmask));
}

// Counted entries per CSR row: warp per tile row, lanes over its segments
// (16-byte count record per segment), one sum per row r.
__global__ void __launch_bounds__(256) row_count_kernel(int64_t rows, uint32_t tile_rows,
                                                       const uint32_t* __restrict__ srp,
                                                       const uint8_t* __restrict__ cnt,
                                                       int64_t* __restrict__ rowcnt) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows) return;
  const uint32_t s0 = srp[I], s1 = srp[I + 1];
  uint32_t sum[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) sum[r] = 0;
  for (uint32_t s = s0 + lane; s < s1; s += 32) {
    const uint4 c = __ldg(reinterpret_cast<const uint4*>(cnt) + s);
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int r = 0; r < 16; ++r) sum[r] += (w[r >> 2] >> (8 * (r & 3))) & 0xffu;
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

// pos[s*16 + r] = row_ptr[16I + r] + counted entries of row r in the
// earlier segments of tile row I: warp per tile row, lanes over segments,
// a warp-wide exclusive scan per row r with the carry kept in lane r.
__global__ void __launch_bounds__(256) position_kernel(int64_t rows, uint32_t tile_rows,
                                                      const uint32_t* __restrict__ srp,
                                                      const uint8_t* __restrict__ cnt,
                                                      const int64_t* __restrict__ row_ptr,
                                                      uint32_t* __restrict__ pos) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows) return;
  const uint32_t s0 = srp[I], s1 = srp[I + 1];
  const int64_t row = int64_t(I) * 16 + (lane & 15);
  uint32_t carry = (lane < 16 && row < rows) ? uint32_t(row_ptr[row]) : 0u;  // lane r: row r
  for (uint32_t sb = s0; sb < s1; sb += 32) {
    const uint32_t s = sb + lane;
    const bool act = s < s1;
    const uint4 c = act ? __ldg(reinterpret_cast<const uint4*>(cnt) + s) : make_uint4(0, 0, 0, 0);
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
    uint32_t out[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint32_t v = (w[r >> 2] >> (8 * (r & 3))) & 0xffu;
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t base = __shfl_sync(kFull, carry, r);
      out[r] = base + incl - v;
      const uint32_t tot = __shfl_sync(kFull, incl, 31);
      if (lane == r) carry += tot;
    }
    if (act) {
      uint4* dst = reinterpret_cast<uint4*>(pos + size_t(s) * 16);
      dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
      dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
      dst[2] = make_uint4(out[8], out[9], out[10], out[11]);
      dst[3] = make_uint4(out[12], out[13], out[14], out[15]);
    }
  }
}

}  // namespace

void launch_merge_count(const TileMat& A, const TileMat& B, uint32_t* row_np, uint32_t* row_ns,
                        uint32_t* row_raw, cudaStream_t st) {
  const unsigned blocks = (A.tile_rows + 7) / 8;
  if (blocks == 0) return;
  merge_kernel<false><<<blocks, 256, 0, st>>>(A, B, row_np, row_ns, row_raw, nullptr, TaskList{});
}

void launch_merge_fill(const TileMat& A, const TileMat& B, const uint32_t* row_pair_off,
                       TaskList& tl, cudaStream_t st) {
  const unsigned blocks = (A.tile_rows + 7) / 8;
  if (blocks == 0) return;
  merge_kernel<true><<<blocks, 256, 0, st>>>(A, B, nullptr, nullptr, nullptr, row_pair_off, tl);
}

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
  seg_kernel<false><<<blocks, 256, 0, st>>>(A.tile_rows, row_pair_off, keys, row_nseg, TaskList{});
}

void launch_seg_fill(const TileMat& A, const uint32_t* row_pair_off, const uint32_t* keys,
                     TaskList& tl, cudaStream_t st) {
  const unsigned blocks = (A.tile_rows + 7) / 8;
  if (blocks == 0) return;
  seg_kernel<true><<<blocks, 256, 0, st>>>(A.tile_rows, row_pair_off, keys, nullptr, tl);
}

void launch_pair_meta(const TileMat& A, const TileMat& B, TaskList& tl, cudaStream_t st) {
  const uint64_t blocks = (tl.npairs + 255) / 256;
  if (blocks == 0) return;
  pair_meta_kernel<<<unsigned(blocks), 256, 0, st>>>(A, B, tl);
}

void launch_counting(const TileMat& A, const TileMat& B, const TaskList& tl, OutPlan& op,
                     cudaStream_t st) {
  const uint64_t blocks = (tl.nseg + 7) / 8;
  if (blocks == 0) return;
  const int v = tuning_variant("TSG_COUNT_BATCH", 4);
  auto k = v == 4 ? counting_kernel<4> : v == 16 ? counting_kernel<16> : counting_kernel<8>;
  k<<<unsigned(blocks), 256, 0, st>>>(A, B, tl, op);
}

void launch_row_counts(int64_t rows, uint32_t tile_rows, const TaskList& tl, OutPlan& op,
                       cudaStream_t st) {
  const unsigned blocks = (tile_rows + 7) / 8;
  if (blocks == 0) return;
  row_count_kernel<<<blocks, 256, 0, st>>>(rows, tile_rows, tl.seg_row_ptr, op.cnt, op.rowcnt);
}

void launch_positions(int64_t rows, uint32_t tile_rows, const TaskList& tl, OutPlan& op,
                      cudaStream_t st) {
  const unsigned blocks = (tile_rows + 7) / 8;
  if (blocks == 0) return;
  position_kernel<<<blocks, 256, 0, st>>>(rows, tile_rows, tl.seg_row_ptr, op.cnt, op.row_ptr,
                                          op.pos);
}

}  // namespace tsg
