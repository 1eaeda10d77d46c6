// tsg_symbolic.cu -- subsystem (2): tile-pair task list and boolean sizing.
//
// GPU restatement at T = 16 of
//   enumerate_pairs       proj/src/pipeline.cpp:37-60
//   filter_zero_products  proj/src/pipeline.cpp:62-70  (tile_product_nonzero :23-35)
//   sort_and_segment      proj/src/pipeline.cpp:72-109
//
// The counting pass (kernels.cpp:79-103) is fused into the numeric kernel
// (tsg_numeric.cu); this file also produces each segment's staging bound
// popc(OR of A row occupancy) * popc(OR of B column occupancy) -- every
// realised output slot of the segment lies in that rectangle.
//
// This is the general path (some tile row of A has more than 32 tiles --
// R-MAT, the rectangular product, the second AMG stage); light rows never
// materialise a task list (tsg_panel.cu).  Fused enumerate+filter (count,
// scan, fill; raw pairs are never materialised), a stable
// segmented radix sort by output tile column per tile row (tsg_api.cu),
// then segment heads.  One warp per 32 consecutive A tiles flattens their
// raw pairs and load-balances them across lanes with a shuffle binary
// search, so skewed B tile rows (R-MAT) keep all lanes busy.
//
#include "tsg_kernels.cuh"

namespace tsg {

namespace {

constexpr uint32_t kInf = 0xffffffffu;

// ------------------------------------------------------------- general rows
template <bool kFill>
__global__ void __launch_bounds__(256) enum_kernel(TileMat A, TileMat B, uint64_t tA,
                                                  uint32_t* __restrict__ tile_cnt,
                                                  const uint32_t* __restrict__ tile_off,
                                                  uint64_t* __restrict__ pairs,
                                                  uint32_t* __restrict__ keys,
                                                  unsigned long long* __restrict__ raw_total,
                                                  uint32_t key_shift) {
  __shared__ uint32_t s_cnt[8][33];
  __shared__ unsigned long long s_raw[8];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t a0 = (uint64_t(blockIdx.x) * 8 + wib) * 32;
  unsigned long long raw = 0;
  if (a0 < tA) {
    const uint64_t a = a0 + lane;
    const bool valid = a < tA;
    // Each A tile's candidate list: a single-column tile (one inner slot kk,
    // ~1 nnz per tile on R-MAT / rect) takes B's CSR row 16k+kk -- its first
    // kept entry per tile names exactly the B tiles that pass the
    // zero-product filter; others take B's tile row k with the occupancy
    // filter (pipeline.cpp:23-35).  Raw pairs are B tile row lengths either way.
    uint32_t bs = 0, bl = 0, colocc = 0, base_off = 0, raw_len = 0, ts = 0;
    bool single = false;
    if (valid) {
      const uint2 ac = __ldg(A.tco + a);
      ts = __ldg(B.trp + ac.x);
      const uint32_t te = __ldg(B.trp + ac.x + 1);
      raw_len = te - ts;
      colocc = ac.y & 0xffffu;
      single = B.etile != nullptr && __popc(colocc) == 1;
      if (single) {
        const int64_t row = int64_t(ac.x) * 16 + (__ffs(colocc) - 1);
        const int64_t e0 = row < B.rows ? __ldg(B.csr_rp + row) : 0, e1 = row < B.rows ? __ldg(B.csr_rp + row + 1) : 0;
        bs = uint32_t(e0);
        bl = uint32_t(e1 - e0);
      } else {
        bs = ts;
        bl = raw_len;
      }
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
    raw = __reduce_add_sync(kFull, raw_len);
    const unsigned single_mask = __ballot_sync(kFull, single);
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
      const uint32_t ts_s = __shfl_sync(kFull, ts, s & 31);
      const bool single_s = (single_mask >> (s & 31)) & 1u;
      uint32_t b = bs_s + (q - ex_s);
      bool pass = false;
      uint32_t J = 0;
      if (active) {
        if (single_s) {
          const uint32_t t = __ldg(B.etile + b);  // b is an entry index here
          pass = (t & kDupEntry) == 0u;            // kNoTile has the bit set too
          b = ts_s + (t & ~kDupEntry);             // the tile's rank within B's tile row
          if (kFill && pass) J = __ldg(&B.tco[b].x);
        } else {
          const uint2 bt = __ldg(B.tco + b);
          pass = (co_s & (bt.y >> 16)) != 0;
          J = bt.x;
        }
      }
      const unsigned grp = __match_any_sync(kFull, s);
      const unsigned pbal = __ballot_sync(kFull, pass);
      const uint32_t before = s_cnt[wib][s];
      if (kFill && pass) {
        const uint32_t pos = off_s + before + __popc(pbal & grp & lanemask_lt());
        pairs[pos] = (a0 + uint64_t(s)) | (uint64_t(b) << 32);
        // (tile row << shift) | tile col; shift 32 drops the row (segmented sort)
        keys[pos] = (key_shift < 32 ? (__ldg(A.trow + a0 + s) << key_shift) : 0u) | J;
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
__global__ void __launch_bounds__(256) seg_kernel(uint32_t jmask, uint32_t tile_rows,
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
      tl.seg_col[s] = key & jmask;
    }
    nseg += __popc(hb);
    carry = __shfl_sync(kFull, key, 31);
  }
  if (!kFill && lane == 0) row_nseg[I] = nseg;
}

// operand metas per sorted pair (general path) and its staging bound
__global__ void pair_meta_kernel(TileMat A, TileMat B, const uint64_t* __restrict__ pairs, TaskList tl,
                                 uint32_t* __restrict__ pair_bound) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i > tl.npairs) return;
  if (i == tl.npairs) {  // pad entry: zero metas (chunk 0), no staging
    tl.pmeta[i] = make_uint4(0, 0, 0, 0);
    tl.pocc[i] = make_uint2(0, 0);
    pair_bound[i] = 0;
    return;
  }
  const uint64_t pr = pairs[i];
  const uint32_t a = uint32_t(pr), b = uint32_t(pr >> 32);
  const uint4 ra = __ldg(A.rec[kRoleA] + a), rb = __ldg(B.rec[kRoleB] + b);  // one sector each
  const uint32_t oa = ra.z, ob = rb.z;
  tl.pmeta[i] = make_uint4(ra.x, ra.y, rb.x, rb.y);
  tl.pocc[i] = make_uint2(oa, ob);  // so the thin kernel reads each pair coalesced
  pair_bound[i] = __popc(oa >> 16) * __popc(ob & 0xffffu);
}

// segment s's staging region starts at the bound prefix of its first pair
__global__ void seg_stage_kernel(TaskList tl, const uint32_t* __restrict__ pair_stage) {
  const uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (s <= tl.nseg) tl.stage_off[s] = pair_stage[tl.seg_off[s]];
}

}  // namespace

void launch_enum_count(const TileMat& A, const TileMat& B, uint64_t tA, uint32_t* tile_cnt,
                       unsigned long long* raw_total, cudaStream_t st) {
  const uint64_t warps = (tA + 31) / 32;
  const uint64_t blocks = (warps + 7) / 8;
  if (blocks == 0) return;
  enum_kernel<false><<<unsigned(blocks), 256, 0, st>>>(A, B, tA, tile_cnt, nullptr, nullptr,
                                                        nullptr, raw_total, 32);
}

void launch_enum_fill(const TileMat& A, const TileMat& B, uint64_t tA, const uint32_t* tile_off,
                      uint64_t* pairs, uint32_t* keys, uint32_t key_shift, cudaStream_t st) {
  const uint64_t warps = (tA + 31) / 32;
  const uint64_t blocks = (warps + 7) / 8;
  if (blocks == 0) return;
  enum_kernel<true><<<unsigned(blocks), 256, 0, st>>>(A, B, tA, nullptr, tile_off, pairs, keys,
                                                       nullptr, key_shift);
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
  seg_kernel<false><<<blocks, 256, 0, st>>>(0xffffffffu, A.tile_rows, row_pair_off, keys, row_nseg, TaskList{});
}

void launch_seg_fill(const TileMat& A, const uint32_t* row_pair_off, const uint32_t* keys, uint32_t jmask,
                     TaskList& tl, cudaStream_t st) {
  const unsigned blocks = (A.tile_rows + 7) / 8;
  if (blocks == 0) return;
  seg_kernel<true><<<blocks, 256, 0, st>>>(jmask, A.tile_rows, row_pair_off, keys, nullptr, tl);
}

void launch_pair_meta(const TileMat& A, const TileMat& B, const uint64_t* pairs, TaskList& tl,
                      uint32_t* pair_bound, cudaStream_t st) {
  const uint64_t blocks = (tl.npairs + 1 + 255) / 256;
  pair_meta_kernel<<<unsigned(blocks), 256, 0, st>>>(A, B, pairs, tl, pair_bound);
}

void launch_seg_stage(const TaskList& tl, const uint32_t* pair_stage, cudaStream_t st) {
  const uint64_t blocks = (tl.nseg + 1 + 255) / 256;
  seg_stage_kernel<<<unsigned(blocks), 256, 0, st>>>(tl, pair_stage);
}

}  // namespace tsg
