// tsg_panel.cu -- the light-row pipeline: task list, counting, SEaC numeric
// and compaction of one tile row (a 16-row panel of A) fused in one warp.
//
// Applies when every tile row of A has at most 32 tiles (FEM27, Poisson,
// the R.A stage of AMG).  Restates, per tile row I:
//   enumerate_pairs / filter_zero_products   pipeline.cpp:37-70
//   sort_and_segment                          pipeline.cpp:72-109
//   counting_pass                             kernels.cpp:79-103
//   multiply_pass / finalize_segment          kernels.cpp:105-203
//   compact                                   kernels.cpp:205-220
// Lane l owns A tile (I, k_l) and walks B tile row k_l (sorted by J).  Each
// step takes the minimum pending output column J (REDUX): the lanes holding
// it are exactly output tile (I, J)'s pairs, already in ascending k (lane
// order) -- the sort happens in registers, the segment is the step.  The
// warp multiplies the step's pairs right there (mma.sync, fp32 accumulators
// in registers; or sequential CUDA-core fp32 in ORDERED mode), counts its
// structural nonzeros (0/1-indicator MMA, see tsg_numeric.cu) and appends
// the realised entries of each of its 16 rows to that CSR row's staging
// region.  Because the warp visits the row's output tiles in column order,
// every staging row fills in final CSR order; no task list, segment table or
// position pass ever reaches HBM.
//
//   elem_bound_kernel     staging bound per CSR row from the CSR alone:
//                         sum over the row's entries k of nnz(B row k)
//                         (device output; the pass below counts the stats)
//   panel_count_kernel    or: raw / filtered pairs, segments (stats) and a
//                         tight staging bound per CSR row (host output, whose
//                         pinned buffers the bound sizes; chained stages)
//   CUB scan              -> staging row offsets                (tsg_api.cu)
//   panel_numeric_kernel  the fused pass above; realised count per row
//   CUB scan              -> row_ptr                            (tsg_api.cu)
//   panel_copy_kernel     staging rows -> CSR (contiguous copies), the
//                         non-finite check of finalize_segment
#include <algorithm>
#include <mutex>

#include "tsg_kernels.cuh"
#include "tsg_mma.cuh"

namespace tsg {

namespace {

constexpr uint32_t kInf = 0xffffffffu;

// Warp state of the 32-way merge over tile row I (NL lists per lane when a tile row holds
// more than 32 A tiles).
// The same merge with NL lists per lane: lane l owns A tiles l, l + 32, ...
// (tile rows of up to 32 NL tiles).  A run's pairs in ascending k are list 0
// lanes 0..31, then list 1, ... (tiles of a tile row are sorted by k).
template <int NL>
struct MergeN {
  uint32_t occ[NL], cur[NL], end[NL];
  uint2 bt[NL], bn[NL];
  __device__ __forceinline__ void start(const TileMat& A, const TileMat& B, uint32_t I, int lane, uint32_t& a0,
                                        uint32_t& na) {
    a0 = A.trp[I];
    na = A.trp[I + 1] - a0;  // <= 32 NL on this path
#pragma unroll
    for (int q = 0; q < NL; ++q) {
      occ[q] = 0;
      cur[q] = 0;
      end[q] = 0;
      const uint32_t t = uint32_t(lane) + 32u * q;
      if (t < na) {
        const uint2 ac = __ldg(A.tco + a0 + t);
        occ[q] = ac.y;
        cur[q] = __ldg(B.trp + ac.x);
        end[q] = __ldg(B.trp + ac.x + 1);
      }
      bt[q] = cur[q] < end[q] ? __ldg(B.tco + cur[q]) : make_uint2(kInf, 0);
      bn[q] = cur[q] + 1 < end[q] ? __ldg(B.tco + cur[q] + 1) : make_uint2(kInf, 0);
    }
  }
  __device__ __forceinline__ uint32_t min_head() const {
    uint32_t j = bt[0].x;
#pragma unroll
    for (int q = 1; q < NL; ++q) j = min(j, bt[q].x);
    return j;
  }
  __device__ __forceinline__ void advance(const TileMat& B, int q) {
    ++cur[q];
    bt[q] = bn[q];
    bn[q] = cur[q] + 1 < end[q] ? __ldg(B.tco + cur[q] + 1) : make_uint2(kInf, 0);
  }
};

// Counts per tile row (raw pairs, filtered pairs, segments) and, per CSR
// row r of the panel, a staging bound: the sum over the row's output tiles
// that cover row r (OR of the run's A row occupancy) of the run's column
// span (OR of its B column occupancy).
template <int NL>
__global__ void __launch_bounds__(256) panel_count_kernel(TileMat A, TileMat B, int64_t rows,
                                                         uint32_t* __restrict__ row_np,
                                                         uint32_t* __restrict__ row_ns,
                                                         uint32_t* __restrict__ row_raw,
                                                         uint32_t* __restrict__ row_bound) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= A.tile_rows) return;
  MergeN<NL> m;
  uint32_t a0, na;
  m.start(A, B, I, lane, a0, na);
  uint32_t raw_len = 0;  // raw pairs of this lane's A tiles (pipeline.cpp:52-58)
#pragma unroll
  for (int q = 0; q < NL; ++q) raw_len += m.end[q] - m.cur[q];
  uint32_t np = 0, ns = 0, bound = 0;
  while (true) {
    const uint32_t J = __reduce_min_sync(kFull, m.min_head());
    if (J == kInf) break;
    uint32_t ro = 0, co = 0, npass = 0;
#pragma unroll
    for (int q = 0; q < NL; ++q) {
      const bool take = m.bt[q].x == J;
      const bool pass = take && (m.occ[q] & (m.bt[q].y >> 16) & 0xffffu) != 0u;
      npass += __popc(__ballot_sync(kFull, pass));
      ro |= pass ? (m.occ[q] >> 16) : 0u;
      co |= pass ? (m.bt[q].y & 0xffffu) : 0u;
      if (take) m.advance(B, q);
    }
    if (npass) {
      ro = __reduce_or_sync(kFull, ro);
      co = __reduce_or_sync(kFull, co);
      bound += ((ro >> (lane & 15)) & 1u) * __popc(co);  // lane r: row r
      np += npass;
      ++ns;
    }
  }
  const uint32_t rw = __reduce_add_sync(kFull, raw_len);
  if (lane == 0) {
    row_np[I] = np;
    row_ns[I] = ns;
    row_raw[I] = rw;
  }
  const int64_t row = int64_t(I) * 16 + lane;
  if (lane < 16 && row < rows) row_bound[row] = bound;
}

// Element-level staging bound: row r of C has at most sum over A's entries
// (r, k) of nnz(B row k) entries (and at most B.cols).  Thread per row (the
// light path bounds a row at 32 tiles = 512 entries; the row's entries are
// consecutive, so the warp's loads stay in L1).  Invalid columns contribute
// nothing (the conversion flags them).
__global__ void __launch_bounds__(256) elem_bound_kernel(CsrView A, const int64_t* __restrict__ rpB,
                                                        int64_t bcols, uint32_t* __restrict__ row_bound,
                                                        unsigned long long* __restrict__ total,
                                                        const unsigned* __restrict__ gate) {
  __shared__ unsigned long long s_sum[8];
  // gate[1]: the conversion's largest A tile row; beyond 128 tiles the call
  // is general and the speculative light pass stands down (the bound is unused)
  if (gate[1] > 128u) return;
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  uint64_t b = 0;
  if (r < A.rows && (*gate & kErrRowPtr)) {
    row_bound[r] = 0;
  } else if (r < A.rows) {
    const int64_t e0 = __ldg(A.row_ptr + r), e1 = __ldg(A.row_ptr + r + 1);
    uint64_t sum = 0;
#pragma unroll 4
    for (int64_t p = e0; p < e1; ++p) {
      const int32_t c = __ldg(A.col + p);
      if (c >= 0 && c < A.cols) sum += uint64_t(__ldg(rpB + c + 1) - __ldg(rpB + c));
    }
    b = sum < uint64_t(bcols) ? sum : uint64_t(bcols);
    row_bound[r] = uint32_t(b);
  }
  // the exact u64 total (guards the u32 staging offsets)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(kFull, b, o);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < 8; ++i) t += s_sum[i];
    if (t) atomicAdd(total, t);
  }
}

// Upper bound of the output tiles of each tile row (chained stages, emit
// mode): min(B tile columns, raw pairs of the row).  Warp per tile row.
__global__ void __launch_bounds__(256) row_tile_bound_kernel(TileMat A, TileMat B, uint32_t* __restrict__ bound) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= A.tile_rows) return;
  const uint32_t a0 = A.trp[I], na = A.trp[I + 1] - a0;
  uint32_t raw = 0;
  for (uint32_t l = lane; l < na; l += 32) {
    const uint32_t k = __ldg(&A.tco[a0 + l].x);
    raw += __ldg(B.trp + k + 1) - __ldg(B.trp + k);
  }
  raw = __reduce_add_sync(kFull, raw);
  if (lane == 0) bound[I] = raw < B.tile_cols ? raw : B.tile_cols;
}

constexpr int kSA = 17;    // padded row stride of the ordered A scratch tile
constexpr int kSRow = 24;  // row stride of the ordered B scratch tile

// Chained products (R.A.P): instead of CSR, the run's output tile is
// emitted as an A-operand tile of the next stage.  The accumulator fragment
// of mma.m16n8k16 (two n8 halves) has exactly the A-operand register layout
// (reg0 = row g cols 2t..2t+1, reg1 = row g+8, reg2/3 = cols +8), so the tile
// is four cvt.rn.f16x2 per lane -- the binary16 downcast between stages
// (kernels.cpp:239-258: RNE, |x| > 65504 overflows, values rounding to zero
// drop) -- and the lane-dense chunk write.  Tiles of a tile row go to slots
// from em.tile_base[I] in column order; the host compacts them afterwards.
__device__ __forceinline__ void emit_tile(const float (&acc)[2][4], uint32_t J, uint32_t I, int lane,
                                          const LaneLayout& L, unsigned lt, const TileEmit& em,
                                          uint32_t& e_tiles, uint32_t& e_chunks) {
  uint32_t hv[4];
  bool over = false, bad = false;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float v0 = acc[h][2 * q], v1 = acc[h][2 * q + 1];
      bad |= !isfinite(v0) || !isfinite(v1);
      over |= fabsf(v0) > 65504.0f || fabsf(v1) > 65504.0f;
      const __half2 hh = __floats2half2_rn(v0, v1);
      hv[q + 2 * h] = *reinterpret_cast<const uint32_t*>(&hh);
    }
  // a non-finite accumulator is the multiplication pass's error (raised
  // before the next stage's conversion would see the overflow)
  const bool any_bad = __any_sync(kFull, bad), any_over = __any_sync(kFull, over);
  if ((any_bad || any_over) && lane == 0)
    atomicOr(em.err_flag, any_bad ? unsigned(kErrPrecision) : unsigned(kErrOverflow));
  // nonzero binary16 slots -> per-lane bits, then the group's two row masks
  uint32_t x = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t w = hv[q + 2 * h];
      if (w & 0x7fffu) x |= 1u << (8 * h + 16 * q);
      if (w & 0x7fff0000u) x |= 1u << (8 * h + 16 * q + 1);
    }
  const bool present = x != 0u;
  x <<= 2 * L.t;
  x |= __shfl_xor_sync(kFull, x, 1);
  x |= __shfl_xor_sync(kFull, x, 2);  // rows g | g+8 << 16
  const unsigned lm = __ballot_sync(kFull, present);
  if (lm == 0u) return;  // every slot cancelled or underflowed: no tile
  const uint32_t t = em.tile_base[I] + e_tiles;
  const uint32_t cb = 1u + 32u * em.tile_base[I] + e_chunks;
  if (present) em.chunk[cb + __popc(lm & lt)] = make_uint4(hv[0], hv[1], hv[2], hv[3]);
  if (L.t == 0) em.rm2[size_t(t) * 8 + L.g] = x;
  const uint32_t colocc = __reduce_or_sync(kFull, (x | (x >> 16)) & 0xffffu);
  const uint32_t rowocc =
      __reduce_or_sync(kFull, (((x & 0xffffu) != 0u) << L.g) | (((x >> 16) != 0u) << (L.g + 8)));
  if (lane == 0) {
    const uint32_t occ = colocc | (rowocc << 16);
    em.tco[t] = make_uint2(J, occ);
    em.meta[t] = make_uint2(lm, cb);
    em.rec[t] = make_uint4(lm, cb, occ, J);
  }
  ++e_tiles;
  e_chunks += __popc(lm);
}

template <bool kOrdered, int kMinBlocks, bool kEmit, int NL>
__global__ void __launch_bounds__(256, kMinBlocks) panel_numeric_kernel(TileMat A, TileMat B, int64_t rows,
                                                              const uint32_t* __restrict__ row_stage,
                                                              uint64_t stage_cap, uint2* __restrict__ stage,
                                                              int64_t* __restrict__ rowcnt,
                                                              unsigned long long* __restrict__ counted,
                                                              const unsigned long long* __restrict__ need,
                                                              unsigned long long* __restrict__ stats,
                                                              uint32_t I0, uint32_t I1, TileEmit em,
                                                              const unsigned* __restrict__ gate,
                                                              unsigned* __restrict__ work) {
  // the run's pairs: {A lane mask, A chunk base, B lane mask, B chunk base}
  // (one list, TENSOR: {A tile of the row, -, B meta} with the A chunk index
  // of every lane precomputed per tile row in s_aidx)
  constexpr bool kTable = !kOrdered && NL == 1;
  __shared__ __align__(16) uint4 s_meta[8][32 * NL];
  __shared__ uint32_t s_aidx[kTable ? 8 : 1][32][32];
  __shared__ float sA[kOrdered ? 8 : 1][16 * kSA];
  __shared__ float sB[kOrdered ? 8 : 1][16 * kSRow];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  if (!kEmit && (*need > stage_cap || (*need >> 32))) return;  // arena too small: the host reruns the pass
  // speculative launch: {error flags, max A tiles per tile row} of the
  // conversion; invalid input or rows that are not light -> nothing to do
  if (gate && ((gate[0] & (kErrInvariant | kErrRowPtr)) || gate[1] > 32u * NL)) return;
  const uint4* cA = A.chunk[kRoleA];
  const uint4* cB = B.chunk[kRoleB];
  const unsigned lt = lanemask_lt(), bit = 1u << lane;
  const LaneLayout L(lane);
  uint32_t nstruct = 0, np = 0, ns = 0, rw = 0;
  // persistent warps (`work` != null) take tile rows from a counter, so the
  // last wave does not leave SMs idle; otherwise warp w of block b owns one
  for (uint32_t it = 0;; ++it) {
  uint32_t I;
  if (work) {
    I = 0;
    if (lane == 0) I = I0 + atomicAdd(work, 1u);
    I = __shfl_sync(kFull, I, 0);
  } else {
    I = it == 0 ? I0 + blockIdx.x * 8 + w : I1;
  }
  if (I >= I1) break;
  __syncwarp();  // the previous row's shared scratch is no longer read
  MergeN<NL> m;
  uint32_t a0, na;
  m.start(A, B, I, lane, a0, na);
  {
    uint32_t raw_len = 0;  // raw pairs of this tile row
#pragma unroll
    for (int q = 0; q < NL; ++q) raw_len += m.end[q] - m.cur[q];
    rw += __reduce_add_sync(kFull, raw_len);
  }
  uint2 am[NL];
#pragma unroll
  for (int q = 0; q < NL; ++q)
    am[q] = uint32_t(lane) + 32u * q < na ? __ldg(A.meta[kRoleA] + a0 + lane + 32 * q) : make_uint2(0, 0);
  if (kTable) {
    // this lane's chunk index in each of the row's A tiles (they are reused
    // by every output tile of the row)
    for (uint32_t l = 0; l < na; ++l) {
      const uint32_t lm = __shfl_sync(kFull, am[0].x, l), base = __shfl_sync(kFull, am[0].y, l);
      s_aidx[w][l][lane] = (lm & bit) ? base + __popc(lm & lt) : 0u;
    }
  }
  // lanes of group g track the staging cursors of rows g and g+8
  const int64_t rg = int64_t(I) * 16 + L.g, rg8 = rg + 8;
  uint32_t wg = !kEmit && rg < rows ? __ldg(row_stage + rg) : 0u;
  uint32_t wg8 = !kEmit && rg8 < rows ? __ldg(row_stage + rg8) : 0u;
  const uint32_t wg0 = wg, wg80 = wg8;
  uint32_t e_tiles = 0, e_chunks = 0;  // emit mode: tiles / chunks written for this tile row
  while (true) {
    const uint32_t J = __reduce_min_sync(kFull, m.min_head());
    if (J == kInf) break;
    // the run's pairs, in ascending k (list, then lane) order
    uint32_t n = 0;
    bool take[NL];
#pragma unroll
    for (int q = 0; q < NL; ++q) {
      take[q] = m.bt[q].x == J;
      const bool pass = take[q] && (m.occ[q] & (m.bt[q].y >> 16) & 0xffffu) != 0u;
      const unsigned pb = __ballot_sync(kFull, pass);
      if (pass) {
        const uint2 bm = __ldg(B.meta[kRoleB] + m.cur[q]);
        s_meta[w][n + __popc(pb & lt)] = kTable ? make_uint4(uint32_t(lane), 0u, bm.x, bm.y)
                                                : make_uint4(am[q].x, am[q].y, bm.x, bm.y);
      }
      n += __popc(pb);
    }
    if (n) {
      np += n;
      ++ns;
      __syncwarp();
      float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      if (!kOrdered) {
        uint32_t sac[2][2] = {{0u, 0u}, {0u, 0u}};
        for (uint32_t u = 0; u < n; u += 2) {
          const uint4 m0 = s_meta[w][u];
          const uint4 m1 = u + 1 < n ? s_meta[w][u + 1] : make_uint4(0, 0, 0, 0);
          const uint4 fa0 = kTable ? __ldg(cA + s_aidx[w][m0.x][lane]) : load_chunk(cA, m0.x, m0.y, lt, bit);
          const uint4 fb0 = load_chunk(cB, m0.z, m0.w, lt, bit);
          // an absent second pair reads the zero chunk: adds exact zeros
          const uint4 fa1 = kTable ? __ldg(cA + (u + 1 < n ? s_aidx[w][m1.x][lane] : 0u))
                                   : load_chunk(cA, m1.x, m1.y, lt, bit);
          const uint4 fb1 = load_chunk(cB, m1.z, m1.w, lt, bit);
          mma16816(acc[0], fa0, fb0.x, fb0.y);
          mma16816(acc[1], fa0, fb0.z, fb0.w);
          const uint4 xa0 = nz_h2(fa0), xb0 = nz_h2(fb0);
          mma16816_h(sac[0], xa0, xb0.x, xb0.y);
          mma16816_h(sac[1], xa0, xb0.z, xb0.w);
          mma16816(acc[0], fa1, fb1.x, fb1.y);
          mma16816(acc[1], fa1, fb1.z, fb1.w);
          const uint4 xa1 = nz_h2(fa1), xb1 = nz_h2(fb1);
          mma16816_h(sac[0], xa1, xb1.x, xb1.y);
          mma16816_h(sac[1], xa1, xb1.z, xb1.w);
        }
        nstruct += count_nz_counts(sac[0][0], sac[0][1], sac[1][0], sac[1][1]);
      } else {
        bool snz[2][4] = {{false, false, false, false}, {false, false, false, false}};
        for (uint32_t u = 0; u < n; ++u) {
          const uint4 mt = s_meta[w][u];
          // expand_tile (kernels.cpp:17-26): every lane writes all 8 of its slots
#pragma unroll
          for (int role = 0; role < 2; ++role) {
            const uint4 ch = role == kRoleA ? load_chunk(cA, mt.x, mt.y, lt, bit)
                                            : load_chunk(cB, mt.z, mt.w, lt, bit);
            const uint32_t regs[4] = {ch.x, role == kRoleA ? ch.y : ch.z, role == kRoleA ? ch.z : ch.y, ch.w};
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              int r, c;
              rc_of(role, lane, j, r, c);
              const float v = __half2float(__ushort_as_half(uint16_t(regs[j >> 1] >> (16 * (j & 1)))));
              if (role == kRoleA)
                sA[w][r * kSA + c] = v;
              else
                sB[w][r * kSRow + c] = v;
            }
          }
          __syncwarp();
          // tile_mm_reference (kernels.cpp:28-38): k ascending, no FMA; an
          // exact binary16 x binary16 product is nonzero iff both factors are
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int r = L.g + 8 * (i >> 1), c = 2 * L.t + (i & 1) + 8 * h;
              float x = acc[h][i];
              bool nz = snz[h][i];
#pragma unroll
              for (int kk = 0; kk < 16; ++kk) {
                const float pr = __fmul_rn(sA[w][r * kSA + kk], sB[w][kk * kSRow + c]);
                nz |= pr != 0.0f;
                x = __fadd_rn(x, pr);
              }
              acc[h][i] = x;
              snz[h][i] = nz;
            }
          __syncwarp();
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int i = 0; i < 4; ++i) nstruct += snz[h][i];
      }
      if (kEmit) {
        emit_tile(acc, J, I, lane, L, lt, em, e_tiles, e_chunks);
        __syncwarp();
      } else {
      // finalize_segment: bitmap = accumulators != 0 (cancelled slots and -0
      // drop: compact()); row r's entries append to row r's staging region
      const uint32_t rmg = group_row_masks(acc, L.t);  // rows g | g+8 << 16
      const int32_t cj = int32_t(J * 16u) + 2 * L.t;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t p = q ? wg8 : wg, mr = q ? (rmg >> 16) : (rmg & 0xffffu);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float v0 = acc[h][2 * q], v1 = acc[h][2 * q + 1];
          const uint32_t e0 = p + __popc(mr & L.cm[h]);
          if (v0 != 0.0f) stage[e0] = make_uint2(__float_as_uint(v0), uint32_t(cj + 8 * h));
          if (v1 != 0.0f) stage[e0 + (v0 != 0.0f)] = make_uint2(__float_as_uint(v1), uint32_t(cj + 8 * h + 1));
        }
      }
      wg += __popc(rmg & 0xffffu);
      wg8 += __popc(rmg >> 16);
      __syncwarp();  // s_meta is rewritten by the next run
      }
    }
#pragma unroll
    for (int q = 0; q < NL; ++q)
      if (take[q]) m.advance(B, q);
  }
  if (kEmit) {
    if (lane == 0) em.rtiles[I] = e_tiles;
  } else if (L.t == 0) {
    if (rg < rows) rowcnt[rg] = int64_t(wg - wg0);
    if (rg8 < rows) rowcnt[rg8] = int64_t(wg8 - wg80);
  }
  }  // tile rows
  nstruct = __reduce_add_sync(kFull, nstruct);
  if (lane == 0 && nstruct) atomicAdd(counted, (unsigned long long)nstruct);
  if (stats && lane == 0 && (np | rw)) {  // the statistics panel_count_kernel would have produced
    atomicAdd(stats, (unsigned long long)np);
    atomicAdd(stats + 1, (unsigned long long)ns);
    atomicAdd(stats + 2, (unsigned long long)rw);
  }
}

// Staging rows -> CSR: warp per panel, lanes over the panel's output
// positions (the 16 rows are consecutive in the CSR), each taken from its
// row's staging region.  Non-finite values raise kErrPrecision
// (finalize_segment, kernels.cpp:115-127).
#ifndef TSG_PANEL_KB
#define TSG_PANEL_KB 4
#endif
#ifndef TSG_COPY_U
#define TSG_COPY_U 16
#endif
constexpr int kCopyU = TSG_COPY_U;  // staged entries per lane in flight

__global__ void __launch_bounds__(256) panel_copy_kernel(int64_t rows, uint32_t tile_rows,
                                                        const uint32_t* __restrict__ row_stage,
                                                        const int64_t* __restrict__ row_ptr,
                                                        const uint2* __restrict__ stage,
                                                        int32_t* __restrict__ col,
                                                        float* __restrict__ val,
                                                        unsigned* __restrict__ err_flag, uint32_t I0) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = I0 + blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows) return;
  const int64_t r0 = int64_t(I) * 16;
  const int64_t r1 = r0 + 16 < rows ? r0 + 16 : rows;
  const int64_t base = row_ptr[r0];
  const uint32_t T = uint32_t(row_ptr[r1] - base);
  const int64_t row = r0 + (lane & 15);
  // lane r: offset of row r within the panel (rows past the end: T)
  const uint32_t off = row < r1 ? uint32_t(row_ptr[row] - base) : T;
  const uint32_t src0 = row < r1 ? row_stage[row] : 0u;
  bool bad = false;
  // kCopyU entries per lane per step: the row lookups and loads first, then the stores
  for (uint32_t q0 = 0; q0 < T; q0 += 32 * kCopyU) {
    uint2 e[kCopyU];
#pragma unroll
    for (int u = 0; u < kCopyU; ++u) {
      const uint32_t q = q0 + 32 * u + lane;
      int r = 0;  // last row whose offset is <= q (empty rows resolve to the next one)
#pragma unroll
      for (int b = 8; b > 0; b >>= 1) {
        const uint32_t v = __shfl_sync(kFull, off, r + b);
        if (v <= q) r += b;
      }
      const uint32_t o = __shfl_sync(kFull, off, r), sr = __shfl_sync(kFull, src0, r);
      e[u] = q < T ? __ldg(stage + sr + (q - o)) : make_uint2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < kCopyU; ++u) {
      const uint32_t q = q0 + 32 * u + lane;
      if (q < T) {
        const float x = __uint_as_float(e[u].x);
        bad |= !isfinite(x);
        col[base + q] = int32_t(e[u].y);
        val[base + q] = x;
      }
    }
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(err_flag, unsigned(kErrPrecision));
}

}  // namespace

void launch_panel_count(const TileMat& A, const TileMat& B, int64_t rows, uint32_t* row_np,
                        uint32_t* row_ns, uint32_t* row_raw, uint32_t* row_bound, int nl, cudaStream_t st) {
  const unsigned blocks = (A.tile_rows + 7) / 8;
  if (blocks == 0) return;
  auto k = nl <= 1 ? panel_count_kernel<1> : nl == 2 ? panel_count_kernel<2> : panel_count_kernel<4>;
  k<<<blocks, 256, 0, st>>>(A, B, rows, row_np, row_ns, row_raw, row_bound);
}

void launch_elem_bound(const CsrView& A, const int64_t* rpB, int64_t bcols, uint32_t* row_bound,
                       unsigned long long* total, const unsigned* gate, cudaStream_t st) {
  const unsigned blocks = unsigned((A.rows + 255) / 256);
  if (blocks == 0) return;
  elem_bound_kernel<<<blocks, 256, 0, st>>>(A, rpB, bcols, row_bound, total, gate);
}

namespace {
using PanelK = void (*)(TileMat, TileMat, int64_t, const uint32_t*, uint64_t, uint2*, int64_t*, unsigned long long*,
                        const unsigned long long*, unsigned long long*, uint32_t, uint32_t, TileEmit, const unsigned*,
                        unsigned*);
template <int NL>
PanelK pick_panel(int mode, bool emit) {
  constexpr int kB = NL == 1 ? TSG_PANEL_KB : 3;  // resident blocks per SM (registers of the NL merge lists)
  if (mode == 1) return emit ? panel_numeric_kernel<true, kB, true, NL> : panel_numeric_kernel<true, kB, false, NL>;
  return emit ? panel_numeric_kernel<false, kB, true, NL> : panel_numeric_kernel<false, kB, false, NL>;
}
}  // namespace

cudaError_t launch_panel_numeric(const TileMat& A, const TileMat& B, int64_t rows, const uint32_t* row_stage,
                                 uint64_t stage_cap, uint2* stage, int64_t* rowcnt, unsigned long long* counted,
                                 const unsigned long long* need, unsigned long long* stats, int mode, uint32_t I0,
                                 uint32_t I1, cudaStream_t st, const TileEmit* emit, const unsigned* gate,
                                 unsigned* work, int nl) {
  unsigned blocks = (I1 - I0 + 7) / 8;
  if (I1 <= I0) return cudaSuccess;
  const TileEmit em = emit ? *emit : TileEmit{};
  const int li = nl <= 1 ? 0 : nl == 2 ? 1 : 2;
  const PanelK k = li == 0 ? pick_panel<1>(mode, emit) : li == 1 ? pick_panel<2>(mode, emit) : pick_panel<4>(mode, emit);
  if (work) {  // persistent: one resident wave takes the tile rows from the counter
    // resident blocks of each kernel variant, per device (a process may drive several GPUs)
    static std::mutex mu;
    static int cached[16][12] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const int slot = li * 4 + (mode == 1 ? 2 : 0) + (emit ? 1 : 0);
    int waves;
    {
      std::lock_guard<std::mutex> g(mu);
      int& c = cached[dev & 15][slot];
      if (!c) {
        int per_sm = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(k), 256, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        c = std::max(1, per_sm) * std::max(1, sms);
      }
      waves = c;
    }
    if (blocks <= unsigned(waves)) {
      work = nullptr;  // one wave covers every tile row: static assignment
    } else {
      blocks = unsigned(waves);
      e = cudaMemsetAsync(work, 0, sizeof(unsigned), st);
      if (e != cudaSuccess) return e;
    }
  }
  k<<<blocks, 256, 0, st>>>(A, B, rows, row_stage, stage_cap, stage, rowcnt, counted, need, stats, I0, I1, em, gate,
                            work);
  return cudaSuccess;
}

// Emitted tiles (gapped per tile row) -> dense CSR-of-tiles: warp per tile row.
__global__ void emit_compact_kernel(uint32_t tile_rows, TileEmit em, const uint32_t* __restrict__ trp, TileMat T) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows) return;
  const uint32_t src = em.tile_base[I], dst = trp[I], n = em.rtiles[I];
  for (uint32_t i = lane; i < n; i += 32) {
    T.tco[dst + i] = em.tco[src + i];
    T.meta[kRoleA][dst + i] = em.meta[src + i];
    T.rec[kRoleA][dst + i] = em.rec[src + i];
  }
  for (uint32_t i = lane; i < 8 * n; i += 32) T.rm2[size_t(dst) * 8 + i] = em.rm2[size_t(src) * 8 + i];
}

void launch_row_tile_bound(const TileMat& A, const TileMat& B, uint32_t* bound, cudaStream_t st) {
  const unsigned blocks = (A.tile_rows + 7) / 8;
  if (blocks == 0) return;
  row_tile_bound_kernel<<<blocks, 256, 0, st>>>(A, B, bound);
}

void launch_emit_compact(uint32_t tile_rows, const TileEmit& em, const uint32_t* trp, TileMat& T, cudaStream_t st) {
  const unsigned blocks = (tile_rows + 7) / 8;
  if (blocks == 0) return;
  emit_compact_kernel<<<blocks, 256, 0, st>>>(tile_rows, em, trp, T);
}

void launch_panel_copy(int64_t rows, const uint32_t* row_stage, const int64_t* row_ptr, const uint2* stage,
                       int32_t* col, float* val, unsigned* err_flag, uint32_t I0, uint32_t I1, cudaStream_t st) {
  if (I1 <= I0) return;
  const unsigned blocks = (I1 - I0 + 7) / 8;
  panel_copy_kernel<<<blocks, 256, 0, st>>>(rows, I1, row_stage, row_ptr, stage, col, val, err_flag, I0);
}

}  // namespace tsg
