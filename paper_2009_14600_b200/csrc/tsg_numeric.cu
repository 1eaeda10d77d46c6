// tsg_numeric.cu -- subsystem (3): SEaC numeric phase (sort, expand, compress).
//
// GPU restatement of multiply_pass / finalize_segment
// (proj/src/kernels.cpp:105-203) at T = 16.  One warp per segment (= one
// output tile, TaskList order).  The warp walks the segment's pairs in
// ascending inner tile k and keeps the 16x16 fp32 output tile in registers
// for the whole run (two m16n8 accumulators, 8 floats per lane).
//
//   TENSOR mode: per pair each lane loads its A and B operand chunk (one
//     LDG.128 each, tsg_common.cuh) and the warp issues two
//     mma.sync.m16n8k16.f32.f16.f16.f32 -- the 16x16 tile product is exactly
//     one m16n16k16, so the 8x8 diagonal pairing of the reference
//     (kernels.cpp:40-77) has no waste left to remove.
//   ORDERED mode: CUDA-core fp32, one rounding per product, ascending k,
//     __fmul_rn/__fadd_rn (no FMA contraction, proj/CMakeLists.txt:12-14):
//     bit-identical to tile_mm_reference (kernels.cpp:28-38) and to
//     dense_spgemm_mixed_ordered (oracle.cpp:102-121).
//
// Compress (finalize_segment, kernels.cpp:109-127) writes straight into the
// final CSR: the counting pass already fixed every structurally nonzero
// slot's position (pos[seg, r] = row_ptr + counted entries of row r in the
// row's earlier tiles), so value (r, c) of output tile (I, J) goes to
// pos[seg, r] + rank of c in the counted row mask.  An
// accumulator that is exactly 0 there (cancellation; v != 0 is false for
// -0 too) is written as a col = -1 hole and flagged; the host then runs the
// compaction fix-up (compact(), kernels.cpp:205-220).  Non-finite
// accumulators raise kErrPrecision (PrecisionError, kernels.cpp:199-201).
#include "tsg_kernels.cuh"

namespace tsg {

namespace {

__device__ __forceinline__ void mma16816(float (&d)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// chunk index of this lane for a tile with meta {lane mask, base}; 0 = zeros
__device__ __forceinline__ uint32_t chunk_index(uint32_t lm, uint32_t base, int lane, bool ok) {
  const bool present = ok && ((lm >> lane) & 1u);
  return present ? base + __popc(lm & lanemask_lt()) : 0u;
}

// Where segment s's output goes: everything the epilogue needs that does
// not depend on the accumulators, loaded at the top of the kernel so the
// loads overlap the MMA work.
struct TileDest {
  uint32_t rowm;   // counted mask of row lane & 15
  uint32_t pos;    // CSR position of that row's first counted entry
  int32_t cbase;   // 16 * output tile column
};

__device__ __forceinline__ TileDest tile_dest(uint64_t s, const TaskList& tl, const OutPlan& op,
                                              int lane) {
  const uint32_t J = tl.seg_col[s];
  const int r = lane & 15;
  const uint32_t w = op.bm2[s * 8 + (r & 7)];  // counted rows (r&7) | +8 << 16
  TileDest d;
  d.rowm = (r >> 3) ? (w >> 16) : (w & 0xffffu);
  d.pos = op.pos[s * 16 + r];  // 64 contiguous bytes per segment (64-bit index: 16S > 2^32)
  d.cbase = int32_t(J * 16);
  return d;
}

constexpr int kSRow = 24;  // staging row stride (floats): conflict-free STS.64

// acc[h][i] holds (row g + 8*(i>>1), col 2t + (i&1) + 8h).  The tile is
// staged in shared memory (four STS.64 per lane), then lane r & 15 walks the
// counted entries of row r -- lanes 0-15 take the even entries, 16-31 the
// odd ones -- and stores them at pos + entry index.  sacc is this warp's
// 16 x 16 float scratch.
__device__ __forceinline__ void store_tile(const float (&acc)[2][4], const TileDest& d,
                                           const OutPlan& op, int lane,
                                           float* __restrict__ sacc,
                                           unsigned* __restrict__ err_flag) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int q = 0; q < 2; ++q)
      *reinterpret_cast<float2*>(sacc + (g + 8 * q) * kSRow + 2 * t + 8 * h) =
          make_float2(acc[h][2 * q], acc[h][2 * q + 1]);
  __syncwarp();
  const int r = lane & 15, par = lane >> 4;
  bool bad = false, cancelled = false;
  uint32_t m = par ? (d.rowm & (d.rowm - 1)) : d.rowm;  // odd lanes start at entry 1
  uint32_t e = par;
  while (m) {
    const int c = __ffs(m) - 1;
    const float v = sacc[r * kSRow + c];
    bad |= !isfinite(v);
    const bool zero = v == 0.0f;
    cancelled |= zero;
    op.col[d.pos + e] = zero ? -1 : d.cbase + c;
    op.val[d.pos + e] = v;
    m &= m - 1;  // skip this entry ...
    m &= m - 1;  // ... and the other parity's next one
    e += 2;
  }
  const unsigned flags = (__any_sync(kFull, bad) ? unsigned(kErrPrecision) : 0u) |
                         (__any_sync(kFull, cancelled) ? unsigned(kCancelled) : 0u);
  if (flags && lane == 0) atomicOr(err_flag, flags);
}

// One warp per segment.  The serial load chain is kept to three steps:
// (1) segment bounds, (2) one coalesced LDG.128 per lane of the operand
// metas of up to 32 pairs (TaskList.pmeta) together with the epilogue's
// index loads, (3) the operand chunks of kBatch pairs at a time (metas
// broadcast by shuffle; absent lanes and pairs past the end read the zero
// chunk), then the MMAs.  Accumulation order is ascending k.
// Absent lanes skip the load (no L1 sector) and use zeros.
__device__ __forceinline__ uint4 load_chunk(const uint4* __restrict__ base, uint32_t lm,
                                            uint32_t first, unsigned lt, unsigned bit) {
  uint4 v = make_uint4(0, 0, 0, 0);
  if (lm & bit) v = __ldg(base + first + __popc(lm & lt));
  return v;
}

template <int kBatch>
__global__ void __launch_bounds__(256) numeric_tc_kernel(TileMat A, TileMat B, TaskList tl,
                                                        OutPlan op,
                                                        unsigned* __restrict__ err_flag) {
  __shared__ __align__(16) float s_acc[8][16 * kSRow];
  const int lane = threadIdx.x & 31;
  const uint64_t s = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (s >= tl.nseg) return;
  const uint32_t p0 = tl.seg_off[s], p1 = tl.seg_off[s + 1];
  const TileDest dest = tile_dest(s, tl, op, lane);
  float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  const uint4* cA = A.chunk[kRoleA];
  const uint4* cB = B.chunk[kRoleB];
  const unsigned lt = lanemask_lt(), bit = 1u << lane;
  for (uint32_t pb = p0; pb < p1; pb += 32) {
    const uint32_t n = min(32u, p1 - pb);
    const uint4 ml = lane < n ? __ldg(tl.pmeta + pb + lane) : make_uint4(0, 0, 0, 0);
    for (uint32_t u0 = 0; u0 < n; u0 += kBatch) {
      uint4 fa[kBatch], fb[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int q = int(u0) + u;  // lanes >= n hold zero metas
        const uint32_t lma = __shfl_sync(kFull, ml.x, q), bsa = __shfl_sync(kFull, ml.y, q);
        const uint32_t lmb = __shfl_sync(kFull, ml.z, q), bsb = __shfl_sync(kFull, ml.w, q);
        fa[u] = load_chunk(cA, lma, bsa, lt, bit);
        fb[u] = load_chunk(cB, lmb, bsb, lt, bit);
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        if (u0 + u < n) {
          // B chunk: {x, y} = {b0, b1} of the n0..7 MMA, {z, w} of the n8..15 MMA
          mma16816(acc[0], fa[u], fb[u].x, fb[u].y);
          mma16816(acc[1], fa[u], fb[u].z, fb[u].w);
        }
      }
    }
  }
  store_tile(acc, dest, op, lane, s_acc[threadIdx.x >> 5], err_flag);
}

constexpr int kSA = 17;  // padded row stride of the A scratch tile

__global__ void __launch_bounds__(256) numeric_ordered_kernel(TileMat A, TileMat B, TaskList tl,
                                                             OutPlan op,
                                                             unsigned* __restrict__ err_flag) {
  __shared__ float sA[8][16 * kSA];
  __shared__ __align__(16) float sB[8][16 * kSRow];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const uint64_t s = uint64_t(blockIdx.x) * 8 + w;
  if (s >= tl.nseg) return;
  const uint32_t p0 = tl.seg_off[s], p1 = tl.seg_off[s + 1];
  const int g = lane >> 2, t = lane & 3;
  float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  const unsigned long long* pairs = reinterpret_cast<const unsigned long long*>(tl.pairs);
  for (uint32_t p = p0; p < p1; ++p) {
    const uint64_t pr = __ldg(pairs + p);
    // expand_tile (kernels.cpp:17-26): every lane writes all 8 of its slots
    // (absent lanes read the zero chunk), so no separate clearing is needed
#pragma unroll
    for (int role = 0; role < 2; ++role) {
      const TileMat& M = role == kRoleA ? A : B;
      const uint32_t tt = role == kRoleA ? uint32_t(pr) : uint32_t(pr >> 32);
      const uint2 m = __ldg(M.meta[role] + tt);
      const uint4 ch = __ldg(M.chunk[role] + chunk_index(m.x, m.y, lane, true));
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
    // tile_mm_reference: acc += a[r][k] * b[k][c], k ascending, no FMA
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = g + 8 * (i >> 1), c = 2 * t + (i & 1) + 8 * h;
        float x = acc[h][i];
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          x = __fadd_rn(x, __fmul_rn(sA[w][r * kSA + kk], sB[w][kk * kSRow + c]));
        acc[h][i] = x;
      }
    __syncwarp();
  }
  store_tile(acc, tile_dest(s, tl, op, lane), op, lane, sB[w], err_flag);  // sB is free again
}

}  // namespace

void launch_numeric(const TileMat& A, const TileMat& B, const TaskList& tl, OutPlan& op, int mode,
                    unsigned* err_flag, cudaStream_t st) {
  const uint64_t blocks = (tl.nseg + 7) / 8;
  if (blocks == 0) return;
  if (mode == 1) {
    numeric_ordered_kernel<<<unsigned(blocks), 256, 0, st>>>(A, B, tl, op, err_flag);
  } else {
    const int v = tuning_variant("TSG_NUMERIC_BATCH", 2);
    auto k = v == 2 ? numeric_tc_kernel<2> : v == 8 ? numeric_tc_kernel<8> : numeric_tc_kernel<4>;
    k<<<unsigned(blocks), 256, 0, st>>>(A, B, tl, op, err_flag);
  }
}

}  // namespace tsg
