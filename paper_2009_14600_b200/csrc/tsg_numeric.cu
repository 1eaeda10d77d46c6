// tsg_numeric.cu -- subsystem (3): SEaC numeric phase (sort, expand, compress).
//
// GPU restatement of multiply_pass / finalize_segment
// (proj/src/kernels.cpp:105-203) at T = 16.  One warp per segment (= one
// output tile, TaskList order).  The warp walks the segment's pairs in
// ascending inner tile k and keeps the 16x16 fp32 output tile in registers
// for the whole run (two m16n8 accumulators, 8 floats per lane).
//
//   TENSOR mode: per pair, the A and B operand fragments are built straight
//     from the packed fragment-order values (tsg_common.cuh) and multiplied
//     with two mma.sync.m16n8k16 f32.f16.f16.f32 -- the 16x16 tile product
//     is exactly one m16n16k16, so the 8x8 diagonal pairing of the
//     reference (kernels.cpp:40-77) has no waste to remove.
//   ORDERED mode: CUDA-core fp32, one rounding per product, ascending k,
//     __fmul_rn/__fadd_rn (no FMA contraction, proj/CMakeLists.txt:12-14):
//     bit-identical to tile_mm_reference (kernels.cpp:28-38) and to
//     dense_spgemm_mixed_ordered (oracle.cpp:102-121).
//
// Compress (finalize_segment, kernels.cpp:109-127): ballot the nonzero
// accumulators (v != 0, so -0 drops), rebuild the 16 row masks, and store
// the realised values in row-major bit order into the segment's counted
// slot range; non-finite accumulators raise kErrPrecision (-> PrecisionError,
// kernels.cpp:199-201).  Empty tiles are simply all-zero masks; compaction
// is fused into the tiled -> CSR output (tsg_output.cu).
#include "tsg_kernels.cuh"

namespace tsg {

namespace {

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ unsigned spread4(unsigned n) {  // bit t -> bit 2t
  return (n & 1u) | ((n & 2u) << 1) | ((n & 4u) << 2) | ((n & 8u) << 3);
}

// acc[h][i] holds (row g + 8*(i>>1), col 2t + (i&1) + 8h).
__device__ __forceinline__ void compress_store(const float (&acc)[2][4], uint64_t s,
                                               const OutTiles& ot, int lane,
                                               unsigned* __restrict__ err_flag) {
  unsigned B[2][4];
  bool bad = false;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      B[h][i] = __ballot_sync(kFull, acc[h][i] != 0.0f);
      bad |= !isfinite(acc[h][i]);
    }
  if (__any_sync(kFull, bad)) {
    if (lane == 0) atomicOr(err_flag, kErrPrecision);
  }
  const int g = lane >> 2, t = lane & 3;
  const unsigned low = (1u << (4 * g)) - 1u;
  const unsigned lt = (1u << t) - 1u, le = (1u << (t + 1)) - 1u;
  float* dst = ot.vals + ot.elem_off[s];
  unsigned pre = 0;
  unsigned tot_upper = 0;
#pragma unroll
  for (int half = 0; half < 2; ++half) {  // half 0: row g, half 1: row g+8
    const int i0 = 2 * half;              // acc index of col 2t (i0) / 2t+1 (i0+1)
    if (half == 1) pre = tot_upper;
    pre += __popc(B[0][i0] & low) + __popc(B[0][i0 + 1] & low) + __popc(B[1][i0] & low) +
           __popc(B[1][i0 + 1] & low);
    if (half == 0)
      tot_upper = __popc(B[0][0]) + __popc(B[0][1]) + __popc(B[1][0]) + __popc(B[1][1]);
    const unsigned n0 = (B[0][i0] >> (4 * g)) & 0xfu, n1 = (B[0][i0 + 1] >> (4 * g)) & 0xfu;
    const unsigned n2 = (B[1][i0] >> (4 * g)) & 0xfu, n3 = (B[1][i0 + 1] >> (4 * g)) & 0xfu;
    const unsigned left = __popc(n0) + __popc(n1);
    const unsigned rk0 = __popc(n0 & lt) + __popc(n1 & lt);
    const unsigned rk1 = __popc(n0 & le) + __popc(n1 & lt);
    const unsigned rk2 = left + __popc(n2 & lt) + __popc(n3 & lt);
    const unsigned rk3 = left + __popc(n2 & le) + __popc(n3 & lt);
    if (acc[0][i0] != 0.0f) dst[pre + rk0] = acc[0][i0];
    if (acc[0][i0 + 1] != 0.0f) dst[pre + rk1] = acc[0][i0 + 1];
    if (acc[1][i0] != 0.0f) dst[pre + rk2] = acc[1][i0];
    if (acc[1][i0 + 1] != 0.0f) dst[pre + rk3] = acc[1][i0 + 1];
  }
  // row masks: lane r (< 16) writes row r
  {
    const int r = lane & 15, rr = r & 7, i0 = (r >> 3) * 2;
    const unsigned n0 = (B[0][i0] >> (4 * rr)) & 0xfu, n1 = (B[0][i0 + 1] >> (4 * rr)) & 0xfu;
    const unsigned n2 = (B[1][i0] >> (4 * rr)) & 0xfu, n3 = (B[1][i0 + 1] >> (4 * rr)) & 0xfu;
    const unsigned m = spread4(n0) | (spread4(n1) << 1) | (spread4(n2) << 8) | (spread4(n3) << 9);
    if (lane < 16) ot.cmask[s * 16 + r] = uint16_t(m);
  }
}

// Fragment of tile t given its header word h and value base vbase.
__device__ __forceinline__ void expand_frag(unsigned h, const unsigned short* __restrict__ vals,
                                            uint32_t vbase, uint32_t (&r)[4]) {
  const unsigned byte = h & 0xffu;
  const unsigned short* src = vals + vbase + (h >> 8);
  unsigned v[8];
  int q = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const bool on = (byte >> j) & 1u;
    v[j] = on ? unsigned(__ldg(src + q)) : 0u;
    q += on;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) r[i] = v[2 * i] | (v[2 * i + 1] << 16);
}

// One warp per segment.  Memory-level parallelism: lane j first loads pair
// j of the segment and both value offsets (one coalesced round), then the
// warp takes the pairs kBatch at a time, issuing every header and value
// load of the batch before its MMAs.  Accumulation order is unchanged
// (pairs in ascending k).
constexpr int kBatch = 4;

__global__ void __launch_bounds__(256) numeric_tc_kernel(TileMat A, TileMat B, TaskList tl,
                                                        OutTiles ot,
                                                        unsigned* __restrict__ err_flag) {
  const int lane = threadIdx.x & 31;
  const uint64_t s = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (s >= tl.nseg) return;
  const uint32_t p0 = tl.seg_off[s], p1 = tl.seg_off[s + 1];
  float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  const unsigned long long* pairs = reinterpret_cast<const unsigned long long*>(tl.pairs);
  const uint16_t* fhA = A.fhdr[kRoleA];
  const uint16_t* fhB = B.fhdr[kRoleB];
  const unsigned short* vA = reinterpret_cast<const unsigned short*>(A.vals[kRoleA]);
  const unsigned short* vB = reinterpret_cast<const unsigned short*>(B.vals[kRoleB]);
  for (uint32_t pb = p0; pb < p1; pb += 32) {
    const uint32_t n = min(32u, p1 - pb);
    uint32_t a_l = 0, b_l = 0, va_l = 0, vb_l = 0;
    if (lane < n) {
      const uint64_t pr = __ldg(pairs + pb + lane);
      a_l = uint32_t(pr);
      b_l = uint32_t(pr >> 32);
      va_l = __ldg(A.voff + a_l);
      vb_l = __ldg(B.voff + b_l);
    }
    for (uint32_t u0 = 0; u0 < n; u0 += kBatch) {
      unsigned hA[kBatch], hB[kBatch];
      uint32_t vaB[kBatch], vbB[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const uint32_t idx = u0 + u;
        const uint32_t a = __shfl_sync(kFull, a_l, idx & 31);
        const uint32_t b = __shfl_sync(kFull, b_l, idx & 31);
        vaB[u] = __shfl_sync(kFull, va_l, idx & 31);
        vbB[u] = __shfl_sync(kFull, vb_l, idx & 31);
        const bool ok = idx < n;
        hA[u] = ok ? __ldg(fhA + size_t(a) * 32 + lane) : 0u;
        hB[u] = ok ? __ldg(fhB + size_t(b) * 32 + lane) : 0u;
      }
      uint32_t fa[kBatch][4], fb[kBatch][4];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        expand_frag(hA[u], vA, vaB[u], fa[u]);
        expand_frag(hB[u], vB, vbB[u], fb[u]);
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        if (u0 + u < n) {
          // B regs: 0 = (k<8, n<8), 1 = (k<8, n>=8), 2 = (k>=8, n<8), 3 = (k>=8, n>=8)
          mma16816(acc[0], fa[u], fb[u][0], fb[u][2]);
          mma16816(acc[1], fa[u], fb[u][1], fb[u][3]);
        }
      }
    }
  }
  compress_store(acc, s, ot, lane, err_flag);
}

constexpr int kSA = 17;  // padded row stride of the A scratch tile

__global__ void __launch_bounds__(256) numeric_ordered_kernel(TileMat A, TileMat B, TaskList tl,
                                                             OutTiles ot,
                                                             unsigned* __restrict__ err_flag) {
  __shared__ float sA[8][16 * kSA];
  __shared__ float sB[8][16 * 16];
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
    const uint32_t a = uint32_t(pr), b = uint32_t(pr >> 32);
    for (int i = lane; i < 16 * kSA; i += 32) sA[w][i] = 0.f;
    for (int i = lane; i < 256; i += 32) sB[w][i] = 0.f;
    __syncwarp();
    // expand_tile (kernels.cpp:17-26) for both operands
#pragma unroll
    for (int role = 0; role < 2; ++role) {
      const TileMat& M = role == kRoleA ? A : B;
      const uint32_t tt = role == kRoleA ? a : b;
      const unsigned h = __ldg(M.fhdr[role] + size_t(tt) * 32 + lane);
      const unsigned short* src =
          reinterpret_cast<const unsigned short*>(M.vals[role]) + __ldg(M.voff + tt) + (h >> 8);
      int q = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if ((h >> j) & 1u) {
          int r, c;
          rc_of(role, lane, j, r, c);
          const float v = __half2float(__ushort_as_half(__ldg(src + q)));
          ++q;
          if (role == kRoleA)
            sA[w][r * kSA + c] = v;
          else
            sB[w][r * 16 + c] = v;
        }
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
          x = __fadd_rn(x, __fmul_rn(sA[w][r * kSA + kk], sB[w][kk * 16 + c]));
        acc[h][i] = x;
      }
    __syncwarp();
  }
  compress_store(acc, s, ot, lane, err_flag);
}

}  // namespace

void launch_numeric(const TileMat& A, const TileMat& B, const TaskList& tl, OutTiles& ot, int mode,
                    unsigned* err_flag, cudaStream_t st) {
  const uint64_t blocks = (tl.nseg + 7) / 8;
  if (blocks == 0) return;
  if (mode == 1)
    numeric_ordered_kernel<<<unsigned(blocks), 256, 0, st>>>(A, B, tl, ot, err_flag);
  else
    numeric_tc_kernel<<<unsigned(blocks), 256, 0, st>>>(A, B, tl, ot, err_flag);
}

}  // namespace tsg
