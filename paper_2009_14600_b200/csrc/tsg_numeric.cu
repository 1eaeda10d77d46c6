// tsg_numeric.cu -- subsystem (3): SEaC numeric phase (sort, expand, compress)
// with the counting pass fused in.
//
// GPU restatement of counting_pass + multiply_pass + finalize_segment
// (proj/src/kernels.cpp:79-203) at T = 16.  A warp owns one segment (= one
// output tile, TaskList order) at a time and walks its pairs in ascending
// inner tile k, keeping the 16x16 fp32 output tile in registers for the
// whole run (two m16n8 accumulators, 8 floats per lane).  Warps stride over
// the segments (persistent grid, one resident wave).
//
//   TENSOR mode: per pair each lane loads its A and B operand chunk (one
//     LDG.128 each, tsg_common.cuh) and the warp issues two
//     mma.sync.m16n8k16.f32.f16.f16.f32 -- the 16x16 tile product is exactly
//     one m16n16k16, so the 8x8 diagonal pairing of the reference
//     (kernels.cpp:40-77) has no waste left to remove.
//     Two more MMAs on the 0/1 indicators of the same operand registers
//     (set.ne.f16x2) count, per output slot, the products with two nonzero
//     factors: the slot is structurally nonzero (boolean_tile_mm,
//     pipeline.cpp:11-21) iff that count is.  This is the counting pass
//     (kernels.cpp:79-103) at no extra operand traffic.
//   ORDERED mode: CUDA-core fp32, one rounding per product, ascending k,
//     __fmul_rn/__fadd_rn (no FMA contraction, proj/CMakeLists.txt:12-14):
//     bit-identical to tile_mm_reference (kernels.cpp:28-38) and to
//     dense_spgemm_mixed_ordered (oracle.cpp:102-121).
//
// Compress (finalize_segment, kernels.cpp:109-127): the bitmap is the set of
// accumulators != 0 (so -0 and cancelled slots drop, which is compact(),
// kernels.cpp:205-220); it is stored as 16 row masks, and the nonzeros are
// packed row-major at the segment's staging offset for the CSR assembly.
// Non-finite accumulators raise kErrPrecision (PrecisionError,
// kernels.cpp:199-201) in the assembly pass, which reads every value.
#include "tsg_kernels.cuh"
#include "tsg_mma.cuh"

namespace tsg {

namespace {

// finalize_segment: realised bitmap (16 row masks) and the nonzeros packed
// row-major (compressed in this warp's shared scratch, written coalesced).
__device__ __forceinline__ void emit_tile(const float (&acc)[2][4], uint32_t so, uint64_t s,
                                          int lane, const LaneLayout& L, const Staged& sg,
                                          float* __restrict__ sv) {
  unsigned B[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int i = 0; i < 4; ++i) B[h][i] = __ballot_sync(kFull, acc[h][i] != 0.0f);
  const unsigned rm = row_mask_from_ballots(B, lane);  // row lane & 15
  const unsigned n = __popc(rm);
  unsigned incl = n;  // inclusive prefix over the 16 rows (each half-warp alike)
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const unsigned y = __shfl_up_sync(kFull, incl, o, 16);
    if ((lane & 15) >= o) incl += y;
  }
  if (lane < 16) sg.rmask[s * 16 + lane] = uint16_t(rm);  // 64-bit: 16 S > 2^32 on R-MAT
  const unsigned pk = (incl - n) | (rm << 16);
  const unsigned p0 = __shfl_sync(kFull, pk, L.g), p1 = __shfl_sync(kFull, pk, L.g + 8);
  const unsigned total = __shfl_sync(kFull, incl, 15);
  // entry index of (row, col 2t + 8h) = row prefix + nonzeros left of it in
  // the row; its odd neighbour follows directly when it is nonzero itself
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const unsigned p = q ? p1 : p0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float v0 = acc[h][2 * q], v1 = acc[h][2 * q + 1];
      const unsigned e0 = (p & 0xffffu) + __popc((p >> 16) & L.cm[h]);
      if (v0 != 0.0f) sv[e0] = v0;
      if (v1 != 0.0f) sv[e0 + (v0 != 0.0f)] = v1;
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) {  // total <= 256
    if (32u * k >= total) break;
    const unsigned e = lane + 32u * k;
    if (e < total) sg.val[so + e] = sv[e];
  }
  __syncwarp();
}

__device__ __forceinline__ void finish(uint32_t nstruct, const Staged& sg, int lane) {
  nstruct = __reduce_add_sync(kFull, nstruct);
  if (lane == 0 && nstruct) atomicAdd(sg.counted, (unsigned long long)nstruct);
}

// Per segment: (1) its bounds and staging offset, (2) one coalesced
// LDG.128 per lane of the operand metas of up to 32 pairs, parked in shared
// memory and read back as broadcasts, (3) the operand chunks of kBatch pairs
// at a time, then the MMAs.  Accumulation order is ascending k.
template <int kBatch, int kMinBlocks>
__global__ void __launch_bounds__(256, kMinBlocks) numeric_tc_kernel(TaskList tl, const uint4* __restrict__ cA,
                                                           const uint4* __restrict__ cB, Staged sg,
                                                           const uint32_t* __restrict__ list,
                                                           const uint32_t* __restrict__ list_len) {
  __shared__ __align__(16) uint4 s_meta[8][32];
  __shared__ __align__(16) float s_v[8][256];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const unsigned lt = lanemask_lt(), bit = 1u << lane;
  const LaneLayout L(lane);
  uint32_t nstruct = 0;
  const uint64_t stride = uint64_t(gridDim.x) * 8;
  const uint64_t nwork = list ? uint64_t(*list_len) : tl.nseg;
  for (uint64_t i = uint64_t(blockIdx.x) * 8 + w; i < nwork; i += stride) {
    const uint64_t s = list ? uint64_t(__ldg(list + i)) : i;
    const uint32_t p0 = tl.seg_off[s], p1 = tl.seg_off[s + 1];
    const uint32_t so = tl.stage_off[s];
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    uint32_t sac[2][2] = {{0u, 0u}, {0u, 0u}};  // .f16x2 counts of nonzero products
    for (uint32_t pb = p0; pb < p1; pb += 32) {
      const uint32_t n = min(32u, p1 - pb);
      s_meta[w][lane] = lane < n ? __ldg(tl.pmeta + pb + lane) : make_uint4(0, 0, 0, 0);
      __syncwarp();
      // kBatch | 32, so u0 + u <= 31; pairs past n hold zero metas and add
      // exact zeros (absent slots already are zeros: the sums cannot change)
      for (uint32_t u0 = 0; u0 < n; u0 += kBatch) {
        uint4 fa[kBatch], fb[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          const uint4 m = s_meta[w][u0 + u];
          fa[u] = load_chunk(cA, m.x, m.y, lt, bit);
          fb[u] = load_chunk(cB, m.z, m.w, lt, bit);
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
          // B chunk: {x, y} = {b0, b1} of the n0..7 MMA, {z, w} of the n8..15 MMA
          mma16816(acc[0], fa[u], fb[u].x, fb[u].y);
          mma16816(acc[1], fa[u], fb[u].z, fb[u].w);
          // boolean product as 0/1 counts (fp16 sums of positive integers
          // never return to zero; overflow saturates at inf, still nonzero)
          const uint4 xa = nz_h2(fa[u]), xb = nz_h2(fb[u]);
          mma16816_h(sac[0], xa, xb.x, xb.y);
          mma16816_h(sac[1], xa, xb.z, xb.w);
        }
      }
      __syncwarp();
    }
    nstruct += count_nz_counts(sac[0][0], sac[0][1], sac[1][0], sac[1][1]);
    emit_tile(acc, so, s, lane, L, sg, s_v[w]);
  }
  finish(nstruct, sg, lane);
}

constexpr int kSA = 17;    // padded row stride of the A scratch tile
constexpr int kSRow = 24;  // row stride of the B scratch tile

__global__ void __launch_bounds__(256) numeric_ordered_kernel(TaskList tl, const uint4* __restrict__ cA,
                                                             const uint4* __restrict__ cB, Staged sg,
                                                             const uint32_t* __restrict__ list,
                                                             const uint32_t* __restrict__ list_len) {
  __shared__ float sA[8][16 * kSA];
  __shared__ __align__(16) float sB[8][16 * kSRow];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const LaneLayout L(lane);
  uint32_t nstruct = 0;
  const uint64_t stride = uint64_t(gridDim.x) * 8;
  const uint64_t nwork = list ? uint64_t(*list_len) : tl.nseg;
  for (uint64_t i = uint64_t(blockIdx.x) * 8 + w; i < nwork; i += stride) {
    const uint64_t s = list ? uint64_t(__ldg(list + i)) : i;
    const uint32_t p0 = tl.seg_off[s], p1 = tl.seg_off[s + 1];
    const uint32_t so = tl.stage_off[s];
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    bool snz[2][4] = {{false, false, false, false}, {false, false, false, false}};
    for (uint32_t p = p0; p < p1; ++p) {
      const uint4 m = __ldg(tl.pmeta + p);
      // expand_tile (kernels.cpp:17-26): every lane writes all 8 of its slots
      // (absent lanes read the zero chunk), so no separate clearing is needed
#pragma unroll
      for (int role = 0; role < 2; ++role) {
        const uint4 ch = role == kRoleA ? __ldg(cA + chunk_index(m.x, m.y, lane))
                                        : __ldg(cB + chunk_index(m.z, m.w, lane));
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
      // tile_mm_reference: acc += a[r][k] * b[k][c], k ascending, no FMA.
      // A product of two binary16 values is exact in fp32, so it is nonzero
      // iff both factors are: that is the boolean product of the counting pass.
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
    emit_tile(acc, so, s, lane, L, sg, sA[w]);
  }
  finish(nstruct, sg, lane);
}

// ------------------------------------------------------------------ thin
// Segments whose staging bound is at most kThin slots (ultra-sparse tiles:
// R-MAT, the rectangular uniform product -- about one nonzero per tile and
// one pair per segment) get one thread each instead of one warp: the
// thread walks its pairs, and per pair the common inner slots k
// (A column occupancy & B row occupancy, pipeline.cpp:23-35), and
// accumulates every product a[r][k]*b[k][c] in sequential fp32 (k
// ascending, pairs in segment order, no FMA: tile_mm_reference,
// kernels.cpp:28-38) into a <= kThin-entry slot list -- bit-identical to
// the reference in both modes.  Heavier segments are flagged for the warp
// kernels.
constexpr int kThin = 8;

// binary16 value of slot (r, c) of a tile stored in `role` order
__device__ __forceinline__ float tile_value(const uint4* __restrict__ chunks, uint2 meta, int role,
                                            int r, int c) {
  int lane, j;
  slot_of(role, r, c, lane, j);
  if (!((meta.x >> lane) & 1u)) return 0.0f;
  const uint4 ch = __ldg(chunks + meta.y + __popc(meta.x & ((1u << lane) - 1u)));
  const int reg = j >> 1;
  // B chunks store the fragment registers as {reg0, reg2, reg1, reg3}
  const int at = role == kRoleB ? ((reg & 1) << 1 | (reg >> 1)) : reg;
  const uint32_t word = at == 0 ? ch.x : at == 1 ? ch.y : at == 2 ? ch.z : ch.w;
  return __half2float(__ushort_as_half(uint16_t(word >> (16 * (j & 1)))));
}

__global__ void __launch_bounds__(256) numeric_thin_kernel(TaskList tl, TileMat A, TileMat B, Staged sg,
                                                          uint8_t* __restrict__ heavy) {
  const uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  uint32_t nstruct = 0;
  if (s < tl.nseg) {
    const uint32_t so = tl.stage_off[s];
    const bool thin = tl.stage_off[s + 1] - so <= uint32_t(kThin);
    heavy[s] = !thin;
    if (thin) {
      uint32_t slot[kThin];
      float acc[kThin];
#pragma unroll
      for (int i = 0; i < kThin; ++i) {
        slot[i] = 0xffffu;
        acc[i] = 0.0f;
      }
      int n = 0;
      const uint32_t p0 = tl.seg_off[s], p1 = tl.seg_off[s + 1];
      for (uint32_t p = p0; p < p1; ++p) {
        // operand metas and occupancies of the pair, stored per pair by
        // pair_meta_kernel: consecutive segments read consecutive pairs
        const uint4 mt = __ldg(tl.pmeta + p);
        const uint2 oc = __ldg(tl.pocc + p);
        const uint32_t oa = oc.x, ob = oc.y;
        const uint2 ma = make_uint2(mt.x, mt.y), mb = make_uint2(mt.z, mt.w);
        for (uint32_t km = (oa & 0xffffu) & (ob >> 16); km; km &= km - 1) {
          const int k = __ffs(km) - 1;
          for (uint32_t rm = oa >> 16; rm; rm &= rm - 1) {
            const int r = __ffs(rm) - 1;
            const float a = tile_value(A.chunk[kRoleA], ma, kRoleA, r, k);
            if (a == 0.0f) continue;
            for (uint32_t cmk = ob & 0xffffu; cmk; cmk &= cmk - 1) {
              const int c = __ffs(cmk) - 1;
              const float b = tile_value(B.chunk[kRoleB], mb, kRoleB, k, c);
              if (b == 0.0f) continue;
              const uint32_t want = uint32_t(r << 4 | c);
              const float pr2 = __fmul_rn(a, b);
              // slot list kept sorted (row-major): position = slots below
              int pos = 0;
              bool hit = false;
#pragma unroll
              for (int i = 0; i < kThin; ++i) {
                if (i >= n) break;
                pos += slot[i] < want;
                hit |= slot[i] == want;
              }
              if (hit) {
#pragma unroll
                for (int i = 0; i < kThin; ++i)
                  if (i == pos) acc[i] = __fadd_rn(acc[i], pr2);
              } else {  // new structural slot (n < kThin: the bound holds it)
#pragma unroll
                for (int i = kThin - 1; i > 0; --i)
                  if (i > pos && i <= n) {
                    slot[i] = slot[i - 1];
                    acc[i] = acc[i - 1];
                  }
#pragma unroll
                for (int i = 0; i < kThin; ++i)
                  if (i == pos) {
                    slot[i] = want;
                    acc[i] = __fadd_rn(0.0f, pr2);
                  }
                ++n;
              }
            }
          }
        }
      }
      nstruct = uint32_t(n);
      uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // row masks, rows 2q | 2q+1 << 16
      uint32_t e = 0;
#pragma unroll
      for (int i = 0; i < kThin; ++i) {
        if (i >= n) break;
        if (acc[i] != 0.0f) {  // realised (cancelled slots drop: compact())
          const uint32_t r = slot[i] >> 4, bitpos = (slot[i] & 15u) + 16u * (r & 1u);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (uint32_t(q) == (r >> 1)) w[q] |= 1u << bitpos;
          sg.val[so + e] = acc[i];
          ++e;
        }
      }
      uint4* rec = reinterpret_cast<uint4*>(sg.rmask) + 2 * s;
      rec[0] = make_uint4(w[0], w[1], w[2], w[3]);
      rec[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
  }
  nstruct = __reduce_add_sync(kFull, nstruct);
  if ((threadIdx.x & 31) == 0 && nstruct) atomicAdd(sg.counted, (unsigned long long)nstruct);
}

// One resident wave: warps stride over the segments.  Occupancy is cached
// per kernel (host-side lookup, no device work).
unsigned resident_blocks(const void* kernel, uint64_t nseg) {
  struct Entry {
    const void* k;
    int per_sm;
  };
  static Entry cache[8];
  static int ncache = 0, sms = 0;
  int per_sm = 0;
  for (int i = 0; i < ncache; ++i)
    if (cache[i].k == kernel) per_sm = cache[i].per_sm;
  if (per_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    if (ncache < 8) cache[ncache++] = {kernel, per_sm};
  }
  const uint64_t want = (nseg + 7) / 8;
  const uint64_t cap = uint64_t(per_sm) * uint64_t(sms);
  return unsigned(want < cap ? want : cap);
}

}  // namespace

void launch_numeric_thin(const TaskList& tl, const TileMat& A, const TileMat& B, Staged& sg, uint8_t* heavy,
                         cudaStream_t st) {
  if (tl.nseg == 0) return;
  const uint64_t blocks = (tl.nseg + 255) / 256;
  numeric_thin_kernel<<<unsigned(blocks), 256, 0, st>>>(tl, A, B, sg, heavy);
}

void launch_numeric(const TaskList& tl, const TileMat& A, const TileMat& B, Staged& sg, int mode,
                    const uint32_t* list, const uint32_t* list_len, cudaStream_t st) {
  if (tl.nseg == 0) return;
  const uint4* cA = A.chunk[kRoleA];
  const uint4* cB = B.chunk[kRoleB];
  using K = void (*)(TaskList, const uint4*, const uint4*, Staged, const uint32_t*, const uint32_t*);
  K k = numeric_tc_kernel<2, 4>;
  if (mode == 1) {
    k = numeric_ordered_kernel;
  } else {
    const int v = tuning_variant("TSG_NUMERIC_BATCH", 2);
    const int mb = tuning_variant("TSG_NUMERIC_MINB", 4);
    if (v == 1) k = mb == 6 ? numeric_tc_kernel<1, 6> : numeric_tc_kernel<1, 5>;
    if (v == 2) k = mb == 4 ? numeric_tc_kernel<2, 4> : mb == 6 ? numeric_tc_kernel<2, 6> : numeric_tc_kernel<2, 5>;
    if (v == 4) k = mb == 3 ? numeric_tc_kernel<4, 3> : numeric_tc_kernel<4, 4>;
  }
  k<<<resident_blocks(reinterpret_cast<const void*>(k), tl.nseg), 256, 0, st>>>(tl, cA, cB, sg, list, list_len);
}

}  // namespace tsg
