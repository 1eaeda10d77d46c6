// tsg_esc.cu -- general rows: the tSparse symbolic + SEaC numeric phases for
// tile rows of A with more than 32 tiles (R-MAT, the rectangular product,
// the second AMG stage), fused per work unit in shared memory.
//
// GPU restatement at T = 16 of
//   enumerate_pairs / filter_zero_products  proj/src/pipeline.cpp:37-70
//   sort_and_segment                        proj/src/pipeline.cpp:72-109
//   counting_pass                           proj/src/kernels.cpp:79-103
//   expand_tile / tile_mm_reference         proj/src/kernels.cpp:17-38
//   multiply_pass / finalize_segment        proj/src/kernels.cpp:105-203
//   compact + to_element_coo                proj/src/kernels.cpp:205-220,
//                                           proj/src/tile_format.cpp:131-154
// On these matrices a tile holds ~1 nonzero, so a tile pair is ~1 product:
// the tile pairs of a unit are expanded straight into their element products
// (r, c, a*b) -- the "expand" of SEaC, done at enumeration -- and radix-sorted
// in shared memory by the output tile key (tile row, J, in-tile column,
// in-tile row), stable, so products of one slot keep ascending k.  Runs of
// equal (tile row, J) are the segments (output tiles, sort_and_segment);
// runs of equal slot are summed in that order with one fp32 rounding per
// product (tile_mm_reference: bit-identical to the reference in both numeric
// modes); sums != 0 are the realised bitmap (finalize_segment / compact()),
// written row-major, one piece per tile row.  No task list reaches HBM.
//
// Work units: up to 16 aligned light tile rows whose products fit one sort
// (kCap), or one column range of a heavy tile row (cut at quantiles of the
// global product-column distribution, 16-aligned so segment counts add up).
// A heavy unit whose products exceed kCap anyway is halved by column until it
// fits, or becomes a dense ordered leaf (<= 256 columns).
//
//   esc_brec        B row records {first entry, end, first col, last col}
//   esc_colcount/colhist/scan   product histogram over output columns -> G
//   esc_plan_prod/scan/group/fill   units and output records
//   esc_kernel      persistent CTAs over the units
//   esc_rowcount / scan / esc_copy   pieces -> CSR
//   esc_njt / esc_pairstats         raw and filtered tile-pair counts
#include <algorithm>
#include <cstdio>
#include <type_traits>

#include "tsg_kernels.cuh"

namespace tsg {

namespace {

constexpr int kNT = kEscThreads;  // threads per CTA
constexpr int kWarps = kNT / 32;
constexpr int kMaxIPT = 4096 / kNT;     // products per thread, at most (16 at 256 threads, 8 at 512)
static_assert(kNT == 256 || kNT == 512, "esc_kernel is written for 256 or 512 threads");
constexpr int kCap = kNT * kMaxIPT;     // products per sorted leaf
constexpr int kGroup = 16;              // light tile rows per unit, at most
constexpr uint32_t kDenseW = 256;       // columns of a dense leaf (16 x 256 accumulators)
constexpr uint32_t kMaxWidth = 1u << 28;  // sorted-leaf width: J < 2^24 keeps the key in 32 bits
constexpr uint32_t kGroupFlag = 0x80000000u;

struct EscSmem {
  union {
    // the leaf's A entries with products in range (compacted): {first B
    // entry in range, product prefix | row within the unit (16 b + r) << 16}
    // and the entry's A value (binary16 bits); entry ne is the sentinel {-, P}
    struct {
      uint2 t[kCap + 1];
      uint16_t av[kCap + 1];
    } tab;
    struct {
      uint32_t key[kCap];  // products: blocked, vectors rotated (phys())
      float val[kCap];
      uint32_t ctr[8 * kNT + 8 * kNT / 32];  // radix digit counters, [digit pair][thread], padded
    } s;
    struct {
      float acc[16 * kDenseW];
      uint8_t flag[16 * kDenseW];
    } d;
  };
  int64_t rowp[kGroup * 16 + 1];
  int32_t adj[256];   // staging index - realised rank, per (r, b)
  uint32_t cnt[256];  // realised entries per (b, r)
  uint32_t wsum[2 * kWarps];
  uint32_t stk[80];
  uint32_t bc[16];
};

__device__ __forceinline__ uint32_t half_nz(uint16_t h) { return h & 0x7fffu; }

#ifdef TSG_ESC_DIAG
// build-time diagnostics (-DTSG_ESC_DIAG): leaf shapes of one esc_kernel launch
// [0] sorted leaves [1] products [2] slots (kNT IPT) [3] pass-slots [4] nb==1 leaves
// [5] dense leaves [6] halvings [7] units [8..12] leaves by IPT 4/8/16 and products in nb>1 leaves
__device__ unsigned long long g_esc_diag[16];
#define ESC_DIAG(i, v) (tid == 0 ? (void)atomicAdd(&g_esc_diag[i], (unsigned long long)(v)) : (void)0)
#else
#define ESC_DIAG(i, v) ((void)0)
#endif
__device__ __forceinline__ uint32_t cpad(uint32_t L) { return L + (L >> 5); }

// Blocked layout: thread t owns items IPT t .. IPT t + IPT-1; its 16-byte
// vectors are rotated so an LDS.128 phase of 8 lanes hits 8 bank groups.
#ifndef TSG_ESC_ROT
#define TSG_ESC_ROT 1
#endif
template <int IPT>
__device__ __forceinline__ uint32_t phys(uint32_t g) {
  constexpr uint32_t NV = IPT / 4;
  if (NV == 1 || !TSG_ESC_ROT) return g;
  const uint32_t t = g / IPT, i = g % IPT, q = i >> 2;
  const uint32_t rot = NV == 4 ? ((t >> 1) & 3u) : ((t >> 2) & 1u);
  return t * IPT + (((q + rot) & (NV - 1)) << 2) + (i & 3u);
}

// Exclusive prefix (for warp w) and total of the per-warp sums ws[0 .. kWarps):
// every warp reads them with one lane each and scans in registers (no loop
// over the warps in every thread).
__device__ __forceinline__ void warp_sums(const uint32_t* ws, int w, int lane, uint32_t& pre, uint32_t& tot) {
  uint32_t x = lane < kWarps ? ws[lane] : 0u;
#pragma unroll
  for (int o = 1; o < kWarps; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  tot = __shfl_sync(kFull, x, kWarps - 1);
  pre = w > 0 ? __shfl_sync(kFull, x, w - 1) : 0u;
}

// exclusive block scan of two u32 (totals in ta, tb)
__device__ __forceinline__ void block_scan2(EscSmem& sm, uint32_t& a, uint32_t& b, uint32_t& ta, uint32_t& tb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t ia = a, ib = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t va = __shfl_up_sync(kFull, ia, o), vb = __shfl_up_sync(kFull, ib, o);
    if (lane >= o) {
      ia += va;
      ib += vb;
    }
  }
  if (lane == 31) {
    sm.wsum[w] = ia;
    sm.wsum[kWarps + w] = ib;
  }
  __syncthreads();
  uint32_t pa, pb;
  warp_sums(sm.wsum, w, lane, pa, ta);
  warp_sums(sm.wsum + kWarps, w, lane, pb, tb);
  a = pa + ia - a;
  b = pb + ib - b;
  __syncthreads();
}

// Exclusive scan of the per-thread 4-bit-digit counts w8[j] = count(j) |
// count(j + 8) << 16 over (digit, thread) order: afterwards
// ctr[cpad(j kNT + t)] holds the starts of digits j and j + 8 (the latter
// relative to tlo = items with digits 0..7) for thread t.  Returns the packed
// totals (lo16: digits 0..7, hi16: digits 8..15).
__device__ __forceinline__ uint32_t digit_scan(EscSmem& sm, const uint32_t (&w8)[8]) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int j = 0; j < 8; ++j) sm.s.ctr[cpad(j * kNT + tid)] = w8[j];
  __syncthreads();
  // raking: thread t sums the linear counters 8t .. 8t+7 (digit-major order)
  uint32_t v[8], sum = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = sm.s.ctr[cpad(8 * tid + i)];
    sum += v[i];
  }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sm.wsum[w] = inc;
  __syncthreads();
  uint32_t pre, T;
  warp_sums(sm.wsum, w, lane, pre, T);
  uint32_t run = inc - sum + pre;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    sm.s.ctr[cpad(8 * tid + i)] = run;
    run += v[i];
  }
  __syncthreads();
  return T;
}

// Blocked reload of the sorted items (thread t: items IPT t .. IPT t + IPT-1)
template <int IPT>
__device__ __forceinline__ void reload_blocked(const EscSmem& sm, uint32_t (&key)[IPT], float (&val)[IPT]) {
  const int tid = threadIdx.x;
  const uint4* k4 = reinterpret_cast<const uint4*>(sm.s.key) + tid * (IPT / 4);
  const float4* v4 = reinterpret_cast<const float4*>(sm.s.val) + tid * (IPT / 4);
#pragma unroll
  for (int q = 0; q < IPT / 4; ++q) {
    const uint32_t rot = !TSG_ESC_ROT ? 0u : IPT == 16 ? ((uint32_t(tid) >> 1) & 3u) : IPT == 8 ? ((uint32_t(tid) >> 2) & 1u) : 0u;
    const uint32_t pq = (q + rot) & (IPT / 4 - 1);
    const uint4 kk = k4[pq];
    const float4 vv = v4[pq];
    key[4 * q] = kk.x;
    key[4 * q + 1] = kk.y;
    key[4 * q + 2] = kk.z;
    key[4 * q + 3] = kk.w;
    val[4 * q] = vv.x;
    val[4 * q + 1] = vv.y;
    val[4 * q + 2] = vv.z;
    val[4 * q + 3] = vv.w;
  }
}

// One stable LSD pass on the 4-bit digit at `shift` over the valid items
// (mask vm) in registers: per-thread digit counts as 4-bit fields of a u64,
// a raking scan of the [digit][thread] counters, scatter, blocked reload.
// Returns the item count (dense from now on).
template <int IPT>
__device__ __forceinline__ uint32_t radix_pass(EscSmem& sm, uint32_t (&key)[IPT], float (&val)[IPT], uint32_t vm,
                                               int shift) {
  const int tid = threadIdx.x;
  // rk: each item's rank among the thread's earlier items of its digit (4 bits each)
  using Rk = typename std::conditional<(IPT <= 8), uint32_t, unsigned long long>::type;
  unsigned long long C = 0;
  Rk rk = 0;
  uint32_t nv = 0, d0 = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    if ((vm >> i) & 1u) {
      const uint32_t s = ((key[i] >> shift) & 15u) << 2;
      if (nv == 0) d0 = s;
      rk |= Rk((C >> s) & 15ull) << (4 * i);
      C += 1ull << s;
      ++nv;
    }
  }
  uint32_t w8[8];
  {
    // nibble j of each half -> byte j (even / odd digits), then one PRMT per
    // counter pair: w8[j] = count(j) | count(j + 8) << 16
    const uint32_t lo = uint32_t(C), hi = uint32_t(C >> 32);
    const uint32_t le = lo & 0x0f0f0f0fu, lod = (lo >> 4) & 0x0f0f0f0fu;
    const uint32_t he = hi & 0x0f0f0f0fu, hod = (hi >> 4) & 0x0f0f0f0fu;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t a = (j & 1) ? lod : le, b = (j & 1) ? hod : he;  // compile-time selects
      const uint32_t bj = uint32_t(j >> 1);                            // byte within the word
      // byte bj of a -> byte 0, byte bj of b -> byte 2, zeros elsewhere (selector 4 = b byte 0 ... ; 0x7 of the
      // zero operand): __byte_perm(x, y, s) picks bytes of {y:x} by nibbles of s
      w8[j] = __byte_perm(a, b, (bj) | (0xcu << 4) | ((4u + bj) << 8) | (0xcu << 12)) & 0x00ff00ffu;
    }
  }
  if (IPT == 16 && nv == 16 && C == (d0 == 60 ? 0ull : (1ull << (d0 + 4)))) {
    // all 16 items share digit d: its count (16) carried out of the 4-bit field
    const uint32_t d = d0 >> 2;
#pragma unroll
    for (int j = 0; j < 8; ++j) w8[j] = uint32_t(j) == (d & 7u) ? (16u << (16 * (d >> 3))) : 0u;
  }
  const uint32_t T = digit_scan(sm, w8);
  const uint32_t tlo = T & 0xffffu;  // items with digits 0..7: the base of digit 8
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    if ((vm >> i) & 1u) {
      const uint32_t d = (key[i] >> shift) & 15u;
      const uint32_t p = sm.s.ctr[cpad((d & 7u) * kNT + tid)];
      const uint32_t dst = (d < 8 ? (p & 0xffffu) : (p >> 16) + tlo) + uint32_t((rk >> (4 * i)) & 15u);
      const uint32_t q = phys<IPT>(dst);
      sm.s.key[q] = key[i];
      sm.s.val[q] = val[i];
    }
  }
  __syncthreads();
  reload_blocked<IPT>(sm, key, val);
  return tlo + (T >> 16);
}

template <int IPT>
__device__ __forceinline__ uint32_t valid_mask(uint32_t n) {
  const uint32_t g0 = threadIdx.x * IPT;
  if (n <= g0) return 0u;
  const uint32_t k = n - g0;
  return k >= uint32_t(IPT) ? (1u << IPT) - 1u : (1u << k) - 1u;
}

// first B entry of [b0, b1) with column >= c
__device__ __forceinline__ uint32_t lower_col(const int32_t* __restrict__ colB, uint32_t b0, uint32_t b1, uint32_t c) {
  while (b0 < b1) {
    const uint32_t m = (b0 + b1) >> 1;
    if (uint32_t(__ldg(colB + m)) < c)
      b0 = m + 1;
    else
      b1 = m;
  }
  return b0;
}

struct Unit {
  uint32_t I, lo, hi, nb, rec0;  // first tile row, column range, tile rows, first output record
};

// Output records of a unit (thread 0's chain state for a heavy unit).
struct PieceChain {
  uint32_t prev = kNoPiece;  // last record written by this unit
};

// A leaf's output: thread 0 reserves n staging slots and the piece record
// (published in sm.bc[0] = record, sm.bc[2..3] = staging base); the
// entries are then written straight to global staging.  All threads.
__device__ void begin_piece(EscSmem& sm, const EscArgs& g, const Unit& u, uint32_t n, PieceChain& pc) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    const unsigned long long base = n ? atomicAdd(g.stage_top, (unsigned long long)n) : 0ull;
    uint32_t rec = kNoPiece;
    if (u.nb > 1 || pc.prev == kNoPiece) {
      rec = u.rec0;
    } else if (n > 0) {  // a later leaf of a halved heavy unit: a pool piece chained after the last
      const uint32_t slot = atomicAdd(g.piece_top, 1u);
      if (slot < g.pool_cap)
        rec = *g.nrec + slot;
      else
        atomicOr(g.err_flag, unsigned(kErrPool));
    }
    if (u.nb == 1 && rec != kNoPiece) {
      if (pc.prev != kNoPiece) g.pieces[pc.prev].next = rec;
      pc.prev = rec;
    }
    sm.bc[0] = rec;
    sm.bc[2] = uint32_t(base);
    sm.bc[3] = uint32_t(base >> 32);
  }
  __syncthreads();
}

// The piece records (realised entries per row from sm.cnt[b][r]); the
// trailing barrier frees shared memory for the next leaf.
__device__ void end_piece(EscSmem& sm, const EscArgs& g, const Unit& u) {
  const int tid = threadIdx.x;
  const uint32_t rec = sm.bc[0];
  const unsigned long long base = (unsigned long long)sm.bc[2] | ((unsigned long long)sm.bc[3] << 32);
  if (rec != kNoPiece && tid < int(u.nb)) {  // thread b: the record of tile row I + b
    EscPiece& p = g.pieces[rec + tid];
    uint32_t off = 0;
    for (int b = 0; b < tid; ++b)
      for (int r = 0; r < 16; ++r) off += sm.cnt[b * 16 + r];
    p.I = u.I + tid;
    p.next = kNoPiece;
    p.off = base + off;
#pragma unroll
    for (int r = 0; r < 16; ++r) p.cnt[r] = sm.cnt[tid * 16 + r];
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long piece_base(const EscSmem& sm) {
  return (unsigned long long)sm.bc[2] | ((unsigned long long)sm.bc[3] << 32);
}

// Lockstep lower bounds: for each k, the first index of [b0[k], b1[k]) whose
// column is >= c[k] (returned in b0).  The K searches issue their loads
// together, so their latency chains overlap.
template <int K>
__device__ __forceinline__ void lower_cols(const int32_t* __restrict__ colB, uint32_t (&b0)[K], uint32_t (&b1)[K],
                                           const uint32_t (&c)[K]) {
  while (true) {
    bool any = false;
    uint32_t m[K];
    uint32_t v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      m[k] = (b0[k] + b1[k]) >> 1;
      if (b0[k] < b1[k]) {
        v[k] = uint32_t(__ldg(colB + m[k]));
        any = true;
      }
    }
    if (!any) break;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (b0[k] < b1[k]) {
        if (v[k] < c[k])
          b0[k] = m[k] + 1;
        else
          b1[k] = m[k];
      }
  }
}

// The leaf's entry table; false (nothing built) when its products exceed kCap.
// Thread t takes entries 2t and 2t+1 of each 2 kNT-entry round: their loads
// and the four range searches (entry x {lo, hi}) run concurrently.
__device__ bool build_table(EscSmem& sm, const EscArgs& g, const Unit& u, uint32_t lo, uint32_t hi,
                            uint32_t& P, uint32_t& ne) {
  const int tid = threadIdx.x;
  const int nrow = 16 * int(u.nb);
  const int64_t E0 = sm.rowp[0], E1 = sm.rowp[nrow];
  const bool full = lo == 0 && int64_t(hi) >= g.colsB;
  int bsearch0 = 128;  // the row search's first step: below the unit's row count
  while (bsearch0 > 1 && bsearch0 >= nrow) bsearch0 >>= 1;
  P = 0;
  ne = 0;
  for (int64_t e0 = E0; e0 < E1; e0 += 2 * kNT) {
    int64_t e[2];
    uint16_t a[2] = {0, 0};
    int32_t ca[2] = {0, 0};
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      e[x] = e0 + 2 * tid + x;
      if (e[x] < E1) {
        a[x] = __ldg(g.hA + e[x]);
        ca[x] = __ldg(g.colA + e[x]);
      }
    }
    uint4 rb[2];
#pragma unroll
    for (int x = 0; x < 2; ++x)  // {first entry, end, first col, last col}
      rb[x] = e[x] < E1 && half_nz(a[x]) ? __ldg(g.brec + ca[x]) : make_uint4(0, 0, 0, 0);
    // searches: k = 2x (first entry >= lo), 2x+1 (first entry >= hi)
    uint32_t s0[4], s1[4], sc[4];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const bool in = rb[x].y > rb[x].x && (full || (rb[x].z < hi && rb[x].w >= lo));
      const bool need_lo = in && !full && rb[x].z < lo, need_hi = in && !full && rb[x].w >= hi;
      s0[2 * x] = rb[x].x;
      s1[2 * x] = need_lo ? rb[x].y : rb[x].x;
      sc[2 * x] = lo;
      s0[2 * x + 1] = in ? rb[x].x : rb[x].x;
      s1[2 * x + 1] = need_hi ? rb[x].y : rb[x].x;
      sc[2 * x + 1] = hi;
      if (in && !need_hi) s0[2 * x + 1] = s1[2 * x + 1] = rb[x].y;  // the whole row tail is below hi
    }
    lower_cols<4>(g.colB, s0, s1, sc);
    uint32_t len[2], blo[2], br[2];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      blo[x] = s0[2 * x];
      len[x] = s0[2 * x + 1] > blo[x] ? s0[2 * x + 1] - blo[x] : 0u;
      br[x] = 0;
      if (len[x])
        for (int b = bsearch0; b > 0; b >>= 1)  // row within the unit: last rowp <= e
          if (int(br[x]) + b < nrow && sm.rowp[br[x] + b] <= e[x]) br[x] += b;
    }
    const uint32_t fa = len[0] > 0, fb = len[1] > 0;
    const uint32_t la = min(len[0], uint32_t(kCap) + 1u), lb = min(len[1], uint32_t(kCap) + 1u);
    uint32_t f = fa + fb, lc = la + lb, ft, lt;
    block_scan2(sm, f, lc, ft, lt);
    if (P + lt > uint32_t(kCap)) return false;
    if (fa) {
      sm.tab.t[ne + f] = make_uint2(blo[0], (P + lc) | (br[0] << 16));
      sm.tab.av[ne + f] = a[0];
    }
    if (fb) {
      sm.tab.t[ne + f + fa] = make_uint2(blo[1], (P + lc + la) | (br[1] << 16));
      sm.tab.av[ne + f + fa] = a[1];
    }
    ne += ft;
    P += lt;
  }
  if (tid == 0) sm.tab.t[ne] = make_uint2(0u, P);
  __syncthreads();
  return true;
}

// A single-tile-row leaf after its cc and J passes.  The products arrived in
// row order and every pass was stable, so the items are sorted by (J, cc, r)
// -- equal output slots adjacent, in ascending k -- and each row's entries
// come in column order.  A digit scan over the rows of the realised entries
// (digit_scan, as in a radix pass but without the scatter) gives every entry
// its row-major staging index directly: no row pass, no shared-memory emit.
template <int IPT>
__device__ void rowmajor_emit(EscSmem& sm, const EscArgs& g, const Unit& u, uint32_t lo, int jb, uint32_t n,
                              const uint32_t (&key)[IPT], const float (&val)[IPT], PieceChain& pc,
                              unsigned long long& segs, unsigned long long& structural) {
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t g0 = uint32_t(tid) * IPT;
  const uint32_t vmn = valid_mask<IPT>(n);
  const bool cont = g0 > 0 && g0 < n && sm.s.key[phys<IPT>(g0 - 1)] == key[0];
  auto run_tail = [&](uint32_t kcur, float s) {  // a run continuing into later threads
    for (uint32_t gg = g0 + IPT; gg < n; ++gg) {
      const uint32_t q = phys<IPT>(gg);
      if (sm.s.key[q] != kcur) break;
      s = __fadd_rn(s, sm.s.val[q]);
    }
    return s;
  };
  // the runs this thread owns (heads in its items), summed in k order; f(key, sum) per run
  auto for_runs = [&](auto&& f) {
    bool owned = false;
    uint32_t kcur = 0;
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      if ((vmn >> i) & 1u) {
        const bool head = i == 0 ? !cont : key[i] != key[i - 1];
        if (head) {
          if (owned) f(kcur, s);
          owned = true;
          kcur = key[i];
          s = val[i];
        } else if (owned) {
          s = __fadd_rn(s, val[i]);
        }
      }
    }
    if (owned) f(kcur, run_tail(kcur, s));
  };
  // pass 1: structural slots, realised entries per row (8-bit fields: a thread
  // may own 16 entries of one row)
  unsigned long long c0 = 0, c1 = 0;
  uint32_t nstruct = 0;
  bool bad = false;
  for_runs([&](uint32_t k, float x) {
    ++nstruct;
    bad |= !isfinite(x);
    if (x != 0.0f) {
      const uint32_t r = k & 15u;
      if (r < 8)
        c0 += 1ull << (8 * r);
      else
        c1 += 1ull << (8 * (r - 8));
    }
  });
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(g.err_flag, unsigned(kErrPrecision));
  nstruct = __reduce_add_sync(kFull, nstruct);
  if (lane == 0 && nstruct) atomicAdd(&sm.bc[1], nstruct);
  uint32_t w8[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) w8[j] = uint32_t((c0 >> (8 * j)) & 0xffu) | (uint32_t((c1 >> (8 * j)) & 0xffu) << 16);
  const uint32_t T = digit_scan(sm, w8);
  const uint32_t tlo = T & 0xffffu, tot = tlo + (T >> 16);
  auto start_of = [&](uint32_t r, int t) {  // staging index of row r's first entry of thread t
    const uint32_t p = sm.s.ctr[cpad((r & 7u) * kNT + t)];
    return r < 8 ? (p & 0xffffu) : (p >> 16) + tlo;
  };
  if (tid < 16) {  // the piece's per-row counts (sm.cnt[b = 0][r])
    const uint32_t st = start_of(uint32_t(tid), 0), en = tid == 15 ? tot : start_of(uint32_t(tid) + 1, 0);
    sm.cnt[tid] = en - st;
  }
  begin_piece(sm, g, u, tot, pc);  // (its barrier publishes sm.cnt)
  // pass 2: each realised entry at its row-major staging index
  if (sm.bc[0] != kNoPiece) {
    uint2* __restrict__ dst = g.stage + piece_base(sm);
    const uint32_t jmask = (1u << jb) - 1u;
    unsigned long long l0 = 0, l1 = 0;
    for_runs([&](uint32_t k, float x) {
      if (x == 0.0f) return;
      const uint32_t r = k & 15u;
      uint32_t rank;
      if (r < 8) {
        rank = uint32_t((l0 >> (8 * r)) & 0xffu);
        l0 += 1ull << (8 * r);
      } else {
        rank = uint32_t((l1 >> (8 * (r - 8))) & 0xffu);
        l1 += 1ull << (8 * (r - 8));
      }
      dst[start_of(r, tid) + rank] = make_uint2(lo + (((k >> 8) & jmask) << 4) + ((k >> 4) & 15u), __float_as_uint(x));
    });
  }
  if (tid == 0) {
    segs += sm.bc[7];
    structural += sm.bc[1];
    sm.bc[7] = 0;
    sm.bc[1] = 0;
  }
  end_piece(sm, g, u);
}

// Sorted leaf: expand, sort by (tile row, J, cc, r), segments, combine, write.
template <int IPT>
__device__ void sort_leaf(EscSmem& sm, const EscArgs& g, const Unit& u, uint32_t lo, uint32_t hi, uint32_t P,
                          uint32_t ne, PieceChain& pc, unsigned long long& segs, unsigned long long& structural) {
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t jr = (hi - lo + 15u) >> 4;  // tile columns of the leaf
  int jb = 0;
  while ((1u << jb) < jr) ++jb;
  const int bshift = 8 + jb;  // tile row within the unit above J
  // ---- expand: thread t generates products IPT t .. IPT t + IPT-1
  uint32_t key[IPT];
  float val[IPT];
  uint32_t vm = 0;
  const uint32_t g0 = uint32_t(tid) * IPT;
  uint32_t cc[IPT];
  uint16_t hb[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    key[i] = 0;
    val[i] = 0.f;
    cc[i] = 0;
    hb[i] = 0;
  }
  if (g0 < P) {
    uint32_t e = 0, top = ne;  // largest e with pre[e] <= g0
    while (top - e > 1) {
      const uint32_t m = (e + top) >> 1;
      if ((sm.tab.t[m].y & 0xffffu) <= g0)
        e = m;
      else
        top = m;
    }
    uint2 te = sm.tab.t[e];
    uint32_t nxt = sm.tab.t[e + 1].y & 0xffffu;
    float av = __half2float(__ushort_as_half(sm.tab.av[e]));
    // (1) B entry index of every item (shared memory only), the row in key[i]
    // and the A value in val[i]; (2) all the thread's global loads in flight at
    // once; (3) keys and exact products
    uint32_t idx[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t gi = g0 + i;
      idx[i] = 0;
      if (gi < P) {
        while (gi >= nxt) {
          te = sm.tab.t[++e];
          nxt = sm.tab.t[e + 1].y & 0xffffu;
          av = __half2float(__ushort_as_half(sm.tab.av[e]));
        }
        idx[i] = te.x + (gi - (te.y & 0xffffu));
        key[i] = te.y >> 16;
        val[i] = av;
      }
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      cc[i] = g0 + i < P ? uint32_t(__ldg(g.colB + idx[i])) : 0u;
      hb[i] = g0 + i < P ? __ldg(g.hB + idx[i]) : uint16_t(0);
    }
  }
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    if (half_nz(hb[i])) {
      const uint32_t c = cc[i], br = key[i];
      vm |= 1u << i;
      key[i] = ((br >> 4) << bshift) | (((c - lo) >> 4) << 8) | ((c & 15u) << 4) | (br & 15u);
      val[i] = __fmul_rn(val[i], __half2float(__ushort_as_half(hb[i])));
    }
  }
  __syncthreads();  // the table (aliased by the sort buffer) is consumed
  ESC_DIAG(0, 1);
  ESC_DIAG(1, P);
  ESC_DIAG(2, kNT * IPT);
  ESC_DIAG(3, uint64_t(kNT * IPT) * (1 + (bshift - 8 + 3) / 4 + (u.nb > 1 ? 2 : 0)));
  ESC_DIAG(4, u.nb == 1);
  ESC_DIAG(IPT == 4 ? 8 : IPT == 8 ? 9 : 10, 1);
  if (u.nb > 1) ESC_DIAG(11, P);
  // ---- sort: cc, J digits, tile row (stable: ascending k survives)
  uint32_t n = radix_pass<IPT>(sm, key, val, vm, 4);
  for (int s = 8; s < bshift; s += 4) n = radix_pass<IPT>(sm, key, val, valid_mask<IPT>(n), s);
  if (u.nb > 1) n = radix_pass<IPT>(sm, key, val, valid_mask<IPT>(n), bshift);
  // segments: runs of (tile row, J) -- the output tiles of sort_and_segment
  {
    const uint32_t vmn = valid_mask<IPT>(n);
    const uint32_t prev = (g0 > 0 && g0 < n) ? (sm.s.key[phys<IPT>(g0 - 1)] >> 8) : 0xffffffffu;
    uint32_t heads = 0;
#pragma unroll
    for (int i = 0; i < IPT; ++i)
      if ((vmn >> i) & 1u) heads += (key[i] >> 8) != (i == 0 ? prev : (key[i - 1] >> 8)) ? 1u : 0u;
    heads = __reduce_add_sync(kFull, heads);
    if (lane == 0 && heads) atomicAdd(&sm.bc[7], heads);
  }
  if (u.nb == 1) {
    rowmajor_emit<IPT>(sm, g, u, lo, jb, n, key, val, pc, segs, structural);
    return;
  }
  // ---- row: order (r, tile row, J, cc); a (tile row, r) group is one CSR row slice
  n = radix_pass<IPT>(sm, key, val, valid_mask<IPT>(n), 0);
  const uint32_t vmn = valid_mask<IPT>(n);
  const bool cont = g0 > 0 && g0 < n && sm.s.key[phys<IPT>(g0 - 1)] == key[0];
  // group index (r, b) of a key: 16 r + b
  auto rb_of = [&](uint32_t k) { return ((k & 15u) << 4) | (k >> bshift); };
  auto run_tail = [&](uint32_t kcur, float s) {  // a run continuing into later threads
    for (uint32_t gg = g0 + IPT; gg < n; ++gg) {
      const uint32_t q = phys<IPT>(gg);
      if (sm.s.key[q] != kcur) break;
      s = __fadd_rn(s, sm.s.val[q]);
    }
    return s;
  };
  // pass 1: realised entries per (b, r) (runs owned by this thread)
  if (tid < 256) sm.cnt[tid] = 0;
  __syncthreads();
  uint32_t nreal = 0, nstruct = 0;
  bool bad = false;
  {
    bool owned = false;
    uint32_t kcur = 0, gcur = 0xffffffffu, crun = 0;
    float s = 0.f;
    auto close_run = [&](float x) {
      if (x != 0.0f) {
        ++nreal;
        const uint32_t gr = rb_of(kcur);
        if (gr != gcur) {
          if (crun) atomicAdd(&sm.cnt[((gcur & 15u) << 4) | (gcur >> 4)], crun);  // sm.cnt is [b][r]
          gcur = gr;
          crun = 0;
        }
        ++crun;
      }
      bad |= !isfinite(x);
    };
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      if ((vmn >> i) & 1u) {
        const bool head = i == 0 ? !cont : key[i] != key[i - 1];
        if (head) {
          if (owned) close_run(s);
          owned = true;
          kcur = key[i];
          s = val[i];
          ++nstruct;
        } else if (owned) {
          s = __fadd_rn(s, val[i]);
        }
      }
    }
    if (owned) close_run(run_tail(kcur, s));
    if (crun) atomicAdd(&sm.cnt[((gcur & 15u) << 4) | (gcur >> 4)], crun);
  }
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(g.err_flag, unsigned(kErrPrecision));
  nstruct = __reduce_add_sync(kFull, nstruct);
  if (lane == 0 && nstruct) atomicAdd(&sm.bc[1], nstruct);
  uint32_t off = nreal, zero = 0, tot, dt;
  block_scan2(sm, off, zero, tot, dt);  // (its barriers also publish sm.cnt)
  begin_piece(sm, g, u, tot, pc);
  // staging index = realised rank + adj[r][b]: the unit's tile rows one after
  // another, each row-major.  Thread t: group (r, b) = (t >> 4, t & 15) for the
  // rank of its first entry (entries of the groups before it in (r, b) order),
  // and (b, r) = (t >> 4, t & 15) for its staging index (row-major order)
  {
    const bool grp = tid < 256;  // one thread per (b, r) group
    uint32_t x = grp ? sm.cnt[((tid & 15) << 4) | (tid >> 4)] : 0u, y = grp ? sm.cnt[tid] : 0u, tx, ty;
    block_scan2(sm, x, y, tx, ty);
    if (grp) sm.adj[((tid & 15) << 4) | (tid >> 4)] = int32_t(y);  // (r, b) slot <- staging start of (b, r)
    __syncthreads();
    if (grp) sm.adj[tid] -= int32_t(x);
  }
  __syncthreads();
  // pass 2: write the realised entries at their staging index (global)
  if (sm.bc[0] != kNoPiece) {
    bool owned = false;
    uint32_t kcur = 0, o = off;
    float s = 0.f;
    const uint32_t jmask = (1u << jb) - 1u;
    uint2* __restrict__ dst = g.stage + piece_base(sm);
    auto emit = [&](float x) {
      if (x != 0.0f) {
        const uint32_t q = uint32_t(int32_t(o) + sm.adj[rb_of(kcur)]);
        dst[q] = make_uint2(lo + (((kcur >> 8) & jmask) << 4) + ((kcur >> 4) & 15u), __float_as_uint(x));
        ++o;
      }
    };
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      if ((vmn >> i) & 1u) {
        const bool head = i == 0 ? !cont : key[i] != key[i - 1];
        if (head) {
          if (owned) emit(s);
          owned = true;
          kcur = key[i];
          s = val[i];
        } else if (owned) {
          s = __fadd_rn(s, val[i]);
        }
      }
    }
    if (owned) emit(run_tail(kcur, s));
  }
  if (tid == 0) {  // (bc[1], bc[7] are complete: block_scan2 and begin_piece synchronised since)
    segs += sm.bc[7];
    structural += sm.bc[1];
    sm.bc[7] = 0;
    sm.bc[1] = 0;
  }
  end_piece(sm, g, u);
}

// Dense leaf (a heavy unit's <= 256 columns whose products exceed kCap):
// 16 x 256 fp32 accumulators; warp w owns rows w and w + 8 and walks their A
// entries in ascending k, lanes over the B row's entries in range -- per slot
// the products are added in k order (the reference's sequence).
__device__ void dense_leaf(EscSmem& sm, const EscArgs& g, const Unit& u, uint32_t lo, uint32_t hi, PieceChain& pc,
                           unsigned long long& segs, unsigned long long& structural) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t width = hi - lo;
  for (uint32_t i = tid; i < 16 * kDenseW; i += kNT) {
    sm.d.acc[i] = 0.f;
    sm.d.flag[i] = 0;
  }
  if (tid == 0) sm.bc[7] = 0;
  __syncthreads();
  for (int rr = w; rr < 16; rr += kWarps) {
    const int64_t e0 = sm.rowp[rr], e1 = sm.rowp[rr + 1];
    for (int64_t e = e0; e < e1; ++e) {
      const uint16_t a = __ldg(g.hA + e);
      if (!half_nz(a)) continue;
      const uint4 rb = __ldg(g.brec + __ldg(g.colA + e));
      const uint32_t blo = lower_col(g.colB, rb.x, rb.y, lo), bhi = lower_col(g.colB, blo, rb.y, hi);
      const float af = __half2float(__ushort_as_half(a));
      for (uint32_t j = blo + lane; j < bhi; j += 32) {
        const uint16_t hb = __ldg(g.hB + j);
        if (!half_nz(hb)) continue;
        const uint32_t slot = uint32_t(rr) * kDenseW + (uint32_t(__ldg(g.colB + j)) - lo);
        const float p = __fmul_rn(af, __half2float(__ushort_as_half(hb)));
        sm.d.acc[slot] = sm.d.flag[slot] ? __fadd_rn(sm.d.acc[slot], p) : p;
        sm.d.flag[slot] = 1;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  // thread t < 256: row t >> 4, columns 16 (t & 15) .. +15 (one tile column)
  const uint32_t row = tid >> 4, tc = tid & 15;
  const bool dl = tid < 256;
  uint32_t nreal = 0, nst = 0;
  bool bad = false;
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t c = tc * 16 + i, s = row * kDenseW + c;
    v[i] = 0.f;
    if (dl && c < width && sm.d.flag[s]) {
      ++nst;
      v[i] = sm.d.acc[s];
      nreal += v[i] != 0.0f;
      bad |= !isfinite(v[i]);
    }
  }
  if (nst) atomicOr(&sm.bc[7], 1u << tc);  // tile column tc holds a structural entry
  if (__any_sync(kFull, bad) && lane == 0) atomicOr(g.err_flag, unsigned(kErrPrecision));
  if (tid < 256) sm.cnt[tid] = 0;
  __syncthreads();  // the accumulators are in registers before the output aliases them
  uint32_t off = nreal, zero = 0, tot, dt;
  if (nreal) atomicAdd(&sm.cnt[row], nreal);
  nst = __reduce_add_sync(kFull, nst);
  if (lane == 0 && nst) atomicAdd(&sm.bc[1], nst);
  block_scan2(sm, off, zero, tot, dt);
  begin_piece(sm, g, u, tot, pc);
  if (sm.bc[0] != kNoPiece) {
    uint2* __restrict__ dst = g.stage + piece_base(sm);
    uint32_t o = off;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (v[i] != 0.0f) dst[o++] = make_uint2(lo + tc * 16 + i, __float_as_uint(v[i]));
  }
  if (tid == 0) {
    segs += __popc(sm.bc[7]);
    structural += sm.bc[1];
    sm.bc[7] = 0;
    sm.bc[1] = 0;
  }
  end_piece(sm, g, u);
}

template <int kMinBlocks>
__global__ void __launch_bounds__(kNT, kMinBlocks) esc_kernel(EscArgs g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EscSmem& sm = *reinterpret_cast<EscSmem*>(smem_raw);
  const int tid = threadIdx.x;
  unsigned long long segs = 0, structural = 0;  // thread 0's tallies
  if (tid == 0) {
    sm.bc[1] = 0;
    sm.bc[7] = 0;
  }
  const uint32_t nunits = min(*g.nunits, g.unit_end);
  for (;;) {
    if (tid == 0) sm.bc[0] = g.unit0 + atomicAdd(g.work, 1u);
    __syncthreads();
    const uint32_t ui = sm.bc[0];
    __syncthreads();
    if (ui >= nunits) break;
    ESC_DIAG(7, 1);
    const uint4 wu = g.units[ui];
    Unit u;
    u.I = wu.x;
    u.lo = wu.y;
    u.hi = wu.z;
    u.nb = (wu.w & kGroupFlag) ? (wu.w & 0xffu) : 1u;
    u.rec0 = g.rec_base[u.I] + ((wu.w & kGroupFlag) ? 0u : wu.w);
    for (int i = tid; i <= 16 * int(u.nb); i += kNT) {
      int64_t r = int64_t(u.I) * 16 + i;
      if (r > g.rowsA) r = g.rowsA;
      sm.rowp[i] = __ldg(g.rpA + r);
    }
    PieceChain pc;
    if (u.nb == 1) {  // a heavy unit's record starts empty (a unit without products keeps it)
      if (tid < 16) g.pieces[u.rec0].cnt[tid] = 0;
      if (tid == 0) {
        g.pieces[u.rec0].I = u.I;
        g.pieces[u.rec0].next = kNoPiece;
        g.pieces[u.rec0].off = 0;
      }
    }
    if (tid == 0) {
      sm.stk[0] = u.lo;
      sm.stk[1] = u.hi;
      sm.bc[4] = 1;  // stack depth
    }
    __syncthreads();
    while (true) {
      const uint32_t depth = sm.bc[4];
      if (depth == 0) break;
      const uint32_t lo = sm.stk[2 * (depth - 1)], hi = sm.stk[2 * (depth - 1) + 1];
      __syncthreads();
      if (tid == 0) sm.bc[4] = depth - 1;
      uint32_t P = 0, ne = 0;
      const bool fits = hi > lo && hi - lo <= kMaxWidth && build_table(sm, g, u, lo, hi, P, ne);
      if (hi <= lo) {
      } else if (fits) {
        if (P <= uint32_t(kNT) * 4)
          sort_leaf<4>(sm, g, u, lo, hi, P, ne, pc, segs, structural);
        else if (kMaxIPT == 8 || P <= uint32_t(kNT) * 8)
          sort_leaf<8>(sm, g, u, lo, hi, P, ne, pc, segs, structural);
        else if constexpr (kMaxIPT >= 16)
          sort_leaf<16>(sm, g, u, lo, hi, P, ne, pc, segs, structural);
      } else if (u.nb > 1) {  // cannot happen: a group's products fit (planned exactly)
        if (tid == 0) atomicOr(g.err_flag, unsigned(kErrPool));
      } else if (hi - lo <= kDenseW) {
        ESC_DIAG(5, 1);
        dense_leaf(sm, g, u, lo, hi, pc, segs, structural);
      } else {  // halve (16-aligned), left half first
        ESC_DIAG(6, 1);
        if (tid == 0) {
          uint32_t mid = (lo + ((hi - lo) >> 1)) & ~15u;
          if (mid <= lo) mid = lo + 16;
          const uint32_t d = sm.bc[4];
          sm.stk[2 * d] = mid;
          sm.stk[2 * d + 1] = hi;
          sm.stk[2 * d + 2] = lo;
          sm.stk[2 * d + 3] = mid;
          sm.bc[4] = d + 2;
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    if (segs) atomicAdd(g.segs, segs);
    if (structural) atomicAdd(g.counted, structural);
  }
}

// ---------------------------------------------------------------- planning

__global__ void esc_brec_kernel(int64_t rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                uint4* __restrict__ brec) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < rows; k += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t b0 = uint32_t(rp[k]), b1 = uint32_t(rp[k + 1]);
    brec[k] = make_uint4(b0, b1, b1 > b0 ? uint32_t(__ldg(col + b0)) : 0u, b1 > b0 ? uint32_t(__ldg(col + b1 - 1)) : 0u);
  }
}

// colcnt[k] = kept A entries in column k
__global__ void esc_colcount_kernel(int64_t nnz, const int32_t* __restrict__ col, const uint16_t* __restrict__ h,
                                    uint32_t* __restrict__ colcnt) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nnz; e += int64_t(gridDim.x) * blockDim.x)
    if (half_nz(__ldg(h + e))) atomicAdd(colcnt + __ldg(col + e), 1u);
}

// hist[c] += colcnt[k] for every kept B entry (k, c): warp per B row
__global__ void esc_colhist_kernel(int64_t rowsB, const int64_t* __restrict__ rpB, const int32_t* __restrict__ colB,
                                   const uint16_t* __restrict__ hB, const uint32_t* __restrict__ colcnt,
                                   unsigned long long* __restrict__ hist) {
  // eight lanes per B row, four rows per warp step (R-MAT rows hold ~16 entries)
  const int lane = threadIdx.x & 31, sl = lane & 7;
  for (int64_t k0 = ((blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5) * 4; k0 < rowsB;
       k0 += ((int64_t(gridDim.x) * blockDim.x) >> 5) * 4) {
    const int64_t k = k0 + (lane >> 3);
    const uint32_t w = k < rowsB ? __ldg(colcnt + k) : 0u;
    if (!w) continue;
    const int64_t b1 = __ldg(rpB + k + 1);
    for (int64_t e = __ldg(rpB + k) + sl; e < b1; e += 8)
      if (half_nz(__ldg(hB + e))) atomicAdd(hist + __ldg(colB + e), (unsigned long long)w);
  }
}

// products of each tile row: kept A entries x their B row lengths
__global__ void __launch_bounds__(256) esc_plan_prod_kernel(int64_t rowsA, uint32_t tile_rows,
                                                           const int64_t* __restrict__ rpA,
                                                           const int32_t* __restrict__ colA,
                                                           const uint16_t* __restrict__ hA,
                                                           const uint4* __restrict__ brec,
                                                           unsigned long long* __restrict__ prod,
                                                           unsigned long long* __restrict__ total) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows) return;
  const int64_t r0 = int64_t(I) * 16, r1 = r0 + 16 < rowsA ? r0 + 16 : rowsA;
  const int64_t e0 = rpA[r0], e1 = rpA[r1];
  unsigned long long p = 0;
  for (int64_t e = e0 + lane; e < e1; e += 32)
    if (half_nz(__ldg(hA + e))) {
      const uint4 rb = __ldg(brec + __ldg(colA + e));
      p += rb.y - rb.x;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(kFull, p, o);
  if (lane == 0) {
    prod[I] = p;
    if (p) atomicAdd(total, p);
  }
}

// the aligned group of 2^gbits tile rows that tile row I joins (gbits = 0:
// alone); a heavy row (> kCap products) returns -1
__device__ __forceinline__ int group_bits(uint32_t I, uint32_t tile_rows, const unsigned long long* __restrict__ pre,
                                          bool allow) {
  if (pre[I + 1] - pre[I] > uint64_t(kCap)) return -1;
  int gb = 0;
  if (allow)
    for (int b = 4; b >= 1; --b) {
      const uint32_t I0 = I & ~((1u << b) - 1u), I1 = min(I0 + (1u << b), tile_rows);
      if (pre[I1] - pre[I0] <= uint64_t(kCap)) {
        gb = b;
        break;
      }
    }
  return gb;
}

// output records (nrec) and work units (nwk) per tile row
__global__ void esc_plan_group_kernel(uint32_t tile_rows, const unsigned long long* __restrict__ pre, bool allow,
                                      uint32_t max_chunks, uint32_t target, uint32_t* __restrict__ nrec,
                                      uint32_t* __restrict__ nwk) {
  const uint32_t I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= tile_rows) return;
  const int gb = group_bits(I, tile_rows, pre, allow);
  if (gb < 0) {
    const uint64_t p = pre[I + 1] - pre[I];
    const uint64_t n = std::min<uint64_t>(max_chunks, (p + target - 1) / target);
    nrec[I] = uint32_t(n);
    nwk[I] = uint32_t(n);
  } else {
    nrec[I] = 1;
    nwk[I] = (I & ((1u << gb) - 1u)) == 0u ? 1u : 0u;
  }
}

// unit descriptors {I, c0, c1, j | kGroupFlag + nb}: a heavy tile row's
// column ranges at quantiles of the global product-column distribution G
__global__ void __launch_bounds__(256) esc_plan_fill_kernel(uint32_t tile_rows, int64_t colsB,
                                                           const unsigned long long* __restrict__ pre, bool allow,
                                                           const uint32_t* __restrict__ nwk,
                                                           const uint32_t* __restrict__ wbase,
                                                           const unsigned long long* __restrict__ G,
                                                           uint4* __restrict__ units) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows) return;
  const uint32_t n = nwk[I], b = wbase[I];
  if (n == 0) return;
  const int gb = group_bits(I, tile_rows, pre, allow);
  if (gb >= 0) {
    if (lane == 0) {
      const uint32_t nb = min(1u << gb, tile_rows - I);
      units[b] = make_uint4(I, 0u, uint32_t(colsB), kGroupFlag | nb);
    }
    return;
  }
  const double Gt = double(G[colsB]);
  auto quant = [&](uint32_t j) -> uint32_t {  // 16-aligned column of the j/n quantile
    if (j == 0) return 0u;
    if (j >= n) return uint32_t(colsB);
    const double want = Gt * double(j) / double(n);
    int64_t lo = 0, hi = colsB;  // smallest c with G[c] >= want
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (double(__ldg(G + m)) < want)
        lo = m + 1;
      else
        hi = m;
    }
    return uint32_t(lo) & ~15u;
  };
  for (uint32_t j = lane; j < n; j += 32) units[b + j] = make_uint4(I, quant(j), quant(j + 1), j);
}

// ---------------------------------------------------------------- assembly

// rowcnt[16 I + r] = realised entries of row r; each piece gets its offset
// within the row.  Warp per tile row, lane r < 16 = row r.
__global__ void __launch_bounds__(256) esc_rowcount_kernel(int64_t rows, uint32_t tile_rows,
                                                          const uint32_t* __restrict__ base, EscPiece* pieces,
                                                          int64_t* __restrict__ rowcnt, uint32_t I0) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = I0 + blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= tile_rows || lane >= 16) return;
  uint32_t acc = 0;
  for (uint32_t c = base[I]; c < base[I + 1]; ++c)
    for (uint32_t p = c; p != kNoPiece; p = pieces[p].next) {
      const uint32_t n = pieces[p].cnt[lane];
      pieces[p].roff[lane] = acc;
      acc += n;
    }
  const int64_t row = int64_t(I) * 16 + lane;
  if (row < rows) rowcnt[row] = acc;
}

// A piece's header as the copy needs it: lane r < 16 holds row r's count and
// its entries of the row in earlier pieces; I and the staging offset.
struct PieceHdr {
  uint32_t cnt = 0, ro = 0, I = 0;
  unsigned long long off = 0;
};
__device__ __forceinline__ PieceHdr load_hdr(const EscPiece* __restrict__ pieces, uint32_t p, int lane) {
  PieceHdr h;
  const EscPiece& pc = pieces[p];
  h.cnt = lane < 16 ? pc.cnt[lane] : 0u;
  h.ro = lane < 16 ? pc.roff[lane] : 0u;
  h.I = pc.I;
  h.off = pc.off;
  return h;
}
// row r's first CSR slot for this piece (lane r < 16)
__device__ __forceinline__ int64_t piece_dst0(const PieceHdr& h, const int64_t* __restrict__ row_ptr, int lane) {
  return lane < 16 && h.cnt ? row_ptr[int64_t(h.I) * 16 + lane] + h.ro : 0;
}

// One staged piece -> its CSR slots: lanes over the piece's entries; entry q
// belongs to the last row whose start within the piece is <= q.
#ifndef TSG_ESC_COPY_U
#define TSG_ESC_COPY_U 16
#endif
constexpr int kEscCopyU = TSG_ESC_COPY_U;

__device__ __forceinline__ void copy_piece(const PieceHdr& h, int64_t dst0, int lane, const uint2* __restrict__ stage,
                                           int32_t* __restrict__ col, float* __restrict__ val) {
  uint32_t inc = h.cnt;  // each row's start within the piece
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += v;
  }
  const uint32_t total = __shfl_sync(kFull, inc, 15);
  const uint32_t start = inc - h.cnt;
  // kEscCopyU entries per lane in flight: all loads first, then the row lookups and stores
  for (uint32_t q0 = 0; q0 < total; q0 += 32 * kEscCopyU) {
    uint2 e[kEscCopyU];
#pragma unroll
    for (int u = 0; u < kEscCopyU; ++u) {
      const uint32_t q = q0 + 32 * u + lane;
      e[u] = q < total ? __ldg(stage + h.off + q) : make_uint2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < kEscCopyU; ++u) {
      const uint32_t q = q0 + 32 * u + lane;
      if (q0 + 32 * u >= total) break;
      int r = 0;
#pragma unroll
      for (int b = 8; b > 0; b >>= 1) {
        const uint32_t st = __shfl_sync(kFull, start, r + b);
        if (st <= q) r += b;
      }
      const uint32_t sr = __shfl_sync(kFull, start, r);
      const int64_t d = __shfl_sync(kFull, dst0, r);
      if (q < total) {
        col[d + (q - sr)] = int32_t(e[u].x);
        val[d + (q - sr)] = __uint_as_float(e[u].y);
      }
    }
  }
}

// staged pieces -> CSR: a warp takes pieces p, p + W, ...; the header two
// pieces ahead and the row pointers one piece ahead are in flight while the
// current piece's entries move
__global__ void __launch_bounds__(256) esc_copy_kernel(const uint32_t* __restrict__ nrec,
                                                      const uint32_t* __restrict__ piece_top, uint32_t pool_cap,
                                                      const EscPiece* __restrict__ pieces,
                                                      const uint2* __restrict__ stage,
                                                      const int64_t* __restrict__ row_ptr,
                                                      int32_t* __restrict__ col, float* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const uint32_t np = *nrec + min(*piece_top, pool_cap);
  const uint32_t W = (gridDim.x * blockDim.x) >> 5;
  uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= np) return;
  PieceHdr h = load_hdr(pieces, p, lane);
  PieceHdr h1 = p + W < np ? load_hdr(pieces, p + W, lane) : PieceHdr{};
  int64_t d0 = piece_dst0(h, row_ptr, lane);
  for (; p < np; p += W) {
    const PieceHdr h2 = p + 2 * W < np ? load_hdr(pieces, p + 2 * W, lane) : PieceHdr{};
    const int64_t d1 = p + W < np ? piece_dst0(h1, row_ptr, lane) : 0;
    copy_piece(h, d0, lane, stage, col, val);
    h = h1;
    h1 = h2;
    d0 = d1;
  }
}

// records [rec0, rec1) and the pool pieces chained after them: warp per record
__global__ void __launch_bounds__(256) esc_copy_records_kernel(uint32_t rec0, uint32_t rec1,
                                                              const EscPiece* __restrict__ pieces,
                                                              const uint2* __restrict__ stage,
                                                              const int64_t* __restrict__ row_ptr,
                                                              int32_t* __restrict__ col, float* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  for (uint32_t p = rec0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); p < rec1;
       p += (gridDim.x * blockDim.x) >> 5)
    for (uint32_t q = p; q != kNoPiece; q = pieces[q].next) {
      const PieceHdr h = load_hdr(pieces, q, lane);
      copy_piece(h, piece_dst0(h, row_ptr, lane), lane, stage, col, val);
    }
}

// ---------------------------------------------------------------- statistics

// njt[k] = distinct tiles CSR row k of B touches (its entries that are the
// first of their (row, tile)).  Eight lanes per row, four rows per warp step
// (R-MAT rows hold ~16 entries).
__global__ void esc_njt_kernel(int64_t rows, const int64_t* __restrict__ rp, const uint32_t* __restrict__ etile,
                               uint32_t* __restrict__ njt) {
  const int lane = threadIdx.x & 31, sl = lane & 7;
  for (int64_t k0 = ((blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5) * 4; k0 < rows;
       k0 += ((int64_t(gridDim.x) * blockDim.x) >> 5) * 4) {
    const int64_t k = k0 + (lane >> 3);
    uint32_t n = 0;
    if (k < rows) {
      const int64_t e1 = __ldg(rp + k + 1);
      for (int64_t e = __ldg(rp + k) + sl; e < e1; e += 8) n += (__ldg(etile + e) & kDupEntry) == 0u;
    }
    n += __shfl_xor_sync(kFull, n, 1);
    n += __shfl_xor_sync(kFull, n, 2);
    n += __shfl_xor_sync(kFull, n, 4);
    if (sl == 0 && k < rows) njt[k] = n;
  }
}

// raw pairs = sum over A tiles of B tile-row lengths (pipeline.cpp:52-58);
// filtered = pairs passing tile_product_nonzero (pipeline.cpp:23-35): a
// single-column A tile passes exactly the tiles its B row touches (njt);
// others test B's row occupancies.  Warp per 32 A tiles.
constexpr uint32_t kPairBits = 8192;  // tile ranks of a B tile row the pair-statistics bitmap covers

// Per B tile row k, rinfo[k] = its occupied rows (lo16: rows with a kept
// entry) | kSingleRows when every tile occupies exactly one row (R-MAT's
// ~1-entry tiles).  The tiles of row k with row x occupied are the distinct
// tiles CSR row 16 k + x touches, njt[16 k + x]; so an A tile with column
// occupancy c passes
//   all len tiles        when c covers every occupied row,
//   none                 when it meets none,
//   sum_{x in c} njt     when the tiles are single-row.
// Warp per tile row.
constexpr uint32_t kSingleRows = 1u << 16;

// row occupancy of B's tile b (a converted B's tco, or a B summary's ro)
__device__ __forceinline__ uint32_t tile_ro(const TileMat& B, uint32_t b) {
  return B.ro16 ? uint32_t(__ldg(B.ro16 + b)) : __ldg(&B.tco[b].y) >> 16;
}

__global__ void __launch_bounds__(256) esc_brow_bits_kernel(TileMat B, uint32_t* __restrict__ rinfo) {
  const int lane = threadIdx.x & 31;
  const uint32_t k = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (k >= B.tile_rows) return;
  const uint32_t b0 = B.trp[k], b1 = B.trp[k + 1];
  uint32_t rows = 0;
  bool one = true;
  for (uint32_t b = b0 + lane; b < b1; b += 32) {
    const uint32_t ro = tile_ro(B, b);
    one &= __popc(ro) == 1;
    rows |= ro;
  }
  rows = __reduce_or_sync(kFull, rows);
  const bool all = __all_sync(kFull, one);
  if (lane == 0) rinfo[k] = rows | (all ? kSingleRows : 0u);
}

// The B tiles of tile row k meeting column occupancy c (an A tile with several
// occupied columns, B tiles with several occupied rows).  Long B tile rows
// (R-MAT hubs): the union of the tiles the occupied B CSR rows touch, as a
// bitmap over the tile row's tile ranks (B tile (k, J) has row kk occupied iff
// CSR row 16 k + kk keeps an entry in tile J, whose etile is J's rank); short
// ones: the occupancy test over the tile row.  Warp-collective; bm: the warp's
// kPairBits-bit scratch.
__device__ __forceinline__ uint32_t meets_count(const TileMat& B, uint32_t k, uint32_t c, uint32_t* bm, int lane) {
  const uint32_t b0 = __ldg(B.trp + k), b1 = __ldg(B.trp + k + 1), len = b1 - b0;
  uint32_t entries = 0;
  for (uint32_t ci = c; ci; ci &= ci - 1u) {
    const int64_t row = int64_t(k) * 16 + (__ffs(ci) - 1);
    if (row < B.rows) entries += uint32_t(__ldg(B.csr_rp + row + 1) - __ldg(B.csr_rp + row));
  }
  uint32_t n = 0;
  if (len <= kPairBits && entries < len) {
    for (uint32_t i = lane; i < (len + 31) / 32; i += 32) bm[i] = 0;
    __syncwarp();
    for (uint32_t ci = c; ci; ci &= ci - 1u) {
      const int64_t row = int64_t(k) * 16 + (__ffs(ci) - 1);
      if (row >= B.rows) continue;
      const int64_t e1 = __ldg(B.csr_rp + row + 1);
      for (int64_t e = __ldg(B.csr_rp + row) + lane; e < e1; e += 32) {
        const uint32_t et = __ldg(B.etile + e);
        if (et != kNoTile) {
          const uint32_t t = et & ~kDupEntry;
          if (t < len) atomicOr(&bm[t >> 5], 1u << (t & 31));  // (a summary from another B cannot write past bm)
        }
      }
    }
    __syncwarp();
    for (uint32_t i = lane; i < (len + 31) / 32; i += 32) n += __popc(bm[i]);
    __syncwarp();
  } else {
    for (uint32_t b = b0 + lane; b < b1; b += 32) n += (tile_ro(B, b) & c) != 0u;
  }
  return __reduce_add_sync(kFull, n);
}

// Thread per A tile (warp per 32): raw pairs, and the filtered pairs of the
// cheap cases; the warp counts its A tiles that need meets_count together.
#ifndef TSG_PS_TILES
#define TSG_PS_TILES 2
#endif
constexpr int kPsTiles = TSG_PS_TILES;  // A tiles per lane (their gathers in flight together)

__global__ void __launch_bounds__(256) esc_pairstats_kernel(TileMat A, TileMat B, uint32_t tA,
                                                           const uint32_t* __restrict__ njt,
                                                           const uint32_t* __restrict__ rinfo,
                                                           unsigned long long* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint32_t a0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 32 * kPsTiles;
  if (a0 >= tA) return;
  unsigned long long raw = 0, filt = 0;
  uint32_t K[kPsTiles], co[kPsTiles], b0[kPsTiles], b1[kPsTiles], info[kPsTiles];
  unsigned multi = 0;  // bit q: tile q of this lane needs meets_count
  // (1) every gather of the lane's tiles in flight together
#pragma unroll
  for (int q = 0; q < kPsTiles; ++q) {
    const uint32_t a = a0 + 32u * q + lane;
    K[q] = 0;
    co[q] = 0;
    if (a < tA) {
      const uint2 t = __ldg(A.tco + a);
      K[q] = t.x;
      co[q] = t.y & 0xffffu;
    }
  }
#pragma unroll
  for (int q = 0; q < kPsTiles; ++q) {
    const bool in = co[q] != 0u;
    b0[q] = in ? __ldg(B.trp + K[q]) : 0u;
    b1[q] = in ? __ldg(B.trp + K[q] + 1) : 0u;
    info[q] = in && __popc(co[q]) > 1 ? __ldg(rinfo + K[q]) : 0u;
  }
  // (2) raw pairs and the cheap filtered cases
#pragma unroll
  for (int q = 0; q < kPsTiles; ++q) {
    const uint32_t r = b1[q] - b0[q];
    raw += r;
    if (co[q] == 0u || r == 0u) continue;
    if (__popc(co[q]) == 1) {
      const int64_t row = int64_t(K[q]) * 16 + (__ffs(co[q]) - 1);
      filt += row < B.rows ? __ldg(njt + row) : 0u;
    } else {
      const uint32_t rm = info[q] & 0xffffu;
      if ((co[q] & rm) == rm) {  // every tile has an occupied row, all of them inside c
        filt += r;
      } else if (co[q] & rm) {
        if (info[q] & kSingleRows) {
          for (uint32_t c = co[q] & rm; c; c &= c - 1u) filt += __ldg(njt + size_t(K[q]) * 16 + (__ffs(c) - 1));
        } else {
          multi |= 1u << q;
        }
      }
    }
  }
  __shared__ uint32_t s_bm[8][kPairBits / 32];
#pragma unroll
  for (int q = 0; q < kPsTiles; ++q) {
    for (unsigned m = __ballot_sync(kFull, (multi >> q) & 1u); m; m &= m - 1) {
      const int src = __ffs(m) - 1;
      const uint32_t n = meets_count(B, __shfl_sync(kFull, K[q], src), __shfl_sync(kFull, co[q], src),
                                     s_bm[threadIdx.x >> 5], lane);
      if (lane == src) filt += n;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    raw += __shfl_xor_sync(kFull, raw, o);
    filt += __shfl_xor_sync(kFull, filt, o);
  }
  if (lane == 0) {
    if (raw) atomicAdd(out, raw);
    if (filt) atomicAdd(out + 1, filt);
  }
}

// A converted panel's tile counts per tile row and row occupancy per tile (tsg_bsum)
__global__ void bsum_tiles_kernel(TileMat B, uint64_t tiles, uint32_t* __restrict__ tile_count,
                                  uint16_t* __restrict__ ro) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < tiles; i += stride)
    ro[i] = uint16_t(__ldg(&B.tco[i].y) >> 16);
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < B.tile_rows; k += stride)
    tile_count[k] = B.trp[k + 1] - B.trp[k];
}

// ---------------------------------------------------------------- chained A
// A chained stage's A arrives as A-role tiles (the previous stage's emitted
// output, tsg_panel.cu emit_tile); the general path reads CSR.  Warp per tile
// row, lane r < 16 = row r walks the row's tiles in column order.
__device__ __forceinline__ uint32_t tile_row_mask(const TileMat& A, uint32_t t, int r) {
  return (__ldg(A.rm2 + size_t(t) * 8 + (r & 7)) >> (16 * (r >> 3))) & 0xffffu;
}

__global__ void __launch_bounds__(256) tiles_rowcount_kernel(TileMat A, int64_t* __restrict__ rowcnt) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= A.tile_rows || lane >= 16) return;
  uint32_t n = 0;
  for (uint32_t t = A.trp[I]; t < A.trp[I + 1]; ++t) n += __popc(tile_row_mask(A, t, lane));
  const int64_t row = int64_t(I) * 16 + lane;
  if (row < A.rows) rowcnt[row] = n;
}

__global__ void __launch_bounds__(256) tiles_to_csr_kernel(TileMat A, const int64_t* __restrict__ rp,
                                                          int32_t* __restrict__ col, uint16_t* __restrict__ h16) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (I >= A.tile_rows || lane >= 16) return;
  const int64_t row = int64_t(I) * 16 + lane;
  if (row >= A.rows) return;
  int64_t p = rp[row];
  for (uint32_t t = A.trp[I]; t < A.trp[I + 1]; ++t) {
    uint32_t m = tile_row_mask(A, t, lane);
    if (!m) continue;
    const uint32_t J = __ldg(&A.tco[t].x);
    const uint2 mt = __ldg(A.meta[kRoleA] + t);
    for (; m; m &= m - 1u) {
      const int cc = __ffs(m) - 1;
      int L, j;
      slot_of(kRoleA, lane, cc, L, j);
      const uint4 ch = __ldg(A.chunk[kRoleA] + ((mt.x >> L) & 1u ? mt.y + __popc(mt.x & ((1u << L) - 1u)) : 0u));
      const uint32_t wd = (j >> 1) == 0 ? ch.x : (j >> 1) == 1 ? ch.y : (j >> 1) == 2 ? ch.z : ch.w;
      col[p] = int32_t(J * 16u + uint32_t(cc));
      h16[p] = uint16_t(wd >> (16 * (j & 1)));
      ++p;
    }
  }
}

bool allow_groups(const EscArgs& g) { return (g.colsB + 15) / 16 <= (int64_t(1) << 20); }

}  // namespace

size_t esc_smem_bytes() { return sizeof(EscSmem); }

void launch_esc_brec(const EscArgs& g, int64_t rowsB, uint4* brec, cudaStream_t st) {
  if (rowsB > 0)
    esc_brec_kernel<<<unsigned(std::min<int64_t>((rowsB + 255) / 256, 4096)), 256, 0, st>>>(rowsB, g.rpB, g.colB,
                                                                                            brec);
}

void launch_esc_hist(const EscArgs& g, int64_t nnzA, int64_t rowsB, uint32_t* colcnt, unsigned long long* hist,
                     cudaStream_t st) {
  if (nnzA > 0) esc_colcount_kernel<<<1184, 256, 0, st>>>(nnzA, g.colA, g.hA, colcnt);
  if (rowsB > 0) esc_colhist_kernel<<<2368, 256, 0, st>>>(rowsB, g.rpB, g.colB, g.hB, colcnt, hist);
}

void launch_esc_plan_prod(const EscArgs& g, unsigned long long* prod, unsigned long long* total, cudaStream_t st) {
  if (g.tile_rows == 0) return;
  esc_plan_prod_kernel<<<(g.tile_rows + 7) / 8, 256, 0, st>>>(g.rowsA, g.tile_rows, g.rpA, g.colA, g.hA, g.brec,
                                                              prod, total);
}

void launch_esc_plan_group(const EscArgs& g, const unsigned long long* pre, uint32_t* nrec, uint32_t* nwk,
                           cudaStream_t st) {
  if (g.tile_rows == 0) return;
  const uint32_t max_chunks = uint32_t(std::max<int64_t>(1, std::min<int64_t>((g.colsB + 15) / 16, 1 << 30)));
  esc_plan_group_kernel<<<(g.tile_rows + 255) / 256, 256, 0, st>>>(g.tile_rows, pre, allow_groups(g), max_chunks,
                                                                   g.target, nrec, nwk);
}

void launch_esc_plan_fill(const EscArgs& g, const unsigned long long* pre, const uint32_t* nwk, const uint32_t* wbase,
                          const unsigned long long* G, uint4* units, cudaStream_t st) {
  if (g.tile_rows == 0) return;
  esc_plan_fill_kernel<<<(g.tile_rows + 7) / 8, 256, 0, st>>>(g.tile_rows, g.colsB, pre, allow_groups(g), nwk, wbase,
                                                              G, units);
}

void launch_esc(const EscArgs& g, int device, cudaStream_t st) {
  // resident CTAs per SM: 3 (80 registers) or 4 (64 registers; TSG_ESC_MINB=4)
  static int per_sm[16][2] = {}, sms[16] = {0};
  // 256 threads: 3 CTAs/SM (80 registers) or 4 (TSG_ESC_MINB=4, 64 registers);
  // 512 threads: 2 CTAs/SM (64 registers) or 3 (TSG_ESC_MINB=3)
  constexpr int kB0 = kNT == 512 ? 2 : 3;
  const int d = device & 15, v = tuning_variant("TSG_ESC_MINB", kB0) == kB0 + 1 ? 1 : 0;
  auto k = v ? esc_kernel<kB0 + 1> : esc_kernel<kB0>;
  const size_t smem = sizeof(EscSmem);
  if (!per_sm[d][v]) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kNT, smem);
    cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, device);
    per_sm[d][v] = std::max(1, n);
  }
  k<<<unsigned(per_sm[d][v] * sms[d]), kNT, smem, st>>>(g);
#ifdef TSG_ESC_DIAG
  unsigned long long h[16];
  cudaStreamSynchronize(st);
  cudaMemcpyFromSymbol(h, g_esc_diag, sizeof(h));
  std::fprintf(stderr, "esc_diag leaves %llu products %llu slots %llu pass_slots %llu nb1 %llu dense %llu halve %llu units %llu ipt4 %llu ipt8 %llu ipt16 %llu grp_products %llu\n",
               h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9], h[10], h[11]);
  const unsigned long long z[16] = {};
  cudaMemcpyToSymbol(g_esc_diag, z, sizeof(z));
#endif
}

void launch_esc_rowcount(const EscArgs& g, const uint32_t* base, int64_t* rowcnt, cudaStream_t st, uint32_t I0,
                         uint32_t I1) {
  if (I1 == 0) I1 = g.tile_rows;
  if (I1 <= I0) return;
  esc_rowcount_kernel<<<(I1 - I0 + 7) / 8, 256, 0, st>>>(g.rowsA, I1, base, g.pieces, rowcnt, I0);
}

void launch_esc_copy_records(const EscArgs& g, uint32_t rec0, uint32_t rec1, const int64_t* row_ptr, int32_t* col,
                             float* val, cudaStream_t st) {
  if (rec1 <= rec0) return;
  const unsigned blocks = std::min<unsigned>((rec1 - rec0 + 7) / 8, 148u * 16u);
  esc_copy_records_kernel<<<blocks, 256, 0, st>>>(rec0, rec1, g.pieces, g.stage, row_ptr, col, val);
}

void launch_esc_copy(const EscArgs& g, const int64_t* row_ptr, int32_t* col, float* val, cudaStream_t st) {
  esc_copy_kernel<<<148 * 16, 256, 0, st>>>(g.nrec, g.piece_top, g.pool_cap, g.pieces, g.stage, row_ptr, col, val);
}

void launch_esc_bsummary(const TileMat& B, uint32_t* njt, uint32_t* rinfo, cudaStream_t st) {
  if (B.rows > 0) esc_njt_kernel<<<2368, 256, 0, st>>>(B.rows, B.csr_rp, B.etile, njt);
  if (B.tile_rows > 0) esc_brow_bits_kernel<<<(B.tile_rows + 7) / 8, 256, 0, st>>>(B, rinfo);
}

void launch_esc_pairstats(const TileMat& A, const TileMat& B, uint64_t tA, const uint32_t* njt, const uint32_t* rinfo,
                          unsigned long long* out, cudaStream_t st) {
  if (tA > 0)
    esc_pairstats_kernel<<<unsigned((tA + 256 * kPsTiles - 1) / (256 * kPsTiles)), 256, 0, st>>>(A, B, uint32_t(tA), njt,
                                                                                                rinfo, out);
}

void launch_bsum_tiles(const TileMat& B, uint64_t tiles, uint32_t* tile_count, uint16_t* ro, cudaStream_t st) {
  if (tiles == 0 && B.tile_rows == 0) return;
  bsum_tiles_kernel<<<1184, 256, 0, st>>>(B, tiles, tile_count, ro);
}

void launch_tiles_rowcount(const TileMat& A, int64_t* rowcnt, cudaStream_t st) {
  if (A.tile_rows == 0) return;
  tiles_rowcount_kernel<<<(A.tile_rows + 7) / 8, 256, 0, st>>>(A, rowcnt);
}

void launch_tiles_to_csr(const TileMat& A, const int64_t* rp, int32_t* col, uint16_t* h16, cudaStream_t st) {
  if (A.tile_rows == 0) return;
  tiles_to_csr_kernel<<<(A.tile_rows + 7) / 8, 256, 0, st>>>(A, rp, col, h16);
}

}  // namespace tsg
