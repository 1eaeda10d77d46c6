// tsg_convert.cu -- subsystem (1): CSR -> 16x16 tiled bitmap format.
//
// GPU restatement of from_element_coo(m, Fp16Stored)
// (proj/src/tile_format.cpp:61-129) at T = 16:
//   * validation of the COO/CSR invariant        tile_format.cpp:34-51
//   * non-finite -> OverflowError (or dropped)   tile_format.cpp:82-86
//   * exact zero dropped                         tile_format.cpp:87
//   * round_to_half (RNE, |x| > 65504 throws)    tile_format.cpp:89-90, half.cpp:12-36
//   * values that round to zero dropped          tile_format.cpp:98
//   * tiles keyed (tile_row, tile_col), slots in-tile, tiles sorted
//     (the std::sort at tile_format.cpp:106-110 is replaced by a 16-way
//      merge across the rows of a tile row: CSR rows are already sorted).
//
// One warp per tile row (16 CSR rows), one pass, no host synchronisation:
// every array is sized by nnz (a tile row never holds more tiles or chunks
// than entries), so tile row I writes its tiles at gapped slots starting at
// row_ptr[16 I]; a scan of the per-tile-row counts and tiles_compact_kernel
// give the dense CSR-of-tiles afterwards.  Per tile row: the fast path ranks
// tile columns with a shared-memory bitmap (or, when the panel is wide or has
// many tiles, merges its 16 already-sorted row runs), builds the 256-bit
// masks with shared-memory atomics and stores each fp16 value straight into
// its lane-dense operand chunk (A order and/or B order, tsg_common.cuh);
// panels of 512-8192 entries in a general call take convert_hub_kernel (a CTA
// bitmap over the tile columns), the rest the 16-way merge walk, one tile at
// a time.
#include <algorithm>
#include <type_traits>

#include "tsg_kernels.cuh"

namespace tsg {

namespace {

// Single-step RNE double -> binary16 (no double rounding through float).
__device__ __forceinline__ unsigned short f64_to_half_bits(double x) {
  unsigned short h;
  asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(x));
  return h;
}

// Loads value p as binary16 bits (kDtype: 0 f16 bits, 1 f32, 2 f64).  Sets
// kErrOverflow on |x| > 65504 or non-finite input (unless dropped); `keep`
// is false when the entry is dropped (zero, underflow, dropped non-finite).
template <int kDtype>
__device__ __forceinline__ unsigned short load_half(const void* val, int64_t p,
                                                    bool drop_nonfinite, unsigned& err,
                                                    bool& keep) {
  unsigned short h = 0;
  keep = false;
  if (kDtype == 1) {
    const float x = __ldg(static_cast<const float*>(val) + p);
    if (!isfinite(x)) {
      if (!drop_nonfinite) err |= kErrOverflow;
      return 0;
    }
    if (fabsf(x) > 65504.0f) {
      err |= kErrOverflow;
      return 0;
    }
    h = __half_as_ushort(__float2half_rn(x));
  } else if (kDtype == 2) {
    const double x = __ldg(static_cast<const double*>(val) + p);
    if (!isfinite(x)) {
      if (!drop_nonfinite) err |= kErrOverflow;
      return 0;
    }
    if (fabs(x) > 65504.0) {
      err |= kErrOverflow;
      return 0;
    }
    h = f64_to_half_bits(x);
  } else {
    h = __ldg(static_cast<const unsigned short*>(val) + p);
    if ((h & 0x7c00u) == 0x7c00u) {  // inf / nan
      if (!drop_nonfinite) err |= kErrOverflow;
      return 0;
    }
  }
  keep = (h & 0x7fffu) != 0;  // exact zero or underflow-to-(+-)0 dropped
  return h;
}

// load_half on an already loaded value (same checks and rounding).
template <int kDtype, class Raw>
__device__ __forceinline__ unsigned short raw_to_half(Raw x, bool drop_nonfinite, unsigned& err, bool& keep) {
  unsigned short h = 0;
  keep = false;
  if constexpr (kDtype == 0) {
    h = x;
    if ((h & 0x7c00u) == 0x7c00u) {  // inf / nan
      if (!drop_nonfinite) err |= kErrOverflow;
      return 0;
    }
  } else {
    if (!isfinite(x)) {
      if (!drop_nonfinite) err |= kErrOverflow;
      return 0;
    }
    if (fabs(double(x)) > 65504.0) {
      err |= kErrOverflow;
      return 0;
    }
    if constexpr (kDtype == 1)
      h = __half_as_ushort(__float2half_rn(x));
    else
      h = f64_to_half_bits(x);
  }
  keep = (h & 0x7fffu) != 0;  // exact zero or underflow-to-(+-)0 dropped
  return h;
}

constexpr int kBitW = 256;  // fast path: bitmap words (panels spanning <= 8192 tile columns)
constexpr int kFastT = 64;  // fast path: tiles per panel
constexpr int kFastU = 16;  // fast path: entries per lane (panels of <= 512 entries)

// Output of the conversion kernels before compaction: tile row I's tiles at
// slots [E0, E0 + n) with E0 = its first CSR entry (a panel never holds more
// tiles than entries), chunks from 1 + E0 per role; the dense CSR-of-tiles
// arrays are derived from rm2 + rec by tiles_compact_kernel.
struct Gapped {
  uint32_t* rm2 = nullptr;
  uint4* rec[2] = {nullptr, nullptr};  // {lane mask, first chunk, occupancy, tile col}
  uint4* chunk[2] = {nullptr, nullptr};
  uint32_t* etile = nullptr;  // per entry: tile rank within its tile row | kDupEntry, or kNoTile
  uint16_t* h16 = nullptr;    // per entry: rounded binary16 value, 0 when dropped
  uint32_t* ntiles = nullptr;  // per tile row
  uint8_t* mark = nullptr;     // optional: mark[J] = 1 for every tile column J (the B tile rows A needs)
  // "general" flag: set by the A-role conversion when a tile row has more than
  // kLightMax tiles -- the call then takes the general path, which reads no
  // operand chunks, 256-bit masks or lane metadata, so every tile row that sees
  // it writes only what the general path reads (tile columns, occupancy,
  // etile, h16)
  unsigned* general = nullptr;
  bool may_set = false;        // this conversion is A's (its tile rows decide the path)
};

constexpr uint32_t kLightMax = 128;  // the light path's largest tile row (tsg_api.cu decide())

// the role whose records a lite (general-call) conversion writes and the compaction reads
__device__ __forceinline__ int lite_role(int roles) { return (roles & 1) ? 0 : 1; }

__device__ __forceinline__ void mark_column(const Gapped& out, uint32_t J) {
  if (out.mark && !out.mark[J]) out.mark[J] = 1;  // most tiles share their column's flag: skip the store
}

// The general flag as a tile row starts (read early: its latency overlaps the
// row's loads) ...
__device__ __forceinline__ bool general_seen(const Gapped& out) {
  return out.general && *reinterpret_cast<volatile unsigned*>(out.general) != 0u;
}
// ... and once its tile count is known: true when the call is general (this row
// of A has more than kLightMax tiles, or the flag was already set)
__device__ __forceinline__ bool general_call(const Gapped& out, uint32_t ntiles, bool seen) {
  if (!out.general) return false;
  if (out.may_set && ntiles > kLightMax) {
    atomicOr(out.general, 1u);
    return true;
  }
  return seen;
}

// Tile-slot (r, c) of a 16x16 tile -> its lane and fp16 position in the
// lane's 16-byte chunk.  A order: lane (g, t) holds rows g, g+8 x cols 2t,
// 2t+1, 2t+8, 2t+9 in regs i = (r>>3) + 2(c>>3).  B order (the transposed
// tile, regs stored {0, 2, 1, 3}): lane (c&7, (r&7)>>1), word
// 2(c>>3) + (r>>3), half r&1.
__device__ __forceinline__ void slot_lane(int role, int r, int c, int& L, int& h16) {
  if (role == kRoleA) {
    L = (r & 7) * 4 + ((c & 7) >> 1);
    h16 = 2 * ((r >> 3) + 2 * (c >> 3)) + (c & 1);
  } else {
    L = (c & 7) * 4 + ((r & 7) >> 1);
    h16 = 2 * (2 * (c >> 3) + (r >> 3)) + (r & 1);
  }
}

struct __align__(16) FastSmem {  // 16-byte multiple: the tiles use 16-byte accesses
  uint8_t row[32 * kFastU];  // row of each entry of the panel
  union {
    struct {                    // bitmap path
      uint32_t bits[kBitW];     // tile-column bitmap of the panel
      uint16_t pre[kBitW];      // tiles before each bitmap word
      uint32_t rm[kFastT][8];   // per tile: word g = row g | row g+8 << 16
      uint32_t lm[kFastT][2];   // per tile and role: lane presence mask
      uint2 cl[kFastT][2];      // per tile and role: {first chunk, lane mask}
    };
    struct {                              // sort path
      unsigned long long items[32 * kFastU];  // (tile col, row, col, entry, fp16) sorted
      uint16_t ts[32 * kFastU + 1];       // first item of each tile
      uint32_t bnd[kTile + 1];            // first item of each row (runs of the merge)
    };
  };
};

// Sort path for panels the bitmap cannot rank (wider than 8192 tile columns,
// or more than kFastT tiles: R-MAT, the rectangular products): the panel's
// kept entries, as 64-bit items (tile col << 40 | row << 36 | col & 15 << 32
// | entry << 16 | fp16), arrive in CSR order -- 16 runs (the rows), each
// already sorted because a CSR row is -- and four levels of pairwise
// merge-path merges in shared memory order them; runs of equal tile column
// are the tiles, in (row, col) order inside; lanes then emit one tile each.
//
// One merge level: lane l produces outputs [l S, l S + S) (S = ceil(nk/32)
// <= 16) of the runs' pairwise merges, in registers -- a merge-path search
// finds where its first output comes from, then S sequential steps -- and
// writes them back in place once the warp has read the level.
__device__ __forceinline__ void merge_rows(unsigned long long* it, const uint32_t* bnd, uint32_t nk, int lane) {
  const uint32_t S = (nk + 31u) >> 5;
  const uint32_t q0 = min(nk, uint32_t(lane) * S), q1 = min(nk, q0 + S);
  for (int w = 1; w < kTile; w <<= 1) {
    unsigned long long o[kFastU];
    uint32_t ia = 0, ib = 0, am = 0, be = 0;
    unsigned long long va = ~0ull, vb = ~0ull;
    if (q0 < q1) {
      int p = 0;  // the pair of runs (p .. p+w-1, p+w .. p+2w-1) holding output q0
      while (bnd[p + 2 * w] <= q0) p += 2 * w;
      const uint32_t a = bnd[p];
      am = bnd[p + w];
      be = bnd[p + 2 * w];
      const uint32_t d = q0 - a, la = am - a, lb = be - am;
      uint32_t lo = d > lb ? d - lb : 0u, hi = min(d, la);
      while (lo < hi) {  // outputs before q0 take lo items of the first run (keys are distinct)
        const uint32_t m = (lo + hi) >> 1;
        if (it[a + m] < it[am + d - 1u - m])
          lo = m + 1u;
        else
          hi = m;
      }
      ia = a + lo;
      ib = am + (d - lo);
      va = ia < am ? it[ia] : ~0ull;
      vb = ib < be ? it[ib] : ~0ull;
      while (q0 == be) {  // (empty pair ends) the next non-empty pair
        p += 2 * w;
        ia = bnd[p];
        am = ib = bnd[p + w];
        be = bnd[p + 2 * w];
        va = ia < am ? it[ia] : ~0ull;
        vb = ib < be ? it[ib] : ~0ull;
      }
      int pp = p;
#pragma unroll
      for (int s2 = 0; s2 < kFastU; ++s2) {
        const uint32_t q = q0 + uint32_t(s2);
        if (q < q1) {
          while (q == be) {  // this pair is done: the next one starts at its beginning
            pp += 2 * w;
            ia = bnd[pp];
            am = ib = bnd[pp + w];
            be = bnd[pp + 2 * w];
            va = ia < am ? it[ia] : ~0ull;
            vb = ib < be ? it[ib] : ~0ull;
          }
          if (va < vb) {
            o[s2] = va;
            ++ia;
            va = ia < am ? it[ia] : ~0ull;
          } else {
            o[s2] = vb;
            ++ib;
            vb = ib < be ? it[ib] : ~0ull;
          }
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int s2 = 0; s2 < kFastU; ++s2)
      if (q0 + uint32_t(s2) < q1) it[q0 + s2] = o[s2];
    __syncwarp();
  }
}

__device__ __forceinline__ uint32_t sparse_panel(FastSmem& sm, const Gapped& out, int roles, int64_t E0, uint32_t E,
                                                 uint32_t nk, int lane, bool seen) {
  unsigned long long* it = sm.items;
  // run starts: the kept items are in CSR order, so row r's run begins at the
  // first item whose row is >= r
  if (lane <= kTile) {
    uint32_t lo = 0, hi = nk;
    while (lo < hi) {
      const uint32_t m = (lo + hi) >> 1;
      if (((it[m] >> 36) & 15u) < uint32_t(lane))
        lo = m + 1u;
      else
        hi = m;
    }
    sm.bnd[lane] = lane == kTile ? nk : lo;
  }
  __syncwarp();
  merge_rows(it, sm.bnd, nk, lane);
  // tile starts -> tile ranks; etile (first kept entry of each (row, tile))
  uint32_t ntiles = 0;
  const unsigned lt = lanemask_lt();
  for (uint32_t i0 = 0; i0 < nk; i0 += 32) {
    const uint32_t i = i0 + lane;
    const unsigned long long x = i < nk ? it[i] : ~0ull;
    const unsigned long long xp = i > 0 && i < nk ? it[i - 1] : ~0ull;
    const bool start = i < nk && (i == 0 || (x >> 40) != (xp >> 40));
    const unsigned sb = __ballot_sync(kFull, start);
    const uint32_t t = ntiles + __popc(sb & lt) + (start ? 1u : 0u) - 1u;  // tile of item i
    if (start) sm.ts[t] = uint16_t(i);
    if (i < nk && out.etile) {
      const bool first_row = start || ((x >> 36) & 15u) != ((xp >> 36) & 15u);
      out.etile[E0 + ((x >> 16) & 0xffffu)] = t | (first_row ? 0u : kDupEntry);
    }
    ntiles += __popc(sb);
  }
  if (lane == 0) sm.ts[ntiles] = uint16_t(nk);
  const bool lite = __shfl_sync(kFull, lane == 0 ? general_call(out, ntiles, seen) : false, 0);
  __syncwarp();
  if (lite) {  // the general path reads only each tile's column and occupancy
    for (uint32_t t = lane; t < ntiles; t += 32) {
      const uint32_t a = sm.ts[t], b = sm.ts[t + 1];
      const uint32_t J = uint32_t(it[a] >> 40);
      uint32_t co = 0, ro = 0;
      for (uint32_t i = a; i < b; ++i) {
        const unsigned long long x = it[i];
        ro |= 1u << uint32_t((x >> 36) & 15u);
        co |= 1u << uint32_t((x >> 32) & 15u);
      }
      mark_column(out, J);
      out.rec[lite_role(roles)][E0 + t] = make_uint4(0u, 0u, co | (ro << 16), J);
    }
    return ntiles;
  }
  // lanes emit tiles t = lane, lane + 32, ...; chunk bases by a warp scan
  uint32_t runA = 1u + uint32_t(E0), runB = 1u + uint32_t(E0);
  for (uint32_t t0 = 0; t0 < ntiles; t0 += 32) {
    const uint32_t t = t0 + lane;
    uint32_t rm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t lmA = 0, lmB = 0, a = 0, b = 0, J = 0;
    if (t < ntiles) {
      a = sm.ts[t];
      b = sm.ts[t + 1];
      J = uint32_t(it[a] >> 40);
      for (uint32_t i = a; i < b; ++i) {
        const unsigned long long x = it[i];
        const int r = int(x >> 36) & 15, cc = int(x >> 32) & 15;
#pragma unroll
        for (int g = 0; g < 8; ++g)
          if (g == (r & 7)) rm[g] |= 1u << (cc + 16 * (r >> 3));
        int L, h16;
        slot_lane(kRoleA, r, cc, L, h16);
        lmA |= 1u << L;
        slot_lane(kRoleB, r, cc, L, h16);
        lmB |= 1u << L;
      }
    }
    const uint32_t nA = (roles & 1) ? __popc(lmA) : 0u, nB = (roles & 2) ? __popc(lmB) : 0u;
    uint32_t iA = nA, iB = nB;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t va = __shfl_up_sync(kFull, iA, o), vb = __shfl_up_sync(kFull, iB, o);
      if (lane >= o) {
        iA += va;
        iB += vb;
      }
    }
    const uint32_t cbA = runA + iA - nA, cbB = runB + iB - nB;
    runA += __shfl_sync(kFull, iA, 31);
    runB += __shfl_sync(kFull, iB, 31);
    if (t < ntiles) {
      uint32_t colocc = 0, rowocc = 0;
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        colocc |= rm[g] | (rm[g] >> 16);
        rowocc |= ((rm[g] & 0xffffu) != 0u ? 1u << g : 0u) | ((rm[g] >> 16) != 0u ? 1u << (g + 8) : 0u);
      }
      const uint32_t occ = (colocc & 0xffffu) | (rowocc << 16);
      mark_column(out, J);
      uint4* dst = reinterpret_cast<uint4*>(out.rm2 + size_t(E0 + t) * 8);
      dst[0] = make_uint4(rm[0], rm[1], rm[2], rm[3]);
      dst[1] = make_uint4(rm[4], rm[5], rm[6], rm[7]);
#pragma unroll
      for (int role = 0; role < 2; ++role) {
        if (!(roles & (1 << role))) continue;
        const uint32_t lm = role == kRoleA ? lmA : lmB, cb = role == kRoleA ? cbA : cbB;
        out.rec[role][E0 + t] = make_uint4(lm, cb, occ, J);
        uint32_t n = 0;
        for (uint32_t m = lm; m; m &= m - 1u, ++n) {  // present lanes, ascending
          const int Lw = __ffs(m) - 1;
          uint32_t w[4] = {0, 0, 0, 0};
          for (uint32_t i = a; i < b; ++i) {
            const unsigned long long x = it[i];
            int L, h16;
            slot_lane(role, int(x >> 36) & 15, int(x >> 32) & 15, L, h16);
            if (L != Lw) continue;
            const uint32_t hv = uint32_t(x & 0xffffu) << (16 * (h16 & 1));
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q == (h16 >> 1)) w[q] |= hv;
          }
          out.chunk[role][cb + n] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
  }
  return ntiles;
}


// Fast path, warp per tile row (panel): the panel's entries are loaded once
// (coalesced, up to kFastU per lane, kept in registers); their tile columns
// are marked in a bitmap whose prefix popcounts rank the tiles; shared-memory
// atomics build each tile's 256-bit mask and lane presence masks; a prefix
// over the tiles gives the chunk bases; the chunk ranges are zeroed and
// every entry stores its fp16 value at its chunk slot.  Panels outside the
// limits go to the walk list.
template <int kDtype>
#ifndef TSG_CONV_MINB
#define TSG_CONV_MINB 4
#endif
__global__ void __launch_bounds__(256, TSG_CONV_MINB) convert_fast_kernel(CsrView in, uint32_t tile_rows, Gapped out, int roles,
                                                          uint32_t* __restrict__ walk_list,
                                                          uint32_t* __restrict__ walk_count,
                                                          unsigned* __restrict__ err_flag, int drop_nonfinite,
                                                          const uint8_t* __restrict__ needed) {
  __shared__ __align__(16) FastSmem smem[8];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // the scan's tail and the zero chunk of each role
    out.ntiles[tile_rows] = 0;
    if (roles & 1) out.chunk[kRoleA][0] = make_uint4(0, 0, 0, 0);
    if (roles & 2) out.chunk[kRoleB][0] = make_uint4(0, 0, 0, 0);
  }
  const uint32_t I = blockIdx.x * 8 + wib;
  if (I >= tile_rows) return;
  if (*err_flag & kErrRowPtr) {  // malformed row pointers (validate_rowptr_kernel): no tiles, no reads
    if (lane == 0) out.ntiles[I] = 0;
    return;
  }
  FastSmem& sm = smem[wib];
  const bool seen = lane == 0 && general_seen(out);
  const int64_t r0 = int64_t(I) * kTile, r1 = r0 + kTile < in.rows ? r0 + kTile : in.rows;
  const int64_t row = r0 + lane;
  const bool has_row = lane < kTile && row < in.rows;
  const int64_t p = has_row ? in.row_ptr[row] : 0;
  const int64_t end = has_row ? in.row_ptr[row + 1] : 0;
  const int64_t E0 = in.row_ptr[r0], E1 = in.row_ptr[r1];
  const bool rows_ok = __all_sync(kFull, !has_row || (end >= p && p >= E0 && end <= E1));
  if (!rows_ok || E1 - E0 > 32 * kFastU || E1 < E0) {  // the walk (it validates an unreferenced panel too)
    if (lane == 0) walk_list[atomicAdd(walk_count, 1u)] = I;
    return;
  }
  const uint32_t E = uint32_t(E1 - E0);
  // every load of the panel in flight at once: columns and raw values
  int32_t c[kFastU];
  using Raw = typename std::conditional<kDtype == 2, double, typename std::conditional<kDtype == 1, float,
                                                                                      unsigned short>::type>::type;
  Raw v[kFastU];
#pragma unroll
  for (int u = 0; u < kFastU; ++u) {
    c[u] = -1;
    v[u] = Raw(0);
  }
#pragma unroll
  for (int u = 0; u < kFastU; ++u) {
    if (32u * u >= E) break;
    const uint32_t q = 32 * u + lane;
    if (q < E) {
      c[u] = __ldg(in.col + E0 + q);
      v[u] = __ldg(static_cast<const Raw*>(in.val) + E0 + q);
    }
  }
  const bool skip = needed && !needed[I];
  uint32_t jlo = 0xffffffffu, jhi = 0;
#pragma unroll
  for (int u = 0; u < kFastU; ++u) {
    if (32u * u >= E) break;
    if (c[u] >= 0) {
      jlo = min(jlo, uint32_t(c[u]) >> 4);
      jhi = max(jhi, uint32_t(c[u]) >> 4);
    }
  }
  jlo = __reduce_min_sync(kFull, jlo);
  jhi = __reduce_max_sync(kFull, jhi);
  // too wide for the bitmap: the sort path (tile columns must fit 24 bits)
  const bool wide = jlo != 0xffffffffu && jhi - jlo >= uint32_t(kBitW) * 32u;
  if (wide && jhi >= (1u << 24)) {
    if (lane == 0) walk_list[atomicAdd(walk_count, 1u)] = I;
    return;
  }
  // lane r < 16: offset of row r's first entry in the panel (rows past the end: E)
  const uint32_t rs = lane < kTile && row < in.rows ? uint32_t(p - E0) : E;
  // panels spanning <= 1024 tile columns (most banded ones) use one bitmap
  // word per lane
  const bool narrow = jlo == 0xffffffffu || jhi - jlo < 1024u;
  if (!wide)
    for (int i = lane; i < (narrow ? 32 : kBitW); i += 32) sm.bits[i] = 0;
  if (has_row)
    for (uint32_t q = rs; q < uint32_t(end - E0); ++q) sm.row[q] = uint8_t(lane);
  __syncwarp();
  unsigned err = 0;
  // entries: column, and packed {fp16 bits, row, kept}
  uint32_t pk[kFastU];
#pragma unroll
  for (int u = 0; u < kFastU; ++u) {
    pk[u] = 0;
    if (32u * u >= E) break;
    const uint32_t q = 32 * u + lane;
    const int32_t up = __shfl_up_sync(kFull, c[u], 1);
    const int32_t last = __shfl_sync(kFull, c[u > 0 ? u - 1 : 0], 31);  // lane 31 of the previous step
    const int32_t cprev = lane > 0 ? up : (u > 0 ? last : -1);
    if (q < E) {
      const int r = sm.row[q];
      const bool later = q > 0 && sm.row[q - 1] == r;  // not the first entry of its row
      bool keep;
      const uint16_t h = raw_to_half<kDtype>(v[u], drop_nonfinite, err, keep);
      if (c[u] >= in.cols || c[u] < 0 || (later && c[u] <= cprev)) err |= kErrInvariant;
      const uint32_t j = (uint32_t(c[u]) >> 4) - jlo;
      // out-of-range columns (flagged) never form tiles: the tile structure
      // stays in range even for invalid input
      keep = keep && !skip && c[u] >= 0 && c[u] < in.cols && (wide || j < uint32_t(kBitW) * 32u);
      if (keep && !wide) atomicOr(&sm.bits[j >> 5], 1u << (j & 31));
      if (!keep && out.etile) out.etile[E0 + q] = kNoTile;
      if (out.h16) out.h16[E0 + q] = keep ? h : uint16_t(0);
      pk[u] = uint32_t(h) | (uint32_t(r) << 16) | (keep ? 1u << 20 : 0u);
    }
  }
  __syncwarp();
  // the sort path: the panel's kept entries as items
  auto sort_path = [&]() {
    uint32_t P2 = 32;
    while (P2 < E) P2 <<= 1;
    uint32_t nk = 0;  // kept items, compacted in CSR order
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int u = 0; u < kFastU; ++u) {
      if (32u * u >= P2) break;
      const uint32_t q = 32 * u + lane;
      const bool kp = q < E && ((pk[u] >> 20) & 1u);
      const unsigned kb = __ballot_sync(kFull, kp);
      if (kp)
        sm.items[nk + __popc(kb & lt)] = (static_cast<unsigned long long>(uint32_t(c[u]) >> 4) << 40) |
                                         (static_cast<unsigned long long>((pk[u] >> 16) & 15u) << 36) |
                                         (static_cast<unsigned long long>(uint32_t(c[u]) & 15u) << 32) |
                                         (static_cast<unsigned long long>(q) << 16) | (pk[u] & 0xffffu);
      nk += __popc(kb);
    }
    __syncwarp();
    const uint32_t nt = sparse_panel(sm, out, roles, E0, E, nk, lane, seen);
    const unsigned e = __reduce_or_sync(kFull, err);
    if (lane == 0) {
      out.ntiles[I] = nt;
      if (e) atomicOr(err_flag, e);
    }
  };
  if (wide && !skip) {
    sort_path();
    return;
  }
  // ranks: tiles before each bitmap word (lane owns word lane, or words
  // 8 lane .. 8 lane + 7)
  uint32_t ntiles = 0;
  if (wide) {
  } else if (narrow) {
    const uint32_t wc = __popc(sm.bits[lane]);
    uint32_t incl = wc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    ntiles = __shfl_sync(kFull, incl, 31);
    sm.pre[lane] = uint16_t(incl - wc);
  } else {
    uint32_t wc[8], lsum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      wc[i] = __popc(sm.bits[8 * lane + i]);
      lsum += wc[i];
    }
    uint32_t incl = lsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    ntiles = __shfl_sync(kFull, incl, 31);
    uint32_t run = incl - lsum;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      sm.pre[8 * lane + i] = uint16_t(run);
      run += wc[i];
    }
  }
  const unsigned e_all = __reduce_or_sync(kFull, err);
  if (skip) {
    if (lane == 0) {
      out.ntiles[I] = 0;
      if (e_all) atomicOr(err_flag, e_all);
    }
    return;
  }
  if (ntiles > uint32_t(kFastT)) {  // too many tiles to stage: the sort path
    __syncwarp();
    sort_path();
    return;
  }
  // a general call reads no chunks / masks / lane metadata of this tile row
  const bool lite = __shfl_sync(kFull, lane == 0 ? general_call(out, ntiles, seen) : false, 0);
  for (uint32_t i = lane; i < ntiles * 8u; i += 32) sm.rm[i >> 3][i & 7] = 0;
  for (uint32_t i = lane; i < ntiles * 2u; i += 32) sm.lm[i >> 1][i & 1] = 0;
  __syncwarp();
  // tile rank of each kept entry; masks
  uint32_t carry = 0xffffffffu;  // (row, tile) key of the last kept entry so far
#pragma unroll
  for (int u = 0; u < kFastU; ++u) {
    if (32u * u >= E) break;
    const bool keep = (pk[u] >> 20) & 1u;
    const int r = (pk[u] >> 16) & 15;
    uint32_t k = 0;
    if (keep) {
      const uint32_t j = (uint32_t(c[u]) >> 4) - jlo;
      k = sm.pre[j >> 5] + __popc(sm.bits[j >> 5] & ((1u << (j & 31)) - 1u));
      const int cc = c[u] & 15;
      atomicOr(&sm.rm[k][r & 7], 1u << (cc + 16 * (r >> 3)));
      if (!lite) {
        int L, h16;
        slot_lane(kRoleA, r, cc, L, h16);
        atomicOr(&sm.lm[k][0], 1u << L);
        slot_lane(kRoleB, r, cc, L, h16);
        atomicOr(&sm.lm[k][1], 1u << L);
      }
      pk[u] |= k << 21;  // k < 64: bits 21..26
    }
    if (out.etile) {  // the first kept entry of each (row, tile) names the tile; later ones are duplicates
      const uint32_t key = keep ? (uint32_t(r) << 16) | k : 0xfffffffeu;
      const unsigned kb = __ballot_sync(kFull, keep);
      const unsigned peers = __match_any_sync(kFull, key) & kb;
      if (keep) {
        const bool dup = (peers & lanemask_lt()) != 0u || key == carry;
        out.etile[E0 + 32 * u + lane] = k | (dup ? kDupEntry : 0u);
      }
      if (kb) carry = __shfl_sync(kFull, key, 31 - __clz(kb));
    }
  }
  __syncwarp();
  // per tile (lane k, k + 32): chunk bases, metadata
  uint32_t cbA[2], cbB[2];
  {
    uint32_t nA[2], nB[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t k = lane + 32 * h;
      nA[h] = k < ntiles ? __popc(sm.lm[k][0]) : 0u;
      nB[h] = k < ntiles ? __popc(sm.lm[k][1]) : 0u;
    }
    uint32_t ia = nA[0], ib = nB[0];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t va = __shfl_up_sync(kFull, ia, o), vb = __shfl_up_sync(kFull, ib, o);
      if (lane >= o) {
        ia += va;
        ib += vb;
      }
    }
    const uint32_t ta = __shfl_sync(kFull, ia, 31), tb = __shfl_sync(kFull, ib, 31);
    uint32_t ja = nA[1], jb = nB[1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t va = __shfl_up_sync(kFull, ja, o), vb = __shfl_up_sync(kFull, jb, o);
      if (lane >= o) {
        ja += va;
        jb += vb;
      }
    }
    const uint32_t base = 1u + uint32_t(E0);
    cbA[0] = base + ia - nA[0];
    cbB[0] = base + ib - nB[0];
    cbA[1] = base + ta + ja - nA[1];
    cbB[1] = base + tb + jb - nB[1];
    const uint32_t totA = ta + __shfl_sync(kFull, ja, 31), totB = tb + __shfl_sync(kFull, jb, 31);
    // zero the panel's chunk ranges (the values are stored into them below)
    for (uint32_t i = lane; i < totA && (roles & 1); i += 32) out.chunk[kRoleA][base + i] = make_uint4(0, 0, 0, 0);
    for (uint32_t i = lane; i < totB && (roles & 2); i += 32) out.chunk[kRoleB][base + i] = make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t k = lane + 32 * h;
    if (k >= ntiles) continue;
    // tile column: the k-th set bit of the bitmap
    int w = 0;
    for (int b = narrow ? 16 : kBitW / 2; b > 0; b >>= 1)
      if (sm.pre[w + b] <= k) w += b;
    uint32_t word = sm.bits[w];
    for (uint32_t n = k - sm.pre[w]; n > 0; --n) word &= word - 1u;
    const uint32_t J = jlo + uint32_t(w) * 32u + uint32_t(__ffs(word) - 1);
    uint32_t colocc = 0, rowocc = 0;
    const uint4* rmv = reinterpret_cast<const uint4*>(sm.rm[k]);
    uint4 m0 = rmv[0], m1 = rmv[1];
    const uint32_t mw[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
    for (int gg = 0; gg < 8; ++gg) {
      colocc |= mw[gg] | (mw[gg] >> 16);
      rowocc |= ((mw[gg] & 0xffffu) != 0u ? 1u << gg : 0u) | ((mw[gg] >> 16) != 0u ? 1u << (gg + 8) : 0u);
    }
    const uint32_t occ = (colocc & 0xffffu) | (rowocc << 16);
    if (!lite) {
      uint4* dst = reinterpret_cast<uint4*>(out.rm2 + size_t(E0 + k) * 8);
      dst[0] = m0;
      dst[1] = m1;
    }
    mark_column(out, J);
    if (lite) {
      out.rec[lite_role(roles)][E0 + k] = make_uint4(0u, 0u, occ, J);
    } else {
      if (roles & 1) out.rec[kRoleA][E0 + k] = make_uint4(sm.lm[k][0], cbA[h], occ, J);
      if (roles & 2) out.rec[kRoleB][E0 + k] = make_uint4(sm.lm[k][1], cbB[h], occ, J);
    }
    sm.cl[k][0] = make_uint2(cbA[h], sm.lm[k][0]);
    sm.cl[k][1] = make_uint2(cbB[h], sm.lm[k][1]);
  }
  __syncwarp();  // chunk zeros before the value stores (same warp: ordered by the barrier)
  // every kept entry stores its fp16 value into its chunk slots
#pragma unroll
  for (int u = 0; u < kFastU; ++u) {
    if (32u * u >= E || lite) break;
    if (!((pk[u] >> 20) & 1u)) continue;
    const uint32_t k = (pk[u] >> 21) & 63u;
    const int r = (pk[u] >> 16) & 15, cc = c[u] & 15;
    const uint16_t hv = uint16_t(pk[u]);
#pragma unroll
    for (int role = 0; role < 2; ++role) {
      if (!(roles & (1 << role))) continue;
      int L, h16;
      slot_lane(role, r, cc, L, h16);
      const uint2 cl = sm.cl[k][role];
      const uint32_t idx = cl.x + __popc(cl.y & ((1u << L) - 1u));
      reinterpret_cast<uint16_t*>(out.chunk[role] + idx)[h16] = hv;
    }
  }
  if (lane == 0) {
    out.ntiles[I] = ntiles;
    if (e_all) atomicOr(err_flag, e_all);
  }
}

// A-order regs of a densely staged tile (row-major fp16 bits): lane (g, t)
// holds reg i = rows g + 8(i&1), cols 2t + 8(i>>1) .. +1.
__device__ __forceinline__ void staged_regs(const uint16_t* tl, int lane, uint32_t (&r)[4]) {
  const int g = lane >> 2, tq = lane & 3;
  const uint32_t* tw = reinterpret_cast<const uint32_t*>(tl);
#pragma unroll
  for (int i = 0; i < 4; ++i) r[i] = tw[((g + 8 * (i & 1)) * 16 + 2 * tq + 8 * (i >> 1)) >> 1];
}

constexpr int kHubThreads = 256;
constexpr uint32_t kHubMax = 8192;      // entries of a hub panel
constexpr uint32_t kHubWords = 2048;    // tile-column bitmap: spans of <= 65536 tile columns
constexpr uint32_t kHubDefer = 0xfffffffeu;  // ntiles[I]: the hub kernel handed the row to the walk

// Which listed tile rows convert_hub_kernel may take (the walk kernel takes
// the rest, and the ones the hub kernel hands back): needed, well-formed row
// pointers, 512 < entries <= kHubMax.  Warp-collective; every warp of both
// kernels computes the same answer.
__device__ __forceinline__ bool hub_takes(const CsrView& in, uint32_t I, const uint8_t* needed, int lane) {
  if (needed && !needed[I]) return false;
  const int64_t r0 = int64_t(I) * kTile, r1 = r0 + kTile < in.rows ? r0 + kTile : in.rows;
  const int nr = int(r1 - r0);
  const int64_t v = lane <= nr ? in.row_ptr[r0 + lane] : 0;
  const int64_t nxt = __shfl_down_sync(kFull, v, 1);
  const bool mono = lane >= nr || nxt >= v;
  const int64_t E = __shfl_sync(kFull, v, nr) - __shfl_sync(kFull, v, 0);
  return __all_sync(kFull, mono) && E > 32 * kFastU && E <= int64_t(kHubMax);
}

// The general panel walk (any column span, any number of tiles): warp per
// listed tile row, lanes r < 16 own CSR rows; each step takes the minimum
// pending tile column (REDUX), every row lane consumes its entries in that
// tile, and the tile is staged densely and cut.
template <int kDtype>
__global__ void __launch_bounds__(256) convert_walk_kernel(CsrView in, Gapped out, int roles,
                                                          const uint32_t* __restrict__ walk_list,
                                                          const uint32_t* __restrict__ walk_count,
                                                          unsigned* __restrict__ err_flag, int drop_nonfinite,
                                                          const uint8_t* __restrict__ needed) {
  __shared__ __align__(16) uint16_t s_tile[8][2][256];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint16_t* st = s_tile[wib][0];
  uint16_t* stT = s_tile[wib][1];
  const uint32_t n_list = *walk_count;
  for (uint32_t li = blockIdx.x * 8 + wib; li < n_list; li += gridDim.x * 8) {
    const uint32_t I = walk_list[li];
    if (hub_takes(in, I, needed, lane) && out.ntiles[I] != kHubDefer) continue;  // convert_hub_kernel's
    const int64_t row = int64_t(I) * kTile + lane;
    const bool has_row = lane < kTile && row < in.rows;
    int64_t p = has_row ? in.row_ptr[row] : 0;
    const int64_t end = has_row ? in.row_ptr[row + 1] : 0;
    const int64_t E0 = in.row_ptr[int64_t(I) * kTile];
    unsigned err = 0;
    if (has_row && end < p) err |= kErrInvariant;
    if (needed && !needed[I]) {  // validation only (tile_format.cpp:34-51): no tiles
      int32_t prev_col = -1;
      for (int64_t q = p; q < end; ++q) {
        const int32_t c = __ldg(in.col + q);
        if (c <= prev_col || c >= in.cols || c < 0) err |= kErrInvariant;
        prev_col = c;
        bool keep;
        load_half<kDtype>(in.val, q, drop_nonfinite, err, keep);
        if (out.etile) out.etile[q] = kNoTile;
        if (out.h16) out.h16[q] = 0;
      }
      const unsigned e = __reduce_or_sync(kFull, err);
      if (lane == 0) {
        out.ntiles[I] = 0;
        if (e) atomicOr(err_flag, e);
      }
      continue;
    }
    uint32_t ntiles = 0;
    uint32_t cbase[2] = {1u + uint32_t(E0), 1u + uint32_t(E0)};
    int32_t prev_col = -1;
    // a general call (flagged by some tile row of A with > kLightMax tiles) reads
    // no chunks, masks or lane metadata: only tile columns, occupancy, etile, h16
    const bool lite = __shfl_sync(kFull, lane == 0 ? general_seen(out) : false, 0);
    int32_t c_cur = p < end ? __ldg(in.col + p) : 0;  // one entry ahead: the walk is not a chain of loads
    while (true) {
      const uint32_t my_tc = (p < end) ? uint32_t(c_cur) >> 4 : 0xffffffffu;
      const uint32_t J = __reduce_min_sync(kFull, my_tc);
      if (J == 0xffffffffu) break;
      reinterpret_cast<uint4*>(st)[lane] = make_uint4(0, 0, 0, 0);
      reinterpret_cast<uint4*>(stT)[lane] = make_uint4(0, 0, 0, 0);
      __syncwarp();
      uint32_t rm = 0;
      bool first = true;  // first kept entry of this tile in this row
      while (p < end) {
        const int32_t c = c_cur;
        if ((uint32_t(c) >> 4) != J) break;
        const int32_t c_next = p + 1 < end ? __ldg(in.col + p + 1) : 0;
        if (c <= prev_col || c >= in.cols || c < 0) err |= kErrInvariant;
        prev_col = c;
        bool keep;
        const unsigned short h = load_half<kDtype>(in.val, p, drop_nonfinite, err, keep);
        keep = keep && c >= 0 && c < in.cols;  // out-of-range columns (flagged) never form tiles
        if (out.h16) out.h16[p] = keep ? h : (unsigned short)0;
        if (keep) {
          rm |= 1u << (c & 15);
          st[lane * 16 + (c & 15)] = h;
          stT[(c & 15) * 16 + lane] = h;
        }
        if (out.etile) {
          out.etile[p] = keep ? (ntiles | (first ? 0u : kDupEntry)) : kNoTile;
          first &= !keep;
        }
        ++p;
        c_cur = c_next;
      }
      // Termination holds for any input: the lane holding the minimum tile
      // column always consumes at least one entry.  Invalid input only sets
      // the flag; the host discards the results.
      const unsigned any = __ballot_sync(kFull, rm != 0);
      if (any == 0) continue;  // every value of this tile dropped
      __syncwarp();
      const uint32_t t = uint32_t(E0) + ntiles;
      const uint32_t occ = (__reduce_or_sync(kFull, rm) & 0xffffu) | ((any & 0xffffu) << 16);
      // the 256-bit mask as interleaved row masks: word g = row g | row g+8 << 16
      const uint32_t rm_hi = __shfl_sync(kFull, rm, (lane & 7) + 8);
      if (lane < 8 && !lite) out.rm2[size_t(t) * 8 + lane] = rm | (rm_hi << 16);
      if (lane == 0) mark_column(out, J);
#pragma unroll
      for (int role = 0; role < 2; ++role) {
        if (!(roles & (1 << role))) continue;
        if (lite) {
          if (lane == 0 && role == lite_role(roles)) out.rec[role][t] = make_uint4(0u, 0u, occ, J);
          continue;
        }
        uint32_t rg[4];
        staged_regs(role == kRoleA ? st : stT, lane, rg);
        if (role == kRoleB) {  // the transposed tile in A order, stored {reg0, reg2, reg1, reg3}
          const uint32_t t1 = rg[1];
          rg[1] = rg[2];
          rg[2] = t1;
        }
        const bool present = (rg[0] | rg[1] | rg[2] | rg[3]) != 0u;
        const unsigned lm = __ballot_sync(kFull, present);
        if (present) out.chunk[role][cbase[role] + __popc(lm & lanemask_lt())] = make_uint4(rg[0], rg[1], rg[2], rg[3]);
        if (lane == 0) out.rec[role][t] = make_uint4(lm, cbase[role], occ, J);
        cbase[role] += __popc(lm);
      }
      __syncwarp();
      ++ntiles;
    }
    const unsigned e = __reduce_or_sync(kFull, err);
    if (lane == 0) {
      out.ntiles[I] = ntiles;
      if (e) atomicOr(err_flag, e);
    }
  }
}

// Hub panels of a general call (512 < entries <= kHubMax: R-MAT's dense
// tile rows), CTA per listed tile row.  A general call reads no operand
// chunks, masks or lane metadata, so no sort is needed: the kept entries mark
// their tile columns in a shared-memory bitmap, the bitmap's prefix popcounts
// rank the tiles (tile columns ascending, like from_element_coo's sort), and
// shared-memory atomics gather each tile's occupancy words.  Tile rows of a
// call that is not (yet) known to be general, or spanning more than 65536 tile
// columns, are handed back to convert_walk_kernel (ntiles = kHubDefer).
struct HubSmem {
  uint32_t bits[kHubWords];
  uint16_t wpre[kHubWords];  // tiles before each bitmap word (<= kHubMax)
  uint32_t occ[kHubMax];     // per tile: column occupancy | row occupancy << 16
  int64_t rp[kTile + 1];
  uint32_t wsum[kHubThreads / 32];
  uint32_t jlo, jhi, flag;
};

// exclusive block scan (kHubThreads threads)
__device__ __forceinline__ uint32_t hub_scan(HubSmem& sm, uint32_t x, uint32_t& tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sm.wsum[w] = inc;
  __syncthreads();
  uint32_t pre = 0;
  tot = 0;
#pragma unroll
  for (int i = 0; i < kHubThreads / 32; ++i) {
    const uint32_t v = sm.wsum[i];
    if (i < w) pre += v;
    tot += v;
  }
  __syncthreads();
  return pre + inc - x;
}

template <int kDtype>
__global__ void __launch_bounds__(kHubThreads) convert_hub_kernel(CsrView in, Gapped out, int roles,
                                                                 const uint32_t* __restrict__ walk_list,
                                                                 const uint32_t* __restrict__ walk_count,
                                                                 unsigned* __restrict__ err_flag, int drop_nonfinite,
                                                                 const uint8_t* __restrict__ needed) {
  __shared__ HubSmem sm;
  const int tid = threadIdx.x;
  const uint32_t n_list = *walk_count;
  for (uint32_t li = blockIdx.x; li < n_list; li += gridDim.x) {
    const uint32_t I = walk_list[li];
    if (!hub_takes(in, I, needed, tid & 31)) continue;  // the walk kernel's
    const int64_t r0 = int64_t(I) * kTile, r1 = r0 + kTile < in.rows ? r0 + kTile : in.rows;
    const int nr = int(r1 - r0);
    if (tid <= kTile) sm.rp[tid] = in.row_ptr[r0 + tid < r1 ? r0 + tid : r1];
    if (tid == 0) {
      sm.jlo = 0xffffffffu;
      sm.jhi = 0;
      sm.flag = general_seen(out) ? 1u : 0u;
    }
    __syncthreads();
    // the panel's tile-column span from each row's first and last column
    if (tid < nr && sm.rp[tid + 1] > sm.rp[tid]) {
      const int32_t c0 = __ldg(in.col + sm.rp[tid]), c1 = __ldg(in.col + sm.rp[tid + 1] - 1);
      if (c0 >= 0 && c0 < in.cols) atomicMin(&sm.jlo, uint32_t(c0) >> 4);
      if (c1 >= 0 && c1 < in.cols) atomicMax(&sm.jhi, uint32_t(c1) >> 4);
    }
    for (uint32_t i = tid; i < kHubWords; i += kHubThreads) sm.bits[i] = 0;
    __syncthreads();
    const uint32_t jlo = sm.jlo;
    if (!sm.flag || (jlo != 0xffffffffu && sm.jhi - jlo >= kHubWords * 32u)) {
      if (tid == 0) out.ntiles[I] = kHubDefer;  // not known general yet, or too wide: the walk
      __syncthreads();
      continue;
    }
    const int64_t E0 = sm.rp[0];
    const uint32_t E = uint32_t(sm.rp[nr] - E0);
    unsigned err = 0;
    // (1) validation, rounding, kept entries mark their tile columns
    for (uint32_t q = tid; q < E; q += kHubThreads) {
      const int64_t e = E0 + q;
      int r = 0;
#pragma unroll
      for (int b = 8; b > 0; b >>= 1)
        if (r + b <= nr - 1 && sm.rp[r + b] <= e) r += b;
      const int32_t c = __ldg(in.col + e);
      const bool later = e > sm.rp[r];
      const int32_t cp = later ? __ldg(in.col + e - 1) : -1;
      if (c >= in.cols || c < 0 || (later && c <= cp)) err |= kErrInvariant;
      bool keep;
      const unsigned short h = load_half<kDtype>(in.val, e, drop_nonfinite, err, keep);
      keep = keep && c >= 0 && c < in.cols && (uint32_t(c) >> 4) >= jlo && (uint32_t(c) >> 4) - jlo < kHubWords * 32u;
      if (out.h16) out.h16[e] = keep ? h : (unsigned short)0;
      if (keep) {
        const uint32_t j = (uint32_t(c) >> 4) - jlo;
        atomicOr(&sm.bits[j >> 5], 1u << (j & 31));
      } else if (out.etile) {
        out.etile[e] = kNoTile;
      }
    }
    __syncthreads();
    // (2) tile ranks: tiles before each bitmap word
    uint32_t wc[kHubWords / kHubThreads], lsum = 0;
#pragma unroll
    for (int i = 0; i < int(kHubWords / kHubThreads); ++i) {
      wc[i] = __popc(sm.bits[tid * (kHubWords / kHubThreads) + i]);
      lsum += wc[i];
    }
    uint32_t ntiles;
    uint32_t run = hub_scan(sm, lsum, ntiles);
#pragma unroll
    for (int i = 0; i < int(kHubWords / kHubThreads); ++i) {
      sm.wpre[tid * (kHubWords / kHubThreads) + i] = uint16_t(run);
      run += wc[i];
    }
    for (uint32_t t = tid; t < ntiles; t += kHubThreads) sm.occ[t] = 0;
    if (tid == 0 && out.may_set && ntiles > kLightMax) atomicOr(out.general, 1u);
    __syncthreads();
    // (3) occupancy words; etile = tile rank | duplicate flag (an earlier kept
    // entry of the same row in the same tile)
    for (uint32_t q = tid; q < E; q += kHubThreads) {
      const int64_t e = E0 + q;
      if (out.h16 && out.h16[e] == 0) continue;  // dropped
      int r = 0;
#pragma unroll
      for (int b = 8; b > 0; b >>= 1)
        if (r + b <= nr - 1 && sm.rp[r + b] <= e) r += b;
      const uint32_t c = uint32_t(__ldg(in.col + e)), j = (c >> 4) - jlo;
      const uint32_t t = sm.wpre[j >> 5] + __popc(sm.bits[j >> 5] & ((1u << (j & 31)) - 1u));
      atomicOr(&sm.occ[t], (1u << (c & 15u)) | (1u << (16 + r)));
      if (out.etile) {
        bool dup = false;  // walk back over the row's entries in the same tile
        for (int64_t p = e - 1; p >= sm.rp[r]; --p) {
          if ((uint32_t(__ldg(in.col + p)) >> 4) != (c >> 4)) break;
          if (out.h16[p] != 0) {
            dup = true;
            break;
          }
        }
        out.etile[e] = t | (dup ? kDupEntry : 0u);
      }
    }
    __syncthreads();
    // (4) the tile records: tile t = the t-th set bit of the bitmap
    for (uint32_t w = tid; w < kHubWords; w += kHubThreads) {
      uint32_t word = sm.bits[w], t = sm.wpre[w];
      for (; word; word &= word - 1u, ++t) {
        const uint32_t J = jlo + w * 32u + uint32_t(__ffs(word) - 1);
        const uint32_t o = sm.occ[t];
        mark_column(out, J);
        out.rec[lite_role(roles)][E0 + t] = make_uint4(0u, 0u, o, J);
      }
    }
    const unsigned e_or = __reduce_or_sync(kFull, err);
    if (e_or && (tid & 31) == 0) atomicOr(err_flag, e_or);
    if (tid == 0) out.ntiles[I] = ntiles;
    __syncthreads();  // shared memory is rewritten by the next tile row
  }
}

// Gapped tiles -> the dense CSR-of-tiles arrays (warp per tile row).
__global__ void __launch_bounds__(256) tiles_compact_kernel(CsrView in, uint32_t tile_rows, Gapped g, TileMat T,
                                                           int roles, unsigned* __restrict__ max_row_tiles) {
  const int lane = threadIdx.x & 31;
  const uint32_t I = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (max_row_tiles) {  // the largest tile row (the light-path test), one atomic per block
    __shared__ unsigned s_max;
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    if (lane == 0 && I < tile_rows) atomicMax(&s_max, g.ntiles[I]);
    __syncthreads();
    if (threadIdx.x == 0 && s_max) atomicMax(max_row_tiles, s_max);
  }
  if (I >= tile_rows) return;
  const uint32_t src = uint32_t(in.row_ptr[int64_t(I) * kTile]), dst = T.trp[I], n = g.ntiles[I];
  const int r0 = lite_role(roles);
  const bool lite = g.general && *g.general;  // final here: the conversion kernels are done
  if (lite) {  // tile column + occupancy only; four records per lane in flight
    for (uint32_t i0 = lane; i0 < n; i0 += 128) {
      uint4 r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + 32u * u < n) r[u] = g.rec[r0][src + i0 + 32u * u];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + 32u * u < n) T.tco[dst + i0 + 32u * u] = make_uint2(r[u].w, r[u].z);
    }
    return;
  }
  for (uint32_t i = lane; i < n; i += 32) {
    const uint4 rec0 = g.rec[r0][src + i];
    T.tco[dst + i] = make_uint2(rec0.w, rec0.z);
#pragma unroll
    for (int role = 0; role < 2; ++role) {
      if (!(roles & (1 << role))) continue;
      const uint4 rc = role == r0 ? rec0 : g.rec[role][src + i];
      T.meta[role][dst + i] = make_uint2(rc.x, rc.y);
      T.rec[role][dst + i] = rc;
    }
  }
  const uint4* s4 = reinterpret_cast<const uint4*>(g.rm2 + size_t(src) * 8);
  uint4* d4 = reinterpret_cast<uint4*>(T.rm2 + size_t(dst) * 8);
  for (uint32_t i = lane; i < 2 * n; i += 32) d4[i] = s4[i];
}

// B tile rows that some A tile refers to (A's tile columns).
__global__ void mark_needed_kernel(const TileMat A, uint8_t* __restrict__ needed) {
  const uint32_t nt = A.trp[A.tile_rows];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    const uint32_t J = __ldg(&A.tco[t].x);
    if (!needed[J]) needed[J] = 1;  // most A tiles share their column's flag: skip the contended store
  }
}

__global__ void row_stats_kernel(const uint32_t* __restrict__ trp, uint32_t tile_rows,
                                 unsigned* __restrict__ max_row_tiles) {
  unsigned m = 0;
  for (uint32_t I = blockIdx.x * blockDim.x + threadIdx.x; I < tile_rows;
       I += gridDim.x * blockDim.x)
    m = max(m, trp[I + 1] - trp[I]);
  m = __reduce_max_sync(kFull, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(max_row_tiles, m);
}

// Column counts of A (histogram) for C-bar.
__global__ void col_hist_kernel(const int32_t* __restrict__ col, int64_t nnz, int64_t ncols,
                                unsigned* __restrict__ hist) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nnz;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t c = __ldg(col + i);
    if (c >= 0 && c < ncols) atomicAdd(hist + c, 1u);
  }
}

__global__ void cbar_dot_kernel(const unsigned* __restrict__ hist, const int64_t* __restrict__ rpB,
                                int64_t n, unsigned long long* __restrict__ out) {
  unsigned long long acc = 0;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n;
       k += int64_t(gridDim.x) * blockDim.x)
    acc += (unsigned long long)hist[k] * (unsigned long long)(rpB[k + 1] - rpB[k]);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(kFull, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// row_ptr[0] == 0, row_ptr[rows] == nnz, non-decreasing: checked before any
// kernel indexes the entries through it (every later reader is gated on
// kErrRowPtr).  Thread per row pointer.
__global__ void validate_rowptr_kernel(const int64_t* __restrict__ rp, int64_t rows, int64_t nnz,
                                       unsigned* __restrict__ err_flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= rows; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t v = rp[i];
    if (i == 0) bad |= v != 0;
    if (i == rows) bad |= v != nnz;
    else bad |= rp[i + 1] < v;
  }
  if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(err_flag, unsigned(kErrRowPtr));
}

}  // namespace

void launch_validate_rowptr(const CsrView& in, unsigned* err_flag, cudaStream_t st) {
  const int64_t n = in.rows + 1;
  const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 2368));
  validate_rowptr_kernel<<<blocks, 256, 0, st>>>(in.row_ptr, in.rows, in.nnz, err_flag);
}

void launch_convert(const CsrView& in, TileMat& out, int roles, const ConvertScratch& cs, unsigned* err_flag,
                    int drop_nonfinite, const uint8_t* needed, cudaStream_t st) {
  if (out.tile_rows == 0) return;
  Gapped g;
  g.rm2 = cs.rm2;
  g.rec[0] = cs.rec[0];
  g.rec[1] = cs.rec[1];
  g.chunk[0] = out.chunk[0];
  g.chunk[1] = out.chunk[1];
  g.etile = out.etile;
  g.h16 = out.h16;
  g.ntiles = cs.ntiles;
  g.mark = cs.mark;
  g.general = cs.general;
  g.may_set = (roles & 1) != 0;
  auto kf = in.dtype == 0 ? convert_fast_kernel<0> : in.dtype == 2 ? convert_fast_kernel<2> : convert_fast_kernel<1>;
  kf<<<(out.tile_rows + 7) / 8, 256, 0, st>>>(in, out.tile_rows, g, roles, cs.walk_list, cs.walk_count, err_flag,
                                    drop_nonfinite, needed);
  auto kh = in.dtype == 0 ? convert_hub_kernel<0> : in.dtype == 2 ? convert_hub_kernel<2> : convert_hub_kernel<1>;
  kh<<<std::min<unsigned>((out.tile_rows + 7) / 8, 148u * 4u), kHubThreads, 0, st>>>(in, g, roles, cs.walk_list,
                                                                                   cs.walk_count, err_flag,
                                                                                   drop_nonfinite, needed);
  auto kw = in.dtype == 0 ? convert_walk_kernel<0> : in.dtype == 2 ? convert_walk_kernel<2> : convert_walk_kernel<1>;
  const unsigned wblocks = std::min<unsigned>((out.tile_rows + 7) / 8, 148u * 8u);
  kw<<<wblocks, 256, 0, st>>>(in, g, roles, cs.walk_list, cs.walk_count, err_flag, drop_nonfinite, needed);
}

void launch_tiles_compact(const CsrView& in, const ConvertScratch& cs, TileMat& out, int roles, cudaStream_t st,
                          unsigned* max_row_tiles) {
  if (out.tile_rows == 0) return;
  Gapped g;
  g.rm2 = cs.rm2;
  g.rec[0] = cs.rec[0];
  g.rec[1] = cs.rec[1];
  g.ntiles = cs.ntiles;
  g.general = cs.general;
  tiles_compact_kernel<<<(out.tile_rows + 7) / 8, 256, 0, st>>>(in, out.tile_rows, g, out, roles, max_row_tiles);
}

void launch_mark_needed(const TileMat& A, uint8_t* needed, cudaStream_t st) {
  if (A.cap == 0) return;
  unsigned blocks = unsigned((A.cap + 255) / 256);
  if (blocks > 2368) blocks = 2368;
  mark_needed_kernel<<<blocks, 256, 0, st>>>(A, needed);
}

void launch_row_stats(const TileMat& A, unsigned* max_row_tiles, cudaStream_t st) {
  if (A.tile_rows == 0) return;
  unsigned blocks = (A.tile_rows + 255) / 256;
  if (blocks > 592) blocks = 592;
  row_stats_kernel<<<blocks, 256, 0, st>>>(A.trp, A.tile_rows, max_row_tiles);
}

void launch_cbar(const int32_t* colA, int64_t nnzA, int64_t inner, const int64_t* rpB,
                 unsigned* hist, unsigned long long* out, cudaStream_t st) {
  if (nnzA > 0) col_hist_kernel<<<1184, 256, 0, st>>>(colA, nnzA, inner, hist);
  if (inner > 0) cbar_dot_kernel<<<592, 256, 0, st>>>(hist, rpB, inner, out);
}

}  // namespace tsg
