// tsg_kernels.cuh -- launchers of the four subsystems (host side view).
#pragma once
#include <cuda_runtime.h>

#include "tsg_common.cuh"

namespace tsg {

// Build-time-fixed kernel variants selectable for tuning runs through an
// environment variable (read once); the default is the tuned choice.
int tuning_variant(const char* name, int dflt);

struct CsrView {  // device CSR input
  int64_t rows = 0, cols = 0, nnz = 0;
  const int64_t* row_ptr = nullptr;
  const int32_t* col = nullptr;
  const void* val = nullptr;
  int dtype = 1;  // 0 f16 bits, 1 f32, 2 f64
};

// (1) conversion
// `needed` (nullable): per tile row, whether the other operand refers to it;
// unneeded tile rows are validated but get no tiles
// CSR -> tiles: convert_fast_kernel (block per panel) for panels spanning
// <= 8192 tile columns with <= 1024 entries and <= 64 tiles, the panel walk
// for the rest (listed by the fast kernel), both writing tiles at gapped
// slots (tile row I at row_ptr[16 I]); then a scan of cs.ntiles -> out.trp
// and launch_tiles_compact -> out's dense arrays.  Chunks stay where they
// were written (tile row I's from 1 + row_ptr[16 I]).
struct ConvertScratch {
  uint32_t* rm2 = nullptr;             // gapped, cap * 8
  uint4* rec[2] = {nullptr, nullptr};  // gapped, cap each (roles in use)
  uint32_t* ntiles = nullptr;          // tile_rows + 1
  uint32_t* walk_list = nullptr;       // tile_rows
  uint32_t* walk_count = nullptr;      // 1, zeroed
  uint8_t* mark = nullptr;             // optional, zeroed: set for every tile column
  unsigned* general = nullptr;         // optional, zeroed: set when a tile row of A has > 128 tiles
                                       // (general path); later tile rows then skip chunks / masks
};
// sets kErrRowPtr in err_flag unless row_ptr[0] == 0, row_ptr[rows] == nnz and non-decreasing
void launch_validate_rowptr(const CsrView& in, unsigned* err_flag, cudaStream_t st);
void launch_convert(const CsrView& in, TileMat& out, int roles, const ConvertScratch& cs, unsigned* err_flag,
                    int drop_nonfinite, const uint8_t* needed, cudaStream_t st);
// max_row_tiles (nullable): atomicMax of the tiles per tile row
void launch_tiles_compact(const CsrView& in, const ConvertScratch& cs, TileMat& out, int roles, cudaStream_t st,
                          unsigned* max_row_tiles = nullptr);
void launch_mark_needed(const TileMat& A, uint8_t* needed, cudaStream_t st);
void launch_row_stats(const TileMat& A, unsigned* max_row_tiles, cudaStream_t st);
void launch_cbar(const int32_t* colA, int64_t nnzA, int64_t inner, const int64_t* rpB,
                 unsigned* hist, unsigned long long* out, cudaStream_t st);

// light rows (<= 32 A tiles per tile row): the fused panel pass (tsg_panel.cu)
// nl: merge lists per lane (1, 2, 4): tile rows of up to 32 nl A tiles
void launch_panel_count(const TileMat& A, const TileMat& B, int64_t rows, uint32_t* row_np,
                        uint32_t* row_ns, uint32_t* row_raw, uint32_t* row_bound, int nl, cudaStream_t st);
// staging slot = {value bits, column}, row r's region at row_stage[r]; both
// passes work on the tile rows [I0, I1)
// Emit mode (chained products): output tiles become A-operand tiles of the
// next stage instead of CSR (tsg_panel.cu emit_tile); slots per tile row
// from tile_base, realised tiles per tile row in rtiles.
struct TileEmit {
  uint2* tco = nullptr;
  uint32_t* rm2 = nullptr;
  uint2* meta = nullptr;
  uint4* rec = nullptr;
  uint4* chunk = nullptr;  // chunk 0 = zeros; tile row I's chunks from 1 + 32 * tile_base[I]
  const uint32_t* tile_base = nullptr;
  uint32_t* rtiles = nullptr;
  unsigned* err_flag = nullptr;
};
// The pass does nothing when the staging total row_stage[rows] exceeds
// stage_cap slots (the host checks and reruns with a bigger arena).
// `need`: device u64 total of the staging bound (the pass returns at once when
// it exceeds stage_cap); `stats`: when non-null, {filtered pairs, segments,
// raw pairs} are accumulated there (the element-bound flow has no count pass)
cudaError_t launch_panel_numeric(const TileMat& A, const TileMat& B, int64_t rows, const uint32_t* row_stage,
                                 uint64_t stage_cap, uint2* stage, int64_t* rowcnt, unsigned long long* counted,
                                 const unsigned long long* need, unsigned long long* stats, int mode, uint32_t I0,
                                 uint32_t I1, cudaStream_t st, const TileEmit* emit = nullptr,
                                 const unsigned* gate = nullptr, unsigned* work = nullptr, int nl = 1);
// The same light-row pass on tcgen05 (tsg_tc05.cu; TENSOR mode, tile rows of
// <= 32 A tiles): persistent CTAs over panels of 8 tile rows, M = 128 MMAs
// with TMEM accumulators.  Sets *fallback when a panel gathers more B tiles
// than its shared memory holds (the host then runs launch_panel_numeric).
cudaError_t launch_tc05_panel(const TileMat& A, const TileMat& B, int64_t rows, const uint32_t* row_stage,
                              uint64_t stage_cap, uint2* stage, int64_t* rowcnt, unsigned long long* counted,
                              const unsigned long long* need, unsigned long long* stats, const unsigned* gate,
                              unsigned* work, unsigned* fallback, int device, cudaStream_t st);
// row_bound[r] = min(B.cols, sum over A's entries (r, k) of nnz(B row k));
// *total += sum of row_bound
// (gate: the call's error flags; malformed row pointers -> all bounds 0)
void launch_elem_bound(const CsrView& A, const int64_t* rpB, int64_t bcols, uint32_t* row_bound,
                       unsigned long long* total, const unsigned* gate, cudaStream_t st);
void launch_emit_compact(uint32_t tile_rows, const TileEmit& em, const uint32_t* trp, TileMat& T, cudaStream_t st);
// bound[I] = min(B.tile_cols, raw pairs of A's tile row I): output tiles of the row at most
void launch_row_tile_bound(const TileMat& A, const TileMat& B, uint32_t* bound, cudaStream_t st);
void launch_panel_copy(int64_t rows, const uint32_t* row_stage, const int64_t* row_ptr, const uint2* stage,
                       int32_t* col, float* val, unsigned* err_flag, uint32_t I0, uint32_t I1, cudaStream_t st);
// (2)+(3) general rows: per (tile row, column range) chunk, the tile pairs
// expanded into element products, sorted by output tile key in shared
// memory, summed in k order, written as row-major pieces (tsg_esc.cu)
#ifndef TSG_ESC_NT
#define TSG_ESC_NT 512  // threads per esc_kernel CTA (512: 22.8 ms vs 256: 23.4 ms on R-MAT; build-time switch)
#endif
constexpr int kEscThreads = TSG_ESC_NT;
constexpr uint32_t kEscTarget = 3584;  // products per unit of a heavy tile row (sorted leaves hold 4096; R-MAT: 22.4 ms vs 22.8 at 3072, a cliff near 4000)
constexpr uint32_t kNoPiece = 0xffffffffu;
struct EscPiece {             // one sorted output piece: rows of tile row I, row-major
  uint32_t I, next;           // tile row; next piece of the same record (kNoPiece: last)
  unsigned long long off;     // its first staged {col, value} slot
  uint32_t cnt[16];           // realised entries per row
  uint32_t roff[16];          // (assembly) entries of the row in earlier pieces
};
struct EscArgs {
  int64_t rowsA = 0;
  uint32_t tile_rows = 0;
  uint32_t target = kEscTarget;       // products per unit of a heavy tile row
  const int64_t* rpA = nullptr;
  const int32_t* colA = nullptr;
  const uint16_t* hA = nullptr;  // rounded A values (binary16 bits, 0 = dropped)
  int64_t colsB = 0;
  const int64_t* rpB = nullptr;
  const int32_t* colB = nullptr;
  const uint16_t* hB = nullptr;
  const uint4* brec = nullptr;        // per B row {first entry, end, first col, last col}
  const uint4* units = nullptr;       // {tile row, c0, c1, heavy piece index | group flag + tile rows}
  const uint32_t* nunits = nullptr;   // device: number of units
  const uint32_t* rec_base = nullptr; // first output record of each tile row
  const uint32_t* nrec = nullptr;     // device: number of records (the pool follows them)
  EscPiece* pieces = nullptr;
  uint32_t* piece_top = nullptr;      // pool pieces used
  uint32_t pool_cap = 0;
  uint2* stage = nullptr;             // {col, value bits}
  unsigned long long* stage_top = nullptr;
  unsigned* work = nullptr;
  uint32_t unit0 = 0, unit_end = 0xffffffffu;  // the launch's unit range (pipelined host output: a chunk)
  unsigned* err_flag = nullptr;
  unsigned long long* counted = nullptr;
  unsigned long long* segs = nullptr;
};
size_t esc_smem_bytes();
void launch_esc_brec(const EscArgs& g, int64_t rowsB, uint4* brec, cudaStream_t st);
void launch_esc_hist(const EscArgs& g, int64_t nnzA, int64_t rowsB, uint32_t* colcnt, unsigned long long* hist,
                     cudaStream_t st);
void launch_esc_plan_prod(const EscArgs& g, unsigned long long* prod, unsigned long long* total, cudaStream_t st);
void launch_esc_plan_group(const EscArgs& g, const unsigned long long* pre, uint32_t* nrec, uint32_t* nwk,
                           cudaStream_t st);
void launch_esc_plan_fill(const EscArgs& g, const unsigned long long* pre, const uint32_t* nwk, const uint32_t* wbase,
                          const unsigned long long* G, uint4* units, cudaStream_t st);
void launch_esc(const EscArgs& g, int device, cudaStream_t st);
// tile rows [I0, I1) (I1 = 0: all)
void launch_esc_rowcount(const EscArgs& g, const uint32_t* base, int64_t* rowcnt, cudaStream_t st, uint32_t I0 = 0,
                         uint32_t I1 = 0);
void launch_esc_copy(const EscArgs& g, const int64_t* row_ptr, int32_t* col, float* val, cudaStream_t st);
// the pieces of output records [rec0, rec1) and their chains (a chunk of tile rows)
void launch_esc_copy_records(const EscArgs& g, uint32_t rec0, uint32_t rec1, const int64_t* row_ptr, int32_t* col,
                             float* val, cudaStream_t st);
// njt: B rows + 1; nx: 16 per B tile row; single: one per B tile row (scratch)
// B's per-row / per-tile-row summaries (njt, rinfo) from a converted B
void launch_esc_bsummary(const TileMat& B, uint32_t* njt, uint32_t* rinfo, cudaStream_t st);
void launch_esc_pairstats(const TileMat& A, const TileMat& B, uint64_t tA, const uint32_t* njt, const uint32_t* rinfo,
                          unsigned long long* out, cudaStream_t st);
void launch_bsum_tiles(const TileMat& B, uint64_t tiles, uint32_t* tile_count, uint16_t* ro, cudaStream_t st);
// 8x8 tiles of the reference's TiledMatrix (tsg_tiles8.cu): device arrays
struct Tiles8View {
  const uint32_t* tile_col = nullptr;
  const unsigned long long* bitmap = nullptr;
  const unsigned long long* elem_index = nullptr;
  const float* val = nullptr;
};
struct Tiles8Out {
  uint32_t* tile_row = nullptr;
  uint32_t* tile_col = nullptr;
  unsigned long long* bitmap = nullptr;
  unsigned long long* elem_index = nullptr;
  float* val = nullptr;
};
// trp[T] = first tile of tile row T (tiles sorted by row); kErrInvariant if not
void launch_tiles8_trp(const uint32_t* tile_row, int64_t ntiles, int64_t tile_rows, uint32_t* trp, unsigned* err,
                       cudaStream_t st);
// count: rowcnt[r] = elements of row r; else: the CSR at row pointers rp
void launch_tiles8_to_csr(const Tiles8View& t, const uint32_t* trp, int64_t rows, int64_t* rowcnt, const int64_t* rp,
                          int32_t* col, float* val, unsigned* err, bool count, cudaStream_t st);
// per 8-row group: tiles (gt) and elements (ge); then the tiles at the scanned offsets
void launch_csr_tiles8_count(const CsrView& C, const float* val, uint32_t* gt, uint32_t* ge, unsigned* err,
                             cudaStream_t st);
void launch_csr_tiles8_write(const CsrView& C, const float* val, const unsigned long long* toff,
                             const unsigned long long* eoff, const Tiles8Out& o, cudaStream_t st);

// A given as A-role tiles (a chained stage) -> CSR with binary16 values
void launch_tiles_rowcount(const TileMat& A, int64_t* rowcnt, cudaStream_t st);
void launch_tiles_to_csr(const TileMat& A, const int64_t* rp, int32_t* col, uint16_t* h16, cudaStream_t st);

}  // namespace tsg
