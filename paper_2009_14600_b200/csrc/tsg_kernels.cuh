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

// Sorted tile-pair task list (pipeline.hpp:22-34 at T=16): pairs sorted by
// (output tile row, output tile col, inner k), one segment per output tile.
// Each pair is stored as its two operands' metas (pmeta), so the numeric
// kernels reach the lane chunks with one indirection.
struct TaskList {
  uint64_t npairs = 0, nseg = 0;
  uint4* pmeta = nullptr;           // [P+1] {A lane mask, A chunk base, B lane mask, B chunk base}; [P] = 0
  uint2* pocc = nullptr;            // [P+1] {A occupancy, B occupancy} (tco.y of the two tiles)
  uint32_t* seg_row_ptr = nullptr;  // [tile_rows+1] first segment of each tile row
  uint32_t* seg_off = nullptr;      // [S+1] first pair of each segment
  uint32_t* seg_col = nullptr;      // [S] output tile column J
  uint32_t* stage_off = nullptr;    // [S+1] staged-entry region of each segment (upper bound)
};

// Numeric output in tile order (MulResult, kernels.hpp:24-30): each
// segment's realised (nonzero) bitmap as 16 row masks, and its values packed
// row-major (bit order, like TiledMatrix.elements) at stage_off[s].  The
// assembly pass turns it into CSR (compact + to_element_coo,
// kernels.cpp:205-220, tile_format.cpp:131-154).
struct Staged {
  float* val = nullptr;                   // [stage cap]
  uint16_t* rmask = nullptr;              // [S*16] realised row masks (bit c of row r)
  unsigned long long* counted = nullptr;  // structural (counted) nonzeros, CountResult.total_elements
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
};
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
void launch_panel_count(const TileMat& A, const TileMat& B, int64_t rows, uint32_t* row_np,
                        uint32_t* row_ns, uint32_t* row_raw, uint32_t* row_bound, cudaStream_t st);
// staging slot = {value bits, column}, row r's region at row_stage[r]; both
// passes work on the tile rows [I0, I1)
// Emit mode (chained products): output tiles become A-operand tiles of the
// next stage instead of CSR (tsg_panel.cu emit_tile); slots per tile row
// from tile_base, realised tiles per tile row in rtiles.
struct TileEmit {
  uint2* tco = nullptr;
  uint32_t* rm2 = nullptr;
  uint32_t* trow = nullptr;
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
void launch_panel_numeric(const TileMat& A, const TileMat& B, int64_t rows, const uint32_t* row_stage,
                          uint64_t stage_cap, uint2* stage, int64_t* rowcnt, unsigned long long* counted,
                          const unsigned long long* need, unsigned long long* stats, int mode,
                          uint32_t I0, uint32_t I1, cudaStream_t st, const TileEmit* emit = nullptr,
                          const unsigned* gate = nullptr, unsigned* work = nullptr);
// row_bound[r] = min(B.cols, sum over A's entries (r, k) of nnz(B row k));
// *total += sum of row_bound
void launch_elem_bound(const CsrView& A, const int64_t* rpB, int64_t bcols, uint32_t* row_bound,
                       unsigned long long* total, cudaStream_t st);
void launch_emit_compact(uint32_t tile_rows, const TileEmit& em, const uint32_t* trp, TileMat& T, cudaStream_t st);
// bound[I] = min(B.tile_cols, raw pairs of A's tile row I): output tiles of the row at most
void launch_row_tile_bound(const TileMat& A, const TileMat& B, uint32_t* bound, cudaStream_t st);
// dcol (nullable): also writes the host transport -- first[row] = the row's
// first column, dcol[p] = column delta to the previous entry of the row (0 at
// a row start); *ovf |= 1 when some delta exceeds 16 bits
void launch_panel_copy(int64_t rows, const uint32_t* row_stage, const int64_t* row_ptr, const uint2* stage,
                       int32_t* col, float* val, unsigned* err_flag, uint32_t I0, uint32_t I1,
                       cudaStream_t st, uint16_t* dcol = nullptr, int32_t* first = nullptr,
                       unsigned* ovf = nullptr);
// (2) symbolic -- general: enumerate + filter, stable sort, segment heads
void launch_enum_count(const TileMat& A, const TileMat& B, uint64_t tA, uint32_t* tile_cnt,
                       unsigned long long* raw_total, cudaStream_t st);
void launch_enum_fill(const TileMat& A, const TileMat& B, uint64_t tA, const uint32_t* tile_off,
                      uint64_t* pairs, uint32_t* keys, uint32_t key_shift, cudaStream_t st);
void launch_row_pair_off(const TileMat& A, const uint32_t* tile_off, uint32_t* row_pair_off,
                         cudaStream_t st);
void launch_seg_count(const TileMat& A, const uint32_t* row_pair_off, const uint32_t* keys,
                      uint32_t* row_nseg, cudaStream_t st);
void launch_seg_fill(const TileMat& A, const uint32_t* row_pair_off, const uint32_t* keys, uint32_t jmask,
                     TaskList& tl, cudaStream_t st);
// per sorted pair: operand metas and the staging bound popc(rows A) * popc(cols B)
void launch_pair_meta(const TileMat& A, const TileMat& B, const uint64_t* pairs, TaskList& tl,
                      uint32_t* pair_bound, cudaStream_t st);
void launch_seg_stage(const TaskList& tl, const uint32_t* pair_stage, cudaStream_t st);

// (3) numeric -- fused boolean count (counting_pass) + SEaC multiply, staged output.
// Thin segments (tiny staging bound): thread per segment, sequential fp32;
// flags the others in `heavy` (general path, where the tile pairs exist).
void launch_numeric_thin(const TaskList& tl, const TileMat& A, const TileMat& B, Staged& sg, uint8_t* heavy,
                         cudaStream_t st);
// warp per segment over all segments, or over list[0 .. *list_len) when list != null
void launch_numeric(const TaskList& tl, const TileMat& A, const TileMat& B, Staged& sg, int mode,
                    const uint32_t* list, const uint32_t* list_len, cudaStream_t st);

// (4) assembly.  A tile row's segments are cut into chunks of at most
// kChunkSegs (one warp each, so hub tile rows spread over many warps):
//   launch_asm_chunks (chunks per tile row) -> host scan -> launch_asm_chunk_fill
//   launch_row_counts (realised (chunk, row) counts, row totals) -> host scan -> row_ptr
//   launch_chunk_offsets (CSR offset of each chunk's rows) -> launch_assemble
constexpr uint32_t kChunkSegs = 512;
struct AsmChunks {
  uint32_t* n = nullptr;          // number of chunks (device)
  uint32_t* tile_row = nullptr;   // [chunks]
  uint32_t* seg_begin = nullptr;  // [chunks]
  uint32_t* seg_end = nullptr;    // [chunks]
  uint32_t* off = nullptr;        // [chunks*16] row counts, then CSR offsets
};
void launch_asm_chunks(uint32_t tile_rows, const uint32_t* seg_row_ptr, uint32_t* nchunks, cudaStream_t st);
void launch_asm_chunk_fill(uint32_t tile_rows, const uint32_t* seg_row_ptr, const uint32_t* chunk_base,
                           AsmChunks& ch, cudaStream_t st);
void launch_row_counts(int64_t rows, const AsmChunks& ch, uint64_t max_chunks, const Staged& sg,
                       int64_t* rowcnt, cudaStream_t st);
void launch_chunk_offsets(int64_t rows, uint32_t tile_rows, const uint32_t* chunk_base, const int64_t* row_ptr,
                          AsmChunks& ch, cudaStream_t st);
void launch_assemble(int64_t rows, const AsmChunks& ch, uint64_t max_chunks, const TaskList& tl,
                     const Staged& sg, int32_t* col, float* val, unsigned* err_flag, cudaStream_t st);

}  // namespace tsg
