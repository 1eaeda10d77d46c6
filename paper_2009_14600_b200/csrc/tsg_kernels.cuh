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
struct TaskList {
  uint64_t npairs = 0, nseg = 0;
  uint64_t* pairs = nullptr;        // [P] a | b << 32
  uint4* pmeta = nullptr;           // [P] {A lane mask, A chunk base, B lane mask, B chunk base}
  uint32_t* seg_row_ptr = nullptr;  // [tile_rows+1] first segment of each tile row
  uint32_t* seg_off = nullptr;      // [S+1] first pair of each segment
  uint32_t* seg_col = nullptr;      // [S] output tile column J
  uint32_t* seg_row = nullptr;      // [S] output tile row I
};

// Output sizing and the final CSR (CountResult + compact, kernels.hpp:15-30).
struct OutPlan {
  uint32_t* bm2 = nullptr;    // [S*8] boolean (counted) row masks, interleaved like rm2
  uint8_t* cnt = nullptr;     // [S*16] counted entries per (segment, row)
  uint32_t* pos = nullptr;    // [S*16] CSR position of each (segment, row) run
  int64_t* rowcnt = nullptr;  // [rows+1] counted entries per CSR row
  int64_t* row_ptr = nullptr;
  int32_t* col = nullptr;
  float* val = nullptr;
};

// (1) conversion
void launch_convert_count(const CsrView& in, TileMat& out, uint32_t* row_ntiles,
                          uint32_t* row_nvals, unsigned* err_flag, int drop_nonfinite,
                          cudaStream_t st);
void launch_convert_fill(const CsrView& in, TileMat& out, int roles, const uint32_t* tile_base,
                         const uint32_t* val_base, int drop_nonfinite, cudaStream_t st);
void launch_row_stats(const TileMat& A, unsigned* max_row_tiles, cudaStream_t st);
void launch_cbar(const int32_t* colA, int64_t nnzA, int64_t inner, const int64_t* rpB,
                 unsigned* hist, unsigned long long* out, cudaStream_t st);

// (2) symbolic -- light rows (<= 32 A tiles per tile row): sort-free merge
void launch_merge_count(const TileMat& A, const TileMat& B, uint32_t* row_np, uint32_t* row_ns,
                        uint32_t* row_raw, cudaStream_t st);
void launch_merge_fill(const TileMat& A, const TileMat& B, const uint32_t* row_pair_off,
                       TaskList& tl, cudaStream_t st);
// (2) symbolic -- general: enumerate + filter, stable sort, segment heads
void launch_enum_count(const TileMat& A, const TileMat& B, uint64_t tA, uint32_t* tile_cnt,
                       unsigned long long* raw_total, cudaStream_t st);
void launch_enum_fill(const TileMat& A, const TileMat& B, uint64_t tA, const uint32_t* tile_off,
                      uint64_t* pairs, uint32_t* keys, cudaStream_t st);
void launch_row_pair_off(const TileMat& A, const uint32_t* tile_off, uint32_t* row_pair_off,
                         cudaStream_t st);
void launch_seg_count(const TileMat& A, const uint32_t* row_pair_off, const uint32_t* keys,
                      uint32_t* row_nseg, cudaStream_t st);
void launch_seg_fill(const TileMat& A, const uint32_t* row_pair_off, const uint32_t* keys,
                     TaskList& tl, cudaStream_t st);
void launch_pair_meta(const TileMat& A, const TileMat& B, TaskList& tl, cudaStream_t st);
// counting pass (boolean products on the u8 tensor cores)
void launch_counting(const TileMat& A, const TileMat& B, const TaskList& tl, OutPlan& op,
                     cudaStream_t st);
// counted row sums -> (CUB scan -> row_ptr) -> per (segment, row) positions
void launch_row_counts(int64_t rows, uint32_t tile_rows, const TaskList& tl, OutPlan& op,
                       cudaStream_t st);
void launch_positions(int64_t rows, uint32_t tile_rows, const TaskList& tl, OutPlan& op,
                      cudaStream_t st);

// (3) numeric -- writes the final CSR at the counted positions
void launch_numeric(const TileMat& A, const TileMat& B, const TaskList& tl, OutPlan& op, int mode,
                    unsigned* err_flag, cudaStream_t st);

// (4) compaction fix-up, only when some slot cancelled to zero
void launch_compact_count(int64_t rows, const OutPlan& op, int64_t* rowcnt, cudaStream_t st);
void launch_compact_fill(int64_t rows, const OutPlan& op, const int64_t* new_rp, int32_t* col,
                         float* val, cudaStream_t st);

}  // namespace tsg
