// tsg_kernels.cuh -- launchers of the four subsystems (host side view).
#pragma once
#include <cuda_runtime.h>

#include "tsg_common.cuh"

namespace tsg {

struct CsrView {  // device CSR input
  int64_t rows = 0, cols = 0, nnz = 0;
  const int64_t* row_ptr = nullptr;
  const int32_t* col = nullptr;
  const void* val = nullptr;
  int dtype = 1;  // 0 f16 bits, 1 f32, 2 f64
};

struct TaskList {  // sorted tile-pair task list (pipeline.hpp:22-34 at T=16)
  uint64_t npairs = 0, nseg = 0;
  uint32_t* tile_pair_off = nullptr;  // [tA+1] first pair of each A tile (enumeration order)
  uint32_t* row_pair_off = nullptr;   // [tile_rows+1]
  uint64_t* pairs = nullptr;          // [P] a | b << 32, sorted by (row, J, k)
  uint32_t* keys = nullptr;           // [P] J
  uint32_t* seg_row_ptr = nullptr;    // [tile_rows+1] first segment of each tile row
  uint32_t* seg_off = nullptr;        // [S+1] first pair of each segment
  uint32_t* seg_col = nullptr;        // [S] output tile column J
};

struct OutTiles {  // pre-compaction multiply output (MulResult, kernels.hpp:24-30)
  uint32_t* counted = nullptr;   // [S] boolean upper bound per tile
  uint32_t* elem_off = nullptr;  // [S+1] exclusive prefix of counted
  uint16_t* cmask = nullptr;     // [S*16] realised row masks
  float* vals = nullptr;         // [counted total] row-major bit order per tile
};

// (1) conversion
void launch_convert_count(const CsrView& in, TileMat& out, uint32_t* row_ntiles,
                          uint32_t* row_nvals, unsigned* err_flag, int drop_nonfinite,
                          cudaStream_t st);
void launch_convert_fill(const CsrView& in, TileMat& out, int roles, const uint32_t* tile_base,
                         const uint32_t* val_base, int drop_nonfinite, cudaStream_t st);
void launch_cbar(const int32_t* colA, int64_t nnzA, int64_t inner, const int64_t* rpB,
                 unsigned* hist, unsigned long long* out, cudaStream_t st);

// (2) symbolic
void launch_enum_count(const TileMat& A, const TileMat& B, uint64_t tA, uint32_t* tile_cnt,
                       unsigned long long* raw_total, cudaStream_t st);
void launch_enum_fill(const TileMat& A, const TileMat& B, uint64_t tA, const uint32_t* tile_off,
                      uint64_t* pairs, uint32_t* keys, cudaStream_t st);
void launch_row_pair_off(const TileMat& A, const uint32_t* tile_off, uint32_t* row_pair_off,
                         cudaStream_t st);
void launch_seg_count(const TileMat& A, const uint32_t* row_pair_off, const uint32_t* keys,
                      uint32_t* row_nseg, cudaStream_t st);
void launch_seg_fill(const TileMat& A, const uint32_t* row_pair_off, const uint32_t* keys,
                     const uint32_t* seg_row_ptr, uint32_t* seg_off, uint32_t* seg_col,
                     cudaStream_t st);
void launch_counting(const TileMat& A, const TileMat& B, const TaskList& tl, uint32_t* counted,
                     cudaStream_t st);

// (3) numeric
void launch_numeric(const TileMat& A, const TileMat& B, const TaskList& tl, OutTiles& ot,
                    int mode, unsigned* err_flag, cudaStream_t st);

// (4) output
void launch_out_rowcount(const TileMat& A, int64_t rows, const TaskList& tl, const OutTiles& ot,
                         int64_t* rowcnt, cudaStream_t st);
void launch_out_fill(const TileMat& A, int64_t rows, const TaskList& tl, const OutTiles& ot,
                     const int64_t* row_ptr, int32_t* col, float* val, cudaStream_t st);

}  // namespace tsg
