/* tsparse_b200.h -- C ABI of the B200-native tSparse spGEMM path (C = A.B).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (tilemul, /root/reference/proj) is a C++ library whose hot path is the
 * pass chain
 *
 *   from_element_coo                      proj/include/tilemul/tile_format.hpp:71-72
 *   enumerate_pairs / filter_zero_products proj/include/tilemul/pipeline.hpp:46-52
 *   sort_and_segment                      proj/include/tilemul/pipeline.hpp:56-57
 *   counting_pass                         proj/include/tilemul/kernels.hpp:52-53
 *   multiply_pass                         proj/include/tilemul/kernels.hpp:62-64
 *   compact                               proj/include/tilemul/kernels.hpp:67
 *   spgemm_square                         proj/include/tilemul/kernels.hpp:88-89
 *   to_element_coo                        proj/include/tilemul/tile_format.hpp:75
 *
 * tsg_spgemm() replaces that whole chain in one call (sorted duplicate-free
 * COO == CSR, so CSR is the interchange format: SURVEY.md Appendix A.2).
 * tsg_spgemm_chain() replaces the R.A.P composition with the fp32 -> binary16
 * downcast between stages (proj/src/kernels.cpp:239-258).  The per-phase
 * functions are not exported individually: on a GPU they would force a
 * device<->host copy per phase.  include/tilemul_gpu.hpp re-exposes the
 * reference's C++ names (tilemul::spgemm_square etc.) on top of this ABI.
 *
 * Plain C: no torch, no CUDA types.  Pointers are host or device as the
 * `mem` field says.  Every call is synchronous at return and deterministic
 * (byte-identical output for any launch configuration or GPU count).
 * One context per host thread.
 */
#ifndef TSPARSE_B200_H
#define TSPARSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSG_ABI_VERSION 4

/* Only the functions below are exported (the library builds with
 * -fvisibility=hidden). */
#if defined(__GNUC__)
#define TSG_API __attribute__((visibility("default")))
#else
#define TSG_API
#endif

/* Status codes mirror the reference CLI exit codes
 * (proj/tools/tilemul.cpp:30-35,285-306; proj/include/tilemul/errors.hpp:9-51). */
typedef enum {
  TSG_OK = 0,
  TSG_ERR_OTHER = 1,      /* tilemul::Error (anything else), CUDA failures      */
  TSG_ERR_INVARIANT = 2,  /* InvariantError: unsorted/duplicate/out-of-range CSR */
  TSG_ERR_OVERFLOW = 3,   /* OverflowError: |x| > 65504 or non-finite input       */
  TSG_ERR_DIMENSION = 4,  /* DimensionError: A.cols != B.rows                      */
  TSG_ERR_PRECISION = 5   /* PrecisionError: non-finite accumulator               */
} tsg_status;

typedef enum { TSG_F16 = 0, TSG_F32 = 1, TSG_F64 = 2 } tsg_dtype; /* value carrier */
typedef enum { TSG_MEM_HOST = 0, TSG_MEM_DEVICE = 1 } tsg_mem;

/* Numeric mode of the multiply.
 * TENSOR:  fp16 x fp16 -> fp32 on the tensor cores (mma.m16n8k16), the
 *          tSparse design.  Bit-exact wherever partial sums are exact
 *          (integer / dyadic inputs), else within the stated tolerance.
 * ORDERED: CUDA-core fp32 adds, one rounding per product in ascending k,
 *          no FMA contraction: bit-identical to dense_spgemm_mixed_ordered
 *          (proj/src/oracle.cpp:102-121) on every input. */
typedef enum { TSG_MODE_TENSOR = 0, TSG_MODE_ORDERED = 1 } tsg_mode;

/* Read-only CSR view: rows sorted by column, no duplicates (== the
 * reference's ElementCoo invariant, proj/include/tilemul/coo.hpp:11-33). */
typedef struct {
  int64_t rows, cols, nnz;
  const int64_t* row_ptr; /* rows + 1 */
  const int32_t* col;     /* nnz      */
  const void* val;        /* nnz values of type `dtype` (TSG_F16 = binary16 bits) */
  int32_t dtype;          /* tsg_dtype */
  int32_t mem;            /* tsg_mem   */
} tsg_csr;

/* Output CSR, allocated by the library (fp32 values, like compact()'s
 * Fp32Stored output, proj/src/kernels.cpp:205-220).  Release with
 * tsg_free_csr().  `mem` is set by the caller before the call. */
typedef struct {
  int64_t rows, cols, nnz;
  int64_t* row_ptr;
  int32_t* col;
  float* val;
  int32_t mem;
  int32_t _pad;
  void* _owner; /* library bookkeeping */
} tsg_csr_out;

/* Optional 16x16 tiled view of C (pre-CSR), for the tile-structure parity
 * bridge: tile coords, 16 row masks (u16, bit c of row r =
 * slot (r,c)), element offsets (row-major bit order), realised values.
 * Host memory, allocated by the library; release with tsg_free_tiles(). */
typedef struct {
  int64_t ntiles, nnz;
  uint32_t* tile_row;
  uint32_t* tile_col;
  uint16_t* row_masks; /* 16 per tile */
  uint64_t* elem_index;
  float* val;
} tsg_tiles_out;

typedef struct {
  int32_t mode;           /* tsg_mode (default TENSOR)                          */
  int32_t drop_nonfinite; /* from_element_coo(..., drop_nonfinite) semantics    */
  int32_t phase_timing;   /* record CUDA events per phase into tsg_run_stats    */
  int32_t want_tiles;     /* also fill a tsg_tiles_out (host) for parity tests  */
} tsg_options;

/* Phase names follow PhaseTiming (proj/include/tilemul/report.hpp:10-17)
 * plus the two boundary conversions the GPU path owns.  Seconds of device
 * time between CUDA events; zero unless options.phase_timing. */
typedef struct {
  double convert;    /* CSR -> 16x16 tiles (both operands)          */
  double task_list;  /* enumerate + zero-product filter             */
  double sort;       /* per-tile-row sort by output tile, segments  */
  double counting;   /* fused into multiply: always ~0              */
  double multiply;   /* counting + SEaC numeric (one fused kernel)  */
  double compaction; /* tiled -> CSR assembly (zeros already gone) */
  double total;      /* first kernel to last, device time           */
  /* counters (T = 16 tiles) */
  uint64_t tiles_a, tiles_b, raw_pairs, filtered_pairs, segments;
  uint64_t counted_elements; /* symbolic nnz(C), tile-size invariant      */
  uint64_t nnz_c;            /* realised nnz(C)                            */
  uint64_t cbar;             /* sum_k nnzA(:,k) * nnzB(k,:)  (flops / 2)  */
  uint64_t kernel_launches;  /* own kernels launched by this call         */
  uint64_t h2d_bytes, d2h_bytes;
  uint64_t staged_slots;     /* numeric staging capacity (bound on nnz)   */
  /* Device memory of the call in bytes: the B200 counterpart of the
   * reference's MemoryReport (proj/include/tilemul/report.hpp:19-27, filled
   * by memory_report, proj/src/analytics.cpp:120-152).  Allocated sizes by
   * role; mem_peak is the high-water mark of the context's device pool
   * during the call (everything the call held at once, staging arena
   * included).  Summed over the devices of a multi-device context. */
  uint64_t mem_input_tiles;    /* tile records of A and B (trp, tco, masks, metas) */
  uint64_t mem_input_elements; /* operand chunks and rounded binary16 values      */
  uint64_t mem_task_list;      /* work units / output pieces (general rows; the
                                  light-row task list never leaves registers)    */
  uint64_t mem_counting;       /* per-row bounds, offsets and counts              */
  uint64_t mem_pre_compaction; /* staged {column, value} slots                    */
  uint64_t mem_output;         /* output CSR                                      */
  uint64_t mem_peak;
  int32_t path;    /* numeric path of the (last) stage: tsg_path               */
  int32_t devices; /* panel workers (GPUs) the call ran on                     */
} tsg_run_stats;

/* Which numeric kernel a call ran (tsg_run_stats.path). */
typedef enum {
  TSG_PATH_PANEL = 0,      /* light tile rows: panel_numeric_kernel (tensor-core SEaC) */
  TSG_PATH_GENERAL = 1,    /* general tile rows: esc_kernel (element SEaC in smem)      */
  TSG_PATH_PANEL_EMIT = 2  /* chained stage emitting the next stage's A tiles           */
} tsg_path;

typedef struct tsg_ctx tsg_ctx;

TSG_API void tsg_default_options(tsg_options* opt);

/* device < 0: current device.  stream: cudaStream_t or NULL (own stream). */
TSG_API int tsg_create(tsg_ctx** ctx, int device, void* stream);

/* A context over n_devices GPUs (devices[i] = CUDA ordinals; NULL = 0 .. n-1).
 * Every call splits A into n contiguous tile-row panels balanced by work
 * (intermediate products per tile row); panel i runs on
 * devices[i] with its own stream and host thread; B is replicated to every
 * device (peer copies over NVLink from the device holding it, or H2D from
 * host memory); the panels' CSR slices are concatenated in row order into
 * one output on devices[0] (or the host), byte-identical to one GPU.  A
 * chain (tsg_spgemm_chain) splits its first operand the same way: rank p
 * computes X0_p . X1 . ... (AMG's R_p.A.P).  An ordinal may repeat: several
 * panel workers then share one GPU (used to exercise the multi-device path
 * on a single-GPU box).  Device inputs must live on devices[0].  The
 * counterpart of one reference process using every host core
 * (proj/include/tilemul/threading.hpp:14-45). */
TSG_API int tsg_create_multi(tsg_ctx** ctx, int n_devices, const int* devices);

/* Per-panel device times (ms, CUDA events on each panel's stream) of the
 * last call of a multi-device context: out[i] for panel i, n entries at most;
 * returns the panel count.  The max over panels is the call's critical path. */
TSG_API int tsg_last_panel_ms(const tsg_ctx* ctx, double* out, int n);
TSG_API int tsg_destroy(tsg_ctx* ctx);
TSG_API const char* tsg_last_error(const tsg_ctx* ctx);
TSG_API int tsg_abi_version(void);

/* C = A . B.  tiles may be NULL. */
TSG_API int tsg_spgemm(tsg_ctx* ctx, const tsg_csr* A, const tsg_csr* B, tsg_csr_out* C,
               const tsg_options* opt, tsg_run_stats* stats, tsg_tiles_out* tiles);

/* C = X0 . X1 . ... . X{n-1}, left to right; each intermediate is rounded
 * to binary16 (drop exact zeros / underflow, OverflowError beyond 65504)
 * before the next stage, as spgemm_square does for fp32-stored input
 * (proj/src/kernels.cpp:239-258).  stats accumulates over stages. */
TSG_API int tsg_spgemm_chain(tsg_ctx* ctx, int n, const tsg_csr* const* X, tsg_csr_out* C,
                     const tsg_options* opt, tsg_run_stats* stats);

TSG_API void tsg_free_csr(tsg_ctx* ctx, tsg_csr_out* C);
TSG_API void tsg_free_tiles(tsg_tiles_out* t);

/* The reference's 8x8 TiledMatrix (proj/include/tilemul/tile_format.hpp:24-55)
 * as a struct of arrays: tiles sorted by (tile_row, tile_col), bit 8r + c of
 * a 64-bit bitmap marks slot (r, c), each tile's elements contiguous from
 * elem_index in ascending bit order.  Input view (host or device). */
typedef struct {
  int64_t rows, cols, ntiles, nnz;
  const uint32_t* tile_row;
  const uint32_t* tile_col;
  const uint64_t* bitmap;
  const uint64_t* elem_index;
  const float* val;
  int32_t mem; /* tsg_mem */
  int32_t _pad;
} tsg_tiles8;

/* Host output of tsg_csr_to_tiles8, allocated by the library. */
typedef struct {
  int64_t rows, cols, ntiles, nnz;
  uint32_t* tile_row;
  uint32_t* tile_col;
  uint64_t* bitmap;
  uint64_t* elem_index;
  float* val;
} tsg_tiles8_out;

/* 8x8 tiles -> CSR on the GPU (to_element_coo, tile_format.cpp:131-154,
 * without its global sort); C->mem chooses host or device output (fp32). */
TSG_API int tsg_tiles8_to_csr(tsg_ctx* ctx, const tsg_tiles8* T, tsg_csr_out* C);
/* CSR (fp32 values, host or device) -> 8x8 tiles on the GPU, equal to
 * from_element_coo(to COO, Fp32Stored) (tile_format.cpp:61-129): zeros
 * dropped, non-finite values raise status 3.  Host output. */
TSG_API int tsg_csr_to_tiles8(tsg_ctx* ctx, const tsg_csr* C, tsg_tiles8_out* T);
TSG_API void tsg_free_tiles8(tsg_tiles8_out* T);

/* B's share of a general-row product, per row panel of B: the
 * per-row and per-tile summaries the general path reads of B besides its CSR
 * (the 16x16 tile structure behind the T = 16 pair counters, and the binary16
 * values).  In an N-GPU run each GPU summarises its own panel of B rows and
 * the panels are all-gathered -- concatenated in row order, array by array --
 * instead of every GPU converting all of B.  Arrays are device memory on the
 * context's device; tsg_bsum_create allocates them (tsg_bsum_free releases),
 * a gathered summary passed to tsg_spgemm_bsum may live anywhere on that
 * device (e.g. torch tensors).
 *   njt        [rows]        distinct 16x16 tiles each row touches
 *   tile_count [tile_rows]   tiles per 16-row tile row
 *   rinfo      [tile_rows]   rows holding an entry (lo 16 bits) | 1 << 16
 *                            when every tile occupies a single row
 *   ro         [tiles]       row occupancy of each tile (tile-row order)
 *   etile      [nnz]         per entry: its tile's rank in its tile row |
 *                            0x80000000 unless first of its tile in its row;
 *                            0xffffffff when the entry is dropped
 *   h16        [nnz]         per entry: binary16 value (0 = dropped)       */
typedef struct {
  int64_t rows, tile_rows, tiles, nnz;
  uint32_t* njt;
  uint32_t* tile_count;
  uint32_t* rinfo;
  uint16_t* ro;
  uint32_t* etile;
  uint16_t* h16;
  void* _owner;
} tsg_bsum;

/* Summary of a row panel of B given as its own CSR (row_ptr from 0; the
 * panel's first row a multiple of 16 in B).  Validation and binary16
 * rounding as tsg_spgemm's conversion (status 2 / 3). */
TSG_API int tsg_bsum_create(tsg_ctx* ctx, const tsg_csr* Bpanel, tsg_bsum* out);
TSG_API void tsg_bsum_free(tsg_ctx* ctx, tsg_bsum* s);
/* C = A.B as tsg_spgemm, with B's summary given (all of B's rows).  Rows of A
 * that take the general path read B only through Bsum and B's CSR; when A's
 * rows are light the call converts B itself (as tsg_spgemm). */
TSG_API int tsg_spgemm_bsum(tsg_ctx* ctx, const tsg_csr* A, const tsg_csr* B, const tsg_bsum* Bsum,
                            tsg_csr_out* C, const tsg_options* opt, tsg_run_stats* stats);

/* sum_k nnzA(:,k) * nnzB(k,:) on the device (analytics.cpp:51-65,
 * generalised to A != B): the GFLOPS denominator / 2. */
TSG_API int tsg_cbar(tsg_ctx* ctx, const tsg_csr* A, const tsg_csr* B, uint64_t* cbar);

/* Total own-kernel launches by this context since creation. */
TSG_API uint64_t tsg_launch_count(const tsg_ctx* ctx);

/* Device time (ms) of a phase ("convert", "task_list", "sort", "counting",
 * "multiply", "compaction", "total") or of a single kernel launch
 * ("numeric_kernel", "assemble_kernel") during the last call made with
 * phase_timing set, or of the last tsg_bsum_create ("bsum") -- CUDA events
 * on the context's stream. */
TSG_API double tsg_last_kernel_ms(const tsg_ctx* ctx, const char* phase);

#ifdef __cplusplus
}
#endif
#endif /* TSPARSE_B200_H */
