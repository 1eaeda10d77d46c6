// tsg_api.cu -- host driver and C ABI (include/tsparse_b200.h).
//
// Sequences the four subsystems for C = A.B, like spgemm_square
// (proj/src/kernels.cpp:222-302) sequences the reference passes:
//
//   validate row pointers, convert A, B (CSR -> 16x16 tiles)    tsg_convert.cu   "convert"
//   light tile rows (<= 32 tiles, or <= 128 dense tiles): one fused panel
//     pass per tile row -- enumerate, filter, merge-order sort, counting
//     and SEaC multiply on the tensor cores, staged rows -> CSR  tsg_panel.cu     "multiply", "compaction"
//   general tile rows: planning (product histogram, work units), then per
//     unit the element SEaC in shared memory -- enumerate, radix sort by
//     output tile, counting, ordered sums -- pieces -> CSR      tsg_esc.cu       "task_list", "multiply", "compaction"
//
// Everything runs stream-ordered on the context's stream with scratch from
// a stream-ordered memory pool (cudaMallocFromPoolAsync), so steady-state
// calls do not touch the driver allocator.  The host synchronises only to
// read data-dependent sizes; a device-output light call needs one readback.
// Host output overlaps the device->host copy of finished tile-row chunks
// with the computation of later ones (both paths).  A multi-device context
// (tsg_create_multi) runs one panel of A's tile rows per GPU.
#include <cub/device/device_scan.cuh>

#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/tsparse_b200.h"
#include "tsg_kernels.cuh"

namespace tsg {
constexpr int kGatherMax = 48;  // scalars per gathered readback (3 + 2 (kPipeChunks + 1) at most)
constexpr int kPipeChunks = 16;  // max tile-row chunks of the pipelined host-output path (TSG_PIPE, default 8)
// Tuning switches for A/B runs: read from the environment once
// per name and process; the defaults are the measured best.
int tuning_variant(const char* name, int dflt) {
  static std::mutex mu;
  static std::vector<std::pair<std::string, int>> seen;
  std::lock_guard<std::mutex> g(mu);
  for (const auto& [n, v] : seen)
    if (n == name) return v;
  const char* e = std::getenv(name);
  const int v = e ? std::atoi(e) : dflt;
  seen.emplace_back(name, v);
  return v;
}
int pipe_chunks() {
  static const int n = std::max(1, std::min(kPipeChunks, tuning_variant("TSG_PIPE", 8)));
  return n;
}
}  // namespace tsg

struct tsg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaMemPool_t pool = nullptr;
  uint64_t* pinned = nullptr;  // small pinned readback buffer
  std::string err;
  uint64_t launches = 0;
  double last_phase_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double last_numeric_kernel_ms = 0, last_assemble_kernel_ms = 0;
  double last_bsum_ms = 0;  // device time of the last tsg_bsum_create
  // pipelined host output: a second stream for device->host slices, its events,
  // and pinned slots for the chunk ends
  cudaStream_t d2h = nullptr;
  cudaEvent_t pipe_ev[tsg::kPipeChunks + 1] = {};
  void* pinned_pipe = nullptr;
  cudaEvent_t d2h_ev[tsg::kPipeChunks] = {};  // chunk c's slices landed on the host
  cudaEvent_t ev[8] = {};
  cudaEvent_t kev[4] = {};  // bracket the numeric and assembly kernels alone
  // pinned host blocks released by tsg_free_csr, reused by later host outputs
  std::vector<std::pair<void*, size_t>> pinned_free;
  // grow-only device arena for the numeric staging buffer (the one large,
  // data-sized scratch of a call): kept across calls so steady-state calls
  // never ask the pool for gigabytes at a new size
  void* stage_buf = nullptr;
  size_t stage_cap = 0;
  // multi-device context (tsg_create_multi): one single-device context per
  // panel worker; panel i runs on sub[i]; the last call's per-panel times
  std::vector<tsg_ctx*> sub;
  std::vector<double> panel_ms;
};

namespace {

using namespace tsg;

struct Fail {
  int code;
  std::string msg;
};

#define TSG_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw Fail{TSG_ERR_OTHER, std::string(#call) + ": " + cudaGetErrorString(e_)};    \
  } while (0)

// Stream-ordered scratch, released (to the pool) when the scope ends.
// Allocations are tallied by role (the MemoryReport fields of tsg_run_stats).
enum MemCat : int { kMemTiles = 0, kMemElements, kMemTaskList, kMemCounting, kMemStaging, kMemOutput, kMemCats };
struct Scratch {
  tsg_ctx* ctx;
  std::vector<void*> ptrs;
  int cat = kMemCounting;          // role of the next allocations
  uint64_t bytes[kMemCats] = {};   // bytes allocated per role
  explicit Scratch(tsg_ctx* c) : ctx(c) {}
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, ctx->stream);
  }
  template <class T>
  T* alloc(uint64_t n, bool keep = false) {
    if (n == 0) n = 1;
    void* p = nullptr;
    TSG_CUDA(cudaMallocFromPoolAsync(&p, n * sizeof(T), ctx->pool, ctx->stream));
    if (!keep) ptrs.push_back(p);
    bytes[cat] += n * sizeof(T);
    return static_cast<T*>(p);
  }
};
// RAII role switch for a block of allocations
struct MemRole {
  Scratch& sc;
  int prev;
  MemRole(Scratch& s, int c) : sc(s), prev(s.cat) { s.cat = c; }
  ~MemRole() { sc.cat = prev; }
};

void check_launch(tsg_ctx* ctx, int n = 1) {
  ctx->launches += n;
  TSG_CUDA(cudaGetLastError());
}

template <class T>
T readback(tsg_ctx* ctx, const T* dptr) {
  TSG_CUDA(cudaMemcpyAsync(ctx->pinned, dptr, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  TSG_CUDA(cudaStreamSynchronize(ctx->stream));
  T v;
  std::memcpy(&v, ctx->pinned, sizeof(T));
  return v;
}

// Sum of n u32 (exact, u64) -- guards every u32 offset array against wrap.
__global__ void sum_u32_kernel(const uint32_t* __restrict__ in, uint64_t n,
                               unsigned long long* __restrict__ out) {
  unsigned long long acc = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    acc += in[i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

template <class Tin, class Tout>
void exclusive_sum(tsg_ctx* ctx, Scratch& sc, const Tin* in, Tout* out, uint64_t n) {
  size_t bytes = 0;
  TSG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, ctx->stream));
  void* tmp = sc.alloc<char>(bytes);
  TSG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, ctx->stream));
}

uint64_t total_u32(tsg_ctx* ctx, Scratch& sc, const uint32_t* in, uint64_t n) {
  auto* d = sc.alloc<unsigned long long>(1);
  TSG_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), ctx->stream));
  if (n) {
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    sum_u32_kernel<<<unsigned(blocks), 256, 0, ctx->stream>>>(in, n, d);
    check_launch(ctx);
  }
  return readback(ctx, d);
}

void record(tsg_ctx* ctx, bool timing, int i) {
  if (timing) TSG_CUDA(cudaEventRecord(ctx->ev[i], ctx->stream));
}

size_t dtype_size(int dt) { return dt == TSG_F16 ? 2 : dt == TSG_F32 ? 4 : 8; }

void check_csr(const tsg_csr* M, const char* name) {
  if (!M) throw Fail{TSG_ERR_OTHER, std::string(name) + " is NULL"};
  if (M->rows < 0 || M->cols < 0 || M->nnz < 0)
    throw Fail{TSG_ERR_INVARIANT, std::string(name) + ": negative dimension"};
  if (M->dtype < TSG_F16 || M->dtype > TSG_F64)
    throw Fail{TSG_ERR_OTHER, std::string(name) + ": unknown dtype"};
  if (M->rows > (int64_t(1) << 35) || M->cols > (int64_t(1) << 31) - 16)
    throw Fail{TSG_ERR_OTHER, std::string(name) + ": dimensions beyond the 16x16 tile index range"};
  if (M->nnz >= (int64_t(1) << 29))
    throw Fail{TSG_ERR_OTHER, std::string(name) + ": nnz beyond 2^29 needs row-panel batching"};
  if ((M->rows > 0 || M->nnz > 0) && (!M->row_ptr || (M->nnz > 0 && (!M->col || !M->val))))
    throw Fail{TSG_ERR_OTHER, std::string(name) + ": missing arrays"};
  // host row pointers: the endpoints here (the full check, also for device
  // input, is validate_rowptr_kernel before any entry is read)
  if (M->mem == TSG_MEM_HOST && M->row_ptr && (M->row_ptr[0] != 0 || M->row_ptr[M->rows] != M->nnz))
    throw Fail{TSG_ERR_INVARIANT, std::string(name) + ": row_ptr[0] must be 0 and row_ptr[rows] must equal nnz"};
}

// Device view of a CSR (copies host input; the H2D bytes are counted).
CsrView stage(tsg_ctx* ctx, Scratch& sc, const tsg_csr* M, tsg_run_stats* st) {
  CsrView v;
  v.rows = M->rows;
  v.cols = M->cols;
  v.nnz = M->nnz;
  v.dtype = M->dtype;
  if (M->mem == TSG_MEM_DEVICE) {
    v.row_ptr = M->row_ptr;
    v.col = M->col;
    v.val = M->val;
    return v;
  }
  auto* rp = sc.alloc<int64_t>(M->rows + 1);
  auto* col = sc.alloc<int32_t>(M->nnz);
  auto* val = sc.alloc<char>(M->nnz * dtype_size(M->dtype));
  const size_t b0 = (M->rows + 1) * sizeof(int64_t), b1 = M->nnz * sizeof(int32_t),
               b2 = M->nnz * dtype_size(M->dtype);
  TSG_CUDA(cudaMemcpyAsync(rp, M->row_ptr, b0, cudaMemcpyHostToDevice, ctx->stream));
  if (M->nnz) {
    TSG_CUDA(cudaMemcpyAsync(col, M->col, b1, cudaMemcpyHostToDevice, ctx->stream));
    TSG_CUDA(cudaMemcpyAsync(val, M->val, b2, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (st) st->h2d_bytes += b0 + b1 + b2;
  v.row_ptr = rp;
  v.col = col;
  v.val = val;
  return v;
}

// Several device scalars -> host with one synchronisation.
template <class T, int N>
void readback_many(tsg_ctx* ctx, const T* const (&src)[N], T (&dst)[N]) {
  static_assert(N * sizeof(T) <= 48, "pinned staging is 64 bytes");
  for (int i = 0; i < N; ++i)
    TSG_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(ctx->pinned) + i * sizeof(T), src[i], sizeof(T),
                             cudaMemcpyDeviceToHost, ctx->stream));
  TSG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(dst, ctx->pinned, N * sizeof(T));
}

// Chunk c's end offset and the error flags written straight into pinned host
// memory (mapped under UVA) by the device: a small cudaMemcpy here would
// queue on the copy engine behind the large D2H slices of earlier chunks and
// stall the compute stream.
__global__ void publish_chunk_kernel(const int64_t* __restrict__ end, const unsigned* __restrict__ ovf,
                                     int64_t* ends_h, unsigned* ovf_h) {
  *reinterpret_cast<volatile int64_t*>(ends_h) = *end;
  *reinterpret_cast<volatile unsigned*>(ovf_h) = *ovf;
  __threadfence_system();
}

// Device scalars (u32 or u64) -> host in one copy and one synchronisation:
// a one-block kernel gathers them into a device array first.
struct ScalarGather {
  const void* p[kGatherMax];
  uint32_t wide = 0;  // bit i: p[i] is a u64
  int n = 0;
};
__global__ void gather_scalars_kernel(ScalarGather g, unsigned long long* out) {
  const int i = threadIdx.x;
  if (i < g.n)
    out[i] = ((g.wide >> i) & 1u) ? *static_cast<const unsigned long long*>(g.p[i])
                                  : *static_cast<const uint32_t*>(g.p[i]);
}
void readback_gather(tsg_ctx* ctx, Scratch& sc, const ScalarGather& g, unsigned long long* dst) {
  auto* d = sc.alloc<unsigned long long>(kGatherMax);
  gather_scalars_kernel<<<1, 32, 0, ctx->stream>>>(g, d);
  check_launch(ctx);
  unsigned long long* h = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(ctx->pinned) + 64);
  TSG_CUDA(cudaMemcpyAsync(h, d, g.n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  TSG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(dst, h, g.n * sizeof(unsigned long long));
}

// CSR -> 16x16 tiles (one conversion pass at gapped slots, scan of the tile
// counts, compaction of the tile metadata).  No host synchronisation: every
// array is sized by the input nnz (an upper bound on tiles and chunks).
// Returns the device address of the tile count (trp[tile_rows]).
const uint32_t* convert(tsg_ctx* ctx, Scratch& sc, const CsrView& in, TileMat& T, int roles,
                        unsigned* err_flag, int drop_nonfinite, const uint8_t* needed = nullptr,
                        uint8_t* mark = nullptr, uint32_t* walk_count_zeroed = nullptr,
                        unsigned* max_row_tiles = nullptr, unsigned* general = nullptr) {
  T.rows = in.rows;
  T.cols = in.cols;
  T.tile_rows = uint32_t((in.rows + 15) / 16);
  T.tile_cols = uint32_t((in.cols + 15) / 16);
  const uint64_t nr = uint64_t(T.tile_rows) + 1;
  const uint64_t cap = uint64_t(in.nnz);
  T.cap = cap;
  MemRole role_tiles(sc, kMemTiles);
  ConvertScratch cs;
  cs.rm2 = sc.alloc<uint32_t>(cap * 8);
  cs.ntiles = sc.alloc<uint32_t>(nr);
  cs.walk_list = sc.alloc<uint32_t>(nr);
  cs.mark = mark;
  cs.general = general;
  if (walk_count_zeroed) {
    cs.walk_count = walk_count_zeroed;
  } else {
    cs.walk_count = sc.alloc<uint32_t>(1);
    TSG_CUDA(cudaMemsetAsync(cs.walk_count, 0, sizeof(uint32_t), ctx->stream));
  }
  // ntiles[tile_rows] and chunk 0 of each role are zeroed by the fast kernel
  // (which is not launched for an empty matrix)
  if (T.tile_rows == 0) TSG_CUDA(cudaMemsetAsync(cs.ntiles, 0, sizeof(uint32_t), ctx->stream));
  if (roles & 2) {
    T.etile = sc.alloc<uint32_t>(cap);
    T.csr_rp = in.row_ptr;
  }
  {
    MemRole role_el(sc, kMemElements);
    T.h16 = sc.alloc<uint16_t>(cap);
    for (int role = 0; role < 2; ++role)
      if (roles & (1 << role)) T.chunk[role] = sc.alloc<uint4>(cap + 1);
  }
  for (int role = 0; role < 2; ++role)
    if (roles & (1 << role)) cs.rec[role] = sc.alloc<uint4>(cap);
  launch_validate_rowptr(in, err_flag, ctx->stream);
  launch_convert(in, T, roles, cs, err_flag, drop_nonfinite, needed, ctx->stream);
  check_launch(ctx, 4);
  T.trp = sc.alloc<uint32_t>(nr);
  exclusive_sum(ctx, sc, cs.ntiles, T.trp, nr);
  T.tco = sc.alloc<uint2>(cap);
  T.rm2 = sc.alloc<uint32_t>(cap * 8);
  for (int role = 0; role < 2; ++role) {
    if (!(roles & (1 << role))) continue;
    T.meta[role] = sc.alloc<uint2>(cap);
    T.rec[role] = sc.alloc<uint4>(cap);
  }
  launch_tiles_compact(in, cs, T, roles, ctx->stream, max_row_tiles);
  check_launch(ctx);
  return T.trp + nr - 1;
}

void raise_flags(unsigned flags) {
  if (flags & kErrRowPtr)
    throw Fail{TSG_ERR_INVARIANT, "CSR row pointers malformed (row_ptr[0] != 0, row_ptr[rows] != nnz, or decreasing)"};
  if (flags & kErrInvariant)
    throw Fail{TSG_ERR_INVARIANT, "CSR entries unsorted, duplicated, or out of range"};
  if (flags & kErrOverflow)
    throw Fail{TSG_ERR_OVERFLOW, "value outside binary16 finite range (|x| <= 65504) or non-finite"};
  if (flags & kErrPrecision)
    throw Fail{TSG_ERR_PRECISION, "non-finite accumulator in multiplication pass"};
}

struct OutOwner {  // device or pinned-host output buffers
  bool host = false;
  void* p[3] = {nullptr, nullptr, nullptr};
  size_t sz[3] = {0, 0, 0};
};

// Pinned host block from the context cache (best fit) or cudaMallocHost.
void* pinned_alloc(tsg_ctx* ctx, size_t bytes, size_t* got) {
  if (bytes == 0) bytes = 1;
  size_t best = SIZE_MAX, bi = 0;
  for (size_t i = 0; i < ctx->pinned_free.size(); ++i) {
    const size_t sz = ctx->pinned_free[i].second;
    if (sz >= bytes && sz < best) {
      best = sz;
      bi = i;
    }
  }
  if (best != SIZE_MAX) {
    void* p = ctx->pinned_free[bi].first;
    *got = best;
    ctx->pinned_free.erase(ctx->pinned_free.begin() + bi);
    return p;
  }
  void* p = nullptr;
  TSG_CUDA(cudaMallocHost(&p, bytes));
  *got = bytes;
  return p;
}

// Host-side 16x16 tiled view of a CSR (pattern + values), for the parity
// bridge only (tsg_tiles_out).  Tiles sorted by (row, col), row-major slots.
void tiles_from_csr(int64_t rows, const std::vector<int64_t>& rp, const std::vector<int32_t>& col,
                    const std::vector<float>& val, tsg_tiles_out* out) {
  struct Ent {
    uint64_t key;  // tile_row << 32 | tile_col
    uint32_t slot;
    float v;
  };
  std::vector<Ent> e;
  e.reserve(col.size());
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t p = rp[r]; p < rp[r + 1]; ++p)
      e.push_back({(uint64_t(r >> 4) << 32) | uint32_t(col[p] >> 4),
                   uint32_t((r & 15) * 16 + (col[p] & 15)), val[p]});
  std::stable_sort(e.begin(), e.end(), [](const Ent& a, const Ent& b) {
    return a.key != b.key ? a.key < b.key : a.slot < b.slot;
  });
  std::vector<uint32_t> tr, tc;
  std::vector<uint16_t> rm;
  std::vector<uint64_t> ei;
  for (size_t i = 0; i < e.size();) {
    const uint64_t k = e[i].key;
    tr.push_back(uint32_t(k >> 32));
    tc.push_back(uint32_t(k));
    ei.push_back(i);
    uint16_t m[16] = {0};
    for (; i < e.size() && e[i].key == k; ++i) m[e[i].slot >> 4] |= uint16_t(1u << (e[i].slot & 15));
    rm.insert(rm.end(), m, m + 16);
  }
  auto dup = [](const void* src, size_t bytes) {
    void* p = std::malloc(bytes ? bytes : 1);
    if (bytes) std::memcpy(p, src, bytes);
    return p;
  };
  std::vector<float> vv(e.size());
  for (size_t i = 0; i < e.size(); ++i) vv[i] = e[i].v;
  out->ntiles = int64_t(tr.size());
  out->nnz = int64_t(vv.size());
  out->tile_row = static_cast<uint32_t*>(dup(tr.data(), tr.size() * 4));
  out->tile_col = static_cast<uint32_t*>(dup(tc.data(), tc.size() * 4));
  out->row_masks = static_cast<uint16_t*>(dup(rm.data(), rm.size() * 2));
  out->elem_index = static_cast<uint64_t*>(dup(ei.data(), ei.size() * 8));
  out->val = static_cast<float*>(dup(vv.data(), vv.size() * 4));
}

// One tsg_spgemm call.  The phases share the call's stream, scratch and
// output bookkeeping, so they are members of one object; spgemm_impl runs
// them in order (the pass chain of spgemm_square, kernels.cpp:222-302).
struct Call {
  tsg_ctx* ctx;
  const tsg_csr* Ain;
  const tsg_csr* Bin;
  tsg_csr_out* C;
  const tsg_options& opt;
  tsg_run_stats* st;
  const bool timing;
  cudaStream_t s;
  Scratch sc;
  uint64_t launches0;

  unsigned long long* zblk = nullptr;  // zero-initialised scalars (convert_operands)
  unsigned* dscal = nullptr;  // [0] error flags, [1] max A tiles per tile row
  unsigned* work = nullptr;
  unsigned* err_flag = nullptr;
  bool same = false;
  CsrView dA, dB;
  TileMat TA, TB_own;
  const TileMat* TB = nullptr;
  uint64_t tA = 0, tB = 0;
  bool light = false;
  int path = TSG_PATH_PANEL;  // numeric kernel that ran (tsg_run_stats.path)
  int nl = 1;  // merge lists per lane of the light-row pass (tile rows of up to 32 nl A tiles)

  // Light-row (tensor-core panel) pass or general rows (element SEaC): tile
  // rows of at most 32 A tiles always take the panel pass; up to 128 when the
  // tiles are dense enough for the MMA to pay (>= 4 entries per A tile on
  // average; a chained stage's A is a product, dense); thinner or longer tile
  // rows take the general path.
  void decide(uint32_t max_row_tiles) {
    nl = max_row_tiles <= 32 ? 1 : max_row_tiles <= 64 ? 2 : 4;
    const bool dense = pre_a || (tA > 0 && uint64_t(dA.nnz) >= 4 * tA);
    light = max_row_tiles <= 32 || (max_row_tiles <= 128 && dense);
  }

  int64_t rows = 0;
  uint64_t nr = 0;  // tile rows + 1
  uint64_t P = 0, S = 0, raw = 0, stage_total = 0, counted = 0;
  int64_t nnzC = 0;
  OutOwner* owner = nullptr;
  bool host_done = false;  // the pipelined light path ships the output itself
  int64_t* d_rp = nullptr;
  int32_t* d_col = nullptr;
  float* d_val = nullptr;
  unsigned long long* counted_d = nullptr;
  int64_t* rowcnt = nullptr;  // realised entries per CSR row

  // chained products: A given as tiles by the previous stage (pre_a), and/or
  // this stage's result emitted as the next stage's A tiles (emit_out); the
  // emitted arrays outlive this call and are listed in `keep`
  const TileMat* pre_a = nullptr;
  TileMat* emit_out = nullptr;
  // B's summary (tsg_spgemm_bsum): the general path reads B through it and
  // B's CSR; B is converted only if the rows turn out light
  const tsg_bsum* bsum = nullptr;
  unsigned long long* emit_tot = nullptr;  // emit mode: P, S, raw accumulated by the numeric pass
  std::vector<void*>* keep = nullptr;

  Call(tsg_ctx* c, const tsg_csr* a, const tsg_csr* b, tsg_csr_out* out, const tsg_options& o,
       tsg_run_stats* stats)
      : ctx(c), Ain(a), Bin(b), C(out), opt(o), st(stats), timing(o.phase_timing != 0), s(c->stream),
        sc(c), launches0(c->launches) {
    // the pool's high-water mark restarts at what is held now (mem_peak)
    uint64_t zero = 0;
    cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrUsedMemHigh, &zero);
  }

  // ---- (1) validation, staging of host inputs, CSR -> 16x16 tiles ----------------
  // readback of the conversion results deferred to the speculative light pass
  const unsigned* ntA_dev = nullptr;
  const unsigned* ntB_dev = nullptr;

  // zeroed with the call's scalars (the high half of zblk[6]): set by A's
  // conversion when a tile row has more than 128 tiles (the call is general)
  unsigned* general_flag() { return reinterpret_cast<unsigned*>(zblk + 6) + 1; }

  void convert_operands(bool defer = false) {
    if (!pre_a) check_csr(Ain, "A");
    check_csr(Bin, "B");
    if (!C) throw Fail{TSG_ERR_OTHER, "C is NULL"};
    if (Ain->cols != Bin->rows)
      throw Fail{TSG_ERR_DIMENSION, "inner dimensions differ: A is " + std::to_string(Ain->rows) + "x" +
                                        std::to_string(Ain->cols) + ", B is " + std::to_string(Bin->rows) +
                                        "x" + std::to_string(Bin->cols)};
    record(ctx, timing, 0);
    // the call's small zero-initialised device scalars, one memset:
    // [0] error flags + max A tiles per tile row, [1] counted, [2..5] totals
    // of the speculative light pass, [6] [7] the conversions' walk counters
    zblk = sc.alloc<unsigned long long>(8);
    TSG_CUDA(cudaMemsetAsync(zblk, 0, 8 * sizeof(unsigned long long), s));
    dscal = reinterpret_cast<unsigned*>(zblk);
    counted_d = zblk + 1;
    work = sc.alloc<unsigned>(1);  // tile-row counter of the persistent numeric pass
    err_flag = dscal;
    same = !pre_a && !bsum && (Ain == Bin || (Ain->row_ptr == Bin->row_ptr && Ain->col == Bin->col &&
                                     Ain->val == Bin->val && Ain->rows == Bin->rows && Ain->cols == Bin->cols &&
                                     Ain->mem == Bin->mem && Ain->dtype == Bin->dtype && Ain->nnz == Bin->nnz));
    const uint32_t* ntA_d;
    // the B tile rows A's tiles refer to (A's tile columns), marked by A's
    // conversion: only those are tiled (a row panel of A -- multi-GPU, or any
    // A that touches part of B -- converts its slice of B)
    uint8_t* needed = nullptr;
    if (!same && !bsum) {
      needed = sc.alloc<uint8_t>((Bin->rows + 15) / 16 + 1);
      TSG_CUDA(cudaMemsetAsync(needed, 0, (Bin->rows + 15) / 16 + 1, s));
    }
    if (pre_a) {  // the previous stage's emitted tiles
      TA = *pre_a;
      ntA_d = TA.trp + TA.tile_rows;
      if (needed) {
        launch_mark_needed(TA, needed, s);
        check_launch(ctx);
      }
    } else {
      dA = stage(ctx, sc, Ain, st);
      ntA_d = convert(ctx, sc, dA, TA, same ? 3 : 1, err_flag, opt.drop_nonfinite, nullptr, needed,
                      reinterpret_cast<uint32_t*>(zblk + 6), dscal + 1, general_flag());
    }
    dB = same ? dA : stage(ctx, sc, Bin, st);
    const uint32_t* ntB_d = ntA_d;
    if (bsum)
      ntB_d = bsum_view();
    else if (!same)
      ntB_d = convert(ctx, sc, dB, TB_own, 2, err_flag, opt.drop_nonfinite, needed, nullptr,
                      reinterpret_cast<uint32_t*>(zblk + 7), nullptr, general_flag());
    TB = same ? &TA : &TB_own;
    if (pre_a) {  // converted A tiles report their largest tile row in the compaction
      launch_row_stats(TA, dscal + 1, s);
      check_launch(ctx);
    }
    ntA_dev = ntA_d;
    ntB_dev = ntB_d;
    if (!defer) {
      const unsigned* src[4] = {dscal, dscal + 1, ntA_d, ntB_d};
      unsigned v[4];
      readback_many(ctx, src, v);
      raise_flags(v[0]);
      tA = v[2];
      tB = v[3];
      if (bsum && tB != uint64_t(bsum->tiles))
        throw Fail{TSG_ERR_DIMENSION, "B summary: tile counts sum to " + std::to_string(tB) + ", not its " +
                                          std::to_string(bsum->tiles) + " tiles"};
      decide(v[1]);
    }
    record(ctx, timing, 1);

    rows = Ain->rows;
    nr = uint64_t(TA.tile_rows) + 1;
    owner = new OutOwner();
    owner->host = C->mem == TSG_MEM_HOST;
    C->_owner = owner;  // released by free_out on any later failure
    {
      MemRole role_out(sc, kMemOutput);
      d_rp = owner->host ? sc.alloc<int64_t>(rows + 1) : sc.alloc<int64_t>(rows + 1, true);
    }
    if (!owner->host) owner->p[0] = d_rp;
    rowcnt = sc.alloc<int64_t>(rows + 1);  // rowcnt[rows] = 0: written by the numeric kernels
    TSG_CUDA(cudaMemsetAsync(rowcnt + rows, 0, sizeof(int64_t), s));
  }

  // B as its summary: tile-row pointers from the tile counts, per-tile row
  // occupancies, per-entry tile ranks and binary16 values (tsg_bsum); returns
  // the device tile count
  const uint32_t* bsum_view() {
    const int64_t tr = (Bin->rows + 15) / 16;
    if (bsum->rows != Bin->rows || bsum->nnz != Bin->nnz || bsum->tile_rows != tr)
      throw Fail{TSG_ERR_DIMENSION, "B summary does not match B (rows " + std::to_string(bsum->rows) + ", nnz " +
                                        std::to_string(bsum->nnz) + ", tile rows " + std::to_string(bsum->tile_rows) +
                                        ")"};
    if ((tr && (!bsum->tile_count || !bsum->rinfo || !bsum->njt)) ||
        (bsum->nnz && (!bsum->etile || !bsum->h16)) || (bsum->tiles && !bsum->ro))
      throw Fail{TSG_ERR_OTHER, "B summary arrays missing"};
    TB_own = TileMat{};
    TB_own.rows = Bin->rows;
    TB_own.cols = Bin->cols;
    TB_own.tile_rows = uint32_t(tr);
    TB_own.tile_cols = uint32_t((Bin->cols + 15) / 16);
    const uint64_t nr1 = uint64_t(tr) + 1;
    auto* cnt = sc.alloc<uint32_t>(nr1);
    if (tr) TSG_CUDA(cudaMemcpyAsync(cnt, bsum->tile_count, tr * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    TSG_CUDA(cudaMemsetAsync(cnt + tr, 0, sizeof(uint32_t), s));
    TB_own.trp = sc.alloc<uint32_t>(nr1);
    exclusive_sum(ctx, sc, cnt, TB_own.trp, nr1);
    TB_own.ro16 = bsum->ro;
    TB_own.etile = bsum->etile;
    TB_own.csr_rp = dB.row_ptr;
    TB_own.h16 = bsum->h16;
    return TB_own.trp + tr;
  }

  // B converted after all (a summary call whose rows are light)
  void convert_b() {
    const uint32_t* ntB_d = convert(ctx, sc, dB, TB_own, 2, err_flag, opt.drop_nonfinite, nullptr, nullptr,
                                    reinterpret_cast<uint32_t*>(zblk + 7), nullptr, general_flag());
    TB = &TB_own;
    const unsigned* src[2] = {dscal, ntB_d};
    unsigned v[2];
    readback_many(ctx, src, v);
    raise_flags(v[0]);
    tB = v[1];
  }

  // realised row counts -> row_ptr; nnz(C) and counted elements to the host,
  // plus (optionally) four more contiguous device totals in the same sync
  void scan_rows(const unsigned long long* extra = nullptr, unsigned long long* out = nullptr, bool check = true) {
    exclusive_sum(ctx, sc, rowcnt, d_rp, uint64_t(rows) + 1);
    const unsigned long long* nz = reinterpret_cast<const unsigned long long*>(d_rp + rows);
    unsigned long long v[6];
    if (extra) {
      const unsigned long long* src[6] = {counted_d, nz, extra, extra + 1, extra + 2, extra + 3};
      readback_many(ctx, src, v);
      for (int i = 0; i < 4; ++i) out[i] = v[2 + i];
    } else {
      const unsigned long long* src[2] = {counted_d, nz};
      readback_many(ctx, src, *reinterpret_cast<unsigned long long(*)[2]>(v));
    }
    counted = v[0];
    nnzC = int64_t(v[1]);
    if (check && uint64_t(nnzC) >= (uint64_t(1) << 32))
      throw Fail{TSG_ERR_OTHER, "output beyond 2^32 elements needs row-panel batching"};
  }

  void alloc_out() {
    MemRole role_out(sc, kMemOutput);
    d_col = sc.alloc<int32_t>(nnzC, !owner->host);
    d_val = sc.alloc<float>(nnzC, !owner->host);
    if (!owner->host) {
      owner->p[1] = d_col;
      owner->p[2] = d_val;
    }
  }

  // grow-only staging arena (bytes)
  void* arena(size_t need) {
    need = std::max<size_t>(need, 16);
    if (need > ctx->stage_cap) {
      if (ctx->stage_buf) TSG_CUDA(cudaFreeAsync(ctx->stage_buf, s));
      ctx->stage_buf = nullptr;
      ctx->stage_cap = 0;
      const size_t cap = need + need / 4;
      TSG_CUDA(cudaMallocFromPoolAsync(&ctx->stage_buf, cap, ctx->pool, s));
      ctx->stage_cap = cap;
    }
    return ctx->stage_buf;
  }

  void check_stage_total() const {
    if (stage_total >= (uint64_t(1) << 32))
      throw Fail{TSG_ERR_OTHER, "staged slots beyond 2^32 need row-panel batching"};
  }

  // ---- light rows: one fused pass per tile row (tsg_panel.cu) --------------------
  // Device output, CSR operands, staging arena in place: the whole light
  // pass is enqueued before the conversion results are read -- the numeric
  // kernel itself returns when the rows are not light, the input is invalid
  // or the arena is too small -- and ONE synchronisation then reads the
  // conversion results, the statistics and nnz(C).  Returns false when the
  // rows are not light (the caller takes the general path).
  bool light_speculative() {
    auto* row_bound = sc.alloc<uint32_t>(rows + 1);
    auto* row_stage = sc.alloc<uint32_t>(rows + 1);
    TSG_CUDA(cudaMemsetAsync(row_bound + rows, 0, 4, s));
    auto* tot_d = zblk + 2;  // zeroed with the call's scalars
    launch_elem_bound(dA, dB.row_ptr, Bin->cols, row_bound, tot_d + 3, err_flag, s);
    check_launch(ctx);
    exclusive_sum(ctx, sc, row_bound, row_stage, uint64_t(rows) + 1);
    record(ctx, timing, 2);
    record(ctx, timing, 3);
    record(ctx, timing, 4);
    uint2* stage = static_cast<uint2*>(ctx->stage_buf);
    const uint64_t cap_slots = ctx->stage_cap / sizeof(uint2);
    // TSG_TC05=1: the tcgen05 variant of the light pass (TENSOR mode; the
    // measured comparison of DESIGN.md §6)
    const bool tc05 = opt.mode == TSG_MODE_TENSOR && tuning_variant("TSG_TC05", 0) == 1;
    unsigned* fallback = sc.alloc<unsigned>(1);
    TSG_CUDA(cudaMemsetAsync(fallback, 0, sizeof(unsigned), s));
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[0], s));
    if (tc05)
      TSG_CUDA(launch_tc05_panel(TA, *TB, rows, row_stage, cap_slots, stage, rowcnt, counted_d, tot_d + 3, tot_d, dscal,
                                 work, fallback, ctx->device, s));
    else
      TSG_CUDA(launch_panel_numeric(TA, *TB, rows, row_stage, cap_slots, stage, rowcnt, counted_d, tot_d + 3, tot_d,
                                    opt.mode, 0, TA.tile_rows, s, nullptr, dscal, work, 1));
    check_launch(ctx);
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[1], s));
    record(ctx, timing, 5);
    exclusive_sum(ctx, sc, rowcnt, d_rp, uint64_t(rows) + 1);
    ScalarGather g;
    const void* ps[11] = {dscal, dscal + 1, ntA_dev, ntB_dev, counted_d, d_rp + rows, tot_d, tot_d + 1, tot_d + 2,
                          tot_d + 3, fallback};
    for (int i = 0; i < 11; ++i) g.p[i] = ps[i];
    g.wide = 0x3f0u;  // counted, nnz and the four totals are u64
    g.n = 11;
    unsigned long long v[11];
    readback_gather(ctx, sc, g, v);
    raise_flags(unsigned(v[0]));
    tA = v[2];
    tB = v[3];
    decide(unsigned(v[1]));
    if (!light) return false;
    if (nl > 1) {  // the speculative pass (one merge list) stood down: the multi-list pass
      light_path();
      return true;
    }
    counted = v[4];
    nnzC = int64_t(v[5]);
    P = v[6];
    S = v[7];
    raw = v[8];
    stage_total = v[9];
    if (stage_total >> 32) {  // element bound beyond the u32 staging offsets: the tight bound
      TSG_CUDA(cudaMemsetAsync(counted_d, 0, sizeof(unsigned long long), s));
      light_path();
      return true;
    }
    if (stage_total > cap_slots || v[10]) {  // the rare arena overflow (or a tcgen05 panel fallback): redo the pass
      stage = static_cast<uint2*>(arena(stage_total * sizeof(uint2)));
      TSG_CUDA(cudaMemsetAsync(counted_d, 0, sizeof(unsigned long long), s));
      TSG_CUDA(cudaMemsetAsync(tot_d, 0, 3 * sizeof(unsigned long long), s));
      TSG_CUDA(launch_panel_numeric(TA, *TB, rows, row_stage, stage_total, stage, rowcnt, counted_d, tot_d + 3, tot_d,
                           opt.mode, 0, TA.tile_rows, s, nullptr, nullptr, work, nl));
      check_launch(ctx);
      unsigned long long t[4];
      scan_rows(tot_d, t);
      P = t[0];
      S = t[1];
      raw = t[2];
    } else if (uint64_t(nnzC) >= (uint64_t(1) << 32)) {
      throw Fail{TSG_ERR_OTHER, "output beyond 2^32 elements needs row-panel batching"};
    }
    alloc_out();
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[2], s));
    launch_panel_copy(rows, row_stage, d_rp, stage, d_col, d_val, err_flag, 0, TA.tile_rows, s);
    check_launch(ctx);
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[3], s));
    record(ctx, timing, 6);
    return true;
  }

  void light_path() {
    if (emit_out) {  // chained stage: no staging, only the output tiles per tile row are bounded
      auto* row_tb = sc.alloc<uint32_t>(nr);
      TSG_CUDA(cudaMemsetAsync(row_tb + nr - 1, 0, sizeof(uint32_t), s));
      launch_row_tile_bound(TA, *TB, row_tb, s);
      check_launch(ctx);
      emit_tot = sc.alloc<unsigned long long>(4);  // P, S, raw (numeric pass), tile bound
      TSG_CUDA(cudaMemsetAsync(emit_tot, 0, 4 * sizeof(unsigned long long), s));
      const unsigned blocks = unsigned(std::min<uint64_t>((nr + 255) / 256, 1184));
      sum_u32_kernel<<<blocks, 256, 0, s>>>(row_tb, nr - 1, emit_tot + 3);
      check_launch(ctx);
      const uint64_t cap = readback(ctx, emit_tot + 3);
      if (cap >= (uint64_t(1) << 31)) throw Fail{TSG_ERR_OTHER, "emitted tiles beyond 2^31 need row-panel batching"};
      light_emit(row_tb, cap);
      return;
    }
    auto* row_np = sc.alloc<uint32_t>(nr);
    auto* row_ns = sc.alloc<uint32_t>(nr);
    auto* row_raw = sc.alloc<uint32_t>(nr);
    auto* row_bound = sc.alloc<uint32_t>(rows + 1);
    auto* row_stage = sc.alloc<uint32_t>(rows + 1);
    TSG_CUDA(cudaMemsetAsync(row_bound + rows, 0, 4, s));
    // exact u64 totals: P, S, raw pairs, staging slots (guards the u32 offsets)
    auto* tot_d = sc.alloc<unsigned long long>(4);
    TSG_CUDA(cudaMemsetAsync(tot_d, 0, 4 * sizeof(unsigned long long), s));
    const unsigned sblocks = unsigned(std::min<uint64_t>((std::max<uint64_t>(nr, rows + 1) + 255) / 256, 1184));
    // Staging bound.  Device output from CSR operands: the element-level bound
    // (one cheap pass over A's column indices; the numeric pass then counts
    // the statistics).  Host output (the bound sizes the pinned buffers) and
    // chained stages: the tight per-output-tile bound of panel_count_kernel.
    bool elem = !owner->host && !pre_a && !emit_out && tuning_variant("TSG_LIGHT_BOUND", 1) == 1;
    auto count_bound = [&]() {
      launch_panel_count(TA, *TB, rows, row_np, row_ns, row_raw, row_bound, nl, s);
      check_launch(ctx);
      sum_u32_kernel<<<sblocks, 256, 0, s>>>(row_np, nr - 1, tot_d);
      sum_u32_kernel<<<sblocks, 256, 0, s>>>(row_ns, nr - 1, tot_d + 1);
      sum_u32_kernel<<<sblocks, 256, 0, s>>>(row_raw, nr - 1, tot_d + 2);
      check_launch(ctx, 4);
    };
    if (elem) {
      launch_elem_bound(dA, dB.row_ptr, Bin->cols, row_bound, tot_d + 3, err_flag, s);
    } else {
      count_bound();
      sum_u32_kernel<<<sblocks, 256, 0, s>>>(row_bound, uint64_t(rows), tot_d + 3);
    }
    check_launch(ctx);
    exclusive_sum(ctx, sc, row_bound, row_stage, uint64_t(rows) + 1);
    auto take_totals = [&](const unsigned long long (&v)[4]) {
      P = v[0];
      S = v[1];
      raw = v[2];
      stage_total = v[3];
    };
    auto read_totals = [&]() {
      const unsigned long long* src[4] = {tot_d, tot_d + 1, tot_d + 2, tot_d + 3};
      unsigned long long v[4];
      readback_many(ctx, src, v);
      take_totals(v);
    };
    // an element bound beyond the u32 staging offsets: the tight bound instead
    auto fall_back = [&]() {
      elem = false;
      TSG_CUDA(cudaMemsetAsync(tot_d, 0, 4 * sizeof(unsigned long long), s));
      count_bound();
      sum_u32_kernel<<<sblocks, 256, 0, s>>>(row_bound, uint64_t(rows), tot_d + 3);
      check_launch(ctx);
      exclusive_sum(ctx, sc, row_bound, row_stage, uint64_t(rows) + 1);
      read_totals();
      check_stage_total();
    };
    // Device output with a staging arena already in place: launch the panel
    // pass without reading the staging total back first; the kernel checks it
    // against the arena on the device and the totals are read with nnz(C)
    // (a too-small arena -- rare after the first call -- reruns the pass).
    const bool speculative = !owner->host && ctx->stage_cap >= 16;
    if (!speculative) {
      read_totals();
      if (elem && stage_total >= (uint64_t(1) << 32)) fall_back();
      check_stage_total();
    }
    record(ctx, timing, 2);
    record(ctx, timing, 3);  // the merge is the sort: no separate phase
    record(ctx, timing, 4);  // the counting pass is fused into the numeric pass
    uint2* stage = static_cast<uint2*>(speculative ? ctx->stage_buf : arena(stage_total * sizeof(uint2)));
    uint64_t cap_slots = speculative ? ctx->stage_cap / sizeof(uint2) : stage_total;
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[0], s));
    if (owner->host && TA.tile_rows >= 8u * uint32_t(pipe_chunks())) {
      light_host_pipelined(row_stage, tot_d + 3, stage, cap_slots);
      return;
    }
    TSG_CUDA(launch_panel_numeric(TA, *TB, rows, row_stage, cap_slots, stage, rowcnt, counted_d, tot_d + 3,
                         elem ? tot_d : nullptr, opt.mode, 0, TA.tile_rows, s, nullptr, nullptr, work, nl));
    check_launch(ctx);
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[1], s));
    record(ctx, timing, 5);
    if (speculative) {
      unsigned long long t[4];
      // one synchronisation: counted, nnz(C), P, S, raw, staging slots (the
      // row counts are meaningless when the pass found the arena too small)
      scan_rows(tot_d, t, false);
      take_totals(t);
      if (stage_total > cap_slots || (stage_total >> 32)) {  // the rare arena overflow: redo the pass
        if (elem && stage_total >= (uint64_t(1) << 32)) fall_back();
        check_stage_total();
        stage = static_cast<uint2*>(arena(stage_total * sizeof(uint2)));
        cap_slots = stage_total;
        TSG_CUDA(cudaMemsetAsync(counted_d, 0, sizeof(unsigned long long), s));
        if (elem) TSG_CUDA(cudaMemsetAsync(tot_d, 0, 3 * sizeof(unsigned long long), s));
        TSG_CUDA(launch_panel_numeric(TA, *TB, rows, row_stage, cap_slots, stage, rowcnt, counted_d, tot_d + 3,
                             elem ? tot_d : nullptr, opt.mode, 0, TA.tile_rows, s, nullptr, nullptr, work, nl));
        check_launch(ctx);
        scan_rows(tot_d, t);
        take_totals(t);
      } else if (uint64_t(nnzC) >= (uint64_t(1) << 32)) {
        throw Fail{TSG_ERR_OTHER, "output beyond 2^32 elements needs row-panel batching"};
      }
    } else {
      if (elem) {
        unsigned long long t[4];
        scan_rows(tot_d, t);
        take_totals(t);
      } else {
        scan_rows();
      }
    }
    alloc_out();
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[2], s));
    launch_panel_copy(rows, row_stage, d_rp, stage, d_col, d_val, err_flag, 0, TA.tile_rows, s);
    check_launch(ctx);
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[3], s));
    record(ctx, timing, 6);
  }

  // Chained product, light rows: the result goes to the next stage as A tiles
  // (panel pass in emit mode, then compaction into a dense CSR-of-tiles).
  // Chained product, light rows, `cap` = the bound on the emitted tiles
  void light_emit(const uint32_t* row_tb, uint64_t cap) {
    path = TSG_PATH_PANEL_EMIT;
    auto kept = [&](auto* p) {
      keep->push_back(p);
      return p;
    };
    record(ctx, timing, 2);
    record(ctx, timing, 3);
    record(ctx, timing, 4);
    TileEmit em;
    auto* tile_base = sc.alloc<uint32_t>(nr);
    exclusive_sum(ctx, sc, row_tb, tile_base, nr);
    em.tile_base = tile_base;
    const uint64_t S = std::max<uint64_t>(cap, 1);
    em.tco = sc.alloc<uint2>(S);
    em.rm2 = sc.alloc<uint32_t>(S * 8);
    em.meta = sc.alloc<uint2>(S);
    em.rec = sc.alloc<uint4>(S);
    em.chunk = kept(sc.alloc<uint4>(32 * S + 1, true));
    TSG_CUDA(cudaMemsetAsync(em.chunk, 0, sizeof(uint4), s));
    em.rtiles = sc.alloc<uint32_t>(nr);
    TSG_CUDA(cudaMemsetAsync(em.rtiles + nr - 1, 0, sizeof(uint32_t), s));
    em.err_flag = err_flag;
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[0], s));
    TSG_CUDA(launch_panel_numeric(TA, *TB, rows, nullptr, 0, nullptr, nullptr, counted_d, nullptr, emit_tot, opt.mode, 0,
                         TA.tile_rows, s, &em, nullptr, work, nl));
    check_launch(ctx);
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[1], s));
    record(ctx, timing, 5);
    TileMat& T = *emit_out;
    T = TileMat{};
    T.rows = rows;
    T.cols = TB->cols;
    T.tile_rows = TA.tile_rows;
    T.tile_cols = uint32_t((T.cols + 15) / 16);
    T.trp = kept(sc.alloc<uint32_t>(nr, true));
    exclusive_sum(ctx, sc, em.rtiles, T.trp, nr);
    // the dense arrays are sized by the bound (no readback here); counted
    // and the statistics are read by finish()
    const uint64_t nt = S;
    T.cap = cap;
    T.tco = kept(sc.alloc<uint2>(nt, true));
    T.rm2 = kept(sc.alloc<uint32_t>(nt * 8, true));
    T.meta[kRoleA] = kept(sc.alloc<uint2>(nt, true));
    T.rec[kRoleA] = kept(sc.alloc<uint4>(nt, true));
    T.chunk[kRoleA] = em.chunk;
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[2], s));
    launch_emit_compact(TA.tile_rows, em, T.trp, T, s);
    check_launch(ctx);
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[3], s));
    nnzC = 0;
    stage_total = 0;  // no staging: the tiles are written in place
    record(ctx, timing, 6);
  }

  // Host output: the result crosses PCIe (the slowest leg), so the panel pass
  // runs in kPipeChunks tile-row chunks and chunk c's CSR slice goes to the
  // host on a second stream while chunk c+1 computes.  Row pointers are a
  // chained scan (each chunk starts from the previous chunk's end, read on
  // the device); host buffers are sized by the staging bound, an upper bound
  // on nnz(C).
  void light_host_pipelined(const uint32_t* row_stage, const unsigned long long* need, uint2* stage,
                            uint64_t cap_slots) {
    TSG_CUDA(cudaMemsetAsync(d_rp, 0, sizeof(int64_t), s));
    owner->p[0] = pinned_alloc(ctx, (rows + 1) * sizeof(int64_t), &owner->sz[0]);
    owner->p[1] = pinned_alloc(ctx, std::max<uint64_t>(stage_total, 1) * sizeof(int32_t), &owner->sz[1]);
    owner->p[2] = pinned_alloc(ctx, std::max<uint64_t>(stage_total, 1) * sizeof(float), &owner->sz[2]);
    d_col = sc.alloc<int32_t>(stage_total);
    d_val = sc.alloc<float>(stage_total);
    auto* ends = reinterpret_cast<int64_t*>(ctx->pinned_pipe);  // row_ptr at each chunk end
    auto* flag_h = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(ctx->pinned_pipe) + 8 * (kPipeChunks + 1));
    size_t tmp_bytes = 0;
    TSG_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, tmp_bytes, rowcnt, d_rp, cuda::std::plus<int64_t>(),
                                            cub::FutureValue<int64_t>(d_rp), rows + 1, s));
    void* tmp = sc.alloc<char>(tmp_bytes);
    const int nch = pipe_chunks();
    int64_t cr0[kPipeChunks], cr1[kPipeChunks];
    // (1) every chunk's compute, with its end offset to the host
    for (int c = 0; c < nch; ++c) {
      const uint32_t I0 = uint32_t(uint64_t(TA.tile_rows) * c / nch);
      const uint32_t I1 = uint32_t(uint64_t(TA.tile_rows) * (c + 1) / nch);
      const int64_t r0 = int64_t(I0) * 16, r1 = std::min<int64_t>(int64_t(I1) * 16, rows);
      cr0[c] = r0;
      cr1[c] = r1;
      TSG_CUDA(launch_panel_numeric(TA, *TB, rows, row_stage, cap_slots, stage, rowcnt, counted_d, need, nullptr, opt.mode,
                           I0, I1, s, nullptr, nullptr, work, nl));
      check_launch(ctx);
      // row_ptr[r0 .. r1] = row_ptr[r0] + exclusive prefix (row_ptr[r0] from the previous chunk)
      TSG_CUDA(cub::DeviceScan::ExclusiveScan(tmp, tmp_bytes, rowcnt + r0, d_rp + r0, cuda::std::plus<int64_t>(),
                                              cub::FutureValue<int64_t>(d_rp + r0), r1 - r0 + 1, s));
      launch_panel_copy(rows, row_stage, d_rp, stage, d_col, d_val, err_flag, I0, I1, s);
      check_launch(ctx);
      publish_chunk_kernel<<<1, 1, 0, s>>>(d_rp + r1, err_flag, ends + c, flag_h + c);
      check_launch(ctx);
      TSG_CUDA(cudaEventRecord(ctx->pipe_ev[c], s));
    }
    // (2) each chunk's slices to the host on stream 2 as soon as it is computed
    int32_t* h_col = static_cast<int32_t*>(owner->p[1]);
    int64_t* h_rp = static_cast<int64_t*>(owner->p[0]);
    uint64_t sent = 0, d2h_bytes = 0;
    for (int c = 0; c < nch; ++c) {
      TSG_CUDA(cudaEventSynchronize(ctx->pipe_ev[c]));  // its end is readable now
      const uint64_t lo = sent, hi = uint64_t(ends[c]);
      TSG_CUDA(cudaStreamWaitEvent(ctx->d2h, ctx->pipe_ev[c], 0));
      TSG_CUDA(cudaMemcpyAsync(h_rp + cr0[c], d_rp + cr0[c], (cr1[c] - cr0[c]) * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, ctx->d2h));
      d2h_bytes += (cr1[c] - cr0[c]) * sizeof(int64_t);
      if (hi > lo) {
        TSG_CUDA(cudaMemcpyAsync(h_col + lo, d_col + lo, (hi - lo) * 4, cudaMemcpyDeviceToHost, ctx->d2h));
        TSG_CUDA(cudaMemcpyAsync(static_cast<float*>(owner->p[2]) + lo, d_val + lo, (hi - lo) * 4,
                                 cudaMemcpyDeviceToHost, ctx->d2h));
        d2h_bytes += (hi - lo) * 8;
      }
      sent = hi;
    }
    nnzC = int64_t(sent);
    if (uint64_t(nnzC) >= (uint64_t(1) << 32))
      throw Fail{TSG_ERR_OTHER, "output beyond 2^32 elements needs row-panel batching"};
    TSG_CUDA(cudaMemcpyAsync(h_rp + rows, d_rp + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->d2h));
    TSG_CUDA(cudaEventRecord(ctx->pipe_ev[kPipeChunks], ctx->d2h));
    TSG_CUDA(cudaStreamWaitEvent(s, ctx->pipe_ev[kPipeChunks], 0));  // the final sync covers stream 2
    counted = readback(ctx, counted_d);
    if (st) st->d2h_bytes += sizeof(int64_t) + d2h_bytes;
    host_done = true;
    if (timing) {
      TSG_CUDA(cudaEventRecord(ctx->kev[1], s));
      TSG_CUDA(cudaEventRecord(ctx->kev[2], s));
      TSG_CUDA(cudaEventRecord(ctx->kev[3], s));
    }
    record(ctx, timing, 5);
    record(ctx, timing, 6);
  }

  // ---- general rows: per-chunk element SEaC in shared memory (tsg_esc.cu) ----------
  void general_path() {
    path = TSG_PATH_GENERAL;
    const TileMat& B = *TB;
    EscArgs g;
    g.rowsA = rows;
    g.tile_rows = TA.tile_rows;
    g.target = uint32_t(std::max(256, tuning_variant("TSG_ESC_TARGET", int(kEscTarget))));
    int64_t nnzA = 0;
    if (pre_a) {  // the previous stage's A tiles -> CSR with binary16 values
      auto* rp = sc.alloc<int64_t>(rows + 1);
      TSG_CUDA(cudaMemsetAsync(rowcnt + rows, 0, sizeof(int64_t), s));
      launch_tiles_rowcount(TA, rowcnt, s);
      exclusive_sum(ctx, sc, rowcnt, rp, uint64_t(rows) + 1);
      nnzA = int64_t(readback(ctx, rp + rows));
      auto* col = sc.alloc<int32_t>(nnzA);
      auto* h = sc.alloc<uint16_t>(nnzA);
      launch_tiles_to_csr(TA, rp, col, h, s);
      check_launch(ctx, 2);
      g.rpA = rp;
      g.colA = col;
      g.hA = h;
    } else {
      nnzA = dA.nnz;
      g.rpA = dA.row_ptr;
      g.colA = dA.col;
      g.hA = TA.h16;
    }
    g.colsB = Bin->cols;
    g.rpB = dB.row_ptr;
    g.colB = dB.col;
    g.hB = B.h16;
    // B row records {first entry, end, first col, last col}: one gather per A entry
    auto* brec = sc.alloc<uint4>(uint64_t(std::max<int64_t>(Bin->rows, 1)));
    launch_esc_brec(g, Bin->rows, brec, s);
    g.brec = brec;
    // (1) product histogram over output columns -> its prefix G (heavy-row cuts)
    const uint64_t inner = uint64_t(std::max<int64_t>(Bin->rows, 1));
    auto* colcnt = sc.alloc<uint32_t>(inner);
    TSG_CUDA(cudaMemsetAsync(colcnt, 0, inner * sizeof(uint32_t), s));
    const uint64_t nc1 = uint64_t(Bin->cols) + 1;
    auto* hist = sc.alloc<unsigned long long>(nc1);
    TSG_CUDA(cudaMemsetAsync(hist, 0, nc1 * sizeof(unsigned long long), s));
    launch_esc_hist(g, nnzA, Bin->rows, colcnt, hist, s);
    check_launch(ctx, 4);
    auto* G = sc.alloc<unsigned long long>(nc1);
    exclusive_sum(ctx, sc, hist, G, nc1);
    // (2) products per tile row -> units (groups of light rows, column ranges
    // of heavy rows) and output records; tile-pair statistics
    // tot: [0] products, [1] segments, [2] raw pairs, [3] filtered pairs, [4] pool pieces (u32)
    auto* tot = sc.alloc<unsigned long long>(8);
    TSG_CUDA(cudaMemsetAsync(tot, 0, 8 * sizeof(unsigned long long), s));
    auto* prod = sc.alloc<unsigned long long>(nr);
    TSG_CUDA(cudaMemsetAsync(prod + nr - 1, 0, sizeof(unsigned long long), s));
    launch_esc_plan_prod(g, prod, tot, s);
    check_launch(ctx);
    auto* ppre = sc.alloc<unsigned long long>(nr);
    exclusive_sum(ctx, sc, prod, ppre, nr);
    auto* nrec = sc.alloc<uint32_t>(nr);
    auto* nwk = sc.alloc<uint32_t>(nr);
    TSG_CUDA(cudaMemsetAsync(nrec + nr - 1, 0, sizeof(uint32_t), s));
    TSG_CUDA(cudaMemsetAsync(nwk + nr - 1, 0, sizeof(uint32_t), s));
    launch_esc_plan_group(g, ppre, nrec, nwk, s);
    check_launch(ctx);
    auto* rbase = sc.alloc<uint32_t>(nr);
    auto* wbase = sc.alloc<uint32_t>(nr);
    exclusive_sum(ctx, sc, nrec, rbase, nr);
    exclusive_sum(ctx, sc, nwk, wbase, nr);
    const uint32_t* njt = bsum ? bsum->njt : nullptr;
    const uint32_t* rinfo = bsum ? bsum->rinfo : nullptr;
    if (!bsum) {
      auto* nj = sc.alloc<uint32_t>(uint64_t(B.rows) + 1);
      auto* ri = sc.alloc<uint32_t>(uint64_t(B.tile_rows) + 1);
      launch_esc_bsummary(B, nj, ri, s);
      check_launch(ctx, 2);
      njt = nj;
      rinfo = ri;
    }
    launch_esc_pairstats(TA, B, tA, njt, rinfo, tot + 2, s);
    check_launch(ctx);
    record(ctx, timing, 2);
    uint64_t nrecs = 0, nunits = 0, products = 0;
    // host output of a large product: the tile rows run in chunks whose CSR
    // slices cross PCIe while later chunks compute (the chunks' record and
    // unit boundaries come with this readback)
    const int nch = owner->host && !pre_a && TA.tile_rows >= 8u * uint32_t(pipe_chunks()) ? pipe_chunks() : 0;
    uint32_t cut_rec[kPipeChunks + 1] = {}, cut_unit[kPipeChunks + 1] = {};
    {
      ScalarGather sg;
      sg.p[0] = rbase + nr - 1;
      sg.p[1] = wbase + nr - 1;
      sg.p[2] = tot;
      sg.wide = 0x4u;
      sg.n = 3;
      for (int c = 0; c <= nch && nch; ++c) {
        const uint32_t I = uint32_t(uint64_t(TA.tile_rows) * c / nch);
        sg.p[sg.n++] = rbase + I;
        sg.p[sg.n++] = wbase + I;
      }
      unsigned long long v[kGatherMax];
      readback_gather(ctx, sc, sg, v);
      nrecs = v[0];
      nunits = v[1];
      products = v[2];
      for (int c = 0; c <= nch && nch; ++c) {
        cut_rec[c] = uint32_t(v[3 + 2 * c]);
        cut_unit[c] = uint32_t(v[4 + 2 * c]);
      }
    }
    uint4* units;
    {
      MemRole role_tl(sc, kMemTaskList);
      units = sc.alloc<uint4>(nunits);
    }
    launch_esc_plan_fill(g, ppre, nwk, wbase, G, units, s);
    check_launch(ctx);
    record(ctx, timing, 3);
    record(ctx, timing, 4);
    // (3) multiply: staging for every product (realised entries <= products)
    auto* ctr = sc.alloc<unsigned long long>(2);  // [0] work counter (u32), [1] staging top
    g.units = units;
    g.nunits = wbase + nr - 1;
    g.rec_base = rbase;
    g.nrec = rbase + nr - 1;
    g.stage = static_cast<uint2*>(arena(std::max<uint64_t>(products, 1) * sizeof(uint2)));
    g.err_flag = err_flag;
    g.counted = counted_d;
    g.segs = tot + 1;
    g.piece_top = reinterpret_cast<uint32_t*>(tot + 4);
    g.work = reinterpret_cast<unsigned*>(ctr);
    g.stage_top = ctr + 1;
    uint64_t pool = std::max<uint64_t>(4096, nunits / 8);
    if (nch && general_host_pipelined(g, nch, cut_rec, cut_unit, nrecs, pool, products, rbase)) return;
    unsigned long long t[4];
    for (int attempt = 0;; ++attempt) {
      g.pool_cap = uint32_t(std::min<uint64_t>(pool, 0xfffffff0ull - nrecs));
      {
        MemRole role_tl(sc, kMemTaskList);
        g.pieces = sc.alloc<EscPiece>(nrecs + g.pool_cap);
      }
      TSG_CUDA(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), s));
      if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[0], s));
      launch_esc(g, ctx->device, s);
      check_launch(ctx);
      if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[1], s));
      record(ctx, timing, 5);
      launch_esc_rowcount(g, rbase, rowcnt, s);
      check_launch(ctx);
      scan_rows(tot + 1, t);
      if (t[3] <= g.pool_cap || attempt > 8) break;
      // the overflow-piece pool was too small (pathological column skew): rerun
      pool = t[3] * 2;
      TSG_CUDA(cudaMemsetAsync(counted_d, 0, sizeof(unsigned long long), s));
      TSG_CUDA(cudaMemsetAsync(tot + 1, 0, sizeof(unsigned long long), s));
      TSG_CUDA(cudaMemsetAsync(tot + 4, 0, sizeof(unsigned long long), s));
      TSG_CUDA(cudaMemsetAsync(err_flag, 0, sizeof(unsigned), s));
    }
    S = t[0];
    raw = t[1];
    P = t[2];
    stage_total = products;
    alloc_out();
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[2], s));
    launch_esc_copy(g, d_rp, d_col, d_val, s);
    check_launch(ctx);
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[3], s));
    record(ctx, timing, 6);
  }

  // General rows, host output: the tile rows run in nch chunks (their units
  // [cut_unit[c], cut_unit[c+1]) and output records [cut_rec[c],
  // cut_rec[c+1])); chunk c's row pointers chain from chunk c-1's end on the
  // device, its pieces are copied into CSR buffers sized by the product bound,
  // and its slices go to the host on the copy stream while chunk c+1
  // computes.  Returns false (nothing shipped) when the overflow-piece pool
  // ran out: the caller then takes the unpipelined path with its retry.
  bool general_host_pipelined(EscArgs& g, int nch, const uint32_t* cut_rec, const uint32_t* cut_unit, uint64_t nrecs,
                              uint64_t pool, uint64_t products, const uint32_t* rbase) {
    g.pool_cap = uint32_t(std::min<uint64_t>(pool, 0xfffffff0ull - nrecs));
    {
      MemRole role_tl(sc, kMemTaskList);
      g.pieces = sc.alloc<EscPiece>(nrecs + g.pool_cap);
    }
    auto* ctr = sc.alloc<unsigned long long>(2);
    g.work = reinterpret_cast<unsigned*>(ctr);
    g.stage_top = ctr + 1;
    TSG_CUDA(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), s));
    TSG_CUDA(cudaMemsetAsync(d_rp, 0, sizeof(int64_t), s));
    const uint64_t bound = std::max<uint64_t>(products, 1);
    {
      MemRole role_out(sc, kMemOutput);
      d_col = sc.alloc<int32_t>(bound);
      d_val = sc.alloc<float>(bound);
    }
    owner->p[0] = pinned_alloc(ctx, (rows + 1) * sizeof(int64_t), &owner->sz[0]);
    owner->p[1] = pinned_alloc(ctx, bound * sizeof(int32_t), &owner->sz[1]);
    owner->p[2] = pinned_alloc(ctx, bound * sizeof(float), &owner->sz[2]);
    auto* ends = reinterpret_cast<int64_t*>(ctx->pinned_pipe);
    auto* flag_h = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(ctx->pinned_pipe) + 8 * (kPipeChunks + 1));
    size_t tmp_bytes = 0;
    TSG_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, tmp_bytes, rowcnt, d_rp, cuda::std::plus<int64_t>(),
                                            cub::FutureValue<int64_t>(d_rp), rows + 1, s));
    void* tmp = sc.alloc<char>(tmp_bytes);
    int64_t cr0[kPipeChunks], cr1[kPipeChunks];
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[0], s));
    for (int c = 0; c < nch; ++c) {
      const uint32_t I0 = uint32_t(uint64_t(TA.tile_rows) * c / nch);
      const uint32_t I1 = uint32_t(uint64_t(TA.tile_rows) * (c + 1) / nch);
      cr0[c] = int64_t(I0) * 16;
      cr1[c] = std::min<int64_t>(int64_t(I1) * 16, rows);
      g.unit0 = cut_unit[c];
      g.unit_end = cut_unit[c + 1];
      TSG_CUDA(cudaMemsetAsync(g.work, 0, sizeof(unsigned), s));
      launch_esc(g, ctx->device, s);
      launch_esc_rowcount(g, rbase, rowcnt, s, I0, I1);
      check_launch(ctx, 2);
      TSG_CUDA(cub::DeviceScan::ExclusiveScan(tmp, tmp_bytes, rowcnt + cr0[c], d_rp + cr0[c],
                                              cuda::std::plus<int64_t>(), cub::FutureValue<int64_t>(d_rp + cr0[c]),
                                              cr1[c] - cr0[c] + 1, s));
      launch_esc_copy_records(g, cut_rec[c], cut_rec[c + 1], d_rp, d_col, d_val, s);
      publish_chunk_kernel<<<1, 1, 0, s>>>(d_rp + cr1[c], err_flag, ends + c, flag_h + c);
      check_launch(ctx, 2);
      TSG_CUDA(cudaEventRecord(ctx->pipe_ev[c], s));
    }
    if (timing) TSG_CUDA(cudaEventRecord(ctx->kev[1], s));
    // each chunk's slices to the host as soon as it is computed
    int32_t* h_col = static_cast<int32_t*>(owner->p[1]);
    float* h_val = static_cast<float*>(owner->p[2]);
    int64_t* h_rp = static_cast<int64_t*>(owner->p[0]);
    uint64_t sent = 0, d2h_bytes = 0;
    bool pool_short = false;
    for (int c = 0; c < nch; ++c) {
      TSG_CUDA(cudaEventSynchronize(ctx->pipe_ev[c]));
      pool_short |= (flag_h[c] & kErrPool) != 0;
      if (pool_short) break;
      const uint64_t lo = sent, hi = uint64_t(ends[c]);
      TSG_CUDA(cudaStreamWaitEvent(ctx->d2h, ctx->pipe_ev[c], 0));
      TSG_CUDA(cudaMemcpyAsync(h_rp + cr0[c], d_rp + cr0[c], (cr1[c] - cr0[c]) * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, ctx->d2h));
      d2h_bytes += (cr1[c] - cr0[c]) * sizeof(int64_t);
      if (hi > lo) {
        TSG_CUDA(cudaMemcpyAsync(h_col + lo, d_col + lo, (hi - lo) * 4, cudaMemcpyDeviceToHost, ctx->d2h));
        TSG_CUDA(cudaMemcpyAsync(h_val + lo, d_val + lo, (hi - lo) * 4, cudaMemcpyDeviceToHost, ctx->d2h));
        d2h_bytes += (hi - lo) * 8;
      }
      sent = hi;
    }
    TSG_CUDA(cudaMemcpyAsync(h_rp + rows, d_rp + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->d2h));
    TSG_CUDA(cudaEventRecord(ctx->pipe_ev[kPipeChunks], ctx->d2h));
    TSG_CUDA(cudaStreamWaitEvent(s, ctx->pipe_ev[kPipeChunks], 0));
    if (pool_short) {  // pathological column skew: give the buffers back, rerun unpipelined
      TSG_CUDA(cudaStreamSynchronize(ctx->d2h));
      for (int i = 0; i < 3; ++i) {
        ctx->pinned_free.emplace_back(owner->p[i], owner->sz[i]);
        owner->p[i] = nullptr;
      }
      TSG_CUDA(cudaMemsetAsync(counted_d, 0, sizeof(unsigned long long), s));
      TSG_CUDA(cudaMemsetAsync(g.segs, 0, sizeof(unsigned long long), s));
      TSG_CUDA(cudaMemsetAsync(g.piece_top, 0, sizeof(uint32_t), s));
      TSG_CUDA(cudaMemsetAsync(err_flag, 0, sizeof(unsigned), s));
      g.unit0 = 0;
      g.unit_end = 0xffffffffu;
      return false;
    }
    record(ctx, timing, 5);
    // statistics: segments, raw and filtered pairs (tot[1..3]), counted; nnz(C)
    const unsigned long long* src[4] = {g.segs, g.segs + 1, g.segs + 2, counted_d};
    unsigned long long v[4];
    readback_many(ctx, src, v);
    S = v[0];
    raw = v[1];
    P = v[2];
    counted = v[3];
    nnzC = int64_t(sent);
    stage_total = products;
    if (uint64_t(nnzC) >= (uint64_t(1) << 32))
      throw Fail{TSG_ERR_OTHER, "output beyond 2^32 elements needs row-panel batching"};
    if (st) st->d2h_bytes += sizeof(int64_t) + d2h_bytes;
    host_done = true;
    if (timing) {
      TSG_CUDA(cudaEventRecord(ctx->kev[2], s));
      TSG_CUDA(cudaEventRecord(ctx->kev[3], s));
    }
    record(ctx, timing, 6);
    return true;
  }

  // ---- output hand-off, error flags, phase times and counters ----------------------
  void finish(tsg_tiles_out* tiles) {
    // non-finite accumulators are flagged by the CSR pass (read at the final sync)
    unsigned* flags_host = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(ctx->pinned) + 56);
    TSG_CUDA(cudaMemcpyAsync(flags_host, err_flag, 4, cudaMemcpyDeviceToHost, s));
    unsigned long long* counted_host = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(ctx->pinned) + 40);
    unsigned long long* tot_host = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(ctx->pinned) + 64);
    if (emit_out) {
      TSG_CUDA(cudaMemcpyAsync(counted_host, counted_d, 8, cudaMemcpyDeviceToHost, s));
      if (emit_tot) TSG_CUDA(cudaMemcpyAsync(tot_host, emit_tot, 24, cudaMemcpyDeviceToHost, s));
    }
    C->rows = rows;
    C->cols = Bin->cols;
    C->nnz = nnzC;
    if (owner->host && !host_done && !emit_out) {
      owner->p[0] = pinned_alloc(ctx, (rows + 1) * sizeof(int64_t), &owner->sz[0]);
      owner->p[1] = pinned_alloc(ctx, nnzC * sizeof(int32_t), &owner->sz[1]);
      owner->p[2] = pinned_alloc(ctx, nnzC * sizeof(float), &owner->sz[2]);
      TSG_CUDA(cudaMemcpyAsync(owner->p[0], d_rp, (rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      if (nnzC) {
        TSG_CUDA(cudaMemcpyAsync(owner->p[1], d_col, nnzC * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        TSG_CUDA(cudaMemcpyAsync(owner->p[2], d_val, nnzC * sizeof(float), cudaMemcpyDeviceToHost, s));
      }
      if (st) st->d2h_bytes += (rows + 1) * sizeof(int64_t) + nnzC * (sizeof(int32_t) + sizeof(float));
    }
    C->row_ptr = static_cast<int64_t*>(owner->p[0]);
    C->col = static_cast<int32_t*>(owner->p[1]);
    C->val = static_cast<float*>(owner->p[2]);

    TSG_CUDA(cudaStreamSynchronize(s));
    if (emit_out) {
      counted = *counted_host;
      if (emit_tot) {
        P = tot_host[0];
        S = tot_host[1];
        raw = tot_host[2];
      }
    }
    raise_flags(*flags_host);
    if (tiles) {  // test path: 16x16 tiled view of the realised C
      std::vector<int64_t> h_rp(rows + 1);
      std::vector<int32_t> h_col(nnzC);
      std::vector<float> h_val(nnzC);
      TSG_CUDA(cudaMemcpy(h_rp.data(), d_rp, (rows + 1) * 8, cudaMemcpyDeviceToHost));
      if (nnzC) {
        TSG_CUDA(cudaMemcpy(h_col.data(), d_col, nnzC * 4, cudaMemcpyDeviceToHost));
        TSG_CUDA(cudaMemcpy(h_val.data(), d_val, nnzC * 4, cudaMemcpyDeviceToHost));
      }
      tiles_from_csr(rows, h_rp, h_col, h_val, tiles);
    }
    if (timing) {
      float ms[7] = {0};
      for (int i = 1; i <= 6; ++i) TSG_CUDA(cudaEventElapsedTime(&ms[i], ctx->ev[i - 1], ctx->ev[i]));
      float tot = 0;
      TSG_CUDA(cudaEventElapsedTime(&tot, ctx->ev[0], ctx->ev[6]));
      for (int i = 1; i <= 6; ++i) ctx->last_phase_ms[i] = ms[i];
      ctx->last_phase_ms[7] = tot;
      float kn = 0, kc = 0;
      TSG_CUDA(cudaEventElapsedTime(&kn, ctx->kev[0], ctx->kev[1]));
      TSG_CUDA(cudaEventElapsedTime(&kc, ctx->kev[2], ctx->kev[3]));
      ctx->last_numeric_kernel_ms = kn;
      ctx->last_assemble_kernel_ms = kc;
      if (st) {
        st->convert += ms[1] * 1e-3;
        st->task_list += ms[2] * 1e-3;
        st->sort += ms[3] * 1e-3;
        st->counting += ms[4] * 1e-3;
        st->multiply += ms[5] * 1e-3;
        st->compaction += ms[6] * 1e-3;
        st->total += tot * 1e-3;
      }
    }
    if (emit_out && !light) throw Fail{TSG_ERR_OTHER, "internal: tile emission needs the light-row path"};
    if (st) {
      st->tiles_a += tA;
      st->tiles_b += tB;
      st->raw_pairs += raw;
      st->filtered_pairs += P;
      st->segments += S;
      st->counted_elements += counted;
      st->nnz_c = uint64_t(nnzC);
      st->staged_slots += stage_total;
      st->kernel_launches += ctx->launches - launches0;
      st->mem_input_tiles += sc.bytes[kMemTiles];
      st->mem_input_elements += sc.bytes[kMemElements];
      st->mem_task_list += sc.bytes[kMemTaskList];
      st->mem_counting += sc.bytes[kMemCounting];
      st->mem_pre_compaction += stage_total * sizeof(uint2) + sc.bytes[kMemStaging];
      st->mem_output += sc.bytes[kMemOutput];
      uint64_t high = 0;
      if (cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrUsedMemHigh, &high) == cudaSuccess)
        st->mem_peak = std::max<uint64_t>(st->mem_peak, uint64_t(high));
      st->path = path;
      st->devices = 1;
    }
  }
};

void spgemm_impl(tsg_ctx* ctx, const tsg_csr* Ain, const tsg_csr* Bin, tsg_csr_out* C,
                 const tsg_options& opt, tsg_run_stats* st, tsg_tiles_out* tiles) {
  Call call(ctx, Ain, Bin, C, opt, st);
  // one synchronisation for conversion + light pass when it can be speculated
  const bool spec = C && C->mem != TSG_MEM_HOST && ctx->stage_cap >= 16 &&
                    tuning_variant("TSG_LIGHT_BOUND", 1) == 1 && tuning_variant("TSG_SPECULATE", 1) == 1;
  call.convert_operands(spec);
  if (spec) {
    if (!call.light_speculative()) call.general_path();
  } else if (call.light) {
    call.light_path();
  } else {
    call.general_path();
  }
  call.finish(tiles);
}

// tsg_spgemm_bsum: A converted as usual, B through its summary; light rows
// (the MMA pass reads B's operand tiles) convert B after all.
void spgemm_bsum_impl(tsg_ctx* ctx, const tsg_csr* Ain, const tsg_csr* Bin, const tsg_bsum* bsum, tsg_csr_out* C,
                      const tsg_options& opt, tsg_run_stats* st) {
  if (!bsum) throw Fail{TSG_ERR_OTHER, "B summary is NULL"};
  Call call(ctx, Ain, Bin, C, opt, st);
  call.bsum = bsum;
  call.convert_operands();
  if (call.light) {
    call.convert_b();
    call.light_path();
  } else {
    call.general_path();
  }
  call.finish(nullptr);
}

// A panel of B -> its summary (tsg_bsum_create): B-role conversion with the
// general flag raised (no operand chunks), then the per-row and per-tile-row
// summaries; outputs outlive the call (pool allocations owned by the summary).
void bsum_create_impl(tsg_ctx* ctx, const tsg_csr* Bp, tsg_bsum* out) {
  check_csr(Bp, "B panel");
  *out = tsg_bsum{};
  TSG_CUDA(cudaEventRecord(ctx->kev[0], ctx->stream));
  Scratch sc(ctx);
  const CsrView dB = stage(ctx, sc, Bp, nullptr);
  auto* z = sc.alloc<unsigned>(4);  // [0] error flags, [1] walk counter, [2] general flag
  TSG_CUDA(cudaMemsetAsync(z, 0, 2 * sizeof(unsigned), ctx->stream));
  const unsigned one = 1;
  TSG_CUDA(cudaMemcpyAsync(z + 2, &one, sizeof(unsigned), cudaMemcpyHostToDevice, ctx->stream));
  TileMat T;
  const uint32_t* nt_d = convert(ctx, sc, dB, T, 2, z, 0, nullptr, nullptr, z + 1, nullptr, z + 2);
  const unsigned* src[2] = {z, nt_d};
  unsigned v[2];
  readback_many(ctx, src, v);
  raise_flags(v[0]);
  const int64_t rows = Bp->rows, tr = (rows + 15) / 16, nnz = Bp->nnz, tiles = int64_t(v[1]);
  auto* own = new std::vector<void*>();
  auto keep = [&](size_t bytes) {
    void* p = nullptr;
    TSG_CUDA(cudaMallocFromPoolAsync(&p, std::max<size_t>(bytes, 4), ctx->pool, ctx->stream));
    own->push_back(p);
    return p;
  };
  try {
    out->rows = rows;
    out->tile_rows = tr;
    out->tiles = tiles;
    out->nnz = nnz;
    out->njt = static_cast<uint32_t*>(keep((rows + 1) * 4));
    out->tile_count = static_cast<uint32_t*>(keep((tr + 1) * 4));
    out->rinfo = static_cast<uint32_t*>(keep((tr + 1) * 4));
    out->ro = static_cast<uint16_t*>(keep(tiles * 2));
    out->etile = static_cast<uint32_t*>(keep(nnz * 4));
    out->h16 = static_cast<uint16_t*>(keep(nnz * 2));
    out->_owner = own;
    launch_esc_bsummary(T, out->njt, out->rinfo, ctx->stream);
    launch_bsum_tiles(T, uint64_t(tiles), out->tile_count, out->ro, ctx->stream);
    check_launch(ctx, 3);
    if (nnz) {
      TSG_CUDA(cudaMemcpyAsync(out->etile, T.etile, nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      TSG_CUDA(cudaMemcpyAsync(out->h16, T.h16, nnz * 2, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    TSG_CUDA(cudaEventRecord(ctx->kev[1], ctx->stream));
    TSG_CUDA(cudaStreamSynchronize(ctx->stream));
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->kev[0], ctx->kev[1]) == cudaSuccess) ctx->last_bsum_ms = ms;
  } catch (...) {
    for (void* p : *own) cudaFreeAsync(p, ctx->stream);
    delete own;
    *out = tsg_bsum{};
    throw;
  }
}

// One stage of a chain (tsg_spgemm_chain).  `pre_a`: A as the previous
// stage's tiles (else Ain as CSR).  `emit`: when this stage takes the
// light-row path, its result becomes the next stage's A tiles (returns
// true); otherwise C receives CSR as usual (returns false).
bool chain_stage(tsg_ctx* ctx, const tsg_csr* Ain, const TileMat* pre_a,
                 const tsg_csr* Bin, tsg_csr_out* C, TileMat* emit, std::vector<void*>* keep,
                 const tsg_options& opt, tsg_run_stats* st) {
  Call call(ctx, Ain, Bin, C, opt, st);
  call.pre_a = pre_a;
  call.keep = keep;
  call.convert_operands();
  if (call.light) {
    call.emit_out = emit;
    call.light_path();
  } else {
    call.general_path();
  }
  call.finish(nullptr);
  return emit && call.light;
}

void free_out(tsg_ctx* ctx, tsg_csr_out* C) {
  if (!C || !C->_owner) return;
  auto* o = static_cast<OutOwner*>(C->_owner);
  for (int i = 0; i < 3; ++i) {
    void* p = o->p[i];
    if (!p) continue;
    if (o->host)
      ctx->pinned_free.emplace_back(p, o->sz[i]);
    else
      cudaFreeAsync(p, ctx->stream);
  }
  delete o;
  C->_owner = nullptr;
  C->row_ptr = nullptr;
  C->col = nullptr;
  C->val = nullptr;
}


// ---------------------------------------------------------------- multi-device
// tsg_create_multi: C = X0 . X1 ... with X0 split into contiguous tile-row
// panels of ~equal work; panel i runs the single-device
// path on sub[i] (own stream, own host thread per distinct GPU), the other
// operands replicated per device; the panels' CSR slices are concatenated
// in row order (byte-identical to one device: a C tile row depends only on
// X0's tile row and the other operands).

// A tile row's cost for the panel split: its intermediate products w plus,
// for the general path, the range searches of its work units (each unit of
// ~kEscTarget products searches the B rows of all the tile row's entries)
__host__ __device__ inline unsigned long long panel_cost(unsigned long long w, int64_t entries) {
  constexpr double kSearchWeight = 0.9;  // one (entry, unit) search, in products (distributed.py SEARCH_WEIGHT)
  const double units = w ? double((w + kEscTarget - 1) / kEscTarget) : 0.0;
  return w + (unsigned long long)(kSearchWeight * units * double(entries));
}

// work[I] = panel_cost(sum over X0's entries (r, k) in tile row I of nnz(X1 row k), entries)
__global__ void tile_row_work_kernel(CsrView A, const int64_t* __restrict__ rpB, unsigned long long* __restrict__ work) {
  const int lane = threadIdx.x & 31;
  const int64_t I = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t r0 = I * 16;
  if (r0 >= A.rows) return;
  const int64_t r1 = r0 + 16 < A.rows ? r0 + 16 : A.rows;
  const int64_t e0 = A.row_ptr[r0], e1 = A.row_ptr[r1];
  unsigned long long w = 0;
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const int32_t c = A.col[e];
    if (c >= 0 && c < A.cols) w += (unsigned long long)(rpB[c + 1] - rpB[c]);
  }
  for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  if (lane == 0) work[I] = panel_cost(w, e1 - e0);
}

// dst[i] = src[i] - src[0] + add, i < n (a row-pointer slice rebased)
__global__ void rebase_kernel(const int64_t* __restrict__ src, int64_t n, int64_t add, int64_t* __restrict__ dst) {
  const int64_t b = src[0];
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i] - b + add;
}

// x[i] += add, i < n (in place)
__global__ void add_kernel(int64_t* __restrict__ x, int64_t n, int64_t add) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    x[i] += add;
}

void add_offset(int64_t* x, int64_t n, int64_t add, cudaStream_t st) {
  if (n <= 0 || add == 0) return;
  const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 1184));
  add_kernel<<<blocks, 256, 0, st>>>(x, n, add);
  TSG_CUDA(cudaGetLastError());
}

void rebase(const int64_t* src, int64_t n, int64_t add, int64_t* dst, cudaStream_t st) {
  if (n <= 0) return;
  const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 1184));
  rebase_kernel<<<blocks, 256, 0, st>>>(src, n, add, dst);
  TSG_CUDA(cudaGetLastError());
}

// Panel boundaries (rows, 16-aligned): cut p = the first tile row whose
// exclusive cost prefix reaches p/n of the total (paper_2009_14600_b200/
// distributed.py panel_bounds restates the same rule).
std::vector<int64_t> panel_cuts(tsg_ctx* ctx, const tsg_csr* A, const tsg_csr* B, int n) {
  const int64_t T = (A->rows + 15) / 16;
  std::vector<unsigned long long> cum(T + 1, 0);
  if (A->mem == TSG_MEM_HOST && B->mem == TSG_MEM_HOST) {
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        for (int64_t I = T * t / nt; I < T * (t + 1) / nt; ++I) {
          unsigned long long w = 0;
          const int64_t r1 = std::min<int64_t>(A->rows, I * 16 + 16);
          for (int64_t e = A->row_ptr[I * 16]; e < A->row_ptr[r1]; ++e) {
            const int32_t c = A->col[e];
            if (c >= 0 && c < A->cols) w += (unsigned long long)(B->row_ptr[c + 1] - B->row_ptr[c]);
          }
          cum[I + 1] = panel_cost(w, A->row_ptr[r1] - A->row_ptr[I * 16]);
        }
      });
    for (auto& x : th) x.join();
  } else {  // device operands (on devices[0]): the work per tile row on the device
    tsg_ctx* c0 = ctx->sub[0];
    TSG_CUDA(cudaSetDevice(c0->device));
    Scratch sc(c0);
    CsrView va = stage(c0, sc, A, nullptr);
    CsrView vb = stage(c0, sc, B, nullptr);
    auto* w = sc.alloc<unsigned long long>(uint64_t(std::max<int64_t>(T, 1)));
    if (T > 0) {
      tile_row_work_kernel<<<unsigned((T * 32 + 255) / 256), 256, 0, c0->stream>>>(va, vb.row_ptr, w);
      check_launch(c0);
      TSG_CUDA(cudaMemcpyAsync(cum.data() + 1, w, T * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c0->stream));
    }
    TSG_CUDA(cudaStreamSynchronize(c0->stream));
  }
  for (int64_t I = 0; I < T; ++I) cum[I + 1] += cum[I];
  std::vector<int64_t> cut(n + 1, 0);
  const double total = double(cum[T]);
  for (int p = 1; p < n; ++p) {
    const double want = total * p / n;
    const int64_t I = std::lower_bound(cum.begin(), cum.end(), want,
                                       [](unsigned long long a, double b) { return double(a) < b; }) - cum.begin();
    cut[p] = std::max(cut[p - 1], std::min<int64_t>(I, T));
  }
  cut[n] = T;
  for (int p = 0; p <= n; ++p) cut[p] = std::min<int64_t>(cut[p] * 16, A->rows);
  return cut;
}

// Device copy of operand M (on devices[0]) for another device (peer copy
// over NVLink); owner pointers in `keep`.
tsg_csr replicate(const tsg_csr* M, tsg_ctx* to, int from_dev, std::vector<std::pair<tsg_ctx*, void*>>& keep) {
  tsg_csr r = *M;
  const size_t b0 = (M->rows + 1) * sizeof(int64_t), b1 = M->nnz * sizeof(int32_t), b2 = M->nnz * dtype_size(M->dtype);
  void* p[3] = {nullptr, nullptr, nullptr};
  const size_t b[3] = {b0, b1, b2};
  const void* src[3] = {M->row_ptr, M->col, M->val};
  for (int i = 0; i < 3; ++i) {
    TSG_CUDA(cudaMallocFromPoolAsync(&p[i], std::max<size_t>(b[i], 1), to->pool, to->stream));
    keep.emplace_back(to, p[i]);
    if (b[i]) TSG_CUDA(cudaMemcpyPeerAsync(p[i], to->device, src[i], from_dev, b[i], to->stream));
  }
  r.row_ptr = static_cast<int64_t*>(p[0]);
  r.col = static_cast<int32_t*>(p[1]);
  r.val = p[2];
  return r;
}

void merge_stats(tsg_run_stats* into, const tsg_run_stats& s, bool first) {
  double* t = &into->convert;
  const double* u = &s.convert;
  for (int i = 0; i < 7; ++i) t[i] = std::max(t[i], u[i]);  // phase times: the critical path
  uint64_t* a = &into->tiles_a;
  const uint64_t* b = &s.tiles_a;
  for (int i = 0; i < 19; ++i) a[i] += b[i];  // counters and memory: sums over panels
  if (first) into->path = s.path;
}

int spgemm_multi(tsg_ctx* ctx, int nops, const tsg_csr* const* X, tsg_csr_out* C, const tsg_options& o,
                 tsg_run_stats* stats) {
  const int n = int(ctx->sub.size());
  const int dev0 = ctx->sub[0]->device;
  if (!C) throw Fail{TSG_ERR_OTHER, "C is NULL"};
  if (o.want_tiles) throw Fail{TSG_ERR_OTHER, "the tiled parity view needs a single-device context"};
  for (int i = 0; i < nops; ++i) check_csr(X[i], i == 0 ? "A" : "B");
  for (int i = 0; i + 1 < nops; ++i)
    if (X[i]->cols != X[i + 1]->rows)
      throw Fail{TSG_ERR_DIMENSION, "inner dimensions differ: " + std::to_string(X[i]->rows) + "x" +
                                        std::to_string(X[i]->cols) + " . " + std::to_string(X[i + 1]->rows) + "x" +
                                        std::to_string(X[i + 1]->cols)};
  const tsg_csr* A = X[0];
  const std::vector<int64_t> cut = panel_cuts(ctx, A, X[1], n);
  // panels, grouped by device (one host thread per distinct GPU; panels
  // sharing a GPU run one after another)
  std::vector<int> devs;
  for (auto* c : ctx->sub)
    if (std::find(devs.begin(), devs.end(), c->device) == devs.end()) devs.push_back(c->device);
  std::vector<tsg_csr_out> outs(n);
  std::vector<tsg_run_stats> pst(n);
  std::vector<Fail> fails(n, Fail{TSG_OK, ""});
  ctx->panel_ms.assign(n, 0.0);
  std::vector<std::vector<std::pair<tsg_ctx*, void*>>> keeps(devs.size());
  auto run_device = [&](size_t di) {
    const int d = devs[di];
    std::vector<tsg_csr> rep(nops);  // X1.. on this device
    bool have_rep = false;
    for (int p = 0; p < n; ++p) {
      tsg_ctx* c = ctx->sub[p];
      if (c->device != d) continue;
      try {
        TSG_CUDA(cudaSetDevice(d));
        if (!have_rep) {
          for (int i = 1; i < nops; ++i)
            rep[i] = (X[i]->mem == TSG_MEM_DEVICE && d != dev0) ? replicate(X[i], c, dev0, keeps[di]) : *X[i];
          have_rep = true;
        }
        cudaEvent_t ev[2];
        TSG_CUDA(cudaEventCreate(&ev[0]));
        TSG_CUDA(cudaEventCreate(&ev[1]));
        TSG_CUDA(cudaEventRecord(ev[0], c->stream));
        // X0's panel [r0, r1) with rebased row pointers (on this device)
        const int64_t r0 = cut[p], r1 = cut[p + 1];
        tsg_csr a = *A;
        a.rows = r1 - r0;
        std::vector<int64_t> hrp;
        if (A->mem == TSG_MEM_HOST) {
          const int64_t e0 = A->row_ptr[r0];
          hrp.resize(r1 - r0 + 1);
          for (int64_t r = r0; r <= r1; ++r) hrp[r - r0] = A->row_ptr[r] - e0;
          a.row_ptr = hrp.data();
          a.nnz = hrp.back();
          a.col = A->col + e0;
          a.val = static_cast<const char*>(A->val) + e0 * dtype_size(A->dtype);
        } else {
          int64_t e[2];
          TSG_CUDA(cudaMemcpyAsync(e, A->row_ptr + r0, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
          TSG_CUDA(cudaMemcpyAsync(e + 1, A->row_ptr + r1, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
          TSG_CUDA(cudaStreamSynchronize(c->stream));
          a.nnz = e[1] - e[0];
          void* rp = nullptr;
          TSG_CUDA(cudaMallocFromPoolAsync(&rp, (a.rows + 1) * sizeof(int64_t), c->pool, c->stream));
          keeps[di].emplace_back(c, rp);
          if (d == dev0) {
            rebase(A->row_ptr + r0, a.rows + 1, 0, static_cast<int64_t*>(rp), c->stream);
            a.col = A->col + e[0];
            a.val = static_cast<const char*>(A->val) + e[0] * dtype_size(A->dtype);
          } else {
            void* tmp = nullptr;
            TSG_CUDA(cudaMallocFromPoolAsync(&tmp, (a.rows + 1) * sizeof(int64_t), c->pool, c->stream));
            keeps[di].emplace_back(c, tmp);
            TSG_CUDA(cudaMemcpyPeerAsync(tmp, d, A->row_ptr + r0, dev0, (a.rows + 1) * sizeof(int64_t), c->stream));
            rebase(static_cast<int64_t*>(tmp), a.rows + 1, 0, static_cast<int64_t*>(rp), c->stream);
            void* cv[2] = {nullptr, nullptr};
            const size_t bb[2] = {a.nnz * sizeof(int32_t), a.nnz * dtype_size(A->dtype)};
            const void* src[2] = {A->col + e[0], static_cast<const char*>(A->val) + e[0] * dtype_size(A->dtype)};
            for (int i = 0; i < 2; ++i) {
              TSG_CUDA(cudaMallocFromPoolAsync(&cv[i], std::max<size_t>(bb[i], 1), c->pool, c->stream));
              keeps[di].emplace_back(c, cv[i]);
              if (bb[i]) TSG_CUDA(cudaMemcpyPeerAsync(cv[i], d, src[i], dev0, bb[i], c->stream));
            }
            a.col = static_cast<int32_t*>(cv[0]);
            a.val = cv[1];
          }
          a.row_ptr = static_cast<int64_t*>(rp);
        }
        outs[p] = tsg_csr_out{};
        outs[p].mem = TSG_MEM_DEVICE;
        std::memset(&pst[p], 0, sizeof(tsg_run_stats));
        if (nops == 2) {
          spgemm_impl(c, &a, &rep[1], &outs[p], o, &pst[p], nullptr);
        } else {
          std::vector<const tsg_csr*> xs(nops);
          xs[0] = &a;
          for (int i = 1; i < nops; ++i) xs[i] = &rep[i];
          const int rc = tsg_spgemm_chain(c, nops, xs.data(), &outs[p], &o, &pst[p]);
          if (rc != TSG_OK) throw Fail{rc, c->err};
        }
        TSG_CUDA(cudaEventRecord(ev[1], c->stream));
        TSG_CUDA(cudaEventSynchronize(ev[1]));
        float ms = 0;
        TSG_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
        ctx->panel_ms[p] = ms;
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
      } catch (const Fail& f) {
        fails[p] = f;
      }
    }
  };
  {
    std::vector<std::thread> th;
    for (size_t di = 0; di < devs.size(); ++di) th.emplace_back(run_device, di);
    for (auto& t : th) t.join();
  }
  auto release = [&]() {
    for (int p = 0; p < n; ++p)
      if (outs[p]._owner) {
        cudaSetDevice(ctx->sub[p]->device);
        free_out(ctx->sub[p], &outs[p]);
      }
    for (auto& k : keeps)
      for (auto& [c, ptr] : k) {
        cudaSetDevice(c->device);
        cudaFreeAsync(ptr, c->stream);
      }
    for (auto* c : ctx->sub) cudaStreamSynchronize(c->stream);
    cudaSetDevice(dev0);
  };
  for (int p = 0; p < n; ++p)
    if (fails[p].code != TSG_OK) {
      release();
      throw fails[p];
    }
  // concatenate: panel p's entries start at the sum of the earlier panels' nnz
  int64_t nnz = 0;
  std::vector<int64_t> base(n + 1, 0);
  for (int p = 0; p < n; ++p) base[p + 1] = base[p] + outs[p].nnz;
  nnz = base[n];
  const int64_t rows = A->rows;
  tsg_ctx* c0 = ctx->sub[0];
  auto* owner = new OutOwner();
  owner->host = C->mem == TSG_MEM_HOST;
  C->_owner = owner;
  uint64_t d2h = 0;
  try {
    if (owner->host) {
      owner->p[0] = pinned_alloc(c0, (rows + 1) * sizeof(int64_t), &owner->sz[0]);
      owner->p[1] = pinned_alloc(c0, std::max<int64_t>(nnz, 1) * sizeof(int32_t), &owner->sz[1]);
      owner->p[2] = pinned_alloc(c0, std::max<int64_t>(nnz, 1) * sizeof(float), &owner->sz[2]);
      for (int p = 0; p < n; ++p) {  // every device ships its slice straight into place
        tsg_ctx* c = ctx->sub[p];
        TSG_CUDA(cudaSetDevice(c->device));
        const int64_t nr = cut[p + 1] - cut[p];
        add_offset(outs[p].row_ptr, nr, base[p], c->stream);
        TSG_CUDA(cudaMemcpyAsync(static_cast<int64_t*>(owner->p[0]) + cut[p], outs[p].row_ptr, nr * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, c->stream));
        if (outs[p].nnz) {
          TSG_CUDA(cudaMemcpyAsync(static_cast<int32_t*>(owner->p[1]) + base[p], outs[p].col,
                                   outs[p].nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
          TSG_CUDA(cudaMemcpyAsync(static_cast<float*>(owner->p[2]) + base[p], outs[p].val,
                                   outs[p].nnz * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        }
        d2h += nr * sizeof(int64_t) + outs[p].nnz * (sizeof(int32_t) + sizeof(float));
      }
      for (auto* c : ctx->sub) TSG_CUDA(cudaStreamSynchronize(c->stream));
      static_cast<int64_t*>(owner->p[0])[rows] = nnz;
    } else {
      TSG_CUDA(cudaSetDevice(dev0));
      for (int i = 0; i < 3; ++i) {
        const size_t b = i == 0 ? (rows + 1) * sizeof(int64_t) : std::max<int64_t>(nnz, 1) * 4;
        TSG_CUDA(cudaMallocFromPoolAsync(&owner->p[i], b, c0->pool, c0->stream));
      }
      for (auto* c : ctx->sub) TSG_CUDA(cudaStreamSynchronize(c->stream));  // every slice is final
      auto* rp = static_cast<int64_t*>(owner->p[0]);
      for (int p = 0; p < n; ++p) {
        const int dp = ctx->sub[p]->device;
        const int64_t nr = cut[p + 1] - cut[p];
        if (nr > 0) {
          TSG_CUDA(cudaMemcpyPeerAsync(rp + cut[p], dev0, outs[p].row_ptr, dp, nr * sizeof(int64_t), c0->stream));
          add_offset(rp + cut[p], nr, base[p], c0->stream);
        }
        if (outs[p].nnz) {
          TSG_CUDA(cudaMemcpyPeerAsync(static_cast<int32_t*>(owner->p[1]) + base[p], dev0, outs[p].col, dp,
                                       outs[p].nnz * sizeof(int32_t), c0->stream));
          TSG_CUDA(cudaMemcpyPeerAsync(static_cast<float*>(owner->p[2]) + base[p], dev0, outs[p].val, dp,
                                       outs[p].nnz * sizeof(float), c0->stream));
        }
      }
      TSG_CUDA(cudaMemcpyAsync(rp + rows, &base[n], sizeof(int64_t), cudaMemcpyHostToDevice, c0->stream));
      TSG_CUDA(cudaStreamSynchronize(c0->stream));
    }
  } catch (...) {
    release();
    throw;
  }
  release();
  C->rows = rows;
  C->cols = X[nops - 1]->cols;
  C->nnz = nnz;
  C->row_ptr = static_cast<int64_t*>(owner->p[0]);
  C->col = static_cast<int32_t*>(owner->p[1]);
  C->val = static_cast<float*>(owner->p[2]);
  if (stats) {
    tsg_run_stats agg;
    std::memset(&agg, 0, sizeof(agg));
    for (int p = 0; p < n; ++p) merge_stats(&agg, pst[p], p == 0);
    agg.nnz_c = uint64_t(nnz);
    agg.d2h_bytes += d2h;
    agg.devices = n;
    double* t = &stats->convert;
    const double* u = &agg.convert;
    for (int i = 0; i < 7; ++i) t[i] += u[i];
    uint64_t* a = &stats->tiles_a;
    const uint64_t* b = &agg.tiles_a;
    for (int i = 0; i < 19; ++i) a[i] += b[i];
    stats->nnz_c = agg.nnz_c;
    stats->path = agg.path;
    stats->devices = n;
  }
  return TSG_OK;
}

}  // namespace

extern "C" {

void tsg_default_options(tsg_options* opt) {
  if (!opt) return;
  std::memset(opt, 0, sizeof(*opt));
  opt->mode = TSG_MODE_TENSOR;
}

int tsg_abi_version(void) { return TSG_ABI_VERSION; }

int tsg_create(tsg_ctx** out, int device, void* stream) {
  if (!out) return TSG_ERR_OTHER;
  *out = nullptr;
  auto* ctx = new tsg_ctx();
  cudaError_t e = cudaSuccess;
  if (device < 0) e = cudaGetDevice(&ctx->device);
  else ctx->device = device;
  if (e == cudaSuccess) e = cudaSetDevice(ctx->device);
  if (e == cudaSuccess) {
    if (stream) {
      ctx->stream = static_cast<cudaStream_t>(stream);
    } else {
      e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
      ctx->own_stream = true;
    }
  }
  if (e == cudaSuccess) e = cudaDeviceGetDefaultMemPool(&ctx->pool, ctx->device);
  if (e == cudaSuccess) {
    uint64_t thr = ~uint64_t(0);
    e = cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->pinned, 64 + 8 * kGatherMax);
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->pinned_pipe, 16 * (tsg::kPipeChunks + 1));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking);
  for (int i = 0; i <= tsg::kPipeChunks && e == cudaSuccess; ++i)
    e = cudaEventCreateWithFlags(&ctx->pipe_ev[i], cudaEventDisableTiming);
  for (int i = 0; i < tsg::kPipeChunks && e == cudaSuccess; ++i)
    e = cudaEventCreateWithFlags(&ctx->d2h_ev[i], cudaEventDisableTiming);
  for (int i = 0; i < 8 && e == cudaSuccess; ++i) e = cudaEventCreate(&ctx->ev[i]);
  for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreate(&ctx->kev[i]);
  if (e != cudaSuccess) {
    std::fprintf(stderr, "tsg_create: %s\n", cudaGetErrorString(e));
    delete ctx;
    return TSG_ERR_OTHER;
  }
  *out = ctx;
  return TSG_OK;
}

int tsg_create_multi(tsg_ctx** out, int n, const int* devices) {
  if (!out || n < 1 || n > 1024) return TSG_ERR_OTHER;
  *out = nullptr;
  auto* m = new tsg_ctx();
  for (int i = 0; i < n; ++i) {
    tsg_ctx* c = nullptr;
    const int rc = tsg_create(&c, devices ? devices[i] : i, nullptr);
    if (rc != TSG_OK) {
      for (auto* x : m->sub) tsg_destroy(x);
      m->sub.clear();
      delete m;
      return rc;
    }
    m->sub.push_back(c);
  }
  // the front context: device, stream, pool and pinned cache of panel 0
  m->device = m->sub[0]->device;
  m->stream = m->sub[0]->stream;
  m->pool = m->sub[0]->pool;
  cudaSetDevice(m->device);
  *out = m;
  return TSG_OK;
}

int tsg_last_panel_ms(const tsg_ctx* ctx, double* out, int n) {
  if (!ctx) return 0;
  const int k = int(ctx->panel_ms.size());
  for (int i = 0; i < k && i < n && out; ++i) out[i] = ctx->panel_ms[i];
  return k;
}

int tsg_destroy(tsg_ctx* ctx) {
  if (!ctx) return TSG_OK;
  if (!ctx->sub.empty()) {  // a multi-device front: everything belongs to the panel contexts
    for (auto* c : ctx->sub) tsg_destroy(c);
    delete ctx;
    return TSG_OK;
  }
  cudaStreamSynchronize(ctx->stream);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->kev)
    if (e) cudaEventDestroy(e);
  if (ctx->stage_buf) cudaFreeAsync(ctx->stage_buf, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->pinned_pipe) cudaFreeHost(ctx->pinned_pipe);
  for (auto& e : ctx->pipe_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->d2h_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->d2h) {
    cudaStreamSynchronize(ctx->d2h);
    cudaStreamDestroy(ctx->d2h);
  }
  for (auto& b : ctx->pinned_free) cudaFreeHost(b.first);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return TSG_OK;
}

const char* tsg_last_error(const tsg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int tsg_spgemm(tsg_ctx* ctx, const tsg_csr* A, const tsg_csr* B, tsg_csr_out* C,
               const tsg_options* opt, tsg_run_stats* stats, tsg_tiles_out* tiles) {
  if (!ctx) return TSG_ERR_OTHER;
  tsg_options o;
  tsg_default_options(&o);
  if (opt) o = *opt;
  ctx->err.clear();
  if (C) C->_owner = nullptr;
  try {
    TSG_CUDA(cudaSetDevice(ctx->device));
    if (!ctx->sub.empty()) {
      const tsg_csr* X[2] = {A, B};
      return spgemm_multi(ctx, 2, X, C, o, stats);
    }
    spgemm_impl(ctx, A, B, C, o, stats, o.want_tiles ? tiles : nullptr);
    return TSG_OK;
  } catch (const Fail& f) {
    ctx->err = f.msg;
    cudaStreamSynchronize(ctx->stream);
    if (C && C->_owner) free_out(ctx, C);
    return f.code;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return TSG_ERR_OTHER;
  }
}

int tsg_bsum_create(tsg_ctx* ctx, const tsg_csr* Bpanel, tsg_bsum* out) {
  if (!ctx || !out) return TSG_ERR_OTHER;
  ctx->err.clear();
  if (!ctx->sub.empty()) {
    ctx->err = "B summaries are per device: use a single-device context";
    return TSG_ERR_OTHER;
  }
  try {
    TSG_CUDA(cudaSetDevice(ctx->device));
    bsum_create_impl(ctx, Bpanel, out);
    return TSG_OK;
  } catch (const Fail& f) {
    ctx->err = f.msg;
    cudaStreamSynchronize(ctx->stream);
    return f.code;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return TSG_ERR_OTHER;
  }
}

void tsg_bsum_free(tsg_ctx* ctx, tsg_bsum* s) {
  if (!ctx || !s || !s->_owner) return;
  auto* own = static_cast<std::vector<void*>*>(s->_owner);
  cudaSetDevice(ctx->device);
  for (void* p : *own) cudaFreeAsync(p, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  delete own;
  *s = tsg_bsum{};
}

int tsg_spgemm_bsum(tsg_ctx* ctx, const tsg_csr* A, const tsg_csr* B, const tsg_bsum* Bsum, tsg_csr_out* C,
                    const tsg_options* opt, tsg_run_stats* stats) {
  if (!ctx) return TSG_ERR_OTHER;
  tsg_options o;
  tsg_default_options(&o);
  if (opt) o = *opt;
  o.want_tiles = 0;
  ctx->err.clear();
  if (C) C->_owner = nullptr;
  if (!ctx->sub.empty()) {
    ctx->err = "tsg_spgemm_bsum runs one GPU's panel: use a single-device context";
    return TSG_ERR_OTHER;
  }
  try {
    TSG_CUDA(cudaSetDevice(ctx->device));
    spgemm_bsum_impl(ctx, A, B, Bsum, C, o, stats);
    return TSG_OK;
  } catch (const Fail& f) {
    ctx->err = f.msg;
    cudaStreamSynchronize(ctx->stream);
    if (C && C->_owner) free_out(ctx, C);
    return f.code;
  } catch (const std::exception& e) {
    ctx->err = e.what();
    return TSG_ERR_OTHER;
  }
}

int tsg_spgemm_chain(tsg_ctx* ctx, int n, const tsg_csr* const* X, tsg_csr_out* C,
                     const tsg_options* opt, tsg_run_stats* stats) {
  if (!ctx) return TSG_ERR_OTHER;
  if (n < 2 || !X || !C) {
    ctx->err = "chain needs at least two operands";
    return TSG_ERR_OTHER;
  }
  tsg_options o;
  tsg_default_options(&o);
  if (opt) o = *opt;
  o.want_tiles = 0;
  ctx->err.clear();
  if (!ctx->sub.empty()) {
    try {
      TSG_CUDA(cudaSetDevice(ctx->device));
      return spgemm_multi(ctx, n, X, C, o, stats);
    } catch (const Fail& f) {
      ctx->err = f.msg;
      return f.code;
    }
  }
  // Left to right.  Between stages the intermediate is rounded to binary16
  // (kernels.cpp:239-258).  When a stage takes the light-row path its result
  // goes to the next stage directly as A tiles (the downcast fused into the
  // emission); otherwise as a device fp32 CSR rounded by the next conversion.
  std::vector<void*> keep[2];  // emitted tile arrays of the previous / current stage
  TileMat tiles[2];
  const TileMat* pre = nullptr;
  tsg_csr_out cur{};
  bool have_cur = false;
  int rc = TSG_OK;
  try {
    TSG_CUDA(cudaSetDevice(ctx->device));
    for (int i = 1; i < n && rc == TSG_OK; ++i) {
      const bool last = i == n - 1;
      tsg_csr left{};
      if (!pre) {
        if (!have_cur) {
          left = *X[0];
        } else {
          left.rows = cur.rows;
          left.cols = cur.cols;
          left.nnz = cur.nnz;
          left.row_ptr = cur.row_ptr;
          left.col = cur.col;
          left.val = cur.val;
          left.dtype = TSG_F32;
          left.mem = TSG_MEM_DEVICE;
        }
      } else {
        left.rows = pre->rows;
        left.cols = pre->cols;
      }
      tsg_csr_out next{};
      next.mem = last ? C->mem : TSG_MEM_DEVICE;
      const int w = i & 1;
      for (void* p : keep[w]) cudaFreeAsync(p, ctx->stream);
      keep[w].clear();
      bool emitted = false;
      try {
        emitted = chain_stage(ctx, &left, pre, X[i], &next, last ? nullptr : &tiles[w],
                              &keep[w], o, stats);
      } catch (const Fail& f) {
        ctx->err = f.msg;
        cudaStreamSynchronize(ctx->stream);
        if (next._owner) free_out(ctx, &next);
        rc = f.code;
      } catch (const std::exception& e) {
        ctx->err = e.what();
        cudaStreamSynchronize(ctx->stream);
        if (next._owner) free_out(ctx, &next);
        rc = TSG_ERR_OTHER;
      }
      if (have_cur) free_out(ctx, &cur);
      have_cur = false;
      for (void* p : keep[w ^ 1]) cudaFreeAsync(p, ctx->stream);  // the previous stage's tiles are consumed
      keep[w ^ 1].clear();
      if (rc != TSG_OK) break;
      if (emitted) {
        free_out(ctx, &next);  // no CSR for an emitting stage
        pre = &tiles[w];
      } else {
        pre = nullptr;
        cur = next;
        have_cur = true;
      }
    }
  } catch (const Fail& f) {
    ctx->err = f.msg;
    rc = f.code;
  }
  for (auto& k : keep)
    for (void* p : k) cudaFreeAsync(p, ctx->stream);
  if (rc != TSG_OK) {
    if (have_cur) free_out(ctx, &cur);
    cudaStreamSynchronize(ctx->stream);
    return rc;
  }
  *C = cur;
  cudaStreamSynchronize(ctx->stream);
  return TSG_OK;
}

void tsg_free_csr(tsg_ctx* ctx, tsg_csr_out* C) {
  if (!ctx) return;
  tsg_ctx* c = ctx->sub.empty() ? ctx : ctx->sub[0];  // a multi-device output lives on panel 0's device
  cudaSetDevice(c->device);
  free_out(c, C);
  cudaStreamSynchronize(c->stream);
}

void tsg_free_tiles(tsg_tiles_out* t) {
  if (!t) return;
  std::free(t->tile_row);
  std::free(t->tile_col);
  std::free(t->row_masks);
  std::free(t->elem_index);
  std::free(t->val);
  std::memset(t, 0, sizeof(*t));
}

int tsg_cbar(tsg_ctx* ctx, const tsg_csr* A, const tsg_csr* B, uint64_t* cbar) {
  if (!ctx || !cbar) return TSG_ERR_OTHER;
  if (!ctx->sub.empty()) {
    const int rc = tsg_cbar(ctx->sub[0], A, B, cbar);
    ctx->err = ctx->sub[0]->err;
    return rc;
  }
  ctx->err.clear();
  try {
    check_csr(A, "A");
    check_csr(B, "B");
    if (A->cols != B->rows) throw Fail{TSG_ERR_DIMENSION, "inner dimensions differ"};
    Scratch sc(ctx);
    const CsrView dA = stage(ctx, sc, A, nullptr);
    const CsrView dB = stage(ctx, sc, B, nullptr);
    auto* hist = sc.alloc<unsigned>(A->cols);
    auto* out = sc.alloc<unsigned long long>(1);
    TSG_CUDA(cudaMemsetAsync(hist, 0, A->cols * sizeof(unsigned), ctx->stream));
    TSG_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long), ctx->stream));
    launch_cbar(dA.col, dA.nnz, A->cols, dB.row_ptr, hist, out, ctx->stream);
    check_launch(ctx, 2);
    *cbar = readback(ctx, out);
    return TSG_OK;
  } catch (const Fail& f) {
    ctx->err = f.msg;
    return f.code;
  }
}

int tsg_tiles8_to_csr(tsg_ctx* ctx, const tsg_tiles8* T, tsg_csr_out* C) {
  if (!ctx || !T || !C) return TSG_ERR_OTHER;
  if (!ctx->sub.empty()) {
    const int rc = tsg_tiles8_to_csr(ctx->sub[0], T, C);
    ctx->err = ctx->sub[0]->err;
    return rc;
  }
  ctx->err.clear();
  C->_owner = nullptr;
  try {
    TSG_CUDA(cudaSetDevice(ctx->device));
    if (T->rows < 0 || T->cols < 0 || T->ntiles < 0 || T->nnz < 0)
      throw Fail{TSG_ERR_INVARIANT, "tiles8: negative size"};
    if (T->nnz >= (int64_t(1) << 32)) throw Fail{TSG_ERR_OTHER, "tiles8: more than 2^32 elements"};
    Scratch sc(ctx);
    cudaStream_t s = ctx->stream;
    const int64_t rows = T->rows, nt = T->ntiles, tile_rows = (rows + 7) / 8;
    auto dev = [&](const void* p, size_t bytes) -> const void* {  // host arrays -> device
      if (T->mem == TSG_MEM_DEVICE || bytes == 0) return p;
      char* d = sc.alloc<char>(bytes);
      TSG_CUDA(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, s));
      return d;
    };
    const auto* trow = static_cast<const uint32_t*>(dev(T->tile_row, nt * 4));
    Tiles8View v;
    v.tile_col = static_cast<const uint32_t*>(dev(T->tile_col, nt * 4));
    v.bitmap = static_cast<const unsigned long long*>(dev(T->bitmap, nt * 8));
    v.elem_index = static_cast<const unsigned long long*>(dev(T->elem_index, nt * 8));
    v.val = static_cast<const float*>(dev(T->val, T->nnz * 4));
    auto* err = sc.alloc<unsigned>(1);
    TSG_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned), s));
    auto* trp = sc.alloc<uint32_t>(tile_rows + 1);
    TSG_CUDA(cudaMemsetAsync(trp, 0, (tile_rows + 1) * sizeof(uint32_t), s));
    launch_tiles8_trp(trow, nt, tile_rows, trp, err, s);
    auto* rowcnt = sc.alloc<int64_t>(rows + 1);
    TSG_CUDA(cudaMemsetAsync(rowcnt, 0, (rows + 1) * sizeof(int64_t), s));
    launch_tiles8_to_csr(v, trp, rows, rowcnt, nullptr, nullptr, nullptr, err, true, s);
    auto* rp = sc.alloc<int64_t>(rows + 1);
    exclusive_sum(ctx, sc, rowcnt, rp, uint64_t(rows) + 1);
    check_launch(ctx, 2);
    const int64_t nnz = readback(ctx, rp + rows);
    const unsigned ev = readback(ctx, err);
    if (ev & kErrInvariant) throw Fail{TSG_ERR_INVARIANT, "tiles8: tiles not sorted by row"};
    if (nnz != T->nnz) throw Fail{TSG_ERR_INVARIANT, "tiles8: bitmap population != element count"};
    auto* col = sc.alloc<int32_t>(nnz);
    auto* val = sc.alloc<float>(nnz);
    launch_tiles8_to_csr(v, trp, rows, nullptr, rp, col, val, err, false, s);
    check_launch(ctx);
    auto* owner = new OutOwner();
    owner->host = C->mem == TSG_MEM_HOST;
    C->_owner = owner;
    if (owner->host) {
      owner->p[0] = pinned_alloc(ctx, (rows + 1) * sizeof(int64_t), &owner->sz[0]);
      owner->p[1] = pinned_alloc(ctx, std::max<int64_t>(nnz, 1) * sizeof(int32_t), &owner->sz[1]);
      owner->p[2] = pinned_alloc(ctx, std::max<int64_t>(nnz, 1) * sizeof(float), &owner->sz[2]);
      TSG_CUDA(cudaMemcpyAsync(owner->p[0], rp, (rows + 1) * 8, cudaMemcpyDeviceToHost, s));
      if (nnz) {
        TSG_CUDA(cudaMemcpyAsync(owner->p[1], col, nnz * 4, cudaMemcpyDeviceToHost, s));
        TSG_CUDA(cudaMemcpyAsync(owner->p[2], val, nnz * 4, cudaMemcpyDeviceToHost, s));
      }
    } else {  // keep the device arrays
      owner->p[0] = rp;
      owner->p[1] = col;
      owner->p[2] = val;
      sc.ptrs.erase(std::remove_if(sc.ptrs.begin(), sc.ptrs.end(),
                                   [&](void* q) { return q == rp || q == col || q == val; }),
                    sc.ptrs.end());
    }
    TSG_CUDA(cudaStreamSynchronize(s));
    C->rows = rows;
    C->cols = T->cols;
    C->nnz = nnz;
    C->row_ptr = static_cast<int64_t*>(owner->p[0]);
    C->col = static_cast<int32_t*>(owner->p[1]);
    C->val = static_cast<float*>(owner->p[2]);
    return TSG_OK;
  } catch (const Fail& f) {
    ctx->err = f.msg;
    cudaStreamSynchronize(ctx->stream);
    if (C->_owner) free_out(ctx, C);
    return f.code;
  }
}

int tsg_csr_to_tiles8(tsg_ctx* ctx, const tsg_csr* C, tsg_tiles8_out* T) {
  if (!ctx || !C || !T) return TSG_ERR_OTHER;
  if (!ctx->sub.empty()) {
    const int rc = tsg_csr_to_tiles8(ctx->sub[0], C, T);
    ctx->err = ctx->sub[0]->err;
    return rc;
  }
  ctx->err.clear();
  std::memset(T, 0, sizeof(*T));
  try {
    TSG_CUDA(cudaSetDevice(ctx->device));
    check_csr(C, "C");
    if (C->dtype != TSG_F32) throw Fail{TSG_ERR_OTHER, "tiles8: fp32 values expected (the product's output)"};
    Scratch sc(ctx);
    cudaStream_t s = ctx->stream;
    const CsrView v = stage(ctx, sc, C, nullptr);
    const int64_t groups = (C->rows + 7) / 8;
    auto* err = sc.alloc<unsigned>(1);
    TSG_CUDA(cudaMemsetAsync(err, 0, sizeof(unsigned), s));
    auto* gt = sc.alloc<uint32_t>(groups + 1);
    auto* ge = sc.alloc<uint32_t>(groups + 1);
    TSG_CUDA(cudaMemsetAsync(gt + groups, 0, 4, s));
    TSG_CUDA(cudaMemsetAsync(ge + groups, 0, 4, s));
    launch_validate_rowptr(v, err, s);
    launch_csr_tiles8_count(v, static_cast<const float*>(v.val), gt, ge, err, s);
    check_launch(ctx, 2);
    auto* toff = sc.alloc<unsigned long long>(groups + 1);
    auto* eoff = sc.alloc<unsigned long long>(groups + 1);
    exclusive_sum(ctx, sc, gt, toff, uint64_t(groups) + 1);
    exclusive_sum(ctx, sc, ge, eoff, uint64_t(groups) + 1);
    const unsigned long long* src[2] = {toff + groups, eoff + groups};
    unsigned long long tot[2];
    readback_many(ctx, src, tot);
    raise_flags(readback(ctx, err));
    const int64_t nt = int64_t(tot[0]), ne = int64_t(tot[1]);
    Tiles8Out o;
    o.tile_row = sc.alloc<uint32_t>(nt);
    o.tile_col = sc.alloc<uint32_t>(nt);
    o.bitmap = sc.alloc<unsigned long long>(nt);
    o.elem_index = sc.alloc<unsigned long long>(nt);
    o.val = sc.alloc<float>(ne);
    launch_csr_tiles8_write(v, static_cast<const float*>(v.val), toff, eoff, o, s);
    check_launch(ctx);
    T->rows = C->rows;
    T->cols = C->cols;
    T->ntiles = nt;
    T->nnz = ne;
    T->tile_row = static_cast<uint32_t*>(std::malloc(std::max<int64_t>(nt, 1) * 4));
    T->tile_col = static_cast<uint32_t*>(std::malloc(std::max<int64_t>(nt, 1) * 4));
    T->bitmap = static_cast<uint64_t*>(std::malloc(std::max<int64_t>(nt, 1) * 8));
    T->elem_index = static_cast<uint64_t*>(std::malloc(std::max<int64_t>(nt, 1) * 8));
    T->val = static_cast<float*>(std::malloc(std::max<int64_t>(ne, 1) * 4));
    if (nt) {
      TSG_CUDA(cudaMemcpyAsync(T->tile_row, o.tile_row, nt * 4, cudaMemcpyDeviceToHost, s));
      TSG_CUDA(cudaMemcpyAsync(T->tile_col, o.tile_col, nt * 4, cudaMemcpyDeviceToHost, s));
      TSG_CUDA(cudaMemcpyAsync(T->bitmap, o.bitmap, nt * 8, cudaMemcpyDeviceToHost, s));
      TSG_CUDA(cudaMemcpyAsync(T->elem_index, o.elem_index, nt * 8, cudaMemcpyDeviceToHost, s));
    }
    if (ne) TSG_CUDA(cudaMemcpyAsync(T->val, o.val, ne * 4, cudaMemcpyDeviceToHost, s));
    TSG_CUDA(cudaStreamSynchronize(s));
    return TSG_OK;
  } catch (const Fail& f) {
    ctx->err = f.msg;
    cudaStreamSynchronize(ctx->stream);
    tsg_free_tiles8(T);
    return f.code;
  }
}

void tsg_free_tiles8(tsg_tiles8_out* T) {
  if (!T) return;
  std::free(T->tile_row);
  std::free(T->tile_col);
  std::free(T->bitmap);
  std::free(T->elem_index);
  std::free(T->val);
  std::memset(T, 0, sizeof(*T));
}

uint64_t tsg_launch_count(const tsg_ctx* ctx) {
  if (!ctx) return 0;
  uint64_t n = ctx->launches;
  for (auto* c : ctx->sub) n += c->launches;
  return n;
}

double tsg_last_kernel_ms(const tsg_ctx* ctx, const char* phase) {
  if (!ctx || !phase) return 0.0;
  if (!ctx->sub.empty()) return tsg_last_kernel_ms(ctx->sub[0], phase);
  if (std::strcmp(phase, "numeric_kernel") == 0) return ctx->last_numeric_kernel_ms;
  if (std::strcmp(phase, "assemble_kernel") == 0) return ctx->last_assemble_kernel_ms;
  if (std::strcmp(phase, "bsum") == 0) return ctx->last_bsum_ms;
  static const char* names[] = {"", "convert", "task_list", "sort", "counting", "multiply",
                                "compaction", "total"};
  for (int i = 1; i < 8; ++i)
    if (std::strcmp(phase, names[i]) == 0) return ctx->last_phase_ms[i];
  return 0.0;
}

}  // extern "C"
