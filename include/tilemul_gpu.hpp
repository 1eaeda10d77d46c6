// tilemul_gpu.hpp -- header-only C++ drop-in over the C ABI (tsparse_b200.h).
//
// Re-exposes the reference's hot-path API (namespace tilemul in
// /root/reference/proj/include/tilemul) with the same type and function
// names, field meanings and exception taxonomy, backed by the B200 CUDA
// library.  Code written against the reference switches by replacing
//
//   #include "tilemul/kernels.hpp"        ->  #include "tilemul_gpu.hpp"
//   using namespace tilemul;              ->  using namespace tilemul_gpu;
//
// Mirrored names (reference file:line):
//   ElementCoo                  coo.hpp:11-26
//   ElementKind, TileEntry,
//   TiledMatrix (8x8 tiles)     tile_format.hpp:12-55
//   validate_coo                tile_format.hpp:66-69  (InvariantError)
//   from_element_coo            tile_format.hpp:71-72  (host, 8x8 -- for callers
//   to_element_coo              tile_format.hpp:75      that hold TiledMatrix)
//   MemoryReport                report.hpp:19-27       (device accounting)
//   PhaseTiming                 report.hpp:10-17
//   SquareOptions/SquareResult  kernels.hpp:69-89
//   spgemm_square               kernels.hpp:88-89      (runs on the GPU)
//   Error ... PrecisionError    errors.hpp:9-51
// New: spgemm(A, B) and spgemm_chain({R, A, P}).
//
// The 8x8 TiledMatrix stays the interchange type of spgemm_square so callers
// keep working unchanged; internally the GPU uses 16x16 tiles and the result
// comes back as the Fp32Stored 8x8 tiling of its CSR -- the same tiles the
// reference tests build as their expected output with
// from_element_coo(Fp32Stored) (proj/tests/test_kernels.cpp:280-283).
#pragma once

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsparse_b200.h"

namespace tilemul_gpu {

// ---- errors (errors.hpp:9-51) ---------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvariantError : Error {
  using Error::Error;
};
struct OverflowError : Error {
  using Error::Error;
};
struct DimensionError : Error {
  using Error::Error;
};
struct PrecisionError : Error {
  using Error::Error;
};
// input-side taxonomy of the reference front end (errors.hpp:14-33)
struct ParseError : Error {
  using Error::Error;
};
struct UnsupportedError : ParseError {
  using ParseError::ParseError;
};
struct IoError : Error {
  using Error::Error;
};
struct FormatError : Error {
  using Error::Error;
};

inline void throw_status(int st, const std::string& msg) {
  switch (st) {
    case TSG_OK: return;
    case TSG_ERR_INVARIANT: throw InvariantError(msg);
    case TSG_ERR_OVERFLOW: throw OverflowError(msg);
    case TSG_ERR_DIMENSION: throw DimensionError(msg);
    case TSG_ERR_PRECISION: throw PrecisionError(msg);
    default: throw Error(msg);
  }
}

// ---- data model (coo.hpp, tile_format.hpp, report.hpp) ----------------------
struct ElementCoo {
  std::uint64_t rows = 0, cols = 0;
  struct Entry {
    std::uint64_t row = 0, col = 0;
    double value = 0.0;
  };
  std::vector<Entry> entries;  // sorted by (row, col), no duplicates
};

inline constexpr int kTileDim = 8;
enum class ElementKind : std::uint8_t { Fp16Stored = 0, Fp32Stored = 1 };

struct TileEntry {
  std::uint32_t tile_row = 0, tile_col = 0;
  std::uint64_t elem_index = 0;
  std::uint64_t bitmap = 0;  // bit 8r+c <=> slot (r, c)
  friend bool operator==(const TileEntry&, const TileEntry&) = default;
};

struct TiledMatrix {
  std::uint64_t rows = 0, cols = 0;
  ElementKind kind = ElementKind::Fp16Stored;
  std::vector<TileEntry> tiles;
  std::vector<float> elements;
  std::uint64_t nnz() const { return elements.size(); }
  std::uint64_t tile_rows() const { return (rows + kTileDim - 1) / kTileDim; }
  std::uint64_t tile_cols() const { return (cols + kTileDim - 1) / kTileDim; }
  friend bool operator==(const TiledMatrix&, const TiledMatrix&) = default;  // tile_format.hpp:54
};

struct PhaseTiming {
  double task_list = 0, sort = 0, counting = 0, multiply = 0, compaction = 0, total = 0;
};

// report.hpp:19-27 field names; filled from the device's own accounting
// (tsg_run_stats.mem_*): allocated bytes by role and the pool's high-water
// mark of the call, not the reference's CPU model (analytics.cpp:120-152).
struct MemoryReport {
  std::uint64_t input_tiles_bytes = 0, input_elements_bytes = 0, task_list_bytes = 0, counting_bytes = 0,
                pre_compaction_bytes = 0, output_bytes = 0, peak_bytes = 0;
};

struct SquareOptions {
  bool pairing = true;    // accepted for compatibility; 16x16 tiles need no pairing
  // the reference's worker count (kernels.hpp:71, threading.hpp:14-25) maps to
  // GPUs: 0 = TILEMUL_GPUS from the environment, else 1; n > 1 splits A into
  // n work-balanced tile-row panels on GPUs 0 .. n-1 (tsg_create_multi)
  unsigned threads = 0;
  bool ordered = false;   // true: bit-exact CUDA-core numerics (TSG_MODE_ORDERED)
};

struct SquareResult {
  TiledMatrix output;
  PhaseTiming timing;
  MemoryReport memory;
  std::uint64_t raw_pairs = 0, filtered_pairs = 0, output_tiles_allocated = 0,
                counted_elements = 0;
  unsigned threads_used = 1;  // GPUs the call ran on
};

// ---- ElementCoo validation and 8x8 tiling ------------------------------------
// validate_coo (the reference's contract, tile_format.hpp:66-69): every
// entry inside rows x cols, strictly increasing (row, col) -- sorted and
// duplicate-free -- else InvariantError.
inline void validate_coo(const ElementCoo& m) {
  const ElementCoo::Entry* prev = nullptr;
  for (std::size_t i = 0; i < m.entries.size(); ++i) {
    const auto& e = m.entries[i];
    if (e.row >= m.rows || e.col >= m.cols)
      throw InvariantError("ElementCoo entry " + std::to_string(i) + " at (" + std::to_string(e.row) + ", " +
                           std::to_string(e.col) + ") is outside " + std::to_string(m.rows) + "x" +
                           std::to_string(m.cols));
    if (prev && !(prev->row < e.row || (prev->row == e.row && prev->col < e.col)))
      throw InvariantError("ElementCoo entry " + std::to_string(i) + " breaks the strictly increasing (row, col) order");
    prev = &e;
  }
}

namespace detail {
// RNE to binary16 as an exact double; OverflowError beyond 65504 (half.cpp:12-36).
inline double round_to_half(double x) {
  if (!std::isfinite(x) || std::fabs(x) > 65504.0) throw OverflowError("value outside binary16 range");
  if (x == 0.0) return x;
  int e2 = 0;
  std::frexp(std::fabs(x), &e2);
  const double q = std::ldexp(1.0, std::max(e2 - 1, -14) - 10);  // spacing of binary16 at |x|
  return std::nearbyint(x / q) * q;  // default rounding mode: ties to even
}

// Kept entries of an 8-row group, in row-major order, grouped into 8x8 tiles
// by tile column without a global sort: the group's distinct tile columns
// (sorted, unique) index a counting scatter; row-major arrival order is the
// tiles' bit order.  Appends to t.
struct Kept {
  std::uint32_t tc;
  std::uint32_t bit;
  float v;
};
inline void emit_group(std::uint32_t tr, std::vector<Kept>& g, std::vector<std::uint32_t>& cols, TiledMatrix& t) {
  if (g.empty()) return;
  cols.clear();
  for (const auto& k : g) cols.push_back(k.tc);
  std::sort(cols.begin(), cols.end());
  cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
  const std::size_t t0 = t.tiles.size();
  std::vector<std::uint64_t> start(cols.size() + 1, 0);
  for (const auto& k : g) ++start[std::lower_bound(cols.begin(), cols.end(), k.tc) - cols.begin() + 1];
  for (std::size_t j = 1; j < start.size(); ++j) start[j] += start[j - 1];
  const std::uint64_t e0 = t.elements.size();
  t.elements.resize(e0 + g.size());
  for (std::size_t j = 0; j < cols.size(); ++j) t.tiles.push_back(TileEntry{tr, cols[j], e0 + start[j], 0});
  for (const auto& k : g) {
    const std::size_t j = std::lower_bound(cols.begin(), cols.end(), k.tc) - cols.begin();
    t.tiles[t0 + j].bitmap |= 1ull << k.bit;
    t.elements[e0 + start[j]++] = k.v;
  }
  g.clear();
}
}  // namespace detail

// from_element_coo (tile_format.hpp:71-72): validate, drop zeros, non-finite
// values raise OverflowError unless drop_nonfinite, Fp16Stored rounds to
// binary16 (OverflowError beyond 65504), values that round to zero drop.
inline TiledMatrix from_element_coo(const ElementCoo& m, ElementKind kind, bool drop_nonfinite = false) {
  validate_coo(m);
  TiledMatrix t;
  t.rows = m.rows;
  t.cols = m.cols;
  t.kind = kind;
  t.elements.reserve(m.entries.size());
  std::vector<detail::Kept> group;
  std::vector<std::uint32_t> cols;
  std::uint64_t cur = ~0ull;
  for (const auto& e : m.entries) {
    if (!std::isfinite(e.value)) {
      if (drop_nonfinite) continue;
      throw OverflowError("non-finite value at (" + std::to_string(e.row) + ", " + std::to_string(e.col) + ")");
    }
    if (e.value == 0.0) continue;
    const float v = kind == ElementKind::Fp16Stored ? float(detail::round_to_half(e.value)) : float(e.value);
    if (!std::isfinite(v)) throw OverflowError("value overflows fp32 at (" + std::to_string(e.row) + ")");
    if (v == 0.0f) continue;
    const std::uint64_t tr = e.row / kTileDim;
    if (tr != cur) {
      detail::emit_group(std::uint32_t(cur), group, cols, t);
      cur = tr;
    }
    group.push_back({std::uint32_t(e.col / kTileDim), std::uint32_t((e.row % kTileDim) * kTileDim + e.col % kTileDim), v});
  }
  detail::emit_group(std::uint32_t(cur), group, cols, t);
  return t;
}

// to_element_coo (tile_format.hpp:75): tiles are ordered by (row, col), so a
// tile row's 8 element rows are produced by walking its tiles once per row
// (ascending columns) -- (row, col) order without a sort.
inline ElementCoo to_element_coo(const TiledMatrix& m) {
  ElementCoo out;
  out.rows = m.rows;
  out.cols = m.cols;
  out.entries.reserve(m.elements.size());
  for (std::size_t a = 0; a < m.tiles.size();) {
    std::size_t b = a;
    while (b < m.tiles.size() && m.tiles[b].tile_row == m.tiles[a].tile_row) ++b;
    for (int r = 0; r < kTileDim; ++r)
      for (std::size_t i = a; i < b; ++i) {
        const TileEntry& t = m.tiles[i];
        std::uint64_t row_bits = (t.bitmap >> (kTileDim * r)) & 0xffull;
        // elements of rows above r precede this row's in the tile's run
        std::uint64_t idx = t.elem_index + std::uint64_t(std::popcount(t.bitmap & ((1ull << (kTileDim * r)) - 1)));
        for (; row_bits; row_bits &= row_bits - 1)
          out.entries.push_back({std::uint64_t(t.tile_row) * kTileDim + r,
                                 std::uint64_t(t.tile_col) * kTileDim + std::countr_zero(row_bits),
                                 double(m.elements[idx++])});
      }
    a = b;
  }
  return out;
}

// ---- the GPU path ------------------------------------------------------------
class Context {
 public:
  explicit Context(int device = -1) { throw_status(tsg_create(&ctx_, device, nullptr), "tsg_create failed"); }
  // several GPUs: A is split into work-balanced tile-row panels, one per device
  explicit Context(const std::vector<int>& devices) {
    throw_status(tsg_create_multi(&ctx_, int(devices.size()), devices.data()), "tsg_create_multi failed");
    n_ = unsigned(devices.size());
  }
  ~Context() { tsg_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  tsg_ctx* get() const { return ctx_; }
  unsigned devices() const { return n_; }

 private:
  tsg_ctx* ctx_ = nullptr;
  unsigned n_ = 1;
};

inline Context& default_context() {
  thread_local Context c;  // one context per host thread (tsparse_b200.h)
  return c;
}

namespace detail {
// CSR view over host arrays (values as f64, or f32 for TiledMatrix elements)
struct HostCsr {
  std::int64_t rows = 0, cols = 0;
  std::vector<std::int64_t> rp;
  std::vector<std::int32_t> col;
  std::vector<double> val;
  std::vector<float> fval;
  tsg_csr view() const {
    tsg_csr v{};
    v.rows = rows;
    v.cols = cols;
    v.nnz = std::int64_t(col.size());
    v.row_ptr = rp.data();
    v.col = col.data();
    if (!fval.empty() || val.empty()) {
      v.val = fval.data();
      v.dtype = TSG_F32;
    } else {
      v.val = val.data();
      v.dtype = TSG_F64;
    }
    v.mem = TSG_MEM_HOST;
    return v;
  }
};

inline HostCsr to_csr(const ElementCoo& m) {
  validate_coo(m);  // sorted, duplicate-free, in range: entry order is CSR order
  HostCsr c;
  c.rows = std::int64_t(m.rows);
  c.cols = std::int64_t(m.cols);
  c.rp.assign(m.rows + 1, 0);
  c.col.reserve(m.entries.size());
  c.val.reserve(m.entries.size());
  for (const auto& e : m.entries) {
    c.rp[e.row + 1]++;
    c.col.push_back(std::int32_t(e.col));
    c.val.push_back(e.value);
  }
  for (std::size_t r = 1; r < c.rp.size(); ++r) c.rp[r] += c.rp[r - 1];
  return c;
}

// 8x8 TiledMatrix -> CSR (f32 values) directly: per tile row, each element
// row walks the row's tiles in column order
inline HostCsr tiled_to_csr(const TiledMatrix& m) {
  HostCsr c;
  c.rows = std::int64_t(m.rows);
  c.cols = std::int64_t(m.cols);
  c.rp.assign(m.rows + 1, 0);
  c.col.resize(m.elements.size());
  c.fval.resize(m.elements.size());
  for (const auto& t : m.tiles)
    for (int r = 0; r < kTileDim; ++r)
      c.rp[std::uint64_t(t.tile_row) * kTileDim + r + 1] += std::popcount((t.bitmap >> (kTileDim * r)) & 0xffull);
  for (std::size_t r = 1; r < c.rp.size(); ++r) c.rp[r] += c.rp[r - 1];
  std::vector<std::int64_t> w(c.rp.begin(), c.rp.end() - 1);
  for (const auto& t : m.tiles) {  // tiles in (row, col) order: each row fills left to right
    std::uint64_t bm = t.bitmap, idx = t.elem_index;
    for (; bm; bm &= bm - 1, ++idx) {
      const int b = std::countr_zero(bm);
      const std::uint64_t row = std::uint64_t(t.tile_row) * kTileDim + b / kTileDim;
      const std::int64_t p = w[row]++;
      c.col[p] = std::int32_t(std::uint64_t(t.tile_col) * kTileDim + b % kTileDim);
      c.fval[p] = m.elements[idx];
    }
  }
  return c;
}

// output CSR (fp32) -> 8x8 Fp32Stored tiles (bit-preserving; cancelled zeros
// never reach the CSR), per 8-row group with detail::emit_group
inline TiledMatrix csr_to_tiled(const tsg_csr_out& o) {
  TiledMatrix t;
  t.rows = std::uint64_t(o.rows);
  t.cols = std::uint64_t(o.cols);
  t.kind = ElementKind::Fp32Stored;
  t.elements.reserve(std::size_t(o.nnz));
  std::vector<Kept> group;
  std::vector<std::uint32_t> cols;
  for (std::int64_t r0 = 0; r0 < o.rows; r0 += kTileDim) {
    const std::int64_t r1 = std::min<std::int64_t>(o.rows, r0 + kTileDim);
    for (std::int64_t r = r0; r < r1; ++r)
      for (std::int64_t p = o.row_ptr[r]; p < o.row_ptr[r + 1]; ++p)
        group.push_back({std::uint32_t(o.col[p] / kTileDim), std::uint32_t((r - r0) * kTileDim + o.col[p] % kTileDim),
                         o.val[p]});
    emit_group(std::uint32_t(r0 / kTileDim), group, cols, t);
  }
  return t;
}

inline ElementCoo from_out(const tsg_csr_out& o) {
  ElementCoo m;
  m.rows = std::uint64_t(o.rows);
  m.cols = std::uint64_t(o.cols);
  m.entries.reserve(std::size_t(o.nnz));
  for (std::int64_t r = 0; r < o.rows; ++r)
    for (std::int64_t p = o.row_ptr[r]; p < o.row_ptr[r + 1]; ++p)
      m.entries.push_back({std::uint64_t(r), std::uint64_t(o.col[p]), double(o.val[p])});
  return m;
}

inline tsg_options options(bool ordered) {
  tsg_options opt;
  tsg_default_options(&opt);
  opt.mode = ordered ? TSG_MODE_ORDERED : TSG_MODE_TENSOR;
  return opt;
}

// RAII output CSR
struct Out {
  tsg_ctx* ctx;
  tsg_csr_out o{};
  explicit Out(tsg_ctx* c) : ctx(c) { o.mem = TSG_MEM_HOST; }
  ~Out() { tsg_free_csr(ctx, &o); }
};
}  // namespace detail

// C = A.B on the GPU (the pass composition of proj/tests/test_kernels.cpp:197-202).
inline ElementCoo spgemm(const ElementCoo& A, const ElementCoo& B, bool ordered = false,
                         tsg_run_stats* stats = nullptr, Context& ctx = default_context()) {
  const auto a = detail::to_csr(A), b = detail::to_csr(B);
  const tsg_csr va = a.view(), vb = b.view();
  const tsg_options opt = detail::options(ordered);
  detail::Out out(ctx.get());
  throw_status(tsg_spgemm(ctx.get(), &va, &vb, &out.o, &opt, stats, nullptr), tsg_last_error(ctx.get()));
  return detail::from_out(out.o);
}

// X0.X1...Xn-1 left to right with the binary16 downcast between stages
// (proj/src/kernels.cpp:239-258).
inline ElementCoo spgemm_chain(const std::vector<ElementCoo>& X, bool ordered = false,
                               tsg_run_stats* stats = nullptr, Context& ctx = default_context()) {
  std::vector<detail::HostCsr> hs;
  for (const auto& m : X) hs.push_back(detail::to_csr(m));
  std::vector<tsg_csr> views;
  for (const auto& h : hs) views.push_back(h.view());
  std::vector<const tsg_csr*> ptrs;
  for (const auto& v : views) ptrs.push_back(&v);
  const tsg_options opt = detail::options(ordered);
  detail::Out out(ctx.get());
  throw_status(tsg_spgemm_chain(ctx.get(), int(ptrs.size()), ptrs.data(), &out.o, &opt, stats),
               tsg_last_error(ctx.get()));
  return detail::from_out(out.o);
}

inline unsigned resolve_gpus(unsigned requested) {
  if (requested) return requested;
  if (const char* e = std::getenv("TILEMUL_GPUS")) {
    const long v = std::strtol(e, nullptr, 10);
    if (v > 0) return unsigned(v);
  }
  return 1;
}

// spgemm_square (kernels.hpp:88-89): same contract -- DimensionError for a
// non-square input, output Fp32Stored 8x8 tiles, the SquareResult counters.
// Counters come from the GPU's 16x16 pipeline; counted_elements (symbolic
// nnz(C)) is tile-size invariant and equals the reference's.  The 8x8 tiles
// are re-tiled on the GPU both ways (tsg_tiles8_to_csr into the pipeline's
// CSR, tsg_csr_to_tiles8 out of it); only the tile arrays cross PCIe.
inline SquareResult spgemm_square(const TiledMatrix& A, const SquareOptions& o = {}) {
  if (A.rows != A.cols)
    throw DimensionError("matrix squaring needs a square input, got " + std::to_string(A.rows) + "x" +
                         std::to_string(A.cols));
  const unsigned gpus = resolve_gpus(o.threads);
  std::vector<int> devs(gpus);
  for (unsigned i = 0; i < gpus; ++i) devs[i] = int(i);
  std::unique_ptr<Context> multi;
  if (gpus > 1) multi = std::make_unique<Context>(devs);
  Context& ctx = multi ? *multi : default_context();
  // the 8x8 tiles as a struct of arrays, to a device CSR on the GPU
  std::vector<std::uint32_t> tr(A.tiles.size()), tc(A.tiles.size());
  std::vector<std::uint64_t> bm(A.tiles.size()), ei(A.tiles.size());
  for (std::size_t i = 0; i < A.tiles.size(); ++i) {
    tr[i] = A.tiles[i].tile_row;
    tc[i] = A.tiles[i].tile_col;
    bm[i] = A.tiles[i].bitmap;
    ei[i] = A.tiles[i].elem_index;
  }
  tsg_tiles8 t8{};
  t8.rows = std::int64_t(A.rows);
  t8.cols = std::int64_t(A.cols);
  t8.ntiles = std::int64_t(A.tiles.size());
  t8.nnz = std::int64_t(A.elements.size());
  t8.tile_row = tr.data();
  t8.tile_col = tc.data();
  t8.bitmap = bm.data();
  t8.elem_index = ei.data();
  t8.val = A.elements.data();
  t8.mem = TSG_MEM_HOST;
  detail::Out ain(ctx.get());
  ain.o.mem = TSG_MEM_DEVICE;
  throw_status(tsg_tiles8_to_csr(ctx.get(), &t8, &ain.o), tsg_last_error(ctx.get()));
  tsg_csr va{};
  va.rows = ain.o.rows;
  va.cols = ain.o.cols;
  va.nnz = ain.o.nnz;
  va.row_ptr = ain.o.row_ptr;
  va.col = ain.o.col;
  va.val = ain.o.val;
  va.dtype = TSG_F32;
  va.mem = TSG_MEM_DEVICE;
  tsg_options opt = detail::options(o.ordered);
  opt.phase_timing = 1;  // SquareResult::timing is always filled (kernels.cpp:260-280)
  tsg_run_stats st{};
  detail::Out out(ctx.get());
  out.o.mem = TSG_MEM_DEVICE;
  throw_status(tsg_spgemm(ctx.get(), &va, &va, &out.o, &opt, &st, nullptr), tsg_last_error(ctx.get()));
  // the product back to 8x8 tiles on the GPU
  tsg_csr vc{};
  vc.rows = out.o.rows;
  vc.cols = out.o.cols;
  vc.nnz = out.o.nnz;
  vc.row_ptr = out.o.row_ptr;
  vc.col = out.o.col;
  vc.val = out.o.val;
  vc.dtype = TSG_F32;
  vc.mem = TSG_MEM_DEVICE;
  tsg_tiles8_out t8o{};
  throw_status(tsg_csr_to_tiles8(ctx.get(), &vc, &t8o), tsg_last_error(ctx.get()));
  SquareResult r;
  r.output.rows = A.rows;
  r.output.cols = A.cols;
  r.output.kind = ElementKind::Fp32Stored;
  r.output.tiles.resize(std::size_t(t8o.ntiles));
  for (std::size_t i = 0; i < r.output.tiles.size(); ++i)
    r.output.tiles[i] = TileEntry{t8o.tile_row[i], t8o.tile_col[i], t8o.elem_index[i], t8o.bitmap[i]};
  r.output.elements.assign(t8o.val, t8o.val + t8o.nnz);
  tsg_free_tiles8(&t8o);
  r.timing = {st.task_list, st.sort, st.counting, st.multiply, st.compaction, st.total};
  r.memory = {st.mem_input_tiles, st.mem_input_elements, st.mem_task_list, st.mem_counting,
              st.mem_pre_compaction, st.mem_output, st.mem_peak};
  r.raw_pairs = st.raw_pairs;
  r.filtered_pairs = st.filtered_pairs;
  r.output_tiles_allocated = st.segments;
  r.counted_elements = st.counted_elements;
  r.threads_used = unsigned(std::max(1, st.devices));
  return r;
}

}  // namespace tilemul_gpu
