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
//   from_element_coo            tile_format.hpp:71-72  (host, 8x8 -- for callers
//   to_element_coo              tile_format.hpp:75      that hold TiledMatrix)
//   PhaseTiming                 report.hpp:10-17
//   SquareOptions/SquareResult  kernels.hpp:69-89
//   spgemm_square               kernels.hpp:88-89      (runs on the GPU)
//   Error ... PrecisionError    errors.hpp:9-51
// New: spgemm(A, B) and spgemm_chain({R, A, P}).
//
// The 8x8 TiledMatrix stays the interchange type of spgemm_square so callers
// keep working unchanged; internally the GPU uses 16x16 tiles and the result
// is re-tiled with from_element_coo(Fp32Stored), exactly how the reference
// tests build their expected output (proj/tests/test_kernels.cpp:280-283).
#pragma once

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdint>
#include <cstring>
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

struct SquareOptions {
  bool pairing = true;    // accepted for compatibility; 16x16 tiles need no pairing
  unsigned threads = 0;   // accepted for compatibility; the GPU ignores it
  bool ordered = false;   // true: bit-exact CUDA-core numerics (TSG_MODE_ORDERED)
};

struct SquareResult {
  TiledMatrix output;
  PhaseTiming timing;
  std::uint64_t raw_pairs = 0, filtered_pairs = 0, output_tiles_allocated = 0,
                counted_elements = 0;
  unsigned threads_used = 1;
};

// ---- host conversions (8x8, tile_format.cpp:61-154 semantics) -------------
namespace detail {
// RNE to binary16 as an exact double; status 3 beyond 65504 / non-finite
// (half.cpp:12-36).
inline double round_to_half(double x) {
  if (!std::isfinite(x) || std::fabs(x) > 65504.0) throw OverflowError("value outside binary16 range");
  if (x == 0.0) return x;
  int e2 = 0;
  std::frexp(std::fabs(x), &e2);
  const int e = e2 - 1;
  const double q = std::ldexp(1.0, e >= -14 ? e - 10 : -24);
  const double y = x / q, f = std::floor(y), r = y - f;
  double rr = f;
  if (r > 0.5 || (r == 0.5 && std::fmod(f, 2.0) != 0.0)) rr = f + 1.0;
  if (rr == 0.0) return std::copysign(0.0, x);
  return rr * q;
}
}  // namespace detail

inline TiledMatrix from_element_coo(const ElementCoo& m, ElementKind kind) {
  struct Slot {
    std::uint64_t tr, tc;
    std::uint32_t bit;
    float v;
  };
  std::vector<Slot> slots;
  for (const auto& e : m.entries) {
    if (e.row >= m.rows || e.col >= m.cols) throw InvariantError("COO entry out of range");
    if (!std::isfinite(e.value)) throw OverflowError("non-finite value");
    if (e.value == 0.0) continue;
    const float v = kind == ElementKind::Fp16Stored ? float(detail::round_to_half(e.value)) : float(e.value);
    if (v == 0.0f) continue;
    slots.push_back({e.row / 8, e.col / 8, std::uint32_t((e.row % 8) * 8 + e.col % 8), v});
  }
  std::sort(slots.begin(), slots.end(), [](const Slot& a, const Slot& b) {
    return a.tr != b.tr ? a.tr < b.tr : a.tc != b.tc ? a.tc < b.tc : a.bit < b.bit;
  });
  TiledMatrix t;
  t.rows = m.rows;
  t.cols = m.cols;
  t.kind = kind;
  for (std::size_t i = 0; i < slots.size();) {
    TileEntry te{std::uint32_t(slots[i].tr), std::uint32_t(slots[i].tc), t.elements.size(), 0};
    for (; i < slots.size() && slots[i].tr == te.tile_row && slots[i].tc == te.tile_col; ++i) {
      te.bitmap |= 1ULL << slots[i].bit;
      t.elements.push_back(slots[i].v);
    }
    t.tiles.push_back(te);
  }
  return t;
}

inline ElementCoo to_element_coo(const TiledMatrix& m) {
  ElementCoo out;
  out.rows = m.rows;
  out.cols = m.cols;
  for (const auto& t : m.tiles) {
    std::uint64_t bm = t.bitmap, idx = t.elem_index;
    while (bm) {
      const int b = std::countr_zero(bm);
      out.entries.push_back({std::uint64_t(t.tile_row) * 8 + b / 8, std::uint64_t(t.tile_col) * 8 + b % 8,
                             double(m.elements[idx++])});
      bm &= bm - 1;
    }
  }
  std::sort(out.entries.begin(), out.entries.end(), [](const auto& a, const auto& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  return out;
}

// ---- the GPU path ------------------------------------------------------------
class Context {
 public:
  explicit Context(int device = -1) {
    throw_status(tsg_create(&ctx_, device, nullptr), "tsg_create failed");
  }
  ~Context() { tsg_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  tsg_ctx* get() const { return ctx_; }

 private:
  tsg_ctx* ctx_ = nullptr;
};

inline Context& default_context() {
  thread_local Context c;  // one context per host thread (tsparse_b200.h)
  return c;
}

namespace detail {
struct HostCsr {
  std::int64_t rows = 0, cols = 0;
  std::vector<std::int64_t> rp;
  std::vector<std::int32_t> col;
  std::vector<double> val;
  tsg_csr view() const {
    tsg_csr v{};
    v.rows = rows;
    v.cols = cols;
    v.nnz = std::int64_t(col.size());
    v.row_ptr = rp.data();
    v.col = col.data();
    v.val = val.data();
    v.dtype = TSG_F64;
    v.mem = TSG_MEM_HOST;
    return v;
  }
};

inline HostCsr to_csr(const ElementCoo& m) {
  HostCsr c;
  c.rows = std::int64_t(m.rows);
  c.cols = std::int64_t(m.cols);
  c.rp.assign(m.rows + 1, 0);
  for (const auto& e : m.entries) {
    if (e.row >= m.rows || e.col >= m.cols) throw InvariantError("COO entry out of range");
    c.rp[e.row + 1]++;
    c.col.push_back(std::int32_t(e.col));
    c.val.push_back(e.value);
  }
  for (std::size_t r = 1; r < c.rp.size(); ++r) c.rp[r] += c.rp[r - 1];
  return c;
}

inline ElementCoo from_out(tsg_csr_out& o) {
  ElementCoo m;
  m.rows = std::uint64_t(o.rows);
  m.cols = std::uint64_t(o.cols);
  m.entries.reserve(std::size_t(o.nnz));
  for (std::int64_t r = 0; r < o.rows; ++r)
    for (std::int64_t p = o.row_ptr[r]; p < o.row_ptr[r + 1]; ++p)
      m.entries.push_back({std::uint64_t(r), std::uint64_t(o.col[p]), double(o.val[p])});
  return m;
}
}  // namespace detail

// C = A.B on the GPU (the pass composition of proj/tests/test_kernels.cpp:197-202).
inline ElementCoo spgemm(const ElementCoo& A, const ElementCoo& B, bool ordered = false,
                         tsg_run_stats* stats = nullptr, Context& ctx = default_context()) {
  const auto a = detail::to_csr(A), b = detail::to_csr(B);
  const tsg_csr va = a.view(), vb = b.view();
  tsg_options opt;
  tsg_default_options(&opt);
  opt.mode = ordered ? TSG_MODE_ORDERED : TSG_MODE_TENSOR;
  tsg_csr_out out{};
  out.mem = TSG_MEM_HOST;
  throw_status(tsg_spgemm(ctx.get(), &va, &vb, &out, &opt, stats, nullptr), tsg_last_error(ctx.get()));
  ElementCoo c = detail::from_out(out);
  tsg_free_csr(ctx.get(), &out);
  return c;
}

// X0.X1...Xn-1 left to right with the binary16 downcast between stages
// (proj/src/kernels.cpp:239-258).
inline ElementCoo spgemm_chain(const std::vector<ElementCoo>& X, bool ordered = false,
                               Context& ctx = default_context()) {
  std::vector<detail::HostCsr> hs;
  for (const auto& m : X) hs.push_back(detail::to_csr(m));
  std::vector<tsg_csr> views;
  for (const auto& h : hs) views.push_back(h.view());
  std::vector<const tsg_csr*> ptrs;
  for (const auto& v : views) ptrs.push_back(&v);
  tsg_options opt;
  tsg_default_options(&opt);
  opt.mode = ordered ? TSG_MODE_ORDERED : TSG_MODE_TENSOR;
  tsg_csr_out out{};
  out.mem = TSG_MEM_HOST;
  throw_status(tsg_spgemm_chain(ctx.get(), int(ptrs.size()), ptrs.data(), &out, &opt, nullptr),
               tsg_last_error(ctx.get()));
  ElementCoo c = detail::from_out(out);
  tsg_free_csr(ctx.get(), &out);
  return c;
}

// spgemm_square (kernels.hpp:88-89): same contract -- DimensionError for a
// non-square input, output Fp32Stored 8x8 tiles, the SquareResult counters.
// Counters come from the GPU's 16x16 pipeline; counted_elements (symbolic
// nnz(C)) is tile-size invariant and equals the reference's.
inline SquareResult spgemm_square(const TiledMatrix& A, const SquareOptions& o = {}) {
  if (A.rows != A.cols)
    throw DimensionError("matrix squaring needs a square input, got " + std::to_string(A.rows) + "x" +
                         std::to_string(A.cols));
  tsg_run_stats st{};
  const ElementCoo a = to_element_coo(A);
  const ElementCoo c = spgemm(a, a, o.ordered, &st);
  SquareResult r;
  r.output = from_element_coo(c, ElementKind::Fp32Stored);
  r.timing = {st.task_list, st.sort, st.counting, st.multiply, st.compaction, st.total};
  r.raw_pairs = st.raw_pairs;
  r.filtered_pairs = st.filtered_pairs;
  r.output_tiles_allocated = st.segments;
  r.counted_elements = st.counted_elements;
  return r;
}

}  // namespace tilemul_gpu
