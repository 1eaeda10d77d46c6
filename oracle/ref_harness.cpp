// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY (never shipped, never
// on the product path).
//
// A thin extern "C" wrapper around the *unmodified* tilemul reference
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libref_tilemul.so).  It lets the Python tests and bench.py's
// CPU-baseline / `--impl reference` arm drive the reference's own entry
// points on CSR inputs:
//
//   * spgemm_square                       proj/src/kernels.cpp:222-302
//   * the A.B pass composition            proj/tests/test_kernels.cpp:197-202
//     (enumerate_pairs -> filter_zero_products -> sort_and_segment ->
//      counting_pass -> multiply_pass -> compact)
//   * the fp32 -> binary16 re-tiling of   proj/src/kernels.cpp:239-258
//     an intermediate (chains R.A.P)
//   * dense_spgemm_mixed_ordered / fp64   proj/src/oracle.cpp:95-121
//   * smape                               proj/src/oracle.cpp:123-150
//   * serialize_tiled + FNV-1a            proj/src/tiled_io.cpp:154-158,
//                                         proj/tests/support/corpus.hpp:177-184
//   * make_random_coo (golden fixtures)   proj/tests/support/corpus.hpp:71-91
//
// Status codes follow the CLI's exit codes (proj/tools/tilemul.cpp:285-306):
// 0 ok, 2 parse/format/invariant, 3 overflow, 4 dimension, 5 precision,
// 1 anything else.
#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "support/corpus.hpp"
#include "tilemul/errors.hpp"
#include "tilemul/half.hpp"
#include "tilemul/kernels.hpp"
#include "tilemul/oracle.hpp"
#include "tilemul/pipeline.hpp"
#include "tilemul/tile_format.hpp"
#include "tilemul/threading.hpp"
#include "tilemul/tiled_io.hpp"

using namespace tilemul;

namespace {

struct RefCsr {
  std::int64_t rows = 0, cols = 0;
  std::vector<std::int64_t> rp;
  std::vector<std::int32_t> col;
  std::vector<double> val;
};

struct RefResult {
  RefCsr C;
  std::vector<std::uint32_t> trow, tcol;
  std::vector<std::uint64_t> bitmap, elem_index;
  double t[6] = {0, 0, 0, 0, 0, 0};  // taskList, sort, counting, multiply, compaction, total
  std::uint64_t u[6] = {0, 0, 0, 0, 0, 0};  // raw, filtered, segments, counted, realized, threads
  std::uint64_t fnv = 0;
};

thread_local std::string g_err;

int status_of(const std::exception& e) {
  if (dynamic_cast<const OverflowError*>(&e)) return 3;
  if (dynamic_cast<const DimensionError*>(&e)) return 4;
  if (dynamic_cast<const PrecisionError*>(&e)) return 5;
  if (dynamic_cast<const ParseError*>(&e) || dynamic_cast<const FormatError*>(&e) ||
      dynamic_cast<const InvariantError*>(&e))
    return 2;
  return 1;
}

ElementCoo coo_from_csr(std::int64_t rows, std::int64_t cols, const std::int64_t* rp,
                        const std::int32_t* col, const double* val) {
  ElementCoo m;
  m.rows = static_cast<std::uint64_t>(rows);
  m.cols = static_cast<std::uint64_t>(cols);
  m.entries.reserve(rows > 0 ? static_cast<std::size_t>(rp[rows]) : 0);
  for (std::int64_t r = 0; r < rows; ++r)
    for (std::int64_t p = rp[r]; p < rp[r + 1]; ++p)
      m.entries.push_back({static_cast<std::uint64_t>(r), static_cast<std::uint64_t>(col[p]), val[p]});
  return m;
}

RefCsr csr_from_coo(const ElementCoo& m) {
  RefCsr c;
  c.rows = static_cast<std::int64_t>(m.rows);
  c.cols = static_cast<std::int64_t>(m.cols);
  c.rp.assign(m.rows + 1, 0);
  c.col.reserve(m.entries.size());
  c.val.reserve(m.entries.size());
  for (const auto& e : m.entries) {
    c.rp[e.row + 1]++;
    c.col.push_back(static_cast<std::int32_t>(e.col));
    c.val.push_back(e.value);
  }
  for (std::size_t r = 1; r < c.rp.size(); ++r) c.rp[r] += c.rp[r - 1];
  return c;
}

void fill_result_from_tiled(RefResult& r, const TiledMatrix& T) {
  r.C = csr_from_coo(to_element_coo(T));
  r.trow.reserve(T.tiles.size());
  for (const auto& t : T.tiles) {
    r.trow.push_back(t.tile_row);
    r.tcol.push_back(t.tile_col);
    r.bitmap.push_back(t.bitmap);
    r.elem_index.push_back(t.elem_index);
  }
  r.fnv = testsupport::fnv1a(serialize_tiled(T));
}

using clk = std::chrono::steady_clock;
double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

// The pass composition of proj/tests/test_kernels.cpp:197-202 with the phase
// stamps of proj/src/kernels.cpp:260-287.
TiledMatrix compose(const TiledMatrix& A, const TiledMatrix& B, unsigned threads, bool pairing,
                    RefResult& r, double* t) {
  const auto t0 = clk::now();
  auto raw = enumerate_pairs(A, B);
  r.u[0] += raw.size();
  auto filtered = filter_zero_products(std::move(raw), A, B);
  r.u[1] += filtered.size();
  const auto t1 = clk::now();
  const TaskList tl = sort_and_segment(std::move(filtered), A, B);
  r.u[2] += tl.num_segments();
  const auto t2 = clk::now();
  const CountResult cr = counting_pass(A, B, tl, threads);
  r.u[3] += cr.total_elements;
  const auto t3 = clk::now();
  const MulResult mr = multiply_pass(A, B, tl, cr, {pairing, threads});
  const auto t4 = clk::now();
  TiledMatrix C = compact(mr);
  const auto t5 = clk::now();
  t[0] += secs(t0, t1);
  t[1] += secs(t1, t2);
  t[2] += secs(t2, t3);
  t[3] += secs(t3, t4);
  t[4] += secs(t4, t5);
  return C;
}

// fp32-stored -> binary16, rebuilt when rounding underflows an element:
// the semantics of proj/src/kernels.cpp:239-258.
TiledMatrix downcast(const TiledMatrix& X) {
  TiledMatrix c = X;
  c.kind = ElementKind::Fp16Stored;
  bool any_zero = false;
  for (float& v : c.elements) {
    v = static_cast<float>(round_to_half(static_cast<double>(v)));
    any_zero |= v == 0.0f;
  }
  if (any_zero) c = from_element_coo(to_element_coo(c), ElementKind::Fp16Stored);
  return c;
}

std::vector<ElementCoo>& main_corpus() {
  // proj/tests/acceptance.cpp:45-58 (seed 42, 200 matrices).
  static std::vector<ElementCoo> corpus;
  if (corpus.empty()) {
    std::mt19937_64 rng(42);
    std::uniform_int_distribution<std::uint64_t> dim_dist(8, 512);
    std::uniform_real_distribution<double> logden(std::log(0.0005), std::log(0.10));
    for (int i = 0; i < 200; ++i) {
      const std::uint64_t dims = dim_dist(rng);
      const double density = std::exp(logden(rng));
      corpus.push_back(testsupport::make_random_coo(rng, dims, dims, density,
                                                    testsupport::ValueMode::SignedHalves));
    }
  }
  return corpus;
}

std::vector<ElementCoo>& wild_corpus() {
  // proj/tests/test_kernels.cpp:332-348 (seed 111, 30 matrices, odd dims).
  static std::vector<ElementCoo> corpus;
  if (corpus.empty()) {
    std::mt19937_64 rng(111);
    std::uniform_int_distribution<std::uint64_t> dim_dist(9, 203);
    for (int rep = 0; rep < 30; ++rep) {
      std::uint64_t dims = dim_dist(rng);
      if (dims % 8 == 0) ++dims;
      corpus.push_back(testsupport::make_random_coo(rng, dims, dims, 0.15,
                                                    testsupport::ValueMode::WildHalves));
    }
  }
  return corpus;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// C = A.B through the reference.  square != 0 calls spgemm_square(A) (B is
// ignored), otherwise the pass composition.  Input tiling is untimed
// (SPEC.md:522), as in the reference CLI.
int ref_spgemm(std::int64_t mA, std::int64_t nA, const std::int64_t* rpA, const std::int32_t* colA,
               const double* valA, std::int64_t mB, std::int64_t nB, const std::int64_t* rpB,
               const std::int32_t* colB, const double* valB, int square, int threads, int pairing,
               void** out) {
  try {
    auto* r = new RefResult();
    const TiledMatrix A = from_element_coo(coo_from_csr(mA, nA, rpA, colA, valA), ElementKind::Fp16Stored);
    if (square) {
      const SquareResult sr = spgemm_square(A, {pairing != 0, static_cast<unsigned>(threads)});
      r->t[0] = sr.timing.task_list;
      r->t[1] = sr.timing.sort;
      r->t[2] = sr.timing.counting;
      r->t[3] = sr.timing.multiply;
      r->t[4] = sr.timing.compaction;
      r->t[5] = sr.timing.total;
      r->u[0] = sr.raw_pairs;
      r->u[1] = sr.filtered_pairs;
      r->u[2] = sr.output_tiles_allocated;
      r->u[3] = sr.counted_elements;
      r->u[5] = sr.threads_used;
      fill_result_from_tiled(*r, sr.output);
    } else {
      const TiledMatrix B = from_element_coo(coo_from_csr(mB, nB, rpB, colB, valB), ElementKind::Fp16Stored);
      const unsigned th = resolve_threads(static_cast<unsigned>(threads));
      const auto t0 = clk::now();
      TiledMatrix C = compose(A, B, th, pairing != 0, *r, r->t);
      r->t[5] = secs(t0, clk::now());
      r->u[5] = th;
      fill_result_from_tiled(*r, C);
    }
    r->u[4] = r->C.col.size();
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// (X0 . X1) . X2 ... left to right, each intermediate downcast to binary16
// as proj/src/kernels.cpp:239-258 does; the downcast is timed (total).
int ref_chain(int n, const std::int64_t* ms, const std::int64_t* ns, const std::int64_t* const* rps,
              const std::int32_t* const* cols, const double* const* vals, int threads, int pairing,
              void** out) {
  try {
    auto* r = new RefResult();
    std::vector<TiledMatrix> X;
    for (int i = 0; i < n; ++i)
      X.push_back(from_element_coo(coo_from_csr(ms[i], ns[i], rps[i], cols[i], vals[i]),
                                   ElementKind::Fp16Stored));
    const unsigned th = resolve_threads(static_cast<unsigned>(threads));
    const auto t0 = clk::now();
    TiledMatrix acc = X[0];
    for (int i = 1; i < n; ++i) {
      if (i > 1) acc = downcast(acc);
      acc = compose(acc, X[i], th, pairing != 0, *r, r->t);
    }
    r->t[5] = secs(t0, clk::now());
    r->u[5] = th;
    fill_result_from_tiled(*r, acc);
    r->u[4] = r->C.col.size();
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// Element-level oracles: mode 0 = dense_spgemm_mixed_ordered, 1 = fp64.
// The result's fnv is FNV-1a(serialize_tiled(from_element_coo(C, Fp32Stored)))
// for mode 0 -- the golden-hash recipe of proj/tests/test_cli.cpp:149-169.
int ref_oracle(int mode, std::int64_t mA, std::int64_t nA, const std::int64_t* rpA,
               const std::int32_t* colA, const double* valA, std::int64_t mB, std::int64_t nB,
               const std::int64_t* rpB, const std::int32_t* colB, const double* valB, void** out) {
  try {
    auto* r = new RefResult();
    const ElementCoo A = coo_from_csr(mA, nA, rpA, colA, valA);
    const ElementCoo B = coo_from_csr(mB, nB, rpB, colB, valB);
    const auto t0 = clk::now();
    const ElementCoo C = mode == 0 ? dense_spgemm_mixed_ordered(A, B) : dense_spgemm_fp64(A, B);
    r->t[5] = secs(t0, clk::now());
    r->C = csr_from_coo(C);
    r->u[4] = r->C.col.size();
    if (mode == 0) {
      const TiledMatrix T = from_element_coo(C, ElementKind::Fp32Stored);
      for (const auto& t : T.tiles) {
        r->trow.push_back(t.tile_row);
        r->tcol.push_back(t.tile_col);
        r->bitmap.push_back(t.bitmap);
        r->elem_index.push_back(t.elem_index);
      }
      r->fnv = testsupport::fnv1a(serialize_tiled(T));
    }
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// from_element_coo(Fp16Stored) of a CSR: the reference's 8x8 tiling
// (proj/src/tile_format.cpp:61-129), for the conversion parity bridge.
int ref_tile(std::int64_t m, std::int64_t n, const std::int64_t* rp, const std::int32_t* col,
             const double* val, int kind, void** out) {
  try {
    auto* r = new RefResult();
    const TiledMatrix T = from_element_coo(coo_from_csr(m, n, rp, col, val),
                                           kind == 0 ? ElementKind::Fp16Stored : ElementKind::Fp32Stored);
    fill_result_from_tiled(*r, T);
    r->u[4] = T.elements.size();
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// Generated matrices (values fp64): 0 = make_random_coo(mt19937_64(seed), ...)
// on a fresh generator; the acceptance / wild corpora by index.
int ref_random_coo(std::uint64_t seed, std::uint64_t rows, std::uint64_t cols, double density, int mode,
                   void** out) {
  try {
    auto* r = new RefResult();
    std::mt19937_64 rng(seed);
    r->C = csr_from_coo(testsupport::make_random_coo(rng, rows, cols, density,
                                                     static_cast<testsupport::ValueMode>(mode)));
    r->u[4] = r->C.col.size();
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

int ref_corpus(int which, int index, void** out) {
  try {
    auto& c = which == 0 ? main_corpus() : wild_corpus();
    if (index < 0 || index >= static_cast<int>(c.size())) return 1;
    auto* r = new RefResult();
    r->C = csr_from_coo(c[index]);
    r->u[4] = r->C.col.size();
    *out = r;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

double ref_round_to_half(double x, int* status) {
  try {
    *status = 0;
    return round_to_half(x);
  } catch (const std::exception& e) {
    *status = status_of(e);
    return 0.0;
  }
}

double ref_smape(std::int64_t m, std::int64_t n, const std::int64_t* rpX, const std::int32_t* colX,
                 const double* valX, const std::int64_t* rpY, const std::int32_t* colY, const double* valY) {
  return smape(coo_from_csr(m, n, rpX, colX, valX), coo_from_csr(m, n, rpY, colY, valY));
}

// Result accessors.
void ref_result_dims(void* h, std::int64_t* out4) {
  auto* r = static_cast<RefResult*>(h);
  out4[0] = r->C.rows;
  out4[1] = r->C.cols;
  out4[2] = static_cast<std::int64_t>(r->C.col.size());
  out4[3] = static_cast<std::int64_t>(r->trow.size());
}
void ref_result_csr(void* h, std::int64_t* rp, std::int32_t* col, double* val) {
  auto* r = static_cast<RefResult*>(h);
  std::memcpy(rp, r->C.rp.data(), r->C.rp.size() * sizeof(std::int64_t));
  std::memcpy(col, r->C.col.data(), r->C.col.size() * sizeof(std::int32_t));
  std::memcpy(val, r->C.val.data(), r->C.val.size() * sizeof(double));
}
void ref_result_tiles(void* h, std::uint32_t* trow, std::uint32_t* tcol, std::uint64_t* bitmap,
                      std::uint64_t* elem_index) {
  auto* r = static_cast<RefResult*>(h);
  const std::size_t n = r->trow.size();
  std::memcpy(trow, r->trow.data(), n * 4);
  std::memcpy(tcol, r->tcol.data(), n * 4);
  std::memcpy(bitmap, r->bitmap.data(), n * 8);
  std::memcpy(elem_index, r->elem_index.data(), n * 8);
}
void ref_result_stats(void* h, double* t6, std::uint64_t* u6, std::uint64_t* fnv) {
  auto* r = static_cast<RefResult*>(h);
  std::memcpy(t6, r->t, sizeof(r->t));
  std::memcpy(u6, r->u, sizeof(r->u));
  *fnv = r->fnv;
}
void ref_result_free(void* h) { delete static_cast<RefResult*>(h); }

}  // extern "C"
