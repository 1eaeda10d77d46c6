// tests/cpp/shim_acceptance.cpp -- the reference's acceptance-style gates
// (proj/tests/acceptance.cpp) written against the C++ drop-in header
// include/tilemul_gpu.hpp, i.e. as a reference user would after switching.
// Prints one PASS/FAIL line per gate; exit status = number of failures.
// Built by __graft_entry__.build(); run on the GPU by tests/test_gpu_shim.py.
#include <bit>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <map>
#include <string>

#include "tilemul_gpu.hpp"

using namespace tilemul_gpu;

namespace {

std::uint64_t sm_state = 42;
std::uint64_t splitmix() {
  std::uint64_t z = (sm_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
double unif() { return double(splitmix() >> 11) * 0x1.0p-53; }

// SignedHalves-like values (corpus.hpp:61-66): binary16 values in [-4, 4].
ElementCoo random_coo(std::uint64_t n, double density) {
  std::map<std::pair<std::uint64_t, std::uint64_t>, double> m;
  const auto target = std::uint64_t(density * double(n) * double(n));
  while (m.size() < target) {
    const std::uint64_t r = splitmix() % n, c = splitmix() % n;
    double v = 0.0;
    while (v == 0.0) v = detail::round_to_half(-4.0 + 8.0 * unif());
    m.emplace(std::make_pair(r, c), v);
  }
  ElementCoo coo;
  coo.rows = coo.cols = n;
  for (const auto& [k, v] : m) coo.entries.push_back({k.first, k.second, v});
  return coo;
}

// Independent element-level oracle (dense_spgemm_mixed_ordered semantics,
// oracle.cpp:102-121): binary16 inputs, exact fp32 products, one fp32 add
// per product in ascending k.
ElementCoo oracle(const ElementCoo& A, const ElementCoo& B) {
  std::vector<std::vector<std::pair<std::uint64_t, float>>> brow(B.rows);
  for (const auto& e : B.entries) brow[e.row].push_back({e.col, float(detail::round_to_half(e.value))});
  std::map<std::uint64_t, std::map<std::uint64_t, float>> acc;
  for (const auto& e : A.entries) {
    const float a = float(detail::round_to_half(e.value));
    if (a == 0.0f) continue;
    for (const auto& [j, b] : brow[e.col]) {
      volatile float p = a * b;  // exact
      volatile float s = acc[e.row][j] + p;
      acc[e.row][j] = s;
    }
  }
  ElementCoo C;
  C.rows = A.rows;
  C.cols = B.cols;
  for (const auto& [i, row] : acc)
    for (const auto& [j, v] : row)
      if (v != 0.0f) C.entries.push_back({i, j, double(v)});
  return C;
}

bool bit_equal(const ElementCoo& x, const ElementCoo& y) {
  if (x.rows != y.rows || x.cols != y.cols || x.entries.size() != y.entries.size()) return false;
  for (std::size_t i = 0; i < x.entries.size(); ++i) {
    const auto &a = x.entries[i], &b = y.entries[i];
    if (a.row != b.row || a.col != b.col) return false;
    if (std::bit_cast<std::uint32_t>(float(a.value)) != std::bit_cast<std::uint32_t>(float(b.value)))
      return false;
  }
  return true;
}

bool pattern_equal(const ElementCoo& x, const ElementCoo& y) {
  if (x.entries.size() != y.entries.size()) return false;
  for (std::size_t i = 0; i < x.entries.size(); ++i)
    if (x.entries[i].row != y.entries[i].row || x.entries[i].col != y.entries[i].col) return false;
  return true;
}

int failures = 0;
void report(bool ok, const char* gate, const std::string& detail) {
  std::printf("%s %s -- %s\n", ok ? "PASS" : "FAIL", gate, detail.c_str());
  if (!ok) ++failures;
}

}  // namespace

int main() {
  // gate 1: spgemm_square == mixed oracle, bit-exact in ORDERED mode; TENSOR pattern-exact
  {
    int n_ok = 0, n_pat = 0;
    const int N = 60;
    for (int i = 0; i < N; ++i) {
      const std::uint64_t dims = 8 + splitmix() % 300;
      const double dens = 0.0005 * std::exp(unif() * std::log(200.0));
      const ElementCoo coo = random_coo(dims, dens);
      const TiledMatrix A = from_element_coo(coo, ElementKind::Fp16Stored);
      const ElementCoo want = oracle(coo, coo);
      SquareOptions o;
      o.ordered = true;
      n_ok += bit_equal(to_element_coo(spgemm_square(A, o).output), want);
      n_pat += pattern_equal(to_element_coo(spgemm_square(A).output), want);
    }
    report(n_ok == N && n_pat == N, "oracle equivalence (acceptance.cpp:114-135)",
           std::to_string(n_ok) + "/" + std::to_string(N) + " bit-exact ordered, " + std::to_string(n_pat) +
               " pattern-exact tensor");
  }
  // gate 2: counting upper bound with cancellation (acceptance.cpp:62-98)
  {
    ElementCoo m;
    m.rows = m.cols = 16;
    m.entries = {{0, 1, 1.0}, {0, 2, -1.0}, {1, 8, 5.0}, {2, 8, 5.0}};
    const SquareResult r = spgemm_square(from_element_coo(m, ElementKind::Fp16Stored));
    report(r.counted_elements == 1 && r.output.tiles.empty(), "counting bound + compaction",
           "counted " + std::to_string(r.counted_elements) + ", realized " + std::to_string(r.output.nnz()));
  }
  // gate: identity reproduces B (test_kernels.cpp:193-210 via spgemm)
  {
    ElementCoo I;
    I.rows = I.cols = 64;
    for (std::uint64_t k = 0; k < 64; ++k) I.entries.push_back({k, k, 1.0});
    const ElementCoo B = random_coo(64, 0.08);
    report(bit_equal(spgemm(I, B), oracle(I, B)), "identity . B == B", "64x64");
  }
  // gate: error taxonomy (errors.hpp, tilemul.cpp exit codes)
  {
    bool dim = false, ovf = false;
    TiledMatrix rect;
    rect.rows = 8;
    rect.cols = 16;
    try {
      spgemm_square(rect);
    } catch (const DimensionError&) {
      dim = true;
    }
    ElementCoo big;
    big.rows = big.cols = 8;
    big.entries = {{0, 0, 70000.0}};
    try {
      spgemm(big, big);
    } catch (const OverflowError&) {
      ovf = true;
    }
    report(dim && ovf, "DimensionError / OverflowError", "non-square and |x| > 65504");
  }
  // gate: chain with binary16 downcast (kernels.cpp:239-258)
  {
    const ElementCoo R = random_coo(48, 0.05), A = random_coo(48, 0.05), P = random_coo(48, 0.05);
    ElementCoo RA = oracle(R, A);
    const ElementCoo want = oracle(RA, P);  // oracle rounds RA to binary16 on entry
    report(bit_equal(spgemm_chain({R, A, P}, true), want), "R.A.P chain", "48^3 ordered");
  }
  // gate: validate_coo (tile_format.hpp:66-69) -- unsorted, duplicated and
  // out-of-range entries raise InvariantError before anything runs
  {
    int raised = 0;
    ElementCoo bad;
    bad.rows = bad.cols = 8;
    bad.entries = {{1, 0, 1.0}, {0, 5, 1.0}};  // unsorted rows
    try { spgemm(bad, bad); } catch (const InvariantError&) { ++raised; }
    bad.entries = {{0, 3, 1.0}, {0, 3, 2.0}};  // duplicate
    try { (void)from_element_coo(bad, ElementKind::Fp16Stored); } catch (const InvariantError&) { ++raised; }
    bad.entries = {{0, 8, 1.0}};  // out of range
    try { validate_coo(bad); } catch (const InvariantError&) { ++raised; }
    report(raised == 3, "validate_coo -> InvariantError", std::to_string(raised) + "/3 raised");
  }
  // gate: from_element_coo(..., drop_nonfinite) (tile_format.cpp:82-86 contract)
  {
    ElementCoo m;
    m.rows = m.cols = 16;
    m.entries = {{0, 0, 2.0}, {0, 9, INFINITY}, {3, 3, 1e-9}, {9, 1, -0.5}};
    bool raised = false;
    try { (void)from_element_coo(m, ElementKind::Fp16Stored); } catch (const OverflowError&) { raised = true; }
    const TiledMatrix t = from_element_coo(m, ElementKind::Fp16Stored, true);
    const ElementCoo back = to_element_coo(t);
    // inf dropped, 1e-9 underflows binary16 and drops, the rest round-trips
    const bool ok = raised && back.entries.size() == 2 && back.entries[0].col == 0 && back.entries[1].row == 9 &&
                    back.entries[1].value == -0.5 && t.tiles.size() == 2;
    report(ok, "drop_nonfinite + underflow drop + round trip", std::to_string(back.entries.size()) + " entries");
  }
  // gate: to_element_coo(from_element_coo(x)) == x for a binary16 matrix, and
  // SquareResult carries the device memory report and the GPU count
  {
    const ElementCoo coo = random_coo(200, 0.03);
    const TiledMatrix A = from_element_coo(coo, ElementKind::Fp16Stored);
    const bool rt = bit_equal(to_element_coo(A), coo);
    const SquareResult r = spgemm_square(A);
    const bool mem = r.memory.peak_bytes > 0 && r.memory.output_bytes > 0 && r.memory.input_tiles_bytes > 0 &&
                     r.threads_used == 1;
    report(rt && mem, "tiling round trip + MemoryReport",
           "peak " + std::to_string(r.memory.peak_bytes) + " B, threads_used " + std::to_string(r.threads_used));
  }
  // gate: a multi-device context (several panel workers on GPU 0) returns the
  // single-device product bit for bit
  {
    const ElementCoo A = random_coo(300, 0.02), B = random_coo(300, 0.02);
    Context multi(std::vector<int>{0, 0, 0});
    tsg_run_stats st{};
    const ElementCoo one = spgemm(A, B, true);
    const ElementCoo three = spgemm(A, B, true, &st, multi);
    report(bit_equal(one, three) && st.devices == 3, "multi-device panels == one device",
           std::to_string(one.entries.size()) + " entries, devices " + std::to_string(st.devices));
  }
  return failures;
}
