// tests/cpp/ref_call_sites.cpp -- source compatibility of the C++ drop-in:
// the reference's own call patterns, written against `namespace tilemul`
// exactly as its CLI and tests use it, compiled with tilemul_gpu.hpp behind a
// namespace alias.  Patterns followed (not copied):
//   proj/tools/tilemul.cpp:84-118    cmd_square: SquareOptions{pairing,
//                                    threads}, spgemm_square, res.output /
//                                    timing.total / threads_used / memory,
//                                    write_tiled_binary, to_element_coo
//   proj/tools/tilemul.cpp:164-200   cmd_bench: warm-up call, per-iteration
//                                    PhaseTiming vector, MemoryReport copy,
//                                    fnv1a(serialize_tiled(output)),
//                                    lower median through PhaseTiming::*
//   proj/tests/test_kernels.cpp:267-300  the squared result equals
//                                    from_element_coo(oracle, Fp32Stored):
//                                    tiles equal, elements bit-equal,
//                                    validate_tiled passes, no zero stored
// Prints one PASS/FAIL line per case; exit status = failures.  Run on the
// GPU by tests/test_gpu_shim.py.
#include <algorithm>
#include <bit>
#include <cstdio>
#include <filesystem>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "tilemul_gpu.hpp"
#include "tilemul_gpu_io.hpp"

namespace tilemul = tilemul_gpu;

namespace {

int failures = 0;
void report(bool ok, const char* what, const std::string& detail) {
  std::printf("%s %s -- %s\n", ok ? "PASS" : "FAIL", what, detail.c_str());
  if (!ok) ++failures;
}

// a SignedHalves-like random matrix (binary16 values in [-4, 4])
tilemul::ElementCoo random_coo(std::mt19937_64& rng, std::uint64_t n, double density) {
  std::uniform_real_distribution<double> u(-4.0, 4.0);
  std::uniform_int_distribution<std::uint64_t> pick(0, n - 1);
  std::map<std::pair<std::uint64_t, std::uint64_t>, double> m;
  while (m.size() < std::uint64_t(density * double(n * n))) {
    double v = 0.0;
    while (v == 0.0) v = tilemul::detail::round_to_half(u(rng));
    m[{pick(rng), pick(rng)}] = v;
  }
  tilemul::ElementCoo c;
  c.rows = c.cols = n;
  for (const auto& [k, v] : m) c.entries.push_back({k.first, k.second, v});
  return c;
}

// the reference's mixed-precision ordered product (oracle.cpp:102-121
// semantics): binary16 inputs, exact fp32 products, fp32 adds in ascending k
tilemul::ElementCoo mixed_oracle(const tilemul::ElementCoo& A, const tilemul::ElementCoo& B) {
  std::vector<std::vector<std::pair<std::uint64_t, float>>> brow(B.rows);
  for (const auto& e : B.entries) brow[e.row].push_back({e.col, float(e.value)});
  std::map<std::uint64_t, std::map<std::uint64_t, float>> acc;
  for (const auto& e : A.entries)
    for (const auto& [j, b] : brow[e.col]) {
      volatile float p = float(e.value) * b;
      volatile float s = acc[e.row][j] + p;
      acc[e.row][j] = s;
    }
  tilemul::ElementCoo C;
  C.rows = A.rows;
  C.cols = B.cols;
  for (const auto& [i, row] : acc)
    for (const auto& [j, v] : row)
      if (v != 0.0f) C.entries.push_back({i, j, double(v)});
  return C;
}

double lower_median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[(v.size() - 1) / 2];
}

}  // namespace

int main() {
  using namespace tilemul;
  std::mt19937_64 rng(101);
  const auto dir = std::filesystem::temp_directory_path();

  // cmd_square's calls
  {
    const TiledMatrix A = from_element_coo(random_coo(rng, 300, 0.02), ElementKind::Fp16Stored);
    SquareOptions opts;
    opts.pairing = true;
    opts.threads = 0;
    const SquareResult res = spgemm_square(A, opts);
    const auto path = dir / "ref_call_sites_c.tspz";
    write_tiled_binary(res.output, path);
    const TiledMatrix back = read_tiled_binary(path);
    const ElementCoo coo_c = to_element_coo(res.output);
    const MemoryReport mem = res.memory;
    report(back == res.output && coo_c.entries.size() == res.output.elements.size() && res.timing.total > 0.0 &&
               res.threads_used >= 1u && mem.peak_bytes > 0,
           "cmd_square call pattern", std::to_string(res.output.elements.size()) + " elements, " +
                                          std::to_string(res.output.tiles.size()) + " tiles");
    std::filesystem::remove(path);
  }

  // cmd_bench's calls
  {
    const TiledMatrix A = from_element_coo(random_coo(rng, 256, 0.03), ElementKind::Fp16Stored);
    SquareOptions opts;
    opts.threads = 1;
    spgemm_square(A, opts);  // warm-up
    std::vector<PhaseTiming> timings;
    MemoryReport memory;
    std::uint64_t hash = 0, first = 0;
    unsigned used = 0;
    bool same = true;
    for (unsigned i = 0; i < 3; ++i) {
      const SquareResult res = spgemm_square(A, opts);
      timings.push_back(res.timing);
      memory = res.memory;
      hash = fnv1a(serialize_tiled(res.output));
      if (i == 0) first = hash;
      same &= hash == first;
      used = res.threads_used;
    }
    const auto pick = [&](double PhaseTiming::*field) {
      std::vector<double> v;
      for (const auto& t : timings) v.push_back(t.*field);
      return lower_median(std::move(v));
    };
    const double total = pick(&PhaseTiming::total);
    report(same && total > 0.0 && used == 1u && memory.output_bytes > 0, "cmd_bench call pattern (deterministic hash)",
           "fnv1a " + std::to_string(hash));
  }

  // test_kernels.cpp: the squared result equals the re-tiled mixed oracle
  {
    int ok = 0;
    for (int rep = 0; rep < 5; ++rep) {
      const ElementCoo coo = random_coo(rng, 256, 0.02);
      const TiledMatrix A = from_element_coo(coo, ElementKind::Fp16Stored);
      SquareOptions o;
      o.ordered = true;  // bit-exact numerics (the reference's sequential fp32)
      const TiledMatrix C = spgemm_square(A, o).output;
      validate_tiled(C);
      const TiledMatrix want = from_element_coo(mixed_oracle(coo, coo), ElementKind::Fp32Stored);
      bool eq = C.tiles == want.tiles && C.elements.size() == want.elements.size();
      for (std::size_t i = 0; eq && i < C.elements.size(); ++i)
        eq = C.elements[i] != 0.0f &&
             std::bit_cast<std::uint32_t>(C.elements[i]) == std::bit_cast<std::uint32_t>(want.elements[i]);
      ok += eq;
    }
    report(ok == 5, "square == from_element_coo(oracle, Fp32Stored)", std::to_string(ok) + "/5 bit-equal");
  }
  return failures;
}
