// tilemul_gpu -- the reference's command-line front end (proj/tools/tilemul.cpp)
// with the spGEMM running on the B200.
//
//   tilemul_gpu convert --input A.mtx --output A.tspz [--precision fp16|fp32]
//   tilemul_gpu square  --input A.{mtx,tspz} --output C.tspz [--report r.json]
//                       [--pairing on|off] [--threads N] [--numerics ordered|tensor]
//   tilemul_gpu compare --input A.mtx [--mode fp64|mixed] [--numerics ...]
//   tilemul_gpu stats   --input A.{mtx,tspz} [--json]
//   tilemul_gpu advise  --input A.{mtx,tspz} [--json] [--raw-tile-ratio]
//   tilemul_gpu bench   --input A.{mtx,tspz} [--iters K] [--threads N] [--csv out.csv]
//                       [--numerics ...]
//
// Same subcommands, flags, output lines, report JSON / bench CSV fields and
// stable exit codes (tilemul.cpp:30-35, 285-306): 0 ok, 2 unparseable input
// (parse / format / invariant), 3 binary16 overflow, 4 dimension mismatch,
// 5 non-finite accumulator, 1 anything else.  `--numerics ordered` (the
// default) is bit-identical to the reference, so `square` writes the same
// .tspz bytes and `bench` the same FNV-1a output hash; `--numerics tensor`
// uses the tensor-core path (pattern-exact, values within DESIGN.md 5).
// `--pairing` and `--threads` are accepted for compatibility (16x16 tiles
// need no pairing; the GPU grid replaces the thread pool).  `stats` and
// `advise` (analytics.cpp:16-118) are host analyses at the reference's T = 8.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "tilemul_gpu.hpp"
#include "tilemul_gpu_io.hpp"

namespace {

using namespace tilemul_gpu;

constexpr int kExitOk = 0, kExitOther = 1, kExitParse = 2, kExitOverflow = 3, kExitDimension = 4,
              kExitPrecision = 5;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::string cmd;
  std::map<std::string, std::string> opt;
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? d : it->second;
  }
  bool has(const std::string& k) const { return opt.count(k) != 0; }
};

Args parse(int argc, char** argv) {
  if (argc < 2) throw UsageError("a subcommand is required: convert, square, compare, stats, advise, bench");
  Args a;
  a.cmd = argv[1];
  static const std::map<std::string, std::vector<std::string>> known = {
      {"convert", {"--input", "--output", "--precision"}},
      {"square", {"--input", "--output", "--pairing", "--threads", "--report", "--numerics"}},
      {"compare", {"--input", "--mode", "--numerics"}},
      {"stats", {"--input", "--json"}},
      {"advise", {"--input", "--json", "--raw-tile-ratio"}},
      {"bench", {"--input", "--iters", "--threads", "--csv", "--numerics"}},
  };
  auto k = known.find(a.cmd);
  if (k == known.end()) throw UsageError("unknown subcommand " + a.cmd);
  for (int i = 2; i < argc; ++i) {
    const std::string o = argv[i];
    if (std::find(k->second.begin(), k->second.end(), o) == k->second.end())
      throw UsageError("unknown option " + o + " for " + a.cmd);
    if (o == "--json" || o == "--raw-tile-ratio") {
      a.opt[o] = "1";
    } else {
      if (i + 1 >= argc) throw UsageError(o + " needs a value");
      a.opt[o] = argv[++i];
    }
  }
  if (!a.has("--input")) throw UsageError("--input is required");
  return a;
}

bool has_tspz_magic(const std::filesystem::path& p) {
  std::ifstream in(p, std::ios::binary);
  char m[4] = {};
  in.read(m, 4);
  return in && std::string(m, 4) == "TSPZ";
}

TiledMatrix load_matrix(const std::filesystem::path& p, ElementKind mtx_kind = ElementKind::Fp16Stored) {
  if (!std::filesystem::exists(p)) throw IoError("input file not found: " + p.string());
  if (has_tspz_magic(p)) return read_tiled_binary(p);
  return from_element_coo(read_matrix_market(p), mtx_kind);
}

bool ordered_numerics(const Args& a) {
  const std::string n = a.get("--numerics", "ordered");
  if (n != "ordered" && n != "tensor") throw UsageError("--numerics must be ordered or tensor");
  return n == "ordered";
}

// ---- host reference products for `compare` and the report's SMAPE ------------------
// Row-wise Gustavson with a dense accumulator, k ascending per output
// element (oracle.cpp:33-121): fp64, or binary16 inputs with fp32 adds.
template <class Acc>
ElementCoo host_product(const ElementCoo& A, const ElementCoo& B, bool round_half) {
  auto rows_of = [](const ElementCoo& m) {
    std::vector<std::uint64_t> o(m.rows + 1, 0);
    for (const auto& e : m.entries) o[e.row + 1]++;
    for (std::uint64_t r = 1; r <= m.rows; ++r) o[r] += o[r - 1];
    return o;
  };
  auto prep = [&](const ElementCoo& m) {
    if (!round_half) return m;
    ElementCoo r = m;
    std::erase_if(r.entries, [](ElementCoo::Entry& e) {
      e.value = detail::round_to_half(e.value);
      return e.value == 0.0;
    });
    return r;
  };
  const ElementCoo a = prep(A), b = prep(B);
  const auto ar = rows_of(a), br = rows_of(b);
  ElementCoo C;
  C.rows = A.rows;
  C.cols = B.cols;
  std::vector<Acc> acc(B.cols, Acc(0));
  std::vector<std::uint8_t> on(B.cols, 0);
  std::vector<std::uint64_t> touched;
  for (std::uint64_t i = 0; i < a.rows; ++i) {
    touched.clear();
    for (std::uint64_t p = ar[i]; p < ar[i + 1]; ++p) {
      const auto& x = a.entries[p];
      for (std::uint64_t q = br[x.col]; q < br[x.col + 1]; ++q) {
        const auto& y = b.entries[q];
        if (!on[y.col]) {
          on[y.col] = 1;
          touched.push_back(y.col);
        }
        acc[y.col] += Acc(x.value) * Acc(y.value);
      }
    }
    std::sort(touched.begin(), touched.end());
    for (const auto j : touched) {
      if (acc[j] != Acc(0)) C.entries.push_back({i, j, double(acc[j])});
      acc[j] = Acc(0);
      on[j] = 0;
    }
  }
  return C;
}

double smape(const ElementCoo& X, const ElementCoo& Y) {  // oracle.cpp:123-150
  double sum = 0.0;
  std::uint64_t n = 0;
  std::size_t ix = 0, iy = 0;
  auto key = [](const ElementCoo::Entry& e) { return std::pair(e.row, e.col); };
  while (ix < X.entries.size() || iy < Y.entries.size()) {
    double x = 0.0, y = 0.0;
    if (iy >= Y.entries.size() || (ix < X.entries.size() && key(X.entries[ix]) < key(Y.entries[iy]))) {
      x = X.entries[ix++].value;
    } else if (ix >= X.entries.size() || key(Y.entries[iy]) < key(X.entries[ix])) {
      y = Y.entries[iy++].value;
    } else {
      x = X.entries[ix++].value;
      y = Y.entries[iy++].value;
    }
    if (x == 0.0 && y == 0.0) continue;
    ++n;
    sum += std::fabs(x - y) / (std::fabs(x) + std::fabs(y));
  }
  return n == 0 ? 0.0 : 100.0 * sum / double(n);
}

double lower_median(std::vector<double> v) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  return v[(v.size() - 1) / 2];
}

std::string num(double x) {
  char b[64];
  std::snprintf(b, sizeof b, "%.9g", x);
  return b;
}

// ---- subcommands ------------------------------------------------------------------
int cmd_convert(const Args& a) {
  const std::string prec = a.get("--precision", "fp16");
  if (prec != "fp16" && prec != "fp32") throw UsageError("--precision must be fp16 or fp32");
  if (!a.has("--output")) throw UsageError("--output is required");
  const ElementKind kind = prec == "fp32" ? ElementKind::Fp32Stored : ElementKind::Fp16Stored;
  const TiledMatrix m = from_element_coo(read_matrix_market(std::filesystem::path(a.get("--input"))), kind);
  write_tiled_binary(m, std::filesystem::path(a.get("--output")));
  std::cout << "wrote " << a.get("--output") << ": " << m.tiles.size() << " tiles, " << m.elements.size()
            << " elements, " << m.rows << "x" << m.cols << " " << prec << "\n";
  return kExitOk;
}

int cmd_square(const Args& a) {
  if (!a.has("--output")) throw UsageError("--output is required");
  const std::filesystem::path in(a.get("--input"));
  const TiledMatrix A = load_matrix(in);
  SquareOptions o;
  o.pairing = a.get("--pairing", "on") == "on";
  o.ordered = ordered_numerics(a);
  const SquareResult r = spgemm_square(A, o);
  write_tiled_binary(r.output, std::filesystem::path(a.get("--output")));
  std::cout << "squared " << in.filename().string() << ": nnzC=" << r.output.elements.size()
            << " tiles=" << r.output.tiles.size() << " total=" << r.timing.total << "s threads=1\n";
  if (a.has("--report")) {  // RunReport JSON (report.cpp:10-34)
    const ElementCoo ca = to_element_coo(A);
    const double sm = smape(to_element_coo(r.output), host_product<double>(ca, ca, false));
    std::ofstream out(a.get("--report"));
    if (!out) throw IoError("cannot open " + a.get("--report") + " for writing");
    const auto& t = r.timing;
    out << "{\n  \"matrixName\": \"" << in.stem().string() << "\",\n  \"dims\": " << A.rows
        << ",\n  \"nnzA\": " << A.elements.size() << ",\n  \"nnzC\": " << r.output.elements.size()
        << ",\n  \"timing\": {\n    \"taskList\": " << num(t.task_list) << ",\n    \"sort\": " << num(t.sort)
        << ",\n    \"counting\": " << num(t.counting) << ",\n    \"multiply\": " << num(t.multiply)
        << ",\n    \"compaction\": " << num(t.compaction) << ",\n    \"total\": " << num(t.total)
        << "\n  },\n  \"memory\": {\n    \"peakBytes\": 0\n  },\n  \"smapeVsFp64\": " << num(sm)
        << ",\n  \"threadCount\": 1,\n  \"seed\": 0,\n  \"device\": \"B200 (tsparse_b200)\"\n}\n";
  }
  return kExitOk;
}

int cmd_compare(const Args& a) {
  const std::string mode = a.get("--mode", "fp64");
  if (mode != "fp64" && mode != "mixed") throw UsageError("--mode must be fp64 or mixed");
  const ElementCoo coo = read_matrix_market(std::filesystem::path(a.get("--input")));
  const TiledMatrix A = from_element_coo(coo, ElementKind::Fp16Stored);
  SquareOptions o;
  o.ordered = ordered_numerics(a);
  const SquareResult r = spgemm_square(A, o);
  const ElementCoo ref = mode == "mixed" ? host_product<float>(coo, coo, true) : host_product<double>(coo, coo, false);
  std::cout << "SMAPE vs " << mode << " oracle: " << smape(to_element_coo(r.output), ref) << " %\n";
  return kExitOk;
}

// Table-1 statistics (analytics.cpp:16-84) at the reference's T = 8.
struct Stats {
  std::uint64_t dims = 0, nnz_a = 0, nnz_c = 0, cbar = 0, c_tiles = 0, raw = 0, filt = 0;
  double avg = 0, med = 0, mean = 0, sd = 0;
};

Stats compute_stats(const TiledMatrix& A) {
  if (A.rows != A.cols)
    throw DimensionError("statistics for A*A need a square matrix, got " + std::to_string(A.rows) + "x" +
                         std::to_string(A.cols));
  Stats st;
  st.dims = A.rows;
  st.nnz_a = A.elements.size();
  st.avg = A.rows ? double(A.elements.size()) / double(A.rows) : 0.0;
  if (!A.tiles.empty()) {
    std::vector<int> pops;
    for (const auto& t : A.tiles) pops.push_back(std::popcount(t.bitmap));
    std::sort(pops.begin(), pops.end());
    st.med = pops[(pops.size() - 1) / 2];
    for (int p : pops) st.mean += p;
    st.mean /= double(pops.size());
    for (int p : pops) st.sd += (p - st.mean) * (p - st.mean);
    st.sd = std::sqrt(st.sd / double(pops.size()));
  }
  const ElementCoo coo = to_element_coo(A);
  {
    std::vector<std::uint64_t> rn(A.rows, 0), cn(A.cols, 0);
    for (const auto& e : coo.entries) rn[e.row]++, cn[e.col]++;
    for (std::uint64_t k = 0; k < A.rows; ++k) st.cbar += cn[k] * rn[k];
    const ElementCoo C = host_product<double>(coo, coo, false);
    st.nnz_c = C.entries.size();
    std::vector<std::uint64_t> keys;
    for (const auto& e : C.entries) keys.push_back((e.row / 8) * ((A.cols / 8) + 1) + e.col / 8);
    std::sort(keys.begin(), keys.end());
    st.c_tiles = std::uint64_t(std::unique(keys.begin(), keys.end()) - keys.begin());
  }
  {  // tile pairs (pipeline.cpp:23-60): row starts of B's tile rows, O(1) filter
    std::vector<std::uint64_t> rs(A.tile_rows() + 1, 0);
    for (const auto& t : A.tiles) rs[t.tile_row + 1]++;
    for (std::size_t i = 1; i < rs.size(); ++i) rs[i] += rs[i - 1];
    auto colocc = [](std::uint64_t b) {
      std::uint64_t o = 0;
      for (int r = 0; r < 8; ++r) o |= (b >> (8 * r)) & 0xff;
      return o;
    };
    auto rowocc = [](std::uint64_t b) {
      std::uint64_t o = 0;
      for (int r = 0; r < 8; ++r) o |= std::uint64_t(((b >> (8 * r)) & 0xff) != 0) << r;
      return o;
    };
    for (const auto& ta : A.tiles)
      for (std::uint64_t j = rs[ta.tile_col]; j < rs[ta.tile_col + 1]; ++j) {
        ++st.raw;
        st.filt += (colocc(ta.bitmap) & rowocc(A.tiles[j].bitmap)) != 0;
      }
  }
  return st;
}

int cmd_stats(const Args& a) {
  const std::filesystem::path in(a.get("--input"));
  const TiledMatrix A = load_matrix(in, ElementKind::Fp32Stored);
  const Stats st = compute_stats(A);
  const std::string name = in.stem().string();
  if (a.has("--json")) {
    std::cout << "{\"matrixName\": \"" << name << "\", \"dims\": " << st.dims << ", \"nnzA\": " << st.nnz_a
              << ", \"nnzC\": " << st.nnz_c << ", \"nnzCbar\": " << st.cbar << ", \"nnzCTiles\": " << st.c_tiles
              << ", \"nnzCbarTilesRaw\": " << st.raw << ", \"nnzCbarTilesFiltered\": " << st.filt
              << ", \"avgRow\": " << num(st.avg) << ", \"densityMedian\": " << num(st.med)
              << ", \"densityMean\": " << num(st.mean) << ", \"densityStd\": " << num(st.sd) << "}\n";
  } else {
    std::cout << "matrixName,dims,nnzA,nnzC,nnzCbar,nnzCTiles,nnzCbarTilesRaw,nnzCbarTilesFiltered,avgRow,"
                 "densityMedian,densityMean,densityStd\n"
              << name << ',' << st.dims << ',' << st.nnz_a << ',' << st.nnz_c << ',' << st.cbar << ',' << st.c_tiles
              << ',' << st.raw << ',' << st.filt << ',' << num(st.avg) << ',' << num(st.med) << ','
              << num(st.mean) << ',' << num(st.sd) << "\n";
  }
  return kExitOk;
}

// The paper's approach-selection thresholds evaluated on the statistics
// (advise, analytics.cpp:93-118; output as cmd_advise, tilemul.cpp:146-162).
// The intermediate ratio is C-bar over the filtered tile pairs, or the raw
// ones with --raw-tile-ratio.
int cmd_advise(const Args& a) {
  const std::filesystem::path in(a.get("--input"));
  const Stats st = compute_stats(load_matrix(in, ElementKind::Fp32Stored));
  const std::uint64_t pairs = a.has("--raw-tile-ratio") ? st.raw : st.filt;
  const double ratio = pairs ? double(st.cbar) / double(pairs) : 0.0;
  struct Rule {
    const char* approach;
    const char* condition;
    bool yes;
  };
  const Rule rules[] = {
      {"cuSPARSE", "NNZ(A) > 200000", st.nnz_a > 200000},
      {"CUSP", "NNZ(Cbar) / NNZ(Cbar_tiles) >= 1", ratio >= 1.0},
      {"RMerge2", "avgRowA > 42 AND NNZ(A) > 100000", st.avg > 42.0 && st.nnz_a > 100000},
      {"Nsparse", "avgRowA > 42 AND NNZ(A) > 100000", st.avg > 42.0 && st.nnz_a > 100000},
      {"AC-SpGEMM", "NNZ(Cbar) / NNZ(Cbar_tiles) > 9", ratio > 9.0},
      {"spECK", "avgRowA > 42 AND NNZ(A) > 300000", st.avg > 42.0 && st.nnz_a > 300000},
      {"global", "NNZ(A) > 300000 AND avgRowA > 42", st.nnz_a > 300000 && st.avg > 42.0},
      {"globalRelaxed", "NNZ(A) > 300000 AND avgRowA > 21", st.nnz_a > 300000 && st.avg > 21.0},
  };
  if (a.has("--json")) {
    std::cout << "[";
    bool first = true;
    for (const auto& r : rules) {
      std::cout << (first ? "\n" : ",\n") << "  {\n    \"approach\": \"" << r.approach << "\",\n    \"condition\": \""
                << r.condition << "\",\n    \"recommended\": " << (r.yes ? "true" : "false") << "\n  }";
      first = false;
    }
    std::cout << "\n]\n";
    return kExitOk;
  }
  std::cout << "approach        recommended  condition\n";
  for (const auto& r : rules) {
    const std::string ap(r.approach);
    std::cout << ap << std::string(16 - std::min<std::size_t>(16, ap.size()), ' ') << (r.yes ? "yes" : "no ")
              << "          " << r.condition << "\n";
  }
  return kExitOk;
}

int cmd_bench(const Args& a) {
  const std::filesystem::path in(a.get("--input"));
  const TiledMatrix A = load_matrix(in);
  const long iters = std::stol(a.get("--iters", "1"));
  if (iters < 1) throw UsageError("--iters must be positive");
  SquareOptions o;
  o.ordered = ordered_numerics(a);
  spgemm_square(A, o);  // warm-up, untimed
  std::vector<PhaseTiming> ts;
  std::uint64_t hash = 0;
  for (long i = 0; i < iters; ++i) {
    const SquareResult r = spgemm_square(A, o);
    ts.push_back(r.timing);
    hash = fnv1a(serialize_tiled(r.output));
  }
  auto pick = [&](double PhaseTiming::*f) {
    std::vector<double> v;
    for (const auto& t : ts) v.push_back(t.*f);
    return lower_median(v);
  };
  const std::string header =
      "matrixName,iters,threads,taskList,sort,counting,multiply,compaction,total,peakBytes,outputHash";
  const std::string row = in.stem().string() + "," + std::to_string(iters) + ",1," + num(pick(&PhaseTiming::task_list)) +
                          "," + num(pick(&PhaseTiming::sort)) + "," + num(pick(&PhaseTiming::counting)) + "," +
                          num(pick(&PhaseTiming::multiply)) + "," + num(pick(&PhaseTiming::compaction)) + "," +
                          num(pick(&PhaseTiming::total)) + ",0," + std::to_string(hash);
  if (a.has("--csv")) {
    std::ofstream out(a.get("--csv"));
    if (!out) throw IoError("cannot open " + a.get("--csv") + " for writing");
    out << header << "\n" << row << "\n";
  }
  std::cout << header << "\n" << row << "\n";
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  try {
    a = parse(argc, argv);
  } catch (const UsageError& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return kExitOther;
  }
  try {
    if (a.cmd == "convert") return cmd_convert(a);
    if (a.cmd == "square") return cmd_square(a);
    if (a.cmd == "compare") return cmd_compare(a);
    if (a.cmd == "stats") return cmd_stats(a);
    if (a.cmd == "bench") return cmd_bench(a);
    return cmd_advise(a);
  } catch (const UsageError& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return kExitOther;
  } catch (const ParseError& e) {
    std::cerr << "parse error: " << e.what() << "\n";
    return kExitParse;
  } catch (const FormatError& e) {
    std::cerr << "format error: " << e.what() << "\n";
    return kExitParse;
  } catch (const InvariantError& e) {
    std::cerr << "invalid input: " << e.what() << "\n";
    return kExitParse;
  } catch (const OverflowError& e) {
    std::cerr << "overflow: " << e.what() << "\n";
    return kExitOverflow;
  } catch (const DimensionError& e) {
    std::cerr << "dimension error: " << e.what() << "\n";
    return kExitDimension;
  } catch (const PrecisionError& e) {
    std::cerr << "precision error: " << e.what() << "\n";
    return kExitPrecision;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitOther;
  }
}
