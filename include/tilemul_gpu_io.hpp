// tilemul_gpu_io.hpp -- the reference's file formats for the B200 front end
// (SURVEY.md 8(f) rows 2-3), header-only C++20 over tilemul_gpu.hpp:
//
//   read_matrix_market            mm_io.cpp:29-135   coordinate real/integer/
//                                                    pattern, general/symmetric,
//                                                    1-based, duplicates summed
//   normalize_coo                 tile_format.cpp:14-32
//   validate_tiled                tile_format.cpp:174-225
//   write/read_tiled_binary,      tiled_io.cpp:55-158  the ".tspz" format:
//   serialize_tiled                  LE "TSPZ", u32 version 1, u8 kind, u64 rows,
//                                    cols, tiles, elements; SoA tileRow u32[],
//                                    tileCol u32[], bitmap u64[], elemIndex u64[],
//                                    payload (u16 binary16 bits or f32)
//   fnv1a                         tools/tilemul.cpp:37-44 (the bench output hash)
//
// Same error taxonomy and messages' intent: ParseError / UnsupportedError for
// Matrix Market, FormatError for a broken .tspz, InvariantError for a .tspz
// whose tiles break the format invariants, IoError for files.
#pragma once

#include <bit>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <istream>
#include <sstream>
#include <string>
#include <vector>

#include "tilemul_gpu.hpp"

static_assert(std::endian::native == std::endian::little, "the .tspz format is little-endian");

namespace tilemul_gpu {

// ---- binary16 bit patterns (half.cpp:43-79) ---------------------------------
inline float half_bits_to_float(std::uint16_t h) {
  const int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
  double v;
  if (e == 0) v = std::ldexp(double(m), -24);
  else if (e == 31) v = m ? std::nan("") : INFINITY;
  else v = std::ldexp(double(m | 1024), e - 25);
  return float(s ? -v : v);
}

// exact for binary16-representable values (the Fp16Stored invariant)
inline std::uint16_t half_bits_from_float(float f) {
  const std::uint32_t x = std::bit_cast<std::uint32_t>(f);
  const std::uint16_t sign = std::uint16_t((x >> 16) & 0x8000u);
  const float a = std::fabs(f);
  if (a == 0.0f) return sign;
  if (std::isinf(a)) return std::uint16_t(sign | 0x7c00u);
  if (std::isnan(a)) return std::uint16_t(sign | 0x7e00u);
  int e2 = 0;
  std::frexp(double(a), &e2);
  const int e = e2 - 1;  // a in [2^e, 2^(e+1))
  if (e < -14)  // subnormal: m * 2^-24
    return std::uint16_t(sign | std::uint16_t(std::lround(std::ldexp(double(a), 24))));
  const int m = int(std::lround(std::ldexp(double(a), 10 - e))) - 1024;
  return std::uint16_t(sign | std::uint16_t((e + 15) << 10) | std::uint16_t(m));
}

inline bool is_binary16(float f) {
  return std::isfinite(f) && half_bits_to_float(half_bits_from_float(f)) == f;
}

// ---- COO normalisation (tile_format.cpp:14-32) ----------------------------------
inline void normalize_coo(ElementCoo& m) {
  std::sort(m.entries.begin(), m.entries.end(), [](const auto& a, const auto& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  std::size_t out = 0;
  for (std::size_t i = 0; i < m.entries.size();) {
    ElementCoo::Entry e = m.entries[i];
    std::size_t j = i + 1;
    for (; j < m.entries.size() && m.entries[j].row == e.row && m.entries[j].col == e.col; ++j)
      e.value += m.entries[j].value;
    m.entries[out++] = e;
    i = j;
  }
  m.entries.resize(out);
}

// ---- Matrix Market (mm_io.cpp:29-135) --------------------------------------------
namespace detail {
inline std::string lower(std::string s) {
  for (auto& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
  return s;
}
inline bool content_line(std::istream& in, std::string& line) {
  while (std::getline(in, line)) {
    const auto p = line.find_first_not_of(" \t\r");
    if (p == std::string::npos || line[p] == '%') continue;
    return true;
  }
  return false;
}
}  // namespace detail

inline ElementCoo read_matrix_market(std::istream& in) {
  std::string line;
  if (!std::getline(in, line)) throw ParseError("empty Matrix Market file");
  if (!line.empty() && line.back() == '\r') line.pop_back();
  std::istringstream hs(line);
  std::string tag, object, format, field, symmetry;
  hs >> tag >> object >> format >> field >> symmetry;
  if (hs.fail() || tag != "%%MatrixMarket") throw ParseError("malformed Matrix Market banner: \"" + line + "\"");
  if (detail::lower(object) != "matrix") throw ParseError("unexpected Matrix Market object \"" + object + "\"");
  if (detail::lower(format) != "coordinate")
    throw UnsupportedError("only coordinate format is supported, got \"" + format + "\"");
  const std::string f = detail::lower(field), sy = detail::lower(symmetry);
  if (f == "complex") throw UnsupportedError("complex matrices are not supported");
  if (f != "real" && f != "integer" && f != "pattern") throw ParseError("unknown Matrix Market field \"" + field + "\"");
  if (sy == "skew-symmetric" || sy == "hermitian")
    throw UnsupportedError("symmetry \"" + symmetry + "\" is not supported");
  if (sy != "general" && sy != "symmetric") throw ParseError("unknown Matrix Market symmetry \"" + symmetry + "\"");
  const bool pattern = f == "pattern", symmetric = sy == "symmetric";
  if (!detail::content_line(in, line)) throw ParseError("missing Matrix Market size line");
  long long r = -1, c = -1, n = -1;
  {
    std::istringstream ss(line);
    std::string rest;
    ss >> r >> c >> n;
    if (ss.fail() || (ss >> rest, !rest.empty()) || r < 0 || c < 0 || n < 0)
      throw ParseError("malformed size line: \"" + line + "\"");
  }
  if (symmetric && r != c) throw ParseError("symmetric matrix must be square");
  ElementCoo out;
  out.rows = std::uint64_t(r);
  out.cols = std::uint64_t(c);
  out.entries.reserve(std::size_t(symmetric ? 2 * n : n));
  for (long long i = 0; i < n; ++i) {
    long long er = 0, ec = 0;
    double v = 1.0;
    in >> er >> ec;
    if (!pattern) in >> v;
    if (in.fail()) throw ParseError("malformed entry " + std::to_string(i + 1) + " of " + std::to_string(n));
    if (er < 1 || ec < 1 || er > r || ec > c)
      throw ParseError("entry " + std::to_string(i + 1) + " index (" + std::to_string(er) + ", " +
                       std::to_string(ec) + ") out of range");
    out.entries.push_back({std::uint64_t(er - 1), std::uint64_t(ec - 1), v});
    if (symmetric && er != ec) out.entries.push_back({std::uint64_t(ec - 1), std::uint64_t(er - 1), v});
  }
  normalize_coo(out);
  return out;
}

inline ElementCoo read_matrix_market(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open " + path.string());
  return read_matrix_market(in);
}

inline void write_matrix_market(const ElementCoo& m, std::ostream& out) {
  out << "%%MatrixMarket matrix coordinate real general\n" << m.rows << ' ' << m.cols << ' ' << m.entries.size() << '\n';
  out.precision(17);
  for (const auto& e : m.entries) out << e.row + 1 << ' ' << e.col + 1 << ' ' << e.value << '\n';
}

// ---- tiled-format invariants (tile_format.cpp:174-225) -------------------------
inline void validate_tiled(const TiledMatrix& m) {
  std::uint64_t expected = 0;
  const TileEntry* prev = nullptr;
  for (const auto& t : m.tiles) {
    if (prev && (prev->tile_row > t.tile_row || (prev->tile_row == t.tile_row && prev->tile_col >= t.tile_col)))
      throw InvariantError("tiles unsorted or duplicated at (" + std::to_string(t.tile_row) + ", " +
                           std::to_string(t.tile_col) + ")");
    if (t.tile_row >= m.tile_rows() || t.tile_col >= m.tile_cols())
      throw InvariantError("tile outside the tile grid");
    if (t.bitmap == 0) throw InvariantError("empty bitmap in a tile");
    // slots past the matrix edge (the padding of edge tiles) must be empty
    const std::uint64_t vr = std::min<std::uint64_t>(kTileDim, m.rows - std::uint64_t(t.tile_row) * kTileDim);
    const std::uint64_t vc = std::min<std::uint64_t>(kTileDim, m.cols - std::uint64_t(t.tile_col) * kTileDim);
    std::uint64_t interior = 0;
    for (std::uint64_t r = 0; r < vr; ++r) interior |= ((vc == 8 ? 0xffull : ((1ull << vc) - 1)) << (8 * r));
    if (t.bitmap & ~interior) throw InvariantError("tile has bits in the padding region");
    if (t.elem_index != expected) throw InvariantError("tile element runs are not contiguous");
    expected += std::uint64_t(std::popcount(t.bitmap));
    prev = &t;
  }
  if (expected != m.elements.size()) throw InvariantError("bitmap population != element count");
  for (const float v : m.elements) {
    if (!std::isfinite(v) || v == 0.0f) throw InvariantError("stored element is zero or non-finite");
    if (m.kind == ElementKind::Fp16Stored && !is_binary16(v))
      throw InvariantError("fp16-stored element is not binary16-representable");
  }
}

// ---- .tspz (tiled_io.cpp:55-158) --------------------------------------------------
namespace detail {
template <typename T>
void put(std::ostream& out, T v) {
  out.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
T get(std::istream& in) {
  T v{};
  in.read(reinterpret_cast<char*>(&v), sizeof(T));
  if (!in) throw FormatError("truncated tiled binary file");
  return v;
}
template <typename T>
std::vector<T> get_array(std::istream& in, std::uint64_t n) {
  if (n > (1ull << 40)) throw FormatError("implausible array length " + std::to_string(n));
  std::vector<T> v(n);
  in.read(reinterpret_cast<char*>(v.data()), std::streamsize(n * sizeof(T)));
  if (!in) throw FormatError("truncated tiled binary file");
  return v;
}
}  // namespace detail

inline void write_tiled_binary(const TiledMatrix& m, std::ostream& out) {
  out.write("TSPZ", 4);
  detail::put<std::uint32_t>(out, 1);
  detail::put<std::uint8_t>(out, std::uint8_t(m.kind));
  detail::put<std::uint64_t>(out, m.rows);
  detail::put<std::uint64_t>(out, m.cols);
  detail::put<std::uint64_t>(out, m.tiles.size());
  detail::put<std::uint64_t>(out, m.elements.size());
  for (const auto& t : m.tiles) detail::put<std::uint32_t>(out, t.tile_row);
  for (const auto& t : m.tiles) detail::put<std::uint32_t>(out, t.tile_col);
  for (const auto& t : m.tiles) detail::put<std::uint64_t>(out, t.bitmap);
  for (const auto& t : m.tiles) detail::put<std::uint64_t>(out, t.elem_index);
  if (m.kind == ElementKind::Fp16Stored) {
    for (const float v : m.elements) detail::put<std::uint16_t>(out, half_bits_from_float(v));
  } else {
    out.write(reinterpret_cast<const char*>(m.elements.data()), std::streamsize(m.elements.size() * 4));
  }
  if (!out) throw IoError("write to tiled binary stream failed");
}

inline void write_tiled_binary(const TiledMatrix& m, const std::filesystem::path& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot open " + path.string() + " for writing");
  write_tiled_binary(m, out);
}

inline TiledMatrix read_tiled_binary(std::istream& in) {
  char magic[4] = {};
  in.read(magic, 4);
  if (!in || std::memcmp(magic, "TSPZ", 4) != 0) throw FormatError("bad magic, not a tiled binary file");
  const auto version = detail::get<std::uint32_t>(in);
  if (version != 1) throw FormatError("unsupported tiled binary version " + std::to_string(version));
  const auto kind = detail::get<std::uint8_t>(in);
  if (kind > 1) throw FormatError("unknown element kind " + std::to_string(kind));
  TiledMatrix m;
  m.kind = ElementKind(kind);
  m.rows = detail::get<std::uint64_t>(in);
  m.cols = detail::get<std::uint64_t>(in);
  const auto nt = detail::get<std::uint64_t>(in), ne = detail::get<std::uint64_t>(in);
  const auto pos = in.tellg();  // declared payload vs remaining bytes before allocating
  if (pos != std::istream::pos_type(-1)) {
    in.seekg(0, std::ios::end);
    const auto end = in.tellg();
    in.seekg(pos);
    const auto remaining = std::uint64_t(end - pos);
    if (nt > remaining / 24 || ne > remaining / (m.kind == ElementKind::Fp16Stored ? 2 : 4))
      throw FormatError("truncated tiled binary file");
  }
  const auto tr = detail::get_array<std::uint32_t>(in, nt);
  const auto tc = detail::get_array<std::uint32_t>(in, nt);
  const auto bm = detail::get_array<std::uint64_t>(in, nt);
  const auto ei = detail::get_array<std::uint64_t>(in, nt);
  m.tiles.resize(nt);
  for (std::uint64_t i = 0; i < nt; ++i) m.tiles[i] = {tr[i], tc[i], ei[i], bm[i]};
  if (m.kind == ElementKind::Fp16Stored) {
    const auto bits = detail::get_array<std::uint16_t>(in, ne);
    m.elements.resize(ne);
    for (std::uint64_t i = 0; i < ne; ++i) m.elements[i] = half_bits_to_float(bits[i]);
  } else {
    m.elements = detail::get_array<float>(in, ne);
  }
  validate_tiled(m);
  return m;
}

inline TiledMatrix read_tiled_binary(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path.string());
  return read_tiled_binary(in);
}

inline std::string serialize_tiled(const TiledMatrix& m) {
  std::ostringstream out(std::ios::binary);
  write_tiled_binary(m, out);
  return std::move(out).str();
}

inline std::uint64_t fnv1a(const std::string& bytes) {
  std::uint64_t h = 1469598103934665603ull;
  for (const unsigned char c : bytes) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

}  // namespace tilemul_gpu
