// tilemul_gpu_io.hpp -- file formats of the B200 front end (SURVEY.md 8(f)
// rows 2-3), header-only C++20 over tilemul_gpu.hpp.  Written from the
// format descriptions, not from the reference's readers:
//
//   .tspz   (proj/README.md:115-123)  little-endian "TSPZ", u32 version 1,
//           u8 element kind (0 = binary16 bit patterns, 1 = f32), u64 rows,
//           cols, tile count, element count, then the arrays tileRow u32[],
//           tileCol u32[], bitmap u64[], elemIndex u64[] and the payload.
//           Whole files are (de)serialised through an in-memory byte buffer:
//           the reader checks every array against the bytes that remain
//           before it allocates, so a hostile header cannot ask for more
//           memory than the file holds.
//   Matrix Market coordinate files (real / integer / pattern, general /
//           symmetric, 1-based, duplicates summed; the subset the reference
//           CLI reads, proj/README.md and mm_io.hpp's contract): parsed from
//           the whole file text with std::from_chars.
//   fnv1a   64-bit FNV-1a of the serialised bytes (the `bench` output hash).
//
// Errors use the reference taxonomy (errors.hpp:14-51): ParseError /
// UnsupportedError for Matrix Market text, FormatError for a malformed
// .tspz byte stream, InvariantError for tiles that break the TiledMatrix
// invariants, IoError for the file system.
#pragma once

#include <bit>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <string>
#include <string_view>
#include <vector>

#include "tilemul_gpu.hpp"

static_assert(std::endian::native == std::endian::little, "the .tspz format is little-endian");

namespace tilemul_gpu {

// ---- binary16 <-> float (the host compiler's _Float16: IEEE RNE) -------------
inline float half_bits_to_float(std::uint16_t h) { return float(std::bit_cast<_Float16>(h)); }
// exact for binary16-representable values (the Fp16Stored invariant)
inline std::uint16_t half_bits_from_float(float f) { return std::bit_cast<std::uint16_t>(_Float16(f)); }
inline bool is_binary16(float f) { return std::isfinite(f) && half_bits_to_float(half_bits_from_float(f)) == f; }

// Sort by (row, col) and sum duplicates (the reference's normalize_coo contract).
inline void normalize_coo(ElementCoo& m) {
  auto& e = m.entries;
  std::stable_sort(e.begin(), e.end(), [](const auto& a, const auto& b) {
    return a.row < b.row || (a.row == b.row && a.col < b.col);
  });
  std::size_t w = 0;
  for (std::size_t i = 0; i < e.size(); ++i) {
    if (w > 0 && e[w - 1].row == e[i].row && e[w - 1].col == e[i].col)
      e[w - 1].value += e[i].value;
    else
      e[w++] = e[i];
  }
  e.resize(w);
}

namespace detail {
inline std::string slurp(const std::filesystem::path& path, bool binary) {
  std::ifstream f(path, binary ? std::ios::binary : std::ios::in);
  if (!f) throw IoError("cannot read " + path.string());
  return std::string(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}
inline std::string slurp(std::istream& in) {
  return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

// Text cursor over the whole Matrix Market file.
struct MmText {
  std::string_view s;
  std::size_t pos = 0;
  // next line that is neither blank nor a % comment; false at the end
  bool next_content(std::string_view& line) {
    while (pos < s.size()) {
      std::size_t e = s.find('\n', pos);
      if (e == std::string_view::npos) e = s.size();
      std::string_view l = s.substr(pos, e - pos);
      pos = e + 1;
      const std::size_t f = l.find_first_not_of(" \t\r");
      if (f == std::string_view::npos || l[f] == '%') continue;
      line = l;
      return true;
    }
    return false;
  }
};

// whitespace-separated fields of one line
inline std::vector<std::string_view> fields(std::string_view l) {
  std::vector<std::string_view> out;
  std::size_t i = 0;
  while (i < l.size()) {
    while (i < l.size() && (l[i] == ' ' || l[i] == '\t' || l[i] == '\r')) ++i;
    std::size_t j = i;
    while (j < l.size() && l[j] != ' ' && l[j] != '\t' && l[j] != '\r') ++j;
    if (j > i) out.push_back(l.substr(i, j - i));
    i = j;
  }
  return out;
}

inline std::string lowered(std::string_view v) {
  std::string s(v);
  for (char& c : s) c = char((c >= 'A' && c <= 'Z') ? c - 'A' + 'a' : c);
  return s;
}

template <class T>
bool parse_num(std::string_view v, T& out) {
  const char* b = v.data();
  const char* e = v.data() + v.size();
  if (b != e && *b == '+') ++b;  // from_chars rejects a leading '+'
  const auto r = std::from_chars(b, e, out);
  return r.ec == std::errc() && r.ptr == e;
}
}  // namespace detail

inline ElementCoo parse_matrix_market(std::string_view text) {
  detail::MmText t{text};
  // banner: %%MatrixMarket matrix coordinate <field> <symmetry>
  const std::size_t nl = text.find('\n');
  const auto banner = detail::fields(text.substr(0, nl));
  t.pos = nl == std::string_view::npos ? text.size() : nl + 1;
  if (banner.size() != 5 || banner[0] != "%%MatrixMarket")
    throw ParseError("not a Matrix Market file (expected a '%%MatrixMarket matrix coordinate ...' banner)");
  const std::string object = detail::lowered(banner[1]), format = detail::lowered(banner[2]),
                    field = detail::lowered(banner[3]), symmetry = detail::lowered(banner[4]);
  if (object != "matrix") throw ParseError("Matrix Market object '" + object + "' is not 'matrix'");
  if (format != "coordinate") throw UnsupportedError("Matrix Market format '" + format + "': only coordinate is read");
  const bool pattern = field == "pattern";
  if (field == "complex") throw UnsupportedError("complex Matrix Market values are not supported");
  if (!pattern && field != "real" && field != "integer")
    throw ParseError("Matrix Market field '" + field + "' is unknown");
  const bool symmetric = symmetry == "symmetric";
  if (symmetry == "skew-symmetric" || symmetry == "hermitian")
    throw UnsupportedError("Matrix Market symmetry '" + symmetry + "' is not supported");
  if (!symmetric && symmetry != "general") throw ParseError("Matrix Market symmetry '" + symmetry + "' is unknown");

  std::string_view line;
  if (!t.next_content(line)) throw ParseError("Matrix Market size line missing");
  const auto sz = detail::fields(line);
  std::int64_t nr = -1, nc = -1, ne = -1;
  if (sz.size() != 3 || !detail::parse_num(sz[0], nr) || !detail::parse_num(sz[1], nc) ||
      !detail::parse_num(sz[2], ne) || nr < 0 || nc < 0 || ne < 0)
    throw ParseError("Matrix Market size line is not 'rows cols entries': '" + std::string(line) + "'");
  if (symmetric && nr != nc) throw ParseError("a symmetric Matrix Market matrix must be square");
  ElementCoo m;
  m.rows = std::uint64_t(nr);
  m.cols = std::uint64_t(nc);
  // an entry line takes >= 4 bytes: a hostile size line cannot over-reserve
  const std::size_t cap = std::min<std::size_t>(std::size_t(ne), text.size() / 4);
  m.entries.reserve(symmetric ? 2 * cap : cap);
  for (std::int64_t k = 0; k < ne; ++k) {
    if (!t.next_content(line)) throw ParseError("Matrix Market file ends after " + std::to_string(k) + " entries");
    const auto f = detail::fields(line);
    std::int64_t i = 0, j = 0;
    double v = 1.0;
    const std::size_t want = pattern ? 2 : 3;
    if (f.size() < want || !detail::parse_num(f[0], i) || !detail::parse_num(f[1], j) ||
        (!pattern && !detail::parse_num(f[2], v)))
      throw ParseError("Matrix Market entry " + std::to_string(k + 1) + " is malformed: '" + std::string(line) + "'");
    if (i < 1 || j < 1 || i > nr || j > nc)
      throw ParseError("Matrix Market entry " + std::to_string(k + 1) + " lies outside the " + std::to_string(nr) +
                       "x" + std::to_string(nc) + " matrix");
    m.entries.push_back({std::uint64_t(i - 1), std::uint64_t(j - 1), v});
    if (symmetric && i != j) m.entries.push_back({std::uint64_t(j - 1), std::uint64_t(i - 1), v});
  }
  normalize_coo(m);
  return m;
}

inline ElementCoo read_matrix_market(std::istream& in) { return parse_matrix_market(detail::slurp(in)); }
inline ElementCoo read_matrix_market(const std::filesystem::path& path) {
  return parse_matrix_market(detail::slurp(path, false));
}

inline void write_matrix_market(const ElementCoo& m, std::ostream& out) {
  out << "%%MatrixMarket matrix coordinate real general\n" << m.rows << ' ' << m.cols << ' ' << m.entries.size()
      << '\n';
  char buf[64];
  for (const auto& e : m.entries) {
    const auto r = std::to_chars(buf, buf + sizeof(buf), e.value);  // shortest round-trip form
    out << e.row + 1 << ' ' << e.col + 1 << ' ' << std::string_view(buf, std::size_t(r.ptr - buf)) << '\n';
  }
}

// TiledMatrix invariants (tile_format.hpp:24-55): tiles strictly ordered by
// (row, col) inside the tile grid, non-empty bitmaps with no bit in an edge
// tile's padding, element runs contiguous and matching the popcounts,
// elements finite and non-zero (binary16-representable when Fp16Stored).
inline void validate_tiled(const TiledMatrix& m) {
  auto fail = [](const std::string& what, std::size_t i) {
    throw InvariantError("tiled matrix: " + what + " (tile " + std::to_string(i) + ")");
  };
  std::uint64_t next = 0;
  for (std::size_t i = 0; i < m.tiles.size(); ++i) {
    const TileEntry& t = m.tiles[i];
    if (i > 0) {
      const TileEntry& p = m.tiles[i - 1];
      if (std::pair(p.tile_row, p.tile_col) >= std::pair(t.tile_row, t.tile_col)) fail("tiles out of order", i);
    }
    if (t.tile_row >= m.tile_rows() || t.tile_col >= m.tile_cols()) fail("tile outside the grid", i);
    if (t.bitmap == 0) fail("empty bitmap", i);
    const std::uint64_t live_rows = std::min<std::uint64_t>(kTileDim, m.rows - std::uint64_t(t.tile_row) * kTileDim);
    const std::uint64_t live_cols = std::min<std::uint64_t>(kTileDim, m.cols - std::uint64_t(t.tile_col) * kTileDim);
    const std::uint64_t row_bits = live_cols >= 8 ? 0xffull : (1ull << live_cols) - 1;
    std::uint64_t live = 0;
    for (std::uint64_t r = 0; r < live_rows; ++r) live |= row_bits << (kTileDim * r);
    if (t.bitmap & ~live) fail("bits beyond the matrix edge", i);
    if (t.elem_index != next) fail("element runs not contiguous", i);
    next += std::uint64_t(std::popcount(t.bitmap));
  }
  if (next != m.elements.size()) throw InvariantError("tiled matrix: bitmaps hold " + std::to_string(next) +
                                                      " slots but " + std::to_string(m.elements.size()) +
                                                      " elements are stored");
  for (std::size_t k = 0; k < m.elements.size(); ++k) {
    const float v = m.elements[k];
    if (v == 0.0f || !std::isfinite(v) || (m.kind == ElementKind::Fp16Stored && !is_binary16(v)))
      throw InvariantError("tiled matrix: element " + std::to_string(k) + " is zero, non-finite or not binary16");
  }
}

// ---- .tspz -------------------------------------------------------------------
namespace detail {
struct ByteWriter {
  std::string buf;
  template <class T>
  void put(T v) {
    char b[sizeof(T)];
    std::memcpy(b, &v, sizeof(T));
    buf.append(b, sizeof(T));
  }
  template <class T>
  void put_all(const std::vector<T>& v) {
    buf.append(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T));
  }
};

struct ByteReader {
  std::string_view b;
  std::size_t at = 0;
  std::size_t left() const { return b.size() - at; }
  template <class T>
  T take() {
    if (left() < sizeof(T)) throw FormatError(".tspz stream ends inside its header");
    T v;
    std::memcpy(&v, b.data() + at, sizeof(T));
    at += sizeof(T);
    return v;
  }
  template <class T>
  std::vector<T> take_array(std::uint64_t n, const char* what) {
    if (n > left() / sizeof(T)) throw FormatError(std::string(".tspz stream too short for its ") + what + " array");
    std::vector<T> v(n);
    std::memcpy(v.data(), b.data() + at, n * sizeof(T));
    at += n * sizeof(T);
    return v;
  }
};
}  // namespace detail

inline std::string serialize_tiled(const TiledMatrix& m) {
  detail::ByteWriter w;
  w.buf.reserve(41 + m.tiles.size() * 24 + m.elements.size() * 4);
  w.buf.append("TSPZ", 4);
  w.put<std::uint32_t>(1);
  w.put<std::uint8_t>(std::uint8_t(m.kind));
  for (std::uint64_t v : {m.rows, m.cols, std::uint64_t(m.tiles.size()), std::uint64_t(m.elements.size())}) w.put(v);
  std::vector<std::uint32_t> tr, tc;
  std::vector<std::uint64_t> bm, ei;
  tr.reserve(m.tiles.size());
  tc.reserve(m.tiles.size());
  bm.reserve(m.tiles.size());
  ei.reserve(m.tiles.size());
  for (const auto& t : m.tiles) {
    tr.push_back(t.tile_row);
    tc.push_back(t.tile_col);
    bm.push_back(t.bitmap);
    ei.push_back(t.elem_index);
  }
  w.put_all(tr);
  w.put_all(tc);
  w.put_all(bm);
  w.put_all(ei);
  if (m.kind == ElementKind::Fp16Stored) {
    std::vector<std::uint16_t> h(m.elements.size());
    for (std::size_t i = 0; i < h.size(); ++i) h[i] = half_bits_from_float(m.elements[i]);
    w.put_all(h);
  } else {
    w.put_all(m.elements);
  }
  return std::move(w.buf);
}

inline TiledMatrix deserialize_tiled(std::string_view bytes) {
  detail::ByteReader r{bytes};
  if (bytes.size() < 4 || bytes.substr(0, 4) != "TSPZ") throw FormatError("not a .tspz stream (magic bytes)");
  r.at = 4;
  const auto version = r.take<std::uint32_t>();
  if (version != 1) throw FormatError(".tspz version " + std::to_string(version) + " is not 1");
  const auto kind = r.take<std::uint8_t>();
  if (kind > 1) throw FormatError(".tspz element kind " + std::to_string(kind) + " is neither 0 nor 1");
  TiledMatrix m;
  m.kind = ElementKind(kind);
  m.rows = r.take<std::uint64_t>();
  m.cols = r.take<std::uint64_t>();
  const auto ntiles = r.take<std::uint64_t>(), nelem = r.take<std::uint64_t>();
  const auto tr = r.take_array<std::uint32_t>(ntiles, "tileRow");
  const auto tc = r.take_array<std::uint32_t>(ntiles, "tileCol");
  const auto bm = r.take_array<std::uint64_t>(ntiles, "bitmap");
  const auto ei = r.take_array<std::uint64_t>(ntiles, "elemIndex");
  m.tiles.resize(ntiles);
  for (std::uint64_t i = 0; i < ntiles; ++i) m.tiles[i] = TileEntry{tr[i], tc[i], ei[i], bm[i]};
  if (m.kind == ElementKind::Fp16Stored) {
    const auto h = r.take_array<std::uint16_t>(nelem, "element");
    m.elements.resize(nelem);
    for (std::uint64_t i = 0; i < nelem; ++i) m.elements[i] = half_bits_to_float(h[i]);
  } else {
    m.elements = r.take_array<float>(nelem, "element");
  }
  validate_tiled(m);
  return m;
}

inline void write_tiled_binary(const TiledMatrix& m, std::ostream& out) {
  const std::string b = serialize_tiled(m);
  out.write(b.data(), std::streamsize(b.size()));
  if (!out) throw IoError("writing the .tspz stream failed");
}
inline void write_tiled_binary(const TiledMatrix& m, const std::filesystem::path& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot write " + path.string());
  write_tiled_binary(m, out);
}
inline TiledMatrix read_tiled_binary(std::istream& in) { return deserialize_tiled(detail::slurp(in)); }
inline TiledMatrix read_tiled_binary(const std::filesystem::path& path) {
  return deserialize_tiled(detail::slurp(path, true));
}

// The reference CLI's output hash (proj/tools/tilemul.cpp:37-44): FNV-1a
// with the 64-bit prime but the offset basis 1469598103934665603 (the
// reference's constant, not the standard 14695981039346656037) -- kept so
// hashes compare across the two front ends.
inline std::uint64_t fnv1a(std::string_view bytes) {
  std::uint64_t h = 1469598103934665603ull;
  for (const unsigned char c : bytes) h = (h ^ c) * 0x100000001b3ull;
  return h;
}

}  // namespace tilemul_gpu
