// NPY reader / writer (reference contract: /root/reference/proj/src/npy.cpp:76-207,
// messages and header layout pinned by tests/test_io.cpp:75-197).
//
// The payload is read in one block and widened with a single pass; for the
// fp32 cubes the GPU path consumes, `npy_to_image` is followed by the upload in
// edaa_set_image_host_checked / edaa_ingest_host, which narrows back to the
// same fp32 bits (the widening is exact).
#include "archetype/npy.hpp"

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string_view>

#include "archetype/error.hpp"
#include "device.hpp"

namespace archetype {

namespace {

constexpr std::string_view kNpyMagic{"\x93NUMPY", 6};

[[noreturn]] void npy_error(const std::string& path, const std::string& what) {
  throw Error(path + ": " + what);
}

// The header is a Python dict literal. Lookups follow numpy's own writer
// layout ('key': value) and tolerate anything after the value: a key is
// located by its quoted name, its value is the next token of the wanted kind.
struct HeaderDict {
  const std::string& text;
  const std::string& path;

  std::size_t locate(const char* key) const {
    const std::string quoted = std::string("'") + key + "'";
    const std::size_t at = text.find(quoted);
    if (at == std::string::npos) npy_error(path, std::string("header missing '") + key + "'");
    return at;
  }

  // The next quoted string after the key's closing quote.
  std::string quoted_value(const char* key) const {
    const std::size_t from = locate(key) + std::strlen(key) + 2;
    const std::size_t q0 = text.find('\'', from);
    const std::size_t q1 = q0 == std::string::npos ? q0 : text.find('\'', q0 + 1);
    if (q1 == std::string::npos)
      npy_error(path, std::string("malformed header value for '") + key + "'");
    return text.substr(q0 + 1, q1 - q0 - 1);
  }

  // Whichever of True / False appears first after the key.
  bool flag_value(const char* key) const {
    const std::size_t from = locate(key) + std::strlen(key) + 2;
    const std::size_t t = text.find("True", from);
    const std::size_t f = text.find("False", from);
    if (t == std::string::npos && f == std::string::npos)
      npy_error(path, std::string("malformed header value for '") + key + "'");
    return t < f;  // npos compares greater than any position
  }

  // The first parenthesised tuple after 'shape': comma-separated decimal
  // extents, blanks ignored, an empty trailing item allowed ("(5,)").
  std::vector<std::size_t> tuple_value(const char* key) const {
    const std::size_t at = locate(key);
    const std::size_t open = text.find('(', at);
    const std::size_t close = text.find(')', at);
    if (open == std::string::npos || close == std::string::npos || close < open)
      npy_error(path, "malformed shape tuple");
    std::vector<std::size_t> dims;
    std::size_t i = open + 1;
    while (i <= close) {
      std::size_t end = text.find(',', i);
      if (end == std::string::npos || end > close) end = close;
      std::size_t a = i, b = end;
      while (a < b && (text[a] == ' ' || text[a] == '\t')) ++a;
      while (b > a && (text[b - 1] == ' ' || text[b - 1] == '\t')) --b;
      if (a < b) {
        std::size_t v = 0;
        for (std::size_t k = a; k < b; ++k) {
          if (text[k] < '0' || text[k] > '9') npy_error(path, "malformed shape tuple");
          v = v * 10 + static_cast<std::size_t>(text[k] - '0');
        }
        dims.push_back(v);
      }  // blank items are skipped, as the reference's tokenizer does
      i = end + 1;
    }
    return dims;
  }
};

}  // namespace

std::size_t NpyArray::element_count() const {
  std::size_t n = 1;
  for (const std::size_t d : shape) n *= d;
  return n;
}

namespace detail {

NpyPayload read_npy_payload(const std::string& path) {
  std::ifstream file(path, std::ios::binary);
  if (!file) npy_error(path, "cannot open file");

  char preamble[8] = {};
  file.read(preamble, sizeof preamble);
  if (!file || std::string_view(preamble, 6) != kNpyMagic) npy_error(path, "not an NPY file (bad magic)");
  const unsigned version = static_cast<unsigned char>(preamble[6]);
  if (version != 1 && version != 2)
    npy_error(path, "unsupported NPY format version " + std::to_string(version));

  // Little-endian header length: 2 bytes in format 1.0, 4 in 2.0.
  unsigned char len_bytes[4] = {};
  const std::size_t len_width = version == 1 ? 2 : 4;
  file.read(reinterpret_cast<char*>(len_bytes), static_cast<std::streamsize>(len_width));
  if (!file) npy_error(path, "truncated header");
  std::uint32_t header_len = 0;
  for (std::size_t k = len_width; k-- > 0;) header_len = (header_len << 8) | len_bytes[k];

  std::string header(header_len, '\0');
  file.read(header.data(), header_len);
  if (!file) npy_error(path, "truncated header");

  const HeaderDict dict{header, path};
  const std::string descr = dict.quoted_value("descr");
  NpyPayload array;
  if (descr == "<f4") {
    array.dtype = NpyDtype::f4;
  } else if (descr == "<f8") {
    array.dtype = NpyDtype::f8;
  } else {
    npy_error(path, "unsupported dtype '" + descr + "' (need <f4 or <f8)");
  }
  if (dict.flag_value("fortran_order")) npy_error(path, "Fortran-order arrays are not supported");
  array.shape = dict.tuple_value("shape");
  if (array.shape.empty()) npy_error(path, "zero-dimensional array");

  std::size_t count = 1;
  for (const std::size_t d : array.shape) count *= d;
  const auto fill = [&](auto& buf) {
    buf.resize(count);
    const auto want = static_cast<std::streamsize>(count * sizeof(buf[0]));
    file.read(reinterpret_cast<char*>(buf.data()), want);
    if (file.gcount() != want) npy_error(path, "truncated data section");
  };
  if (array.dtype == NpyDtype::f8)
    fill(array.f64);
  else
    fill(array.f32);
  return array;
}

}  // namespace detail

NpyArray read_npy(const std::string& path) {
  detail::NpyPayload raw = detail::read_npy_payload(path);
  NpyArray array;
  array.shape = std::move(raw.shape);
  array.dtype = raw.dtype;
  if (raw.dtype == NpyDtype::f8)
    array.values = std::move(raw.f64);
  else
    array.values.assign(raw.f32.begin(), raw.f32.end());  // exact widening
  return array;
}

void write_npy(const std::string& path, std::span<const std::size_t> shape,
               std::span<const double> values, NpyDtype dtype) {
  if (shape.empty()) throw Error(path + ": refusing to write a zero-dimensional array");
  std::size_t count = 1;
  for (const std::size_t d : shape) count *= d;
  if (count != values.size()) throw Error(path + ": shape does not match value count");

  // numpy's own header: "(a, b)" for n-D, "(a,)" for 1-D.
  std::string dims;
  for (std::size_t i = 0; i < shape.size(); ++i) {
    if (i) dims += ", ";
    dims += std::to_string(shape[i]);
  }
  if (shape.size() == 1) dims += ",";
  std::string header = std::string("{'descr': '") + (dtype == NpyDtype::f4 ? "<f4" : "<f8") +
                       "', 'fortran_order': False, 'shape': (" + dims + "), }";
  // magic(6) + version(2) + length(2) + header + '\n', padded to 64 bytes.
  const std::size_t used = 10 + header.size() + 1;
  header.append((64 - used % 64) % 64, ' ');
  header += '\n';

  std::ofstream file(path, std::ios::binary | std::ios::trunc);
  if (!file) throw Error(path + ": cannot open file for writing");
  if (header.size() > 0xffff) throw Error(path + ": header too large for format version 1.0");
  const char lead[10] = {kNpyMagic[0], kNpyMagic[1], kNpyMagic[2], kNpyMagic[3], kNpyMagic[4],
                         kNpyMagic[5], 1, 0, static_cast<char>(header.size() & 0xff),
                         static_cast<char>(header.size() >> 8)};
  file.write(lead, sizeof lead);
  file.write(header.data(), static_cast<std::streamsize>(header.size()));
  if (dtype == NpyDtype::f4) {
    std::vector<float> narrow(values.begin(), values.end());
    file.write(reinterpret_cast<const char*>(narrow.data()),
               static_cast<std::streamsize>(narrow.size() * sizeof(float)));
  } else {
    file.write(reinterpret_cast<const char*>(values.data()),
               static_cast<std::streamsize>(values.size() * sizeof(double)));
  }
  if (!file) throw Error(path + ": write failed");
}

Matrix npy_to_matrix(const NpyArray& array) {
  if (array.shape.size() != 2) throw Error("expected a 2-D array");
  Matrix m(array.shape[0], array.shape[1]);
  const auto dst = m.values();
  for (std::size_t i = 0; i < dst.size(); ++i) dst[i] = array.values[i];
  return m;
}

HsiImage npy_to_image(const NpyArray& array) {
  HsiImage image;
  if (array.shape.size() == 2) {
    image.data = npy_to_matrix(array);
    return image;
  }
  if (array.shape.size() != 3) throw Error("expected a 2-D matrix or 3-D cube");
  // (H, W, L) band-interleaved-by-pixel → BSQ L×(H·W): a blocked transpose of
  // the (H·W)×L payload so both sides stream through cache.
  const std::size_t h = array.shape[0], w = array.shape[1], bands = array.shape[2];
  const std::size_t n = h * w;
  Matrix x(bands, n);
  constexpr std::size_t kBlock = 64;
  for (std::size_t j0 = 0; j0 < n; j0 += kBlock) {
    const std::size_t j1 = j0 + kBlock < n ? j0 + kBlock : n;
    for (std::size_t b0 = 0; b0 < bands; b0 += kBlock) {
      const std::size_t b1 = b0 + kBlock < bands ? b0 + kBlock : bands;
      for (std::size_t j = j0; j < j1; ++j)
        for (std::size_t b = b0; b < b1; ++b) x(b, j) = array.values[j * bands + b];
    }
  }
  image.data = std::move(x);
  image.spatial = Shape2d{h, w};
  return image;
}

}  // namespace archetype
