// Tensor file formats of the reference (imageio.hpp), host side:
//   NDTENSOR  "NDTENSOR <ndim> <d_1> ... <d_n>\n" + element_count little-endian f64 values
//             in storage order (imageio.hpp:24-125): bit-exact round trips, strict
//             header, truncated / trailing / non-finite payload -> FormatError, writing a
//             non-finite value -> NumericError.
//   PGM       P5 / P2 graymaps, maxval <= 65535 (16-bit P5 big-endian) read as raw sample
//             values, shape (height, width); written as 8-bit P5 with round-half-even,
//             optional clamp to [0,255] (imageio.hpp:126-265).
// Plus the streaming NDTENSOR <-> plan paths (Plan::load_observation_ndtensor /
// save_estimate_ndtensor in ndc_plan.cu) that use read_ndtensor_header().
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "ndc_io.h"
#include "ndc_plan.h"

namespace ndc {

namespace {
static_assert(sizeof(double) == 8, "f64");

bool little_endian() {
  const uint16_t one = 1;
  unsigned char b;
  std::memcpy(&b, &one, 1);
  return b == 1;
}

void to_le(double* v, size_t n) {
  if (little_endian()) return;
  for (size_t i = 0; i < n; ++i) {
    unsigned char* p = reinterpret_cast<unsigned char*>(v + i);
    for (int k = 0; k < 4; ++k) std::swap(p[k], p[7 - k]);
  }
}
}  // namespace

NdtHeader read_ndtensor_header(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(NDC_ERR_FORMAT, "cannot open " + path);
  std::string header;
  if (!std::getline(in, header)) fail(NDC_ERR_FORMAT, "read_tensor: missing header");
  std::istringstream hs(header);
  std::string magic;
  hs >> magic;
  if (magic != "NDTENSOR") fail(NDC_ERR_FORMAT, "read_tensor: bad magic '" + magic + "'");
  long long ndim = -1;
  if (!(hs >> ndim) || ndim < 1 || ndim > 16)
    fail(NDC_ERR_FORMAT, "read_tensor: dimension count must be a positive integer");
  NdtHeader h;
  size_t count = 1;
  for (long long i = 0; i < ndim; ++i) {
    long long e = -1;
    if (!(hs >> e) || e < 1)
      fail(NDC_ERR_FORMAT, "read_tensor: expected " + std::to_string(ndim) + " positive extents");
    if (static_cast<size_t>(e) > SIZE_MAX / count)
      fail(NDC_ERR_FORMAT, "read_tensor: Shape: element count overflows");
    count *= static_cast<size_t>(e);
    h.ext.push_back(static_cast<size_t>(e));
  }
  std::string junk;
  if (hs >> junk) fail(NDC_ERR_FORMAT, "read_tensor: trailing tokens in header");
  h.count = count;
  h.payload_offset = static_cast<size_t>(in.tellg());
  in.seekg(0, std::ios::end);
  const size_t size = static_cast<size_t>(in.tellg());
  if (size < h.payload_offset + count * 8) {
    const size_t have = size > h.payload_offset ? (size - h.payload_offset) / 8 : 0;
    fail(NDC_ERR_FORMAT, "read_tensor: truncated payload at element " + std::to_string(have));
  }
  if (size > h.payload_offset + count * 8)
    fail(NDC_ERR_FORMAT, "read_tensor: trailing data after payload");
  return h;
}

void check_finite_payload(const double* v, size_t n, size_t first_index) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i]))
      fail(NDC_ERR_FORMAT, "read_tensor: non-finite value at element " + std::to_string(first_index + i));
}

void read_ndtensor(const std::string& path, double* out, size_t capacity, NdtHeader* hdr) {
  NdtHeader h = read_ndtensor_header(path);
  if (capacity < h.count) fail(NDC_ERR_ARGUMENT, "read_tensor: output capacity too small");
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) fail(NDC_ERR_FORMAT, "cannot open " + path);
  std::fseek(f, static_cast<long>(h.payload_offset), SEEK_SET);
  const size_t got = std::fread(out, 8, h.count, f);
  std::fclose(f);
  if (got != h.count) fail(NDC_ERR_FORMAT, "read_tensor: truncated payload at element " + std::to_string(got));
  to_le(out, h.count);
  check_finite_payload(out, h.count, 0);
  if (hdr) *hdr = h;
}

std::string ndtensor_header_line(const std::vector<size_t>& ext) {
  std::string s = "NDTENSOR " + std::to_string(ext.size());
  for (size_t e : ext) s += " " + std::to_string(e);
  return s + "\n";
}

void write_ndtensor(const std::string& path, const std::vector<size_t>& ext, const double* data) {
  size_t n = 1;
  for (size_t e : ext) n *= e;
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(data[i])) fail(NDC_ERR_NUMERIC, "write_tensor: refusing to store non-finite values");
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) fail(NDC_ERR_FORMAT, "cannot open " + path + " for writing");
  const std::string hl = ndtensor_header_line(ext);
  bool ok = std::fwrite(hl.data(), 1, hl.size(), f) == hl.size();
  if (little_endian()) {
    ok = ok && std::fwrite(data, 8, n, f) == n;
  } else {
    std::vector<double> tmp(data, data + n);
    to_le(tmp.data(), n);
    ok = ok && std::fwrite(tmp.data(), 8, n, f) == n;
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) fail(NDC_ERR_FORMAT, "write_tensor: stream failure");
}

// ---- PGM ------------------------------------------------------------------------------------
namespace {
struct PgmReader {
  std::FILE* f;
  int get() { return std::fgetc(f); }
  void unget(int c) { std::ungetc(c, f); }
  std::string token() {
    int c = get();
    while (c != EOF) {
      if (c == '#') {
        while (c != EOF && c != '\n') c = get();
      } else if (std::isspace(c)) {
        c = get();
      } else {
        break;
      }
    }
    if (c == EOF) fail(NDC_ERR_FORMAT, "read_pgm: unexpected end of header");
    std::string t;
    while (c != EOF && !std::isspace(c)) {
      t.push_back(static_cast<char>(c));
      c = get();
    }
    if (c != EOF) unget(c);
    return t;
  }
  size_t uint(const char* what, size_t max) {
    const std::string t = token();
    size_t v = 0;
    for (char ch : t) {
      if (ch < '0' || ch > '9')
        fail(NDC_ERR_FORMAT, std::string("read_pgm: ") + what + " is not a number: '" + t + "'");
      v = v * 10 + static_cast<size_t>(ch - '0');
      if (v > max) fail(NDC_ERR_FORMAT, std::string("read_pgm: ") + what + " exceeds " + std::to_string(max));
    }
    return v;
  }
};
}  // namespace

void read_pgm(const std::string& path, std::vector<double>* data, size_t* height, size_t* width) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) fail(NDC_ERR_FORMAT, "cannot open " + path);
  struct Closer {
    std::FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  PgmReader r{f};
  const std::string magic = r.token();
  if (magic != "P5" && magic != "P2") fail(NDC_ERR_FORMAT, "read_pgm: bad magic '" + magic + "'");
  const size_t w = r.uint("width", 1u << 20);
  const size_t h = r.uint("height", 1u << 20);
  if (w == 0 || h == 0) fail(NDC_ERR_FORMAT, "read_pgm: zero image dimension");
  const size_t maxval = r.uint("maxval", 65535);
  if (maxval == 0) fail(NDC_ERR_FORMAT, "read_pgm: maxval must be positive");
  data->assign(w * h, 0.0);
  if (magic == "P5") {
    const int sep = r.get();
    if (sep == EOF || !std::isspace(sep))
      fail(NDC_ERR_FORMAT, "read_pgm: expected single whitespace before P5 payload");
    const size_t bpp = maxval > 255 ? 2 : 1;
    std::vector<unsigned char> buf(w * h * bpp);
    if (std::fread(buf.data(), 1, buf.size(), f) != buf.size())
      fail(NDC_ERR_FORMAT, "read_pgm: truncated P5 payload");
    for (size_t i = 0; i < w * h; ++i) {
      const size_t v = bpp == 1 ? buf[i] : (static_cast<size_t>(buf[2 * i]) << 8) | buf[2 * i + 1];
      if (v > maxval) fail(NDC_ERR_FORMAT, "read_pgm: sample " + std::to_string(v) + " exceeds maxval");
      (*data)[i] = static_cast<double>(v);
    }
  } else {
    for (size_t i = 0; i < w * h; ++i) {
      size_t v;
      try {
        v = r.uint("sample", 65535);
      } catch (const Error&) {
        fail(NDC_ERR_FORMAT, "read_pgm: truncated or malformed P2 samples at index " + std::to_string(i));
      }
      if (v > maxval) fail(NDC_ERR_FORMAT, "read_pgm: sample " + std::to_string(v) + " exceeds maxval");
      (*data)[i] = static_cast<double>(v);
    }
  }
  for (int c = r.get(); c != EOF; c = r.get())
    if (!std::isspace(c)) fail(NDC_ERR_FORMAT, "read_pgm: trailing data after samples");
  *height = h;
  *width = w;
}

void write_pgm(const std::string& path, size_t height, size_t width, const double* data, bool clamp) {
  std::vector<unsigned char> bytes(height * width);
  for (size_t i = 0; i < bytes.size(); ++i) {
    const double v = data[i];
    if (!std::isfinite(v)) fail(NDC_ERR_NUMERIC, "write_pgm: non-finite pixel");
    double r = std::nearbyint(v);  // round half to even (default rounding mode)
    if (clamp) {
      r = std::min(255.0, std::max(0.0, r));
    } else if (r < 0.0 || r > 255.0) {
      fail(NDC_ERR_NUMERIC, "write_pgm: pixel " + std::to_string(v) + " outside [0,255] and clamping is off");
    }
    bytes[i] = static_cast<unsigned char>(r);
  }
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) fail(NDC_ERR_FORMAT, "cannot open " + path + " for writing");
  const std::string hdr = "P5\n" + std::to_string(width) + " " + std::to_string(height) + "\n255\n";
  bool ok = std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size();
  ok = ok && std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) fail(NDC_ERR_FORMAT, "write_pgm: stream failure");
}

}  // namespace ndc
