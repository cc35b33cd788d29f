// IBAT batch files (the reference's interchange format, batch.cpp:146-218,
// bandsolve.h:57-62). Layout: a 24-byte little-endian header — the tag
// "IBAT", a u32 format version (1), u64 rows n, u64 systems m — followed by
// n*m IEEE binary64 values in the interleaved order x[i*m + j].
//
// Statuses follow the reference's classification: anything the file system
// refuses is BANDSOLVE_ERR_IO; anything wrong with the bytes (short header,
// wrong tag or version, an empty or absurd shape, a payload of the wrong
// length) is BANDSOLVE_ERR_BAD_FORMAT. The payload length is checked against
// the header before the batch is allocated, so a corrupt header cannot make
// the reader allocate gigabytes. Values are streamed in blocks straight
// into (or out of) the page-locked batch buffer.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.hpp"

namespace bsb {
namespace {

constexpr std::size_t kHeaderBytes = 24;
constexpr uint32_t kVersion = 1;
constexpr uint64_t kMaxDim = uint64_t{1} << 28;  // per dimension; rejects garbage shapes
constexpr std::size_t kBlockValues = 1 << 16;    // values per fread / fwrite

struct Header {
  uint64_t n = 0, m = 0;
  uint32_t version = 0;
  bool tag_ok = false;
};

// little-endian field codec, independent of the host's byte order
template <typename U>
void store_le(unsigned char* dst, U v) {
  for (std::size_t k = 0; k < sizeof(U); ++k) dst[k] = static_cast<unsigned char>(v >> (8 * k));
}
template <typename U>
U load_le(const unsigned char* src) {
  U v = 0;
  for (std::size_t k = sizeof(U); k-- > 0;) v = static_cast<U>((v << 8) | src[k]);
  return v;
}

void encode_header(unsigned char (&h)[kHeaderBytes], uint64_t n, uint64_t m) {
  std::memcpy(h, "IBAT", 4);
  store_le<uint32_t>(h + 4, kVersion);
  store_le<uint64_t>(h + 8, n);
  store_le<uint64_t>(h + 16, m);
}

Header decode_header(const unsigned char (&h)[kHeaderBytes]) {
  Header d;
  d.tag_ok = std::memcmp(h, "IBAT", 4) == 0;
  d.version = load_le<uint32_t>(h + 4);
  d.n = load_le<uint64_t>(h + 8);
  d.m = load_le<uint64_t>(h + 16);
  return d;
}

// one binary64 value <-> its 8 little-endian bytes
void value_to_le(unsigned char* dst, double v) {
  uint64_t bits;
  std::memcpy(&bits, &v, sizeof bits);
  store_le<uint64_t>(dst, bits);
}
double value_from_le(const unsigned char* src) {
  const uint64_t bits = load_le<uint64_t>(src);
  double v;
  std::memcpy(&v, &bits, sizeof v);
  return v;
}

class FileHandle {
 public:
  FileHandle(const char* path, const char* mode) : f_(std::fopen(path, mode)) {}
  ~FileHandle() {
    if (f_) std::fclose(f_);
  }
  FileHandle(const FileHandle&) = delete;
  FileHandle& operator=(const FileHandle&) = delete;
  FILE* get() const { return f_; }
  explicit operator bool() const { return f_ != nullptr; }

 private:
  FILE* f_;
};

bandsolve_status io_error(const char* what, const char* path) {
  return fail(BANDSOLVE_ERR_IO, std::string(what) + " '" + path + "'");
}
bandsolve_status format_error(const char* what, const char* path) {
  return fail(BANDSOLVE_ERR_BAD_FORMAT, std::string("IBAT file '") + path + "': " + what);
}

}  // namespace

bandsolve_status ibat_write(const char* path, const double* data, std::size_t n, std::size_t m) {
  FileHandle f(path, "wb");
  if (!f) return io_error("could not create", path);
  unsigned char header[kHeaderBytes];
  encode_header(header, n, m);
  if (std::fwrite(header, 1, kHeaderBytes, f.get()) != kHeaderBytes) return io_error("write failed on", path);
  const std::size_t total = n * m;
  std::vector<unsigned char> block(8 * std::min(total, kBlockValues));
  for (std::size_t k0 = 0; k0 < total; k0 += kBlockValues) {
    const std::size_t cnt = std::min(kBlockValues, total - k0);
    for (std::size_t k = 0; k < cnt; ++k) value_to_le(block.data() + 8 * k, data[k0 + k]);
    if (std::fwrite(block.data(), 8, cnt, f.get()) != cnt) return io_error("write failed on", path);
  }
  if (std::fflush(f.get()) != 0) return io_error("could not flush", path);
  return BANDSOLVE_OK;
}

bandsolve_status ibat_read(const char* path, std::size_t* n_out, std::size_t* m_out, double** data, bool* pinned) {
  *data = nullptr;
  FileHandle f(path, "rb");
  if (!f) return io_error("could not open", path);
  unsigned char header[kHeaderBytes];
  if (std::fread(header, 1, kHeaderBytes, f.get()) != kHeaderBytes) return format_error("header cut short", path);
  const Header h = decode_header(header);
  if (!h.tag_ok) return format_error("not an IBAT file (tag)", path);
  if (h.version != kVersion) return format_error("format version is not 1", path);
  if (h.n == 0 || h.m == 0 || h.n > kMaxDim || h.m > kMaxDim) return format_error("shape out of range", path);
  // the file length must be exactly header + payload: checked before allocating
  if (std::fseek(f.get(), 0, SEEK_END) != 0) return io_error("could not seek in", path);
  const long length = std::ftell(f.get());
  const uint64_t expect = kHeaderBytes + h.n * h.m * 8;
  if (length < 0 || static_cast<uint64_t>(length) != expect) return format_error("payload length != n*m*8", path);
  if (std::fseek(f.get(), static_cast<long>(kHeaderBytes), SEEK_SET) != 0) return io_error("could not seek in", path);

  const std::size_t total = h.n * h.m;
  double* out = host_alloc_zeroed(total, pinned);
  if (!out) return fail(BANDSOLVE_ERR_INTERNAL, "out of host memory");
  std::vector<unsigned char> block(8 * std::min(total, kBlockValues));
  for (std::size_t k0 = 0; k0 < total; k0 += kBlockValues) {
    const std::size_t cnt = std::min(kBlockValues, total - k0);
    if (std::fread(block.data(), 8, cnt, f.get()) != cnt) {
      host_free(out, *pinned);
      return format_error("payload cut short", path);
    }
    for (std::size_t k = 0; k < cnt; ++k) out[k0 + k] = value_from_le(block.data() + 8 * k);
  }
  *n_out = h.n;
  *m_out = h.m;
  *data = out;
  return BANDSOLVE_OK;
}

}  // namespace bsb
