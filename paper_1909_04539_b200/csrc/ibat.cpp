// IBAT batch files (reference batch.cpp:146-218, bandsolve.h:57-62): 24-byte
// little-endian header "IBAT", u32 version = 1, u64 n, u64 m, then n*m
// binary64 values in interleaved order. Byte-exact round trip; the
// reference's checks, in its order, with its statuses (io_error ->
// BANDSOLVE_ERR_IO, format_error -> BANDSOLVE_ERR_BAD_FORMAT).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.hpp"

namespace bsb {
namespace {
void put_u32_le(unsigned char* p, uint32_t v) {
  for (int k = 0; k < 4; ++k) p[k] = static_cast<unsigned char>(v >> (8 * k));
}
void put_u64_le(unsigned char* p, uint64_t v) {
  for (int k = 0; k < 8; ++k) p[k] = static_cast<unsigned char>(v >> (8 * k));
}
uint64_t get_le(const unsigned char* p, int bytes) {
  uint64_t v = 0;
  for (int k = bytes - 1; k >= 0; --k) v = (v << 8) | p[k];
  return v;
}
struct Closer {
  void operator()(FILE* f) const { std::fclose(f); }
};
using File = std::unique_ptr<FILE, Closer>;
}  // namespace

bandsolve_status ibat_write(const char* path, const double* data, std::size_t n, std::size_t m) {
  File f(std::fopen(path, "wb"));
  if (!f) return fail(BANDSOLVE_ERR_IO, std::string("cannot open for writing: ") + path);
  unsigned char header[24];
  std::memcpy(header, "IBAT", 4);
  put_u32_le(header + 4, 1);
  put_u64_le(header + 8, n);
  put_u64_le(header + 16, m);
  if (std::fwrite(header, 1, sizeof header, f.get()) != sizeof header)
    return fail(BANDSOLVE_ERR_IO, std::string("short write: ") + path);
  std::vector<unsigned char> payload(n * m * 8);
  for (std::size_t k = 0; k < n * m; ++k) {
    uint64_t bits;
    std::memcpy(&bits, data + k, 8);
    put_u64_le(payload.data() + 8 * k, bits);
  }
  if (std::fwrite(payload.data(), 1, payload.size(), f.get()) != payload.size())
    return fail(BANDSOLVE_ERR_IO, std::string("short write: ") + path);
  if (std::fflush(f.get()) != 0) return fail(BANDSOLVE_ERR_IO, std::string("flush failed: ") + path);
  return BANDSOLVE_OK;
}

bandsolve_status ibat_read(const char* path, std::size_t* n_out, std::size_t* m_out, double** data, bool* pinned) {
  *data = nullptr;
  File f(std::fopen(path, "rb"));
  if (!f) return fail(BANDSOLVE_ERR_IO, std::string("cannot open for reading: ") + path);
  unsigned char header[24];
  if (std::fread(header, 1, sizeof header, f.get()) != sizeof header)
    return fail(BANDSOLVE_ERR_BAD_FORMAT, std::string("truncated IBAT header: ") + path);
  if (std::memcmp(header, "IBAT", 4) != 0) return fail(BANDSOLVE_ERR_BAD_FORMAT, std::string("bad IBAT magic: ") + path);
  if (get_le(header + 4, 4) != 1) return fail(BANDSOLVE_ERR_BAD_FORMAT, std::string("unsupported IBAT version: ") + path);
  const uint64_t n = get_le(header + 8, 8), m = get_le(header + 16, 8);
  if (n == 0 || m == 0 || n > (1u << 28) || m > (1u << 28))
    return fail(BANDSOLVE_ERR_BAD_FORMAT, std::string("implausible IBAT shape: ") + path);
  // validate the payload size before allocating anything
  if (std::fseek(f.get(), 0, SEEK_END) != 0) return fail(BANDSOLVE_ERR_IO, std::string("seek failed: ") + path);
  const long size = std::ftell(f.get());
  if (size < 0 || static_cast<uint64_t>(size) != 24 + n * m * 8)
    return fail(BANDSOLVE_ERR_BAD_FORMAT, std::string("IBAT payload size mismatch: ") + path);
  if (std::fseek(f.get(), 24, SEEK_SET) != 0) return fail(BANDSOLVE_ERR_IO, std::string("seek failed: ") + path);
  double* out = host_alloc_zeroed(n * m, pinned);
  if (!out) return fail(BANDSOLVE_ERR_INTERNAL, "out of host memory");
  std::vector<unsigned char> payload(n * m * 8);
  if (std::fread(payload.data(), 1, payload.size(), f.get()) != payload.size()) {
    host_free(out, *pinned);
    return fail(BANDSOLVE_ERR_BAD_FORMAT, std::string("truncated IBAT payload: ") + path);
  }
  for (std::size_t k = 0; k < n * m; ++k) {
    const uint64_t bits = get_le(payload.data() + 8 * k, 8);
    std::memcpy(out + k, &bits, 8);
  }
  *n_out = n;
  *m_out = m;
  *data = out;
  return BANDSOLVE_OK;
}

}  // namespace bsb
