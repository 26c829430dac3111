// skmx.cpp -- SKMX matrix files (core/include/streamk/matrix.hpp:70-93,
// core/src/matrix.cpp:13-61): a 16-byte little-endian header -- magic "SKMX",
// u32 dtype tag (DType: 0 int64, 1 float32, 2 float64; this library adds
// 3 bfloat16 and 4 float16 for device operands), u32 rows, u32 cols -- followed
// by the row-major payload.  Used to hand inputs/outputs of large device runs
// to the offline CPU oracle.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/skb200.h"

namespace {

thread_local std::string g_io_error;

size_t esize(int32_t t) {
  switch (t) {
    case SK_INT64: return 8;
    case SK_FLOAT32: return 4;
    case SK_FLOAT64: return 8;
    case SK_BFLOAT16: return 2;
    case SK_FLOAT16: return 2;
  }
  return 0;
}

void put_u32(unsigned char* p, uint32_t v) {
  p[0] = static_cast<unsigned char>(v & 0xff);
  p[1] = static_cast<unsigned char>((v >> 8) & 0xff);
  p[2] = static_cast<unsigned char>((v >> 16) & 0xff);
  p[3] = static_cast<unsigned char>((v >> 24) & 0xff);
}
uint32_t get_u32(const unsigned char* p) {
  return static_cast<uint32_t>(p[0]) | (static_cast<uint32_t>(p[1]) << 8) |
         (static_cast<uint32_t>(p[2]) << 16) | (static_cast<uint32_t>(p[3]) << 24);
}

struct File {
  FILE* f = nullptr;
  explicit File(FILE* x) : f(x) {}
  ~File() {
    if (f) fclose(f);
  }
};

}  // namespace

extern "C" {

const char* sk_io_error(void) { return g_io_error.c_str(); }

sk_status sk_save_matrix(const char* path, sk_dtype dtype, int64_t rows, int64_t cols,
                         const void* data) {
  const size_t es = esize(dtype);
  if (!path || es == 0 || rows < 0 || cols < 0 || rows > UINT32_MAX || cols > UINT32_MAX ||
      (rows * cols > 0 && !data))
    return SK_EINVAL;
  File f(fopen(path, "wb"));
  if (!f.f) {
    g_io_error = std::string("cannot write matrix file: ") + path;
    return SK_EIO;
  }
  unsigned char h[16];
  std::memcpy(h, "SKMX", 4);
  put_u32(h + 4, static_cast<uint32_t>(dtype));
  put_u32(h + 8, static_cast<uint32_t>(rows));
  put_u32(h + 12, static_cast<uint32_t>(cols));
  const size_t n = static_cast<size_t>(rows * cols);
  if (fwrite(h, 1, 16, f.f) != 16 || (n && fwrite(data, es, n, f.f) != n)) {
    g_io_error = "matrix file: short write";
    return SK_EIO;
  }
  return SK_OK;
}

sk_status sk_load_matrix_header(const char* path, sk_dtype* dtype, int64_t* rows, int64_t* cols) {
  if (!path) return SK_EINVAL;
  File f(fopen(path, "rb"));
  if (!f.f) {
    g_io_error = std::string("cannot read matrix file: ") + path;
    return SK_EIO;
  }
  unsigned char h[16];
  if (fread(h, 1, 16, f.f) != 16) {
    g_io_error = "matrix file: truncated header";
    return SK_EIO;
  }
  if (std::memcmp(h, "SKMX", 4) != 0) {
    g_io_error = "matrix file: bad magic";
    return SK_EIO;
  }
  if (dtype) *dtype = static_cast<sk_dtype>(get_u32(h + 4));
  if (rows) *rows = get_u32(h + 8);
  if (cols) *cols = get_u32(h + 12);
  return SK_OK;
}

// matrix.hpp:86-93 load_matrix<T>: the dtype tag must equal `expect`; rows/cols
// must match the caller's buffer.
sk_status sk_load_matrix(const char* path, sk_dtype expect, int64_t rows, int64_t cols, void* data) {
  sk_dtype tag;
  int64_t r, c;
  sk_status st = sk_load_matrix_header(path, &tag, &r, &c);
  if (st) return st;
  if (tag != expect) {
    g_io_error = "matrix file: dtype tag " + std::to_string(static_cast<int>(tag)) +
                 ", expected " + std::to_string(static_cast<int>(expect));
    return SK_EIO;
  }
  if (r != rows || c != cols) {
    g_io_error = "matrix file: shape " + std::to_string(r) + "x" + std::to_string(c) +
                 " differs from the buffer";
    return SK_EINVAL;
  }
  File f(fopen(path, "rb"));
  if (!f.f || fseek(f.f, 16, SEEK_SET) != 0) {
    g_io_error = "matrix file: reopen failed";
    return SK_EIO;
  }
  const size_t n = static_cast<size_t>(rows * cols), es = esize(expect);
  if (n && fread(data, es, n, f.f) != n) {
    g_io_error = "matrix file: truncated payload";
    return SK_EIO;
  }
  return SK_OK;
}

}  // extern "C"
