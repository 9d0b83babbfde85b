// Host-side helpers shared by the C-ABI translation units: status codes with
// a thread-local message, launch checking, dtype sizes.
#pragma once

#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/xquant.h"

namespace xq {

void set_error(const char* fmt, ...);

inline int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error("%s", buf);
  return status;
}

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(XQ_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return XQ_OK;
}

inline bool valid_bits(int bits) { return bits == 2 || bits == 3 || bits == 4 || bits == 8; }

inline int dtype_size(int dt) {
  switch (dt) {
    case XQ_F32: return 4;
    case XQ_BF16: return 2;
    case XQ_F16: return 2;
    case XQ_F64: return 8;
    default: return 0;
  }
}

inline int64_t row_bytes_for(int64_t cols, int bits) { return (cols * bits + 63) / 64 * 8; }

}  // namespace xq

#define XQ_REQUIRE(cond, status, ...)                  \
  do {                                                  \
    if (!(cond)) return ::xq::fail((status), __VA_ARGS__); \
  } while (0)
