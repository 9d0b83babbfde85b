// Host-side helpers shared by the C-ABI translation units: status codes with
// a thread-local message, launch checking, dtype sizes.
#pragma once

#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include <mutex>
#include <unordered_map>

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

// cudaFuncAttributeMaxDynamicSharedMemorySize is per (kernel, device): one
// process may drive several GPUs (Decoder(device=...)), so the "already raised"
// record is keyed by both, under a lock.
// (Always set: a kernel's static shared memory counts against the default 48 KB.)
inline int ensure_smem(const void* kern, size_t bytes, const char* what) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = reinterpret_cast<uint64_t>(kern) * 64 + static_cast<uint64_t>(dev & 63);
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return XQ_OK;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(bytes)) != cudaSuccess)
    return check_launch(what);
  done[key] = bytes;
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
