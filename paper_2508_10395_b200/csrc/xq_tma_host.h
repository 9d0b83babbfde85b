// Host-side TMA tensor-map helper shared by the newer translation units
// (cuTensorMapEncodeTiled resolved through the runtime's driver entry point,
// so the library links against cudart only).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "xq_host.h"

namespace xq {

inline PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 2-D map over a row-major [rows][inner] tensor, box = [box_rows][box_inner].
inline int tma_map_2d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base,
                      uint64_t inner, uint64_t rows, uint64_t row_pitch_bytes, uint32_t box_inner,
                      uint32_t box_rows, CUtensorMapSwizzle sw, const char* what) {
  auto enc = tma_encode_fn();
  XQ_REQUIRE(enc != nullptr, XQ_ECUDA, "cuTensorMapEncodeTiled unavailable");
  XQ_REQUIRE(reinterpret_cast<uintptr_t>(base) % 16 == 0, XQ_ESHAPE,
             "%s: base not 16-byte aligned", what);
  XQ_REQUIRE(row_pitch_bytes % 16 == 0, XQ_ESHAPE, "%s: row pitch %llu B not a multiple of 16",
             what, (unsigned long long)row_pitch_bytes);
  const cuuint64_t gdim[2] = {inner, rows};
  const cuuint64_t gstride[1] = {row_pitch_bytes};
  const cuuint32_t box[2] = {box_inner, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  XQ_REQUIRE(r == CUDA_SUCCESS, XQ_ECUDA, "%s: cuTensorMapEncodeTiled failed (%d)", what, (int)r);
  return XQ_OK;
}

}  // namespace xq
