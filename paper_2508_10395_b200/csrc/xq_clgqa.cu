// xq-cl-gqa decode append (DeltaLatentCacheGQA, cache.py:538-589) at the new
// tokens, in float64 like the reference so its per-channel codes are the
// reference's:
//
//   k_latent64      lat[b] = (x[b] - acc_row[b]) @ U   (delta layers; x @ U for
//                   base layers, cache.py:562-586), written into row pos_b of
//                   slot b's residual buffer (float64 + its float32 mirror);
//   k_row64_update  acc_row[b] (+)= rec[b] @ U^T       (Accumulator.seed / add
//                   of the new token's reconstruction, cache.py:571-572, 588-589)
//
// Both are GEMVs over U (d x r) with a handful of rows: HBM-bound on U
// (float32 or float64 storage, float64 arithmetic), deterministic fixed-order
// reductions. The full-width accumulator of all cached rows (the remat
// operand) is rebuilt by the tcgen05 remat GEMM (xq_gemm.cu).

#include "xq_common.cuh"
#include "xq_host.h"

namespace xq {
namespace {

constexpr int kL64Cols = 32;      // columns of U per CTA (one per lane)
constexpr int kL64Warps = 16;     // d split over the warps of a CTA
constexpr int kL64Rows = 8;       // rows (slots) per pass (32 KB of static staging)

XQ_DEVINL double load_f64(const void* base, int dt, int64_t i) {
  switch (dt) {
    case XQ_F32: return static_cast<double>(static_cast<const float*>(base)[i]);
    case XQ_BF16: return static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(base)[i]));
    case XQ_F16: return static_cast<double>(__half2float(static_cast<const __half*>(base)[i]));
    default: return static_cast<const double*>(base)[i];
  }
}

template <typename UT>
__global__ void __launch_bounds__(kL64Warps * 32)
    k_latent64(const void* __restrict__ x, int x_dt, int64_t x_stride, int n_rows, int64_t d,
               const double* __restrict__ sub, const UT* __restrict__ u, int64_t r,
               const int32_t* __restrict__ lens, const int32_t* __restrict__ nflushed,
               int64_t G, double* __restrict__ resid64, float* __restrict__ resid32,
               int32_t* __restrict__ flag) {
  __shared__ double xs[kL64Warps][kL64Rows][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * kL64Cols + lane;
  const bool col_ok = col < r;
  const int64_t per_warp = (d + kL64Warps - 1) / kL64Warps;
  const int64_t k_lo = warp * per_warp, k_hi = min(d, k_lo + per_warp);
  for (int b0 = 0; b0 < n_rows; b0 += kL64Rows) {
    const int nb = min(kL64Rows, n_rows - b0);
    double acc[kL64Rows];
#pragma unroll
    for (int i = 0; i < kL64Rows; ++i) acc[i] = 0.0;
    for (int64_t k0 = k_lo; k0 < k_hi; k0 += 32) {
      // stage (x - sub)[b0.., k0 + lane] of this warp's 32 rows of d
      const int64_t kk = k0 + lane;
#pragma unroll
      for (int i = 0; i < kL64Rows; ++i) {
        double v = 0.0;
        if (i < nb && kk < k_hi) {
          v = load_f64(x, x_dt, static_cast<int64_t>(b0 + i) * x_stride + kk);
          if (sub) v = __dsub_rn(v, sub[static_cast<int64_t>(b0 + i) * d + kk]);
        }
        xs[warp][i][lane] = v;
      }
      __syncwarp();
      const int64_t left = k_hi - k0;
      const int kn = left < 32 ? static_cast<int>(left) : 32;
      for (int j = 0; j < kn; ++j) {
        const double uv = col_ok ? static_cast<double>(u[(k0 + j) * r + col]) : 0.0;
#pragma unroll
        for (int i = 0; i < kL64Rows; ++i) acc[i] = __fma_rn(xs[warp][i][j], uv, acc[i]);
      }
      __syncwarp();
    }
    // fixed-order reduction over the warps: xs reused as [warp][row][lane]
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kL64Rows; ++i) xs[warp][i][lane] = acc[i];
    __syncthreads();
    if (warp < nb && col_ok) {
      const int i = warp, b = b0 + i;
      double s = 0.0;
      for (int w = 0; w < kL64Warps; ++w) s = __dadd_rn(s, xs[w][i][lane]);
      if (!isfinite(s)) atomicExch(flag, 1);
      const int64_t pos = lens[b] - 1 - nflushed[b];
      const int64_t o = (static_cast<int64_t>(b) * G + pos) * r + col;
      resid64[o] = s;
      resid32[o] = static_cast<float>(s);
    }
    __syncthreads();
  }
}

// acc_row[b][k] (+)= sum_j rec[b][j] * U[k][j]; rec[b] = row pos_b of slot b's
// float64 residual buffer (the new token's reconstruction). Warp per row k of U; up
// to kL64Rows slots per pass share each U element (independent FMA chains), fixed
// summation order per (b, k).
template <typename UT>
__global__ void __launch_bounds__(256)
    k_row64_update(const double* __restrict__ resid64, const int32_t* __restrict__ rec_pos,
                   int n_rows, int64_t G, const UT* __restrict__ u, int64_t d, int64_t r,
                   int seed, double* __restrict__ acc_row) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t k = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (k >= d) return;
  const UT* urow = u + k * r;
  for (int b0 = 0; b0 < n_rows; b0 += kL64Rows) {
    const int nb = min(kL64Rows, n_rows - b0);
    const double* rec[kL64Rows];
    double s[kL64Rows];
#pragma unroll
    for (int i = 0; i < kL64Rows; ++i) {
      rec[i] = resid64 + (static_cast<int64_t>(b0 + (i < nb ? i : 0)) * G + rec_pos[b0 + (i < nb ? i : 0)]) * r;
      s[i] = 0.0;
    }
    for (int64_t j = lane; j < r; j += 32) {
      const double uv = static_cast<double>(urow[j]);
#pragma unroll
      for (int i = 0; i < kL64Rows; ++i)
        if (i < nb) s[i] = __fma_rn(rec[i][j], uv, s[i]);
    }
#pragma unroll
    for (int i = 0; i < kL64Rows; ++i) {
      if (i >= nb) break;
      double v = s[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0) {
        double* a = acc_row + static_cast<int64_t>(b0 + i) * d + k;
        *a = seed ? v : __dadd_rn(*a, v);
      }
    }
  }
}

}  // namespace
}  // namespace xq

using namespace xq;

extern "C" int xq_clgqa_latent64(const void* x, int32_t x_dtype, int64_t x_row_stride,
                                 int32_t n_rows, int64_t d, const double* acc_row,
                                 const void* u, int32_t u_dtype, int64_t r,
                                 const int32_t* seq_lens, const int32_t* nflushed,
                                 int32_t group_size, double* resid64, float* resid32,
                                 int32_t* nonfinite_flag, void* stream) {
  XQ_REQUIRE(u_dtype == XQ_F32 || u_dtype == XQ_F64, XQ_ECONFIG, "U must be float32 or float64");
  XQ_REQUIRE(dtype_size(x_dtype) > 0, XQ_ECONFIG, "unknown x dtype");
  XQ_REQUIRE(seq_lens && nflushed && resid64 && resid32 && nonfinite_flag, XQ_EUSAGE, "null argument");
  if (n_rows == 0) return XQ_OK;
  const unsigned grid = static_cast<unsigned>((r + kL64Cols - 1) / kL64Cols);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (u_dtype == XQ_F32)
    k_latent64<float><<<grid, kL64Warps * 32, 0, st>>>(x, x_dtype, x_row_stride, n_rows, d, acc_row,
                                                       static_cast<const float*>(u), r, seq_lens,
                                                       nflushed, group_size, resid64, resid32,
                                                       nonfinite_flag);
  else
    k_latent64<double><<<grid, kL64Warps * 32, 0, st>>>(x, x_dtype, x_row_stride, n_rows, d, acc_row,
                                                        static_cast<const double*>(u), r, seq_lens,
                                                        nflushed, group_size, resid64, resid32,
                                                        nonfinite_flag);
  return check_launch("k_latent64");
}

extern "C" int xq_clgqa_row_update(const double* resid64, const int32_t* rec_pos, int32_t n_rows,
                                   int32_t group_size, const void* u, int32_t u_dtype, int64_t d,
                                   int64_t r, int32_t seed, double* acc_row, void* stream) {
  XQ_REQUIRE(u_dtype == XQ_F32 || u_dtype == XQ_F64, XQ_ECONFIG, "U must be float32 or float64");
  XQ_REQUIRE(resid64 && rec_pos && acc_row, XQ_EUSAGE, "null argument");
  if (n_rows == 0) return XQ_OK;
  const unsigned grid = static_cast<unsigned>((d + 7) / 8);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (u_dtype == XQ_F32)
    k_row64_update<float><<<grid, 256, 0, st>>>(resid64, rec_pos, n_rows, group_size,
                                                static_cast<const float*>(u), d, r, seed, acc_row);
  else
    k_row64_update<double><<<grid, 256, 0, st>>>(resid64, rec_pos, n_rows, group_size,
                                                 static_cast<const double*>(u), d, r, seed, acc_row);
  return check_launch("k_row64_update");
}
