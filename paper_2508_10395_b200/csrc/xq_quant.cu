// Quantizer, bit packing, arena append/dequant, RoPE table, weight
// arrangement and the XQuant-CL accumulator -- sm_100a.
//
// Arithmetic contract (bit-exact with the reference quantizer,
// _native.pyx:111-153 / fallback.py:108-131): group min/max on the exactly
// upcast float64 inputs, scale = (max-min)/(2^e-1) (1.0 for a degenerate
// group), code = clamp(floor((x-min)/scale + 0.5), 0, 2^e-1), every step an
// IEEE float64 op with explicit rounding intrinsics so nvcc cannot contract.
#include <math.h>

#include "xq_common.cuh"
#include "xq_host.h"
#include "xq_layout.cuh"

namespace xq {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// ------------------------------------------------------------------ device

XQ_DEVINL double load_as_f64(const void* base, int dt, int64_t i) {
  switch (dt) {
    case XQ_F32: return static_cast<double>(static_cast<const float*>(base)[i]);
    case XQ_BF16:
      return static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(base)[i]));
    case XQ_F16: return static_cast<double>(__half2float(static_cast<const __half*>(base)[i]));
    default: return static_cast<const double*>(base)[i];
  }
}

XQ_DEVINL double shfl_xor_d(double v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }

// Quantize one row (block-cooperative: warps over groups, lanes over
// elements). Codes land in `codes_out` (shared or global bytes); the group
// parameters are handed to `sink(g, scale, zp)` by lane 0 of the owning warp.
// XQuant-CL running row (`acc`, float64): with `acc_mode` 1 the quantized value
// is x - acc and the row then becomes acc + code*scale + zp (cache.py:478-481
// with Accumulator.add, cache.py:139-146); with `acc_mode` 2 (the seeding base
// layer, cache.py:463-467) it becomes code*scale + zp. The reconstruction is the
// reference's float64 dequantize (fallback.py:134-146: one multiply, one add),
// so every later delta is formed exactly as the reference forms it.
template <class Sink>
__device__ void quantize_row(const void* x, int dt, int64_t x_off, int64_t cols, int G, int bits,
                             const float* sub, uint8_t* codes_out, double* x_eff, int* bad,
                             Sink sink, double* acc = nullptr, int acc_mode = 0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int64_t ngroups = (cols + G - 1) / G;
  const double qmax = static_cast<double>((1 << bits) - 1);
  for (int64_t g = warp; g < ngroups; g += nw) {
    const int64_t lo = g * G;
    const int64_t hi = min(lo + G, cols);
    double mn = INFINITY, mx = -INFINITY;
    bool finite = true;
    for (int64_t j = lo + lane; j < hi; j += 32) {
      double v = load_as_f64(x, dt, x_off + j);
      if (sub) v = __dsub_rn(v, static_cast<double>(sub[j]));
      if (acc_mode == 1) v = __dsub_rn(v, acc[j]);
      finite &= isfinite(v);
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, shfl_xor_d(mn, o));
      mx = fmax(mx, shfl_xor_d(mx, o));
    }
    if (!__all_sync(0xffffffffu, finite) && lane == 0) *bad = 1;
    const double span = __dsub_rn(mx, mn);
    const double scale = (span == 0.0) ? 1.0 : __ddiv_rn(span, qmax);
    if (lane == 0) sink(g, scale, mn);
    for (int64_t j = lo + lane; j < hi; j += 32) {
      double v = load_as_f64(x, dt, x_off + j);
      if (sub) v = __dsub_rn(v, static_cast<double>(sub[j]));
      const double a = acc_mode == 1 ? acc[j] : 0.0;
      if (acc_mode == 1) v = __dsub_rn(v, a);
      double q = floor(__dadd_rn(__ddiv_rn(__dsub_rn(v, mn), scale), 0.5));
      q = q < 0.0 ? 0.0 : (q > qmax ? qmax : q);
      codes_out[j] = static_cast<uint8_t>(q);
      if (x_eff) x_eff[j] = v;
      if (acc_mode) {
        const double r = __dadd_rn(__dmul_rn(q, scale), mn);
        acc[j] = acc_mode == 1 ? __dadd_rn(a, r) : r;
      }
    }
  }
}

// 32-bit word w of the LSB-first stream of `n` codes of `bits` bits.
XQ_DEVINL uint32_t stream_word32(const uint8_t* codes, int64_t n, int bits, int64_t w) {
  const int64_t b0 = w * 32;
  int64_t i0 = b0 / bits;
  int64_t i1 = (b0 + 31) / bits;
  if (i1 > n - 1) i1 = n - 1;
  uint32_t word = 0;
  for (int64_t i = i0; i <= i1; ++i) {
    const int64_t off = i * bits - b0;
    const uint32_t c = codes[i];
    word |= off >= 0 ? (c << off) : (c >> (-off));
  }
  return word;
}

__global__ void k_quantize_groups(const double* __restrict__ x, int64_t cols, int G, int bits,
                                  uint8_t* __restrict__ codes, double* __restrict__ scales,
                                  double* __restrict__ zps) {
  const int64_t r = blockIdx.x;
  const int64_t ng = (cols + G - 1) / G;
  int bad = 0;
  quantize_row(x, XQ_F64, r * cols, cols, G, bits, nullptr, codes + r * cols, nullptr, &bad,
               [&](int64_t g, double s, double z) {
                 scales[r * ng + g] = s;
                 zps[r * ng + g] = z;
               });
}

__global__ void k_dequantize_groups(const uint8_t* __restrict__ codes,
                                    const double* __restrict__ scales,
                                    const double* __restrict__ zps, int64_t rows, int64_t cols,
                                    int G, double* __restrict__ out) {
  const int64_t ng = (cols + G - 1) / G;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * cols;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const int64_t p = r * ng + c / G;
    out[i] = __dadd_rn(__dmul_rn(static_cast<double>(codes[i]), scales[p]), zps[p]);
  }
}

__global__ void k_pack(const uint8_t* __restrict__ codes, int64_t n, int bits,
                       uint64_t* __restrict__ words, int64_t n_words) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_words;
       w += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t lo = stream_word32(codes, n, bits, 2 * w);
    const uint64_t hi = stream_word32(codes, n, bits, 2 * w + 1);
    words[w] = lo | (hi << 32);
  }
}

__global__ void k_unpack(const uint64_t* __restrict__ words, int bits, int64_t n,
                         uint8_t* __restrict__ codes) {
  const uint64_t mask = (1ull << bits) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t off = static_cast<uint64_t>(i) * bits;
    const int64_t w = off >> 6;
    const int s = off & 63;
    uint64_t v = words[w] >> s;
    if (s + bits > 64) v |= words[w + 1] << (64 - s);
    codes[i] = static_cast<uint8_t>(v & mask);
  }
}

__global__ void k_quantize_rows(const void* __restrict__ x, int dt, int64_t x_stride,
                                int64_t cols, int G, int bits, const int32_t* __restrict__ lens,
                                int64_t row0, int64_t L_max, const float* __restrict__ sub_rows,
                                uint8_t* __restrict__ codes, int64_t row_bytes,
                                __half2* __restrict__ params, double* __restrict__ x_eff,
                                int32_t* __restrict__ flag, double* __restrict__ acc = nullptr,
                                int acc_mode = 0) {
  extern __shared__ uint8_t s_codes[];
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  const int64_t i = blockIdx.x;
  const int64_t dst = lens ? i * L_max + (lens[i] - 1) : row0 + i;
  const int64_t ng = param_stride(cols, G);
  int bad = 0;
  quantize_row(x, dt, i * x_stride, cols, G, bits, sub_rows ? sub_rows + dst * cols : nullptr,
               s_codes, x_eff ? x_eff + i * cols : nullptr, &bad,
               [&](int64_t g, double s, double z) {
                 params[dst * ng + g] = __halves2half2(__double2half(s), __double2half(z));
               },
               acc ? acc + i * cols : nullptr, acc_mode);
  if (bad) s_bad = 1;
  __syncthreads();
  uint32_t* out = reinterpret_cast<uint32_t*>(codes + dst * row_bytes);
  for (int64_t w = threadIdx.x; w < row_bytes / 4; w += blockDim.x)
    out[w] = stream_word32(s_codes, cols, bits, w);
  if (threadIdx.x == 0 && s_bad && flag) atomicExch(flag, 1);
}

// One CTA per (block, 32-channel slice): per-channel min/max over the G rows.
template <typename T>
__global__ void k_quantize_blocks_per_channel(const T* __restrict__ blocks, int64_t cols,
                                              int bits, int G, const int64_t* __restrict__ dst0,
                                              uint8_t* __restrict__ codes, int64_t row_bytes,
                                              __half* __restrict__ params,
                                              int32_t* __restrict__ flag,
                                              double* __restrict__ recon = nullptr) {
  extern __shared__ uint8_t s_codes[];  // [G][32]
  __shared__ double s_mn[4][32], s_mx[4][32];
  __shared__ double s_scale[32], s_zp[32];
  __shared__ int s_bad;
  const int b = blockIdx.x, slice = blockIdx.y;
  const int c = threadIdx.x & 31, part = threadIdx.x >> 5;
  const int64_t ch = (int64_t)slice * 32 + c;
  const T* blk = blocks + (int64_t)b * G * cols;
  if (threadIdx.x == 0) s_bad = 0;
  double mn = INFINITY, mx = -INFINITY;
  bool finite = true;
  for (int r = part; r < G; r += 4) {
    const double v = static_cast<double>(blk[(int64_t)r * cols + ch]);
    finite &= isfinite(v);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  s_mn[part][c] = mn;
  s_mx[part][c] = mx;
  __syncthreads();
  if (!finite) s_bad = 1;
  const double qmax = static_cast<double>((1 << bits) - 1);
  if (part == 0) {
    for (int p = 1; p < 4; ++p) {
      mn = fmin(mn, s_mn[p][c]);
      mx = fmax(mx, s_mx[p][c]);
    }
    const double span = __dsub_rn(mx, mn);
    const double scale = (span == 0.0) ? 1.0 : __ddiv_rn(span, qmax);
    s_scale[c] = scale;
    s_zp[c] = mn;
    // planar [token group][2][cols] halves in producer channel order (xq_layout.cuh)
    const int bs = perm_block(XQ_A_CODES_CHANNEL, bits);
    const int64_t pos = (int64_t)slice * 32 + (c / bs) * bs + perm_position(c % bs, bs);
    __half* prow = params + (dst0[b] / G) * 2 * cols;
    prow[pos] = __double2half(scale);
    prow[cols + pos] = __double2half(mn);
  }
  __syncthreads();
  const double scale = s_scale[c], zp = s_zp[c];
  for (int r = part; r < G; r += 4) {
    const double v = static_cast<double>(blk[(int64_t)r * cols + ch]);
    double q = floor(__dadd_rn(__ddiv_rn(__dsub_rn(v, zp), scale), 0.5));
    q = q < 0.0 ? 0.0 : (q > qmax ? qmax : q);
    s_codes[r * 32 + c] = static_cast<uint8_t>(q);
    // the reference's float64 reconstruction (fallback.py:134-146), may alias blocks
    if (recon) recon[(int64_t)b * G * cols + (int64_t)r * cols + ch] = __dadd_rn(__dmul_rn(q, scale), zp);
  }
  __syncthreads();
  // row r of this slice: 32 codes -> `bits` 32-bit words at byte 4*bits*slice
  for (int idx = threadIdx.x; idx < G * bits; idx += blockDim.x) {
    const int r = idx / bits, w = idx % bits;
    uint32_t* out = reinterpret_cast<uint32_t*>(codes + (dst0[b] + r) * row_bytes +
                                                (int64_t)slice * 4 * bits);
    out[w] = stream_word32(s_codes + r * 32, 32, bits, w);
  }
  if (threadIdx.x == 0 && s_bad && flag) atomicExch(flag, 1);
}

XQ_DEVINL uint32_t read_code(const uint8_t* row, int64_t c, int bits) {
  const int64_t off = c * bits;
  const int64_t byte = off >> 3;
  const int sh = off & 7;
  uint32_t v = row[byte];
  if (sh + bits > 8) v |= static_cast<uint32_t>(row[byte + 1]) << 8;
  return (v >> sh) & ((1u << bits) - 1);
}

// (scale, zp) of element (arena row r, channel c): per-token half2 grid, or the
// planar permuted per-channel layout written by k_quantize_blocks_per_channel.
XQ_DEVINL float2 load_params(const void* params, int axis, int bits, int G, int64_t cols,
                             int64_t r, int64_t c) {
  if (axis == 0) {
    const int64_t ng = param_stride(cols, G);
    const __half2 p = static_cast<const __half2*>(params)[r * ng + c / G];
    return make_float2(__low2float(p), __high2float(p));
  }
  const int bs = perm_block(XQ_A_CODES_CHANNEL, bits);
  const int64_t pos = (c / bs) * bs + perm_position(static_cast<int>(c % bs), bs);
  const __half* prow = static_cast<const __half*>(params) + (r / G) * 2 * cols;
  return make_float2(__half2float(prow[pos]), __half2float(prow[cols + pos]));
}

__global__ void k_dequant_rows(const uint8_t* __restrict__ codes, int64_t row_bytes,
                               const void* __restrict__ params, int axis, int bits, int G,
                               int64_t cols, int64_t row0, int64_t n_rows,
                               float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows * cols;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = row0 + i / cols, c = i % cols;
    const uint32_t code = read_code(codes + r * row_bytes, c, bits);
    const float2 p = load_params(params, axis, bits, G, cols, r, c);
    out[i] = fmaf(static_cast<float>(code), p.x, p.y);
  }
}

// fp16 operand rows for the remat GEMM: arena rows row0.. (codes) then, from
// row n_codes on, the float32 residual rows (per-channel streams, cache.py:223-230)
__global__ void k_dequant_rows_f16(const uint8_t* __restrict__ codes, int64_t row_bytes,
                                   const void* __restrict__ params, int axis, int bits, int G,
                                   int64_t cols, int64_t row0, int64_t n_codes,
                                   const float* __restrict__ resid, int64_t n_rows,
                                   __half* __restrict__ out, int64_t ldo) {
  // one thread = 8 consecutive channels of one row (16-byte store): the 8*bits
  // code bits are at most 3 bytes apart from a 4-byte aligned window pair
  const int64_t chunks = cols / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows * chunks;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / chunks, c0 = (i % chunks) * 8;
    float v[8];
    if (r < n_codes) {
      const int64_t ar = row0 + r;
      const uint8_t* row = codes + ar * row_bytes;
      const int64_t bit0 = c0 * bits;
      const int64_t w0 = bit0 >> 5;
      const uint32_t* wrow = reinterpret_cast<const uint32_t*>(row);
      const int64_t n_words = row_bytes / 4;
      const uint64_t lo = wrow[w0];
      const uint64_t hi = (w0 + 1 < n_words) ? wrow[w0 + 1] : 0u;
      uint64_t win = (lo | (hi << 32)) >> (bit0 & 31);
      if (axis == 0) {
        const __half2 p = static_cast<const __half2*>(params)[ar * param_stride(cols, G) + c0 / G];
        const float sc = __low2float(p), zp = __high2float(p);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = fmaf(static_cast<float>((win >> (j * bits)) & ((1u << bits) - 1)), sc, zp);
      } else {
        const int bs = perm_block(XQ_A_CODES_CHANNEL, bits);
        const __half* prow = static_cast<const __half*>(params) + (ar / G) * 2 * cols;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int64_t c = c0 + j;
          const int64_t pos = (c / bs) * bs + perm_position(static_cast<int>(c % bs), bs);
          v[j] = fmaf(static_cast<float>((win >> (j * bits)) & ((1u << bits) - 1)),
                      __half2float(prow[pos]), __half2float(prow[cols + pos]));
        }
      }
    } else {
      const float4* rr = reinterpret_cast<const float4*>(resid + (r - n_codes) * cols + c0);
      const float4 a = rr[0], b = rr[1];
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
    uint4 o;
    __half2* oh = reinterpret_cast<__half2*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) oh[j] = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
    *reinterpret_cast<uint4*>(out + r * ldo + c0) = o;
  }
}

// The same for 2/3/4/8-bit codes, specialised: a thread owns 8 channels of kRowsPerBlk
// consecutive rows (one 16-byte store per row, coalesced across the warp); per-channel
// (scale, zp) are loaded once per thread, the rows of a block lie in one 128-token group.
constexpr int kRowsPerBlk = 32;
template <int BITS, int AXIS>
__global__ void __launch_bounds__(128) k_dequant_rows_f16_t(
    const uint8_t* __restrict__ codes, int64_t row_bytes, const void* __restrict__ params, int G,
    int cols, int64_t row0, int n_codes, const float* __restrict__ resid, int n_rows,
    __half* __restrict__ out, int64_t ldo) {
  constexpr uint32_t kMask = (1u << BITS) - 1u;
  const int c0 = 8 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (c0 >= cols) return;
  const int r_lo = blockIdx.y * kRowsPerBlk;
  const int r_hi = min(n_rows, r_lo + kRowsPerBlk);
  float2 pc[8];
  if (AXIS == 1 && r_lo < n_codes) {  // per-channel (scale, zp) of the block's token group
    constexpr int BS = BITS == 2 ? 16 : BITS == 3 ? 32 : BITS == 4 ? 8 : 4;
    const __half* prow = static_cast<const __half*>(params) + ((row0 + r_lo) / G) * 2 * cols;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 + j;
      const int pos = (c / BS) * BS + perm_position(c % BS, BS);
      pc[j] = make_float2(__half2float(prow[pos]), __half2float(prow[cols + pos]));
    }
  }
  const int64_t pstride = param_stride(cols, G);
  for (int r = r_lo; r < r_hi; ++r) {
    float v[8];
    if (r < n_codes) {
      const int64_t ar = row0 + r;
      const uint8_t* cp = codes + ar * row_bytes + (c0 / 8) * BITS;  // 8 codes = BITS bytes
      uint2 cw;
      if constexpr (BITS == 3) {
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(cp) & ~uintptr_t(3));
        const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(cp) & 3u);
        const uint32_t lo = __ldg(wp), hi = sh >= 2u ? __ldg(wp + 1) : 0u;
        cw = make_uint2(__funnelshift_r(lo, hi, 8u * sh), 0u);
      } else if constexpr (BITS == 2) {
        cw = make_uint2(__ldg(reinterpret_cast<const unsigned short*>(cp)), 0u);
      } else if constexpr (BITS == 4) {
        cw = make_uint2(__ldg(reinterpret_cast<const uint32_t*>(cp)), 0u);
      } else {
        cw = __ldg(reinterpret_cast<const uint2*>(cp));
      }
      float2 pt = make_float2(0.f, 0.f);
      if (AXIS == 0) pt = __half22float2(static_cast<const __half2*>(params)[ar * pstride + c0 / G]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t word = (BITS == 8 && j >= 4) ? cw.y : cw.x;
        const float code = static_cast<float>((word >> ((j * BITS) % 32)) & kMask);
        v[j] = AXIS == 0 ? fmaf(code, pt.x, pt.y) : fmaf(code, pc[j].x, pc[j].y);
      }
    } else {
      const float4* rr = reinterpret_cast<const float4*>(resid + (int64_t)(r - n_codes) * cols + c0);
      const float4 a = rr[0], b = rr[1];
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
    uint4 o;
    __half2* oh = reinterpret_cast<__half2*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) oh[j] = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
    *reinterpret_cast<uint4*>(out + (int64_t)r * ldo + c0) = o;
  }
}

__global__ void k_rope_table(float2* __restrict__ cs, int64_t n_pos, int hd, double theta,
                             int j_major) {
  const int half = hd / 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pos * half;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = i / half;
    const int j = i % half;
    const double freq = pow(theta, (-2.0 * j) / hd);  // linalg.py:85
    const double ang = static_cast<double>(pos) * freq;  // linalg.py:86
    const float2 v = make_float2(static_cast<float>(cos(ang)), static_cast<float>(sin(ang)));
    cs[j_major ? (int64_t)j * n_pos + pos : i] = v;
  }
}

__global__ void k_arrange_weights(const void* __restrict__ w_k, const void* __restrict__ w_v,
                                  int dt, int64_t kdim, int n_kv, int bs_k, int bs_v,
                                  __half* __restrict__ out) {
  const int64_t ld = (int64_t)n_kv * 128;
  const int64_t total = (int64_t)n_kv * 256 * kdim;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i % kdim;
    const int64_t rowi = i / kdim;
    const int h = static_cast<int>(rowi / 256), n = static_cast<int>(rowi % 256);
    const bool is_k = n < 128;
    const int bs = is_k ? bs_k : bs_v;
    const int64_t k = (p / bs) * bs + perm_channel(static_cast<int>(p % bs), bs);
    const int64_t col = (int64_t)h * 128 + (is_k ? n : n - 128);
    out[i] = __float2half_rn(load_as_f32(is_k ? w_k : w_v, dt, k * ld + col));
  }
}

// XQuant-CL accumulator (cache.py:139-146, :481): a grid-stride stream over
// (slot, token, 8-channel chunk) items -- 32 B of fp32 acc in and out, 16 B of
// fp16 copy out, bits bytes of codes and one (scale, zp) in per item, all as
// whole-word loads; HBM-bound.
__global__ void __launch_bounds__(256) k_cl_accumulate(
    int seed, const uint8_t* __restrict__ codes, int64_t row_bytes,
    const __half2* __restrict__ params, int bits, int G, int64_t cols,
    const int32_t* __restrict__ lens, int32_t n_seqs, int32_t max_len, int64_t L_max,
    float* __restrict__ acc, __half* __restrict__ x16) {
  const int64_t per_row = cols / 8;
  const int64_t total = (int64_t)n_seqs * max_len * per_row;
  const int64_t ng = param_stride(cols, G);
  const uint32_t mask = (1u << bits) - 1u;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rowi = i / per_row;
    const int b = static_cast<int>(rowi / max_len), t = static_cast<int>(rowi % max_len);
    if (t >= __ldg(lens + b)) continue;
    const int64_t c0 = (i % per_row) * 8;
    const int64_t r = (int64_t)b * L_max + t;
    // 8 codes = `bits` bytes at byte bits*c0/8 of the row (8-byte aligned rows)
    const uint8_t* crow = codes + r * row_bytes;
    const int64_t off = (c0 / 8) * bits;
    uint64_t packed;
    {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(crow + (off & ~int64_t(3)));
      // the second word only when the codes cross into it (never past the row)
      const uint64_t lo = __ldg(w), hi = ((off & 3) + bits > 4) ? __ldg(w + 1) : 0u;
      packed = (lo | (hi << 32)) >> ((off & 3) * 8);
      if (bits == 8) {  // 8 bytes, 8-aligned: the two words are exactly the codes
        packed = lo | (hi << 32);
      }
    }
    const float2 sz = __half22float2(__ldg(params + r * ng + c0 / G));  // one group: 8 | G
    float4* a4 = acc ? reinterpret_cast<float4*>(acc + r * cols + c0) : nullptr;
    float v[8];
    if (seed) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = 0.f;
    } else if (a4) {
      const float4 p0 = a4[0], p1 = a4[1];
      v[0] = p0.x; v[1] = p0.y; v[2] = p0.z; v[3] = p0.w;
      v[4] = p1.x; v[5] = p1.y; v[6] = p1.z; v[7] = p1.w;
    } else {  // fp16-storage accumulator: the fp16 copy is the accumulator
      const uint4 u = *reinterpret_cast<const uint4*>(x16 + r * cols + c0);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
        v[2 * k] = f.x;
        v[2 * k + 1] = f.y;
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      v[k] += fmaf(static_cast<float>((packed >> (k * bits)) & mask), sz.x, sz.y);
    if (a4) {
      a4[0] = make_float4(v[0], v[1], v[2], v[3]);
      a4[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
    if (x16) {
      __half2 h[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) h[k] = __floats2half2_rn(v[2 * k], v[2 * k + 1]);
      *reinterpret_cast<uint4*>(x16 + r * cols + c0) = *reinterpret_cast<uint4*>(h);
    }
  }
}

// The same update for the fp16-storage accumulator -- the engine's per-delta-layer
// hot case (seed: the accumulator starts at zero and is not read). Each thread owns 32 consecutive channels of one row: 64 B
// of accumulator in flight as four 16-byte loads, `BITS` whole words of codes and
// four (scale, zp) loads, with 32-bit index math. Per element the arithmetic is the
// generic kernel's (fp32 add of the fp32 dequantized delta, one fp16 rounding).
#ifndef XQ_ACC_CS
#define XQ_ACC_CS 0
#endif
#ifndef XQ_ACC_CTAS
#define XQ_ACC_CTAS 6
#endif
#ifndef XQ_ACC_COALESCED
#define XQ_ACC_COALESCED 1
#endif
template <int BITS, bool SEED>
__global__ void __launch_bounds__(256) k_cl_accumulate_h(
    const uint8_t* __restrict__ codes, int64_t row_bytes,
    const __half2* __restrict__ params, int G, int cols, const int32_t* __restrict__ lens, int max_len, int64_t L_max,
    uint32_t total, __half* __restrict__ x16) {
  constexpr uint32_t kMask = (1u << BITS) - 1u;
  const uint32_t per_row = static_cast<uint32_t>(cols) / 32;
  const int64_t ng = param_stride(cols, G);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += gridDim.x * blockDim.x) {
    const uint32_t rowi = i / per_row;
    const uint32_t b = rowi / static_cast<uint32_t>(max_len);
    const int t = static_cast<int>(rowi - b * static_cast<uint32_t>(max_len));
    if (t >= __ldg(lens + b)) continue;
    const int c0 = static_cast<int>(i - rowi * per_row) * 32;
    const int64_t r = static_cast<int64_t>(b) * L_max + t;
    uint4* xp = reinterpret_cast<uint4*>(x16 + r * cols + c0);
    uint4 q[4];
#pragma unroll
    // SEED is a template flag: as a runtime flag here it halved the kernel's
    // bandwidth (C3 shape: 3.49 vs 1.77 ms, tools/bench_accumulate.py)
#if XQ_ACC_CS
    for (int k = 0; k < 4; ++k) q[k] = SEED ? make_uint4(0u, 0u, 0u, 0u) : __ldcs(xp + k);
#else
    for (int k = 0; k < 4; ++k) q[k] = SEED ? make_uint4(0u, 0u, 0u, 0u) : xp[k];
#endif
    // 32 codes = BITS words at byte 4*BITS*(c0/32) of the row
    const uint32_t* cw = reinterpret_cast<const uint32_t*>(codes + r * row_bytes) + (c0 / 32) * BITS;
    uint32_t w[BITS + 1];
#pragma unroll
    for (int k = 0; k < BITS; ++k) w[k] = __ldg(cw + k);
    w[BITS] = 0u;
    __half2 sz[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) sz[k] = __ldg(params + r * ng + (c0 + 8 * k) / G);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __half22float2(sz[k]);
      uint32_t hw[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m = 8 * k + 2 * j + e, bit = m * BITS, wi = bit / 32, sh = bit % 32;
          const uint32_t code =
              static_cast<uint32_t>(((static_cast<uint64_t>(w[wi + 1]) << 32) | w[wi]) >> sh) & kMask;
          v[e] = fmaf(static_cast<float>(code), f.x, f.y);
        }
        const float2 old = __half22float2(*reinterpret_cast<const __half2*>(&hw[j]));
        const __half2 h = __floats2half2_rn(old.x + v[0], old.y + v[1]);
        hw[j] = *reinterpret_cast<const uint32_t*>(&h);
      }
#if XQ_ACC_CS
      __stcs(xp + k, make_uint4(hw[0], hw[1], hw[2], hw[3]));
#else
      xp[k] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
#endif
    }
  }
}

// Warp-coalesced form of the fp16 update for cols % 1024 == 0: a
// warp owns 1024 channels of one row, lane l channels 256k + 8l .. +7 (k < 4), so
// every 16-byte accumulator load and store instruction covers 512 contiguous bytes
// (the per-thread-contiguous form touches a quarter of each 64-byte span per
// instruction and leans on L1 to merge them). A lane's 8 codes are BITS whole bytes
// (for 3 bits at any byte alignment).
// Same arithmetic per element as k_cl_accumulate_h.
template <int BITS, bool SEED>
__global__ void __launch_bounds__(256) k_cl_accumulate_w(
    const uint8_t* __restrict__ codes, int64_t row_bytes, const __half2* __restrict__ params,
    int G, int cols, const int32_t* __restrict__ lens, int max_len, int64_t L_max,
    uint32_t total_spans, __half* __restrict__ x16) {
  constexpr uint32_t kMask = (1u << BITS) - 1u;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t spans = static_cast<uint32_t>(cols) / 1024u;
  const int64_t ng = param_stride(cols, G);
  const uint32_t nw = gridDim.x * (blockDim.x / 32u);
  for (uint32_t w = blockIdx.x * (blockDim.x / 32u) + (threadIdx.x >> 5); w < total_spans; w += nw) {
    const uint32_t rowi = w / spans;
    const uint32_t b = rowi / static_cast<uint32_t>(max_len);
    const int t = static_cast<int>(rowi - b * static_cast<uint32_t>(max_len));
    if (t >= __ldg(lens + b)) continue;  // warp-uniform
    const int64_t r = static_cast<int64_t>(b) * L_max + t;
    const int cbase = static_cast<int>(w - rowi * spans) * 1024 + 8 * static_cast<int>(lane);
    uint4* xp = reinterpret_cast<uint4*>(x16 + r * cols + cbase);  // + 32 uint4 per k
    uint4 q[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = SEED ? make_uint4(0u, 0u, 0u, 0u) : xp[32 * k];
    uint2 cw[4];
    __half2 sz[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c0 = cbase + 256 * k;
      const uint8_t* cp = codes + r * row_bytes + c0 * BITS / 8;
      if constexpr (BITS == 3) {  // 3 bytes at any alignment: one or two aligned words
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(cp) & ~uintptr_t(3));
        const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(cp) & 3u);
        // the second word only when the field crosses into it (never past the row end:
        // rows are 8-byte multiples and the field ends at or before it)
        const uint32_t lo = __ldg(wp), hi = sh >= 2u ? __ldg(wp + 1) : 0u;
        cw[k] = make_uint2(__funnelshift_r(lo, hi, 8u * sh), 0u);
      } else if constexpr (BITS == 2) cw[k] = make_uint2(__ldg(reinterpret_cast<const unsigned short*>(cp)), 0u);
      else if constexpr (BITS == 4) cw[k] = make_uint2(__ldg(reinterpret_cast<const uint32_t*>(cp)), 0u);
      else cw[k] = __ldg(reinterpret_cast<const uint2*>(cp));
      sz[k] = __ldg(params + r * ng + c0 / G);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __half22float2(sz[k]);
      uint32_t hw[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m = 2 * j + e;
          const uint32_t word = (BITS == 8 && m >= 4) ? cw[k].y : cw[k].x;
          const uint32_t code = (word >> ((m * BITS) % 32)) & kMask;
          v[e] = fmaf(static_cast<float>(code), f.x, f.y);
        }
        const float2 old = __half22float2(*reinterpret_cast<const __half2*>(&hw[j]));
        const __half2 h = __floats2half2_rn(old.x + v[0], old.y + v[1]);
        hw[j] = *reinterpret_cast<const uint32_t*>(&h);
      }
      xp[32 * k] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    }
  }
}

// one warp per quantization group of a row (the fp64 group math is a latency
// chain; a decode step quantizes only a few rows)
static int rows_threads(int64_t cols, int G) {
  const int64_t w = 32 * ((cols + G - 1) / G);
  return static_cast<int>(w < 128 ? 128 : (w > 512 ? 512 : w));  // 72 registers x 512 threads
}

static int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace xq

using namespace xq;

namespace xq {
template <typename T>
static int quantize_blocks_per_channel(const T* blocks, int64_t n_blocks, int64_t cols, int32_t bits,
                                       int32_t group_size, const int64_t* dst_row0, uint8_t* codes,
                                       int64_t row_bytes, void* params, int32_t* nonfinite_flag,
                                       void* stream, double* recon = nullptr) {
  XQ_REQUIRE(valid_bits(bits), XQ_ECONFIG, "bits must be one of (2, 3, 4, 8), got %d", bits);
  XQ_REQUIRE(cols % 32 == 0, XQ_ESHAPE, "per-channel width must be a multiple of 32");
  XQ_REQUIRE(group_size >= 1 && group_size <= 1024, XQ_ECONFIG, "bad group_size");
  XQ_REQUIRE(row_bytes == row_bytes_for(cols, bits), XQ_ESHAPE, "bad row_bytes");
  if (n_blocks == 0) return XQ_OK;
  dim3 grid(static_cast<unsigned>(n_blocks), static_cast<unsigned>(cols / 32));
  k_quantize_blocks_per_channel<T><<<grid, 128, static_cast<size_t>(group_size) * 32,
                                     (cudaStream_t)stream>>>(blocks, cols, bits, group_size,
                                                             dst_row0, codes, row_bytes,
                                                             static_cast<__half*>(params),
                                                             nonfinite_flag, recon);
  return check_launch("xq_quantize_blocks_per_channel");
}

}  // namespace xq

extern "C" {

const char* xq_version(void) { return "xquant-b200 0.1 (sm_100a)"; }
const char* xq_last_error(void) { return g_err; }

int xq_quantize_groups(const double* x, int64_t rows, int64_t cols, int32_t group_size,
                       int32_t bits, uint8_t* codes, double* scales, double* zero_points,
                       void* stream) {
  XQ_REQUIRE(valid_bits(bits), XQ_ECONFIG, "bits must be one of (2, 3, 4, 8), got %d", bits);
  XQ_REQUIRE(group_size >= 1, XQ_ECONFIG, "group_size must be >= 1, got %d", group_size);
  XQ_REQUIRE(rows >= 0 && cols >= 0, XQ_ESHAPE, "negative shape");
  if (rows == 0 || cols == 0) return XQ_OK;
  XQ_REQUIRE(rows < (1ll << 31), XQ_ESHAPE, "too many rows");
  k_quantize_groups<<<static_cast<unsigned>(rows), 128, 0, (cudaStream_t)stream>>>(
      x, cols, group_size, bits, codes, scales, zero_points);
  return check_launch("xq_quantize_groups");
}

int xq_dequantize_groups(const uint8_t* codes, const double* scales, const double* zero_points,
                         int64_t rows, int64_t cols, int32_t group_size, double* out,
                         void* stream) {
  XQ_REQUIRE(group_size >= 1, XQ_ECONFIG, "group_size must be >= 1");
  if (rows * cols == 0) return XQ_OK;
  k_dequantize_groups<<<grid_for(rows * cols, 256), 256, 0, (cudaStream_t)stream>>>(
      codes, scales, zero_points, rows, cols, group_size, out);
  return check_launch("xq_dequantize_groups");
}

int xq_pack_codes(const uint8_t* codes, int64_t n, int32_t bits, uint64_t* words, void* stream) {
  XQ_REQUIRE(bits >= 1 && bits <= 8, XQ_ECONFIG, "bits must be in 1..8, got %d", bits);
  const int64_t n_words = (n * bits + 63) / 64;
  if (n_words == 0) return XQ_OK;
  k_pack<<<grid_for(n_words, 256), 256, 0, (cudaStream_t)stream>>>(codes, n, bits, words,
                                                                    n_words);
  return check_launch("xq_pack_codes");
}

int xq_unpack_codes(const uint64_t* words, int32_t bits, int64_t n, uint8_t* codes,
                    void* stream) {
  XQ_REQUIRE(bits >= 1 && bits <= 8, XQ_ECONFIG, "bits must be in 1..8, got %d", bits);
  if (n == 0) return XQ_OK;
  k_unpack<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(words, bits, n, codes);
  return check_launch("xq_unpack_codes");
}

int xq_quantize_rows(const void* x, int32_t x_dtype, int64_t x_row_stride, int64_t n_rows,
                     int64_t cols, int32_t bits, int32_t group_size, const int32_t* seq_lens,
                     int64_t row0, int64_t L_max, const float* sub_rows, uint8_t* codes,
                     int64_t row_bytes, void* params, double* x_eff_out, int32_t* nonfinite_flag,
                     void* stream) {
  XQ_REQUIRE(valid_bits(bits), XQ_ECONFIG, "bits must be one of (2, 3, 4, 8), got %d", bits);
  XQ_REQUIRE(group_size >= 1, XQ_ECONFIG, "group_size must be >= 1");
  XQ_REQUIRE(dtype_size(x_dtype) > 0, XQ_ECONFIG, "unknown dtype %d", x_dtype);
  XQ_REQUIRE(row_bytes == row_bytes_for(cols, bits), XQ_ESHAPE,
             "row_bytes %lld != ceil(cols*bits/64)*8 = %lld", (long long)row_bytes,
             (long long)row_bytes_for(cols, bits));
  XQ_REQUIRE(cols <= 48 * 1024, XQ_ESHAPE, "cols %lld too wide for one CTA", (long long)cols);
  if (n_rows == 0 || cols == 0) return XQ_OK;
  k_quantize_rows<<<static_cast<unsigned>(n_rows), rows_threads(cols, group_size), static_cast<size_t>(cols),
                    (cudaStream_t)stream>>>(x, x_dtype, x_row_stride, cols, group_size, bits,
                                            seq_lens, row0, L_max, sub_rows, codes, row_bytes,
                                            static_cast<__half2*>(params), x_eff_out,
                                            nonfinite_flag);
  return check_launch("xq_quantize_rows");
}

int xq_quantize_rows_cl(const void* x, int32_t x_dtype, int64_t x_row_stride, int64_t n_rows,
                        int64_t cols, int32_t bits, int32_t group_size, const int32_t* seq_lens,
                        int64_t row0, int64_t L_max, double* acc_rows, int32_t acc_mode,
                        uint8_t* codes, int64_t row_bytes, void* params, int32_t* nonfinite_flag,
                        void* stream) {
  XQ_REQUIRE(valid_bits(bits), XQ_ECONFIG, "bits must be one of (2, 3, 4, 8), got %d", bits);
  XQ_REQUIRE(group_size >= 1, XQ_ECONFIG, "group_size must be >= 1");
  XQ_REQUIRE(dtype_size(x_dtype) > 0, XQ_ECONFIG, "unknown dtype %d", x_dtype);
  XQ_REQUIRE(acc_rows != nullptr, XQ_EUSAGE, "acc_rows is required");
  XQ_REQUIRE(acc_mode == 1 || acc_mode == 2, XQ_ECONFIG,
             "acc_mode must be 1 (delta) or 2 (seed), got %d", acc_mode);
  XQ_REQUIRE(row_bytes == row_bytes_for(cols, bits), XQ_ESHAPE,
             "row_bytes %lld != ceil(cols*bits/64)*8 = %lld", (long long)row_bytes,
             (long long)row_bytes_for(cols, bits));
  XQ_REQUIRE(cols <= 48 * 1024, XQ_ESHAPE, "cols %lld too wide for one CTA", (long long)cols);
  if (n_rows == 0 || cols == 0) return XQ_OK;
  k_quantize_rows<<<static_cast<unsigned>(n_rows), rows_threads(cols, group_size), static_cast<size_t>(cols),
                    (cudaStream_t)stream>>>(x, x_dtype, x_row_stride, cols, group_size, bits,
                                            seq_lens, row0, L_max, nullptr, codes, row_bytes,
                                            static_cast<__half2*>(params), nullptr,
                                            nonfinite_flag, acc_rows, acc_mode);
  return check_launch("xq_quantize_rows_cl");
}

int xq_quantize_blocks_per_channel(const float* blocks, int64_t n_blocks, int64_t cols,
                                   int32_t bits, int32_t group_size, const int64_t* dst_row0,
                                   uint8_t* codes, int64_t row_bytes, void* params,
                                   int32_t* nonfinite_flag, void* stream) {
  return quantize_blocks_per_channel(blocks, n_blocks, cols, bits, group_size, dst_row0, codes,
                                     row_bytes, params, nonfinite_flag, stream);
}

int xq_quantize_blocks_per_channel_f64(const double* blocks, int64_t n_blocks, int64_t cols,
                                       int32_t bits, int32_t group_size, const int64_t* dst_row0,
                                       uint8_t* codes, int64_t row_bytes, void* params,
                                       int32_t* nonfinite_flag, void* stream) {
  return quantize_blocks_per_channel(blocks, n_blocks, cols, bits, group_size, dst_row0, codes,
                                     row_bytes, params, nonfinite_flag, stream);
}

int xq_dequant_rows(const uint8_t* codes, int64_t row_bytes, const void* params, int32_t axis,
                    int32_t bits, int32_t group_size, int64_t cols, int64_t row0, int64_t n_rows,
                    float* out, void* stream) {
  XQ_REQUIRE(bits >= 1 && bits <= 8, XQ_ECONFIG, "bad bits");
  XQ_REQUIRE(axis == 0 || axis == 1, XQ_ECONFIG, "axis must be 0 or 1");
  if (n_rows * cols == 0) return XQ_OK;
  k_dequant_rows<<<grid_for(n_rows * cols, 256), 256, 0, (cudaStream_t)stream>>>(
      codes, row_bytes, params, axis, bits, group_size, cols, row0, n_rows, out);
  return check_launch("xq_dequant_rows");
}

int xq_quantize_blocks_per_channel_f64_recon(const double* blocks, int64_t n_blocks, int64_t cols,
                                             int32_t bits, int32_t group_size,
                                             const int64_t* dst_row0, uint8_t* codes,
                                             int64_t row_bytes, void* params, double* recon_out,
                                             int32_t* nonfinite_flag, void* stream) {
  XQ_REQUIRE(recon_out != nullptr, XQ_EUSAGE, "recon_out is required");
  return quantize_blocks_per_channel(blocks, n_blocks, cols, bits, group_size, dst_row0, codes,
                                     row_bytes, params, nonfinite_flag, stream, recon_out);
}

int xq_dequant_rows_f16(const uint8_t* codes, int64_t row_bytes, const void* params, int32_t axis,
                        int32_t bits, int32_t group_size, int64_t cols, int64_t row0,
                        int64_t n_codes, const float* resid, int64_t n_rows, void* out,
                        int64_t ldo, void* stream) {
  XQ_REQUIRE(bits >= 1 && bits <= 8, XQ_ECONFIG, "bad bits");
  XQ_REQUIRE(axis == 0 || axis == 1, XQ_ECONFIG, "axis must be 0 or 1");
  XQ_REQUIRE(n_codes <= n_rows && (n_codes == n_rows || resid != nullptr), XQ_EUSAGE,
             "rows past n_codes need the residual buffer");
  XQ_REQUIRE(ldo >= cols, XQ_ESHAPE, "ldo < cols");
  XQ_REQUIRE(cols % 8 == 0 && ldo % 8 == 0 && row_bytes % 4 == 0 &&
                 reinterpret_cast<uintptr_t>(out) % 16 == 0,
             XQ_ESHAPE, "cols / ldo must be multiples of 8 and out 16-byte aligned");
  if (n_rows * cols == 0) return XQ_OK;
  // specialised kernel: whole 128-token groups per block row (per-channel), 32-bit indices
  if (valid_bits(bits) && cols < (int64_t(1) << 30) && n_rows < (int64_t(1) << 30) &&
      (axis == 0 || (group_size % kRowsPerBlk == 0 && row0 % group_size == 0))) {
    const dim3 grid(static_cast<unsigned>((cols / 8 + 127) / 128),
                    static_cast<unsigned>((n_rows + kRowsPerBlk - 1) / kRowsPerBlk));
    auto go = [&](auto kern) {
      kern<<<grid, 128, 0, (cudaStream_t)stream>>>(codes, row_bytes, params, group_size,
                                                    static_cast<int>(cols), row0,
                                                    static_cast<int>(n_codes), resid,
                                                    static_cast<int>(n_rows),
                                                    static_cast<__half*>(out), ldo);
    };
    switch (bits * 2 + axis) {
      case 4: go(k_dequant_rows_f16_t<2, 0>); break;
      case 5: go(k_dequant_rows_f16_t<2, 1>); break;
      case 6: go(k_dequant_rows_f16_t<3, 0>); break;
      case 7: go(k_dequant_rows_f16_t<3, 1>); break;
      case 8: go(k_dequant_rows_f16_t<4, 0>); break;
      case 9: go(k_dequant_rows_f16_t<4, 1>); break;
      case 16: go(k_dequant_rows_f16_t<8, 0>); break;
      default: go(k_dequant_rows_f16_t<8, 1>); break;
    }
    return check_launch("xq_dequant_rows_f16");
  }
  k_dequant_rows_f16<<<grid_for(n_rows * cols / 8, 256), 256, 0, (cudaStream_t)stream>>>(
      codes, row_bytes, params, axis, bits, group_size, cols, row0, n_codes, resid, n_rows,
      static_cast<__half*>(out), ldo);
  return check_launch("xq_dequant_rows_f16");
}

int xq_rope_table(void* cs_out, int64_t n_pos, int32_t head_dim, double theta, int32_t j_major,
                  void* stream) {
  XQ_REQUIRE(head_dim % 2 == 0, XQ_ECONFIG, "head_dim must be even, got %d", head_dim);
  if (n_pos == 0) return XQ_OK;
  k_rope_table<<<grid_for(n_pos * head_dim / 2, 256), 256, 0, (cudaStream_t)stream>>>(
      static_cast<float2*>(cs_out), n_pos, head_dim, theta, j_major);
  return check_launch("xq_rope_table");
}

int xq_arrange_weights(const void* w_k, const void* w_v, int32_t w_dtype, int64_t kdim,
                       int32_t n_kv_heads, int32_t a_mode_k, int32_t bits_k, int32_t a_mode_v,
                       int32_t bits_v, void* w_out, void* stream) {
  XQ_REQUIRE(kdim % 64 == 0, XQ_ESHAPE, "kdim must be a multiple of 64, got %lld",
             (long long)kdim);
  XQ_REQUIRE(dtype_size(w_dtype) > 0, XQ_ECONFIG, "unknown dtype");
  if (a_mode_v == XQ_A_SAME) {
    a_mode_v = a_mode_k;
    bits_v = bits_k;
  }
  const int bs_k = perm_block(a_mode_k, bits_k), bs_v = perm_block(a_mode_v, bits_v);
  const int64_t total = (int64_t)n_kv_heads * 256 * kdim;
  k_arrange_weights<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(
      w_k, w_v, w_dtype, kdim, n_kv_heads, bs_k, bs_v, static_cast<__half*>(w_out));
  return check_launch("xq_arrange_weights");
}

int xq_cl_accumulate(int32_t seed, const uint8_t* codes, int64_t row_bytes, const void* params,
                     int32_t bits, int32_t group_size, int64_t cols, const int32_t* seq_lens,
                     int32_t n_seqs, int32_t max_len, int64_t L_max, float* acc, void* x16_out,
                     void* stream) {
  XQ_REQUIRE(valid_bits(bits), XQ_ECONFIG, "bad bits %d", bits);
  XQ_REQUIRE(cols % 8 == 0, XQ_ESHAPE, "cols must be a multiple of 8");
  XQ_REQUIRE(max_len <= L_max, XQ_ESHAPE, "max_len > L_max");
  if (n_seqs == 0 || max_len == 0) return XQ_OK;
  XQ_REQUIRE(group_size % 8 == 0, XQ_ECONFIG, "group_size must be a multiple of 8");
  XQ_REQUIRE(acc != nullptr || x16_out != nullptr, XQ_EUSAGE, "no accumulator buffer");
  const int64_t items32 = (int64_t)n_seqs * max_len * (cols / 32);
  const int64_t spans = (int64_t)n_seqs * max_len * (cols / 1024);
  if (XQ_ACC_COALESCED && acc == nullptr && cols % 1024 == 0 && group_size % 8 == 0 &&
      cols < (int64_t(1) << 30) && spans + (int64_t)148 * XQ_ACC_CTAS * 8 < (int64_t(1) << 32)) {
    const int64_t blocks = std::min<int64_t>((spans + 7) / 8, 148 * XQ_ACC_CTAS);
    auto launchw = [&](auto kern) {
      kern<<<static_cast<unsigned>(blocks), 256, 0, (cudaStream_t)stream>>>(
          codes, row_bytes, static_cast<const __half2*>(params), group_size,
          static_cast<int>(cols), seq_lens, max_len, L_max, static_cast<uint32_t>(spans),
          static_cast<__half*>(x16_out));
    };
    switch (bits) {
      case 2: seed ? launchw(k_cl_accumulate_w<2, true>) : launchw(k_cl_accumulate_w<2, false>); break;
      case 3: seed ? launchw(k_cl_accumulate_w<3, true>) : launchw(k_cl_accumulate_w<3, false>); break;
      case 4: seed ? launchw(k_cl_accumulate_w<4, true>) : launchw(k_cl_accumulate_w<4, false>); break;
      default: seed ? launchw(k_cl_accumulate_w<8, true>) : launchw(k_cl_accumulate_w<8, false>); break;
    }
    return check_launch("xq_cl_accumulate");
  }
  if (acc == nullptr && cols % 32 == 0 && cols < (int64_t(1) << 30) &&
      items32 + (int64_t)148 * XQ_ACC_CTAS * 256 < (int64_t(1) << 32)) {
    const int64_t blocks = std::min<int64_t>((items32 + 255) / 256, 148 * XQ_ACC_CTAS);  // 38 regs
    auto launch2 = [&](auto kern) {
      kern<<<static_cast<unsigned>(blocks), 256, 0, (cudaStream_t)stream>>>(
          codes, row_bytes, static_cast<const __half2*>(params), group_size,
          static_cast<int>(cols), seq_lens, max_len, L_max, static_cast<uint32_t>(items32),
          static_cast<__half*>(x16_out));
    };
    switch (bits) {
      case 2: seed ? launch2(k_cl_accumulate_h<2, true>) : launch2(k_cl_accumulate_h<2, false>); break;
      case 3: seed ? launch2(k_cl_accumulate_h<3, true>) : launch2(k_cl_accumulate_h<3, false>); break;
      case 4: seed ? launch2(k_cl_accumulate_h<4, true>) : launch2(k_cl_accumulate_h<4, false>); break;
      default: seed ? launch2(k_cl_accumulate_h<8, true>) : launch2(k_cl_accumulate_h<8, false>); break;
    }
    return check_launch("xq_cl_accumulate");
  }
  const int64_t items = (int64_t)n_seqs * max_len * (cols / 8);
  int64_t blocks = (items + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_cl_accumulate<<<static_cast<unsigned>(blocks), 256, 0, (cudaStream_t)stream>>>(
      seed, codes, row_bytes, static_cast<const __half2*>(params), bits, group_size, cols,
      seq_lens, n_seqs, max_len, L_max, acc, static_cast<__half*>(x16_out));
  return check_launch("xq_cl_accumulate");
}

}  // extern "C"
