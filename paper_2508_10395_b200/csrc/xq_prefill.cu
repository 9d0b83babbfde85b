// Prefill attention block (model._Session.prefill, model.py:205-221): causal
// grouped-query attention of n prompt positions over the K/V the remat GEMM
// (xq_gemm.cu) rebuilt from the cache, plus the RoPE of the rows that are not
// produced rotated (q, and the kvq baseline's dequantized K).
//
// k_prefill_attend is a flash-attention kernel (online softmax, K/V never
// materialised beyond one 64-key tile in shared memory): one CTA = 64 query
// rows of one head, 4 warps x 16 rows; S = Q K^T and O += P V on
// mma.sync m16n8k16 (fp16/bf16 in, fp32 accumulate) with ldmatrix fragments
// from XOR-swizzled tiles and a cp.async double buffer. Prefill is a
// one-off per sequence; the decode step is the tcgen05 hot path.

#include "xq_common.cuh"
#include "xq_host.h"

namespace xq {
namespace {

constexpr int kPQ = 64;        // query rows per CTA
constexpr int kPK = 64;        // keys per tile
constexpr int kPThreads = 128;
constexpr int kRowBytes = 256; // 128 x 16-bit

template <typename T>
struct Mma;
template <>
struct Mma<__half> {
  XQ_DEVINL static void run(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  XQ_DEVINL static uint32_t pack(float x, float y) {
    __half2 h = __floats2half2_rn(x, y);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};
template <>
struct Mma<__nv_bfloat16> {
  XQ_DEVINL static void run(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  XQ_DEVINL static uint32_t pack(float x, float y) {
    __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};

XQ_DEVINL void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
XQ_DEVINL void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
XQ_DEVINL void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;  // zero-fill rows past the end
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n)
               : "memory");
}
XQ_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
XQ_DEVINL void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// byte offset of 16-byte chunk c (0..15) of row r in a swizzled [rows][128] tile
XQ_DEVINL uint32_t swz(int r, int c) { return r * kRowBytes + ((c ^ (r & 7)) << 4); }

// 64 rows x 128 elements of a [n][stride] tensor -> swizzled shared tile
template <typename T>
XQ_DEVINL void load_tile(uint32_t dst, const T* base, int64_t stride, int row0, int n_rows) {
  for (int i = threadIdx.x; i < 64 * 16; i += kPThreads) {
    const int r = i >> 4, c = i & 15;
    const int gr = row0 + r;
    const bool ok = gr < n_rows;
    cp_async16(dst + swz(r, c), base + static_cast<int64_t>(ok ? gr : 0) * stride + c * 8, ok);
  }
}

template <typename T>
__global__ void __launch_bounds__(kPThreads)
    k_prefill_attend(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                     int n, int n_heads, int group, int64_t q_stride, int64_t kv_stride,
                     float scale_log2, float* __restrict__ out, int64_t out_stride) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK = sQ + kPQ * kRowBytes;        // [2][64][128]
  const uint32_t sV = sK + 2 * kPK * kRowBytes;    // [2][64][128]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qb = gridDim.x - 1 - blockIdx.x;        // longest (latest) blocks first
  const int h = blockIdx.y, hk = h / group;
  const int q0 = qb * kPQ;
  const T* qh = q + static_cast<int64_t>(h) * 128;
  const T* kh = k + static_cast<int64_t>(hk) * 128;
  const T* vh = v + static_cast<int64_t>(hk) * 128;

  load_tile(sQ, qh + static_cast<int64_t>(q0) * q_stride, q_stride, 0, n - q0);
  const int n_kt = (min(n, q0 + kPQ) + kPK - 1) / kPK;  // causal: keys <= last query row
  load_tile(sK, kh, kv_stride, 0, n);
  load_tile(sV, vh, kv_stride, 0, n);
  cp_async_commit();

  float o[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  uint32_t qf[8][4];
  const int row_a = warp * 16 + (lane >> 2);  // rows row_a, row_a + 8 of this CTA's 64

  for (int t = 0; t < n_kt; ++t) {
    const int buf = t & 1;
    if (t + 1 < n_kt) {
      load_tile(sK + (buf ^ 1) * kPK * kRowBytes, kh, kv_stride, (t + 1) * kPK, n);
      load_tile(sV + (buf ^ 1) * kPK * kRowBytes, vh, kv_stride, (t + 1) * kPK, n);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (t == 0) {  // Q fragments of this warp's 16 rows, all 8 k-steps
      const int r = warp * 16 + (lane & 15);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        ldsm_x4(sQ + swz(r, 2 * ks + (lane >> 4)), qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
    }
    const uint32_t kt = sK + buf * kPK * kRowBytes, vt = sV + buf * kPK * kRowBytes;
    // ---- S = Q K^T: 16 rows x 64 keys (8 n-tiles)
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {  // key n-tiles 2jj, 2jj+1
        const int key = jj * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int chunk = 2 * ks + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kt + swz(key, chunk), b0, b1, b2, b3);
        Mma<T>::run(s[2 * jj], qf[ks], b0, b1);
        Mma<T>::run(s[2 * jj + 1], qf[ks], b2, b3);
      }
    }
    // ---- causal mask (only the diagonal tile) + online softmax
    const int key0 = t * kPK;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int qrow = q0 + row_a + half * 8;
      float mx = m_r[half];
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int key = key0 + j * 8 + 2 * (lane & 3) + e;
          float x = s[j][2 * half + e] * scale_log2;
          if (key > qrow || key >= n) x = -INFINITY;
          s[j][2 * half + e] = x;
          mx = fmaxf(mx, x);
        }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float corr = exp2f(m_r[half] - mx);  // m_r = -inf on the first tile -> 0
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float pexp = exp2f(s[j][2 * half + e] - mx);
          s[j][2 * half + e] = pexp;
          sum += pexp;
        }
      l_r[half] = l_r[half] * corr + sum;
      m_r[half] = mx;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        o[j][2 * half] *= corr;
        o[j][2 * half + 1] *= corr;
      }
    }
    // ---- O += P V: P (16 x 64 keys) as A fragments, V^T fragments by ldmatrix.trans
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // 16 keys per k-step
      uint32_t pa[4];
      pa[0] = Mma<T>::pack(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = Mma<T>::pack(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = Mma<T>::pack(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = Mma<T>::pack(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dj = 0; dj < 8; ++dj) {  // dims 16*dj .. 16*dj+15 (n-tiles 2dj, 2dj+1)
        const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int chunk = 2 * dj + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vt + swz(key, chunk), b0, b1, b2, b3);
        Mma<T>::run(o[2 * dj], pa, b0, b1);
        Mma<T>::run(o[2 * dj + 1], pa, b2, b3);
      }
    }
    __syncthreads();  // the buffer is refilled next iteration
  }
  // ---- normalise and store (fp32)
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    float l = l_r[half];
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    const int qrow = q0 + row_a + half * 8;
    if (qrow >= n) continue;
    const float inv = 1.f / l;
    float* orow = out + static_cast<int64_t>(qrow) * out_stride + static_cast<int64_t>(h) * 128;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int d = j * 8 + 2 * (lane & 3);
      *reinterpret_cast<float2*>(orow + d) = make_float2(o[j][2 * half] * inv, o[j][2 * half + 1] * inv);
    }
  }
}

// RoPE (linalg.py:58-95) of n rows of `width` columns (pairs (2j, 2j+1) of every
// 128-wide head) at positions pos0.., float32 or fp16/bf16 in, fp16/bf16 out.
template <typename TI, typename TO>
__global__ void k_rope_rows(const TI* __restrict__ in, int64_t in_stride, int64_t n, int64_t width,
                            const float2* __restrict__ rope, int64_t pos0, TO* __restrict__ out,
                            int64_t out_stride) {
  const int64_t pairs = width / 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * pairs;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / pairs, pc = i % pairs;
    const int j = static_cast<int>(pc % 64);
    const float2 cs = rope[(pos0 + r) * 64 + j];
    const float e = static_cast<float>(in[r * in_stride + 2 * pc]);
    const float o = static_cast<float>(in[r * in_stride + 2 * pc + 1]);
    out[r * out_stride + 2 * pc] = static_cast<TO>(e * cs.x - o * cs.y);
    out[r * out_stride + 2 * pc + 1] = static_cast<TO>(e * cs.y + o * cs.x);
  }
}

}  // namespace
}  // namespace xq

using namespace xq;

extern "C" int xq_prefill_attend(const void* q, const void* k, const void* v, int32_t dtype,
                                 int32_t n, int32_t n_heads, int32_t group, int64_t q_stride,
                                 int64_t kv_stride, float sm_scale, float* out, int64_t out_stride,
                                 void* stream) {
  XQ_REQUIRE(dtype == XQ_F16 || dtype == XQ_BF16, XQ_ECONFIG, "q/k/v must be fp16 or bf16");
  XQ_REQUIRE(n_heads >= 1 && group >= 1 && n_heads % group == 0, XQ_ECONFIG, "bad head grouping");
  XQ_REQUIRE(q_stride % 8 == 0 && kv_stride % 8 == 0, XQ_ESHAPE, "row strides must be multiples of 8");
  XQ_REQUIRE(reinterpret_cast<uintptr_t>(q) % 16 == 0 && reinterpret_cast<uintptr_t>(k) % 16 == 0 &&
                 reinterpret_cast<uintptr_t>(v) % 16 == 0,
             XQ_ESHAPE, "q/k/v must be 16-byte aligned");
  if (n == 0) return XQ_OK;
  const size_t smem = (kPQ + 4 * kPK) * kRowBytes;
  dim3 grid((n + kPQ - 1) / kPQ, n_heads);
  const float scale_log2 = sm_scale * 1.4426950408889634f;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int s;
  if (dtype == XQ_F16) {
    if ((s = ensure_smem(reinterpret_cast<const void*>(k_prefill_attend<__half>), smem,
                         "cudaFuncSetAttribute(prefill_attend)")) != XQ_OK)
      return s;
    k_prefill_attend<__half><<<grid, kPThreads, smem, st>>>(
        static_cast<const __half*>(q), static_cast<const __half*>(k), static_cast<const __half*>(v),
        n, n_heads, group, q_stride, kv_stride, scale_log2, out, out_stride);
  } else {
    if ((s = ensure_smem(reinterpret_cast<const void*>(k_prefill_attend<__nv_bfloat16>), smem,
                         "cudaFuncSetAttribute(prefill_attend)")) != XQ_OK)
      return s;
    k_prefill_attend<__nv_bfloat16><<<grid, kPThreads, smem, st>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
        static_cast<const __nv_bfloat16*>(v), n, n_heads, group, q_stride, kv_stride, scale_log2,
        out, out_stride);
  }
  return check_launch("k_prefill_attend");
}

extern "C" int xq_rope_rows(const void* in, int32_t in_dtype, int64_t in_stride, int64_t n,
                            int64_t width, const void* rope_cs, int64_t rope_n, int64_t pos0,
                            void* out, int32_t out_dtype, int64_t out_stride, void* stream) {
  XQ_REQUIRE(width % 128 == 0, XQ_ESHAPE, "width must be a multiple of 128 (whole heads)");
  XQ_REQUIRE(pos0 + n <= rope_n, XQ_ESHAPE, "rope table too short");
  XQ_REQUIRE(in_dtype == XQ_F32 || in_dtype == XQ_F16, XQ_ECONFIG, "input must be f32 or f16");
  XQ_REQUIRE(out_dtype == XQ_F16 || out_dtype == XQ_BF16, XQ_ECONFIG, "output must be f16 or bf16");
  if (n == 0) return XQ_OK;
  const int64_t total = n * width / 2;
  const int grid = static_cast<int>(total / 256 + 1 < 4096 ? total / 256 + 1 : 4096);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float2* rope = static_cast<const float2*>(rope_cs);
#define XQ_ROPE(TI, TO)                                                                          \
  k_rope_rows<TI, TO><<<grid, 256, 0, st>>>(static_cast<const TI*>(in), in_stride, n, width, rope, \
                                            pos0, static_cast<TO*>(out), out_stride)
  if (in_dtype == XQ_F32 && out_dtype == XQ_F16) XQ_ROPE(float, __half);
  else if (in_dtype == XQ_F32) XQ_ROPE(float, __nv_bfloat16);
  else if (out_dtype == XQ_F16) XQ_ROPE(__half, __half);
  else XQ_ROPE(__half, __nv_bfloat16);
#undef XQ_ROPE
  return check_launch("k_rope_rows");
}
