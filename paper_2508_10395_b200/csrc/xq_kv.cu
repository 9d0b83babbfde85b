// fp16-KV decode baseline on the same GPU: the reference's FullPrecisionCache
// semantics (cache.py:302-323) with post-RoPE bf16 K/V resident in HBM
// (standard practice, mathematically identical to re-rotating pre-RoPE K each
// step) and a split-K flash-decode that streams K/V once at HBM bandwidth.
#include <math.h>

#include "xq_common.cuh"
#include "xq_host.h"

namespace xq {

__global__ void k_combine(const float* __restrict__ partials, int n_parts, float* __restrict__ out);

constexpr int kKvThreads = 128;
constexpr int kKvUnroll = 8;  // tokens in flight per warp
constexpr int kKvPart = 2 + kHeadDim;

__global__ void k_kv_append(const float* __restrict__ k_new, const float* __restrict__ v_new,
                            const int32_t* __restrict__ lens, int n_seqs, int n_kv, int64_t L_max,
                            const float2* __restrict__ rope, __nv_bfloat16* __restrict__ kc,
                            __nv_bfloat16* __restrict__ vc) {
  const int64_t width = (int64_t)n_kv * kHeadDim;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_seqs * width;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / width, c = i % width;
    const int64_t pos = lens[b] - 1;
    const float2 cs = rope[pos * 64 + (c % kHeadDim) / 2];
    const float e0 = k_new[i & ~1ll], e1 = k_new[i | 1];
    const float k = (c & 1) ? (e0 * cs.y + e1 * cs.x) : (e0 * cs.x - e1 * cs.y);
    const int64_t dst = (b * L_max + pos) * width + c;
    kc[dst] = __float2bfloat16_rn(k);
    vc[dst] = __float2bfloat16_rn(v_new[i]);
  }
}

XQ_DEVINL void bf16x4(uint2 u, float (&f)[4]) {
  const __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&u.x);
  const __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&u.y);
  f[0] = __low2float(a); f[1] = __high2float(a);
  f[2] = __low2float(b); f[3] = __high2float(b);
}

// One CTA per (sequence, KV head, chunk of tokens). Lane l owns dims 4l..4l+3.
template <int GROUP>
__global__ void __launch_bounds__(kKvThreads)
    k_kv_decode(const __nv_bfloat16* __restrict__ K, const __nv_bfloat16* __restrict__ V,
                int64_t L_max, const int32_t* __restrict__ lens, int n_kv, int chunk_tokens,
                int n_chunks, const float* __restrict__ q_pre, const float2* __restrict__ rope,
                float q_scale, float* __restrict__ partials) {
  const int unit = blockIdx.x;
  const int chunk = unit % n_chunks;
  const int h = (unit / n_chunks) % n_kv;
  const int b = unit / (n_chunks * n_kv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int len = lens[b];
  const int t0 = chunk * chunk_tokens;
  const int t1 = min(t0 + chunk_tokens, len);
  const int64_t width = (int64_t)n_kv * kHeadDim;
  const int n_q = n_kv * GROUP;

  float q[GROUP][4];
  {
    const int pos = len - 1;
    const float2 c0 = rope[(int64_t)pos * 64 + 2 * lane], c1 = rope[(int64_t)pos * 64 + 2 * lane + 1];
#pragma unroll
    for (int gi = 0; gi < GROUP; ++gi) {
      const float4 qq = reinterpret_cast<const float4*>(
          q_pre + ((int64_t)b * n_q + h * GROUP + gi) * kHeadDim)[lane];
      q[gi][0] = (qq.x * c0.x - qq.y * c0.y) * q_scale;
      q[gi][1] = (qq.x * c0.y + qq.y * c0.x) * q_scale;
      q[gi][2] = (qq.z * c1.x - qq.w * c1.y) * q_scale;
      q[gi][3] = (qq.z * c1.y + qq.w * c1.x) * q_scale;
    }
  }
  float m[GROUP], l[GROUP], o[GROUP][4];
#pragma unroll
  for (int gi = 0; gi < GROUP; ++gi) {
    m[gi] = -INFINITY;
    l[gi] = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) o[gi][j] = 0.f;
  }
  const int nw = kKvThreads / 32;
  for (int base = t0 + warp * kKvUnroll; base < t1; base += nw * kKvUnroll) {
    uint2 kr[kKvUnroll], vr[kKvUnroll];
#pragma unroll
    for (int u = 0; u < kKvUnroll; ++u) {
      const int t = min(base + u, t1 - 1);
      const int64_t off = ((int64_t)b * L_max + t) * width + (int64_t)h * kHeadDim;
      kr[u] = reinterpret_cast<const uint2*>(K + off)[lane];
      vr[u] = reinterpret_cast<const uint2*>(V + off)[lane];
    }
#pragma unroll
    for (int gi = 0; gi < GROUP; ++gi) {
      float s[kKvUnroll];
      float mt = -INFINITY;
#pragma unroll
      for (int u = 0; u < kKvUnroll; ++u) {
        float kf[4];
        bf16x4(kr[u], kf);
        const float d = warp_sum(q[gi][0] * kf[0] + q[gi][1] * kf[1] + q[gi][2] * kf[2] + q[gi][3] * kf[3]);
        s[u] = (base + u < t1) ? d : -INFINITY;
        mt = fmaxf(mt, s[u]);
      }
      const float mn = fmaxf(m[gi], mt);
      const float alpha = (m[gi] == -INFINITY) ? 0.f : exp2f(m[gi] - mn);
      l[gi] *= alpha;
#pragma unroll
      for (int j = 0; j < 4; ++j) o[gi][j] *= alpha;
#pragma unroll
      for (int u = 0; u < kKvUnroll; ++u) {
        const float pr = (base + u < t1) ? exp2f(s[u] - mn) : 0.f;
        float vf[4];
        bf16x4(vr[u], vf);
        l[gi] += pr;
#pragma unroll
        for (int j = 0; j < 4; ++j) o[gi][j] = fmaf(pr, vf[j], o[gi][j]);
      }
      m[gi] = mn;
    }
  }
  // merge the 4 warps through shared memory, then one partial per CTA
  __shared__ float s_m[4][GROUP], s_l[4][GROUP], s_o[4][GROUP][kHeadDim];
#pragma unroll
  for (int gi = 0; gi < GROUP; ++gi) {
    if (lane == 0) {
      s_m[warp][gi] = m[gi];
      s_l[warp][gi] = l[gi];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) s_o[warp][gi][4 * lane + j] = o[gi][j];
  }
  __syncthreads();
  const int d = threadIdx.x;  // 128 threads = 128 dims
#pragma unroll
  for (int gi = 0; gi < GROUP; ++gi) {
    float M = -INFINITY;
    for (int w = 0; w < nw; ++w) M = fmaxf(M, s_m[w][gi]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY)
      for (int w = 0; w < nw; ++w) {
        if (s_m[w][gi] == -INFINITY) continue;
        const float wgt = exp2f(s_m[w][gi] - M);
        L = fmaf(wgt, s_l[w][gi], L);
        O = fmaf(wgt, s_o[w][gi][d], O);
      }
    float* dst = partials + (((int64_t)b * n_q + h * GROUP + gi) * n_chunks + chunk) * kKvPart;
    if (d == 0) {
      dst[0] = M;
      dst[1] = L;
    }
    dst[2 + d] = O;
  }
}

template <int GROUP>
static int launch_kv(const __nv_bfloat16* K, const __nv_bfloat16* V, int64_t L_max,
                     const int32_t* lens, int n_seqs, int n_kv, int chunk_tokens, int n_chunks,
                     const float* q_pre, const float2* rope, float q_scale, float* partials,
                     cudaStream_t st) {
  k_kv_decode<GROUP><<<static_cast<unsigned>(n_seqs) * n_kv * n_chunks, kKvThreads, 0, st>>>(
      K, V, L_max, lens, n_kv, chunk_tokens, n_chunks, q_pre, rope, q_scale, partials);
  return check_launch("k_kv_decode");
}

}  // namespace xq

using namespace xq;

extern "C" {

int xq_kv_append(const float* k_new, const float* v_new, const int32_t* seq_lens, int32_t n_seqs,
                 int32_t n_kv_heads, int64_t L_max, const void* rope_cs, void* k_cache,
                 void* v_cache, void* stream) {
  const int64_t n = (int64_t)n_seqs * n_kv_heads * kHeadDim;
  if (n == 0) return XQ_OK;
  const int grid = static_cast<int>((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  k_kv_append<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      k_new, v_new, seq_lens, n_seqs, n_kv_heads, L_max, static_cast<const float2*>(rope_cs),
      static_cast<__nv_bfloat16*>(k_cache), static_cast<__nv_bfloat16*>(v_cache));
  return check_launch("xq_kv_append");
}

int64_t xq_kv_decode_workspace_bytes(int32_t n_seqs, int32_t max_len, int32_t n_kv_heads,
                                     int32_t group, int32_t chunk_tokens) {
  if (chunk_tokens < 1) chunk_tokens = 1;
  const int64_t n_chunks = max_len <= 0 ? 1 : (max_len + chunk_tokens - 1) / chunk_tokens;
  return (int64_t)n_seqs * n_kv_heads * group * n_chunks * kKvPart * sizeof(float);
}

int xq_kv_decode_attend(const void* k_cache, const void* v_cache, int64_t L_max,
                        const int32_t* seq_lens, int32_t n_seqs, int32_t max_len,
                        int32_t n_kv_heads, int32_t group, const float* q_pre,
                        const void* rope_cs, float sm_scale, int32_t chunk_tokens,
                        void* workspace, int64_t workspace_bytes, float* out, void* stream) {
  XQ_REQUIRE(chunk_tokens >= 1, XQ_ECONFIG, "chunk_tokens must be >= 1");
  XQ_REQUIRE(max_len <= L_max, XQ_ESHAPE, "max_len > L_max");
  XQ_REQUIRE(workspace_bytes >= xq_kv_decode_workspace_bytes(n_seqs, max_len, n_kv_heads, group,
                                                             chunk_tokens),
             XQ_ESHAPE, "workspace too small");
  const int n_chunks = max_len <= 0 ? 1 : (max_len + chunk_tokens - 1) / chunk_tokens;
  const float qs = sm_scale * 1.4426950408889634f;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto K = static_cast<const __nv_bfloat16*>(k_cache);
  auto V = static_cast<const __nv_bfloat16*>(v_cache);
  auto rope = static_cast<const float2*>(rope_cs);
  auto parts = static_cast<float*>(workspace);
  int status;
  switch (group) {
    case 1: status = launch_kv<1>(K, V, L_max, seq_lens, n_seqs, n_kv_heads, chunk_tokens, n_chunks, q_pre, rope, qs, parts, st); break;
    case 2: status = launch_kv<2>(K, V, L_max, seq_lens, n_seqs, n_kv_heads, chunk_tokens, n_chunks, q_pre, rope, qs, parts, st); break;
    case 4: status = launch_kv<4>(K, V, L_max, seq_lens, n_seqs, n_kv_heads, chunk_tokens, n_chunks, q_pre, rope, qs, parts, st); break;
    case 8: status = launch_kv<8>(K, V, L_max, seq_lens, n_seqs, n_kv_heads, chunk_tokens, n_chunks, q_pre, rope, qs, parts, st); break;
    default: return fail(XQ_ECONFIG, "unsupported group %d", group);
  }
  if (status != XQ_OK) return status;
  k_combine<<<static_cast<unsigned>(n_seqs) * n_kv_heads * group, kHeadDim, 0, st>>>(parts, n_chunks,
                                                                                  out);
  return check_launch("k_combine(kv)");
}

}  // extern "C"
