// fp16-KV decode baseline on the same GPU: the reference's FullPrecisionCache
// semantics (cache.py:302-323) with post-RoPE bf16 K/V resident in HBM
// (standard practice, mathematically identical to re-rotating pre-RoPE K each
// step) and a split-K flash-decode that streams K/V once at HBM bandwidth.
#include <math.h>

#include "xq_common.cuh"
#include "xq_host.h"

namespace xq {

__global__ void k_combine(const float* __restrict__ partials, int n_parts, float* __restrict__ out);

constexpr int kKvThreads = 256;
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

XQ_DEVINL void bf16x8(uint4 u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
    f[2 * i] = __low2float(h);
    f[2 * i + 1] = __high2float(h);
  }
}

// One CTA per (sequence, KV head, chunk of tokens). Each half-warp streams its
// own tokens: lane l of a half owns dims 8l..8l+7 (16-byte loads, one 256-byte
// K row per half-warp load), kKvUnroll rows in flight per half-warp.
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
  const int half = lane >> 4, hl = lane & 15;
  const int stream = warp * 2 + half;  // 0 .. 2*nw-1
  constexpr int kNw = kKvThreads / 32;
  constexpr int kStreams = 2 * kNw;
  const int len = lens[b];
  const int t0 = chunk * chunk_tokens;
  const int t1 = min(t0 + chunk_tokens, len);
  const int64_t width = (int64_t)n_kv * kHeadDim;
  const int n_q = n_kv * GROUP;

  float q[GROUP][8];
  {
    const int pos = len - 1;
#pragma unroll
    for (int gi = 0; gi < GROUP; ++gi) {
      const float4* qp = reinterpret_cast<const float4*>(
          q_pre + ((int64_t)b * n_q + h * GROUP + gi) * kHeadDim + 8 * hl);
      const float4 a = qp[0], c = qp[1];
      const float e[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 cs = rope[(int64_t)pos * 64 + 4 * hl + j];
        q[gi][2 * j] = (e[2 * j] * cs.x - e[2 * j + 1] * cs.y) * q_scale;
        q[gi][2 * j + 1] = (e[2 * j] * cs.y + e[2 * j + 1] * cs.x) * q_scale;
      }
    }
  }
  float m[GROUP], l[GROUP], o[GROUP][8];
#pragma unroll
  for (int gi = 0; gi < GROUP; ++gi) {
    m[gi] = -INFINITY;
    l[gi] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) o[gi][j] = 0.f;
  }
  const __nv_bfloat16* Kb = K + (int64_t)b * L_max * width + (int64_t)h * kHeadDim + 8 * hl;
  const __nv_bfloat16* Vb = V + (int64_t)b * L_max * width + (int64_t)h * kHeadDim + 8 * hl;
  // warp-uniform trip count (the 16-lane shuffles use the full mask): warp w
  // takes blocks of 2*kKvUnroll tokens, half-warp `half` the tokens 2u + half
  for (int wbase = t0 + warp * 2 * kKvUnroll; wbase < t1; wbase += kNw * 2 * kKvUnroll) {
    const int base = wbase + half;
    uint4 kr[kKvUnroll], vr[kKvUnroll];
#pragma unroll
    for (int u = 0; u < kKvUnroll; ++u) {
      const int t = min(base + 2 * u, t1 - 1);
      kr[u] = __ldg(reinterpret_cast<const uint4*>(Kb + (int64_t)t * width));
      vr[u] = __ldg(reinterpret_cast<const uint4*>(Vb + (int64_t)t * width));
    }
#pragma unroll
    for (int gi = 0; gi < GROUP; ++gi) {
      float s[kKvUnroll];
      float mt = -INFINITY;
#pragma unroll
      for (int u = 0; u < kKvUnroll; ++u) {
        float kf[8];
        bf16x8(kr[u], kf);
        float d = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) d = fmaf(q[gi][j], kf[j], d);
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
        s[u] = (base + 2 * u < t1) ? d : -INFINITY;
        mt = fmaxf(mt, s[u]);
      }
      const float mn = fmaxf(m[gi], mt);
      const float alpha = (m[gi] == -INFINITY) ? 0.f : exp2f(m[gi] - mn);
      l[gi] *= alpha;
#pragma unroll
      for (int j = 0; j < 8; ++j) o[gi][j] *= alpha;
#pragma unroll
      for (int u = 0; u < kKvUnroll; ++u) {
        const float pr = (base + 2 * u < t1) ? exp2f(s[u] - mn) : 0.f;
        float vf[8];
        bf16x8(vr[u], vf);
        l[gi] += pr;
#pragma unroll
        for (int j = 0; j < 8; ++j) o[gi][j] = fmaf(pr, vf[j], o[gi][j]);
      }
      m[gi] = mn;
    }
  }
  // merge the 2*nw half-warp streams through shared memory, one partial per CTA
  __shared__ float s_m[kStreams][GROUP], s_l[kStreams][GROUP], s_o[kStreams][GROUP][kHeadDim];
#pragma unroll
  for (int gi = 0; gi < GROUP; ++gi) {
    if (hl == 0) {
      s_m[stream][gi] = m[gi];
      s_l[stream][gi] = l[gi];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s_o[stream][gi][8 * hl + j] = o[gi][j];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < GROUP * kHeadDim; idx += kKvThreads) {
    const int gi = idx / kHeadDim, d = idx % kHeadDim;
    float M = -INFINITY;
    for (int w = 0; w < kStreams; ++w) M = fmaxf(M, s_m[w][gi]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY)
      for (int w = 0; w < kStreams; ++w) {
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
    default: return fail(XQ_ECONFIG, "unsupported group %d", group);
  }
  if (status != XQ_OK) return status;
  k_combine<<<static_cast<unsigned>(n_seqs) * n_kv_heads * group, kHeadDim, 0, st>>>(parts, n_chunks,
                                                                                  out);
  return check_launch("k_combine(kv)");
}

}  // extern "C"
