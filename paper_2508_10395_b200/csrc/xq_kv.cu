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

// ---------------------------------------------------------------- GQA (GROUP > 1)
// The query heads of one KV head share every K/V row, so the scores and the P.V
// product are small matrix products: mma.sync m16n8k16 (bf16 in, fp32 accumulate)
// with the GROUP query heads as rows 0..GROUP-1 of the 16-row A operand. One warp
// takes 16-token blocks: lane (n = lane/4, c = lane%4) loads 16 bytes of token
// rows n and n+8 at dims 32j+8c.. (j = 0..3), the B-fragment layout of K under a
// dim permutation that Q's A fragments share. V goes through movmatrix.trans
// (token-major rows -> the dims x tokens B fragment) with the same loads, and the
// output columns come back in a known permuted order. The S accumulators are
// re-packed as P's A fragments (rows = heads, k = the block's 16 tokens).
XQ_DEVINL void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

XQ_DEVINL uint32_t movmatrix_trans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

XQ_DEVINL uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

XQ_DEVINL uint32_t word_of(const uint4& u, int w) {
  return w == 0 ? u.x : w == 1 ? u.y : w == 2 ? u.z : u.w;
}

constexpr int kGqaWarps = 4;
constexpr int kGqaStages = 3;                 // per-warp ring of 16-token K/V blocks
constexpr uint32_t kGqaStageBytes = 2 * 16 * 256;  // K rows then V rows, 256 B each
constexpr uint32_t kGqaSmem = kGqaWarps * kGqaStages * kGqaStageBytes;

XQ_DEVINL void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
XQ_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
XQ_DEVINL void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// 16-byte chunk q (0..15) of block row r: odd rows swap chunk halves, so the 8
// lanes of an LDS.128 phase (rows g, g+1 x chunks 4j + c) hit 8 distinct bank groups
XQ_DEVINL uint32_t gqa_off(int r, int q) { return r * 256u + ((q ^ ((r & 1) << 2)) * 16u); }

template <int GROUP>
__global__ void __launch_bounds__(32 * kGqaWarps)
    k_kv_decode_gqa(const __nv_bfloat16* __restrict__ K, const __nv_bfloat16* __restrict__ V,
                    int64_t L_max, const int32_t* __restrict__ lens, int n_kv, int chunk_tokens,
                    int n_chunks, const float* __restrict__ q_pre, const float2* __restrict__ rope,
                    float q_scale, float* __restrict__ partials) {
  static_assert(GROUP >= 2 && GROUP <= 8, "GQA group");
  const int unit = blockIdx.x;
  const int chunk = unit % n_chunks;
  const int h = (unit / n_chunks) % n_kv;
  const int b = unit / (n_chunks * n_kv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;  // fragment row (head) / column pair
  const int len = lens[b];
  const int t0 = chunk * chunk_tokens;
  const int t1 = min(t0 + chunk_tokens, len);
  const int64_t width = (int64_t)n_kv * kHeadDim;
  const int n_q = n_kv * GROUP;

  // Q A fragments (rows = heads): k-step ks = 2j + hf covers dims 32j + 8c + 4hf + {0,1}
  // (a0) and + 2 + {0,1} (a2); rotated by RoPE at the query position, pre-scaled
  uint32_t qa0[8], qa2[8];
  {
    const int pos = len - 1;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qa0[ks] = 0u;
      qa2[ks] = 0u;
    }
    if (g < GROUP) {
      const float* qrow = q_pre + ((int64_t)b * n_q + h * GROUP + g) * kHeadDim;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int d0 = 32 * (ks >> 1) + 8 * c + 4 * (ks & 1);
        float r[4];
#pragma unroll
        for (int pr = 0; pr < 2; ++pr) {  // dims d0 + 2pr, d0 + 2pr + 1: one RoPE pair
          const int d = d0 + 2 * pr;
          const float2 cs = rope[(int64_t)pos * 64 + d / 2];
          const float e0 = qrow[d], e1 = qrow[d + 1];
          r[2 * pr] = (e0 * cs.x - e1 * cs.y) * q_scale;
          r[2 * pr + 1] = (e0 * cs.y + e1 * cs.x) * q_scale;
        }
        qa0[ks] = pack_bf16(r[0], r[1]);
        qa2[ks] = pack_bf16(r[2], r[3]);
      }
    }
  }
  float o[16][4];  // virtual n-tile (j, w) = 4j + w: cols 2c, 2c+1 = dims 32j + 8c + 2w + {0,1}
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m = -INFINITY, l = 0.f;  // row g's running max (log2 domain) / this lane's partial sum

  // per-warp cp.async ring: block k of this warp = tokens tb(k) = t0 + 16 (warp + k nw)
  extern __shared__ __align__(128) uint8_t kv_smem[];
  const uint32_t ring = smem_u32(kv_smem) + warp * kGqaStages * kGqaStageBytes;
  const __nv_bfloat16* Kb = K + (int64_t)b * L_max * width + (int64_t)h * kHeadDim;
  const __nv_bfloat16* Vb = V + (int64_t)b * L_max * width + (int64_t)h * kHeadDim;
  constexpr int kStep = 16 * kGqaWarps;
  auto issue = [&](int tb, int stage) {  // 512 chunks of 16 B, 16 per lane (rows past t1 clamp)
    if (tb < t1) {
      const uint32_t st = ring + stage * kGqaStageBytes;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = lane + 32 * k, r = i >> 4, q = i & 15;
        const int64_t t = min(tb + r, t1 - 1);
        cp_async16(st + gqa_off(r, q), Kb + t * width + 8 * q);
        cp_async16(st + 4096u + gqa_off(r, q), Vb + t * width + 8 * q);
      }
    }
    cp_async_commit();
  };
  const int tfirst = t0 + 16 * warp;
#pragma unroll
  for (int k = 0; k < kGqaStages - 1; ++k) issue(tfirst + k * kStep, k);
  int stage = 0;
  for (int tb = tfirst; tb < t1; tb += kStep) {
    cp_async_wait<kGqaStages - 2>();
    __syncwarp();
    const uint32_t st = ring + stage * kGqaStageBytes;
    uint4 kr[2][4], vr[2][4];
#pragma unroll
    for (int tau = 0; tau < 2; ++tau)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        kr[tau][j] = lds128(st + gqa_off(8 * tau + g, 4 * j + c));
        vr[tau][j] = lds128(st + 4096u + gqa_off(8 * tau + g, 4 * j + c));
      }
    // S = Q K^T for tokens tb + 8 tau + (2c, 2c+1) in rows g (c[0], c[1])
    float sc[2][4];
#pragma unroll
    for (int tau = 0; tau < 2; ++tau) {
      sc[tau][0] = sc[tau][1] = sc[tau][2] = sc[tau][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        mma_bf16_16816(sc[tau], qa0[ks], qa2[ks], word_of(kr[tau][ks >> 1], 2 * (ks & 1)),
                       word_of(kr[tau][ks >> 1], 2 * (ks & 1) + 1));
    }
    float s[4];
#pragma unroll
    for (int tau = 0; tau < 2; ++tau)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        s[2 * tau + e] = (tb + 8 * tau + 2 * c + e < t1) ? sc[tau][e] : -INFINITY;
    float bm = fmaxf(fmaxf(s[0], s[1]), fmaxf(s[2], s[3]));
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 1));
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
    const float mn = fmaxf(m, bm);  // finite: every block holds at least one valid token
    const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - mn);
    m = mn;
    float p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = exp2f(s[i] - mn);
    l = fmaf(l, alpha, (p[0] + p[1]) + (p[2] + p[3]));
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      o[i][0] *= alpha;
      o[i][1] *= alpha;
    }
    const uint32_t pa0 = pack_bf16(p[0], p[1]), pa2 = pack_bf16(p[2], p[3]);
    // O += P V: B fragment of virtual tile (j, w) = movmatrix.trans of word w of the
    // token-half rows (k = tokens 2c, 2c+1 of each half)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int w = 0; w < 4; ++w)
        mma_bf16_16816(o[4 * j + w], pa0, pa2, movmatrix_trans(word_of(vr[0][j], w)),
                       movmatrix_trans(word_of(vr[1][j], w)));
    __syncwarp();  // every lane has read this stage before it is refilled
    const int ns = stage == 0 ? kGqaStages - 1 : stage - 1;  // (stage + S - 1) % S
    issue(tb + (kGqaStages - 1) * kStep, ns);
    stage = stage + 1 == kGqaStages ? 0 : stage + 1;
  }
  cp_async_wait<0>();
  l += __shfl_xor_sync(0xffffffffu, l, 1);
  l += __shfl_xor_sync(0xffffffffu, l, 2);

  // merge the warps through shared memory, one partial per (head, CTA)
  __shared__ float s_m[kGqaWarps][GROUP], s_l[kGqaWarps][GROUP], s_o[kGqaWarps][GROUP][kHeadDim];
  if (g < GROUP) {
    if (c == 0) {
      s_m[warp][g] = m;
      s_l[warp][g] = l;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int d = 32 * j + 8 * c + 2 * w;
        s_o[warp][g][d] = o[4 * j + w][0];
        s_o[warp][g][d + 1] = o[4 * j + w][1];
      }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < GROUP * kHeadDim; idx += 32 * kGqaWarps) {
    const int gi = idx / kHeadDim, d = idx % kHeadDim;
    float M = -INFINITY;
    for (int w = 0; w < kGqaWarps; ++w) M = fmaxf(M, s_m[w][gi]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY)
      for (int w = 0; w < kGqaWarps; ++w) {
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
  if constexpr (GROUP == 1) {
    k_kv_decode<GROUP><<<static_cast<unsigned>(n_seqs) * n_kv * n_chunks, kKvThreads, 0, st>>>(
        K, V, L_max, lens, n_kv, chunk_tokens, n_chunks, q_pre, rope, q_scale, partials);
  } else {
    if (int s = ensure_smem(reinterpret_cast<const void*>(k_kv_decode_gqa<GROUP>), kGqaSmem,
                           "cudaFuncSetAttribute(kv_decode_gqa)"))
      return s;
    k_kv_decode_gqa<GROUP><<<static_cast<unsigned>(n_seqs) * n_kv * n_chunks, 32 * kGqaWarps,
                             kGqaSmem, st>>>(K, V, L_max, lens, n_kv, chunk_tokens, n_chunks, q_pre, rope,
                                   q_scale, partials);
  }
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
