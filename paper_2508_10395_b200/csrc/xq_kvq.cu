// Quantized-KV decode baseline "kvq" (QuantizedKvCache, cache.py:326-360),
// the paper's KIVI-style comparison at equal bits: pre-RoPE K quantized per
// channel, V per token, both with residual buffers while decoding
// (cache.py:336-342, the newest < G tokens of each stay in float32).
//
// One CTA per (sequence, chunk of tokens). Per 64-token tile the CTA stages
// the tile's cos/sin rows once, then for each KV head dequantizes the K tile
// into shared memory, rotates it (RoPE at the cached positions,
// cache.py:357-360 + linalg.py:58-95), scores it against the head's query
// heads, updates the per-head online softmax, dequantizes the V tile and
// accumulates p.V. Split partials (m, l, o) per (sequence, query head, chunk)
// are merged by k_combine. HBM traffic per token: 2*kv_width*(bits/8) code
// bytes + the scale / zero-point grids.
#include <math.h>

#include "xq_common.cuh"
#include "xq_host.h"
#include "xq_layout.cuh"

namespace xq {

__global__ void k_combine(const float* __restrict__ partials, int n_parts, float* __restrict__ out);

namespace kvq {

constexpr int kT = 64;          // tokens per tile
constexpr int kThreads = 256;
constexpr int kPart = 2 + kHeadDim;
constexpr int kPad = kHeadDim + 4;  // row stride of the K/V tiles (floats)

struct Params {
  const uint8_t* k_codes;  // [n_seqs*L_max][row_bytes]
  const __half* k_params;  // planar per-channel [rows/G][2][kvw], producer order (xq_layout.cuh)
  const float* k_resid;    // [n_seqs][G][kvw]
  const uint8_t* v_codes;
  const __half2* v_params;  // per-token [rows][vp_stride] (scale, zp)
  const float* v_resid;
  const int32_t* k_nflushed;  // per sequence: tokens < n are in the K codes, the rest in k_resid
  const int32_t* v_nflushed;  // the same for V (prefill quantizes V whole, K by groups)
  int64_t row_bytes, vp_stride, L_max;
  int bits, G;
  const int32_t* seq_lens;
  int n_kv, group, kvw;
  const float* q_pre;
  const float2* rope;  // position-major [n_pos][64]
  float q_scale;
  int chunk_tokens, n_chunks;
  float* partials;  // [n_seqs*n_q][n_chunks][130]
};

// 16 consecutive codes starting at element c0 of a packed row (c0*bits % 8 == 0).
XQ_DEVINL void load16(const uint8_t* row, int64_t c0, int bits, uint32_t (&out)[16]) {
  const uint8_t* p = row + (c0 * bits) / 8;
  uint64_t lo = 0, hi = 0;
  const int nbytes = 2 * bits;  // 16 codes
  for (int i = 0; i < nbytes && i < 8; ++i) lo |= static_cast<uint64_t>(p[i]) << (8 * i);
  for (int i = 8; i < nbytes; ++i) hi |= static_cast<uint64_t>(p[i]) << (8 * (i - 8));
  const uint32_t mask = (1u << bits) - 1u;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int b = i * bits;
    uint32_t v;
    if (b + bits <= 64) v = static_cast<uint32_t>(lo >> b);
    else if (b >= 64) v = static_cast<uint32_t>(hi >> (b - 64));
    else v = static_cast<uint32_t>((lo >> b) | (hi << (64 - b)));
    out[i] = v & mask;
  }
}

__global__ void __launch_bounds__(kThreads) k_kvq_decode(const Params p) {
  extern __shared__ float sm[];
  const int n_q = p.n_kv * p.group;
  float* q_s = sm;                                          // [n_q][128]
  float* o_s = q_s + n_q * kHeadDim;                        // [n_q][128]
  float2* cs_s = reinterpret_cast<float2*>(o_s + n_q * kHeadDim);  // [kT][64]
  __half2* kp_s = reinterpret_cast<__half2*>(cs_s + kT * 64);      // [kvw] (scale, zp), natural order
  float* kt_s = reinterpret_cast<float*>(kp_s + p.kvw);     // [kT][kPad]
  float* vt_s = kt_s + kT * kPad;                           // [kT][kPad]
  float* sc_s = vt_s + kT * kPad;                           // [group][kT]
  float* al_s = sc_s + p.group * kT;                        // [group] tile rescale
  float* m_s = al_s + p.group;                              // [n_q]
  float* l_s = m_s + n_q;                                   // [n_q]

  const int b = blockIdx.x / p.n_chunks, chunk = blockIdx.x % p.n_chunks;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int len = p.seq_lens[b];
  const int t_begin = chunk * p.chunk_tokens;
  const int t_end = min(len, t_begin + p.chunk_tokens);
  const int nfl = p.k_nflushed[b], vnfl = p.v_nflushed[b];
  const int pos = len - 1;
  // q rotated to position len-1 (model.py:234), scaled into the log2 domain
  for (int i = tid; i < n_q * kHeadDim; i += kThreads) {
    const int h = i / kHeadDim, dd = i % kHeadDim;
    const float* qp = p.q_pre + ((int64_t)b * n_q + h) * kHeadDim;
    const float2 cs = p.rope[(int64_t)(pos < 0 ? 0 : pos) * 64 + dd / 2];
    const float e0 = qp[dd & ~1], e1 = qp[dd | 1];
    q_s[i] = ((dd & 1) ? (e0 * cs.y + e1 * cs.x) : (e0 * cs.x - e1 * cs.y)) * p.q_scale;
    o_s[i] = 0.f;
  }
  for (int h = tid; h < n_q; h += kThreads) {
    m_s[h] = -INFINITY;
    l_s[h] = 0.f;
  }
  int kp_group = -1;
  const int bs = perm_block(XQ_A_CODES_CHANNEL, p.bits);
  for (int t0 = t_begin; t0 < t_end; t0 += kT) {
    __syncthreads();
    for (int i = tid; i < kT * 64; i += kThreads) {  // the tile's cos/sin rows
      const int r = i >> 6, j = i & 63;
      const int t = min(t0 + r, len - 1);
      cs_s[i] = p.rope[(int64_t)t * 64 + j];
    }
    const int grp = t0 / p.G;  // tiles never straddle a group (G % kT == 0)
    if (grp != kp_group && t0 < nfl) {
      const __half* prow = p.k_params + ((int64_t)b * p.L_max / p.G + grp) * 2 * p.kvw;
      for (int c = tid; c < p.kvw; c += kThreads) {
        const int ppos = (c / bs) * bs + perm_position(c % bs, bs);
        kp_s[c] = __halves2half2(prow[ppos], prow[p.kvw + ppos]);
      }
      kp_group = grp;
    }
    __syncthreads();
    const int r = tid >> 2, part = tid & 3;  // token row of the tile, 32-channel quarter
    const int t = t0 + r;
    const bool valid = t < t_end;
    const int64_t arow = (int64_t)b * p.L_max + t;
    for (int kvh = 0; kvh < p.n_kv; ++kvh) {
      // ---- K tile: dequant (per-channel params) or residual row, then RoPE
      const int c0 = kvh * kHeadDim + part * 32;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float v[16];
        const int cc = c0 + half * 16;
        if (valid && t < nfl) {
          uint32_t code[16];
          load16(p.k_codes + arow * p.row_bytes, cc, p.bits, code);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 sz = __half22float2(kp_s[cc + i]);
            v[i] = fmaf(static_cast<float>(code[i]), sz.x, sz.y);
          }
        } else if (valid) {
          const float* rr = p.k_resid + ((int64_t)b * p.G + (t - nfl)) * p.kvw + cc;
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = rr[i];
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        const int d0 = part * 32 + half * 16;  // dim within the head
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const float2 cs = cs_s[r * 64 + (d0 + i) / 2];
          kt_s[r * kPad + d0 + i] = v[i] * cs.x - v[i + 1] * cs.y;
          kt_s[r * kPad + d0 + i + 1] = v[i] * cs.y + v[i + 1] * cs.x;
        }
      }
      // ---- V tile: per-token params of this head's 128-channel group (G = 128)
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float v[16];
        const int cc = c0 + half * 16;
        if (valid && t < vnfl) {
          uint32_t code[16];
          load16(p.v_codes + arow * p.row_bytes, cc, p.bits, code);
          const float2 sz = __half22float2(p.v_params[arow * p.vp_stride + cc / p.G]);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = fmaf(static_cast<float>(code[i]), sz.x, sz.y);
        } else if (valid) {
          const float* rr = p.v_resid + ((int64_t)b * p.G + (t - vnfl)) * p.kvw + cc;
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = rr[i];
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        const int d0 = part * 32 + half * 16;
#pragma unroll
        for (int i = 0; i < 16; ++i) vt_s[r * kPad + d0 + i] = v[i];
      }
      __syncthreads();
      // ---- scores of the head's query heads (4 threads per token)
      for (int gi = 0; gi < p.group; ++gi) {
        const float* qh = q_s + (kvh * p.group + gi) * kHeadDim + part * 32;
        const float* kr = kt_s + r * kPad + part * 32;
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) s = fmaf(qh[i], kr[i], s);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (part == 0) sc_s[gi * kT + r] = valid ? s : -INFINITY;
      }
      __syncthreads();
      // ---- online softmax per query head (one warp each, 2 tokens per lane)
      for (int gi = warp; gi < p.group; gi += kThreads / 32) {
        const int h = kvh * p.group + gi;
        const float s0 = sc_s[gi * kT + lane], s1 = sc_s[gi * kT + 32 + lane];
        const float mo = m_s[h];
        const float mn = fmaxf(mo, warp_max(fmaxf(s0, s1)));
        const float p0 = (s0 == -INFINITY) ? 0.f : exp2f(s0 - mn);
        const float p1 = (s1 == -INFINITY) ? 0.f : exp2f(s1 - mn);
        const float alpha = (mo == -INFINITY) ? 0.f : exp2f(mo - mn);
        const float ls = warp_sum(p0 + p1);
        sc_s[gi * kT + lane] = p0;
        sc_s[gi * kT + 32 + lane] = p1;
        if (lane == 0) {
          al_s[gi] = alpha;
          m_s[h] = mn;
          l_s[h] = l_s[h] * alpha + ls;
        }
      }
      __syncthreads();
      // ---- o = o*alpha + p.V (thread = (query head, channel))
      for (int i = tid; i < p.group * kHeadDim; i += kThreads) {
        const int gi = i / kHeadDim, c = i % kHeadDim;
        const float* pp = sc_s + gi * kT;
        float acc = 0.f;
#pragma unroll 8
        for (int rr = 0; rr < kT; ++rr) acc = fmaf(pp[rr], vt_s[rr * kPad + c], acc);
        float* o = o_s + (kvh * p.group + gi) * kHeadDim + c;
        *o = *o * al_s[gi] + acc;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  for (int i = tid; i < n_q * kHeadDim; i += kThreads) {
    const int h = i / kHeadDim, c = i % kHeadDim;
    float* dst = p.partials + (((int64_t)b * n_q + h) * p.n_chunks + chunk) * kPart;
    if (c == 0) {
      dst[0] = m_s[h];
      dst[1] = l_s[h];
    }
    dst[2 + c] = o_s[i];
  }
}

}  // namespace kvq
}  // namespace xq

using namespace xq;
using namespace xq::kvq;

extern "C" {

int64_t xq_kvq_workspace_bytes(int32_t n_seqs, int32_t max_len, int32_t n_q_heads,
                               int32_t chunk_tokens) {
  if (chunk_tokens < kT) chunk_tokens = kT;
  const int64_t n_chunks = max_len <= 0 ? 1 : (max_len + chunk_tokens - 1) / chunk_tokens;
  return (int64_t)n_seqs * n_q_heads * n_chunks * kPart * (int64_t)sizeof(float);
}

int xq_kvq_decode_attend(const uint8_t* k_codes, const void* k_params, const float* k_resid,
                         const uint8_t* v_codes, const void* v_params, const float* v_resid,
                         const int32_t* k_nflushed, const int32_t* v_nflushed, int32_t bits,
                         int32_t group_size,
                         int64_t row_bytes, int64_t L_max, const int32_t* seq_lens, int32_t n_seqs,
                         int32_t max_len, int32_t n_kv_heads, int32_t group, const float* q_pre,
                         const void* rope_cs, float sm_scale, int32_t chunk_tokens,
                         void* workspace, int64_t workspace_bytes, float* out, void* stream) {
  XQ_REQUIRE(valid_bits(bits), XQ_ECONFIG, "bad bits %d", bits);
  XQ_REQUIRE(group_size == 128, XQ_ECONFIG, "kvq decode is specialised for group_size 128");
  XQ_REQUIRE(L_max % group_size == 0, XQ_ECONFIG, "per-channel K needs L_max % 128 == 0");
  XQ_REQUIRE(n_seqs >= 1 && n_kv_heads >= 1 && group >= 1, XQ_ESHAPE, "empty batch");
  XQ_REQUIRE(max_len >= 1 && max_len <= L_max, XQ_ESHAPE, "max_len out of range");
  if (chunk_tokens < kT) chunk_tokens = kT;
  chunk_tokens = (chunk_tokens + kT - 1) / kT * kT;
  XQ_REQUIRE(workspace_bytes >= xq_kvq_workspace_bytes(n_seqs, max_len, n_kv_heads * group,
                                                       chunk_tokens),
             XQ_ESHAPE, "workspace too small");
  const int kvw = n_kv_heads * kHeadDim;
  XQ_REQUIRE(row_bytes == row_bytes_for(kvw, bits), XQ_ESHAPE, "row_bytes mismatch");
  Params p;
  p.k_codes = k_codes;
  p.k_params = static_cast<const __half*>(k_params);
  p.k_resid = k_resid;
  p.v_codes = v_codes;
  p.v_params = static_cast<const __half2*>(v_params);
  p.v_resid = v_resid;
  p.k_nflushed = k_nflushed;
  p.v_nflushed = v_nflushed;
  p.row_bytes = row_bytes;
  p.vp_stride = param_stride(kvw, group_size);
  p.L_max = L_max;
  p.bits = bits;
  p.G = group_size;
  p.seq_lens = seq_lens;
  p.n_kv = n_kv_heads;
  p.group = group;
  p.kvw = kvw;
  p.q_pre = q_pre;
  p.rope = static_cast<const float2*>(rope_cs);
  p.q_scale = sm_scale * 1.4426950408889634f;
  p.chunk_tokens = chunk_tokens;
  p.n_chunks = (max_len + chunk_tokens - 1) / chunk_tokens;
  p.partials = static_cast<float*>(workspace);
  const int n_q = n_kv_heads * group;
  const size_t smem = sizeof(float) * (2 * (size_t)n_q * kHeadDim + 2 * kT * 64 + kvw +
                                       2 * kT * kPad + (size_t)group * kT + group + 2 * n_q);
  XQ_REQUIRE(smem <= 227 * 1024, XQ_ESHAPE, "kvq decode: shared memory plan does not fit");
  static size_t configured = 0;
  if (configured < smem) {
    if (cudaFuncSetAttribute(k_kvq_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return check_launch("cudaFuncSetAttribute(kvq)");
    configured = smem;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_kvq_decode<<<n_seqs * p.n_chunks, kThreads, smem, st>>>(p);
  int status = check_launch("k_kvq_decode");
  if (status != XQ_OK) return status;
  k_combine<<<static_cast<unsigned>(n_seqs) * n_q, kHeadDim, 0, st>>>(p.partials, p.n_chunks, out);
  return check_launch("k_combine(kvq)");
}

}  // extern "C"
