// Quantized-KV decode baseline "kvq" (QuantizedKvCache, cache.py:326-360),
// the paper's KIVI-style comparison at equal bits: pre-RoPE K quantized per
// channel, V per token, both with residual buffers while decoding
// (cache.py:336-342, the newest < G tokens of each stay in float32).
//
// A split-K flash-decode that streams the codes once: one CTA per (sequence,
// KV head, chunk of tokens), half-warps on tokens, dequantization and RoPE of
// K in registers (k_kvq_decode below), split partials merged by k_combine.
// HBM traffic per token and layer: 2*kv_width*bits/8 code bytes + the scale /
// zero-point grids.
#include <math.h>

#include "xq_common.cuh"
#include "xq_host.h"
#include "xq_layout.cuh"

namespace xq {

__global__ void k_combine(const float* __restrict__ partials, int n_parts, float* __restrict__ out);

namespace kvq {

constexpr int kT = 128;  // token chunks are whole K groups (G = 128)
constexpr int kThreads = 256;
constexpr int kPart = 2 + kHeadDim;

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

// `nbytes` (<= 4) bytes of a packed row starting at byte `off` (any alignment;
// rows are 8-byte aligned): two aligned 32-bit loads and a funnel shift.
XQ_DEVINL uint32_t load_bits(const uint8_t* row, int64_t off, int nbytes) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(row + (off & ~int64_t(3)));
  // the second word only when the bits cross into it (never past the row end)
  const uint32_t lo = __ldg(w), hi = ((off & 3) + nbytes > 4) ? __ldg(w + 1) : 0u;
  return __funnelshift_r(lo, hi, static_cast<uint32_t>(off & 3) * 8u);
}

// The 8 codes of channels 8*hl .. 8*hl+7 of head h in a packed row, raw
// (BITS*8 bits; for 8-bit two words).
template <int BITS>
XQ_DEVINL uint2 raw8(const uint8_t* row, int h, int hl) {
  const int64_t off = (int64_t)(h * kHeadDim + 8 * hl) * BITS / 8;  // byte-aligned: 8 codes
  if constexpr (BITS == 8) return __ldg(reinterpret_cast<const uint2*>(row + off));
  return make_uint2(load_bits(row, off, BITS), 0u);
}
template <int BITS>
XQ_DEVINL uint32_t code_j(uint2 raw, int j) {
  if constexpr (BITS == 8) return ((j < 4 ? raw.x : raw.y) >> (8 * (j & 3))) & 0xFFu;
  return (raw.x >> (BITS * j)) & ((1u << BITS) - 1u);
}

// One CTA per (sequence, KV head, chunk of tokens); each half-warp streams its
// own tokens (lane hl owns dims 8hl..8hl+7, kUnroll tokens in flight), like the
// fp16-KV kernel but on codes: K dequantized with the per-channel (scale, zp)
// of the token's group, rotated at its position by angle addition
// cos/sin((t0 + r) theta) from the 16-token block base (global table, one
// coalesced row per block) and a shared offset table r < 16; V dequantized
// with its per-token (scale, zp).
constexpr int kNw = kThreads / 32;
constexpr int kStreams = 2 * kNw;
constexpr int kStages = 3;  // per-warp cp.async ring of token blocks

template <int GROUP>
constexpr int unroll_for() { return GROUP >= 4 ? 4 : 8; }  // tokens per half-warp per block
// one ring stage: a block's K code rows, V code rows (16*BITS bytes per token for
// one head) and V (scale, zp)
template <int BITS, int GROUP>
constexpr uint32_t stage_bytes() { return 2u * 2 * unroll_for<GROUP>() * (16 * BITS + 2); }
template <int BITS, int GROUP>
constexpr uint32_t smem_bytes() { return kNw * kStages * stage_bytes<BITS, GROUP>(); }

XQ_DEVINL void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
XQ_DEVINL void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
XQ_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
XQ_DEVINL void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Codes to floats without a conversion instruction: code j of the lane's 8 is ORed
// in place into the mantissa of 2^23 (one LOP3), 2^23 subtracted, giving the exact
// value code * 2^code_sh(j). Codes whose field would reach the exponent (bit 23) are
// taken from the word shifted right by pre_shift first. The 2^-code_sh factors fold
// into the K scales and into a final rescale of the V accumulators (powers of two:
// the products and sums are the same floats as with the plain codes).
template <int BITS>
constexpr int code_off(int j) { return BITS == 8 ? 8 * (j & 3) : BITS * j; }  // bit in its word
template <int BITS>
constexpr int pre_shift(int j) {
  return code_off<BITS>(j) + BITS - 1 <= 22 ? 0 : BITS * ((23 - BITS) / BITS + 1);
}
template <int BITS>
constexpr int code_sh(int j) { return code_off<BITS>(j) - pre_shift<BITS>(j); }

XQ_DEVINL uint32_t or_magic(uint32_t w) {
  uint32_t r;  // opaque to the optimizer, which would refold the AND / OR pair
  asm("or.b32 %0, %1, 0x4B000000;" : "=r"(r) : "r"(w));
  return r;
}
template <int BITS>
XQ_DEVINL float2 code_pair(uint2 raw, int j) {
  float f[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int c = 2 * j + e;
    const uint32_t w = ((BITS == 8 && c >= 4) ? raw.y : raw.x) >> pre_shift<BITS>(c);
    const uint32_t mask = ((1u << BITS) - 1u) << code_sh<BITS>(c);
    // (w | C) & (mask | C) == (w & mask) | C: one AND per code once the word carries C
    f[e] = __uint_as_float(or_magic(w) & (mask | 0x4B000000u));
  }
  return __fadd2_rn(make_float2(f[0], f[1]), make_float2(-8388608.f, -8388608.f));
}
template <int BITS>
XQ_DEVINL float code_unit(int c) { return __int_as_float((127 - code_sh<BITS>(c)) << 23); }  // 2^-sh

// Sums of N values per lane over the 16 lanes of a half-warp, transposed: each
// exchange step halves the values a lane carries, so N = 8 or 16 sums take N - 1
// (+1) shuffles instead of 4N. Lane hl ends with the sum of value hl >> (4 - log2 N).
template <int N>
XQ_DEVINL float xreduce16(float (&v)[N], int hl) {
#pragma unroll
  for (int st = 0; st < 4; ++st) {
    const int m = 8 >> st, n = N >> (st + 1);
    if (n >= 1) {
      const bool up = (hl & m) != 0;
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const float send = up ? v[i] : v[i + n];
        const float keep = up ? v[i + n] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
      }
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
    }
  }
  return v[0];
}

XQ_DEVINL __half2 from_u32h2(uint32_t u) { return *reinterpret_cast<const __half2*>(&u); }

// raw8 from a staged row (shared address of the head's 16*BITS code bytes)
template <int BITS>
XQ_DEVINL uint2 raw8_s(uint32_t row, int hl) {
  if constexpr (BITS == 8) return lds64(row + 8u * hl);
  const uint32_t off = static_cast<uint32_t>(BITS * hl);
  const uint32_t a = row + (off & ~3u);
  const uint32_t lo = lds32(a), hi = ((off & 3u) + BITS > 4u) ? lds32(a + 4u) : 0u;
  return make_uint2(__funnelshift_r(lo, hi, (off & 3u) * 8u), 0u);
}

template <int BITS, int GROUP>
__global__ void __launch_bounds__(kThreads, 2) k_kvq_decode(const Params p) {
  constexpr int kUnroll = unroll_for<GROUP>();
  constexpr int kBlk = 2 * kUnroll;
  constexpr uint32_t kRowB = 16 * BITS;
  constexpr uint32_t kStageB = stage_bytes<BITS, GROUP>();
  const int unit = blockIdx.x;
  const int chunk = unit % p.n_chunks;
  const int h = (unit / p.n_chunks) % p.n_kv;
  const int b = unit / (p.n_chunks * p.n_kv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, hl = lane & 15;
  const int stream = warp * 2 + half;
  const int len = p.seq_lens[b];
  const int t0 = chunk * p.chunk_tokens;
  const int t1 = min(t0 + p.chunk_tokens, len);
  const int n_q = p.n_kv * GROUP;
  const int nfl = p.k_nflushed[b], vnfl = p.v_nflushed[b];

  constexpr int kN = GROUP * kUnroll;  // (head, token) scores per half-warp and block
  constexpr int kLogN = kN == 16 ? 4 : 3;
  static_assert(kN == 8 || kN == 16, "kvq: 8 or 16 scores per half-warp block");
  // lane-major tables ([.][j][hl] holds channel pair 4hl + j): conflict-free reads
  // cos/sin(r theta_c), r < 16, lane-major: [r][jp][hl] holds the lane's channel pairs
  // 4hl + 2jp and 4hl + 2jp + 1 (one conflict-free 16-byte read per two pairs)
  __shared__ __align__(16) float2 s_off[16][2][16][2];
  for (int i = threadIdx.x; i < 16 * 64; i += kThreads) {
    const int c = i & 63;
    s_off[i >> 6][(c & 3) >> 1][c >> 2][c & 1] = p.rope[i];
  }
  // the query heads rotated to their position and scaled (log2 domain); each warp
  // re-rotates its lanes' channel pairs to every block base below
  __shared__ float2 s_q[GROUP][64];
  for (int i = threadIdx.x; i < GROUP * 64; i += kThreads) {
    const int gi = i >> 6, c = i & 63;
    const float2 cs = p.rope[(int64_t)(len - 1) * 64 + c];
    const float2 e = reinterpret_cast<const float2*>(
        p.q_pre + ((int64_t)b * n_q + h * GROUP + gi) * kHeadDim)[c];
    s_q[gi][(c & 3) * 16 + (c >> 2)] = make_float2((e.x * cs.x - e.y * cs.y) * p.q_scale,
                                                   (e.x * cs.y + e.y * cs.x) * p.q_scale);
  }
  __syncthreads();
  // o = sum_t p_t * (code_t * s_t + z_t) is accumulated as sum_t (p_t s_t) code_t in
  // float2 pairs plus a per-head sum_t p_t z_t (pz), added to every channel at the end
  float m[GROUP], l[GROUP], pz[GROUP];
  float2 o[GROUP][4];
#pragma unroll
  for (int gi = 0; gi < GROUP; ++gi) {
    m[gi] = -INFINITY;
    l[gi] = 0.f;
    pz[gi] = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) o[gi][j] = make_float2(0.f, 0.f);
  }
  // this lane's (head, token) after the transposed reduction
  const int my = hl >> (4 - kLogN), my_g = my / kUnroll, my_u = my % kUnroll;
  const int64_t row0 = (int64_t)b * p.L_max;
  const int bs = perm_block(XQ_A_CODES_CHANNEL, BITS);
  int cur_grp = -1;
  // (scale * 2^-code_sh, zp) of this lane's 8 K channels for the current token group
  float2 kps[4], kpz[4];
  // per-warp cp.async ring of token blocks: warp w takes blocks of kBlk = 2*kUnroll
  // tokens (16-aligned: one RoPE base, one K group); half-warp `half` the tokens
  // 2u + half (rows past t1 clamp to t1 - 1 and are masked).
  extern __shared__ __align__(16) uint8_t kvq_smem[];
  const uint32_t ring = smem_u32(kvq_smem) + warp * kStages * kStageB;
  // this lane's 16-byte chunks of a block (BITS per row): row and byte offsets, fixed
  constexpr int kChunks = kBlk * BITS, kIters = (kChunks + 31) / 32;
  int c_row[kIters], c_q16[kIters];
#pragma unroll
  for (int it = 0; it < kIters; ++it) {
    const int i = lane + 32 * it;
    c_row[it] = i / BITS;
    c_q16[it] = 16 * (i % BITS);
  }
  const uint8_t* kc = p.k_codes + row0 * p.row_bytes;
  const uint8_t* vc = p.v_codes + row0 * p.row_bytes;
  const __half2* vpar = p.v_params + row0 * p.vp_stride + h;
  auto issue = [&](int wb, int stg) {
    if (wb < t1) {
      const uint32_t sa = ring + stg * kStageB;
      const bool full = wb + kBlk <= t1;
#pragma unroll
      for (int it = 0; it < kIters; ++it) {
        if (lane + 32 * it < kChunks) {
          const int t = full ? wb + c_row[it] : min(wb + c_row[it], t1 - 1);
          const int64_t src = (int64_t)t * p.row_bytes + (h * kRowB + c_q16[it]);
          const uint32_t dst = sa + c_row[it] * kRowB + c_q16[it];
          cp_async16(dst, kc + src);
          cp_async16(dst + kBlk * kRowB, vc + src);
        }
      }
      if (lane < kBlk) {
        const int64_t t = min(wb + lane, t1 - 1);
        cp_async4(sa + 2 * kBlk * kRowB + 4u * lane, vpar + t * p.vp_stride);
      }
    }
    cp_async_commit();
  };
  // block k of this warp: warp w takes whole K groups (128 tokens, 128/kBlk blocks)
  // w, w + nw, ...: the per-channel K params load once per group
  constexpr int kBpg = 128 / kBlk;
  auto wb_of = [&](int k) { return t0 + ((k / kBpg) * kNw + warp) * 128 + (k % kBpg) * kBlk; };
  // cos/sin(wbase theta) of the lane's 4 frequencies, loaded one block ahead
  auto base_of = [&](int wb, float2 (&cs)[4]) {
    const int64_t row = (int64_t)min(wb, len - 1) * 64 + 4 * hl;
#pragma unroll
    for (int j = 0; j < 4; ++j) cs[j] = __ldg(p.rope + row + j);
  };
#pragma unroll
  for (int k = 0; k < kStages - 1; ++k) issue(wb_of(k), k);
  float2 nbase[4];
  base_of(wb_of(0), nbase);
  int stage = 0;
  for (int kb = 0, wbase = wb_of(0); wbase < t1; wbase = wb_of(++kb)) {
    const int grp = wbase / kT;  // group_size is 128 (checked on the host)
    if (grp != cur_grp && wbase < nfl) {
      const __half* prow = p.k_params + (row0 / kT + grp) * 2 * p.kvw;
      float ks[8], kz[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = h * kHeadDim + 8 * hl + j;
        const int ppos = (c / bs) * bs + perm_position(c % bs, bs);
        ks[j] = __half2float(prow[ppos]) * code_unit<BITS>(j);
        kz[j] = __half2float(prow[p.kvw + ppos]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        kps[j] = make_float2(ks[2 * j], ks[2 * j + 1]);
        kpz[j] = make_float2(kz[2 * j], kz[2 * j + 1]);
      }
      cur_grp = grp;
    }
    // q rotated back to the block base, qb = R(wbase)^T q, so that
    // q . R(wbase + r) k = qb . R(r) k with R(r) from the shared offset table
    float2 qb[GROUP][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 cs = nbase[j];
#pragma unroll
      for (int gi = 0; gi < GROUP; ++gi) {
        const float2 qq = s_q[gi][j * 16 + hl];
        qb[gi][j] = make_float2(fmaf(qq.x, cs.x, qq.y * cs.y), fmaf(qq.y, cs.x, -qq.x * cs.y));
      }
    }
    base_of(wb_of(kb + 1), nbase);
    cp_async_wait<kStages - 2>();
    __syncwarp();
    const uint32_t sa = ring + stage * kStageB;
    uint2 kraw[kUnroll], vraw[kUnroll];
    __half2 vsz[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int r = 2 * u + half;
      kraw[u] = raw8_s<BITS>(sa + r * kRowB, hl);
      vraw[u] = raw8_s<BITS>(sa + kBlk * kRowB + r * kRowB, hl);
      vsz[u] = from_u32h2(lds32(sa + 2 * kBlk * kRowB + 4u * r));
    }
    // K phase: dequant + RoPE in registers, partial dot products of the group's heads.
    // K groups flush whole (nfl % 128 == 0), so a block is all codes or all residual.
    float part[kN];
    auto k_scores = [&](int u, const float2 (&kv)[4]) {
      const int r = 2 * u + half;
      float2 acc[GROUP];
#pragma unroll
      for (int gi = 0; gi < GROUP; ++gi) acc[gi] = make_float2(0.f, 0.f);
#pragma unroll
      for (int jp = 0; jp < 2; ++jp) {  // RoPE at offset r from the block base (linalg.py:92-93)
        const float4 o4 = *reinterpret_cast<const float4*>(&s_off[r][jp][hl][0]);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = 2 * jp + e;
          const float2 of = e ? make_float2(o4.z, o4.w) : make_float2(o4.x, o4.y);  // (cos, sin)
          // (x c - y s, x s + y c): two packed ops with broadcast / swapped / negated halves
          const float2 t = __fmul2_rn(make_float2(kv[j].y, kv[j].y), make_float2(of.y, of.x));
          const float2 kf = __ffma2_rn(make_float2(kv[j].x, kv[j].x), of, make_float2(-t.x, t.y));
#pragma unroll
          for (int gi = 0; gi < GROUP; ++gi) acc[gi] = __ffma2_rn(qb[gi][j], kf, acc[gi]);
        }
      }
#pragma unroll
      for (int gi = 0; gi < GROUP; ++gi) part[gi * kUnroll + u] = acc[gi].x + acc[gi].y;
    };
    if (wbase < nfl) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        float2 kv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) kv[j] = __ffma2_rn(code_pair<BITS>(kraw[u], j), kps[j], kpz[j]);
        k_scores(u, kv);
      }
    } else {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int t = min(wbase + 2 * u + half, t1 - 1);
        const float4* rr = reinterpret_cast<const float4*>(
            p.k_resid + ((int64_t)b * p.G + (t - nfl)) * p.kvw + h * kHeadDim + 8 * hl);
        const float4 a0 = rr[0], a1 = rr[1];
        const float2 kv[4] = {make_float2(a0.x, a0.y), make_float2(a0.z, a0.w),
                              make_float2(a1.x, a1.y), make_float2(a1.z, a1.w)};
        k_scores(u, kv);
      }
    }
    // this lane's score, the block max of each head, its probability, then every
    // (head, token) probability broadcast to the half-warp for the V phase
    float sc = xreduce16<kN>(part, hl);
    if (wbase + 2 * my_u + half >= t1) sc = -INFINITY;
    float mt = sc;
#pragma unroll
    for (int bit = 4 - kLogN; bit < 4 - kLogN + (kLogN - (GROUP == 4 ? 2 : GROUP == 2 ? 1 : 0)); ++bit)
      mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1 << bit));
    float mn_my = 0.f;
#pragma unroll
    for (int gi = 0; gi < GROUP; ++gi) {
      const float mg = GROUP == 1 ? mt
                                  : __shfl_sync(0xffffffffu, mt, (lane & 16) | ((gi * kUnroll) << (4 - kLogN)));
      const float mn = fmaxf(m[gi], mg);
      const float alpha = (m[gi] == -INFINITY) ? 0.f : exp2f(m[gi] - mn);
      l[gi] *= alpha;
      pz[gi] *= alpha;
      const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
      for (int j = 0; j < 4; ++j) o[gi][j] = __fmul2_rn(o[gi][j], a2);
      m[gi] = mn;
      if (gi == my_g) mn_my = mn;
    }
    const float p_my = (sc == -INFINITY) ? 0.f : exp2f(sc - mn_my);
    // V phase: p * scale times the codes, p * zp into pz; residual rows as floats
    auto v_accum = [&](int u, const float2 (&vf)[4], float2 sz) {
#pragma unroll
      for (int gi = 0; gi < GROUP; ++gi) {
        const float pr = __shfl_sync(0xffffffffu, p_my, (lane & 16) | ((gi * kUnroll + u) << (4 - kLogN)));
        l[gi] += pr;
        pz[gi] = fmaf(pr, sz.y, pz[gi]);
        const float ps = pr * sz.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) o[gi][j] = __ffma2_rn(make_float2(ps, ps), vf[j], o[gi][j]);
      }
    };
    if (wbase + kBlk <= vnfl) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        float2 vf[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) vf[j] = code_pair<BITS>(vraw[u], j);
        v_accum(u, vf, __half22float2(vsz[u]));
      }
    } else {  // the block reaches the V residual rows (V flushes are not group-aligned)
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int t = min(wbase + 2 * u + half, t1 - 1);
        float2 vf[4];
        float2 sz;
        if (t < vnfl) {
          sz = __half22float2(vsz[u]);
#pragma unroll
          for (int j = 0; j < 4; ++j) vf[j] = code_pair<BITS>(vraw[u], j);
        } else {  // scaled like the codes (2^code_sh), undone with them at the end
          sz = make_float2(1.f, 0.f);
          const float4* rr = reinterpret_cast<const float4*>(
              p.v_resid + ((int64_t)b * p.G + (t - vnfl)) * p.kvw + h * kHeadDim + 8 * hl);
          const float4 a0 = rr[0], a1 = rr[1];
          const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            vf[j] = make_float2(a[2 * j] / code_unit<BITS>(2 * j), a[2 * j + 1] / code_unit<BITS>(2 * j + 1));
        }
        v_accum(u, vf, sz);
      }
    }
    __syncwarp();  // every lane has read this stage before it is refilled
    issue(wb_of(kb + kStages - 1), stage == 0 ? kStages - 1 : stage - 1);
    stage = stage + 1 == kStages ? 0 : stage + 1;
  }
  cp_async_wait<0>();
  // merge the half-warp streams, one partial per CTA
  __shared__ float s_m[kStreams][GROUP], s_l[kStreams][GROUP], s_o[kStreams][GROUP][kHeadDim];
#pragma unroll
  for (int gi = 0; gi < GROUP; ++gi) {
    if (hl == 0) {
      s_m[stream][gi] = m[gi];
      s_l[stream][gi] = l[gi];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      s_o[stream][gi][8 * hl + 2 * j] = fmaf(o[gi][j].x, code_unit<BITS>(2 * j), pz[gi]);
      s_o[stream][gi][8 * hl + 2 * j + 1] = fmaf(o[gi][j].y, code_unit<BITS>(2 * j + 1), pz[gi]);
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < GROUP * kHeadDim; idx += kThreads) {
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
    float* dst = p.partials + (((int64_t)b * n_q + h * GROUP + gi) * p.n_chunks + chunk) * kPart;
    if (d == 0) {
      dst[0] = M;
      dst[1] = L;
    }
    dst[2 + d] = O;
  }
}

template <int BITS, int GROUP>
static int launch_one(const Params& p, int grid, cudaStream_t st) {
  constexpr uint32_t smem = smem_bytes<BITS, GROUP>();
  if (int s = ensure_smem(reinterpret_cast<const void*>(k_kvq_decode<BITS, GROUP>), smem,
                         "cudaFuncSetAttribute(kvq_decode)"))
    return s;
  k_kvq_decode<BITS, GROUP><<<grid, kThreads, smem, st>>>(p);
  return check_launch("k_kvq_decode");
}

template <int GROUP>
static int launch_bits(int bits, const Params& p, int grid, cudaStream_t st) {
  switch (bits) {
    case 2: return launch_one<2, GROUP>(p, grid, st);
    case 3: return launch_one<3, GROUP>(p, grid, st);
    case 4: return launch_one<4, GROUP>(p, grid, st);
    case 8: return launch_one<8, GROUP>(p, grid, st);
    default: return fail(XQ_ECONFIG, "bad bits %d", bits);
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
  chunk_tokens = (chunk_tokens + 127) / 128 * 128;
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
  chunk_tokens = (chunk_tokens + 127) / 128 * 128;  // blocks of 16 never straddle a K group
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
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = n_seqs * n_kv_heads * p.n_chunks;
  int status;
  switch (group) {
    case 1: status = launch_bits<1>(bits, p, grid, st); break;
    case 2: status = launch_bits<2>(bits, p, grid, st); break;
    case 4: status = launch_bits<4>(bits, p, grid, st); break;
    default: return fail(XQ_ECONFIG, "unsupported query group %d (1, 2, 4)", group);
  }
  if (status != XQ_OK) return status;
  k_combine<<<static_cast<unsigned>(n_seqs) * n_q, kHeadDim, 0, st>>>(p.partials, p.n_chunks, out);
  return check_launch("k_combine(kvq)");
}

}  // extern "C"
