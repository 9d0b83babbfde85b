// Fused XQuant decode with exact V absorption, for sm_100a.
//
// The reference rebuilds V = x_hat @ W_v for every cached token and then
// takes p @ V (cache.py:385-387, model.py:150-182). Because the product is
// associative, per query head h
//     sum_t p_t,h (x_hat_t @ W_v[:, kv(h)]) = (sum_t p_t,h x_hat_t) @ W_v[:, kv(h)]
// so the V side needs only the probability-weighted sum of the dequantized
// rows -- a [kdim x heads] GEMM over tokens -- plus one tiny projection per
// head at the end. The K side keeps the full rematerialisation (RoPE rotates
// K per position, so q cannot be absorbed into W_k). Per token this halves
// the tensor-core work of MHA (4*d*d_kv -> 2*d*d_kv + 2*H*d FLOP) and cuts
// the dequantisation passes from one per KV head to one per KV-head pair plus
// one for the V side.
//
// One persistent CTA pair (cta_group::2) per two SMs, 512 threads each:
//   warp 0       TMA of the W_k tiles (this CTA's 128 of the pass's 256 rows);
//                fp16 A rows by TMA when the A operand is the CL accumulator
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer (leader)
//   warp 2       TMA of the packed-codes ring
//   warps 4-11   dequant producers (two groups of 4, alternate codes stages)
//   warps 12-15  epilogue
// Per 256-token tile of one sequence (work unit):
//   passes p = 0 .. ceil(n_kv/2)-1: D[256 tok x 256] = A[tok x kdim] W_k^T for
//     KV heads 2p, 2p+1 (M=256 over the pair, N=256, K=kdim). The epilogue
//     RoPEs K in registers and stores the scores q.k of the heads' query heads.
//   exchange: each CTA keeps half of the query heads; the scores of the other
//     half for its 128 tokens go to the peer over DSMEM.
//   softmax over the tile's 256 tokens (tile max m, sum l) -> P (fp16) as the
//     K-major B operand [heads x 256 tokens].
//   V side: O^T[kdim x heads] = X_hat^T[kdim x 256 tok] P[256 tok x heads]:
//     M=256 channels over the pair (128 per CTA, MN-major A tiles written by
//     the same producers), N = heads, K = tokens. O and (m, l) go to HBM as
//     this tile's split partials.
// k_absorb_combine then merges the tile partials per (sequence, head) and
// k_absorb_project applies W_v[:, kv(h)].
#include <cudaTypedefs.h>
#include <math.h>
#include <stdlib.h>

#include <type_traits>

#include "xq_common.cuh"
#include "xq_dequant.cuh"
#include "xq_host.h"
#include "xq_layout.cuh"

namespace xq {
namespace absorb {

// Role profile (built only with -DXQ_ROLE_PROFILE, tools/build_role_profile.sh):
// cycles each role spends blocked on each barrier, summed over the grid.
//  0 W-TMA empty   1 MMA tempty   2 MMA full(K)   3 MMA pready   4 MMA full(V)
//  5 codes-TMA cempty   6 producer cfull   7 producer empty   8 epilogue tfull(K)
//  9 epilogue xfull   10 epilogue tfull(V)   11 CTA cycles (thread 0)
constexpr int kProfCounters = 16;
__device__ unsigned long long g_role_prof[kProfCounters];
#ifdef XQ_ROLE_PROFILE
#define XQ_PROF(c, stmt)                                  \
  do {                                                    \
    const long long t0_ = clock64();                      \
    stmt;                                                 \
    prof_acc[c] += static_cast<unsigned long long>(clock64() - t0_); \
  } while (0)
#else
#define XQ_PROF(c, stmt) stmt
#endif

constexpr int kTileM = 128;   // token rows per CTA (TMEM lanes)
constexpr int kPairM = 256;   // token rows per CTA pair
constexpr int kChunk = 64;    // channels per pass-1 stage
constexpr int kThreads = 512;
constexpr int kProdWarp0 = 4;
constexpr int kEpiWarp0 = 12;
constexpr int kG = 128;
constexpr int kMaxStages = 4;
constexpr int kMaxHeads = 64;
#ifndef XQ_SERPENTINE
#define XQ_SERPENTINE 1
#endif
constexpr bool kSerpentine = XQ_SERPENTINE != 0;  // fp16-row K passes alternate chunk direction
constexpr uint32_t kABytes = kTileM * 128;  // [128 x 64] fp16 = 16 KB
constexpr uint32_t kBSub = 128 * 128;       // 128 W rows x 64 channels (one KV head)
// KV heads per K pass: 4 (two N=256 MMAs share each A stage: half the dequant work
// per FLOP, one 512-column accumulator). GQA ran 2 heads per pass with
// double-buffered accumulators so its heavier score epilogue overlapped the next
// pass; 4 heads per pass halve the producers' per-channel conversions instead,
// which is the larger cost: C4 took 7.5% fewer cycles per launch
// (profiles/r02_gqa_kh4_ab.txt). XQ_GQA_KH=2 restores the pipelined variant.
#ifndef XQ_GQA_KH
#define XQ_GQA_KH 4
#endif
template <int GROUP>
struct Cfg {
  static constexpr int KH = GROUP == 1 ? 4 : XQ_GQA_KH;
  static constexpr int NBUF = KH == 2 ? 2 : 1;         // accumulator buffers
  static constexpr uint32_t kBBytes = (KH / 2) * kBSub;  // this CTA's W rows per stage
  static constexpr uint32_t kABStage = kABytes + kBBytes;
  static constexpr int kStages = KH == 2 ? 4 : 3;
  static constexpr int kUseCols = 512 / NBUF;            // columns of one accumulator
};
constexpr uint32_t kMNHalf = 64 * 128;      // V-side A stage: [64 tok x 64 ch] per channel half

struct Params {
  const float* k_resid;        // CODES_CHANNEL: fp32 residual rows [n_seqs][128][kdim]
  const int32_t* k_nflushed;   // CODES_CHANNEL: flushed token count per sequence
  const float* k_first;        // CODES_CHANNEL: fp32 channel 0 per arena row (outlier channel) or null
  int32_t kdim;
  int64_t L_max;
  const int32_t* seq_lens;
  int32_t n_seqs, n_tiles, n_units;
  int32_t n_kv, n_q, nb, nbh, n_pass;
  int32_t stages, cstages;
  uint32_t cstage_bytes;
  uint32_t k_code_bytes, k_tx, v_tx;  // codes ring: codes bytes / TMA bytes per stage
  const float* q_pre;
  const float2* rope;  // frequency-major [64][rope_n]
  int64_t rope_n;
  float q_scale;
  __half* part_o;      // [n_seqs][n_tiles][n_q][kdim] (fp16: half the partial traffic)
  float2* part_ml;     // [n_seqs][n_tiles][n_q] (m, l), m in the log2 domain
  uint64_t w_hint;
  int32_t a_hint;   // fp16-row A: 0 evict-normal, 1 split (see the K-pass TMA loop), 2 evict-last
  int32_t a_split;  // split: chunks at the start of each sweep loaded evict-first
  // XQ_A_F16_ACC: the accumulator rows (updated in place, one tile ahead of the
  // passes that read them) and this layer's per-token delta codes
  // GROUP 4: q as the B fragments of the score mma, per sequence (k_q_frags, once per
  // launch, in the spare half of the fp16 partials region): [n_seqs][n_kv][8][32]
  const uint2* q_frag;
  int32_t G;  // per-token quantization group (32 / 64 / 128; per-channel token groups: 128)
  __half* acc_out;
  const uint8_t* d_codes;
  const __half2* d_params;
  int64_t d_row_bytes, d_pstride;
  uint32_t off_p, off_codes, off_q, off_sc, off_rope, off_stg, off_bar;
};

// work unit u -> (sequence, tile); false when the tile is past the sequence end
XQ_DEVINL bool get_unit(const Params& p, int u, int& b, int& t, int& len) {
  b = u % p.n_seqs;
  t = u / p.n_seqs;
  len = __ldg(p.seq_lens + b);
  return t * kPairM < len;
}

struct Tile {
  int b, t, len;
};

// Visit this cluster's tiles in the order the pipeline consumes them: the K
// passes (kfn(tile, pass)) and the V side (vfn(tile)) of each tile. With PIPE
// (double-buffered accumulators) the first K pass of the next tile is issued
// before the V side of the current one, so the tensor cores have work while
// the epilogue finishes the current tile's softmax. Every role walks the same
// order, so the stage / accumulator counters stay in lock step.
template <bool PIPE, typename KF, typename VF>
XQ_DEVINL void walk(const Params& p, int cluster, int n_clusters, KF&& kfn, VF&& vfn) {
  auto next_valid = [&](int u, Tile& tl) {
    for (; u < p.n_units; u += n_clusters)
      if (get_unit(p, u, tl.b, tl.t, tl.len)) return u;
    return p.n_units;
  };
  Tile cur, nxt;
  int u = next_valid(cluster, cur);
  bool first = true;
  while (u < p.n_units) {
    const int nu = PIPE ? next_valid(u + n_clusters, nxt) : 0;
    for (int ps = (PIPE && !first) ? 1 : 0; ps < p.n_pass; ++ps) kfn(cur, ps);
    if (PIPE && nu < p.n_units) kfn(nxt, 0);
    vfn(cur);
    first = false;
    if (PIPE) {
      u = nu;
      cur = nxt;
    } else {
      u = next_valid(u + n_clusters, cur);
    }
  }
}

// One warp's accumulator row update: acc = fp16(float(acc) + code * scale + zp) for
// every channel (the arithmetic of k_cl_accumulate_w in xq_quant.cu, bit-identical),
// lane l taking channels 256k + 8l .. +7 (512 contiguous bytes per warp access).
template <int BITS>
XQ_DEVINL void acc_update_row(__half* acc, const uint8_t* codes, const __half2* params, int kdim,
                              int G, int lane) {
  constexpr uint32_t kMask = (1u << BITS) - 1u;
  constexpr int kU = 4;  // 256-channel blocks in flight
  for (int k0 = 0; k0 < kdim; k0 += 256 * kU) {
    uint4 old[kU];
    uint2 cw[kU];
    __half2 sz[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int c0 = k0 + 256 * k + 8 * lane;
      if (c0 >= kdim) continue;
      // evict-first: the next tile's rows must not push the current tile's A rows out
      // of L2 (2% fewer cycles per C3 delta launch, profiles/r02_c3_acc_hint_ab.txt)
      asm volatile("ld.global.L2::cache_hint.v4.b32 {%0, %1, %2, %3}, [%4], %5;"
                   : "=r"(old[k].x), "=r"(old[k].y), "=r"(old[k].z), "=r"(old[k].w)
                   : "l"(acc + c0), "l"(kEvictFirst));
      const uint8_t* cp = codes + c0 * BITS / 8;
      if constexpr (BITS == 3) {  // 3 bytes at any alignment: one or two aligned words
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(cp) & ~uintptr_t(3));
        const uint32_t sh = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(cp) & 3u);
        const uint32_t lo = __ldg(wp), hi = sh >= 2u ? __ldg(wp + 1) : 0u;
        cw[k] = make_uint2(__funnelshift_r(lo, hi, 8u * sh), 0u);
      } else if constexpr (BITS == 2) {
        cw[k] = make_uint2(__ldg(reinterpret_cast<const unsigned short*>(cp)), 0u);
      } else if constexpr (BITS == 4) {
        cw[k] = make_uint2(__ldg(reinterpret_cast<const uint32_t*>(cp)), 0u);
      } else {
        cw[k] = __ldg(reinterpret_cast<const uint2*>(cp));
      }
      sz[k] = __ldg(params + c0 / G);
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int c0 = k0 + 256 * k + 8 * lane;
      if (c0 >= kdim) continue;
      const float2 f = __half22float2(sz[k]);
      uint32_t hw[4] = {old[k].x, old[k].y, old[k].z, old[k].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int m = 2 * j + e;
          const uint32_t word = (BITS == 8 && m >= 4) ? cw[k].y : cw[k].x;
          v[e] = fmaf(static_cast<float>((word >> ((m * BITS) % 32)) & kMask), f.x, f.y);
        }
        const float2 o = __half22float2(from_u32<__half2>(hw[j]));
        hw[j] = as_u32(__floats2half2_rn(o.x + v[0], o.y + v[1]));
      }
      asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(acc + c0),
                   "r"(hw[0]), "r"(hw[1]), "r"(hw[2]), "r"(hw[3]), "l"(kEvictFirst)
                   : "memory");
    }
  }
}

// One entry (kvh, kk, lane) of the GQA score mma's B fragments: q heads kvh*4 + g
// (n = g, 4 of 8 used), k16 block kk of the split RoPE dims, rotated to pos and
// scaled, fp16 pairs {b0b1, b2b3}.
XQ_DEVINL uint2 q_frag_entry(const float* qb, const float2* rope, int64_t rope_n, int pos,
                             float q_scale, int i, int group) {
  const int ln = i & 31, kk = (i >> 5) & 7, kvh = i >> 8;
  const int g = ln >> 2, tig = ln & 3;
  if (g >= group) return make_uint2(0u, 0u);
  const float* qp = qb + (int64_t)(kvh * group + g) * kHeadDim;
  const int j0 = (kk & 3) * 16 + 2 * tig;  // frequency of split dim kk*16 + 2*tig
  const bool odd = kk >= 4;                // dims 64.. hold the second of each pair
  auto rot2 = [&](int j) {                 // split dims (j, j+1) of this half
    const float4 e = *reinterpret_cast<const float4*>(qp + 2 * j);
    const float2 c0 = rope[(int64_t)j * rope_n + pos];
    const float2 c1 = rope[(int64_t)(j + 1) * rope_n + pos];
    const float r0 = odd ? (e.x * c0.y + e.y * c0.x) : (e.x * c0.x - e.y * c0.y);
    const float r1 = odd ? (e.z * c1.y + e.w * c1.x) : (e.z * c1.x - e.w * c1.y);
    const __half2 h = __floats2half2_rn(r0 * q_scale, r1 * q_scale);
    return *reinterpret_cast<const uint32_t*>(&h);
  };
  return make_uint2(rot2(j0), rot2(j0 + 8));
}

// The B fragments of every sequence, once per launch (grid n_seqs): the fused
// kernel copies its sequence's 2 KB per KV head at each tile start instead of
// recomputing them from q and the RoPE table.
__global__ void __launch_bounds__(256) k_q_frags(const float* __restrict__ q_pre,
                                                 const float2* __restrict__ rope, int64_t rope_n,
                                                 const int32_t* __restrict__ seq_lens, int n_q,
                                                 int n_kv, int group, float q_scale,
                                                 uint2* __restrict__ out) {
  // block (sequence b, KV head blockIdx.y): one entry per thread (the RoPE table reads
  // are scattered, so the launch is latency-bound; one entry deep keeps it short)
  const int b = blockIdx.x, n_ent = n_kv * 256;
  const int pos = seq_lens[b] - 1;
  const float* qb = q_pre + (int64_t)b * n_q * kHeadDim;
  const int i = blockIdx.y * 256 + threadIdx.x;
  out[(int64_t)b * n_ent + i] = q_frag_entry(qb, rope, rope_n, pos < 0 ? 0 : pos, q_scale, i, group);
}

// Grouped-query scores of KV heads KB .. KB+NK-1 of K pass ps for the 32 token rows
// of TMEM lane quadrant q4 (the epilogue warps, and with HELP the second producer
// group, which takes the upper half of a 4-head pass). Per m16 tile, K is read from
// TMEM in the mma fragment order (16x256b), rotated in registers (FFMA2, cos/sin by
// angle addition), rounded to fp16 as the A fragments and multiplied with the q
// fragments (n = the 4 query heads of the KV head): 16 mma.sync per KV head and warp
// replace the 4 x 128 FFMA2 and the q loads of the per-row form. The TMEM loads run
// one (mt, c, kh) item ahead: the next item's two loads are issued right after the
// wait for the current one (tcgen05.wait::ld waits for every outstanding load).
// Scores land in sc [q head][128 rows] (-inf past the sequence end).
// kv_of(ps, kh): the KV head in accumulator slot kh of pass ps (see SPLIT in the
// kernel); the q fragments are stored in pass order (slot KH*ps + kh).
template <int KH>
XQ_DEVINL int kv_of(bool split, int ps, int kh) {
  return split ? (kh & 1) + 2 * ps + 4 * (kh >> 1) : KH * ps + kh;
}

template <int KH, int KB, int NK, int GROUP>
XQ_DEVINL void gqa_scores(uint32_t tmem_acc, int q4, int lane, int ps, bool split, int n_kv, int tok0,
                          int len, uint32_t q_a, uint32_t ro_a, uint32_t rb_a, uint32_t sc_a) {
  const int g = lane >> 2, tig = lane & 3;
  constexpr int NI = 2 * 4 * NK;  // (mt, c, kh) items
  uint32_t kbe[2][8], kbo[2][8];  // ping-pong K fragments (even / odd halves)
  auto issue = [&](int it, uint32_t(&ek)[8], uint32_t(&ok)[8]) {
    const int mt = it / (4 * NK), c = (it / NK) & 3, kh = KB + it % NK;
    const uint32_t base =
        tmem_acc + (static_cast<uint32_t>(q4 * 32 + 16 * mt) << 16) + kh * 128 + c * 16;
    tmem_ld16x256b_x2(base, ek);
    tmem_ld16x256b_x2(base + 64, ok);
  };
  issue(0, kbe[0], kbo[0]);
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int r1m = 2 * q4 + mt;
    float acc[NK][4];
#pragma unroll
    for (int j = 0; j < NK; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[j][i] = 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      // cos/sin of rows (g, g+8) x frequencies 16c + 2*tig + {0, 1, 8, 9}, in the
      // fragment register order: i -> row (i & 2 ? g+8 : g), j + (i & 1) + (i & 4 ? 8 : 0)
      float2 cs8[8];
      {
        const int j0 = 16 * c + 2 * tig;
        const float4 b0 = lds_f4(rb_a + 8u * (r1m * 64 + j0));
        const float4 b1 = lds_f4(rb_a + 8u * (r1m * 64 + j0 + 8));
        const float4 o00 = lds_f4(ro_a + 8u * (g * 64 + j0));
        const float4 o01 = lds_f4(ro_a + 8u * (g * 64 + j0 + 8));
        const float4 o10 = lds_f4(ro_a + 8u * ((g + 8) * 64 + j0));
        const float4 o11 = lds_f4(ro_a + 8u * ((g + 8) * 64 + j0 + 8));
        auto cmul = [](float bx, float by, float ox, float oy) {
          return make_float2(bx * ox - by * oy, by * ox + bx * oy);
        };
        cs8[0] = cmul(b0.x, b0.y, o00.x, o00.y);
        cs8[1] = cmul(b0.z, b0.w, o00.z, o00.w);
        cs8[2] = cmul(b0.x, b0.y, o10.x, o10.y);
        cs8[3] = cmul(b0.z, b0.w, o10.z, o10.w);
        cs8[4] = cmul(b1.x, b1.y, o01.x, o01.y);
        cs8[5] = cmul(b1.z, b1.w, o01.z, o01.w);
        cs8[6] = cmul(b1.x, b1.y, o11.x, o11.y);
        cs8[7] = cmul(b1.z, b1.w, o11.z, o11.w);
      }
#pragma unroll
      for (int j = 0; j < NK; ++j) {
        const int slot = KH * ps + KB + j;  // q fragments in pass order
        const int kvh = kv_of<KH>(split, ps, KB + j);
        const int itm = (mt * 4 + c) * NK + j;  // compile time after unrolling
        tmem_wait_ld();
        if (itm + 1 < NI) issue(itm + 1, kbe[(itm + 1) & 1], kbo[(itm + 1) & 1]);
        if (kvh < n_kv) {
          const uint32_t(&ek)[8] = kbe[itm & 1];
          const uint32_t(&ok)[8] = kbo[itm & 1];
          uint32_t are[4], aro[4];
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) {  // RoPE (linalg.py:92-93) of two values
            const float2 e = make_float2(__uint_as_float(ek[2 * q2]), __uint_as_float(ek[2 * q2 + 1]));
            const float2 o = make_float2(__uint_as_float(ok[2 * q2]), __uint_as_float(ok[2 * q2 + 1]));
            const float2 cv = make_float2(cs8[2 * q2].x, cs8[2 * q2 + 1].x);
            const float2 sv = make_float2(cs8[2 * q2].y, cs8[2 * q2 + 1].y);
            const float2 nsv = make_float2(-sv.x, -sv.y);
            const float2 re = __ffma2_rn(e, cv, __fmul2_rn(o, nsv));
            const float2 ro = __ffma2_rn(e, sv, __fmul2_rn(o, cv));
            are[q2] = as_u32(__float22half2_rn(re));
            aro[q2] = as_u32(__float22half2_rn(ro));
          }
          const uint2 qe = lds64(q_a + 8u * ((slot * 8 + c) * 32 + lane));
          const uint2 qo = lds64(q_a + 8u * ((slot * 8 + 4 + c) * 32 + lane));
          mma_16816_f16(acc[j], are, qe.x, qe.y);
          mma_16816_f16(acc[j], aro, qo.x, qo.y);
        }
      }
    }
    // D fragment: (row g, heads 2tig, 2tig+1), (row g+8, the same heads)
    const int rowa = q4 * 32 + 16 * mt + g;
    const int toka = tok0 + rowa;
    const bool va = toka < len, vb = toka + 8 < len;
    if (2 * tig < GROUP) {
#pragma unroll
      for (int j = 0; j < NK; ++j) {
        const int kvh = kv_of<KH>(split, ps, KB + j);
        if (kvh < n_kv) {
          const uint32_t s0 = sc_a + 4u * ((kvh * GROUP + 2 * tig) * kTileM + rowa);
          sts_f32(s0, va ? acc[j][0] : -INFINITY);
          sts_f32(s0 + 4u * kTileM, va ? acc[j][1] : -INFINITY);
          sts_f32(s0 + 32u, vb ? acc[j][2] : -INFINITY);
          sts_f32(s0 + 4u * kTileM + 32u, vb ? acc[j][3] : -INFINITY);
        }
      }
    }
  }
}

template <int AK, int AV, int BITS, int GROUP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_decode_absorbed(const __grid_constant__ CUtensorMap tmap_w,
                      const __grid_constant__ CUtensorMap tmap_ka,
                      const __grid_constant__ CUtensorMap tmap_kp,
                      const __grid_constant__ CUtensorMap tmap_va,
                      const __grid_constant__ CUtensorMap tmap_vp,
                      const __grid_constant__ CUtensorMap tmap_o, const Params p) {
  // PROD: dequant producers fill every A stage from packed codes; otherwise the fp16
  // A rows come by TMA. ACC: the producer warps instead update the accumulator rows
  // of the cluster's next tile in global memory while the current tile's passes run
  constexpr bool ACC = AK == XQ_A_F16_ACC;
  constexpr bool PROD = AK != XQ_A_F16_ROWS && !ACC;
  constexpr bool TMA_A = !PROD;
  static_assert((AK == XQ_A_F16_ROWS) == (AV == XQ_A_F16_ROWS), "fp16 rows feed both sides or neither");
  static_assert((AK == XQ_A_F16_ACC) == (AV == XQ_A_F16_ACC) && (!ACC || GROUP == 1),
                "the fused CL accumulate feeds both sides of an MHA layer");
  static_assert(AV != XQ_A_CODES_CHANNEL || AK == XQ_A_CODES_CHANNEL,
                "a per-channel V side shares the K side's stream (xq-cl-gqa base layers)");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sAB = smem;
  uint8_t* sP = smem + p.off_p;
  uint8_t* sC = smem + p.off_codes;
  float* q_s = reinterpret_cast<float*>(smem + p.off_q);    // [n_q][128]
  // [nb][128 rows]: scores of this CTA's tokens; after the exchange the rows of
  // the peer's heads hold the peer's tokens' scores for this CTA's heads
  float* sc_s = reinterpret_cast<float*>(smem + p.off_sc);
  // RoPE of row r = 16*r1 + r0 of the tile: angle (t0 + 16*r1 + r0)*theta_j
  // = base[r1][j] + off[j][r0], both from the float64-formed table
  float2* rope_off = reinterpret_cast<float2*>(smem + p.off_rope);  // [64 j][16 r0]
  float2* rope_base = rope_off + 64 * 16;                            // [8 r1][64 j]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* empty = full + kMaxStages;
  uint64_t* cfull = empty + kMaxStages;
  uint64_t* cempty = cfull + kMaxStages;
  uint64_t* tfull = cempty + kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* pready = tempty + 2;
  uint64_t* xfull = pready + 1;
  uint64_t* xread = xfull + 1;
  uint64_t* accw = xread + 1;   // ACC: both CTAs' rows of the next tile are updated
  uint64_t* tstart = accw + 1;  // ACC: warp 0 started a tile (the producers may go on)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tstart + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
#ifdef XQ_ROLE_PROFILE
  unsigned long long prof_acc[kProfCounters] = {};
  const long long prof_t0 = clock64();
#endif
  using CF = Cfg<GROUP>;
  // grouped-query scores as mma.sync products (4 query heads per KV head fill half
  // of an n8 tile); MHA keeps per-row FFMA2 dot products
  constexpr bool kMmaScores = GROUP == 4;
  constexpr int STAGES = CF::kStages;
  constexpr int KH = CF::KH;
  // HELP: the second producer group (warps 8-11, TMEM lane quadrants 0-3) drains the
  // upper two KV heads of each 4-head GQA pass while the epilogue drains the lower
  // two. The drain is latency-bound (one warp per SM sub-partition); with one
  // 512-column accumulator the MMA waits for it before every pass.
  constexpr bool kHelp = kMmaScores && KH == 4 && !ACC;
  // SPLIT (8 KV heads, 4 query heads each, two passes): pass ps takes KV heads
  // {2ps, 2ps+1, 2ps+4, 2ps+5}, so each CTA gets half of the query heads it owns
  // (rank r owns KV heads 4r..4r+3) from each pass, and the score exchange and
  // softmax of those heads run after pass 0 under pass 1's MMAs instead of all
  // after pass 1. The pass-0 q fragments (pass order) are dead by then, so P
  // (8 KB, aliasing them) can be written early.
  const bool split = kMmaScores && KH == 4 && p.n_kv == 2 * KH;
  // PACKV: a V-side A stage is 16 KB of the 48 KB ring slot, so with dequant
  // producers both A stages of a V codes stage share one slot (one empty wait and
  // one full arrival): the ring holds twice the V stages the producers can fill
  // while the epilogue runs the softmax, and the V side (producer-bound: its MMAs
  // are N = heads) starts from a deeper buffer
  constexpr bool kPackV = CF::kABStage >= 2 * kABytes;  // (fp16-row A: two TMA boxes per slot)
  constexpr int kVSub = kPackV ? 2 : 1;  // V A stages per ring slot
  constexpr uint32_t kABStage = CF::kABStage;
  constexpr uint32_t kBBytes = CF::kBBytes;
  const int CSTAGES = p.cstages;
  const int ngrp = p.kdim / kG;            // 128-channel groups
  const int nkc = p.kdim / kChunk;         // pass-1 stages per pass
  const int nblk = p.kdim / 256;           // V-side channel blocks (128 per CTA)
  const int bpu = CF::kUseCols / p.nb;     // V-side blocks per accumulator
  const int nuse = (nblk + bpu - 1) / bpu;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], PROD ? 2 + 8 : 2);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < CSTAGES; ++s) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], 4);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kHelp ? 16 : 8);  // epilogue (+ helper) warps of both CTAs
    }
    mbar_init(pready, 8);   // leader's: 4 epilogue warps per CTA
    mbar_init(xfull, 128);  // the peer's 128 epilogue threads (their scores landed here)
    mbar_init(xread, 128);  // the peer's 128 epilogue threads (they read out their landing rows)
    mbar_init(accw, 2 * 256);  // every producer thread (8 warps) of both CTAs, once per tile
    mbar_init(tstart, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    if constexpr (!PROD) {
      tma_prefetch_desc(&tmap_ka);
      tma_prefetch_desc(&tmap_va);
    }
  }
  if (warp == 2 && lane == 0 && PROD) {
    tma_prefetch_desc(&tmap_ka);
    tma_prefetch_desc(&tmap_kp);
    tma_prefetch_desc(&tmap_va);
    tma_prefetch_desc(&tmap_vp);
  }
  if (warp == 1) {
    tmem_alloc2(tmem_slot, 512);
    tmem_relinquish2();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t full_leader0 = mapa_shared(smem_u32(&full[0]), 0);
  const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
  const uint32_t pready_leader = mapa_shared(smem_u32(pready), 0);

  constexpr bool PIPE = Cfg<GROUP>::NBUF == 2;  // see walk(): overlap tile k+1's first K pass with tile k's softmax
  if (warp == 0) {
    // ------------------------------------------------ TMA: W_k halves (+ fp16 A rows)
    uint32_t it = 0, tk = 0;  // tk: tiles whose updated accumulator rows were awaited (ACC)
    walk<PIPE>(p, cluster, n_clusters,
      [&](const Tile& tl, int ps) {
        const int32_t row_tile = static_cast<int32_t>((int64_t)tl.b * p.L_max + tl.t * kPairM);
        // ACC: the tile's rows are read once both CTAs' producers have updated them
        const bool a_tma = TMA_A;
        if (ACC && ps == 0) {
          mbar_wait_cluster(accw, (tk++) & 1u);
          if (elect_one()) mbar_arrive(tstart);
          __syncwarp();
        }
        // fp16 A rows: odd passes walk the channel chunks backwards, so a pass
        // starts on the chunks the previous one read last (still in L2). The
        // 74 clusters' 2 MB tiles exceed L2, and a forward-only walk re-reads
        // every pass from HBM. The MMA accumulates in issue order, so only the
        // fp32 summation order changes. Code-fed passes keep the forward order
        // (the producers' chunk mapping; their codes tiles fit L2).
        const bool rev = TMA_A && kSerpentine && (ps & 1);
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
          const int kcc = rev ? nkc - 1 - kc : kc;
          XQ_PROF(0, mbar_wait(&empty[s], ph ^ 1));
          if (elect_one()) {
            uint8_t* st = sAB + s * kABStage;
            const uint32_t kTx = 2 * (kBBytes + (a_tma ? kABytes : 0u));
            if (leader) mbar_arrive_expect_tx(&full[s], kTx);
            else mbar_arrive_remote(full_leader0 + 8 * s);
#pragma unroll
            for (int sub = 0; sub < KH / 2; ++sub)  // KV head kv_of(ps, 2*sub + rank)
              tma_load_2d_pair(st + kABytes + sub * kBSub, &tmap_w, &full[s], kcc * kChunk,
                               kv_of<KH>(split, ps, 2 * sub + static_cast<int>(rank)) * 128, p.w_hint);
            if (a_tma)
              // split: the first half of a sweep is the part the previous
              // sweep left in L2 (demote it), the second half is what the next
              // sweep reads first (keep it)
              tma_load_2d_pair(st, &tmap_ka, &full[s], kcc * kChunk, row_tile + rank * kTileM,
                               p.a_hint == 1 ? (kc < p.a_split ? kEvictFirst : kEvictLast)
                                             : (p.a_hint == 2 ? kEvictLast : kEvictNormal));
          }
          __syncwarp();
        }
      },
      [&](const Tile& tl) {
        const int32_t row_tile = static_cast<int32_t>((int64_t)tl.b * p.L_max + tl.t * kPairM);
      for (int bb = 0; bb < nblk; ++bb) {
        for (int j = 0; j < 4; j += kVSub, ++it) {
          const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
          XQ_PROF(0, mbar_wait(&empty[s], ph ^ 1));
          if (elect_one()) {
            uint8_t* st = sAB + s * kABStage;
            if constexpr (!TMA_A) {
              if (leader) mbar_arrive(&full[s]);
              else mbar_arrive_remote(full_leader0 + 8 * s);
            } else {
              if (leader) mbar_arrive_expect_tx(&full[s], 2 * kABytes * kVSub);
              else mbar_arrive_remote(full_leader0 + 8 * s);
#pragma unroll
              for (int js = 0; js < kVSub; ++js)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
                  tma_load_2d_pair(st + js * kABytes + hh * kMNHalf, &tmap_va, &full[s],
                                   bb * 256 + rank * 128 + hh * 64, row_tile + 64 * (j + js),
                                   p.a_hint != 0 ? kEvictFirst : kEvictNormal);  // last use
            }
          }
          __syncwarp();
        }
      }
      });
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader CTA only)
    if (leader) {
      constexpr uint32_t kIdescK = idesc_f16_f32(256, 256);
      const uint32_t kIdescV = idesc_f16_f32_amn(256, p.nb);
      const uint64_t desc0 = sdesc_sw128(smem_u32(sAB));
      const uint64_t descv0 = sdesc_mn_sw128(smem_u32(sAB), kMNHalf, 1024);
      const uint64_t descp0 = sdesc_sw128(smem_u32(sP));
      const uint32_t pstage = p.nbh * 128;  // bytes of one 64-token P stage
      uint32_t it = 0, tc = 0, ti = 0;
      walk<PIPE>(p, cluster, n_clusters,
        [&](const Tile&, int) {
          const uint32_t a = CF::NBUF == 2 ? (tc & 1) : 0u;
          const uint32_t aph = CF::NBUF == 2 ? ((tc >> 1) & 1) : (tc & 1);
          XQ_PROF(1, mbar_wait_cluster(&tempty[a], aph ^ 1));
          tc_fence_after();
          const uint32_t d = tmem + a * 256;
          for (int kc = 0; kc < nkc; ++kc, ++it) {
            const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
            XQ_PROF(2, mbar_wait_cluster(&full[s], ph));
            tc_fence_after();
            const uint64_t ad = desc0 + ((s * kABStage) >> 4);
            const uint64_t bd = ad + (kABytes >> 4);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < kChunk / 16; ++k)
#pragma unroll
                for (int sub = 0; sub < KH / 2; ++sub)
                  mma2_f16_ss(d + sub * 256, ad + 2 * k, bd + (sub * kBSub >> 4) + 2 * k, kIdescK,
                              (kc | k) != 0);
              mma2_commit_both(&empty[s]);
            }
            __syncwarp();
          }
          if (elect_one()) mma2_commit_both(&tfull[a]);
          __syncwarp();
          ++tc;
        },
        [&](const Tile&) {
        // V side: needs this tile's P from both CTAs
        XQ_PROF(3, mbar_wait_cluster(pready, ti & 1));
        tc_fence_after();
        int blk = 0;
        for (int us = 0; us < nuse; ++us, ++tc) {
          const uint32_t a = CF::NBUF == 2 ? (tc & 1) : 0u;
          const uint32_t aph = CF::NBUF == 2 ? ((tc >> 1) & 1) : (tc & 1);
          XQ_PROF(1, mbar_wait_cluster(&tempty[a], aph ^ 1));
          tc_fence_after();
          for (int bi = 0; bi < bpu && blk < nblk; ++bi, ++blk) {
            const uint32_t d = tmem + a * 256 + bi * p.nb;
            for (int j0 = 0; j0 < 4; j0 += kVSub, ++it) {
              const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
              XQ_PROF(4, mbar_wait_cluster(&full[s], ph));
              tc_fence_after();
              if (elect_one()) {
#pragma unroll
                for (int js = 0; js < kVSub; ++js) {  // the slot's A stages (token quarters)
                  const int j = j0 + js;
                  const uint64_t ad = descv0 + ((s * kABStage + js * kABytes) >> 4);
                  const uint64_t bd = descp0 + ((j * pstage) >> 4);
#pragma unroll
                  for (int k = 0; k < 4; ++k)  // 16 tokens = two 8-row K groups = 2048 B of A
                    mma2_f16_ss(d, ad + k * (2048 >> 4), bd + 2 * k, kIdescV, (j | k) != 0);
                }
                mma2_commit_both(&empty[s]);
              }
              __syncwarp();
            }
          }
          if (elect_one()) mma2_commit_both(&tfull[a]);
          __syncwarp();
        }
        ++ti;
        });
    }
  } else if (warp == 2) {
    // ------------------------------------------------ TMA: codes ring
    if constexpr (PROD) {
      uint32_t ci = 0, cphase = 0;  // ring slot / phase of the next codes stage
      auto next_slot = [&](uint32_t& cs, uint32_t& cph) {
        cs = ci;
        cph = cphase;
        if (++ci == static_cast<uint32_t>(CSTAGES)) {
          ci = 0;
          cphase ^= 1u;
        }
      };
      walk<PIPE>(p, cluster, n_clusters,
        [&](const Tile& tl, int) {  // K side: group g of this CTA's 128 tokens
          const int32_t arow = static_cast<int32_t>((int64_t)tl.b * p.L_max + tl.t * kPairM) +
                               static_cast<int32_t>(rank) * kTileM;
          for (int g = 0; g < ngrp; ++g) {
            uint32_t cs, cph;
            next_slot(cs, cph);
            XQ_PROF(5, mbar_wait(&cempty[cs], cph ^ 1));
            if (elect_one()) {
              uint8_t* st = sC + cs * p.cstage_bytes;
              mbar_arrive_expect_tx(&cfull[cs], p.k_tx);
              tma_load_2d(st, &tmap_ka, &cfull[cs], g * 16 * BITS, arow, kEvictNormal);
              if constexpr (AK == XQ_A_CODES_TOKEN)
                tma_load_2d(st + p.k_code_bytes, &tmap_kp, &cfull[cs], 4 * (((g * kG) / p.G) & ~3), arow,
                            kEvictNormal);
              else
                tma_load_2d(st + p.k_code_bytes, &tmap_kp, &cfull[cs], g * 128, 2 * (arow / kG),
                            kEvictNormal);
            }
            __syncwarp();
          }
        },
        [&](const Tile& tl) {  // V side: group 2*bb + rank of token half th of the pair tile
          const int32_t row_tile = static_cast<int32_t>((int64_t)tl.b * p.L_max + tl.t * kPairM);
          for (int g = 0; g < ngrp; ++g) {
            uint32_t cs, cph;
            next_slot(cs, cph);
            XQ_PROF(5, mbar_wait(&cempty[cs], cph ^ 1));
            if (elect_one()) {
              uint8_t* st = sC + cs * p.cstage_bytes;
              const int gv = (g & ~1) + static_cast<int>(rank);
              const int32_t arow = row_tile + (g & 1) * kTileM;
              mbar_arrive_expect_tx(&cfull[cs], p.v_tx);
              tma_load_2d(st, &tmap_va, &cfull[cs], gv * 16 * BITS, arow, kEvictNormal);
              if constexpr (AV == XQ_A_CODES_CHANNEL)  // [scales | zps] of this token group
                tma_load_2d(st + 128 * 16 * BITS, &tmap_vp, &cfull[cs], gv * 128, 2 * (arow / kG),
                            kEvictNormal);
              else
                tma_load_2d(st + 128 * 16 * BITS, &tmap_vp, &cfull[cs], 4 * (((gv * kG) / p.G) & ~3), arow,
                            kEvictNormal);
            }
            __syncwarp();
          }
        });
    }
  } else if (warp >= kProdWarp0 && warp < kEpiWarp0) {
    // ------------------------------------------------ dequant producers
    // HELP (warps 8-11): after producing its stages of a K pass, drain the pass's
    // upper two KV heads (scores -> sc_s), then go on with the next item's stages
    uint32_t tch = 0;  // accumulator uses seen (K passes and V-side uses)
    auto help = [&](const Tile& tl, int ps) {
      if constexpr (kHelp) {
        if (ps == 0) named_bar_sync(2, 256);  // the epilogue set up this tile's q / RoPE base
        mbar_wait(&tfull[0], tch & 1u);
        tc_fence_after();
        gqa_scores<KH, KH / 2, KH / 2, GROUP>(tmem, warp & 3, lane, ps, split, p.n_kv,
                                             tl.t * kPairM + static_cast<int>(rank) * kTileM, tl.len,
                                             smem_u32(q_s), smem_u32(rope_off), smem_u32(rope_base),
                                             smem_u32(sc_s));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) mbar_arrive(&tempty[0]);
          else mbar_arrive_remote(tempty_leader0);
        }
        ++tch;
        if (split || ps == p.n_pass - 1) named_bar_arrive(3, 256);  // scores the exchange reads
      }
    };
    if constexpr (ACC) {
      // XQuant-CL accumulate (cache.py:472-481, Accumulator.add cache.py:139-146),
      // one tile ahead: the cluster's first tile is updated before anything reads
      // it; tile i+1 while warp 0 and the tensor cores work on tile i (its rows are
      // disjoint). Warp w takes rows w, w+8, .. of this CTA's 128 and walks each
      // row 256 channels at a time (lane: 8 channels, 16-byte coalesced accesses).
      const int pw = warp - kProdWarp0;
      const uint32_t accw_l = mapa_shared(smem_u32(accw), rank);
      const uint32_t accw_p = mapa_shared(smem_u32(accw), rank ^ 1u);
      uint32_t ti = 0;
      for (int u = cluster; u < p.n_units; u += n_clusters) {
        Tile tl;
        if (!get_unit(p, u, tl.b, tl.t, tl.len)) continue;
        if (ti > 0) mbar_wait(tstart, (ti - 1) & 1u);  // tile ti-1 is under way
        for (int r = pw; r < kTileM; r += 8) {
          const int tok = tl.t * kPairM + static_cast<int>(rank) * kTileM + r;
          if (tok >= tl.len) break;
          const int64_t row = (int64_t)tl.b * p.L_max + tok;
          acc_update_row<BITS>(p.acc_out + row * p.kdim, p.d_codes + row * p.d_row_bytes,
                               p.d_params + row * p.d_pstride, p.kdim, p.G, lane);
        }
        // the updated rows, visible to the TMA loads of both CTAs (async proxy)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mbar_arrive_remote_release(accw_l);
        mbar_arrive_remote_release(accw_p);
        ++ti;
      }
    } else if constexpr (PROD) {
      const int gp = (warp - kProdWarp0) >> 2;
      const int r = ((warp - kProdWarp0) & 3) * 32 + lane;
      const RowSwizzle sw_k(r);       // K side: row = token r of this CTA's 128
      const RowSwizzle sw_v(r & 63);  // V side: row = token within a 64-token stage
      const int hh = r >> 6;          // V side: channel half of the group
      const uint32_t sAB_a = smem_u32(sAB), sC_a = smem_u32(sC);
      // this group's codes stages are the running indices == gp (mod 2) (every
      // K or V item has an even number ngrp of them); ring slot / phase advance
      // by 2 per stage, A stages by 4
      uint32_t cs = static_cast<uint32_t>(gp), cph = 0;
      if (cs >= static_cast<uint32_t>(CSTAGES)) cs -= CSTAGES;  // (CSTAGES >= 2)
      // ai: running ring-slot index of this group's next A stage. K items use two
      // slots per codes stage (this group's at 2*gp + 4k + h of the item); packed V
      // items one (gp + 2k), entered with ai -= gp and left with ai += gp
      uint32_t ai = static_cast<uint32_t>(2 * gp);
      auto advance = [&](uint32_t slots) {
        cs += 2;
        if (cs >= static_cast<uint32_t>(CSTAGES)) {
          cs -= CSTAGES;
          cph ^= 1u;
        }
        ai += 2 * slots;
      };
      // two A stages per codes stage; fill(tile address, h) writes stage h
      // two A stages per codes stage: once stage h is free, conv(st, h, v) converts
      // it into registers and store(tile, h, v) writes it (measured: converting
      // before the wait and releasing the codes stage early did not change C2/C4)
      // packed (V side with PACKV): both A stages into one slot, at +h * 16 KB
      auto stages2 = [&](auto&& conv, auto&& store, auto packed_c) {
        constexpr bool packed = decltype(packed_c)::value;
        const uint32_t st = sC_a + cs * p.cstage_bytes;
        XQ_PROF(6, mbar_wait(&cfull[cs], cph));
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          const uint32_t idx = packed ? ai : ai + h;
          const uint32_t s = idx % STAGES, ph = (idx / STAGES) & 1u;
          if (!packed || h == 0) XQ_PROF(7, mbar_wait(&empty[s], ph ^ 1));
          uint32_t v[32];
          conv(st, h, v);
          store(sAB_a + s * kABStage + (packed ? h * kABytes : 0u), h, v);
          if (!packed || h == 1) {
            fence_proxy_async_smem();
            __syncwarp();
            if (leader) mbar_arrive_if(&full[s], lane == 0);
            else mbar_arrive_remote_if(full_leader0 + 8 * s, lane == 0);
          }
        }
        mbar_arrive_if(&cempty[cs], lane == 0);
        advance(packed ? 1u : 2u);
      };
      using Unpacked = std::integral_constant<bool, false>;
      using PackedV = std::integral_constant<bool, kPackV>;
      walk<PIPE>(p, cluster, n_clusters,
        [&](const Tile& tl, int ps) {
          const int nfl = (AK == XQ_A_CODES_CHANNEL) ? __ldg(p.k_nflushed + tl.b) : 0;
          const int tok_k = tl.t * kPairM + static_cast<int>(rank) * kTileM + r;
          for (int g = gp; g < ngrp; g += 2)
            stages2(
                [&](uint32_t st, int h, uint32_t(&v)[32]) {
                  convert_chunk<AK, BITS>(st, st + p.k_code_bytes, r, tok_k < tl.len, tok_k, tl.b, nfl,
                                          2 * g + h,
                                          p.k_first ? p.k_first + (int64_t)tl.b * p.L_max + tok_k : nullptr,
                                          p.k_resid, p.kdim, v, p.G);
                },
                [&](uint32_t tile, int, const uint32_t(&v)[32]) { sw_k.store(tile, v); }, Unpacked());
          if (kHelp && gp == 1) help(tl, ps);
        },
        [&](const Tile& tl) {
          if (kHelp && gp == 1) tch += nuse;
          if (kPackV) ai -= static_cast<uint32_t>(gp);
          const int nfl = (AK == XQ_A_CODES_CHANNEL) ? __ldg(p.k_nflushed + tl.b) : 0;
          for (int g = gp; g < ngrp; g += 2)
            stages2(
                [&](uint32_t st, int h, uint32_t(&v)[32]) {
                  const int gv = (g & ~1) + static_cast<int>(rank);
                  const int crow = h * 64 + (r & 63);
                  const int tok = tl.t * kPairM + (g & 1) * kTileM + crow;
                  if constexpr (AV == XQ_A_CODES_TOKEN)
                    convert_chunk<AV, BITS>(st, st + 128 * 16 * BITS, crow, tok < tl.len, tok, tl.b,
                                            1 << 30, 2 * gv + hh, nullptr, nullptr, p.kdim, v, p.G);
                  else if constexpr (AV == XQ_A_CODES_CHANNEL)  // same stream as the K side
                    convert_chunk<AV, BITS>(st, st + 128 * 16 * BITS, crow, tok < tl.len, tok, tl.b,
                                            nfl, 2 * gv + hh, nullptr, p.k_resid, p.kdim, v);
                },
                [&](uint32_t tile, int, const uint32_t(&v)[32]) { sw_v.store(tile + hh * kMNHalf, v); },
                PackedV());
          if (kPackV) ai += static_cast<uint32_t>(gp);
        });
    } else if constexpr (kHelp) {  // fp16-row A by TMA: the producer warps only help
      if (warp >= kProdWarp0 + 4)
        walk<PIPE>(p, cluster, n_clusters, [&](const Tile& tl, int ps) { help(tl, ps); },
                   [&](const Tile&) { tch += nuse; });
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------ epilogue (this CTA's 128 rows)
    const int ew = warp - kEpiWarp0;
    const int et = threadIdx.x - kEpiWarp0 * 32;
    const int row = ew * 32 + lane;
    const uint32_t tlane = static_cast<uint32_t>(ew * 32) << 16;
    const int nbh = p.nbh;
    const uint32_t peer = rank ^ 1u;
    const uint32_t sc_peer = mapa_shared(smem_u32(sc_s), peer);
    const uint32_t xfull_peer = mapa_shared(smem_u32(xfull), peer);
    const uint32_t xread_peer = mapa_shared(smem_u32(xread), peer);
    const uint32_t sP_a = smem_u32(sP);
    // 32-bit shared addresses: explicit ld/st.shared (a generic pointer into
    // dynamic shared memory compiles to generic LD/ST)
    const uint32_t q_a = smem_u32(q_s), sc_a = smem_u32(sc_s);
    const uint32_t land_a = sc_a + 4u * (peer * nbh) * kTileM;  // rows of the peer's heads
    const uint32_t ro_a = smem_u32(rope_off), rb_a = smem_u32(rope_base);
    // offsets table: cos/sin(r0*theta_j), r0 < 16 (table positions 0..15); [64 j][16 r0]
    // for the per-row FFMA scores, [16 r0][64 j] for the mma fragments (pairs of j)
    for (int i = et; i < 64 * 16; i += 128)
      rope_off[i] = kMmaScores ? p.rope[(int64_t)(i & 63) * p.rope_n + (i >> 6)]
                               : p.rope[(int64_t)(i >> 4) * p.rope_n + (i & 15)];
    const int r0 = row & 15, r1 = row >> 4;
    const uint32_t stg_a = smem_u32(smem + p.off_stg);
    uint32_t tc = 0, ti = 0, xc = 0;  // xc: score exchanges (xread / xfull phase)
    walk<PIPE>(p, cluster, n_clusters,
      [&](const Tile& tl, int ps) {
      const int b = tl.b, t = tl.t, len = tl.len;
      if (ps == 0) {  // tile setup: q rotated to len-1, the RoPE base rows
#ifdef XQ_ROLE_PROFILE
      const long long pt_s = clock64();
#endif
      const int pos = len - 1;
      if (!PIPE && et == 0) tma_store_wait_read<0>();  // previous tile's O stores have read q_s / sc_s
      named_bar_sync(1, 128);  // previous tile's readers of q_s / sc_s / rope_base are done
      for (int i = et; i < 8 * 64; i += 128) {  // base: cos/sin(t0 + 16*r1), t0 = tile row 0
        const int64_t tp = (int64_t)t * kPairM + rank * kTileM + 16 * (i >> 6);
        rope_base[i] = p.rope[(int64_t)(i & 63) * p.rope_n + (tp < p.rope_n ? tp : 0)];
      }
      if constexpr (kMmaScores) {
        // q as the B fragments of mma m16n8k16 (k_q_frags: entry (kvh, kk, lane) =
        // {b0b1, b2b3} of k16 block kk), copied for this tile's sequence
        const int n_ent4 = p.n_kv * 128;  // 16-byte pairs of entries
        const uint4* src = reinterpret_cast<const uint4*>(p.q_frag + (int64_t)b * p.n_kv * 256);
#pragma unroll 8
        for (int i = et; i < n_ent4; i += 128) {
          const uint4 v = __ldg(src + i);
          const int kvh = i >> 7;  // stored in pass order: slot KH*ps + kh of kv_of(ps, kh)
          const int slot = split ? ((kvh >> 1) & 1) * KH + (kvh & 1) + 2 * (kvh >> 2) : kvh;
          sts128(q_a + 16u * (slot * 128 + (i & 127)), v.x, v.y, v.z, v.w);
        }
      } else {
        const float2 cs = p.rope[(int64_t)(et >> 1) * p.rope_n + pos];
        for (int h = 0; h < p.n_q; ++h) {
          const float* qp = p.q_pre + ((int64_t)b * p.n_q + h) * kHeadDim;
          const float e0 = qp[et & ~1], e1 = qp[et | 1];
          const float rr = (et & 1) ? (e0 * cs.y + e1 * cs.x) : (e0 * cs.x - e1 * cs.y);
          // split layout: even dims (first of each RoPE pair) then odd dims
          sts_f32(q_a + 4u * (h * kHeadDim + ((et & 1) ? 64 : 0) + (et >> 1)), rr * p.q_scale);
        }
      }
      named_bar_sync(1, 128);
      if constexpr (kHelp) named_bar_arrive(2, 256);  // q / RoPE base ready for the helpers
#ifdef XQ_ROLE_PROFILE
      prof_acc[15] += clock64() - pt_s;
#endif
      }
      const int tok = t * kPairM + rank * kTileM + row;
      const bool valid = tok < len;
      // ---- K side: scores of every query head for this CTA's 128 tokens.
      // cos/sin of (t0 + 16*r1 + r0)*theta_j by one angle addition from the two
      // shared tables (shared by the KH heads of a pass)
      auto load_cs = [&](int c, float2(&dst)[16]) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = c * 16 + i;
          const float2 bs = lds_f2(rb_a + 8u * (r1 * 64 + j)), of = lds_f2(ro_a + 8u * (j * 16 + r0));
          dst[i] = make_float2(bs.x * of.x - bs.y * of.y, bs.y * of.x + bs.x * of.y);
        }
      };
        const uint32_t a = CF::NBUF == 2 ? (tc & 1) : 0u;
        const uint32_t aph = CF::NBUF == 2 ? ((tc >> 1) & 1) : (tc & 1);
        XQ_PROF(8, mbar_wait(&tfull[a], aph));
#ifdef XQ_ROLE_PROFILE
        const long long pt_k = clock64();
#endif
        tc_fence_after();
        if constexpr (kMmaScores) {
          // scores on the tensor cores (gqa_scores); with HELP the second producer
          // group takes the pass's KV heads KH/2 .. KH-1 in parallel
          const int tok0 = t * kPairM + static_cast<int>(rank) * kTileM;
          if constexpr (kHelp)
            gqa_scores<KH, 0, KH / 2, GROUP>(tmem + a * 256, ew, lane, ps, split, p.n_kv, tok0, len,
                                            q_a, ro_a, rb_a, sc_a);
          else
            gqa_scores<KH, 0, KH, GROUP>(tmem + a * 256, ew, lane, ps, split, p.n_kv, tok0, len, q_a,
                                        ro_a, rb_a, sc_a);
        } else {
        // K columns of a head come split (W_k rows arranged so): cols 0-63 hold
        // the first element of each RoPE pair, cols 64-127 the second, so
        // pairs of frequencies map to register pairs and the rotation + dot
        // run as packed float2 FMAs (FFMA2)
        float2 sc[KH][GROUP];
#pragma unroll
        for (int kh = 0; kh < KH; ++kh)
#pragma unroll
          for (int gi = 0; gi < GROUP; ++gi) sc[kh][gi] = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // frequencies 16c .. 16c+15
          float2 cc[8], ss[8], ns[8];
          {
            float2 csv[16];
            load_cs(c, csv);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              cc[i] = make_float2(csv[2 * i].x, csv[2 * i + 1].x);
              ss[i] = make_float2(csv[2 * i].y, csv[2 * i + 1].y);
              ns[i] = make_float2(-csv[2 * i].y, -csv[2 * i + 1].y);
            }
          }
#pragma unroll
          for (int kh = 0; kh < KH; ++kh) {
            const int kvh = KH * ps + kh;
            if (kvh < p.n_kv) {
              float ke[16], ko[16];
              tmem_ld16(tmem + tlane + a * 256 + kh * 128 + c * 16, ke);
              tmem_ld16(tmem + tlane + a * 256 + kh * 128 + 64 + c * 16, ko);
              tmem_wait_ld();
              float2 re[8], ro[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {  // RoPE (linalg.py:92-93)
                const float2 e = make_float2(ke[2 * i], ke[2 * i + 1]);
                const float2 o = make_float2(ko[2 * i], ko[2 * i + 1]);
                re[i] = __ffma2_rn(e, cc[i], __fmul2_rn(o, ns[i]));
                ro[i] = __ffma2_rn(e, ss[i], __fmul2_rn(o, cc[i]));
              }
#pragma unroll
              for (int gi = 0; gi < GROUP; ++gi) {
                const uint32_t qe = q_a + 4u * ((kvh * GROUP + gi) * kHeadDim + c * 16);
#pragma unroll
                for (int v4 = 0; v4 < 4; ++v4) {
                  const float4 a4 = lds_f4(qe + 16u * v4), b4 = lds_f4(qe + 256u + 16u * v4);
                  float2 acc = sc[kh][gi];
                  acc = __ffma2_rn(re[2 * v4], make_float2(a4.x, a4.y), acc);
                  acc = __ffma2_rn(re[2 * v4 + 1], make_float2(a4.z, a4.w), acc);
                  acc = __ffma2_rn(ro[2 * v4], make_float2(b4.x, b4.y), acc);
                  acc = __ffma2_rn(ro[2 * v4 + 1], make_float2(b4.z, b4.w), acc);
                  sc[kh][gi] = acc;
                }
              }
            }
          }
        }
#pragma unroll
        for (int kh = 0; kh < KH; ++kh) {
          const int kvh = KH * ps + kh;
          if (kvh < p.n_kv) {
#pragma unroll
            for (int gi = 0; gi < GROUP; ++gi)
              sts_f32(sc_a + 4u * ((kvh * GROUP + gi) * kTileM + row),
                      valid ? sc[kh][gi].x + sc[kh][gi].y : -INFINITY);
          }
        }
        }  // per-row FFMA scores
        // exchange + softmax after this pass: every pass with SPLIT, else the last
        const bool xpass = split || ps == p.n_pass - 1;
        tc_fence_before();
        __syncwarp();
        // HELP: the helpers' scores of this pass are in sc_s (synced before the
        // accumulator is released, so the helpers cannot arrive for the next pass
        // before this wait)
        if (kHelp && xpass) named_bar_sync(3, 256);
        if (lane == 0) {
#ifdef XQ_ROLE_PROFILE
        prof_acc[12] += clock64() - pt_k;
#endif
          if (leader) mbar_arrive(&tempty[a]);
          else mbar_arrive_remote(tempty_leader0 + 8 * a);
        }
        ++tc;
      if (xpass) {
      // this exchange's local heads [h0, h1) (and the peer's same-numbered heads)
      const int h0 = split ? ps * (nbh / 2) : 0;
      const int h1 = split ? h0 + nbh / 2 : nbh;
      // ---- exchange: the peer owns query heads [peer*nbh, peer*nbh + nbh)
#ifdef XQ_ROLE_PROFILE
      const long long pt_x = clock64();
#endif
      // Each CTA's rows of the peer's heads are read out to registers, then
      // receive the peer's tokens' scores for this CTA's heads (no extra buffer).
      {
        float outv[kMaxHeads / 2];
#pragma unroll
        for (int hl = 0; hl < kMaxHeads / 2; ++hl) {
          const int h = static_cast<int>(peer) * nbh + hl;
          outv[hl] = (hl >= h0 && hl < h1 && h < p.n_q) ? lds_f32(sc_a + 4u * (h * kTileM + row))
                                                        : -INFINITY;
        }
        mbar_arrive_remote_release(xread_peer);        // my landing rows may be overwritten
        XQ_PROF(9, mbar_wait_cluster(xread, xc & 1));  // the peer's landing rows are free
#pragma unroll
        for (int hl = 0; hl < kMaxHeads / 2; ++hl)
          if (hl >= h0 && hl < h1)  // into the peer's landing row of my head hl
            st_cluster_f32(sc_peer + 4u * ((static_cast<int>(rank) * nbh + hl) * kTileM + row),
                           outv[hl]);
        mbar_arrive_remote_release(xfull_peer);
        XQ_PROF(9, mbar_wait_cluster(xfull, xc & 1));
        ++xc;
      }
      // ---- softmax over the 256 tokens of the tile for heads [h0, h1) -> P
      named_bar_sync(1, 128);  // every epilogue warp is done with q_s (P overwrites it)
      // ST tokens per thread: 32 (8 threads per head) or, for the 8 heads of a SPLIT
      // exchange, 16 (16 threads per head)
      auto softmax = [&](auto st_c) {
        constexpr int ST = decltype(st_c)::value;
        constexpr int NSEG = 256 / ST;
        constexpr int HPI = 128 / NSEG;  // heads per iteration
        const int seg = et % NSEG;       // tokens seg*ST .. +ST-1 of the pair tile
        const int tk0 = seg * ST;
        const int half = tk0 / kTileM;
        for (int hl = h0 + et / NSEG; hl < h1; hl += HPI) {
          const int h = static_cast<int>(rank) * nbh + hl;
          const uint32_t src = ((half == static_cast<int>(rank)) ? (sc_a + 4u * h * kTileM)
                                                                 : (land_a + 4u * hl * kTileM)) +
                               4u * (tk0 % kTileM);
          float s[ST];
#pragma unroll
          for (int i = 0; i < ST / 4; ++i) {
            const float4 v = (h < p.n_q) ? lds_f4(src + 16u * i)
                                         : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            s[4 * i] = v.x; s[4 * i + 1] = v.y; s[4 * i + 2] = v.z; s[4 * i + 3] = v.w;
          }
          float m = -INFINITY;
#pragma unroll
          for (int i = 0; i < ST; ++i) m = fmaxf(m, s[i]);
#pragma unroll
          for (int o = 1; o < NSEG; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
          float l = 0.f;
          uint32_t pk[ST / 2];
#pragma unroll
          for (int i = 0; i < ST / 2; ++i) {
            const float p0 = (m == -INFINITY) ? 0.f : exp2f(s[2 * i] - m);
            const float p1 = (m == -INFINITY) ? 0.f : exp2f(s[2 * i + 1] - m);
            const __half2 hp = __floats2half2_rn(p0, p1);
            // sum what the MMA will see (the fp16-rounded p)
            const float2 pr = __half22float2(hp);
            l += pr.x + pr.y;
            pk[i] = as_u32(hp);
          }
#pragma unroll
          for (int o = 1; o < NSEG; o <<= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
          // P stage j = tk0/64 holds tokens 64j..64j+63 as one 128-byte row per head
          const uint32_t pst = sP_a + (tk0 / 64) * (nbh * 128);
#pragma unroll
          for (int c = 0; c < ST / 8; ++c)
            sts128(pst + sw128_offset(hl, (tk0 % 64) / 8 + c), pk[4 * c], pk[4 * c + 1],
                   pk[4 * c + 2], pk[4 * c + 3]);
          if (seg == 0 && h < p.n_q)
            p.part_ml[((int64_t)b * p.n_tiles + t) * p.n_q + h] = make_float2(m, l);
        }
      };
      if (split) softmax(std::integral_constant<int, 16>());
      else softmax(std::integral_constant<int, 32>());
      if (ps == p.n_pass - 1) {  // P complete: the V side may start
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
#ifdef XQ_ROLE_PROFILE
        prof_acc[13] += clock64() - pt_x;
#endif
          if (leader) mbar_arrive(pready);
          else mbar_arrive_remote(pready_leader);
        }
        ++ti;
      }
      }
      },
      [&](const Tile& tl) {
      const int b = tl.b, t = tl.t;
      // ---- V side: drain O^T[channels x heads] of this tile
      int blk = 0, vbatch = 0;
      for (int us = 0; us < nuse; ++us, ++tc) {
        const uint32_t a = CF::NBUF == 2 ? (tc & 1) : 0u;
        const uint32_t aph = CF::NBUF == 2 ? ((tc >> 1) & 1) : (tc & 1);
        XQ_PROF(10, mbar_wait(&tfull[a], aph));
#ifdef XQ_ROLE_PROFILE
        const long long pt_v = clock64();
#endif
        tc_fence_after();
        // each [n_q x 128-channel] block is staged in shared memory and written
        // by one TMA bulk store. Staging buffers (8 KB at n_q = 32): both halves of
        // the score region, plus both halves of the q/P region when this is the
        // tile's only V-side accumulator use (with more uses, later uses' MMAs
        // still read P while this one drains). Blocks go out in batches of that
        // many buffers: one barrier and one store wait per batch, not per block.
        // (pipelined: the next tile's scores and q already live there -> one
        // dedicated staging buffer)
        const int nbuf = PIPE ? 1 : (nuse == 1 ? 4 : 2);
        const uint32_t blkb = 256u * p.n_q;  // bytes of one staged block
        auto stg_of = [&](int k) -> uint32_t {
          return PIPE ? stg_a : (k < 2 ? sc_a + k * blkb : q_a + (k - 2) * blkb);
        };
        int k = 0;  // position in the current batch
        for (int bi = 0; bi < bpu && blk < nblk; ++bi, ++blk) {
          const uint32_t stg = stg_of(k);
          if (k == 0 && vbatch > 0) {  // the previous batch's stores have read the buffers
            if (et == 0) tma_store_wait_read<0>();
            named_bar_sync(1, 128);
          }
          for (int c16 = 0; c16 < p.nb / 16; ++c16) {
            float v[16];
            tmem_ld16(tmem + tlane + a * 256 + bi * p.nb + c16 * 16, v);
            tmem_wait_ld();
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const int h = c16 * 16 + jj;
              if (h < p.n_q) {
                const __half hv = __float2half_rn(v[jj]);
                asm volatile("st.shared.b16 [%0], %1;" ::"r"(stg + 2u * (h * kTileM + row)),
                             "h"(*reinterpret_cast<const unsigned short*>(&hv))
                             : "memory");
              }
            }
          }
          ++k;
          if (k == nbuf || bi + 1 == bpu || blk + 1 == nblk) {  // batch complete: store it
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (et == 0) {
              for (int j = 0; j < k; ++j)
                tma_store_2d(&tmap_o, stg_of(j), (blk - k + 1 + j) * 256 + static_cast<int>(rank) * 128,
                             static_cast<int32_t>(((int64_t)b * p.n_tiles + t) * p.n_q));
              tma_store_commit();
            }
            k = 0;
            ++vbatch;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
#ifdef XQ_ROLE_PROFILE
        prof_acc[14] += clock64() - pt_v;
#endif
#pragma unroll
          for (int k = 0; k < (kHelp ? 2 : 1); ++k) {  // HELP: also the helper's share
            if (leader) mbar_arrive(&tempty[a]);
            else mbar_arrive_remote(tempty_leader0 + 8 * a);
          }
        }
      }
      });
  }
  if (warp == kEpiWarp0 && lane == 0) tma_store_wait_all();
#ifdef XQ_ROLE_PROFILE
  if (threadIdx.x == 0) prof_acc[11] = static_cast<unsigned long long>(clock64() - prof_t0);
  if (lane == 0)
    for (int c = 0; c < kProfCounters; ++c)
      if (prof_acc[c]) atomicAdd(&g_role_prof[c], prof_acc[c]);
#endif
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem, 512);
  }
}

// Merge the tile partials: x[b][h][c] = (sum_i 2^(m_i-M) O_i[h][c]) / (sum_i 2^(m_i-M) l_i).
// Grid (n_seqs*n_q, kdim/512), 128 threads x 4 channels (float4 loads, 8 tiles
// in flight per thread: the partials are streamed once from HBM/L2).
__global__ void __launch_bounds__(128) k_absorb_combine(const __half* __restrict__ part_o,
                                                        const float2* __restrict__ part_ml,
                                                        const int32_t* __restrict__ seq_lens,
                                                        int n_tiles, int n_q, int kdim,
                                                        float* __restrict__ x_out) {
  extern __shared__ float wts[];  // [n_tiles]
  __shared__ float red[4];
  const int bh = blockIdx.x, b = bh / n_q, h = bh % n_q, tid = threadIdx.x;
  const int len = seq_lens[b];
  const int nt = (len + kPairM - 1) / kPairM;
  const float2* ml = part_ml + (int64_t)b * n_tiles * n_q + h;
  float M = -INFINITY;
  for (int i = tid; i < nt; i += 128) M = fmaxf(M, ml[(int64_t)i * n_q].x);
  M = warp_max(M);
  if ((tid & 31) == 0) red[tid >> 5] = M;
  __syncthreads();
  M = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  float L = 0.f;
  for (int i = tid; i < nt; i += 128) {
    const float2 v = ml[(int64_t)i * n_q];
    const float wgt = (v.x == -INFINITY) ? 0.f : exp2f(v.x - M);
    wts[i] = wgt;
    L = fmaf(wgt, v.y, L);
  }
  L = warp_sum(L);
  if ((tid & 31) == 0) red[tid >> 5] = L;
  __syncthreads();
  L = red[0] + red[1] + red[2] + red[3];
  const float inv = L > 0.f ? 1.f / L : 0.f;
  const int c = blockIdx.y * 512 + tid * 4;
  if (c >= kdim) return;
  const int64_t stride = (int64_t)n_q * kdim;  // tile stride of the partials
  const __half* po = part_o + (int64_t)b * n_tiles * stride + (int64_t)h * kdim + c;
  auto ld4 = [&](int64_t off) {  // 4 fp16 partials -> float4 (streaming 8-byte load)
    const uint2 u = __ldcs(reinterpret_cast<const uint2*>(po + off));
    const float2 lo = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 hi = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    return make_float4(lo.x, lo.y, hi.x, hi.y);
  };
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int i = 0;
  for (; i + 8 <= nt; i += 8) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ld4((int64_t)(i + k) * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float w = wts[i + k];
      acc.x = fmaf(w, v[k].x, acc.x); acc.y = fmaf(w, v[k].y, acc.y);
      acc.z = fmaf(w, v[k].z, acc.z); acc.w = fmaf(w, v[k].w, acc.w);
    }
  }
  for (; i < nt; ++i) {
    const float4 v = ld4((int64_t)i * stride);
    const float w = wts[i];
    acc.x = fmaf(w, v.x, acc.x); acc.y = fmaf(w, v.y, acc.y);
    acc.z = fmaf(w, v.z, acc.z); acc.w = fmaf(w, v.w, acc.w);
  }
  *reinterpret_cast<float4*>(x_out + (int64_t)bh * kdim + c) =
      make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
}

// out[b][h][:] = x[b][h][:] @ W_v[:, kv(h)], wv fp16 [n_kv][kdim][128] (rows in the
// storage channel order of x). Grid (n_q, 4 column blocks of 32, ceil(n_seqs/8)):
// a CTA streams its [kdim x 32] slice of W_v once for up to 8 sequences (x
// staged in shared memory); 16 threads per row of the slice, 16 channel slices.
// Destinations of the projected output: this GPU's buffer, or under KV-head-group
// sharding this rank's slot in every rank's gather buffer (peer pointers over
// NVLink), so the all-gather is the projection's own stores.
constexpr int kMaxOuts = 9;  // 8 ranks + a local copy
struct OutPtrs {
  float* p[kMaxOuts];
  int n;
};

__global__ void __launch_bounds__(256) k_absorb_project(const float* __restrict__ x,
                                                        int n_seqs, int n_q, int group, int kdim,
                                                        const __half* __restrict__ wv,
                                                        const OutPtrs outs) {
  extern __shared__ float xs[];  // [kdim][8]: the 8 sequences' x of one channel contiguous
  __shared__ float red[8][8][33];
  const int h = blockIdx.x, cb = blockIdx.y, b0 = blockIdx.z * 8, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nb = n_seqs - b0 < 8 ? n_seqs - b0 : 8;
  const int kd4 = kdim / 4;
  for (int i = tid; i < 8 * kd4; i += 256) {
    const int s = i / kd4, c = 4 * (i % kd4);
    const float4 v = s < nb ? *reinterpret_cast<const float4*>(x + ((int64_t)(b0 + s) * n_q + h) * kdim + c)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    xs[c * 8 + s] = v.x;
    xs[(c + 1) * 8 + s] = v.y;
    xs[(c + 2) * 8 + s] = v.z;
    xs[(c + 3) * 8 + s] = v.w;
  }
  __syncthreads();
  // thread = (8-column group q of the 32-column block, channel slice sl of 64):
  // slice sl takes channels sl, sl+64, ... so a warp's 8 slices read 8 adjacent
  // W_v rows (16-byte loads) and 8 adjacent x rows
  const int q = tid & 3, sl = tid >> 2;
  const uint4* w16 = reinterpret_cast<const uint4*>(wv + (int64_t)(h / group) * kdim * 128 + cb * 32 + q * 8);
  float a[8][8];
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[s][j] = 0.f;
#pragma unroll 4
  for (int c = sl; c < kdim; c += 64) {
    const uint4 wr = __ldg(w16 + (int64_t)c * 16);
    const __half2* w2 = reinterpret_cast<const __half2*>(&wr);
    float wf[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __half22float2(w2[j]);
      wf[2 * j] = f.x;
      wf[2 * j + 1] = f.y;
    }
    const float4 x0 = *reinterpret_cast<const float4*>(xs + c * 8);
    const float4 x1 = *reinterpret_cast<const float4*>(xs + c * 8 + 4);
    const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int j = 0; j < 8; ++j) a[s][j] = fmaf(xv[s], wf[j], a[s][j]);
  }
  // lanes q, q+4, ..., q+28 of a warp hold 8 slices of the same outputs
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float v = a[s][j];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      a[s][j] = v;
    }
  if (lane < 4) {
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int j = 0; j < 8; ++j) red[warp][s][lane * 8 + j] = a[s][j];
  }
  __syncthreads();
  if (tid < nb * 32) {
    const int s = tid >> 5, j = tid & 31;
    float v = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) v += red[k][s][j];
    const int64_t o = ((int64_t)(b0 + s) * n_q + h) * kHeadDim + cb * 32 + j;
    for (int k = 0; k < outs.n; ++k) outs.p[k][o] = v;
  }
}

// Arranged weights. wk_out: fp16 [ceil(n_kv/4)*512][kdim], row kvh*128 + j =
// W_k[:, kvh*128 + j]^T with the channels in the K-side producer order (zero
// rows pad an odd n_kv). wv_out: fp16 [n_kv][kdim][128], row c = W_v[perm(c),
// kvh*128 .. +128] with perm the V-side producer order.
__global__ void k_arrange_absorbed(const void* __restrict__ w_k, const void* __restrict__ w_v, int dt,
                                   int64_t kdim, int n_kv, int n_pass, int bs_k, int bs_v,
                                   __half* __restrict__ wk_out, __half* __restrict__ wv_out) {
  const int64_t ld = (int64_t)n_kv * 128;
  const int64_t nk = (int64_t)n_pass * 512 * kdim;
  const int64_t nv = (int64_t)n_kv * kdim * 128;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nk + nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nk) {
      const int64_t pch = i % kdim, rowi = i / kdim;
      const int64_t k = (pch / bs_k) * bs_k + perm_channel(static_cast<int>(pch % bs_k), bs_k);
      // within a head: rows 0-63 = even dims, 64-127 = odd dims (split RoPE pairs)
      const int64_t cp = rowi & 127, dim = cp < 64 ? 2 * cp : 2 * (cp - 64) + 1;
      const int64_t col = (rowi & ~int64_t(127)) + dim;
      wk_out[i] = rowi < ld ? __float2half_rn(load_as_f32(w_k, dt, k * ld + col)) : __float2half_rn(0.f);
    } else {
      const int64_t e = i - nk;
      const int64_t j = e % 128, pch = (e / 128) % kdim, kvh = e / (128 * kdim);
      const int64_t k = (pch / bs_v) * bs_v + perm_channel(static_cast<int>(pch % bs_v), bs_v);
      wv_out[e] = __float2half_rn(load_as_f32(w_v, dt, k * ld + kvh * 128 + j));
    }
  }
}

}  // namespace absorb

// ------------------------------------------------------------ host side
namespace {

using namespace absorb;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

int num_sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

int make_map(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base, uint64_t inner,
             uint64_t rows, uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle sw,
             const char* what, CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
  auto enc = encode_fn();
  XQ_REQUIRE(enc != nullptr, XQ_ECUDA, "cuTensorMapEncodeTiled unavailable");
  XQ_REQUIRE(reinterpret_cast<uintptr_t>(base) % 16 == 0, XQ_ESHAPE, "%s: base not 16-byte aligned", what);
  XQ_REQUIRE((inner * esize) % 16 == 0, XQ_ESHAPE, "%s: row pitch %llu B not a multiple of 16", what,
             (unsigned long long)(inner * esize));
  const cuuint64_t gdim[2] = {inner, rows};
  const cuuint64_t gstride[1] = {inner * esize};
  const cuuint32_t box[2] = {box_inner, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  XQ_REQUIRE(r == CUDA_SUCCESS, XQ_ECUDA, "%s: cuTensorMapEncodeTiled failed (%d)", what, (int)r);
  return XQ_OK;
}

// codes map (box = one 128-channel group of 128 rows) + params map
int stream_maps(int mode, int bits, const void* src, const void* params, int64_t row_bytes,
                int64_t kdim, int G, int64_t rows, uint32_t f16_box_rows, CUtensorMap* codes,
                CUtensorMap* pmap) {
  int st;
  if (mode == XQ_A_F16_ROWS) {
    *pmap = CUtensorMap{};
    return make_map(codes, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, kdim, rows, kChunk, f16_box_rows,
                    CU_TENSOR_MAP_SWIZZLE_128B, "fp16 A rows");
  }
  XQ_REQUIRE(row_bytes == row_bytes_for(kdim, bits), XQ_ESHAPE, "row_bytes mismatch");
  if ((st = make_map(codes, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, src, row_bytes, rows, 16 * bits,
                     kTileM, CU_TENSOR_MAP_SWIZZLE_NONE, "codes", CU_TENSOR_MAP_L2_PROMOTION_L2_128B)) != XQ_OK)
    return st;
  if (mode == XQ_A_CODES_TOKEN)
    return make_map(pmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, params, param_stride(kdim, G) * 4, rows,
                    16, kTileM, CU_TENSOR_MAP_SWIZZLE_NONE, "params", CU_TENSOR_MAP_L2_PROMOTION_NONE);
  return make_map(pmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, params, kdim, 2 * (rows / G), 128, 2,
                  CU_TENSOR_MAP_SWIZZLE_NONE, "channel params", CU_TENSOR_MAP_L2_PROMOTION_NONE);
}

struct Maps {
  CUtensorMap w, ka, kp, va, vp, o;
};

int nb_for(int n_q) {
  const int nb = (n_q + 15) / 16 * 16;
  return nb < 16 ? 16 : nb;
}

int64_t n_tiles_for(int32_t max_len) {
  const int64_t nt = (max_len + kPairM - 1) / kPairM;
  return nt < 1 ? 1 : nt;
}

// Shared-memory plan: [AB ring][P][codes ring][q][scores][peer scores][barriers]
template <int AK, int AV, int BITS, int GROUP>
int plan_smem(Params& p, size_t& total) {
  constexpr bool PROD = AK != XQ_A_F16_ROWS && AK != XQ_A_F16_ACC;  // codes-ring modes
  const uint32_t k_code = PROD ? 128u * 16u * BITS : 0u;
  const uint32_t k_par = AK == XQ_A_CODES_TOKEN ? 128u * 16u : (AK == XQ_A_CODES_CHANNEL ? 512u : 0u);
  const uint32_t v_par = AV == XQ_A_CODES_TOKEN ? 128u * 16u : (AV == XQ_A_CODES_CHANNEL ? 512u : 0u);
  p.k_code_bytes = k_code;
  p.k_tx = k_code + k_par;
  p.v_tx = k_code + v_par;
  const uint32_t cst = PROD ? ((k_code + (k_par > v_par ? k_par : v_par) + 127) / 128 * 128) : 0u;
  p.cstage_bytes = cst;
  // q (fp32 [n_q][128]) and P (fp16 [4][nbh][64]) share one region: P is
  // written after the tile's last use of q, and q is rewritten only after the
  // V-side MMAs that read P have completed
  // pipelined (double-buffered) configs keep P and a V staging buffer apart,
  // the next tile's q and scores are live while this tile's V side drains
  constexpr bool PIPE = Cfg<GROUP>::NBUF == 2;
  const uint32_t qp = PIPE ? (512u * p.n_q + 1023u) / 1024u * 1024u
                           : ((512u * (p.n_q > p.nbh ? p.n_q : p.nbh)) + 1023u) / 1024u * 1024u;
  const uint32_t pbytes = PIPE ? (512u * p.nbh + 1023u) / 1024u * 1024u : 0u;
  const uint32_t stg = PIPE ? 256u * p.n_q : 0u;  // one fp16 [n_q x 128] O block
  const uint32_t fixed = qp + pbytes + stg                  // q / P (+ P, staging)
                         + 512u * p.nb                      // scores (+ the peer's, exchanged)
                         + (64 * 16 + 8 * 64) * 8           // RoPE offset + base tables
                         + (5 * kMaxStages + 8) * 8 + 16;   // barriers + tmem slot
  const uint32_t budget = 227u * 1024u - 1024u;
  using CF = Cfg<GROUP>;
  const int stages = CF::kStages;
  constexpr uint32_t kABStage = CF::kABStage;
  int cstages = PROD ? 4 : 2;
  auto need = [&]() { return stages * kABStage + cstages * cst + fixed; };
  while (need() > budget && cstages > 2) --cstages;
  XQ_REQUIRE(need() <= budget, XQ_ESHAPE, "shared memory plan does not fit (%d heads)", p.n_q);
  p.stages = stages;
  p.cstages = cstages;
  p.off_q = stages * kABStage;
  p.off_p = PIPE ? p.off_q + qp : p.off_q;
  p.off_codes = p.off_q + qp + pbytes;
  p.off_sc = p.off_codes + cstages * cst;
  p.off_stg = p.off_sc + 512u * p.nb;
  p.off_rope = p.off_stg + stg;
  p.off_bar = p.off_rope + (64 * 16 + 8 * 64) * 8;
  total = 1024 + need();
  return XQ_OK;
}

template <int AK, int AV, int BITS, int GROUP>
int launch(const Maps& m, Params p, cudaStream_t st) {
  p.n_pass = (p.n_kv + Cfg<GROUP>::KH - 1) / Cfg<GROUP>::KH;
  size_t smem = 0;
  int status = plan_smem<AK, AV, BITS, GROUP>(p, smem);
  if (status != XQ_OK) return status;
  auto kern = k_decode_absorbed<AK, AV, BITS, GROUP>;
  if ((status = ensure_smem(reinterpret_cast<const void*>(kern), 227 * 1024,
                            "cudaFuncSetAttribute(decode_absorbed)")) != XQ_OK)
    return status;
  if constexpr (GROUP == 4) {  // the score mma's q fragments (spare half of the fp16 partials)
    uint2* qf = reinterpret_cast<uint2*>(p.part_o + (int64_t)p.n_seqs * p.n_tiles * p.n_q * p.kdim);
    k_q_frags<<<dim3(p.n_seqs, p.n_kv), 256, 0, st>>>(p.q_pre, p.rope, p.rope_n, p.seq_lens, p.n_q, p.n_kv, GROUP,
                                        p.q_scale, qf);
    if ((status = check_launch("k_q_frags")) != XQ_OK) return status;
    p.q_frag = qf;
  }
  const int pairs = p.n_units < num_sms() / 2 ? p.n_units : num_sms() / 2;
  kern<<<2 * pairs, kThreads, smem, st>>>(m.w, m.ka, m.kp, m.va, m.vp, m.o, p);
  return check_launch("k_decode_absorbed");
}

template <int AK, int AV, int GROUP>
int dispatch_bits(int bits, const Maps& m, const Params& p, cudaStream_t st) {
  switch (bits) {
    case 2: return launch<AK, AV, 2, GROUP>(m, p, st);
    case 3: return launch<AK, AV, 3, GROUP>(m, p, st);
    case 4: return launch<AK, AV, 4, GROUP>(m, p, st);
    case 8: return launch<AK, AV, 8, GROUP>(m, p, st);
    default: return fail(XQ_ECONFIG, "unsupported bits %d", bits);
  }
}

// k_absorb_combine + k_absorb_project in one launch. A cluster of 4 CTAs takes one
// query head h and S sequences; CTA r merges the tile partials of channels
// [r*kdim/4, (r+1)*kdim/4) into x (shared memory, fp32; 16-byte loads, 8 tiles in
// flight) and projects them through its rows of W_v[:, kv(h)]; CTA 0 sums the four
// [S x 128] partial projections over DSMEM and writes the outputs. Same arithmetic as
// the two kernels up to the fp32 summation order of the projection.
constexpr int kFinishCta = 4;
template <int S>
__global__ void __cluster_dims__(kFinishCta, 1, 1) __launch_bounds__(256)
    k_absorb_finish(const __half* __restrict__ part_o, const float2* __restrict__ part_ml,
                    const int32_t* __restrict__ seq_lens, int n_seqs, int n_tiles, int n_q,
                    int group, int kdim, const __half* __restrict__ wv, const OutPtrs outs) {
  extern __shared__ float fsm[];  // x [S][kq], then weights [S][n_tiles]
  __shared__ float red[8][S][128];
  __shared__ float inv_s[S];
  __shared__ int nt_s[S];
  const uint32_t r = cluster_ctarank();
  const int h = blockIdx.x / kFinishCta, b0 = blockIdx.y * S, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int kq = kdim / kFinishCta, c0 = static_cast<int>(r) * kq;
  float* xs = fsm;
  float* wts = fsm + S * kq;
  // weights of the tiles of sequence s (warp s): 2^(m_i - M), and 1 / L
  for (int s = warp; s < S; s += 8) {
    const int b = b0 + s;
    int nt = 0;
    float inv = 0.f;
    if (b < n_seqs) {
      nt = (seq_lens[b] + kPairM - 1) / kPairM;
      const float2* ml = part_ml + (int64_t)b * n_tiles * n_q + h;
      float M = -INFINITY;
      for (int i = lane; i < nt; i += 32) M = fmaxf(M, ml[(int64_t)i * n_q].x);
      M = warp_max(M);
      float L = 0.f;
      for (int i = lane; i < nt; i += 32) {
        const float2 v = ml[(int64_t)i * n_q];
        const float wgt = (v.x == -INFINITY) ? 0.f : exp2f(v.x - M);
        wts[s * n_tiles + i] = wgt;
        L = fmaf(wgt, v.y, L);
      }
      L = warp_sum(L);
      inv = L > 0.f ? 1.f / L : 0.f;
    }
    if (lane == 0) {
      nt_s[s] = nt;
      inv_s[s] = inv;
    }
  }
  __syncthreads();
  // merge: item = (sequence, 8 channels of this CTA's quarter)
  const int64_t stride = (int64_t)n_q * kdim;  // tile stride of the partials
  for (int it = tid; it < S * (kq / 8); it += 256) {
    const int s = it / (kq / 8), cl = 8 * (it % (kq / 8));
    const int nt = nt_s[s];
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (nt > 0) {
      const __half* po = part_o + (int64_t)(b0 + s) * n_tiles * stride + (int64_t)h * kdim + c0 + cl;
      const float* w = wts + s * n_tiles;
      int i = 0;
      for (; i + 8 <= nt; i += 8) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldcs(reinterpret_cast<const uint4*>(po + (int64_t)(i + k) * stride));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float wk = w[i + k];
          const __half2* h2 = reinterpret_cast<const __half2*>(&v[k]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __half22float2(h2[e]);
            acc[2 * e] = fmaf(wk, f.x, acc[2 * e]);
            acc[2 * e + 1] = fmaf(wk, f.y, acc[2 * e + 1]);
          }
        }
      }
      for (; i < nt; ++i) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(po + (int64_t)i * stride));
        const float wk = w[i];
        const __half2* h2 = reinterpret_cast<const __half2*>(&v);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __half22float2(h2[e]);
          acc[2 * e] = fmaf(wk, f.x, acc[2 * e]);
          acc[2 * e + 1] = fmaf(wk, f.y, acc[2 * e + 1]);
        }
      }
    }
    const float inv = inv_s[s];
#pragma unroll
    for (int e = 0; e < 8; ++e) xs[s * kq + cl + e] = acc[e] * inv;
  }
  __syncthreads();
  // project this quarter: thread = (8-column group cg of 128, channel slice sl of 16)
  const int cg = tid & 15, sl = tid >> 4;
  const uint4* w16 = reinterpret_cast<const uint4*>(wv + ((int64_t)(h / group) * kdim + c0) * 128 + cg * 8);
  float a[S][8];
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[s][j] = 0.f;
#pragma unroll 4
  for (int c = sl; c < kq; c += 16) {
    const uint4 wr = __ldg(w16 + (int64_t)c * 16);
    const __half2* w2 = reinterpret_cast<const __half2*>(&wr);
    float wf[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __half22float2(w2[j]);
      wf[2 * j] = f.x;
      wf[2 * j + 1] = f.y;
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const float xv = xs[s * kq + c];
#pragma unroll
      for (int j = 0; j < 8; ++j) a[s][j] = fmaf(xv, wf[j], a[s][j]);
    }
  }
  // lanes l and l^16 hold slices 2w and 2w+1 of the same columns
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[s][j] += __shfl_xor_sync(0xffffffffu, a[s][j], 16);
  if (lane < 16) {
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int j = 0; j < 8; ++j) red[warp][s][cg * 8 + j] = a[s][j];
  }
  __syncthreads();
  // this CTA's partial projection [S][128] -> red[0]
  for (int i = tid; i < S * 128; i += 256) {
    const int s = i >> 7, j = i & 127;
    float v = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) v += red[k][s][j];
    red[0][s][j] = v;
  }
  cluster_sync();  // every CTA's partial is in its red[0]
  if (r == 0) {
    const uint32_t base = smem_u32(&red[0][0][0]);
    for (int i = tid; i < S * 128; i += 256) {
      const int s = i >> 7, j = i & 127;
      if (b0 + s >= n_seqs) continue;
      float v = red[0][s][j];
#pragma unroll
      for (int q = 1; q < kFinishCta; ++q) v += ld_cluster_f32(mapa_shared(base + 4u * i, q));
      const int64_t o = ((int64_t)(b0 + s) * n_q + h) * kHeadDim + j;
      for (int k = 0; k < outs.n; ++k) outs.p[k][o] = v;
    }
  }
  cluster_sync();  // the peers' red[0] stays alive until CTA 0 has read it
}

// k_absorb_combine + k_absorb_project after a k_decode_absorbed launch
int merge_and_project(const Params& p, const int32_t* seq_lens, int group,
                      const void* wv_arranged, const OutPtrs& op, cudaStream_t st) {
  int status;
  const int n_seqs = p.n_seqs, n_q = p.n_q;
  const int64_t kdim = p.kdim;
#ifndef XQ_SPLIT_FINISH
  if (kdim % (8 * kFinishCta) == 0) {
    // sequences per cluster: the most (<= 8) that still gives >= 128 clusters
    int S = 8;
    while (S > 1 && (int64_t)n_q * ((n_seqs + S - 1) / S) < 128) S >>= 1;
    const dim3 grid(kFinishCta * n_q, (n_seqs + S - 1) / S);
    const size_t fsmem = (size_t)S * (kdim / kFinishCta + p.n_tiles) * sizeof(float);
    const __half* wvh = static_cast<const __half*>(wv_arranged);
    auto go = [&](auto kern) -> int {
      int st2 = ensure_smem(reinterpret_cast<const void*>(kern), fsmem, "cudaFuncSetAttribute(finish)");
      if (st2 != XQ_OK) return st2;
      kern<<<grid, 256, fsmem, st>>>(p.part_o, p.part_ml, seq_lens, n_seqs, p.n_tiles, n_q, group,
                                     static_cast<int>(kdim), wvh, op);
      return check_launch("k_absorb_finish");
    };
    switch (S) {
      case 8: return go(k_absorb_finish<8>);
      case 4: return go(k_absorb_finish<4>);
      case 2: return go(k_absorb_finish<2>);
      default: return go(k_absorb_finish<1>);
    }
  }
#endif
  float* x_attn = reinterpret_cast<float*>(p.part_ml + (int64_t)n_seqs * p.n_tiles * n_q);
  k_absorb_combine<<<dim3(n_seqs * n_q, static_cast<unsigned>((kdim + 511) / 512)), 128,
                     p.n_tiles * sizeof(float), st>>>(p.part_o, p.part_ml, seq_lens, p.n_tiles,
                                                      n_q, p.kdim, x_attn);
  if ((status = check_launch("k_absorb_combine")) != XQ_OK) return status;
  const size_t psmem = 8 * (size_t)kdim * sizeof(float);
  // (dynamic; the kernel's 17 KB static reduction buffer comes on top)
  if ((status = ensure_smem(reinterpret_cast<const void*>(k_absorb_project), psmem,
                            "cudaFuncSetAttribute(project)")) != XQ_OK)
    return status;
  k_absorb_project<<<dim3(n_q, 4, (n_seqs + 7) / 8), 256, psmem, st>>>(
      x_attn, n_seqs, n_q, group, p.kdim, static_cast<const __half*>(wv_arranged), op);
  return check_launch("k_absorb_project");
}

}  // namespace
}  // namespace xq

using namespace xq;
using namespace xq::absorb;

extern "C" {

/* Role profile of the absorbed kernel (zeros unless built with XQ_ROLE_PROFILE):
 * reset != 0 clears the counters; out (if non-NULL) receives 16 uint64. */
int xq_debug_role_profile(uint64_t* out, int32_t reset) {
  if (out && cudaMemcpyFromSymbol(out, g_role_prof, sizeof(unsigned long long) * kProfCounters) !=
                 cudaSuccess)
    return check_launch("role profile read");
  if (reset) {
    static const unsigned long long zeros[kProfCounters] = {};
    if (cudaMemcpyToSymbol(g_role_prof, zeros, sizeof(zeros)) != cudaSuccess)
      return check_launch("role profile reset");
  }
  return XQ_OK;
}

int64_t xq_absorbed_workspace_bytes(int32_t n_seqs, int32_t max_len, int32_t n_q_heads,
                                    int64_t kdim) {
  // O partials (fp16, in a region sized for float32) + (m, l) per tile, then the
  // merged x [n_seqs][n_q][kdim]
  return (int64_t)n_seqs * n_q_heads *
         ((int64_t)n_tiles_for(max_len) * (kdim + 2) + kdim) * (int64_t)sizeof(float);
}

int xq_arrange_weights_absorbed(const void* w_k, const void* w_v, int32_t w_dtype, int64_t kdim,
                                int32_t n_kv_heads, int32_t a_mode_k, int32_t bits_k,
                                int32_t a_mode_v, int32_t bits_v, void* wk_out, void* wv_out,
                                void* stream) {
  XQ_REQUIRE(kdim % 256 == 0 && kdim > 0, XQ_ESHAPE, "kdim must be a positive multiple of 256, got %lld",
             (long long)kdim);
  XQ_REQUIRE(dtype_size(w_dtype) > 0, XQ_ECONFIG, "unknown dtype");
  XQ_REQUIRE(n_kv_heads >= 1, XQ_ESHAPE, "no KV heads");
  if (a_mode_v == XQ_A_SAME) {
    a_mode_v = a_mode_k;
    bits_v = bits_k;
  }
  const int n_pass = (n_kv_heads + 3) / 4;  // rows padded to whole groups of 4 KV heads
  const int bs_k = perm_block(a_mode_k, bits_k), bs_v = perm_block(a_mode_v, bits_v);
  const int64_t total = (int64_t)n_pass * 512 * kdim + (int64_t)n_kv_heads * kdim * 128;
  const int64_t blocks = (total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16;
  k_arrange_absorbed<<<static_cast<unsigned>(blocks), 256, 0, (cudaStream_t)stream>>>(
      w_k, w_v, w_dtype, kdim, n_kv_heads, n_pass, bs_k, bs_v, static_cast<__half*>(wk_out),
      static_cast<__half*>(wv_out));
  return check_launch("xq_arrange_weights_absorbed");
}

int xq_decode_attend_absorbed(int32_t ak_mode, const void* ak_src, const void* ak_params,
                              const float* ak_resid, const int32_t* ak_nflushed,
                              const float* ak_first, int32_t ak_bits,
                              int64_t ak_row_bytes, int32_t av_mode, const void* av_src,
                              const void* av_params, int32_t av_bits, int64_t av_row_bytes,
                              int32_t group_size, int64_t L_max, int64_t kdim,
                              const int32_t* seq_lens, int32_t n_seqs, int32_t max_len,
                              const void* wk_arranged, const void* wv_arranged, int32_t n_kv_heads,
                              int32_t group, const float* q_pre, const void* rope_cs,
                              int64_t rope_n, float sm_scale, void* workspace,
                              int64_t workspace_bytes, float* out, void* stream) {
  return xq_decode_attend_absorbed_peers(
      ak_mode, ak_src, ak_params, ak_resid, ak_nflushed, ak_first, ak_bits, ak_row_bytes, av_mode,
      av_src, av_params, av_bits, av_row_bytes, group_size, L_max, kdim, seq_lens, n_seqs, max_len,
      wk_arranged, wv_arranged, n_kv_heads, group, q_pre, rope_cs, rope_n, sm_scale, workspace,
      workspace_bytes, &out, 1, stream);
}

int xq_decode_attend_absorbed_peers(int32_t ak_mode, const void* ak_src, const void* ak_params,
                                    const float* ak_resid, const int32_t* ak_nflushed,
                                    const float* ak_first, int32_t ak_bits,
                                    int64_t ak_row_bytes, int32_t av_mode, const void* av_src,
                                    const void* av_params, int32_t av_bits, int64_t av_row_bytes,
                                    int32_t group_size, int64_t L_max, int64_t kdim,
                                    const int32_t* seq_lens, int32_t n_seqs, int32_t max_len,
                                    const void* wk_arranged, const void* wv_arranged,
                                    int32_t n_kv_heads, int32_t group, const float* q_pre,
                                    const void* rope_cs, int64_t rope_n, float sm_scale,
                                    void* workspace, int64_t workspace_bytes,
                                    float* const* outs, int32_t n_outs, void* stream) {
  XQ_REQUIRE(outs != nullptr && n_outs >= 1 && n_outs <= kMaxOuts, XQ_EUSAGE,
             "need 1..%d output pointers, got %d", kMaxOuts, n_outs);
  OutPtrs op{};
  op.n = n_outs;
  for (int i = 0; i < n_outs; ++i) {
    XQ_REQUIRE(outs[i] != nullptr, XQ_EUSAGE, "output pointer %d is null", i);
    op.p[i] = outs[i];
  }
  XQ_REQUIRE(rope_n >= max_len, XQ_ESHAPE, "rope table shorter than max_len");
  XQ_REQUIRE(kdim % 256 == 0 && kdim >= 256, XQ_ESHAPE,
             "kdim must be a positive multiple of 256, got %lld", (long long)kdim);
  XQ_REQUIRE(group_size == 32 || group_size == 64 || group_size == kG, XQ_ECONFIG,
             "the fused kernel takes quantization groups of 32, 64 or 128 channels, got %d",
             group_size);
  XQ_REQUIRE(group_size == kG || (ak_mode != XQ_A_CODES_CHANNEL && av_mode != XQ_A_CODES_CHANNEL),
             XQ_ECONFIG, "per-channel streams need 128-token groups (one per CTA tile), got %d",
             group_size);
  XQ_REQUIRE(n_seqs >= 1 && n_kv_heads >= 1, XQ_ESHAPE, "empty batch");
  XQ_REQUIRE(max_len <= L_max && max_len >= 1, XQ_ESHAPE, "max_len out of range");
  const int n_q = n_kv_heads * group;
  XQ_REQUIRE(n_q <= kMaxHeads, XQ_ECONFIG, "at most %d query heads per launch, got %d", kMaxHeads, n_q);
  XQ_REQUIRE(workspace_bytes >= xq_absorbed_workspace_bytes(n_seqs, max_len, n_q, kdim), XQ_ESHAPE,
             "workspace too small");
  const bool mha = av_mode == XQ_A_SAME;
  if (mha) {
    av_mode = ak_mode;
    av_src = ak_src;
    av_params = ak_params;
    av_bits = ak_bits;
    av_row_bytes = ak_row_bytes;
    XQ_REQUIRE(ak_mode == XQ_A_CODES_TOKEN || ak_mode == XQ_A_F16_ROWS ||
                   ak_mode == XQ_A_CODES_CHANNEL,
               XQ_ECONFIG, "shared A operand must be CODES_TOKEN, CODES_CHANNEL or F16_ROWS");
    XQ_REQUIRE(ak_mode != XQ_A_CODES_CHANNEL || L_max % group_size == 0, XQ_ECONFIG,
               "per-channel A operand needs L_max % 128 == 0");
  } else if (ak_mode == XQ_A_F16_ROWS) {  // 16-bit xq-gqa: raw K / V latent rows
    XQ_REQUIRE(av_mode == XQ_A_F16_ROWS, XQ_ECONFIG,
               "split fp16-row K latent needs an fp16-row V latent");
  } else {
    XQ_REQUIRE(ak_mode == XQ_A_CODES_CHANNEL && av_mode == XQ_A_CODES_TOKEN, XQ_ECONFIG,
               "split K/V A operands support (CODES_CHANNEL, CODES_TOKEN) or (F16_ROWS, F16_ROWS)");
    XQ_REQUIRE(ak_bits == av_bits, XQ_ECONFIG, "K and V latent bits must match");
    XQ_REQUIRE(L_max % group_size == 0, XQ_ECONFIG, "per-channel K latent needs L_max % 128 == 0");
  }
  XQ_REQUIRE(ak_mode == XQ_A_F16_ROWS || valid_bits(ak_bits), XQ_ECONFIG, "bad bits %d", ak_bits);
  const int64_t w_rows = (int64_t)(n_kv_heads + 3) / 4 * 512;
  const int64_t arena_rows = (int64_t)n_seqs * L_max;
  Maps maps;
  int st_;
  if ((st_ = make_map(&maps.w, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, wk_arranged, kdim,
                      (uint64_t)w_rows, kChunk, 128, CU_TENSOR_MAP_SWIZZLE_128B, "W_k")) != XQ_OK)
    return st_;
  if ((st_ = stream_maps(ak_mode, ak_bits, ak_src, ak_params, ak_row_bytes, kdim, group_size,
                         arena_rows, 128, &maps.ka, &maps.kp)) != XQ_OK)
    return st_;
  if ((st_ = stream_maps(av_mode, av_bits, av_src, av_params, av_row_bytes, kdim, group_size,
                         arena_rows, 64, &maps.va, &maps.vp)) != XQ_OK)
    return st_;

  const int64_t n_tiles = n_tiles_for(max_len);
  if ((st_ = make_map(&maps.o, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, workspace, kdim,
                      (uint64_t)n_seqs * n_tiles * n_q, 128, static_cast<uint32_t>(n_q),
                      CU_TENSOR_MAP_SWIZZLE_NONE, "O partials")) != XQ_OK)
    return st_;
  Params p{};
  p.k_resid = ak_resid;
  XQ_REQUIRE(ak_first == nullptr || (ak_mode == XQ_A_CODES_CHANNEL && !mha), XQ_ECONFIG,
             "the full-precision first channel applies to the per-channel K latent (xq-gqa)");
  p.k_first = ak_first;
  p.k_nflushed = ak_nflushed;
  p.kdim = static_cast<int32_t>(kdim);
  p.L_max = L_max;
  p.seq_lens = seq_lens;
  p.n_seqs = n_seqs;
  p.n_tiles = static_cast<int32_t>(n_tiles_for(max_len));
  p.n_units = n_seqs * p.n_tiles;
  p.n_kv = n_kv_heads;
  p.n_q = n_q;
  p.nb = nb_for(n_q);
  p.nbh = p.nb / 2;
  p.q_pre = q_pre;
  p.rope = static_cast<const float2*>(rope_cs);
  p.rope_n = rope_n;
  p.q_scale = sm_scale * 1.4426950408889634f;
  float* ws = static_cast<float*>(workspace);
  p.part_o = reinterpret_cast<__half*>(ws);
  p.part_ml = reinterpret_cast<float2*>(ws + (int64_t)n_seqs * p.n_tiles * n_q * kdim);
  // W_k stays L2-resident across the CTA pairs (evict_last). fp16-row A operand
  // (XQuant-CL delta layers): the serpentine sweeps keep the trailing half of each
  // sweep evict-last for the next one (C3: 30.7 -> 23.9 GB of DRAM reads per
  // launch, profiles/r01_c3_l2_policy.txt; 6-8 sixteenths measured best).
  p.w_hint = kEvictLast;
  p.a_hint = 1;
  p.a_split = (p.kdim / kChunk) / 2;
  p.G = group_size;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int status;
  if (mha) {
    // one A stream feeds K and V: X codes (xq-mha), the CL accumulator rows (F16),
    // or the xq-cl-gqa base-layer latent (per-channel codes, any query group)
    if (ak_mode == XQ_A_CODES_TOKEN) {
      XQ_REQUIRE(group == 1, XQ_ECONFIG, "a per-token shared A operand needs group 1, got %d", group);
      status = dispatch_bits<XQ_A_CODES_TOKEN, XQ_A_CODES_TOKEN, 1>(ak_bits, maps, p, st);
    } else if (ak_mode == XQ_A_F16_ROWS) {
      switch (group) {
        case 1: status = launch<XQ_A_F16_ROWS, XQ_A_F16_ROWS, 4, 1>(maps, p, st); break;
        case 2: status = launch<XQ_A_F16_ROWS, XQ_A_F16_ROWS, 4, 2>(maps, p, st); break;
        case 4: status = launch<XQ_A_F16_ROWS, XQ_A_F16_ROWS, 4, 4>(maps, p, st); break;
        default: return fail(XQ_ECONFIG, "unsupported query group %d (1, 2, 4)", group);
      }
    } else {
      switch (group) {
        case 1: status = dispatch_bits<XQ_A_CODES_CHANNEL, XQ_A_CODES_CHANNEL, 1>(ak_bits, maps, p, st); break;
        case 2: status = dispatch_bits<XQ_A_CODES_CHANNEL, XQ_A_CODES_CHANNEL, 2>(ak_bits, maps, p, st); break;
        case 4: status = dispatch_bits<XQ_A_CODES_CHANNEL, XQ_A_CODES_CHANNEL, 4>(ak_bits, maps, p, st); break;
        default: return fail(XQ_ECONFIG, "unsupported query group %d (1, 2, 4)", group);
      }
    }
  } else if (ak_mode == XQ_A_F16_ROWS) {  // K passes read tmap_ka, the V side tmap_va
    switch (group) {
      case 1: status = launch<XQ_A_F16_ROWS, XQ_A_F16_ROWS, 4, 1>(maps, p, st); break;
      case 2: status = launch<XQ_A_F16_ROWS, XQ_A_F16_ROWS, 4, 2>(maps, p, st); break;
      case 4: status = launch<XQ_A_F16_ROWS, XQ_A_F16_ROWS, 4, 4>(maps, p, st); break;
      default: return fail(XQ_ECONFIG, "unsupported GQA group %d (1, 2, 4)", group);
    }
  } else {
    switch (group) {
      case 1: status = dispatch_bits<XQ_A_CODES_CHANNEL, XQ_A_CODES_TOKEN, 1>(ak_bits, maps, p, st); break;
      case 2: status = dispatch_bits<XQ_A_CODES_CHANNEL, XQ_A_CODES_TOKEN, 2>(ak_bits, maps, p, st); break;
      case 4: status = dispatch_bits<XQ_A_CODES_CHANNEL, XQ_A_CODES_TOKEN, 4>(ak_bits, maps, p, st); break;
      default: return fail(XQ_ECONFIG, "unsupported GQA group %d (1, 2, 4)", group);
    }
  }
  if (status != XQ_OK) return status;
  return merge_and_project(p, seq_lens, group, wv_arranged, op, st);
}

int xq_decode_attend_absorbed_cl(void* acc16, const void* codes, const void* params, int32_t bits,
                                 int64_t row_bytes, int32_t group_size, int64_t L_max,
                                 int64_t kdim, const int32_t* seq_lens, int32_t n_seqs,
                                 int32_t max_len, const void* wk_arranged,
                                 const void* wv_arranged, int32_t n_kv_heads, const float* q_pre,
                                 const void* rope_cs, int64_t rope_n, float sm_scale,
                                 void* workspace, int64_t workspace_bytes, float* out,
                                 void* stream) {
  XQ_REQUIRE(acc16 && codes && params && out, XQ_EUSAGE, "null argument");
  XQ_REQUIRE(rope_n >= max_len, XQ_ESHAPE, "rope table shorter than max_len");
  XQ_REQUIRE(kdim % 256 == 0 && kdim >= 256, XQ_ESHAPE,
             "kdim must be a positive multiple of 256, got %lld", (long long)kdim);
  XQ_REQUIRE(group_size == 32 || group_size == 64 || group_size == kG, XQ_ECONFIG,
             "the fused kernel takes quantization groups of 32, 64 or 128 channels, got %d",
             group_size);
  XQ_REQUIRE(valid_bits(bits), XQ_ECONFIG, "bad bits %d", bits);
  XQ_REQUIRE(n_seqs >= 1 && n_kv_heads >= 1, XQ_ESHAPE, "empty batch");
  XQ_REQUIRE(max_len <= L_max && max_len >= 1, XQ_ESHAPE, "max_len out of range");
  const int n_q = n_kv_heads;
  XQ_REQUIRE(n_q <= kMaxHeads, XQ_ECONFIG, "at most %d query heads per launch, got %d", kMaxHeads, n_q);
  XQ_REQUIRE(workspace_bytes >= xq_absorbed_workspace_bytes(n_seqs, max_len, n_q, kdim), XQ_ESHAPE,
             "workspace too small");
  const int64_t w_rows = (int64_t)(n_kv_heads + 3) / 4 * 512;
  const int64_t arena_rows = (int64_t)n_seqs * L_max;
  Maps maps;
  int st_;
  // ka / va: the accumulator rows (K-pass and V-side boxes); the producer warps read
  // the delta codes and their (scale, zp) directly
  if ((st_ = make_map(&maps.w, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, wk_arranged, kdim,
                      (uint64_t)w_rows, kChunk, 128, CU_TENSOR_MAP_SWIZZLE_128B, "W_k")) != XQ_OK)
    return st_;
  if ((st_ = stream_maps(XQ_A_F16_ROWS, 16, acc16, nullptr, 0, kdim, group_size, arena_rows, 128,
                         &maps.ka, &maps.kp)) != XQ_OK)
    return st_;
  if ((st_ = stream_maps(XQ_A_F16_ROWS, 16, acc16, nullptr, 0, kdim, group_size, arena_rows, 64,
                         &maps.va, &maps.vp)) != XQ_OK)
    return st_;
  XQ_REQUIRE(row_bytes == row_bytes_for(kdim, bits), XQ_ESHAPE, "row_bytes mismatch");
  const int64_t n_tiles = n_tiles_for(max_len);
  if ((st_ = make_map(&maps.o, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, workspace, kdim,
                      (uint64_t)n_seqs * n_tiles * n_q, 128, static_cast<uint32_t>(n_q),
                      CU_TENSOR_MAP_SWIZZLE_NONE, "O partials")) != XQ_OK)
    return st_;
  Params p{};
  p.kdim = static_cast<int32_t>(kdim);
  p.L_max = L_max;
  p.seq_lens = seq_lens;
  p.n_seqs = n_seqs;
  p.n_tiles = static_cast<int32_t>(n_tiles);
  p.n_units = n_seqs * p.n_tiles;
  p.n_kv = n_kv_heads;
  p.n_q = n_q;
  p.nb = nb_for(n_q);
  p.nbh = p.nb / 2;
  p.q_pre = q_pre;
  p.rope = static_cast<const float2*>(rope_cs);
  p.rope_n = rope_n;
  p.q_scale = sm_scale * 1.4426950408889634f;
  float* ws = static_cast<float*>(workspace);
  p.part_o = reinterpret_cast<__half*>(ws);
  p.part_ml = reinterpret_cast<float2*>(ws + (int64_t)n_seqs * p.n_tiles * n_q * kdim);
  p.w_hint = kEvictLast;
  p.a_hint = 1;  // the later passes' fp16 rows: the split L2 policy of the F16 path
  p.a_split = (p.kdim / kChunk) / 2;
  p.G = group_size;
  p.acc_out = static_cast<__half*>(acc16);
  p.d_codes = static_cast<const uint8_t*>(codes);
  p.d_params = static_cast<const __half2*>(params);
  p.d_row_bytes = row_bytes;
  p.d_pstride = param_stride(kdim, group_size);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int status;
  switch (bits) {
    case 2: status = launch<XQ_A_F16_ACC, XQ_A_F16_ACC, 2, 1>(maps, p, st); break;
    case 3: status = launch<XQ_A_F16_ACC, XQ_A_F16_ACC, 3, 1>(maps, p, st); break;
    case 4: status = launch<XQ_A_F16_ACC, XQ_A_F16_ACC, 4, 1>(maps, p, st); break;
    default: status = launch<XQ_A_F16_ACC, XQ_A_F16_ACC, 8, 1>(maps, p, st); break;
  }
  if (status != XQ_OK) return status;
  OutPtrs op{};
  op.n = 1;
  op.p[0] = out;
  return merge_and_project(p, seq_lens, 1, wv_arranged, op, st);
}

}  // extern "C"
