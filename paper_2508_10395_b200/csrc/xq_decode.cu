// Fused XQuant decode: dequant -> rematerialise on tcgen05 -> RoPE ->
// flash-decode, for sm_100a. K and V never touch HBM.
//
// Reference semantics (the thing this replaces, per sequence and layer):
//   x_hat = stream.reconstruct()                          cache.py:223-230
//   K = apply_rope(x_hat @ W_k, 0..l-1), V = x_hat @ W_v    cache.py:385-387 (xq-mha)
//   K = RoPE(lat_k_hat @ fused_k), V = lat_v_hat @ fused_v  cache.py:434-437 (xq-gqa)
//   out_h = softmax(q_h K_{h//g}^T / sqrt(hd)) V_{h//g}     model.py:150-182
//
// One persistent CTA per SM (512 threads, warp-specialised):
//   warp 0       TMA producer of the weight tiles (W_k|W_v rows of one KV head)
//   warp 1       TMEM allocator + single-thread tcgen05.mma issuer
//   warps 4-11   two groups of 4 dequant producers (even / odd K-chunks):
//                packed codes -> fp16 pairs (magic-number convert + HFMA2)
//                -> SWIZZLE_128B K-major A tile in shared memory
//   warps 12-15  epilogue: tcgen05.ld the [128 x 256] fp32 accumulator
//                (cols 0-127 = K_pre, 128-255 = V), RoPE, q.k, per-warp online
//                softmax, p.V via warp reduce-scatter -> split partials
// Work unit = (sequence, chunk of 128-token tiles, KV head); a combine
// kernel merges the per-(chunk, warp) partials.
#include <cudaTypedefs.h>
#include <math.h>
#include <stdlib.h>

#include "xq_common.cuh"
#include "xq_host.h"
#include "xq_layout.cuh"
#include "xq_dequant.cuh"

namespace xq {

constexpr int kTileM = 128;  // token rows per CTA (TMEM lanes)
constexpr int kPairM = 256;  // token rows per CTA pair (cta_group::2 MMA, M = 256)
constexpr int kChunk = 64;  // K elements per stage (128 B of fp16 = one swizzle row)
constexpr int kThreads = 512;
constexpr int kProdWarp0 = 4;
constexpr int kEpiWarp0 = 12;
constexpr int kPartStride = 2 + kHeadDim;  // m, l, o[128]
constexpr int kPartsPerChunk = 8;          // 2 CTAs x 4 epilogue warps
constexpr int kG = 128;                    // quantization group (the reference default, cache.py:44)
constexpr uint32_t kABytes = kTileM * 128;  // 16 KB
constexpr uint32_t kBBytes = 128 * 128;     // 16 KB: this CTA's half (N/2 = 128 rows) of W

struct DecodeParams {
  const uint8_t* ak_src;
  const void* ak_params;
  const float* ak_resid;
  const int32_t* ak_nflushed;
  int64_t ak_row_bytes;
  const uint8_t* av_src;
  const void* av_params;
  int64_t av_row_bytes;
  int32_t group_size;
  int64_t L_max;
  int32_t kdim;
  const int32_t* seq_lens;
  int32_t n_chunks;
  int32_t tiles_per_chunk;
  int32_t n_kv;
  int32_t n_units;
  int32_t n_seqs;
  int32_t head_block;  // KV heads per scheduling block (divides n_kv)
  const float* q_pre;
  const float2* rope;  // frequency-major [64][rope_n]
  int64_t rope_n;
  float q_scale;  // sm_scale * log2(e)
  float* partials;
  float* dbg_acc;  // optional: raw [b][h][tile][128][256] accumulator dump
  int32_t dbg_tiles;
  uint64_t w_hint;  // L2 cache policy of the weight TMA loads
};

static float* g_dbg_acc = nullptr;
static int32_t g_dbg_tiles = 0;

struct Unit {
  int b, chunk, h, t0, t1, len;
};

// Unit order: KV head fastest inside a block of `head_block` heads, then token
// chunk, then sequence, then head block. Pairs in flight then share a few
// token ranges (codes re-read from L2) and one block of W (L2-resident).
XQ_DEVINL Unit get_unit(const DecodeParams& p, int u) {
  Unit w;
  const int hbs = p.head_block;
  const int h_in = u % hbs;
  int rest = u / hbs;
  w.chunk = rest % p.n_chunks;
  rest /= p.n_chunks;
  w.b = rest % p.n_seqs;
  w.h = (rest / p.n_seqs) * hbs + h_in;
  w.len = p.seq_lens[w.b];
  const int nt = (w.len + kPairM - 1) / kPairM;  // tiles of 256 tokens (one per CTA pair)
  w.t0 = w.chunk * p.tiles_per_chunk;
  w.t1 = min(w.t0 + p.tiles_per_chunk, nt);
  if (w.t1 < w.t0) w.t1 = w.t0;
  return w;
}

// ---------------------------------------------------------------------------
// Codes ring: a dedicated TMA thread stages, per 128-channel group of a
// 128-token tile, the packed codes of every A stream (box [16*BITS B, 128
// rows]) and, for per-token streams, the half2 (scale, zp) quads (box
// [4 x u32, 128 rows]) into shared memory. Producers then read shared memory
// only, so the LSU pipe carries no uncoalesced global traffic.
// ---------------------------------------------------------------------------
template <int AK, int AV, int BITS>
struct Ring {
  static constexpr bool kProducers = AK != XQ_A_F16_ROWS;
  static constexpr int kStreams = (AV == XQ_A_SAME) ? 1 : 2;
  static constexpr int kGB = 16 * BITS;                           // code bytes per row per group
  static constexpr int kTokenStreams = (AK == XQ_A_CODES_TOKEN) + (AV == XQ_A_CODES_TOKEN);
  static constexpr uint32_t kCodeBytes = kTileM * kGB;
  static constexpr uint32_t kParamBytes = kTileM * 16;        // per-token (scale, zp) quads
  static constexpr uint32_t kChanParamBytes = 2 * 128 * 2;     // per-channel scales + zps
  static constexpr uint32_t kParam0Bytes =
      AK == XQ_A_CODES_TOKEN ? kParamBytes : (AK == XQ_A_CODES_CHANNEL ? kChanParamBytes : 0);
  static constexpr uint32_t kParam1Bytes = AV == XQ_A_CODES_TOKEN ? kParamBytes : 0;
  static constexpr uint32_t kTxBytes = kStreams * kCodeBytes + kParam0Bytes + kParam1Bytes;
  static constexpr uint32_t kStageBytes = kProducers ? ((kTxBytes + 127) / 128 * 128) : 0;
  static constexpr uint32_t kABStage = kStreams * kABytes + kBBytes;
  static constexpr int kABStages = kStreams == 1 ? (BITS == 8 ? 4 : 5) : (BITS == 8 ? 2 : 3);
  static constexpr uint32_t kABBytes = kABStages * kABStage;
  static constexpr uint32_t kEpiScratch = 4 * 32 * 36 * 4 + 4 * 32 * 8 * 4;  // V transpose + p
  static constexpr uint32_t kBudget = 222 * 1024 - kABBytes - 6 * 1024 - kEpiScratch;
  static constexpr int kCodeStages =
      !kProducers ? 0 : (kBudget / kStageBytes >= 4 ? 4 : (kBudget / kStageBytes < 1 ? 1 : kBudget / kStageBytes));
  // stage layout: [s0 codes][s1 codes][s0 params if TOKEN][s1 params if TOKEN]
  __host__ __device__ static constexpr uint32_t code_off(int stream) { return stream * kCodeBytes; }
  __host__ __device__ static constexpr uint32_t param_off(int stream) {
    return kStreams * kCodeBytes + (stream == 1 ? kParam0Bytes : 0);
  }
};

// p rows of the epilogue's shared scratch: padded to a 16-byte vector
template <int GROUP>
constexpr int kPStride = GROUP == 1 ? 1 : (GROUP == 2 ? 2 : 4 * ((GROUP + 3) / 4));
template <int GROUP>
XQ_DEVINL void load_p(const float* src, float (&pv)[kPStride<GROUP>]) {
  if constexpr (GROUP == 1) {
    pv[0] = src[0];
  } else if constexpr (GROUP == 2) {
    const float2 t = *reinterpret_cast<const float2*>(src);
    pv[0] = t.x; pv[1] = t.y;
  } else {
#pragma unroll
    for (int q = 0; q < kPStride<GROUP> / 4; ++q) {
      const float4 t = reinterpret_cast<const float4*>(src)[q];
      pv[4 * q] = t.x; pv[4 * q + 1] = t.y; pv[4 * q + 2] = t.z; pv[4 * q + 3] = t.w;
    }
  }
}

template <int AK, int AV, int BITS, int GROUP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_decode_attend(const __grid_constant__ CUtensorMap tmap_w,
                    const __grid_constant__ CUtensorMap tmap_ca,
                    const __grid_constant__ CUtensorMap tmap_pa,
                    const __grid_constant__ CUtensorMap tmap_cb,
                    const __grid_constant__ CUtensorMap tmap_pb, const DecodeParams p) {
  using R = Ring<AK, AV, BITS>;
  constexpr int A_TILES = R::kStreams;
  constexpr int STAGES = R::kABStages;
  constexpr int CSTAGES = R::kCodeStages;
  constexpr bool PROD = R::kProducers;
  constexpr int AVM = (AV == XQ_A_SAME) ? AK : AV;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  // per stage: [A stream 0][A stream 1][B half]
  uint8_t* sAB = smem;
  uint8_t* sC = sAB + STAGES * R::kABStage;  // codes ring
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + CSTAGES * R::kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* cfull = empty + STAGES;
  uint64_t* cempty = cfull + 4;
  uint64_t* tfull = cempty + 4;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* q_s = reinterpret_cast<float*>(tmem_slot + 4);  // [GROUP][128]
  float* epi_v = q_s + GROUP * kHeadDim;                  // [4 warps][32 rows][36]
  float* epi_p = epi_v + 4 * 32 * 36;                     // [4 warps][32 rows][GROUP pad]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();  // 0 = leader (issues the MMA), 1 = peer
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // leader's full: 2 TMA arrivals (one per CTA) + 8 producer warps (4 per CTA)
      mbar_init(&full[s], PROD ? 2 + 8 : 2);
      mbar_init(&empty[s], 1);  // multicast MMA commit
    }
    for (int s = 0; s < CSTAGES; ++s) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], 4);  // the 4 warps of the producer group that owns the stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);   // multicast MMA commit
      mbar_init(&tempty[a], 8);  // leader's: 4 epilogue warps per CTA
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    if constexpr (!PROD) tma_prefetch_desc(&tmap_ca);
  }
  if (warp == 2 && lane == 0 && PROD) {  // descriptor prefetch
    tma_prefetch_desc(&tmap_ca);
    tma_prefetch_desc(&tmap_pa);
    if constexpr (A_TILES == 2) {
      tma_prefetch_desc(&tmap_cb);
      tma_prefetch_desc(&tmap_pb);
    }
  }
  if (warp == 1) {
    tmem_alloc2(tmem_slot, 512);
    tmem_relinquish2();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nkc = p.kdim / kChunk;
  const uint32_t full_leader0 = mapa_shared(smem_u32(&full[0]), 0);
  const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);

  if (warp == 0) {
    // ------------------------------------------------ TMA: this CTA's W half (+ fp16 A rows)
    uint32_t it = 0;
    for (int u = cluster; u < p.n_units; u += n_clusters) {
      const Unit w = get_unit(p, u);
      for (int t = w.t0; t < w.t1; ++t) {
        const int32_t arow0 = static_cast<int32_t>((int64_t)w.b * p.L_max + t * kPairM + rank * kTileM);
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (elect_one()) {
            uint8_t* st = sAB + s * R::kABStage;
            constexpr uint32_t kTx = 2 * (kBBytes + (PROD ? 0u : kABytes));  // both CTAs
            if (leader) mbar_arrive_expect_tx(&full[s], kTx);
            else mbar_arrive_remote(full_leader0 + 8 * s);
            if constexpr (A_TILES == 1) {  // rows [K_h | V_h] of head h: this CTA's 128
              tma_load_2d_pair(st + kABytes, &tmap_w, &full[s], kc * kChunk,
                               w.h * 256 + rank * 128, p.w_hint);
            } else {  // K half (64 rows of W_k) + V half (64 rows of W_v)
              tma_load_2d_pair(st + 2 * kABytes, &tmap_w, &full[s], kc * kChunk,
                               w.h * 256 + rank * 64, p.w_hint);
              tma_load_2d_pair(st + 2 * kABytes + 64 * 128, &tmap_w, &full[s], kc * kChunk,
                               w.h * 256 + 128 + rank * 64, p.w_hint);
            }
            if constexpr (!PROD)
              tma_load_2d_pair(st, &tmap_ca, &full[s], kc * kChunk, arow0, kEvictNormal);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader CTA only)
    if (leader) {
      constexpr uint32_t kIdesc256 = idesc_f16_f32(256, 256);
      constexpr uint32_t kIdesc128 = idesc_f16_f32(256, 128);
      const uint64_t desc0 = sdesc_sw128(smem_u32(sAB));
      uint32_t it = 0, tc = 0;
      for (int u = cluster; u < p.n_units; u += n_clusters) {
        const Unit w = get_unit(p, u);
        for (int t = w.t0; t < w.t1; ++t, ++tc) {
          const uint32_t a = tc & 1, aph = (tc >> 1) & 1;
          mbar_wait_cluster(&tempty[a], aph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + a * 256;
          for (int kc = 0; kc < nkc; ++kc, ++it) {
            const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
            mbar_wait_cluster(&full[s], ph);
            tc_fence_after();
            // descriptor start-address field is addr>>4: +2 per 32-byte K step
            const uint64_t ad = desc0 + ((s * R::kABStage) >> 4);
            const uint64_t bd = ad + ((A_TILES * kABytes) >> 4);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < kChunk / 16; ++k) {
                const uint32_t acc = (kc | k) != 0;
                if constexpr (A_TILES == 1) {
                  mma2_f16_ss(d, ad + 2 * k, bd + 2 * k, kIdesc256, acc);
                } else {
                  mma2_f16_ss(d, ad + 2 * k, bd + 2 * k, kIdesc128, acc);
                  mma2_f16_ss(d + 128, ad + (kABytes >> 4) + 2 * k, bd + ((64 * 128) >> 4) + 2 * k,
                              kIdesc128, acc);
                }
              }
              mma2_commit_both(&empty[s]);
            }
            __syncwarp();
          }
          if (elect_one()) mma2_commit_both(&tfull[a]);
          __syncwarp();
        }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------ TMA: codes ring (this CTA's rows)
    if constexpr (PROD) {
      uint32_t ci = 0;
      for (int u = cluster; u < p.n_units; u += n_clusters) {
        const Unit w = get_unit(p, u);
        for (int t = w.t0; t < w.t1; ++t) {
          const int32_t arow0 =
              static_cast<int32_t>((int64_t)w.b * p.L_max + t * kPairM + rank * kTileM);
          for (int g = 0; g < nkc / 2; ++g, ++ci) {
            const uint32_t cs = ci % CSTAGES, cph = (ci / CSTAGES) & 1;
            mbar_wait(&cempty[cs], cph ^ 1);
            if (elect_one()) {
              uint8_t* st = sC + cs * R::kStageBytes;
              mbar_arrive_expect_tx(&cfull[cs], R::kTxBytes);
              // params quad holding this 128-channel block's group(s); a TMA box must
              // start on a 16-byte boundary of the inner dimension
              const int32_t pq = g & ~3;  // G = 128: group g of the row
              tma_load_2d(st + R::code_off(0), &tmap_ca, &cfull[cs], g * R::kGB, arow0, kEvictNormal);
              if constexpr (AK == XQ_A_CODES_TOKEN)
                tma_load_2d(st + R::param_off(0), &tmap_pa, &cfull[cs], 4 * pq, arow0, kEvictNormal);
              if constexpr (AK == XQ_A_CODES_CHANNEL)  // [scales | zps] of this token group
                tma_load_2d(st + R::param_off(0), &tmap_pa, &cfull[cs], g * 128,
                            2 * (arow0 / kG), kEvictNormal);
              if constexpr (A_TILES == 2) {
                tma_load_2d(st + R::code_off(1), &tmap_cb, &cfull[cs], g * R::kGB, arow0, kEvictNormal);
                tma_load_2d(st + R::param_off(1), &tmap_pb, &cfull[cs], 4 * pq, arow0, kEvictNormal);
              }
            }
            __syncwarp();
          }
        }
      }
    }
  } else if (warp >= kProdWarp0 && warp < kEpiWarp0) {
    // ------------------------------------------------ dequant producers
    // Group gp owns the codes groups (128 channels = two K-chunks) whose running
    // index is == gp (mod 2); per owned group: one codes-stage wait, two A stages.
    if constexpr (PROD) {
      const int gp = (warp - kProdWarp0) >> 2;
      const int row = ((warp - kProdWarp0) & 3) * 32 + lane;  // tile row = token
      const RowSwizzle sw(row);
      const uint32_t sAB_a = smem_u32(sAB), sC_a = smem_u32(sC);
      const int ngrp = nkc / 2;
      uint32_t tcount = 0;
      for (int u = cluster; u < p.n_units; u += n_clusters) {
        const Unit w = get_unit(p, u);
        const int nfl = (AK == XQ_A_CODES_CHANNEL) ? __ldg(p.ak_nflushed + w.b) : 0;
        for (int t = w.t0; t < w.t1; ++t, ++tcount) {
          const int tok = t * kPairM + rank * kTileM + row;
          const bool valid = tok < w.len;
          const uint32_t ci0 = tcount * ngrp;
          for (int g = (ci0 & 1) == static_cast<uint32_t>(gp) ? 0 : 1; g < ngrp; g += 2) {
            const uint32_t ci = ci0 + g;
            const uint32_t cs = ci % CSTAGES, cph = (ci / CSTAGES) & 1;
            const uint32_t st = sC_a + cs * R::kStageBytes;
            mbar_wait(&cfull[cs], cph);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int kc = 2 * g + h;
              const uint32_t it = tcount * nkc + kc;
              const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
              mbar_wait(&empty[s], ph ^ 1);
              const uint32_t tile = sAB_a + s * R::kABStage;
              produce_chunk<AK, BITS>(tile, st + R::code_off(0), st + R::param_off(0), sw, row,
                                      valid, tok, w.b, nfl, kc, nullptr, p.ak_resid, p.kdim);
              if constexpr (A_TILES == 2)
                produce_chunk<AVM, BITS>(tile + kABytes, st + R::code_off(1), st + R::param_off(1),
                                         sw, row, valid, tok, w.b, 1 << 30, kc, nullptr,
                                         nullptr, p.kdim);
              fence_proxy_async_smem();
              __syncwarp();
              if (leader) mbar_arrive_if(&full[s], lane == 0);
              else mbar_arrive_remote_if(full_leader0 + 8 * s, lane == 0);
            }
            mbar_arrive_if(&cempty[cs], lane == 0);
          }
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ------------------------------------------------ epilogue (this CTA's 128 rows)
    const int ew = warp - kEpiWarp0;  // == warp % 4: TMEM lanes 32*ew ..
    const int et = threadIdx.x - kEpiWarp0 * 32;
    const int row = ew * 32 + lane;
    const uint32_t tlane = static_cast<uint32_t>(ew * 32) << 16;
    const int n_q = p.n_kv * GROUP;
    uint32_t tc = 0;
    for (int u = cluster; u < p.n_units; u += n_clusters) {
      const Unit w = get_unit(p, u);
      const int pos = w.len - 1;
      named_bar_sync(1, 128);
      if (pos >= 0) {
        const float2 cs = p.rope[(int64_t)(et >> 1) * p.rope_n + pos];
#pragma unroll
        for (int gi = 0; gi < GROUP; ++gi) {
          const float* qp = p.q_pre + ((int64_t)w.b * n_q + w.h * GROUP + gi) * kHeadDim;
          const float e0 = qp[et & ~1], e1 = qp[et | 1];
          const float r = (et & 1) ? (e0 * cs.y + e1 * cs.x) : (e0 * cs.x - e1 * cs.y);
          q_s[gi * kHeadDim + et] = r * p.q_scale;
        }
      }
      named_bar_sync(1, 128);
      float m_run[GROUP], l_run[GROUP], o_run[GROUP][4];
#pragma unroll
      for (int gi = 0; gi < GROUP; ++gi) {
        m_run[gi] = -INFINITY;
        l_run[gi] = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) o_run[gi][c] = 0.f;
      }
      for (int t = w.t0; t < w.t1; ++t, ++tc) {
        const uint32_t a = tc & 1, aph = (tc >> 1) & 1;
        const int tok = t * kPairM + rank * kTileM + row;
        const bool valid = tok < w.len;
        // frequency-major table: lanes read consecutive positions (coalesced)
        const float2* rp = p.rope + (valid ? tok : 0);
        mbar_wait(&tfull[a], aph);
        tc_fence_after();
        float sc[GROUP];
#pragma unroll
        for (int gi = 0; gi < GROUP; ++gi) sc[gi] = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float kb[32];
          tmem_ld32(tmem + tlane + a * 256 + c * 32, kb);
          float2 csv[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) csv[i] = __ldg(rp + (int64_t)(c * 16 + i) * p.rope_n);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {  // RoPE in place (linalg.py:92-93)
            const float2 cs = csv[i];
            const float k0 = kb[2 * i], k1 = kb[2 * i + 1];
            kb[2 * i] = k0 * cs.x - k1 * cs.y;
            kb[2 * i + 1] = k0 * cs.y + k1 * cs.x;
          }
#pragma unroll
          for (int gi = 0; gi < GROUP; ++gi) {  // q (broadcast) as 128-bit shared loads
            const float4* qq = reinterpret_cast<const float4*>(q_s + gi * kHeadDim + c * 32);
#pragma unroll
            for (int v4 = 0; v4 < 8; ++v4) {
              const float4 q4 = qq[v4];
              sc[gi] = fmaf(q4.x, kb[4 * v4], sc[gi]);
              sc[gi] = fmaf(q4.y, kb[4 * v4 + 1], sc[gi]);
              sc[gi] = fmaf(q4.z, kb[4 * v4 + 2], sc[gi]);
              sc[gi] = fmaf(q4.w, kb[4 * v4 + 3], sc[gi]);
            }
          }
        }
        if (p.dbg_acc != nullptr && 2 * t + (int)rank < p.dbg_tiles) {
          float* drow = p.dbg_acc +
              ((((int64_t)w.b * p.n_kv + w.h) * p.dbg_tiles + 2 * t + rank) * kTileM + row) * 256;
          for (int c = 0; c < 8; ++c) {
            float tmpv[32];
            tmem_ld32(tmem + tlane + a * 256 + c * 32, tmpv);
            tmem_wait_ld();
            for (int j = 0; j < 32; ++j) drow[c * 32 + j] = tmpv[j];
          }
        }
        float pr[GROUP];
#pragma unroll
        for (int gi = 0; gi < GROUP; ++gi) {
          const float s = valid ? sc[gi] : -INFINITY;
          const float mn = fmaxf(m_run[gi], warp_max(s));
          const float alpha = (m_run[gi] == -INFINITY) ? 0.f : exp2f(m_run[gi] - mn);
          pr[gi] = valid ? exp2f(s - mn) : 0.f;
          l_run[gi] = l_run[gi] * alpha + warp_sum(pr[gi]);
#pragma unroll
          for (int c = 0; c < 4; ++c) o_run[gi][c] *= alpha;
          m_run[gi] = mn;
        }
        // p.V over this warp's 32 rows: transpose each 32x32 block of V through
        // shared memory (row stride 36 floats: 128-bit stores and column reads are
        // both bank-conflict-free), then lane L sums column 32c+L over the rows
        // with the rows' p broadcast from shared memory.
        constexpr int kVS = 36;
        float* vw = epi_v + ew * (32 * kVS);
        float* pw = epi_p + ew * (32 * kPStride<GROUP>);
#pragma unroll
        for (int gi = 0; gi < GROUP; ++gi) pw[lane * kPStride<GROUP> + gi] = pr[gi];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float vb[32];
          tmem_ld32(tmem + tlane + a * 256 + 128 + c * 32, vb);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(vw + lane * kVS + 4 * j) =
                make_float4(vb[4 * j], vb[4 * j + 1], vb[4 * j + 2], vb[4 * j + 3]);
          __syncwarp();
          float acc[GROUP];
#pragma unroll
          for (int gi = 0; gi < GROUP; ++gi) acc[gi] = 0.f;
#pragma unroll 8
          for (int r = 0; r < 32; ++r) {
            const float v = vw[r * kVS + lane];
            float pv[kPStride<GROUP>];
            load_p<GROUP>(pw + r * kPStride<GROUP>, pv);
#pragma unroll
            for (int gi = 0; gi < GROUP; ++gi) acc[gi] = fmaf(pv[gi], v, acc[gi]);
          }
#pragma unroll
          for (int gi = 0; gi < GROUP; ++gi) o_run[gi][c] += acc[gi];
          __syncwarp();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) mbar_arrive(&tempty[a]);
          else mbar_arrive_remote(tempty_leader0 + 8 * a);
        }
      }
#pragma unroll
      for (int gi = 0; gi < GROUP; ++gi) {
        const int hq = w.h * GROUP + gi;
        float* dst = p.partials + ((((int64_t)w.b * n_q + hq) * p.n_chunks + w.chunk) * kPartsPerChunk +
                                   rank * 4 + ew) * kPartStride;
        if (lane == 0) {
          dst[0] = m_run[gi];
          dst[1] = l_run[gi];
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) dst[2 + c * 32 + lane] = o_run[gi][c];
      }
    }
  }
  tc_fence_before();
  cluster_sync();  // the leader's MMAs have finished writing both CTAs' TMEM
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem, 512);
  }
}

// Merge split partials (m in log2 domain): out = sum_i 2^(m_i-M) o_i / sum_i 2^(m_i-M) l_i
__global__ void k_combine(const float* __restrict__ partials, int n_parts, float* __restrict__ out) {
  const int64_t bh = blockIdx.x;
  const int d = threadIdx.x;
  const float* base = partials + bh * n_parts * kPartStride;
  float M = -INFINITY;
  for (int i = 0; i < n_parts; ++i) M = fmaxf(M, base[(int64_t)i * kPartStride]);
  float L = 0.f, O = 0.f;
  if (M != -INFINITY) {
    for (int i = 0; i < n_parts; ++i) {
      const float m = base[(int64_t)i * kPartStride];
      if (m == -INFINITY) continue;
      const float wgt = exp2f(m - M);
      L = fmaf(wgt, base[(int64_t)i * kPartStride + 1], L);
      O = fmaf(wgt, base[(int64_t)i * kPartStride + 2 + d], O);
    }
  }
  out[bh * kHeadDim + d] = L > 0.f ? O / L : 0.f;
}

// ------------------------------------------------------------ debug remat
struct RematParams {
  int ak_mode, av_mode, ak_bits, av_bits, group_size, nflushed, slot;
  const void* ak_src;
  const void* ak_params;
  const float* ak_resid;
  int64_t ak_row_bytes;
  const void* av_src;
  const void* av_params;
  int64_t av_row_bytes;
  int64_t L_max, kdim, n_out;
  const float* w_k;
  const float* w_v;
  const float2* rope;
  float* k_out;
  float* v_out;
};

XQ_DEVINL uint32_t read_code_dbg(const uint8_t* row, int64_t c, int bits) {
  const int64_t off = c * bits;
  const int64_t byte = off >> 3;
  const int sh = off & 7;
  uint32_t v = row[byte];
  if (sh + bits > 8) v |= static_cast<uint32_t>(row[byte + 1]) << 8;
  return (v >> sh) & ((1u << bits) - 1);
}

XQ_DEVINL float deq_natural(int mode, int bits, const void* src, const void* params,
                            const float* resid, int64_t row_bytes, int G, int64_t kdim,
                            int64_t L_max, int slot, int t, int nflushed, int64_t c) {
  const int64_t arow = (int64_t)slot * L_max + t;
  if (mode == XQ_A_F16_ROWS)
    return __half2float(static_cast<const __half*>(src)[arow * kdim + c]);
  if (mode == XQ_A_CODES_TOKEN) {
    const uint32_t code = read_code_dbg(static_cast<const uint8_t*>(src) + arow * row_bytes, c, bits);
    const __half2 sz = static_cast<const __half2*>(params)[arow * param_stride(kdim, G) + c / G];
    return fmaf(static_cast<float>(code), __low2float(sz), __high2float(sz));
  }
  if (t >= nflushed) return resid[((int64_t)slot * G + (t - nflushed)) * kdim + c];
  const uint32_t code = read_code_dbg(static_cast<const uint8_t*>(src) + arow * row_bytes, c, bits);
  const int bs = perm_block(XQ_A_CODES_CHANNEL, bits);
  const int64_t pos = (c / bs) * bs + perm_position(static_cast<int>(c % bs), bs);
  const __half* prow = static_cast<const __half*>(params) + (arow / G) * 2 * kdim;
  return fmaf(static_cast<float>(code), __half2float(prow[pos]), __half2float(prow[kdim + pos]));
}

__global__ void k_remat_f32(const RematParams p) {
  extern __shared__ float sh[];
  float* xk = sh;
  float* xv = sh + p.kdim;
  float* kp = sh + 2 * p.kdim;
  const int t = blockIdx.x;
  const bool same = p.av_mode == XQ_A_SAME;
  for (int64_t c = threadIdx.x; c < p.kdim; c += blockDim.x) {
    xk[c] = deq_natural(p.ak_mode, p.ak_bits, p.ak_src, p.ak_params, p.ak_resid, p.ak_row_bytes,
                        p.group_size, p.kdim, p.L_max, p.slot, t, p.nflushed, c);
    xv[c] = same ? xk[c]
                 : deq_natural(p.av_mode, p.av_bits, p.av_src, p.av_params, nullptr,
                               p.av_row_bytes, p.group_size, p.kdim, p.L_max, p.slot, t, 1 << 30, c);
  }
  __syncthreads();
  for (int64_t n = threadIdx.x; n < p.n_out; n += blockDim.x) {
    float ak = 0.f, av = 0.f;
    for (int64_t c = 0; c < p.kdim; ++c) {
      ak = fmaf(xk[c], p.w_k[c * p.n_out + n], ak);
      av = fmaf(xv[c], p.w_v[c * p.n_out + n], av);
    }
    kp[n] = ak;
    p.v_out[(int64_t)t * p.n_out + n] = av;
  }
  __syncthreads();
  for (int64_t n = threadIdx.x; n < p.n_out; n += blockDim.x) {
    const float2 cs = p.rope[(int64_t)t * 64 + (n % kHeadDim) / 2];
    const float e0 = kp[n & ~1ll], e1 = kp[n | 1];
    p.k_out[(int64_t)t * p.n_out + n] = (n & 1) ? (e0 * cs.y + e1 * cs.x) : (e0 * cs.x - e1 * cs.y);
  }
}

// ------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

static int num_sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

static int64_t n_chunks_for(int32_t max_len, int32_t tpc) {
  const int64_t nt = (max_len + kPairM - 1) / kPairM;
  return nt == 0 ? 1 : (nt + tpc - 1) / tpc;
}

struct Maps {
  CUtensorMap w, ca, pa, cb, pb;
};

template <int AK, int AV, int BITS, int GROUP>
static int launch_decode(const Maps& m, const DecodeParams& p, cudaStream_t st) {
  using R = Ring<AK, AV, BITS>;
  constexpr size_t smem = 1024 + R::kABBytes + R::kCodeStages * R::kStageBytes +
                          (2 * R::kABStages + 8 + 4) * 8 + 16 + GROUP * kHeadDim * 4 +
                          R::kEpiScratch;
  static_assert(R::kABStage % 1024 == 0, "stages must keep 1024-byte swizzle alignment");
  static_assert(smem <= 227 * 1024, "shared memory budget");
  auto kern = k_decode_attend<AK, AV, BITS, GROUP>;
  if (int s = ensure_smem(reinterpret_cast<const void*>(kern), smem, "cudaFuncSetAttribute(decode)"))
    return s;
  // one CTA pair per unit in flight; an even grid of at most one CTA per SM
  const int pairs = p.n_units < num_sms() / 2 ? p.n_units : num_sms() / 2;
  kern<<<2 * pairs, kThreads, smem, st>>>(m.w, m.ca, m.pa, m.cb, m.pb, p);
  return check_launch("k_decode_attend");
}

template <int AK, int AV, int GROUP>
static int dispatch_bits(int bits, const Maps& m, const DecodeParams& p, cudaStream_t st) {
  switch (bits) {
    case 2: return launch_decode<AK, AV, 2, GROUP>(m, p, st);
    case 3: return launch_decode<AK, AV, 3, GROUP>(m, p, st);
    case 4: return launch_decode<AK, AV, 4, GROUP>(m, p, st);
    case 8: return launch_decode<AK, AV, 8, GROUP>(m, p, st);
    default: return fail(XQ_ECONFIG, "unsupported bits %d", bits);
  }
}

static int make_map(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base,
                    uint64_t inner, uint64_t rows, uint32_t box_inner, uint32_t box_rows,
                    CUtensorMapSwizzle sw, const char* what,
                    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
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

// codes (uint8 [rows][row_bytes], box = one 128-channel group) + per-token params
static int stream_maps(int mode, int bits, const void* src, const void* params, int64_t row_bytes,
                       int64_t kdim, int G, int64_t rows, CUtensorMap* codes, CUtensorMap* pmap) {
  int st;
  if (mode == XQ_A_F16_ROWS)
    return make_map(codes, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, kdim, rows, kChunk, kTileM,
                    CU_TENSOR_MAP_SWIZZLE_128B, "fp16 A rows");
  XQ_REQUIRE(row_bytes == row_bytes_for(kdim, bits), XQ_ESHAPE, "row_bytes mismatch");
  if ((st = make_map(codes, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, src, row_bytes, rows, 16 * bits,
                     kTileM, CU_TENSOR_MAP_SWIZZLE_NONE, "codes", CU_TENSOR_MAP_L2_PROMOTION_L2_128B)) != XQ_OK)
    return st;
  if (mode == XQ_A_CODES_TOKEN)  // byte view of the half2 grid: one 16-byte quad per row
    return make_map(pmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, params, param_stride(kdim, G) * 4, rows,
                    16, kTileM, CU_TENSOR_MAP_SWIZZLE_NONE, "params", CU_TENSOR_MAP_L2_PROMOTION_NONE);
  // per-channel: planar halves [rows/G][2][kdim] viewed as [2*rows/G][kdim]; box = one
  // 128-channel group of scales and zps (2 x 256 B)
  return make_map(pmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, params, kdim, 2 * (rows / G), 128, 2,
                  CU_TENSOR_MAP_SWIZZLE_NONE, "channel params", CU_TENSOR_MAP_L2_PROMOTION_NONE);
}

}  // namespace xq

using namespace xq;

extern "C" {

int xq_debug_set_acc_dump(float* buf, int32_t n_tiles) {
  g_dbg_acc = buf;
  g_dbg_tiles = n_tiles;
  return XQ_OK;
}

int64_t xq_decode_workspace_bytes(int32_t n_seqs, int32_t max_len, int32_t n_kv_heads,
                                  int32_t group, int32_t tiles_per_chunk) {
  if (tiles_per_chunk < 1) tiles_per_chunk = 1;
  return (int64_t)n_seqs * n_kv_heads * group * n_chunks_for(max_len, tiles_per_chunk) *
         kPartsPerChunk * kPartStride * sizeof(float);
}

int xq_decode_attend(int32_t ak_mode, const void* ak_src, const void* ak_params,
                     const float* ak_resid, const int32_t* ak_nflushed, int32_t ak_bits,
                     int64_t ak_row_bytes, int32_t av_mode, const void* av_src,
                     const void* av_params, int32_t av_bits, int64_t av_row_bytes,
                     int32_t group_size, int64_t L_max, int64_t kdim, const int32_t* seq_lens,
                     int32_t n_seqs, int32_t max_len, const void* w_arranged, int32_t n_kv_heads,
                     int32_t group, const float* q_pre, const void* rope_cs, int64_t rope_n,
                     float sm_scale, int32_t tiles_per_chunk, void* workspace,
                     int64_t workspace_bytes, float* out, void* stream) {
  XQ_REQUIRE(rope_n >= max_len, XQ_ESHAPE, "rope table shorter than max_len");
  XQ_REQUIRE(kdim % (2 * kChunk) == 0 && kdim >= 2 * kChunk, XQ_ESHAPE,
             "kdim must be a positive multiple of 128, got %lld", (long long)kdim);
  XQ_REQUIRE(group_size == kG, XQ_ECONFIG,
             "the fused kernel is specialised for group_size 128 (the reference default), got %d",
             group_size);
  XQ_REQUIRE(tiles_per_chunk >= 1, XQ_ECONFIG, "tiles_per_chunk must be >= 1");
  XQ_REQUIRE(n_seqs >= 1 && n_kv_heads >= 1, XQ_ESHAPE, "empty batch");
  XQ_REQUIRE(max_len <= L_max, XQ_ESHAPE, "max_len > L_max");
  XQ_REQUIRE(workspace_bytes >= xq_decode_workspace_bytes(n_seqs, max_len, n_kv_heads, group,
                                                          tiles_per_chunk),
             XQ_ESHAPE, "workspace too small");
  const bool mha = av_mode == XQ_A_SAME;
  if (!mha) {
    XQ_REQUIRE(ak_mode == XQ_A_CODES_CHANNEL && av_mode == XQ_A_CODES_TOKEN, XQ_ECONFIG,
               "split K/V A operands support (CODES_CHANNEL, CODES_TOKEN) only");
    XQ_REQUIRE(ak_bits == av_bits, XQ_ECONFIG, "K and V latent bits must match");
    XQ_REQUIRE(L_max % group_size == 0 && group_size == kTileM, XQ_ECONFIG,
               "per-channel K latent needs group_size 128 and L_max % 128 == 0");
  } else {
    XQ_REQUIRE(ak_mode == XQ_A_CODES_TOKEN || ak_mode == XQ_A_F16_ROWS, XQ_ECONFIG,
               "shared A operand must be CODES_TOKEN or F16_ROWS");
  }
  XQ_REQUIRE(ak_mode == XQ_A_F16_ROWS || valid_bits(ak_bits), XQ_ECONFIG, "bad bits %d", ak_bits);
  Maps maps;
  int st_;
  if ((st_ = make_map(&maps.w, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, w_arranged, kdim,
                      (uint64_t)n_kv_heads * 256, kChunk, mha ? 128 : 64,
                      CU_TENSOR_MAP_SWIZZLE_128B, "weights")) != XQ_OK)
    return st_;
  const int64_t arena_rows = (int64_t)n_seqs * L_max;
  if ((st_ = stream_maps(ak_mode, ak_bits, ak_src, ak_params, ak_row_bytes, kdim, group_size,
                         arena_rows, &maps.ca, &maps.pa)) != XQ_OK)
    return st_;
  if (!mha) {
    if ((st_ = stream_maps(av_mode, av_bits, av_src, av_params, av_row_bytes, kdim, group_size,
                           arena_rows, &maps.cb, &maps.pb)) != XQ_OK)
      return st_;
  } else {
    maps.cb = maps.ca;
    maps.pb = maps.pa;
  }

  DecodeParams p;
  p.ak_src = static_cast<const uint8_t*>(ak_src);
  p.ak_params = ak_params;
  p.ak_resid = ak_resid;
  p.ak_nflushed = ak_nflushed;
  p.ak_row_bytes = ak_row_bytes;
  p.av_src = static_cast<const uint8_t*>(mha ? ak_src : av_src);
  p.av_params = mha ? ak_params : av_params;
  p.av_row_bytes = mha ? ak_row_bytes : av_row_bytes;
  p.group_size = group_size;
  p.L_max = L_max;
  p.kdim = static_cast<int32_t>(kdim);
  p.seq_lens = seq_lens;
  p.tiles_per_chunk = tiles_per_chunk;
  p.n_chunks = static_cast<int32_t>(n_chunks_for(max_len, tiles_per_chunk));
  p.n_kv = n_kv_heads;
  p.n_units = n_seqs * p.n_chunks * n_kv_heads;
  p.n_seqs = n_seqs;
  {
    // largest divisor of n_kv whose arranged W block (256 rows x kdim fp16 per head)
    // stays <= 32 MB: the W slice of the pairs in flight then stays L2-resident
    // on both dies (measured: 6.5 -> 1.4 GB of DRAM per C2 layer launch)
    int hb = n_kv_heads;
    while (hb > 1 && ((int64_t)hb * 512 * kdim > (32ll << 20) || n_kv_heads % hb)) --hb;
    p.head_block = hb;
  }
  p.q_pre = q_pre;
  p.rope = static_cast<const float2*>(rope_cs);
  p.rope_n = rope_n;
  p.q_scale = sm_scale * 1.4426950408889634f;
  p.partials = static_cast<float*>(workspace);
  p.dbg_acc = g_dbg_acc;
  p.dbg_tiles = g_dbg_tiles;
  p.w_hint = kEvictLast;  // the W slice of the pairs in flight stays L2-resident
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  int status;
  if (mha) {
    XQ_REQUIRE(group == 1, XQ_ECONFIG, "MHA (shared A) needs group 1, got %d", group);
    if (ak_mode == XQ_A_F16_ROWS)
      status = launch_decode<XQ_A_F16_ROWS, XQ_A_SAME, 4, 1>(maps, p, st);
    else
      status = dispatch_bits<XQ_A_CODES_TOKEN, XQ_A_SAME, 1>(ak_bits, maps, p, st);
  } else {
    switch (group) {
      case 1: status = dispatch_bits<XQ_A_CODES_CHANNEL, XQ_A_CODES_TOKEN, 1>(ak_bits, maps, p, st); break;
      case 2: status = dispatch_bits<XQ_A_CODES_CHANNEL, XQ_A_CODES_TOKEN, 2>(ak_bits, maps, p, st); break;
      case 4: status = dispatch_bits<XQ_A_CODES_CHANNEL, XQ_A_CODES_TOKEN, 4>(ak_bits, maps, p, st); break;
      default: return fail(XQ_ECONFIG, "unsupported GQA group %d (1, 2, 4)", group);
    }
  }
  if (status != XQ_OK) return status;
  const int n_parts = p.n_chunks * kPartsPerChunk;
  k_combine<<<static_cast<unsigned>(n_seqs) * n_kv_heads * group, kHeadDim, 0, st>>>(
      p.partials, n_parts, out);
  return check_launch("k_combine");
}

int xq_remat_f32(int32_t ak_mode, const void* ak_src, const void* ak_params,
                 const float* ak_resid, int32_t ak_nflushed, int32_t ak_bits,
                 int64_t ak_row_bytes, int32_t av_mode, const void* av_src, const void* av_params,
                 int32_t av_bits, int64_t av_row_bytes, int32_t group_size, int64_t L_max,
                 int64_t kdim, int32_t slot, int32_t n_tok, const float* w_k, const float* w_v,
                 int64_t n_out, const void* rope_cs, float* k_out, float* v_out, void* stream) {
  XQ_REQUIRE(n_out % kHeadDim == 0, XQ_ESHAPE, "n_out must be a multiple of 128");
  XQ_REQUIRE(2 * kdim + n_out <= 48 * 1024, XQ_ESHAPE, "debug remat: shapes too large");
  if (n_tok == 0) return XQ_OK;
  RematParams p;
  p.ak_mode = ak_mode; p.av_mode = av_mode; p.ak_bits = ak_bits; p.av_bits = av_bits;
  p.group_size = group_size; p.nflushed = ak_nflushed; p.slot = slot;
  p.ak_src = ak_src; p.ak_params = ak_params; p.ak_resid = ak_resid; p.ak_row_bytes = ak_row_bytes;
  p.av_src = av_src; p.av_params = av_params; p.av_row_bytes = av_row_bytes;
  p.L_max = L_max; p.kdim = kdim; p.n_out = n_out; p.w_k = w_k; p.w_v = w_v;
  p.rope = static_cast<const float2*>(rope_cs); p.k_out = k_out; p.v_out = v_out;
  const size_t smem = (2 * kdim + n_out) * sizeof(float);
  if (int s = ensure_smem(reinterpret_cast<const void*>(k_remat_f32), smem,
                         "cudaFuncSetAttribute(remat_f32)"))
    return s;
  k_remat_f32<<<n_tok, 256, smem, static_cast<cudaStream_t>(stream)>>>(p);
  return check_launch("k_remat_f32");
}

}  // extern "C"
