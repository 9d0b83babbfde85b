// Rematerialization GEMM on tcgen05 for the bulk paths (prefill K/V and the
// XQuant-CL latent accumulator update), where many query rows make the work
// a plain dense GEMM:
//
//   C[M x N] (+)= A[M x K] . B[N x K]^T      fp16 operands, fp32 accumulation
//
// A: dequantized cache rows (tokens x channels), B: a projection stored
// K-major (W^T rows), both staged by TMA in 128-byte-swizzled K-major tiles.
// Epilogues (fused, straight from TMEM):
//   STORE      C = fp16(acc)
//   STORE_ROPE C = fp16(RoPE(acc)) with row i at position pos0 + i (K of a
//              prefill; linalg.py:58-95, pairs (2j, 2j+1) of every 128-wide head)
//   ADD        C = fp16(C + acc) (the accumulator update acc += rec @ U^T,
//              cache.py:588-589)
//
// Persistent CTAs, one 128 x 256 tile at a time; TMEM holds two 256-column
// accumulators so the epilogue of one tile overlaps the MMAs of the next.
// Warp 0: TMA; warp 1: TMEM allocation + the single-thread MMA issuer;
// warps 4-7: epilogue (TMEM lanes 0-127).

#include "xq_common.cuh"
#include "xq_host.h"
#include "xq_tma_host.h"

namespace xq {
namespace {

constexpr int kGemmThreads = 256;
constexpr int kGM = 128, kGN = 256, kGK = 64;  // per CTA: 128 rows of A, 128 of the pair's 256 B rows
constexpr int kGPairM = 2 * kGM;               // a CTA pair computes 256 x 256
constexpr int kGStages = 4;
constexpr uint32_t kGABytes = kGM * 128;       // [128 rows][64 K] fp16
constexpr uint32_t kGBBytes = (kGN / 2) * 128;  // this CTA's half of the pair's B tile
constexpr uint32_t kGStage = kGABytes + kGBBytes;

struct GemmParams {
  int64_t M, N, K;
  int32_t m_tiles, n_tiles;
  __half* C;
  int64_t ldc;
  int32_t epi;
  const float2* rope;  // [n_pos][64] (cos, sin), row-major (rope_table)
  int64_t pos0;
};

// One 256 x 256 output tile per CTA pair (cta_group::2): each CTA stages its 128 rows
// of A and its half of B's 256 rows, the leader issues M=256 N=256 MMAs, and each
// CTA's epilogue drains its 128 rows. Per CTA and 64-deep stage the pair moves 32 KB
// of operands from L2 for 1024 MMA cycles (the 1-SM 128 x 256 form needed 48 KB per
// 512): half the L2 traffic per FLOP, which was the limit of the 1-SM kernel.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    k_gemm_f16(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
               GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kGStages * kGStage);
  uint64_t* empty = full + kGStages;
  uint64_t* tfull = empty + kGStages;   // [2] accumulator ready (both CTAs, multicast commit)
  uint64_t* tempty = tfull + 2;         // [2] accumulator drained (leader's: 4 warps x 2 CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int n_tiles_total = p.m_tiles * p.n_tiles;
  const int nkc = static_cast<int>(p.K / kGK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&full[s], 2);  // the two CTAs' TMA warps (bytes of both land here)
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_mbar_init();
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

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&amap);
      tma_prefetch_desc(&bmap);
      uint32_t it = 0;
      for (int tile = cluster; tile < n_tiles_total; tile += n_clusters) {
        const int mt = tile / p.n_tiles, nt = tile % p.n_tiles;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const uint32_t s = it % kGStages, ph = (it / kGStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * kGStage;
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * kGStage);
          else mbar_arrive_remote(full_leader0 + 8 * s);
          tma_load_2d_pair(st, &amap, &full[s], kc * kGK, mt * kGPairM + static_cast<int>(rank) * kGM,
                           kEvictNormal);
          tma_load_2d_pair(st + kGABytes, &bmap, &full[s], kc * kGK,
                           nt * kGN + static_cast<int>(rank) * (kGN / 2), kEvictLast);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t kIdesc = idesc_f16_f32(kGPairM, kGN);
      const uint64_t a0 = sdesc_sw128(smem_u32(smem));
      const uint64_t b0 = sdesc_sw128(smem_u32(smem + kGABytes));
      uint32_t it = 0, tc = 0;
      for (int tile = cluster; tile < n_tiles_total; tile += n_clusters, ++tc) {
        const uint32_t a = tc & 1, aph = (tc >> 1) & 1;
        mbar_wait_cluster(&tempty[a], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + a * kGN;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const uint32_t s = it % kGStages, ph = (it / kGStages) & 1;
          mbar_wait_cluster(&full[s], ph);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ad = a0 + ((s * kGStage) >> 4), bd = b0 + ((s * kGStage) >> 4);
#pragma unroll
            for (int k = 0; k < kGK / 16; ++k)
              mma2_f16_ss(d, ad + 2 * k, bd + 2 * k, kIdesc, (kc | k) != 0);
            mma2_commit_both(&empty[s]);
          }
          __syncwarp();
        }
        if (elect_one()) mma2_commit_both(&tfull[a]);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int row_in = ew * 32 + lane;
    const uint32_t tlane = static_cast<uint32_t>(ew * 32) << 16;
    uint32_t tc = 0;
    for (int tile = cluster; tile < n_tiles_total; tile += n_clusters, ++tc) {
      const int mt = tile / p.n_tiles, nt = tile % p.n_tiles;
      const uint32_t a = tc & 1, aph = (tc >> 1) & 1;
      const int64_t row = static_cast<int64_t>(mt) * kGPairM + static_cast<int64_t>(rank) * kGM + row_in;
      const bool row_ok = row < p.M;
      __half* crow = p.C + row * p.ldc;
      const bool add = p.epi == 2;
      // the add epilogue's old C rows do not depend on the MMA: the first 32 columns are
      // loaded before the accumulator is ready, each next chunk before the current one's math
      uint4 oldc[4];
      auto load_old = [&](int g) {
        const int64_t n0 = static_cast<int64_t>(nt) * kGN + g * 32;
        if (add && row_ok && n0 + 32 <= p.N) {
          const uint4* src = reinterpret_cast<const uint4*>(crow + n0);
#pragma unroll
          for (int q = 0; q < 4; ++q) oldc[q] = src[q];
        }
      };
      load_old(0);
      mbar_wait(&tfull[a], aph);
      tc_fence_after();
      const float2* rope = p.rope ? p.rope + (p.pos0 + row) * 64 : nullptr;
#pragma unroll 1
      for (int g = 0; g < kGN / 32; ++g) {
        float v[32];
        tmem_ld32(tmem + tlane + a * kGN + g * 32, v);
        uint4 cur[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) cur[q] = oldc[q];
        if (g + 1 < kGN / 32) load_old(g + 1);
        tmem_wait_ld();
        const int64_t n0 = static_cast<int64_t>(nt) * kGN + g * 32;
        if (row_ok && n0 < p.N) {
        if (p.epi == 1) {  // RoPE of pairs (2j, 2j+1), j = (n % 128) / 2
          const int j0 = static_cast<int>((n0 % 128) / 2);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 cs = rope[j0 + i];
            const float e = v[2 * i], o = v[2 * i + 1];
            v[2 * i] = e * cs.x - o * cs.y;
            v[2 * i + 1] = e * cs.y + o * cs.x;
          }
        }
        const int ncols = p.N - n0 < 32 ? static_cast<int>(p.N - n0) : 32;
        if (ncols == 32) {
          uint4* dst = reinterpret_cast<uint4*>(crow + n0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float f[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = v[8 * q + i];
            if (add) {
              const __half2* h = reinterpret_cast<const __half2*>(&cur[q]);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 o = __half22float2(h[i]);
                f[2 * i] += o.x;
                f[2 * i + 1] += o.y;
              }
            }
            uint4 out;
            __half2* oh = reinterpret_cast<__half2*>(&out);
#pragma unroll
            for (int i = 0; i < 4; ++i) oh[i] = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
            dst[q] = out;
          }
        } else {
          for (int i = 0; i < ncols; ++i) {
            float f = v[i];
            if (add) f += __half2float(crow[n0 + i]);
            crow[n0 + i] = __float2half_rn(f);
          }
        }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&tempty[a]);
        else mbar_arrive_remote(tempty_leader0 + 8 * a);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem, 512);
  }
}

int num_sms_dev() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace
}  // namespace xq

using namespace xq;

extern "C" int xq_gemm_f16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                           int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t epilogue,
                           const void* rope_cs, int64_t rope_n, int64_t pos0, void* stream) {
  XQ_REQUIRE(epilogue >= 0 && epilogue <= 2, XQ_ECONFIG, "epilogue must be 0 (store), 1 (store "
             "with RoPE) or 2 (add), got %d", epilogue);
  XQ_REQUIRE(K > 0 && K % kGK == 0, XQ_ESHAPE, "K %lld must be a positive multiple of %d",
             (long long)K, kGK);
  XQ_REQUIRE(M >= 0 && N > 0 && ldc >= N && lda >= K && ldb >= K, XQ_ESHAPE, "bad GEMM shape");
  XQ_REQUIRE(ldc % 8 == 0 && reinterpret_cast<uintptr_t>(C) % 16 == 0, XQ_ESHAPE,
             "C rows must be 16-byte aligned");
  XQ_REQUIRE(epilogue != 1 || (rope_cs != nullptr && pos0 + M <= rope_n && N % 128 == 0),
             XQ_ESHAPE, "RoPE epilogue needs a table covering pos0+M rows and N %% 128 == 0");
  if (M == 0) return XQ_OK;
  CUtensorMap amap, bmap;
  int st;
  if ((st = tma_map_2d(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, A, (uint64_t)K, (uint64_t)M,
                       (uint64_t)lda * 2, kGK, kGM, CU_TENSOR_MAP_SWIZZLE_128B, "A")) != XQ_OK)
    return st;
  if ((st = tma_map_2d(&bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, B, (uint64_t)K, (uint64_t)N,
                       (uint64_t)ldb * 2, kGK, kGN / 2, CU_TENSOR_MAP_SWIZZLE_128B, "B")) != XQ_OK)
    return st;
  GemmParams p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.m_tiles = static_cast<int32_t>((M + kGPairM - 1) / kGPairM);
  p.n_tiles = static_cast<int32_t>((N + kGN - 1) / kGN);
  p.C = static_cast<__half*>(C);
  p.ldc = ldc;
  p.epi = epilogue;
  p.rope = epilogue == 1 ? static_cast<const float2*>(rope_cs) : nullptr;
  p.pos0 = pos0;
  const size_t smem = 1024 + kGStages * kGStage + (2 * kGStages + 4) * 8 + 16;
  if ((st = ensure_smem(reinterpret_cast<const void*>(k_gemm_f16), smem,
                        "cudaFuncSetAttribute(gemm_f16)")) != XQ_OK)
    return st;
  const int tiles = p.m_tiles * p.n_tiles;
  const int pairs = tiles < num_sms_dev() / 2 ? tiles : num_sms_dev() / 2;
  k_gemm_f16<<<2 * pairs, kGemmThreads, smem, static_cast<cudaStream_t>(stream)>>>(amap, bmap, p);
  return check_launch("k_gemm_f16");
}
