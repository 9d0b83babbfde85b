// xq-gqa decode append on tcgen05: the SVD-latent projection of the new
// tokens, x @ [U_k | U_v] (cache.py:429-432), with the V latent quantized and
// packed into its per-token arena and the K latent staged in the per-channel
// residual buffer (cache.py:210-221), in one launch.
//
// The product is transposed so the long side sits on the tensor cores' M:
//   lat^T [2r x B] = U^T [2r x d] . x^T [d x B]
// A = U^T is MN-major in shared memory: U is row-major [d][2r], so a TMA box
// of [64 rows of d][64 columns] with 128-byte swizzle is exactly the canonical
// MN-major SW128 layout (one K row = 64 contiguous M elements). B = x^T is
// K-major: x rows [B][d] in 64-wide SW128 boxes. One CTA owns one 128-column
// block of U (one quantization group) for one d-slice; the 8 CTAs of a
// cluster split d and reduce the [128 x 32] partials through distributed
// shared memory, after which CTA q finishes rows 4q..4q+3: K columns go to the
// residual buffer, V columns are quantized per token (fp64 scale / code math,
// bit-identical to quant.quantize for the same float32 latent) and packed.
//
// HBM roofline: the kernel streams U once (d * 2r * 2 bytes) and is bound by
// it; the MMAs (M=128, N=32, K=16) take a few hundred cycles per CTA.

#include "xq_common.cuh"
#include "xq_host.h"
#include "xq_tma_host.h"

namespace xq {
namespace {

constexpr int kLatThreads = 128;   // 4 warps: the 128 TMEM lanes of the M=128 accumulator
constexpr int kLatCluster = 8;     // d-slices per column block
constexpr int kLatRows = 32;       // N: tokens per launch row-chunk
constexpr int kLatChunk = 64;      // d rows per pipeline stage
constexpr int kLatStages = 4;
constexpr uint32_t kUStage = 2 * 64 * 128;      // two 64-column halves of [64 d][64] bf16 = 16 KB
constexpr uint32_t kXStage = kLatRows * 128;    // [32 rows][64 d] bf16 = 4 KB
constexpr uint32_t kStage = kUStage + kXStage;

struct LatParams {
  int32_t n_rows;        // tokens (slots) in this launch
  int64_t d;             // hidden width (K of the GEMM)
  int32_t r;             // latent rank of each of K and V (U has 2r columns)
  int32_t bits;
  int64_t slice;         // d rows per cluster rank (multiple of 64)
  const int32_t* lens;   // [n_rows] tokens incl. the new one
  const int32_t* nflushed;
  int64_t L_max;
  float* k_resid;        // [n_rows][128][r] per-channel residual rows
  uint8_t* v_codes;      // per-token arena [n_rows * L_max][row_bytes]
  int64_t v_row_bytes;
  __half2* v_params;     // [n_rows * L_max][ngp]
  int64_t v_param_stride;
  float* lat_out;        // optional [n_rows][2r] float32
  int32_t* flag;         // non-finite input
};

__host__ __device__ constexpr uint32_t idesc_bf16_f32_amn(int M, int N) {
  return idesc_f16_f32_amn(M, N) | (1u << 7) | (1u << 10);  // A, B = BF16
}

XQ_DEVINL uint32_t stream_word32_s(const uint8_t* codes, int n, int bits, int w) {
  const int b0 = w * 32;
  const int i0 = b0 / bits;
  int i1 = (b0 + 31) / bits;
  if (i1 > n - 1) i1 = n - 1;
  uint32_t word = 0;
  for (int i = i0; i <= i1; ++i) {
    const int off = i * bits - b0;
    const uint32_t c = codes[i];
    word |= off >= 0 ? (c << off) : (c >> (-off));
  }
  return word;
}

__global__ void __cluster_dims__(1, kLatCluster, 1) __launch_bounds__(kLatThreads, 1)
    k_latent_project(const __grid_constant__ CUtensorMap umap,
                     const __grid_constant__ CUtensorMap xmap, LatParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sStages = smem;
  float* sRed = reinterpret_cast<float*>(smem + kLatStages * kStage);        // [32][128]
  float* sFin = sRed + kLatRows * 128;                                       // [4][128]
  uint8_t* sCodes = reinterpret_cast<uint8_t*>(sFin + 4 * 128);              // [4][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(sCodes + 4 * 128);
  uint64_t* empty = full + kLatStages;
  uint64_t* done = empty + kLatStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int colblk = blockIdx.x;
  const int b0 = blockIdx.z * kLatRows;
  const int64_t k_begin = static_cast<int64_t>(rank) * p.slice;
  const int64_t k_end = min(p.d, k_begin + p.slice);
  const int nchunks = k_begin < k_end ? static_cast<int>((k_end - k_begin + kLatChunk - 1) / kLatChunk) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kLatStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, 32);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------------------------------------------------- TMA producer
    tma_prefetch_desc(&umap);
    tma_prefetch_desc(&xmap);
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % kLatStages;
      if (c >= kLatStages) mbar_wait(&empty[s], ((c / kLatStages) - 1) & 1);
      uint8_t* st = sStages + s * kStage;
      const int32_t k0 = static_cast<int32_t>(k_begin + static_cast<int64_t>(c) * kLatChunk);
      mbar_arrive_expect_tx(&full[s], kStage);
      tma_load_2d(st, &umap, &full[s], colblk * 128, k0, kEvictFirst);
      tma_load_2d(st + kUStage / 2, &umap, &full[s], colblk * 128 + 64, k0, kEvictFirst);
      tma_load_2d(st + kUStage, &xmap, &full[s], k0, b0, kEvictLast);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------------------------------------------------- MMA issuer
    constexpr uint32_t kIdesc = idesc_bf16_f32_amn(128, kLatRows);
    const uint64_t a0 = sdesc_mn_sw128(smem_u32(sStages), kUStage / 2, 1024);
    const uint64_t x0 = sdesc_sw128(smem_u32(sStages + kUStage));
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % kLatStages;
      mbar_wait(&full[s], (c / kLatStages) & 1);
      tc_fence_after();
      const uint64_t ad = a0 + ((s * kStage) >> 4);
      const uint64_t bd = x0 + ((s * kStage) >> 4);
      // a chunk of k rows past the slice end contributes zero (its rows are the
      // next rank's; the final chunk of the tensor is zero-filled by TMA): mask
      // them by issuing only the in-range 16-row steps
      const int64_t left = k_end - (k_begin + static_cast<int64_t>(c) * kLatChunk);
      const int64_t rows = left < kLatChunk ? left : kLatChunk;
#pragma unroll
      for (int k = 0; k < kLatChunk / 16; ++k)
        if (k * 16 < rows)
          mma_f16_ss(tmem, ad + k * (2048 >> 4), bd + 2 * k, kIdesc, (c | k) != 0);
      mma_commit(&empty[s]);
    }
    if (nchunks > 0) mma_commit(done);
  }
  __syncwarp();

  // ---------------------------------------------------------- partial -> shared
  // thread t = TMEM lane t = U column colblk*128 + t; 32 columns = the 32 tokens
  {
    float v[32];
    if (nchunks > 0) {
      mbar_wait(done, 0);
      tc_fence_after();
      tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) sRed[j * 128 + threadIdx.x] = v[j];
  }
  tc_fence_before();
  cluster_sync();  // every rank's partial is in its shared memory

  // ---------------------------------------------------------- DSMEM reduction
  // rank q sums rows 4q..4q+3 over the 8 d-slices
  const int c = threadIdx.x;
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const uint32_t local = smem_u32(&sRed[(rank * 4 + rr) * 128 + c]);
    float sum = 0.f;
#pragma unroll
    for (int q = 0; q < kLatCluster; ++q) {
      float v;
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(mapa_shared(local, q)) : "memory");
      sum += v;
    }
    sFin[rr * 128 + c] = sum;
  }
  cluster_sync();  // remote reads done (peers may exit); sFin visible CTA-wide
  if (warp == 0) tmem_dealloc(tmem, 32);

  // ---------------------------------------------------------- epilogue
  const int n_k_blocks = p.r / 128;
  const bool is_k = colblk < n_k_blocks;
  for (int rr = 0; rr < 4; ++rr) {
    const int b = b0 + static_cast<int>(rank) * 4 + rr;
    if (b >= p.n_rows) break;
    const float val = sFin[rr * 128 + c];
    if (p.lat_out) p.lat_out[static_cast<int64_t>(b) * 2 * p.r + colblk * 128 + c] = val;
    if (!isfinite(val)) atomicExch(p.flag, 1);
    if (is_k) {
      const int64_t pos = p.lens[b] - 1 - p.nflushed[b];
      p.k_resid[(static_cast<int64_t>(b) * 128 + pos) * p.r + colblk * 128 + c] = val;
    }
  }
  if (is_k) return;
  // V latent: warp rr quantizes row rr's group (128 columns) -- quantize_row's math
  const int rr = warp;
  const int b = b0 + static_cast<int>(rank) * 4 + rr;
  if (b >= p.n_rows) return;
  const int g = colblk - n_k_blocks;
  const double qmax = static_cast<double>((1 << p.bits) - 1);
  double mn = INFINITY, mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double v = static_cast<double>(sFin[rr * 128 + lane + 32 * j]);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const double span = __dsub_rn(mx, mn);
  const double scale = (span == 0.0) ? 1.0 : __ddiv_rn(span, qmax);
  uint8_t* codes = sCodes + rr * 128;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int cc = lane + 32 * j;
    const double v = static_cast<double>(sFin[rr * 128 + cc]);
    double q = floor(__dadd_rn(__ddiv_rn(__dsub_rn(v, mn), scale), 0.5));
    q = q < 0.0 ? 0.0 : (q > qmax ? qmax : q);
    codes[cc] = static_cast<uint8_t>(q);
  }
  __syncwarp();
  const int64_t dst = static_cast<int64_t>(b) * p.L_max + (p.lens[b] - 1);
  if (lane < 4 * p.bits) {  // the group is 128*bits bits = 4*bits words of the row
    uint32_t* out = reinterpret_cast<uint32_t*>(p.v_codes + dst * p.v_row_bytes);
    out[g * 4 * p.bits + lane] = stream_word32_s(codes, 128, p.bits, lane);
  }
  if (lane == 0)
    p.v_params[dst * p.v_param_stride + g] = __halves2half2(__double2half(scale), __double2half(mn));
}

}  // namespace
}  // namespace xq

using namespace xq;

extern "C" int xq_latent_project_append(const void* x_bf16, int64_t x_row_stride, int32_t n_rows,
                                        int64_t d, const void* u_bf16, int32_t r, int32_t bits,
                                        int32_t group_size, const int32_t* seq_lens,
                                        const int32_t* k_nflushed, int64_t L_max, float* k_resid,
                                        uint8_t* v_codes, int64_t v_row_bytes, void* v_params,
                                        float* lat_out, int32_t* nonfinite_flag, void* stream) {
  XQ_REQUIRE(valid_bits(bits), XQ_ECONFIG, "bits must be one of (2, 3, 4, 8), got %d", bits);
  XQ_REQUIRE(group_size == 128, XQ_ECONFIG, "the latent kernel is specialised for group_size 128");
  XQ_REQUIRE(r > 0 && r % 128 == 0, XQ_ESHAPE, "latent rank %d must be a multiple of 128", r);
  XQ_REQUIRE(d > 0 && d % 64 == 0, XQ_ESHAPE, "hidden width %lld must be a multiple of 64", (long long)d);
  XQ_REQUIRE(x_row_stride >= d, XQ_ESHAPE, "x row stride < d");
  XQ_REQUIRE(v_row_bytes == row_bytes_for(r, bits), XQ_ESHAPE, "v_row_bytes mismatch");
  XQ_REQUIRE(seq_lens && k_nflushed && k_resid && v_codes && v_params && nonfinite_flag, XQ_EUSAGE,
             "null pointer argument");
  if (n_rows == 0) return XQ_OK;
  CUtensorMap umap, xmap;
  int st;
  if ((st = tma_map_2d(&umap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, u_bf16, 2 * (uint64_t)r,
                       (uint64_t)d, 2 * (uint64_t)r * 2, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B,
                       "U")) != XQ_OK)
    return st;
  if ((st = tma_map_2d(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x_bf16, (uint64_t)d,
                       (uint64_t)n_rows, (uint64_t)x_row_stride * 2, 64, kLatRows,
                       CU_TENSOR_MAP_SWIZZLE_128B, "x")) != XQ_OK)
    return st;
  LatParams p;
  p.n_rows = n_rows;
  p.d = d;
  p.r = r;
  p.bits = bits;
  p.slice = ((d + kLatCluster - 1) / kLatCluster + kLatChunk - 1) / kLatChunk * kLatChunk;
  p.lens = seq_lens;
  p.nflushed = k_nflushed;
  p.L_max = L_max;
  p.k_resid = k_resid;
  p.v_codes = v_codes;
  p.v_row_bytes = v_row_bytes;
  p.v_params = static_cast<__half2*>(v_params);
  p.v_param_stride = (r / 128 + 3) / 4 * 4;  // half2 per row, padded to 16-byte quads
  p.lat_out = lat_out;
  p.flag = nonfinite_flag;
  const size_t smem = 1024 + kLatStages * kStage + (kLatRows * 128 + 4 * 128) * 4 + 4 * 128 +
                      (2 * kLatStages + 1) * 8 + 16;
  if ((st = ensure_smem(reinterpret_cast<const void*>(k_latent_project), smem,
                        "cudaFuncSetAttribute(latent_project)")) != XQ_OK)
    return st;
  dim3 grid(2 * r / 128, kLatCluster, (n_rows + kLatRows - 1) / kLatRows);
  k_latent_project<<<grid, kLatThreads, smem, static_cast<cudaStream_t>(stream)>>>(umap, xmap, p);
  return check_launch("k_latent_project");
}
