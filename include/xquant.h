/*
 * xquant.h -- C ABI of the B200 (sm_100a) XQuant decode hot path.
 *
 * Drop-in boundary for the reference package `xcache` (arxiv 2508.10395,
 * /root/reference/pkg/src/xcache). Every entry point takes plain device
 * pointers, sizes and a cudaStream_t (as void*), performs no allocation and no
 * host synchronisation, enqueues its work on `stream`, and returns a status
 * code (XQ_OK or one of XQ_E*). The Python host layer maps the codes onto the
 * reference's exception classes (errors.py:4-35): 1 -> ShapeError,
 * 2 -> ConfigError, 3 -> UsageError, 4 -> DataError.
 *
 * Data layout in HBM (per layer, per payload stream):
 *   codes  : uint8 [n_slots * L_max * row_bytes]; arena row (slot*L_max + t)
 *            holds token t of sequence `slot` as the exact bytes of the
 *            reference's pack_codes(row, bits) (fallback.py:58-79):
 *            LSB-first little-endian bit stream, row_bytes =
 *            ceil(cols*bits/64)*8.
 *   params : fp16 scale + fp16 zero_point per group -- the 16+16 bits per
 *            group the reference charges (quant.py:44-45, quant.py:58-62).
 *            per-token  : __half2 (scale, zp) [n_slots * L_max][P], row stride
 *                         P = ceil(ceil(cols/G)/4)*4 (padded to whole 16-byte
 *                         quads so the fused kernel can stage it by TMA)
 *            per-channel: planar halves [n_slots * L_max / G][2][cols]
 *                         (scales, then zero points; L_max % G == 0), the
 *                         channels within each block stored in the order the
 *                         fused kernel's dequant producer consumes them
 *                         (paper_2508_10395_b200/csrc/xq_layout.cuh).
 */
#ifndef XQUANT_H_
#define XQUANT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define XQ_OK 0
#define XQ_ESHAPE 1     /* ShapeError  */
#define XQ_ECONFIG 2    /* ConfigError */
#define XQ_EUSAGE 3     /* UsageError  */
#define XQ_ENONFINITE 4 /* DataError   */
#define XQ_ECUDA 5      /* CUDA runtime error (launch / configuration) */

/* element types of caller buffers */
#define XQ_F32 0
#define XQ_BF16 1
#define XQ_F16 2
#define XQ_F64 3

/* A-operand sources of the fused decode kernel */
#define XQ_A_CODES_TOKEN 0   /* per-token packed codes + half2 params            */
#define XQ_A_CODES_CHANNEL 1 /* per-channel packed codes + residual fp32 rows    */
#define XQ_A_F16_ROWS 2      /* plain fp16 rows (XQuant-CL accumulator, 16-bit)  */
#define XQ_A_SAME 3          /* V side reuses the K-side A operand (MHA)         */
#define XQ_A_F16_ACC 4       /* fp16 accumulator rows updated in the first K pass */
                             /* by per-token delta codes (XQuant-CL delta layer)  */

const char* xq_version(void);
/* Message describing the last non-zero status returned on this host thread. */
const char* xq_last_error(void);

/* ======================================================================
 * Lane functions -- replace xcache._kernels (_kernels/__init__.py:20-26)
 * ====================================================================== */

/* quantize_groups: _native.pyx:111-153 / fallback.py:108-131.
 * x: float64 [rows, cols] C-contiguous (device). Per row, contiguous groups
 * of group_size: scale=(max-min)/(2^bits-1) (1 for a degenerate group),
 * zp=min, code=clamp(floor((x-min)/scale+0.5),0,2^bits-1), all in float64,
 * bit-identical to the reference. codes uint8 [rows, cols]; scales/zps
 * float64 [rows, ceil(cols/group_size)]. bits in {2,3,4,8}. */
int xq_quantize_groups(const double* x, int64_t rows, int64_t cols, int32_t group_size,
                       int32_t bits, uint8_t* codes, double* scales, double* zero_points,
                       void* stream);

/* dequantize_groups: _native.pyx:156-177 / fallback.py:134-146.
 * out = code*scale + zp in float64 with two roundings (no FMA). */
int xq_dequantize_groups(const uint8_t* codes, const double* scales, const double* zero_points,
                         int64_t rows, int64_t cols, int32_t group_size, double* out,
                         void* stream);

/* pack_codes / unpack_codes: _native.pyx:64-108 / fallback.py:58-94.
 * words must hold ceil(n*bits/64) uint64. bits in {1..8}. */
int xq_pack_codes(const uint8_t* codes, int64_t n, int32_t bits, uint64_t* words, void* stream);
int xq_unpack_codes(const uint64_t* words, int32_t bits, int64_t n, uint8_t* codes,
                    void* stream);

/* ======================================================================
 * Packed cache arena -- replaces quant.append_rows / cache._Stream.push|bulk
 * for the per-token payloads (cache.py:184-221, quant.py:198-228)
 * ====================================================================== */

/* Quantize n_rows rows (float32/bf16/f16/f64 per x_dtype, row stride in
 * elements) per token in groups of group_size and write packed rows +
 * half2 params into the arena.
 *   destination arena row of input row i:
 *     seq_lens != NULL : i*L_max + seq_lens[i] - 1  (decode: seq_lens counts
 *                        the token being appended; one token per slot)
 *     seq_lens == NULL : row0 + i                   (bulk / prefill)
 *   sub_rows != NULL : quantize x - sub_rows[dst row] instead of x
 *     (XQuant-CL delta against the fp32 accumulator, cache.py:478-479);
 *   x_eff_out != NULL: float64 [n_rows, cols] copy of the exact quantizer
 *     input (stage-wise parity hook).
 *   nonfinite_flag != NULL: set to 1 if any input is NaN/Inf (quant.py:114-115).
 */
int xq_quantize_rows(const void* x, int32_t x_dtype, int64_t x_row_stride, int64_t n_rows,
                     int64_t cols, int32_t bits, int32_t group_size, const int32_t* seq_lens,
                     int64_t row0, int64_t L_max, const float* sub_rows, uint8_t* codes,
                     int64_t row_bytes, void* params, double* x_eff_out, int32_t* nonfinite_flag,
                     void* stream);

/* XQuant-CL quantize-and-append with the running accumulator row in float64
 * (replaces _DeltaBackend._prefill/_decode, cache.py:460-481, with
 * Accumulator.seed/add, cache.py:124-146). Rows as xq_quantize_rows; row i of
 * acc_rows [n_rows, cols] (float64) is the accumulator at that token.
 * acc_mode 1 (delta layer): quantize x - acc, then acc += code*scale + zp.
 * acc_mode 2 (seeding base layer): quantize x, then acc = code*scale + zp.
 * The reconstruction uses the float64 scale/zero point before their fp16
 * storage, so the delta codes of every later layer are bit-exact with the
 * reference's. */
int xq_quantize_rows_cl(const void* x, int32_t x_dtype, int64_t x_row_stride, int64_t n_rows,
                        int64_t cols, int32_t bits, int32_t group_size, const int32_t* seq_lens,
                        int64_t row0, int64_t L_max, double* acc_rows, int32_t acc_mode,
                        uint8_t* codes, int64_t row_bytes, void* params, int32_t* nonfinite_flag,
                        void* stream);

/* xq-gqa decode append (replaces LatentInputCacheGQA._decode, cache.py:429-432,
 * with _Stream.push, cache.py:210-221): lat = x @ [U_k | U_v] on tcgen05 (bf16
 * operands, fp32 accumulation) for n_rows tokens (row b = slot b, appended at
 * position seq_lens[b]-1); the V latent (columns r..2r-1) is quantized per
 * token into the arena (codes + fp16 (scale, zp), as xq_quantize_rows); the K
 * latent (columns 0..r-1) goes to row seq_lens[b]-1-k_nflushed[b] of slot b's
 * float32 residual buffer k_resid [n_rows][128][r]. x: bf16 [n_rows] rows of
 * x_row_stride elements; u_bf16: [d][2r] row-major. lat_out (optional):
 * float32 [n_rows][2r]. group_size must be 128, r a multiple of 128, d of 64. */
int xq_latent_project_append(const void* x_bf16, int64_t x_row_stride, int32_t n_rows, int64_t d,
                             const void* u_bf16, int32_t r, int32_t bits, int32_t group_size,
                             const int32_t* seq_lens, const int32_t* k_nflushed, int64_t L_max,
                             float* k_resid, uint8_t* v_codes, int64_t v_row_bytes, void* v_params,
                             float* lat_out, int32_t* nonfinite_flag, void* stream);

/* The same quantizer writing the reference's float64 reconstruction
 * (codes * scale + zp, fallback.py:134-146) of every block row to recon_out
 * (may alias blocks). xq-cl-gqa keeps its accumulator at the new token in
 * float64 through it. */
int xq_quantize_blocks_per_channel_f64_recon(const double* blocks, int64_t n_blocks, int64_t cols,
                                             int32_t bits, int32_t group_size,
                                             const int64_t* dst_row0, uint8_t* codes,
                                             int64_t row_bytes, void* params, double* recon_out,
                                             int32_t* nonfinite_flag, void* stream);

/* xq-cl-gqa new-token latent (DeltaLatentCacheGQA._push_base / _push_delta,
 * cache.py:562-586): lat[b] = (x[b] - acc_row[b]) @ U in float64 (acc_row NULL
 * for a base layer), U [d][r] float32 or float64; written to row
 * seq_lens[b]-1-nflushed[b] of slot b's residual buffers resid64 (float64) and
 * resid32 (its float32 mirror), each [n_rows][group_size][r]. */
int xq_clgqa_latent64(const void* x, int32_t x_dtype, int64_t x_row_stride, int32_t n_rows,
                      int64_t d, const double* acc_row, const void* u, int32_t u_dtype, int64_t r,
                      const int32_t* seq_lens, const int32_t* nflushed, int32_t group_size,
                      double* resid64, float* resid32, int32_t* nonfinite_flag, void* stream);

/* xq-cl-gqa accumulator at the new token (Accumulator.seed / add of
 * reconstruct() @ U^T, cache.py:571-572, 588-589): acc_row[b] = (seed) or +=
 * resid64[b][rec_pos[b]] @ U^T in float64; acc_row [n_rows][d]. */
int xq_clgqa_row_update(const double* resid64, const int32_t* rec_pos, int32_t n_rows,
                        int32_t group_size, const void* u, int32_t u_dtype, int64_t d, int64_t r,
                        int32_t seed, double* acc_row, void* stream);

/* fp16 operand rows of the remat GEMM (quant.dequantize, quant.py:137-153, then
 * the stream's residual rows, cache.py:223-230): out[i] for i < n_codes is arena
 * row row0+i dequantized (codes * scale + zp, axis 0 per-token / 1 per-channel),
 * for n_codes <= i < n_rows the float32 row resid[i - n_codes]; out row stride ldo. */
int xq_dequant_rows_f16(const uint8_t* codes, int64_t row_bytes, const void* params, int32_t axis,
                        int32_t bits, int32_t group_size, int64_t cols, int64_t row0,
                        int64_t n_codes, const float* resid, int64_t n_rows, void* out,
                        int64_t ldo, void* stream);

/* Remat GEMM on tcgen05 for the bulk paths (prefill K/V rebuild,
 * cache.py:271-281 over a whole prompt; XQuant-CL latent accumulator update
 * acc (+)= reconstruct() @ U^T, cache.py:571-589): C[M x N] (+)= A[M x K] .
 * B[N x K]^T, fp16 row-major operands (lda / ldb / ldc in elements), fp32
 * accumulation. epilogue 0: C = fp16(acc); 1: C = fp16(RoPE(acc)), row i at
 * position pos0+i (rope_cs = the [rope_n][64] (cos, sin) table); 2: C += acc.
 * K must be a multiple of 64. */
int xq_gemm_f16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                int64_t M, int64_t N, int64_t K, int32_t epilogue, const void* rope_cs,
                int64_t rope_n, int64_t pos0, void* stream);

/* Causal grouped-query attention of a prefill (model._attention over the
 * prompt, model.py:150-182, as _Session.prefill calls it, model.py:205-221):
 * q [n][q_stride] (rotated, head h at columns 128h..), k / v [n][kv_stride]
 * (k rotated; KV head h / group), fp16 or bf16 (dtype); out float32
 * [n][out_stride], head h at 128h. Flash-attention (online softmax), K/V read
 * tile by tile. */
int xq_prefill_attend(const void* q, const void* k, const void* v, int32_t dtype, int32_t n,
                      int32_t n_heads, int32_t group, int64_t q_stride, int64_t kv_stride,
                      float sm_scale, float* out, int64_t out_stride, void* stream);

/* RoPE (linalg.apply_rope, linalg.py:58-95) of n rows of width (whole 128-wide
 * heads) at positions pos0.. : in float32 / fp16, out fp16 / bf16 (may alias in
 * when the types match). */
int xq_rope_rows(const void* in, int32_t in_dtype, int64_t in_stride, int64_t n, int64_t width,
                 const void* rope_cs, int64_t rope_n, int64_t pos0, void* out, int32_t out_dtype,
                 int64_t out_stride, void* stream);

/* Per-channel quantization of whole token groups (quant.py:124-134): block b
 * is float32 [group_size, cols] at blocks + b*group_size*cols; its codes go to
 * arena rows dst_row0[b] .. +group_size-1 and its params to param row
 * dst_row0[b]/group_size. Used for the xq-gqa K latent flush (cache.py:218-221). */
int xq_quantize_blocks_per_channel(const float* blocks, int64_t n_blocks, int64_t cols,
                                   int32_t bits, int32_t group_size, const int64_t* dst_row0,
                                   uint8_t* codes, int64_t row_bytes, void* params,
                                   int32_t* nonfinite_flag, void* stream);
/* The same on float64 blocks (the xq-cl-gqa latents, formed in float64 like
 * the reference's so the per-channel codes match it, cache.py:574-586). */
int xq_quantize_blocks_per_channel_f64(const double* blocks, int64_t n_blocks, int64_t cols,
                                       int32_t bits, int32_t group_size, const int64_t* dst_row0,
                                       uint8_t* codes, int64_t row_bytes, void* params,
                                       int32_t* nonfinite_flag, void* stream);

/* Dequantize arena rows [row0, row0+n_rows) to float32 [n_rows, cols]
 * (quant.dequantize, quant.py:137-153). axis 0 per-token, 1 per-channel. */
int xq_dequant_rows(const uint8_t* codes, int64_t row_bytes, const void* params, int32_t axis,
                    int32_t bits, int32_t group_size, int64_t cols, int64_t row0, int64_t n_rows,
                    float* out, void* stream);

/* ======================================================================
 * Rematerialisation + decode attention (cache.py:271-281, model.py:150-182)
 * ====================================================================== */

/* cos/sin table as float2, angle pos*theta^(-2j/hd) formed in float64
 * (linalg.py:84-88). j_major == 0: [n_pos][head_dim/2] (position-major, used
 * by the fp16-KV baseline and the debug remat); j_major != 0:
 * [head_dim/2][n_pos] (frequency-major, coalesced reads in the fused kernel). */
int xq_rope_table(void* cs_out, int64_t n_pos, int32_t head_dim, double theta, int32_t j_major,
                  void* stream);

/* Arrange K/V projection weights for the fused kernel: out is fp16
 * [n_kv_heads][256][kdim]: rows 0..127 of head h are W_k[:, h*128 .. +128]^T,
 * rows 128..255 are W_v[:, h*128 .. +128]^T, each K-major with the channel
 * order permuted to match the dequant producer of the A stream that feeds it
 * (a_mode_* in XQ_A_*, bits_* its code width). w_k / w_v: [kdim, n_kv_heads*128]
 * row-major (x @ W convention, cache.py:385-387), dtype per w_dtype. */
int xq_arrange_weights(const void* w_k, const void* w_v, int32_t w_dtype, int64_t kdim,
                       int32_t n_kv_heads, int32_t a_mode_k, int32_t bits_k, int32_t a_mode_v,
                       int32_t bits_v, void* w_out, void* stream);

/* Workspace (bytes) the fused decode kernel needs for its split partials. */
int64_t xq_decode_workspace_bytes(int32_t n_seqs, int32_t max_len, int32_t n_kv_heads,
                                  int32_t group, int32_t tiles_per_chunk);

/* Fused dequant -> rematerialise (tcgen05, TMEM accumulator) -> RoPE ->
 * flash-decode. K and V are never written to HBM.
 *   For every sequence b and KV head h: K = RoPE(A_K @ W_k[:, h]),
 *   V = A_V @ W_v[:, h] over tokens [0, seq_lens[b]); every query head
 *   h*group .. h*group+group-1 attends with q = RoPE(q_pre, seq_lens[b]-1).
 *   out: float32 [n_seqs, n_kv_heads*group, 128].
 *   A_K: ak_mode XQ_A_CODES_TOKEN / XQ_A_CODES_CHANNEL / XQ_A_F16_ROWS;
 *        for CODES_CHANNEL, tokens t >= ak_nflushed[b] are read from the
 *        float32 residual rows ak_resid + b*G*kdim (cache.py:223-230).
 *   A_V: av_mode as above or XQ_A_SAME (MHA: one X cache feeds K and V).
 *   rows of both A streams are arena rows b*L_max + t with row_bytes bytes
 *   (codes) or kdim fp16 (F16_ROWS).
 *   w_arranged: from xq_arrange_weights. rope_cs: frequency-major table from
 *   xq_rope_table(j_major=1) with rope_n >= max_len positions. sm_scale:
 *   1/sqrt(128) for the reference (model.py:164). */
int xq_decode_attend(int32_t ak_mode, const void* ak_src, const void* ak_params,
                     const float* ak_resid, const int32_t* ak_nflushed, int32_t ak_bits,
                     int64_t ak_row_bytes, int32_t av_mode, const void* av_src,
                     const void* av_params, int32_t av_bits, int64_t av_row_bytes,
                     int32_t group_size, int64_t L_max, int64_t kdim, const int32_t* seq_lens,
                     int32_t n_seqs, int32_t max_len, const void* w_arranged, int32_t n_kv_heads,
                     int32_t group, const float* q_pre, const void* rope_cs, int64_t rope_n,
                     float sm_scale, int32_t tiles_per_chunk, void* workspace,
                     int64_t workspace_bytes, float* out, void* stream);

/* ---- V-absorbed variant (the default hot path) ----
 * Same result as xq_decode_attend, computed with the exact reassociation
 *   sum_t p_t (A_V[t] @ W_v[:, kv]) = (sum_t p_t A_V[t]) @ W_v[:, kv]
 * (cache.py:385-387 + model.py:178-181): the K side is rematerialised on
 * tcgen05 as before (four KV heads per pass); the V side is one
 * [kdim x n_q] tcgen05 GEMM over each 256-token tile's probabilities plus a
 * per-head projection through W_v at the end. kdim % 256 == 0. */

/* Arranged weights of the absorbed kernel. wk_out: fp16
 * [ceil(n_kv/4)*512][kdim], row h*128+j = W_k[:, h*128+j]^T in the K-side
 * producer channel order (zero rows pad an odd n_kv). wv_out: fp16
 * [n_kv][kdim][128], row c = W_v[perm_v(c), h*128 .. +128] with perm_v the
 * V-side producer order. a_mode_v may be XQ_A_SAME. */
int xq_arrange_weights_absorbed(const void* w_k, const void* w_v, int32_t w_dtype, int64_t kdim,
                                int32_t n_kv_heads, int32_t a_mode_k, int32_t bits_k,
                                int32_t a_mode_v, int32_t bits_v, void* wk_out, void* wv_out,
                                void* stream);

/* Workspace (bytes): per-tile partials O [n_seqs][tiles][n_q][kdim] + (m, l). */
int64_t xq_absorbed_workspace_bytes(int32_t n_seqs, int32_t max_len, int32_t n_q_heads,
                                    int64_t kdim);

/* Arguments as xq_decode_attend, with the two arranged weight buffers of
 * xq_arrange_weights_absorbed in place of w_arranged. out: float32
 * [n_seqs, n_kv_heads*group, 128]. ak_first (nullable, CODES_CHANNEL K side
 * only): float32 per arena row, the full-precision channel 0 of the flushed
 * K-latent rows -- the fp16 outlier channel of cache.py:406-411 / :653-658. */
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
                              int64_t workspace_bytes, float* out, void* stream);

/* XQuant-CL delta layer with the accumulate fused in (cache.py:472-481 +
 * Accumulator.add, cache.py:139-146, then the delta layer's remat from the
 * accumulator, cache.py:527-535): acc16 is the fp16 accumulator
 * [n_seqs * L_max, kdim] BEFORE this layer; codes / params are this layer's
 * per-token delta arena (XQ_A_CODES_TOKEN layout, bits 2/3/4/8). In the first K
 * pass over each 256-token tile the dequant producers add the dequantized deltas
 * to the TMA-staged accumulator rows, acc[t] = fp16(float(acc[t]) + code*scale +
 * zp) for t < seq_lens[b] (the arithmetic of xq_cl_accumulate, bit-identical),
 * feed the updated rows to the tensor cores and write them back to acc16; the
 * later K passes and the V side read the updated rows. Replaces xq_cl_accumulate
 * (seed = 0) followed by xq_decode_attend_absorbed on XQ_A_F16_ROWS. MHA (group
 * 1) only; other arguments as xq_decode_attend_absorbed. */
int xq_decode_attend_absorbed_cl(void* acc16, const void* codes, const void* params, int32_t bits,
                                 int64_t row_bytes, int32_t group_size, int64_t L_max,
                                 int64_t kdim, const int32_t* seq_lens, int32_t n_seqs,
                                 int32_t max_len, const void* wk_arranged,
                                 const void* wv_arranged, int32_t n_kv_heads, const float* q_pre,
                                 const void* rope_cs, int64_t rope_n, float sm_scale,
                                 void* workspace, int64_t workspace_bytes, float* out,
                                 void* stream);

/* xq_decode_attend_absorbed with the projected output [n_seqs][H][128] stored
 * to each of n_outs (1..9) destinations. Under KV-head-group sharding
 * (paper_2508_10395_b200/parallel.py) these are this rank's slot
 * in every rank's gather buffer (peer pointers, e.g. torch symmetric memory over
 * NVLink): the all-gather of attention outputs becomes the projection kernel's
 * own stores, followed by a device-side barrier instead of an NCCL call. outs is
 * a host array of device (or peer) pointers. */
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
                                    float* const* outs, int32_t n_outs, void* stream);

/* Debug: cycles each warp role of the absorbed kernel spent blocked per
 * barrier (16 uint64 counters, see csrc/xq_absorb.cu); all zero unless the
 * library was built with -DXQ_ROLE_PROFILE (tools/build_role_profile.sh).
 * reset != 0 clears them after the read. */
int xq_debug_role_profile(uint64_t* out, int32_t reset);

/* Debug hook: when buf != NULL, xq_decode_attend also dumps the raw fp32
 * accumulator of every tile t < n_tiles to buf[b][kv_head][t][128][256]
 * (columns 0-127 = pre-RoPE K, 128-255 = V). NULL disables (default). */
int xq_debug_set_acc_dump(float* buf, int32_t n_tiles);

/* Debug / parity path: SIMT float32 rematerialisation that writes K and V
 * to HBM (cache.rematerialize, cache.py:271-281). a_*: as xq_decode_attend
 * for one sequence slot `slot` and tokens [0, n_tok). w_k/w_v float32
 * [kdim, n_out]. k_out/v_out float32 [n_tok, n_out]; K gets RoPE at
 * positions 0..n_tok-1 (head_dim 128). */
int xq_remat_f32(int32_t ak_mode, const void* ak_src, const void* ak_params,
                 const float* ak_resid, int32_t ak_nflushed, int32_t ak_bits,
                 int64_t ak_row_bytes, int32_t av_mode, const void* av_src, const void* av_params,
                 int32_t av_bits, int64_t av_row_bytes, int32_t group_size, int64_t L_max,
                 int64_t kdim, int32_t slot, int32_t n_tok, const float* w_k, const float* w_v,
                 int64_t n_out, const void* rope_cs, float* k_out, float* v_out, void* stream);

/* ======================================================================
 * XQuant-CL accumulator (cache.py:124-146, 460-481)
 * ====================================================================== */

/* For every slot b and token t < seq_lens[b]:
 *   seed != 0 : acc = deq(codes)          (base layer seeds, cache.py:473-477)
 *   seed == 0 : acc = acc + deq(codes)    (delta layer, cache.py:481)
 * and, if x16_out != NULL, x16_out = fp16(acc) for the remat A operand.
 * acc == NULL: fp16-storage accumulator -- x16_out is the accumulator itself
 * (read, updated, written back in fp16; the reference's accounting charges the
 * accumulator 4 bits, cache.py:45, 129-133). acc/x16_out: [n_slots*L_max][cols]. */
int xq_cl_accumulate(int32_t seed, const uint8_t* codes, int64_t row_bytes, const void* params,
                     int32_t bits, int32_t group_size, int64_t cols, const int32_t* seq_lens,
                     int32_t n_seqs, int32_t max_len, int64_t L_max, float* acc, void* x16_out,
                     void* stream);

/* ======================================================================
 * fp16-KV decode baseline (FullPrecisionCache semantics, cache.py:302-323;
 * the baseline stores post-RoPE K, which is mathematically identical)
 * ====================================================================== */

/* Append RoPE(k_new) and v_new (float32 [n_seqs, n_kv_heads*128]) at position
 * seq_lens[b]-1 of bf16 caches [n_slots*L_max][n_kv_heads*128]. */
int xq_kv_append(const float* k_new, const float* v_new, const int32_t* seq_lens, int32_t n_seqs,
                 int32_t n_kv_heads, int64_t L_max, const void* rope_cs, void* k_cache,
                 void* v_cache, void* stream);

/* Split-K flash-decode over the bf16 caches for tokens [0, seq_lens[b]). */
int64_t xq_kv_decode_workspace_bytes(int32_t n_seqs, int32_t max_len, int32_t n_kv_heads,
                                     int32_t group, int32_t chunk_tokens);
int xq_kv_decode_attend(const void* k_cache, const void* v_cache, int64_t L_max,
                        const int32_t* seq_lens, int32_t n_seqs, int32_t max_len,
                        int32_t n_kv_heads, int32_t group, const float* q_pre,
                        const void* rope_cs, float sm_scale, int32_t chunk_tokens,
                        void* workspace, int64_t workspace_bytes, float* out, void* stream);

/* ======================================================================
 * Quantized-KV decode baseline "kvq" (QuantizedKvCache, cache.py:326-360)
 * ====================================================================== */

/* Workspace (bytes) of xq_kvq_decode_attend's split partials. */
int64_t xq_kvq_workspace_bytes(int32_t n_seqs, int32_t max_len, int32_t n_q_heads,
                               int32_t chunk_tokens);

/* Decode attention over a quantized K/V cache: K pre-RoPE per-channel codes
 * (planar params in the producer order, residual rows k_resid for tokens >=
 * k_nflushed[b]), V per-token codes + half2 params (residual rows v_resid for
 * tokens >= v_nflushed[b]); width n_kv_heads*128, both arenas row_bytes wide.
 * K is rotated at its cached positions (cache.py:357-360), q at
 * seq_lens[b]-1; rope_cs is the position-major table. out: float32
 * [n_seqs, n_kv_heads*group, 128]. */
int xq_kvq_decode_attend(const uint8_t* k_codes, const void* k_params, const float* k_resid,
                         const uint8_t* v_codes, const void* v_params, const float* v_resid,
                         const int32_t* k_nflushed, const int32_t* v_nflushed, int32_t bits,
                         int32_t group_size, int64_t row_bytes, int64_t L_max,
                         const int32_t* seq_lens, int32_t n_seqs, int32_t max_len,
                         int32_t n_kv_heads, int32_t group, const float* q_pre,
                         const void* rope_cs, float sm_scale, int32_t chunk_tokens,
                         void* workspace, int64_t workspace_bytes, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* XQUANT_H_ */
