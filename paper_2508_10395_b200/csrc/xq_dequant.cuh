// Dequant producer building blocks shared by the fused decode kernels:
// packed codes staged in shared memory -> fp16 pairs (magic-number convert,
// one HFMA2 per pair) -> one 128-byte SWIZZLE_128B row of an fp16 A tile.
// The channel order inside a block is the producer order of xq_layout.cuh.
#pragma once

#include "xq_common.cuh"
#include "xq_layout.cuh"

namespace xq {

constexpr int kDqChunk = 64;  // channels per produced row chunk (one 128-byte swizzle row)
constexpr int kDqG = 128;     // quantization group the producers are specialised for

template <typename T>
XQ_DEVINL uint32_t as_u32(T v) {
  return *reinterpret_cast<uint32_t*>(&v);
}
template <typename T>
XQ_DEVINL T from_u32(uint32_t v) {
  return *reinterpret_cast<T*>(&v);
}

// (a & mask) | magic in one LOP3: both constants live in registers (a LOP3
// takes a single immediate, so nvcc would otherwise emit two instructions).
XQ_DEVINL uint32_t and_or(uint32_t a, uint32_t mask, uint32_t magic) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(mask), "r"(magic));
  return d;
}

// codes at bits 0.. and 16.. of `bits` (unmasked) -> fp16 pair c*s + z, one rounding:
// 0x6400|c is the fp16 value 1024+c, exactly; subtracting 1024 is exact.
XQ_DEVINL uint32_t deq_pair(uint32_t bits, uint32_t mask, __half2 s2, __half2 z2) {
  const uint32_t magic = 0x64006400u;
  const __half2 c = __hsub2(from_u32<__half2>(and_or(bits, mask, magic)), __float2half2_rn(1024.f));
  return as_u32(__hfma2(c, s2, z2));
}

// 64 codes -> 32 fp16 pairs in producer order (xq_layout.cuh).
// s2/z2: per pair (per-channel) or uniform.
template <int BITS, bool PER_PAIR>
XQ_DEVINL void convert_raw(const uint32_t (&w)[2 * BITS], const __half2* s2, const __half2* z2,
                           uint32_t (&out)[32]) {
  auto S = [&](int j) { return PER_PAIR ? s2[j] : s2[0]; };
  auto Z = [&](int j) { return PER_PAIR ? z2[j] : z2[0]; };
  if constexpr (BITS == 4) {
#pragma unroll
    for (int wi = 0; wi < 8; ++wi)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        out[4 * wi + j] = deq_pair(w[wi] >> (4 * j), 0x000F000Fu, S(4 * wi + j), Z(4 * wi + j));
  } else if constexpr (BITS == 2) {
#pragma unroll
    for (int wi = 0; wi < 4; ++wi)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        out[8 * wi + j] = deq_pair(w[wi] >> (2 * j), 0x00030003u, S(8 * wi + j), Z(8 * wi + j));
  } else if constexpr (BITS == 8) {
#pragma unroll
    for (int wi = 0; wi < 16; ++wi)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        out[2 * wi + j] = deq_pair(w[wi] >> (8 * j), 0x00FF00FFu, S(2 * wi + j), Z(2 * wi + j));
  } else {  // 3-bit: two 32-code blocks of 3 words each
#pragma unroll
    for (int bi = 0; bi < 2; ++bi) {
      const uint32_t w0 = w[3 * bi], w1 = w[3 * bi + 1], w2 = w[3 * bi + 2];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        // code j at bit 3j, code j+16 at bit 3j+48 of the 96-bit block
        const int o_lo = 3 * j, o_hi = 3 * j + 32;
        const uint32_t lo = (o_lo < 32) ? __funnelshift_r(w0, w1, o_lo) : (w1 >> (o_lo - 32));
        const uint32_t hi = (o_hi < 64) ? __funnelshift_r(w1, w2, o_hi - 32) : (w2 >> (o_hi - 64));
        out[16 * bi + j] = deq_pair(__byte_perm(lo, hi, 0x7610), 0x00070007u, S(16 * bi + j),
                                    Z(16 * bi + j));
      }
    }
  }
}

// 2*BITS words of one row's 64-code chunk from shared memory (32-bit address)
template <int BITS>
XQ_DEVINL void lds_raw(uint32_t src, uint32_t (&w)[2 * BITS]) {
  if constexpr (BITS == 3) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const uint2 a = lds64(src + 8 * q);
      w[2 * q] = a.x;
      w[2 * q + 1] = a.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < BITS / 2; ++q) {
      const uint4 a = lds128(src + 16 * q);
      w[4 * q] = a.x; w[4 * q + 1] = a.y; w[4 * q + 2] = a.z; w[4 * q + 3] = a.w;
    }
  }
}

// Per-thread constants of the SWIZZLE_128B row store: byte offsets of the 8
// 16-byte chunks of this row (chunk c goes to slot c ^ (row % 8)).
struct RowSwizzle {
  uint32_t off[8];
  XQ_DEVINL explicit RowSwizzle(int row) {
#pragma unroll
    for (int c = 0; c < 8; ++c) off[c] = sw128_offset(row, c);
  }
  XQ_DEVINL void store(uint32_t tile, const uint32_t (&v)[32]) const {
#pragma unroll
    for (int c = 0; c < 8; ++c) sts128(tile + off[c], v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
};

// One producer thread: convert its row's 64-channel chunk of one A stream into 32
// fp16 pairs in producer order (registers; the caller stores them once the A stage is
// free, so the conversion overlaps the wait). cstage / pstage are 32-bit shared
// addresses of the staged codes and parameters.
template <int MODE, int BITS>
XQ_DEVINL void convert_chunk(uint32_t cstage, uint32_t pstage, int row, bool valid, int tok, int b,
                             int nflushed, int kc, const float* first_row, const float* resid,
                             int kdim, uint32_t (&v)[32], int G = kDqG) {
#ifdef XQ_EXP_NOCONV  // timing experiment only (tools/build_variant.sh): producers without the conversion
  valid = false;
#endif
  if (!valid) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0u;
    return;
  }
  const uint32_t crow = cstage + row * (16 * BITS) + (kc & 1) * 8 * BITS;
  if constexpr (MODE == XQ_A_CODES_TOKEN) {
    uint32_t raw[2 * BITS];
    lds_raw<BITS>(crow, raw);
    // the chunk's first group is kc*64/G; the staged quad of (scale, zp) starts at a
    // multiple of 4 groups (G = 128: kc/2, G = 64: kc, G = 32: 2kc and 2kc+1)
    const int gi = ((kc * kDqChunk) / G) & 3;
    const __half2 sz = from_u32<__half2>(lds32(pstage + row * 16 + 4 * gi));
    if (G >= kDqChunk) {
      const __half2 s2 = __low2half2(sz), z2 = __high2half2(sz);
      convert_raw<BITS, false>(raw, &s2, &z2, v);
    } else {  // G = 32: pairs 0-15 (channel blocks of the first 32) and 16-31 (producer order)
      const __half2 sz1 = from_u32<__half2>(lds32(pstage + row * 16 + 4 * (gi + 1)));
      __half2 s2[32], z2[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        s2[j] = j < 16 ? __low2half2(sz) : __low2half2(sz1);
        z2[j] = j < 16 ? __high2half2(sz) : __high2half2(sz1);
      }
      convert_raw<BITS, true>(raw, s2, z2, v);
    }
  } else {  // XQ_A_CODES_CHANNEL
    constexpr int BS = BITS == 2 ? 16 : BITS == 3 ? 32 : BITS == 4 ? 8 : 4;
    if (tok < nflushed) {
      uint32_t raw[2 * BITS];
      lds_raw<BITS>(crow, raw);
      // per-channel params of this token group, staged by TMA as [scales(128) | zps(128)]
      // halves in producer order: broadcast shared loads (every row reads the same)
      const uint32_t ps = pstage + (kc & 1) * 128;
      __half2 s2[32], z2[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 a = lds128(ps + 16 * c);
        const uint4 z = lds128(ps + 256 + 16 * c);
        s2[4 * c] = from_u32<__half2>(a.x); s2[4 * c + 1] = from_u32<__half2>(a.y);
        s2[4 * c + 2] = from_u32<__half2>(a.z); s2[4 * c + 3] = from_u32<__half2>(a.w);
        z2[4 * c] = from_u32<__half2>(z.x); z2[4 * c + 1] = from_u32<__half2>(z.y);
        z2[4 * c + 2] = from_u32<__half2>(z.z); z2[4 * c + 3] = from_u32<__half2>(z.w);
      }
      convert_raw<BITS, true>(raw, s2, z2, v);
      // fp16 outlier channel (cache.py:406-411): channel 0 (position 0 of the
      // first block in producer order) kept in full precision beside the codes
      if (first_row != nullptr && kc == 0)
        v[0] = as_u32(__halves2half2(__float2half_rn(*first_row), __high2half(from_u32<__half2>(v[0]))));
    } else {  // residual full-precision row (cache.py:228-229)
      const float* r = resid + ((int64_t)b * kDqG + (tok - nflushed)) * kdim + kc * kDqChunk;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int blk = (2 * j) / BS, jj = j % (BS / 2);
        const int c0 = blk * BS + jj, c1 = c0 + BS / 2;
        v[j] = as_u32(__floats2half2_rn(r[c0], r[c1]));
      }
    }
  }
}

// convert_chunk + the SWIZZLE_128B row store (tile: the A stage's 32-bit shared address)
template <int MODE, int BITS>
XQ_DEVINL void produce_chunk(uint32_t tile, uint32_t cstage, uint32_t pstage, const RowSwizzle& sw,
                             int row, bool valid, int tok, int b, int nflushed, int kc,
                             const float* first_row, const float* resid, int kdim) {
  uint32_t v[32];
  convert_chunk<MODE, BITS>(cstage, pstage, row, valid, tok, b, nflushed, kc, first_row, resid, kdim, v);
  sw.store(tile, v);
}

}  // namespace xq
