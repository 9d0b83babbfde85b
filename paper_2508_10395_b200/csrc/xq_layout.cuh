// Channel order of the fp16 A tiles the dequant producers write into shared
// memory, and the matching order of the arranged weights.
//
// A producer turns packed codes into fp16 *pairs* with one shift+mask per
// pair: for b-bit codes the pair (j, j + BS/2) of a block of BS codes sits at
// bit distance 16 inside one 32-bit window (b=2: BS=16, b=4: BS=8, b=8: BS=4;
// b=3 uses two 32-bit windows 32 bits apart, BS=32). Shared-memory position p
// of a block therefore holds channel perm(p): even p -> p/2, odd p -> BS/2+p/2.
// The GEMM sums over channels, so permuting A columns and W rows by the same
// perm leaves K and V unchanged; xq_arrange_weights applies it to W once.
#pragma once

#include <stdint.h>

#include "../../include/xquant.h"

namespace xq {

__host__ __device__ inline int perm_block(int a_mode, int bits) {
  if (a_mode == XQ_A_F16_ROWS) return 1;
  switch (bits) {
    case 2: return 16;
    case 3: return 32;
    case 4: return 8;
    case 8: return 4;
    default: return 1;
  }
}

// channel (relative to the block start) stored at position p of the block
__host__ __device__ inline int perm_channel(int p, int bs) {
  if (bs == 1) return 0;
  return (p & 1) ? (bs >> 1) + (p >> 1) : (p >> 1);
}

// inverse of perm_channel: storage position of channel j of a block
__host__ __device__ inline int perm_position(int j, int bs) {
  if (bs == 1) return 0;
  const int h = bs >> 1;
  return j < h ? 2 * j : 2 * (j - h) + 1;
}

// Row stride (in half2 entries) of the per-token (scale, zp) grid: padded to a
// multiple of 4 groups so a 128-row TMA box of 16-byte rows can stage it.
__host__ __device__ inline int64_t param_stride(int64_t cols, int G) {
  const int64_t ng = (cols + G - 1) / G;
  return (ng + 3) / 4 * 4;
}

}  // namespace xq
