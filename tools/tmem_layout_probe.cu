// Probe the thread <-> (lane, column) layout of tcgen05.ld.16x256b (debug tool).
// Each of 4 warps writes value lane*1000 + col into its 32 TMEM lanes (32x32b
// store), then reads columns 0..15 of lanes base..base+15 with 16x256b.x2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o build/tmem_probe tools/tmem_layout_probe.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2508_10395_b200/csrc/xq_common.cuh"

__global__ void k(float* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        xq::smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  xq::tc_fence_before();
  __syncthreads();
  xq::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t tl = static_cast<uint32_t>(warp * 32) << 16;
  uint32_t v[16];
  for (int c = 0; c < 16; ++c) v[c] = __float_as_uint(float((warp * 32 + lane) * 1000 + c));
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tmem + tl),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(tmem + tl + (16u << 16))
               : "memory");
  xq::tmem_wait_ld();
  for (int i = 0; i < 8; ++i) out[(warp * 32 + lane) * 8 + i] = __uint_as_float(r[i]);
  xq::tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 8 * sizeof(float));
  k<<<1, 128>>>(d);
  float h[128 * 8];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("status %s\n", cudaGetErrorString(e));
  int bad = 0;
  for (int w = 0; w < 4; ++w)
    for (int t = 0; t < 32; ++t) {
      // expected (mma m16n8 C-fragment order): r0,r1 lane t/4 cols 2(t%4),+1; r2,r3 lane t/4+8;
      // r4..r7 the same for cols +8
      for (int i = 0; i < 8; ++i) {
        const int lanex = w * 32 + 16 + t / 4 + ((i & 2) ? 8 : 0);
        const int col = 2 * (t % 4) + (i & 1) + ((i & 4) ? 8 : 0);
        const float want = lanex * 1000 + col;
        if (h[(w * 32 + t) * 8 + i] != want) ++bad;
      }
      if (w == 1 && t < 6) {
        printf("w1 t%d:", t);
        for (int i = 0; i < 8; ++i) printf(" %.0f", h[(w * 32 + t) * 8 + i]);
        printf("\n");
      }
    }
  printf("mismatches vs mma-fragment layout: %d\n", bad);
  return 0;
}
