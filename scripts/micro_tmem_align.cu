// TMEM load cost vs column alignment: 8 warps (two per lane quarter) each load 40 columns of "E" and 40 of
// "O" (x16, x16, x8 each) starting at column offset `off` (0 or 40), as the Step-3 epilogue halves do.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/micro_tmem_align scripts/micro_tmem_align.cu
#include <cstdio>
#include "../paper_1905_12317_b200/csrc/ftk_sm100.cuh"
using namespace ftk::sm100;

__device__ __forceinline__ void ld8(uint32_t a, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(a));
}

__global__ void __launch_bounds__(288, 1) k(int iters, int mode, unsigned long long* cyc, unsigned* sink) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&tb);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tb;
  if (warp >= 1) {
    const int q = warp & 3, h = (warp - 1) >> 2;
    // mode 0: both halves at h * 40 (h = 1 unaligned); mode 1: both halves at 16-aligned offsets h * 48
    const uint32_t off = mode == 0 ? (uint32_t)(h * 40) : (uint32_t)(h * 48);
    uint32_t acc = 0;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t base = tm + ((uint32_t)(q * 32) << 16) + (uint32_t)((it & 1) * 160) + off;
      uint32_t e0[16], e1[16], e2[8], o0[16], o1[16], o2[8];
      tmem_ld16(base, e0);
      tmem_ld16(base + 80, o0);
      tmem_ld16(base + 16, e1);
      tmem_ld16(base + 96, o1);
      ld8(base + 32, e2);
      ld8(base + 112, o2);
      tmem_wait_ld();
      for (int k2 = 0; k2 < 16; ++k2) acc ^= e0[k2] ^ o0[k2] ^ e1[k2] ^ o1[k2];
      for (int k2 = 0; k2 < 8; ++k2) acc ^= e2[k2] ^ o2[k2];
    }
    if (lane == 0) cyc[blockIdx.x * 8 + warp - 1] = clock64() - t0;
    if (acc == 0x1234567u) sink[0] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tm);
  }
}

int main() {
  unsigned long long* d;
  unsigned* sink;
  cudaMalloc(&d, 148 * 8 * sizeof(unsigned long long));
  cudaMalloc(&sink, 4);
  unsigned long long h[148 * 8];
  for (int mode : {0, 1}) {
    k<<<148, 288>>>(4000, mode, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): cycles per iteration by warp (h=0 x4, h=1 x4):", mode, mode == 0 ? "offsets 0 / 40" : "offsets 0 / 48");
    for (int w = 0; w < 8; ++w) printf(" %.0f", h[w] / 4000.0);
    printf("\n");
  }
  return 0;
}
