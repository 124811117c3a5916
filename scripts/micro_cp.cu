// Validates the tcgen05.cp.cta_group::1.128x256b layout assumption used by Step 3: the shared-memory
// source is a 128-row x 32-byte matrix in the canonical K-major SWIZZLE_NONE layout (core matrix =
// 8 rows x 16 B; LBO = stride between the two K-adjacent cores, SBO = stride between 8-row groups);
// row i lands in TMEM lane i, bytes [0,32) of the row in columns c0..c0+7.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/micro_cp scripts/micro_cp.cu
#include <cstdio>
#include "../paper_1905_12317_b200/csrc/ftk_sm100.cuh"
using namespace ftk::sm100;

__device__ __forceinline__ void tc_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

// src image: 128 rows x 24 words (96 B) -> 3 cp instructions of 8 columns
__global__ void k(uint32_t* out, int lbo, int sbo_cores) {
  __shared__ __align__(1024) uint32_t sm[128 * 24];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  // canonical: core (r/8, w/4): offset (r/8)*SBO + (w/4)*LBO + (r%8)*16 + (w%4)*4 bytes
  const int SBO = sbo_cores * 128;
  for (int i = tid; i < 128 * 24; i += blockDim.x) {
    const int r = i / 24, w = i % 24;
    const int off = (r / 8) * SBO + (w / 4) * lbo + (r % 8) * 16 + (w % 4) * 4;
    sm[off / 4] = (uint32_t)(r * 1000 + w);
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<32>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (tid == 0) {
    for (int j = 0; j < 3; ++j) {  // 8 words (2 cores along K) per instruction
      const uint64_t d = smem_desc_kmajor_noswz(smem_u32(sm) + j * 2 * lbo, lbo, SBO);
      tc_cp_128x256b(tm + 8 * j, d);
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t v[16];
  tmem_ld16(tm + ((uint32_t)(warp * 32) << 16), v);
  uint32_t v2[16];
  tmem_ld16(tm + ((uint32_t)(warp * 32) << 16) + 16, v2);
  tmem_wait_ld();
  for (int c = 0; c < 16; ++c) out[tid * 24 + c] = v[c];
  for (int c = 0; c < 8; ++c) out[tid * 24 + 16 + c] = v2[c];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<32>(tm); }
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 128 * 24 * 4);
  static uint32_t h[128 * 24];
  // layout A: LBO = 128 B (K-adjacent cores contiguous), SBO = 6 cores (rows groups of 8 x 24 words)
  for (int variant = 0; variant < 2; ++variant) {
    const int lbo = variant == 0 ? 128 : 16 * 128, sbo = variant == 0 ? 6 : 1;
    cudaMemset(d, 0xff, 128 * 24 * 4);
    k<<<1, 128>>>(d, lbo, sbo);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 128; ++r)
      for (int w = 0; w < 24; ++w)
        if (h[r * 24 + w] != (uint32_t)(r * 1000 + w)) {
          if (bad < 5) printf("variant %d mismatch r=%d w=%d got %u\n", variant, r, w, h[r * 24 + w]);
          ++bad;
        }
    printf("variant %d (LBO=%d, SBO=%d cores): %s (%d bad)\n", variant, lbo, sbo, bad ? "FAIL" : "OK", bad);
  }
  return 0;
}
