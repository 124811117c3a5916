// tcgen05.mma (A from TMEM, B from shared memory) throughput for a B operand that walks through shared
// memory (Step-1 image stages: N = 128 rows x K = 64 bf16 per stage, 4 K16 steps) in the canonical
// no-swizzle K-major layout vs the 128-byte-swizzled K-major layout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/micro_swz scripts/micro_swz.cu
#include <cstdio>
#include "../paper_1905_12317_b200/csrc/ftk_sm100.cuh"
using namespace ftk::sm100;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {  // K-major, 128 B swizzle, 8-row atoms of 1 KB
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;   // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                        // version
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}

__global__ void __launch_bounds__(128, 1) k(int iters, int N, int mode, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8 * 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tb);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tb;
  if (warp == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint32_t base = smem_u32(sm);
    const uint32_t stage = (uint32_t)N * 64 * 2;  // N rows x 64 bf16
    const unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int c = 0; c < iters; ++c) {
        const int st = (c >> 2) & 7, ks = c & 3;
        uint64_t bd;
        if (mode == 0)  // canonical no-swizzle: core matrix (row8, kgroup) at row8 * (64/8) * 128 + kgroup * 128
          bd = smem_desc_kmajor_noswz(base + st * stage + ks * 256, 128, (64 / 8) * 128);
        else            // 128B swizzle: row r at r * 128 (+ XOR), K16 step = +32 B
          bd = desc_sw128(base + st * stage + ks * 32);
        mma_f16_ts(tm, tm + 256, bd, idesc, c > 0 ? 1u : 0u);
      }
      tc_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  unsigned long long h[148];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  for (int N : {128, 80})
    for (int mode : {0, 1}) {
      const int iters = 8000;
      k<<<148, 128, 8 * 16384>>>(iters, N, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      printf("N=%d B %s: %.1f cycles/MMA (ideal %.0f)\n", N, mode ? "SW128 " : "no-swz", (double)h[0] / iters, 128.0 * N / 256);
    }
  return 0;
}
