// Microbenchmarks of the sm_100a resources the FTK Step-3 kernel is bound by (run on a B200):
//   (1) TMEM -> register load throughput (tcgen05.ld 32x32b.x16 / x32) with 4 / 8 / 16 warps per SM;
//   (2) back-to-back tcgen05.mma kind::f16 (A from TMEM, B from SMEM) cycles per instruction vs N;
//   (3) (2) while 8 warps stream TMEM loads of other columns (interference).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o micro_tc scripts/micro_tc.cu
#include <cstdio>
#include <cstdlib>

#include "../paper_1905_12317_b200/csrc/ftk_sm100.cuh"

using namespace ftk::sm100;

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// (1) + (3): warps >= 1 stream TMEM loads; warp 0 lane 0 optionally issues MMAs into columns [0, 256)
template <int X>
__global__ void __launch_bounds__(544, 1) k_tmem(int iters, int mma_iters, int N, unsigned long long* cyc,
                                                  unsigned* sink) {
  __shared__ __align__(1024) uint8_t sb[256 * 16 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (int)sizeof(sb) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sb)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  const int nld = (blockDim.x >> 5) - 1;  // loader warps
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp == 0) {
    if (lane == 0 && mma_iters > 0) {
      const uint32_t idesc = idesc_bf16_f32(128, N);
      const uint64_t bd = smem_desc_kmajor_noswz(smem_u32(sb), 128, 256);
      for (int i = 0; i < mma_iters; ++i) mma_f16_ts(tm + 0, tm + 384, bd, idesc, i > 0 ? 1u : 0u);
      tc_commit(&bar);
      mbar_wait(&bar, 0);
      cyc[blockIdx.x * 2 + 1] = clock64() - t0;
    }
  } else {
    const int q = warp & 3;
    const int slot = (warp - 1) >> 2;  // which group of 4 warps
    const int nslots = nld / 4 > 0 ? nld / 4 : 1;
    uint32_t acc = 0;
    const uint32_t colbase = mma_iters > 0 ? 256u : 0u;  // avoid the MMA accumulator columns
    const uint32_t ncols = mma_iters > 0 ? 128u : 512u;
    for (int it = 0; it < iters; ++it) {
      for (uint32_t c = (uint32_t)slot * X; c < ncols; c += (uint32_t)nslots * X) {
        uint32_t r[32];
        if constexpr (X == 32) {
          tmem_ld32(tm + ((uint32_t)(q * 32) << 16) + colbase + c, r);
        } else {
          uint32_t r16[16];
          tmem_ld16(tm + ((uint32_t)(q * 32) << 16) + colbase + c, r16);
#pragma unroll
          for (int k = 0; k < 16; ++k) r[k] = r16[k];
        }
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < X; ++k) acc ^= r[k];
      }
    }
    if (acc == 0x12345678u) sink[0] = acc;
    __syncwarp();
    if (lane == 0 && warp == 1) cyc[blockIdx.x * 2] = clock64() - t0;
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
  cudaMalloc(&d, 148 * 2 * sizeof(unsigned long long));
  cudaMalloc(&sink, 4);
  unsigned long long h[296];
  const int iters = 200;
  for (int warps : {4, 8, 16}) {
    for (int x : {16, 32}) {
      cudaMemset(d, 0, sizeof h);
      if (x == 16)
        k_tmem<16><<<148, 32 * (warps + 1)>>>(iters, 0, 64, d, sink);
      else
        k_tmem<32><<<148, 32 * (warps + 1)>>>(iters, 0, 64, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("err %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      double bytes = (double)iters * 512 * 128 * 4;
      printf("TMEM ld x%d, %2d warps: %.1f B/cyc/SM (cycles %llu)\n", x, warps, bytes / h[0], h[0]);
    }
  }
  for (int N : {64, 80, 96, 128, 256}) {
    const int mi = 4000;
    cudaMemset(d, 0, sizeof h);
    k_tmem<32><<<148, 32>>>(0, mi, N, d, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("MMA M128 N%3d K16 (TS): %.2f cyc/instr (floor 128N/256 = %.1f); %.0f MAC/cyc/SM\n", N, (double)h[1] / mi,
           128.0 * N / 256, 128.0 * N * 16 * mi / h[1]);
    cudaMemset(d, 0, sizeof h);
    k_tmem<32><<<148, 32 * 9>>>(mi * N / 64 / 4, mi, N, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("err %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("   with 8 loader warps: MMA %.2f cyc/instr; loads %.1f B/cyc/SM\n", (double)h[1] / mi,
           (double)(mi * N / 64 / 4) * 128 * 128 * 4 / h[0]);
  }
  return 0;
}
