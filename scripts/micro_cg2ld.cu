// TMEM load throughput from 8 warps per CTA while the tensor core runs back-to-back MMAs (A from TMEM, N = 80):
// cta_group::1 (one CTA per SM issuing its own M128 MMAs) vs cta_group::2 (CTA pair, the even CTA issuing
// M256 MMAs for both).  Reports LDTM bytes/cycle/SM and cycles per MMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/micro_cg2ld scripts/micro_cg2ld.cu
#include <cstdio>
#include "../paper_1905_12317_b200/csrc/ftk_tc_dev.cuh"
using namespace ftk;

template <int CG>
__global__ void __launch_bounds__(288, 1) k(int mma_iters, int ld_iters, unsigned long long* cyc) {
  __shared__ __align__(1024) uint8_t sb[80 * 16 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  for (int i = threadIdx.x; i < (int)sizeof(sb) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sb)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (CG == 2) tmem_alloc_cg2<512>(&tb); else tmem_alloc<512>(&tb);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync_all();
  tc_fence_after();
  const uint32_t tm = tb;
  const unsigned long long t0 = clock64();
  if (warp == 0) {
    if (rank == 0 && mma_iters > 0 && elect_one()) {
      const uint32_t idesc = idesc_bf16_f32(128 * CG, 80);
      const uint64_t bd = smem_desc_kmajor_noswz(smem_u32(sb), 128, 256);
      for (int i = 0; i < mma_iters; ++i) {
        if (CG == 2) mma_f16_ts_cg2(tm, tm + 400, bd, idesc, 1u);
        else mma_f16_ts(tm, tm + 400, bd, idesc, 1u);
      }
      if (CG == 2) tc_commit_cg2(&bar); else tc_commit(&bar);
    }
    __syncwarp();
    if (mma_iters > 0) mbar_wait(&bar, 0);
    if (lane == 0) cyc[blockIdx.x * 2] = clock64() - t0;
  } else {
    const int q = warp & 3;
    uint32_t acc = 0;
    for (int it = 0; it < ld_iters; ++it) {
      uint32_t r[16];
      tmem_ld16(tm + ((uint32_t)(q * 32) << 16) + 160u + (uint32_t)((it * 16 + (warp >> 2) * 64) % 224), r);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) acc ^= r[j];
    }
    if (acc == 0x1234567u) cyc[1000] = acc;
    if (lane == 0 && warp == 1) cyc[blockIdx.x * 2 + 1] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_cg2<512>(tm); else tmem_dealloc<512>(tm);
  }
}

template <int CG>
void run(int mi, int li) {
  unsigned long long* d;
  cudaMalloc(&d, 2048 * 8);
  cudaMemset(d, 0, 2048 * 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(288);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k<CG>, mi, li, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  unsigned long long h[4];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const double ldb = 8.0 * li * 32 * 16 * 4;
  printf("cg%d mma %5d ld %5d: mma %.1f cyc/MMA | ld CTA0 %.1f B/cyc, CTA1 %.1f B/cyc (cycles %llu %llu)\n", CG, mi, li,
         mi ? (double)h[0] / mi : 0.0, li ? ldb / h[1] : 0.0, li ? ldb / h[3] : 0.0, h[1], h[3]);
  cudaFree(d);
}

int main() {
  for (int cg : {1, 2}) {
    for (auto p : {std::make_pair(4000, 0), std::make_pair(0, 2000), std::make_pair(4000, 2000), std::make_pair(4000, 8000)}) {
      if (cg == 1) run<1>(p.first, p.second); else run<2>(p.first, p.second);
    }
  }
  return 0;
}
