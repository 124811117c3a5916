// Microbenchmarks for the round-2 kernel designs (run on a B200):
//   (1) tcgen05.mma kind::f16 SS (both operands in shared memory) cycles/instruction for the K-major
//       layouts SWIZZLE_NONE / 32B / 64B / 128B, N = 96 / 128 / 256, plus a numerical check of each layout;
//   (2) TS (A in TMEM) with B in each layout, N = 128;
//   (3) cta_group::2 (CTA pair, M = 256, B split N/2 per CTA), TS and SS, with a numerical check;
//   (4) tcgen05.cp 128x256b throughput alone and interleaved with TS MMAs (N = 80);
//   (5) tcgen05.st from 8 warps concurrent with TS MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/micro_mma2 scripts/micro_mma2.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1905_12317_b200/csrc/ftk_sm100.cuh"
using namespace ftk::sm100;

// layout: 0 none (canonical core matrices, LBO = 128, SBO = K*16), 1 SW32, 2 SW64, 3 SW128
__host__ __device__ inline uint32_t lay_off(int layout, int r, int k, int R, int K) {
  if (layout == 0) return (uint32_t)((r / 8) * (K * 16) + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2);
  const int X = 16 << layout;  // 32, 64, 128 bytes per row of an atom
  const int AW = X / 2;         // atom width in bf16 elements
  uint32_t o = (uint32_t)((k / AW) * (R * X) + (r / 8) * (8 * X) + (r % 8) * X + (k % AW) * 2);
  const uint32_t m = (uint32_t)(X / 16 - 1);
  return o ^ (((o >> 7) & m) << 4);
}
__device__ __forceinline__ uint64_t make_desc(int layout, uint32_t saddr, int R, int K, int ks) {
  if (layout == 0) return smem_desc_kmajor_noswz(saddr + ks * 256, 128, K * 16);
  const int X = 16 << layout, AW = X / 2;
  const int k0 = ks * 16;
  const uint32_t a = saddr + (uint32_t)((k0 / AW) * (R * X) + (k0 % AW) * 2);
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(((8 * X) >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  const uint64_t lt = layout == 1 ? 6 : (layout == 2 ? 4 : 2);
  d |= lt << 61;
  return d;
}
__device__ __forceinline__ void mma_ss2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ts2(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)), "h"((uint16_t)3)
               : "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float hval(int r, int k, int salt) {  // small exact bf16 values
  const unsigned h = (unsigned)(r * 131 + k * 71 + salt * 29) * 2654435761u;
  return (float)((int)((h >> 20) % 9) - 4) * 0.25f;
}
static float hval_h(int r, int k, int salt) {
  const unsigned h = (unsigned)(r * 131 + k * 71 + salt * 29) * 2654435761u;
  return (float)((int)((h >> 20) % 9) - 4) * 0.25f;
}

constexpr int KK = 64;  // K extent of the operands (4 K16 steps)

// cg = 1 or 2; ts: A from TMEM; N = total N; writes D (rows of this CTA x N) if out != null (1 pass)
template <int CG>
__global__ void __launch_bounds__(128, 1) k_mma(int iters, int N, int layoutA, int layoutB, int ts, float* out,
                                                 unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = CG == 2 ? cta_rank() : 0;
  const int NB = N / CG;  // B rows held by this CTA
  uint8_t* sa = sm;
  uint8_t* sb = sm + 128 * KK * 2;
  for (int i = tid; i < 128 * KK; i += blockDim.x) {
    const int r = i / KK, k = i % KK;
    *reinterpret_cast<__nv_bfloat16*>(sa + lay_off(layoutA, r, k, 128, KK)) =
        __float2bfloat16(hval(r + 128 * (int)rank, k, 1));
  }
  for (int i = tid; i < NB * KK; i += blockDim.x) {
    const int r = i / KK, k = i % KK;
    *reinterpret_cast<__nv_bfloat16*>(sb + lay_off(layoutB, r, k, NB, KK)) =
        __float2bfloat16(hval(r + NB * (int)rank, k, 2));
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (CG == 1) {
      tmem_alloc<512>(&tb);
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tb)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tb;
  if (ts) {  // A -> TMEM columns [256, 256 + KK/2)
    const uint32_t base = tm + ((uint32_t)(warp * 32) << 16) + 256;
    uint32_t r16[16];
    for (int c0 = 0; c0 < KK / 2; c0 += 16) {
      for (int j = 0; j < 16; ++j) {
        __nv_bfloat162 h = __floats2bfloat162_rn(hval(tid + 128 * (int)rank, 2 * (c0 + j), 1),
                                                 hval(tid + 128 * (int)rank, 2 * (c0 + j) + 1, 1));
        r16[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      tmem_st16(base + c0, r16);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  if (warp == 0 && rank == 0) {
    const uint32_t idesc = idesc_bf16_f32(128 * CG, N);
    const unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ks = 0; ks < KK / 16; ++ks) {
          const uint64_t bd = make_desc(layoutB, smem_u32(sb), NB, KK, ks);
          const uint32_t acc = (it > 0 || ks > 0) ? 1u : 0u;
          if (ts) {
            if (CG == 1) mma_f16_ts(tm, tm + 256 + ks * 8, bd, idesc, acc);
            else mma_ts2(tm, tm + 256 + ks * 8, bd, idesc, acc);
          } else {
            const uint64_t ad = make_desc(layoutA, smem_u32(sa), 128, KK, ks);
            if (CG == 1) mma_f16_ss(tm, ad, bd, idesc, acc);
            else mma_ss2(tm, ad, bd, idesc, acc);
          }
        }
      }
      if (CG == 1) tc_commit(&bar); else commit2(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    if ((tid & 31) == 0 && cyc) cyc[blockIdx.x] = clock64() - t0;
  }
  if (CG == 2 && !(warp == 0 && rank == 0)) mbar_wait(&bar, 0);
  if (CG == 1 && warp != 0) mbar_wait(&bar, 0);
  tc_fence_after();
  if (out) {
    const uint32_t base = tm + ((uint32_t)(warp * 32) << 16);
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t r16[16];
      tmem_ld16(base + c0, r16);
      tmem_wait_ld();
      for (int e = 0; e < 16; ++e)
        out[((size_t)blockIdx.x * 128 + tid) * N + c0 + e] = __uint_as_float(r16[e]);
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (CG == 1) tmem_dealloc<512>(tm);
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

__device__ __forceinline__ void tc_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
// (4) cp throughput: per iteration ncp copies of 128 x 32 B (+ nmma TS MMAs N=80); (5) with nst > 0 warps 1..8
// streaming tcgen05.st x16 into columns [320, 512)
__global__ void __launch_bounds__(288, 1) k_cp(int iters, int ncp, int nmma, int nst, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tb);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tb;
  const unsigned long long t0 = clock64();
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16_f32(128, 80);
      const uint64_t bd = smem_desc_kmajor_noswz(smem_u32(sm) + 32768, 128, 256);
      for (int it = 0; it < iters; ++it) {
        for (int c = 0; c < ncp; ++c)
          tc_cp_128x256b(tm + 160 + (uint32_t)((c & 7) * 8), smem_desc_kmajor_noswz(smem_u32(sm) + (c & 7) * 4096, 128, 256));
        for (int m = 0; m < nmma; ++m) mma_f16_ts(tm, tm + 160 + (uint32_t)((m & 3) * 8), bd, idesc, 1u);
      }
      tc_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    if ((tid & 31) == 0) cyc[blockIdx.x * 2] = clock64() - t0;
  } else if (warp <= nst) {
    const int q = warp & 3;
    uint32_t r16[16];
    for (int j = 0; j < 16; ++j) r16[j] = (uint32_t)(tid * 16 + j);
    const int per = iters * 4;
    for (int it = 0; it < per; ++it) {
      const uint32_t col = 320u + (uint32_t)(((it * 2 + (warp >> 2)) & 11) * 16);
      tmem_st16(tm + ((uint32_t)(q * 32) << 16) + col, r16);
    }
    tmem_wait_st();
    if ((tid & 31) == 0 && warp == 1) cyc[blockIdx.x * 2 + 1] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tm);
  }
}

static int check(const char* what, int CG, int N, int la, int lb, int ts) {
  const int ctas = CG == 2 ? 2 : 1;
  float* d_out;
  cudaMalloc(&d_out, (size_t)ctas * 128 * N * 4);
  cudaMemset(d_out, 0, (size_t)ctas * 128 * N * 4);
  const size_t smem = 128 * KK * 2 + 256 * KK * 2;
  if (CG == 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_mma<2>, 1, N, la, lb, ts, d_out, (unsigned long long*)nullptr);
  } else {
    k_mma<1><<<1, 128, smem>>>(1, N, la, lb, ts, d_out, nullptr);
  }
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: CUDA error %s\n", what, cudaGetErrorString(e));
    exit(1);
  }
  std::vector<float> h((size_t)ctas * 128 * N);
  cudaMemcpy(h.data(), d_out, h.size() * 4, cudaMemcpyDeviceToHost);
  cudaFree(d_out);
  double mx = 0;
  for (int c = 0; c < ctas; ++c)
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < KK; ++k) ref += (double)hval_h(r + 128 * c, k, 1) * (double)hval_h(n, k, 2);
        mx = std::fmax(mx, std::fabs(ref - h[((size_t)c * 128 + r) * N + n]));
      }
  printf("check %-34s max|err| = %.3g %s\n", what, mx, mx < 1e-3 ? "OK" : "FAIL");
  return mx < 1e-3 ? 0 : 1;
}

static double run_mma(int CG, int N, int la, int lb, int ts, int iters) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaMemset(d, 0, 148 * 8);
  const size_t smem = 128 * KK * 2 + 256 * KK * 2;
  if (CG == 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_mma<2>, iters, N, la, lb, ts, (float*)nullptr, d);
  } else {
    k_mma<1><<<148, 128, smem>>>(iters, N, la, lb, ts, nullptr, d);
  }
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("run: CUDA error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (double)h[0] / (iters * (KK / 16));
}

int main() {
  cudaFuncSetAttribute(k_mma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  cudaFuncSetAttribute(k_mma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const char* ln[4] = {"none", "SW32", "SW64", "SW128"};
  int bad = 0;
  char buf[128];
  for (int l = 0; l < 4; ++l) {
    snprintf(buf, sizeof buf, "SS cg1 N=96 A,B %s", ln[l]);
    bad += check(buf, 1, 96, l, l, 0);
  }
  bad += check("TS cg1 N=128 B SW128", 1, 128, 0, 3, 1);
  bad += check("SS cg2 N=96 A,B SW64", 2, 96, 2, 2, 0);
  bad += check("SS cg2 N=128 A,B SW128", 2, 128, 3, 3, 0);
  bad += check("TS cg2 N=96 B SW64", 2, 96, 0, 2, 1);
  bad += check("TS cg2 N=128 B none", 2, 128, 0, 0, 1);
  if (bad) printf("%d layout checks FAILED\n", bad);
  const int iters = 2000;
  for (int N : {80, 96, 128, 256})
    for (int l = 0; l < 4; ++l)
      printf("SS cg1 M128 N%3d A,B %-5s: %6.1f cyc/MMA (floor %.0f)\n", N, ln[l], run_mma(1, N, l, l, 0, iters),
             128.0 * N / 256);
  for (int N : {80, 128})
    for (int l = 0; l < 4; ++l)
      printf("TS cg1 M128 N%3d B %-5s:   %6.1f cyc/MMA (floor %.0f)\n", N, ln[l], run_mma(1, N, 0, l, 1, iters),
             128.0 * N / 256);
  for (int N : {64, 96, 128, 160, 192, 256}) {
    printf("TS cg2 M256 N%3d B none : %6.1f cyc/MMA (M256: 2x the MACs of cg1 M128)\n", N, run_mma(2, N, 0, 0, 1, iters));
    printf("TS cg2 M256 N%3d B SW64 : %6.1f cyc/MMA\n", N, run_mma(2, N, 0, 2, 1, iters));
    printf("SS cg2 M256 N%3d SW64   : %6.1f cyc/MMA\n", N, run_mma(2, N, 2, 2, 0, iters));
    printf("SS cg2 M256 N%3d SW128  : %6.1f cyc/MMA\n", N, run_mma(2, N, 3, 3, 0, iters));
  }
  {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 16);
    cudaFuncSetAttribute(k_cp, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    unsigned long long h[296];
    struct Cfg { int ncp, nmma, nst; } cfgs[] = {{8, 0, 0}, {0, 18, 0}, {12, 18, 0}, {24, 18, 0}, {0, 18, 8}, {12, 18, 8}, {0, 0, 8}};
    for (auto c : cfgs) {
      const int it = 400;
      cudaMemset(d, 0, 148 * 16);
      k_cp<<<148, 288, 65536>>>(it, c.ncp, c.nmma, c.nst, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("k_cp error %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      printf("cp %2d x 4KB + %2d MMA N80 per iter, %d st warps: %7.1f cyc/iter", c.ncp, c.nmma, c.nst, (double)h[0] / it);
      if (c.ncp && !c.nmma) printf(" (cp %.1f B/cyc)", (double)c.ncp * 4096 * it / h[0]);
      if (c.nst) printf("; st %.1f B/cyc", (double)c.nst * it * 4 * 32 * 64 / (double)h[1]);
      printf("\n");
    }
  }
  return bad;
}
