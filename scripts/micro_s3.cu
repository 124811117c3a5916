// Microbenchmark of the Step-3 MMA issue pattern in isolation (no epilogue): per chunk 3 x (K3p/16)
// tcgen05.mma kind::f16 M128 x N x K16 with A from TMEM (hi/lo slots) and B from SMEM (hi/lo parts, the
// canonical K-major no-swizzle layout [part][row/8][K3p/8][8 rows x 16 B]), E/O accumulators split at Ke,
// one commit per chunk, double-buffered D.  Variants: B fixed vs walking the chunk; 1 vs 3 products.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/micro_s3 scripts/micro_s3.cu
#include <cstdio>
#include <cstring>

#include "../paper_1905_12317_b200/csrc/ftk_sm100.cuh"

using namespace ftk::sm100;

__device__ __forceinline__ void cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

__device__ __forceinline__ void wait_mode(uint64_t* bar, uint32_t parity, int mode) {
  if (mode == 0) {
    mbar_wait(bar, parity);
  } else if (mode == 1) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(a), "r"(parity) : "memory");
  } else {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(a), "r"(parity) : "memory");
  }
}

__global__ void __launch_bounds__(288, 1) k_s3(int chunks, int N, int K3p, int Ke, int nch, int prods, int bfixed,
                                               int wmode, int NB, int flags, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncol = N * nch;
  const uint32_t ypart = (uint32_t)ncol * K3p * 2;
  for (int i = threadIdx.x; i < (int)(2 * ypart / 4); i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  {  // A slots (columns [2 NB N, 512)) = bf16 1.0 pairs, written by the 4 warps (one TMEM lane quarter each)
    const uint32_t a0 = 2u * NB * N;
    for (uint32_t c = a0; c + 4 <= 512; c += 4)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) + c),
                   "r"(0x3f803f80u) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (warp >= 1 && (flags & 8192)) {  // TMEM loader warps: 8 warps (two per lane quarter) read D-buffer columns
    const int q = warp & 3, hh = (warp - 1) >> 2;
    uint32_t acc = 0;
    for (int it = 0; it < chunks; ++it) {
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((it & 1) * 2 * N + hh * (N / 2));
      uint32_t r[16];
      for (int c0 = 0; c0 + 16 <= N / 2; c0 += 16) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(base + c0));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(base + N + c0));
        tmem_wait_ld();
        for (int k = 0; k < 16; ++k) acc ^= r[k];
      }
    }
    if (acc == 0x12345u) cyc[296] = acc;
  }
  if (warp == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint32_t SBO = (uint32_t)K3p * 16u;
    const uint32_t ybase = smem_u32(sm);
    const int ksteps = K3p / 16, ke = Ke / 16, halfk = K3p / 2;
    const uint32_t a_hi0 = tmem + 2u * NB * N;
    const unsigned long long t0 = clock64();
    if (((flags >> 3) & 7) >= 4) {  // the micro_tc loop: constant operands, back-to-back, one final commit
      const uint64_t bd = smem_desc_kmajor_noswz(ybase, 128, ((flags >> 3) & 7) == 4 ? 256u : SBO);
      const int v = (flags >> 7) & 7;  // 0 constant; 1 D alternates; 2 B alternates; 3 acc alternates; 4 A alternates
      if (elect_one()) {
        for (int c = 0; c < chunks; ++c) {
          const uint32_t alt = (uint32_t)(c & 1);
          const uint32_t dd = tmem + ((v == 1) ? alt * (uint32_t)N : 0u);
          const uint64_t bb = bd + ((v == 2) ? (uint64_t)(alt * 16) : 0ull);
          const uint32_t ac = (v == 3) ? alt : (c > 0 ? 1u : 0u);
          const uint32_t aa = a_hi0 + ((v == 4) ? alt * 8u : 0u);
          mma_f16_ts(dd, aa, bb, idesc, ac);
        }
        tc_commit(&bar[0]);
      }
      __syncwarp();
      mbar_wait(&bar[0], 0);
      if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
    } else if (flags & 1024) {  // compile-time 6 k-steps x 3 products, fully unrolled, NB = 2, running counters
      if (elect_one()) {
        int cc = 0;
        for (int c = 0; c < chunks; ++c) {
          const uint32_t db = (uint32_t)(c & 1);
          if (c >= 2 && !(flags & 4)) mbar_wait(&bar[db], (uint32_t)(((c >> 1) - 1) & 1));
          tc_fence_after();
          if ((flags & 16384) && c % 5 == 0) {  // A slot refill per "r-tile" (every 5 chunks), 2 parts x 6 cp
            const uint32_t slot = a_hi0 + (uint32_t)(((c / 5) & 1) * 96);
            for (int part = 0; part < 2; ++part)
              for (int j = 0; j < 6; ++j)
                cp_128x256b(slot + (uint32_t)(part * 48 + 8 * j), smem_desc_kmajor_noswz(ybase + part * 24576 + j * 256, 128, SBO));
          }
          const uint32_t dE = tmem + db * 2u * (uint32_t)N, dO = dE + (uint32_t)N;
          const uint32_t bch = ybase + (uint32_t)(cc * (N / 8)) * SBO;
          cc = (cc + 1 == nch) ? 0 : cc + 1;
          const uint64_t bh0 = smem_desc_kmajor_noswz(bch, 128, SBO);
          const uint64_t bl0 = smem_desc_kmajor_noswz(bch + ypart, 128, SBO);
#pragma unroll
          for (int ks = 0; ks < 6; ++ks) {
            const int kev = (flags & 2048) ? ke : 3;
            const uint32_t d = ks >= kev ? dO : dE;
            const uint32_t acc0 = (ks == 0 || ks == kev) ? 0u : 1u;
            const uint32_t a_hi = a_hi0 + (uint32_t)(ks * 8), a_lo = a_hi + 48u;
            mma_f16_ts(d, a_hi, bh0 + (uint64_t)(ks * 16), idesc, acc0);
            mma_f16_ts(d, a_hi, bl0 + (uint64_t)(ks * 16), idesc, 1u);
            mma_f16_ts(d, a_lo, bh0 + (uint64_t)(ks * 16), idesc, 1u);
          }
          tc_commit(&bar[db]);
        }
        mbar_wait(&bar[(chunks - 1) & 1], (uint32_t)(((chunks - 1) >> 1) & 1));
        mbar_wait(&bar[(chunks - 2) & 1], (uint32_t)(((chunks - 2) >> 1) & 1));
      }
      __syncwarp();
      if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
    } else if (flags & 64) {  // one elected lane runs the whole chunk loop (no per-chunk elect / syncwarp)
      if (elect_one()) {
        for (int c = 0; c < chunks; ++c) {
          const int db = c % NB;
          if (c >= NB && !(flags & 4)) mbar_wait(&bar[db], ((c / NB) - 1) & 1);
          if (!(flags & 1)) tc_fence_after();
          const uint32_t dE = tmem + (uint32_t)(db * 2 * N), dO = dE + (uint32_t)N;
          const int cc = bfixed ? 0 : (c % nch);
          const uint32_t bch = ybase + (uint32_t)(cc * (N / 8)) * SBO;
          const uint64_t bh0 = smem_desc_kmajor_noswz(bch, 128, SBO);
          const uint64_t bl0 = smem_desc_kmajor_noswz(bch + ypart, 128, SBO);
#pragma unroll 1
          for (int ks = 0; ks < ksteps; ++ks) {
            const bool odd = ks >= ke;
            uint32_t d = odd ? dO : dE;
            uint32_t acc0 = (odd ? ks > ke : ks > 0) ? 1u : 0u;
            const int dm = (flags >> 3) & 7;
            if (dm == 1) { d = tmem; acc0 = 1u; }
            if (dm == 2) { d = tmem; }
            if (dm == 3) { acc0 = 1u; }
            const uint32_t a_hi = a_hi0 + (uint32_t)(ks * 8), a_lo = a_hi + (uint32_t)halfk;
            const uint64_t b_hi = bh0 + (uint64_t)(ks * 16), b_lo = bl0 + (uint64_t)(ks * 16);
            mma_f16_ts(d, a_hi, b_hi, idesc, acc0);
            if (prods > 1) {
              mma_f16_ts(d, a_hi, b_lo, idesc, 1u);
              mma_f16_ts(d, a_lo, b_hi, idesc, 1u);
            }
          }
          if (!(flags & 2) || c >= chunks - NB) tc_commit(&bar[db]);
        }
        for (int c = chunks - NB; c < chunks; ++c) mbar_wait(&bar[c % NB], (flags & 2) ? 0u : (uint32_t)((c / NB) & 1));
      }
      __syncwarp();
      if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
    } else {
    for (int c = 0; c < chunks; ++c) {
      const int db = c % NB;
      if (c >= NB && !(flags & 4)) wait_mode(&bar[db], ((c / NB) - 1) & 1, wmode);  // D buffer db free
      if (!(flags & 1)) tc_fence_after();
      const uint32_t dE = tmem + (uint32_t)(db * 2 * N), dO = dE + (uint32_t)N;
      const int cc = bfixed ? 0 : (c % nch);
      const uint32_t bch = ybase + (uint32_t)(cc * (N / 8)) * SBO;
      const uint64_t bh0 = smem_desc_kmajor_noswz(bch, 128, SBO);
      const uint64_t bl0 = smem_desc_kmajor_noswz(bch + ypart, 128, SBO);
      if (elect_one()) {
      for (int ks = 0; ks < ksteps; ++ks) {
        const bool odd = ks >= ke;
        uint32_t d = odd ? dO : dE;
        uint32_t acc0 = (odd ? ks > ke : ks > 0) ? 1u : 0u;
        const int dm = (flags >> 3) & 7;  // 0: as Step 3; 1: one D, always accumulate; 2: one D, init per chunk;
                                    // 3: Step-3 D switching, always accumulate
        if (dm == 1) { d = tmem; acc0 = 1u; }
        if (dm == 2) { d = tmem; }
        if (dm == 3) { acc0 = 1u; }
        const uint32_t a_hi = a_hi0 + (uint32_t)(ks * 8), a_lo = a_hi + (uint32_t)halfk;
        const uint64_t b_hi = bh0 + (uint64_t)(bfixed ? 0 : ks * 16), b_lo = bl0 + (uint64_t)(bfixed ? 0 : ks * 16);
        mma_f16_ts(d, a_hi, b_hi, idesc, acc0);
        if (prods > 1) {
          mma_f16_ts(d, a_hi, b_lo, idesc, 1u);
          mma_f16_ts(d, a_lo, b_hi, idesc, 1u);
        }
      }
      if (!(flags & 2) || c >= chunks - NB) tc_commit(&bar[db]);
      }
      __syncwarp();
    }
    for (int c = chunks - NB; c < chunks; ++c) mbar_wait(&bar[c % NB], (flags & 2) ? 0u : (uint32_t)((c / NB) & 1));
    if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem));
    tmem_wait_ld();
    if (lane == 0) cyc[148 + blockIdx.x] = r[0];
    tc_fence_before();
    __syncwarp();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 300 * sizeof(unsigned long long));
  unsigned long long h[296];
  const int K3p = 96, chunks = 2000;
  struct Cfg { int N, NB, prods, ks, flags, bfixed; };
  // flags: 1 = no fence::after_thread_sync, 2 = no per-chunk commit (only the last NB), 4 = no wait
  // dm (flags bits 3-5): 1 one D always accumulate; 2 one D, reset per chunk; 3 switching D, always accumulate
  const Cfg cfgs[] = {{80, 2, 3, 6, 1024, 0}, {80, 2, 3, 6, 1024 | 16384, 0}, {80, 2, 3, 6, 1024 | 16384 | 8192, 0}};
  for (const Cfg& c : cfgs) {
    const int N = c.N, nch = 400 / N + 1;
    const int K3 = 16 * c.ks;
    const size_t smem = (size_t)2 * N * nch * K3p * 2;
    cudaFuncSetAttribute(k_s3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_s3<<<148, (c.flags & 8192) ? 288 : 128, smem>>>(chunks, N, K3, K3 / 2 > 16 ? (K3 / 32) * 16 : K3, nch, c.prods, c.bfixed, 1, c.NB, c.flags, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("err %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const int mmas = c.prods * c.ks;
    float dv;
    { uint32_t u = (uint32_t)h[148]; memcpy(&dv, &u, 4); }
    printf("N=%2d buffers=%d MMAs/chunk=%2d flags=%d bfixed=%d: D[0][0] = %g; %.0f cycles/chunk = %.1f cycles/MMA\n", N,
           c.NB, mmas, c.flags, c.bfixed, dv,
           (double)h[0] / chunks, (double)h[0] / chunks / mmas);
  }
  return 0;
}
