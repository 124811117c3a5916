// Standalone check of the Step-2 TMA tensor load: Zhat' [pair][p][Hs] (8-byte elements) as a 2-D tensor,
// 8 x box_rows boxes with SWIZZLE_64B into shared memory; verifies the swizzle formula s2_slot().
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/micro_tma scripts/micro_tma.cu
#include <cuda.h>
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_1905_12317_b200/csrc/ftk_sm100.cuh"
using namespace ftk::sm100;

__device__ __forceinline__ void tma_load_2d_(void* dst_smem, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst_smem)), "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}

__global__ void k(const __grid_constant__ CUtensorMap m, int n_in, int x0, int pair, unsigned long long* out, int* bad) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int box = n_in < 256 ? n_in : 256;
    mbar_arrive_expect_tx(&bar, (uint32_t)n_in * 64u);
    for (int k0 = 0; k0 < n_in; k0 += box) tma_load_2d_(sm + (size_t)k0 * 64, &m, x0, pair * n_in + k0, &bar);
  }
  mbar_wait(&bar, 0);
  const unsigned long long* v = reinterpret_cast<const unsigned long long*>(sm);
  for (int i = threadIdx.x; i < n_in * 8; i += blockDim.x) {
    const int p = i / 8, zz = i % 8;
    const int slot = p * 8 + ((((zz >> 1) ^ (p >> 1)) & 3) << 1) + (zz & 1);
    out[i] = v[slot];
  }
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const bool u32 = argc > 1 && std::strcmp(argv[1], "u32") == 0;  // 4-byte elements, x in floats
  printf("element: %s\n", u32 ? "UINT32 (box 16 x rows, x = 2 x0)" : "UINT64 (box 8 x rows)");
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  PFN enc = (PFN)fp;
  struct Case { int Hs, n_in, npair, x0, pair; };
  Case cases[] = {{16, 64, 16, 8, 3}, {34, 256, 100, 16, 7}, {20, 128, 240, 8, 100}, {64, 256, 50, 40, 9},
                  {50, 512, 40, 40, 33}, {50, 512, 40, 46, 39}, {20, 128, 1, 6, 0}, {20, 128, 1, 15, 0},
                  {64, 256, 1, 7, 0}, {64, 256, 1, 62, 0}, {34, 256, 1, 9, 0}, {20, 128, 1, 0, 0}};
  for (auto& c : cases) {
    const size_t ne = (size_t)c.npair * c.n_in * c.Hs;
    std::vector<unsigned long long> h(ne);
    for (size_t i = 0; i < ne; ++i) h[i] = i;
    unsigned long long *d, *o;
    cudaMalloc(&d, ne * 8);
    cudaMalloc(&o, c.n_in * 8 * 8);
    cudaMemcpy(d, h.data(), ne * 8, cudaMemcpyHostToDevice);
    alignas(64) CUtensorMap m;
    const cuuint64_t dims[2] = {(cuuint64_t)(u32 ? 2 * c.Hs : c.Hs), (cuuint64_t)c.npair * c.n_in};
    const cuuint64_t strides[1] = {(cuuint64_t)c.Hs * 8};
    const cuuint32_t box[2] = {u32 ? 16u : 8u, (cuuint32_t)(c.n_in < 256 ? c.n_in : 256)};
    const cuuint32_t es[2] = {1u, 1u};
    CUresult r = enc(&m, u32 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 256, c.n_in * 64>>>(m, c.n_in, u32 ? 2 * c.x0 : c.x0, c.pair, o, nullptr);
    cudaError_t e = cudaDeviceSynchronize();
    int bad = -1;
    if (e == cudaSuccess) {
      std::vector<unsigned long long> out(c.n_in * 8);
      cudaMemcpy(out.data(), o, out.size() * 8, cudaMemcpyDeviceToHost);
      bad = 0;
      for (int p = 0; p < c.n_in; ++p)
        for (int zz = 0; zz < 8; ++zz) {
          const int col = c.x0 + zz;
          const unsigned long long want = col < c.Hs ? ((size_t)c.pair * c.n_in + p) * c.Hs + col : 0ull;
          if (out[p * 8 + zz] != want) ++bad;
        }
    }
    printf("Hs=%d n_in=%d npair=%d x0=%d: encode=%d kernel=%s bad=%d\n", c.Hs, c.n_in, c.npair, c.x0, (int)r,
           cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
    cudaFree(d);
    cudaFree(o);
  }
  return 0;
}
