// Shared-memory radix-2 FFT over rows (used by the load stage and by Step 2).
#pragma once
#include <cuda_runtime.h>

namespace ftk {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// In-place forward DFT X[q] = sum_p x[p] e^{-2 pi i p q / n} of `nr` length-n rows stored
// contiguously in shared memory (iterative radix-2 DIT, bit-reversed input).  tw[j] = e^{-2 pi i j/n}.
__device__ __forceinline__ void smem_fft_rows(float2* s, int nr, int n, int logn, const float2* tw) {
  const int tot = nr << logn;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    const int r = idx >> logn, p = idx & (n - 1);
    const int rp = __brev(p) >> (32 - logn);
    if (rp > p) {
      float2 t = s[(r << logn) + p];
      s[(r << logn) + p] = s[(r << logn) + rp];
      s[(r << logn) + rp] = t;
    }
  }
  __syncthreads();
  const int halfn = n >> 1;
  for (int lh = 0; lh < logn; ++lh) {
    const int half = 1 << lh;
    const int tot2 = nr * halfn;
    for (int idx = threadIdx.x; idx < tot2; idx += blockDim.x) {
      const int r = idx >> (logn - 1);
      const int b = idx & (halfn - 1);
      const int j = b & (half - 1);
      const int k = (b >> lh) << (lh + 1);
      const float2 w = tw[j << (logn - 1 - lh)];
      float2* row = s + (r << logn);
      const float2 u = row[k + j];
      const float2 v = cmul(row[k + j + half], w);
      row[k + j] = make_float2(u.x + v.x, u.y + v.y);
      row[k + j + half] = make_float2(u.x - v.x, u.y - v.y);
    }
    __syncthreads();
  }
}

}  // namespace ftk
