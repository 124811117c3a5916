// SIMT (CUDA-core fp32) kernels of the FTK hot path: the ring FFT used by the load stage and the
// Step-2 FFT, plus straightforward reference versions of Steps 1 and 3 (engine = 1) and the small
// bookkeeping kernels (finalize / merge / export).  The tensor-core engine lives in ftk_tc.cu.
//
// Steps follow PAPER.md Eq. (fbk3), with cyclic q (reading R5) and the
// real-image reduction to ell >= 0 terms (reading R13).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ftk_fft.cuh"
#include "ftk_internal.cuh"

namespace ftk {

// ---------------------------------------------------------------- load: ring FFT
// a(k_m; q) = (1/n_psi) sum_p Ahat(k_m, psi_p) e^{-2 pi i p q / n_psi}   (Eq. aqkcalc)
// in : polar [item][m][p] (p fastest);  out: fb [item][q][m] (m fastest: the Step-1 K-major operand).
__global__ void __launch_bounds__(256) k_ring_fft(const float2* __restrict__ polar, float2* __restrict__ fb, int n_k,
                                                  int n, int logn, int RB, const float2* __restrict__ tw) {
  extern __shared__ float2 sm_fft[];
  float2* tws = sm_fft + (size_t)RB * n;
  const int64_t item = blockIdx.x;
  const int m0 = blockIdx.y * RB;
  const int nr = min(RB, n_k - m0);
  for (int i = threadIdx.x; i < n / 2; i += blockDim.x) tws[i] = tw[i];
  const float2* src = polar + (item * n_k + m0) * (int64_t)n;
  for (int idx = threadIdx.x; idx < nr * n; idx += blockDim.x) sm_fft[idx] = src[idx];
  __syncthreads();
  smem_fft_rows(sm_fft, nr, n, logn, tws);
  const float inv = 1.0f / (float)n;
  float2* dst = fb + item * (int64_t)n * n_k;
  for (int idx = threadIdx.x; idx < nr * n; idx += blockDim.x) {
    const int q = idx / nr, rr = idx - q * nr;
    const float2 v = sm_fft[rr * n + q];
    dst[(int64_t)q * n_k + m0 + rr] = make_float2(v.x * inv, v.y * inv);
  }
}

static int ring_rows_per_block(int n_k, int n) {
  int rb = 8192 / n;
  if (rb < 1) rb = 1;
  if (rb > n_k) rb = n_k;
  return rb;
}

void launch_ring_fft(const float2* polar, float2* fb, int64_t n_items, const DevPlan& P, cudaStream_t s) {
  if (n_items <= 0) return;
  const int rb = ring_rows_per_block(P.n_k, P.n_psi);
  const size_t smem = ((size_t)rb * P.n_psi + P.n_psi / 2) * sizeof(float2);
  FTK_SMEM_OPTIN(k_ring_fft);
  dim3 grid((unsigned)n_items, (P.n_k + rb - 1) / rb);
  k_ring_fft<<<grid, 256, smem, s>>>(polar, fb, P.n_k, P.n_psi, P.log2_psi, rb, P.tw);
}

// ---------------------------------------------------------------- Step 1 (SIMT reference)
// Zhat_zeta(q) = sum_m g_zeta(m) a(m, q - ell_zeta) conj b(m, q),  g = 2 pi w G   (Eq. fbk3 Step 1)
// Zhat layout: [pair][zeta+][q] complex.
constexpr int S1_QC = 32;

__global__ void __launch_bounds__(256) k_step1_simt(const float2* __restrict__ A, const float2* __restrict__ B,
                                                    float2* __restrict__ Zhat, PairBlock pb, DevPlan P) {
  extern __shared__ float4 sm1_raw[];
  const int nk = P.n_k, n = P.n_psi, L = P.ell_max, Hp = P.H_plus, st = nk + 1;
  float2* bs = reinterpret_cast<float2*>(sm1_raw);
  float2* as = bs + S1_QC * st;
  float* gs = reinterpret_cast<float*>(as + (S1_QC + L) * st);
  int* ls = reinterpret_cast<int*>(gs + Hp * nk);
  const int p = blockIdx.x, q0 = blockIdx.y * S1_QC;
  int i, j;
  pair_of(pb, p, i, j);
  const float2* Ai = A + (int64_t)i * n * nk;
  const float2* Bj = B + (int64_t)j * n * nk;
  for (int idx = threadIdx.x; idx < S1_QC * nk; idx += blockDim.x) {
    const int qq = idx / nk, m = idx - qq * nk;
    bs[qq * st + m] = Bj[(int64_t)((q0 + qq) & (n - 1)) * nk + m];
  }
  for (int idx = threadIdx.x; idx < (S1_QC + L) * nk; idx += blockDim.x) {
    const int rr = idx / nk, m = idx - rr * nk;
    const int q = (q0 - L + rr + n) & (n - 1);
    as[rr * st + m] = Ai[(int64_t)q * nk + m];
  }
  for (int idx = threadIdx.x; idx < Hp * nk; idx += blockDim.x) gs[idx] = P.g[idx];
  for (int idx = threadIdx.x; idx < Hp; idx += blockDim.x) ls[idx] = P.ell[idx];
  __syncthreads();
  for (int o = threadIdx.x; o < Hp * S1_QC; o += blockDim.x) {
    const int z = o / S1_QC, qq = o - z * S1_QC;
    const int l = ls[z];
    const float2* ar = as + (qq + L - l) * st;
    const float2* br = bs + qq * st;
    const float* gr = gs + z * nk;
    float re = 0.f, im = 0.f;
    for (int m = 0; m < nk; ++m) {
      const float2 a = ar[m], b = br[m];
      const float g = gr[m];
      re = fmaf(g, a.x * b.x + a.y * b.y, re);
      im = fmaf(g, a.y * b.x - a.x * b.y, im);
    }
    Zhat[((int64_t)p * Hp + z) * n + q0 + qq] = make_float2(re, im);
  }
}

void launch_step1_simt(const float2* A, const float2* B, float2* Zhat, const PairBlock& pb, const DevPlan& P,
                       cudaStream_t s) {
  const int st = P.n_k + 1;
  const size_t smem = (size_t)(S1_QC + S1_QC + P.ell_max) * st * sizeof(float2) + (size_t)P.H_plus * P.n_k * 4 +
                      (size_t)P.H_plus * 4;
  FTK_SMEM_OPTIN(k_step1_simt);
  dim3 grid(pb.count, P.n_psi / S1_QC);
  k_step1_simt<<<grid, 256, smem, s>>>(A, B, Zhat, pb, P);
}

// ---------------------------------------------------------------- Step 2 (FFT over q)
// Z_zeta(r) = sum_q Zhat_zeta(q) e^{-2 pi i q r / n_psi}   (Eq. fbk3 Step 2, forward sign, reading R11)
// Output Z3 [pair][K3p][n_psi] real rows: ell = 0 -> Re Z; ell > 0 -> (Re Z, Im Z)  (reading R13).
constexpr int S2_ZB = 8;

__global__ void __launch_bounds__(256) k_step2_simt(const float2* __restrict__ Zhat, float* __restrict__ Z3,
                                                    PairBlock pb, DevPlan P) {
  extern __shared__ float2 sm2[];
  const int n = P.n_psi, Hp = P.H_plus;
  float2* tws = sm2 + S2_ZB * n;
  const int p = blockIdx.x, z0 = blockIdx.y * S2_ZB;
  const int nz = min(S2_ZB, Hp - z0);
  for (int i = threadIdx.x; i < n / 2; i += blockDim.x) tws[i] = P.tw[i];
  const float2* src = Zhat + ((int64_t)p * Hp + z0) * n;
  for (int idx = threadIdx.x; idx < nz * n; idx += blockDim.x) sm2[idx] = src[idx];
  __syncthreads();
  smem_fft_rows(sm2, nz, n, P.log2_psi, tws);
  float* dst = Z3 + (int64_t)p * P.K3p * n;
  if (blockIdx.y == 0) {  // zero the K padding rows (the region's offset moves with the block size)
    for (int idx = threadIdx.x; idx < P.npads * n; idx += blockDim.x)
      dst[(int64_t)P.pads[idx / n] * n + idx % n] = 0.f;
  }
  for (int idx = threadIdx.x; idx < nz * n; idx += blockDim.x) {
    const int z = idx / n, r = idx - z * n;
    const int c = P.col[z0 + z];
    const float2 v = sm2[idx];
    dst[(int64_t)c * n + r] = v.x;
    if (P.ell[z0 + z] > 0) dst[(int64_t)(c + 1) * n + r] = v.y;
  }
}

void launch_step2_simt(const float2* Zhat, float* Z3, const PairBlock& pb, const DevPlan& P, cudaStream_t s) {
  const size_t smem = ((size_t)S2_ZB * P.n_psi + P.n_psi / 2) * sizeof(float2);
  FTK_SMEM_OPTIN(k_step2_simt);
  dim3 grid(pb.count, (P.H_plus + S2_ZB - 1) / S2_ZB);
  k_step2_simt<<<grid, 256, smem, s>>>(Zhat, Z3, pb, P);
}

// ---------------------------------------------------------------- Step 3 (SIMT reference) + argmax
// X(t, r) = sum_k' Y3[t][k'] Z3[k'][r]  (= Re sum_zeta Y_zeta Z_zeta, Eq. fbk3 Step 3), max/argmax fused.
constexpr int S3_T = 64, S3_R = 64;

__global__ void __launch_bounds__(256) k_step3_simt(const float* __restrict__ Z3, PairBlock pb, DevPlan P, int tm_off,
                                                    unsigned long long* __restrict__ img_keys,
                                                    unsigned long long* __restrict__ pair_keys, int n_tm_local,
                                                    float* __restrict__ land) {
  extern __shared__ float4 sm3_raw[];
  float* Zs = reinterpret_cast<float*>(sm3_raw);   // [K3p][S3_R]
  float* Ys = Zs + P.K3p * S3_R;                   // [K3p][S3_T]
  const int n = P.n_psi, K = P.K3p, Nt = P.N_t;
  const int p = blockIdx.x, r0 = blockIdx.y * S3_R;
  int i, j;
  pair_of(pb, p, i, j);
  const float* zsrc = Z3 + (int64_t)p * K * n;
  for (int idx = threadIdx.x; idx < K * S3_R; idx += blockDim.x) {
    const int k = idx / S3_R, rr = idx - k * S3_R;
    Zs[idx] = zsrc[(int64_t)k * n + r0 + rr];
  }
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float best_v = -INFINITY;
  uint32_t best_f = 0xffffffffu;
  for (int t0 = 0; t0 < Nt; t0 += S3_T) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < K * S3_T; idx += blockDim.x) {
      const int tt = idx / K, k = idx - tt * K;
      Ys[k * S3_T + tt] = (t0 + tt < Nt) ? P.Y3[(int64_t)(t0 + tt) * K + k] : 0.f;
    }
    __syncthreads();
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    for (int k = 0; k < K; ++k) {
      const float4 y = *reinterpret_cast<const float4*>(&Ys[k * S3_T + ty * 4]);
      const float4 z = *reinterpret_cast<const float4*>(&Zs[k * S3_R + tx * 4]);
      const float yy[4] = {y.x, y.y, y.z, y.w}, zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(yy[a], zz[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int t = t0 + ty * 4 + a;
      if (t >= Nt) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int r = r0 + tx * 4 + b;
        const float v = acc[a][b];
        const uint32_t f = (uint32_t)t * (uint32_t)n + (uint32_t)r;
        if (v > best_v || (v == best_v && f < best_f)) {
          best_v = v;
          best_f = f;
        }
        if (land) land[((int64_t)p * Nt + t) * n + r] = v;
      }
    }
  }
  // block reduction of (value, flat) with the lexicographic tie-break
  __shared__ float rv[256];
  __shared__ uint32_t rf[256];
  rv[threadIdx.x] = best_v;
  rf[threadIdx.x] = best_f;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const float v2 = rv[threadIdx.x + s];
      const uint32_t f2 = rf[threadIdx.x + s];
      if (v2 > rv[threadIdx.x] || (v2 == rv[threadIdx.x] && f2 < rf[threadIdx.x])) {
        rv[threadIdx.x] = v2;
        rf[threadIdx.x] = f2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && rf[0] != 0xffffffffu) {
    const uint32_t t = rf[0] / n, r = rf[0] - t * n;
    const uint32_t gflat = ((uint32_t)(tm_off + j) * (uint32_t)Nt + t) * (uint32_t)n + r;
    const unsigned long long key = pack_key(rv[0], gflat);
    if (img_keys) atomicMax(&img_keys[i], key);
    if (pair_keys) atomicMax(&pair_keys[(int64_t)i * n_tm_local + j], key);
  }
}

void launch_step3_simt(const float* Z3, const PairBlock& pb, const DevPlan& P, int tm_offset,
                       unsigned long long* img_keys, unsigned long long* pair_keys, int n_tm_local, float* landscape,
                       cudaStream_t s) {
  const size_t smem = (size_t)P.K3p * (S3_R + S3_T) * sizeof(float);
  FTK_SMEM_OPTIN(k_step3_simt);
  dim3 grid(pb.count, P.n_psi / S3_R);
  k_step3_simt<<<grid, 256, smem, s>>>(Z3, pb, P, tm_offset, img_keys, pair_keys, n_tm_local, landscape);
}

// ---------------------------------------------------------------- bookkeeping
__global__ void k_finalize(const unsigned long long* __restrict__ keys, int64_t n, int N_t, int n_psi,
                           ftk_best_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i];
  ftk_best_t b;
  if (k == 0ull) {
    b.value = -INFINITY;
    b.template_idx = b.shift_idx = b.rot_idx = -1;
  } else {
    b.value = ord_float((uint32_t)(k >> 32));
    const uint32_t flat = 0xffffffffu - (uint32_t)(k & 0xffffffffull);
    b.rot_idx = (int32_t)(flat % (uint32_t)n_psi);
    const uint32_t rest = flat / (uint32_t)n_psi;
    b.shift_idx = (int32_t)(rest % (uint32_t)N_t);
    b.template_idx = (int32_t)(rest / (uint32_t)N_t);
  }
  out[i] = b;
}

void launch_finalize(const unsigned long long* keys, int64_t n, int N_t, int n_psi, ftk_best_t* out, cudaStream_t s) {
  if (n <= 0) return;
  k_finalize<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(keys, n, N_t, n_psi, out);
}

__global__ void k_merge(const ftk_best_t* __restrict__ g, int world, int64_t n, ftk_best_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  ftk_best_t b = g[i];
  for (int r = 1; r < world; ++r) {
    const ftk_best_t c = g[(int64_t)r * n + i];
    if (best_better(c, b)) b = c;
  }
  out[i] = b;
}

void launch_merge(const ftk_best_t* gathered, int world, int64_t n, ftk_best_t* out, cudaStream_t s) {
  if (n <= 0) return;
  k_merge<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(gathered, world, n, out);
}

__global__ void k_fb_export(const float2* __restrict__ fb, int64_t first, int64_t count, int n_k, int n_psi,
                            float2* __restrict__ out) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)n_k * n_psi;
  if (idx >= count * per) return;
  const int64_t it = idx / per;
  const int rem = (int)(idx - it * per);
  const int m = rem / n_psi, q = rem - m * n_psi;
  out[idx] = fb[(first + it) * per + (int64_t)q * n_k + m];
}

void launch_fb_export(const float2* fb, int64_t first, int64_t count, int n_k, int n_psi, float2* out, cudaStream_t s) {
  const int64_t tot = count * n_k * n_psi;
  if (tot <= 0) return;
  k_fb_export<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(fb, first, count, n_k, n_psi, out);
}

}  // namespace ftk
