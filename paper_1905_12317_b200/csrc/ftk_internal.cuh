// Internal device-side declarations shared by the FTK CUDA translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/ftk.h"

namespace ftk {

// A block of (image, template) pairs: either a dense rectangle [i0, i0+ni) x [j0, j0+nj)
// (pair p -> (i0 + p / nj, j0 + p % nj)) or an explicit list (li[p], lj[p]).
struct PairBlock {
  int i0, ni, j0, nj;
  const int32_t* li;
  const int32_t* lj;
  int count;
};

__host__ __device__ inline void pair_of(const PairBlock& b, int p, int& i, int& j) {
  if (b.li) {
    i = b.li[p];
    j = b.lj[p];
  } else {
    i = b.i0 + p / b.nj;
    j = b.j0 + p % b.nj;
  }
}

// Opt `func` into the device's full dynamic shared memory (227 KB on B200, minus its static shared
// memory) on the CURRENT device, once per (call site, device).  The attribute belongs to the function
// and the device, not to a plan, so it is never lowered to one plan's size (distinct plans, and plans
// on different devices, stay independent).  `done` is a per-call-site device bit mask.
inline void smem_optin(const void* func, unsigned long long& done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done & bit) return;
  int mx = 0;
  cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, func) != cudaSuccess) return;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, mx - (int)fa.sharedSizeBytes) ==
      cudaSuccess)
    done |= bit;
}
#define FTK_SMEM_OPTIN(f)                  \
  do {                                     \
    static unsigned long long done_ = 0;   \
    smem_optin((const void*)(f), done_);   \
  } while (0)

// Order-preserving float -> uint32 (larger float -> larger code).  -0.0 is mapped to +0.0 first, so the
// packed-key atomics order values exactly as best_better() / the in-kernel comparisons do (-0 == +0,
// ties broken by the index).
__host__ __device__ inline uint32_t float_ord(float f) {
  f = f + 0.0f;  // -0 + 0 = +0 (round to nearest)
  uint32_t u;
#ifdef __CUDA_ARCH__
  u = __float_as_uint(f);
#else
  __builtin_memcpy(&u, &f, 4);
#endif
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ inline float ord_float(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  float f;
#ifdef __CUDA_ARCH__
  f = __uint_as_float(u);
#else
  __builtin_memcpy(&f, &u, 4);
#endif
  return f;
}
// Packed argmax key: value in the high word, ~flat index in the low word, so atomicMax picks the
// largest value and, among equal values, the smallest flat index (lexicographic tie-break, reading R9).
__host__ __device__ inline unsigned long long pack_key(float v, uint32_t flat) {
  return ((unsigned long long)float_ord(v) << 32) | (unsigned long long)(0xffffffffu - flat);
}

// Is result a strictly better than b (value desc, then (template, shift, rot) asc)?
__host__ __device__ inline bool best_better(const ftk_best_t& a, const ftk_best_t& b) {
  if (a.template_idx < 0) return false;
  if (b.template_idx < 0) return true;
  const float va = (a.value != a.value) ? -INFINITY : a.value;
  const float vb = (b.value != b.value) ? -INFINITY : b.value;
  if (va != vb) return va > vb;
  if (a.template_idx != b.template_idx) return a.template_idx < b.template_idx;
  if (a.shift_idx != b.shift_idx) return a.shift_idx < b.shift_idx;
  return a.rot_idx < b.rot_idx;
}

// Device plan constants used by every engine.
struct DevPlan {
  int n_k, n_psi, log2_psi, N_t, H_plus, K3, K3p, ell_max;
  int n_gamma;           // rotations (Step-2 FFT length); >= n_psi, zero-padded sum (reading R21)
  int Hs;                // row stride (complex) of the engine-0 Step-1 output Zhat' [pair][p][Hs] (H_plus, even)
  int Ke;                // even-ell column block [0, Ke); odd-ell block [Ke, K3p)
  int npads;             // unused (zero) Step-3 columns
  const int* pads;       // [npads]
  const float* g;        // [H_plus][n_k]   2 pi w_m G_zeta(k_m), ell >= 0 terms (ell = 0 block first)
  const int* ell;        // [H_plus]
  const int* col;        // [H_plus] first Step-3 column of the term
  const float* Y3;       // [N_t][K3p]       Step-3 real operand (reading R13), zero-padded
  const float2* tw;      // [n_psi/2] e^{-2 pi i j / n_psi}
  const float2* twg;     // [n_gamma/2] e^{-2 pi i j / n_gamma}
};

// ---------------- SIMT reference engine (ftk_simt.cu) ----------------
void launch_ring_fft(const float2* polar, float2* fb, int64_t n_items, const DevPlan& P, cudaStream_t s);
void launch_step1_simt(const float2* A, const float2* B, float2* Zhat, const PairBlock& pb, const DevPlan& P,
                       cudaStream_t s);
void launch_step2_simt(const float2* Zhat, float* Z3, const PairBlock& pb, const DevPlan& P, cudaStream_t s);
void launch_step3_simt(const float* Z3, const PairBlock& pb, const DevPlan& P, int tm_offset,
                       unsigned long long* img_keys, unsigned long long* pair_keys, int n_tm_local, float* landscape,
                       cudaStream_t s);
void launch_finalize(const unsigned long long* keys, int64_t n, int N_t, int n_psi, ftk_best_t* out, cudaStream_t s);
void launch_merge(const ftk_best_t* gathered, int world, int64_t n, ftk_best_t* out, cudaStream_t s);
void launch_fb_export(const float2* fb, int64_t first, int64_t count, int n_k, int n_psi, float2* out, cudaStream_t s);

// ---------------- pixel front end (ftk_nufft.cu): Eq. Ahattrap by a 2-D type-2 NUFFT ----------------
struct NuPlan {
  int n = 0, nf = 0, lognf = 0, w = 7, n_k = 0;  // pixels per side, fine grid 2n, kernel width
  double beta = 0;                                // ES kernel shape 2.30 w
  float* d_corr = nullptr;                        // [n] 1 / phihat(i - n/2)
  float2* d_twf = nullptr;                        // [nf/2] e^{-2 pi i j / nf}
  float* d_k = nullptr;                           // [n_k] radial nodes (rad/px)
  bool ready = false;
};
int nu_plan_init(NuPlan& nu, int n, const std::vector<double>& k, int w, std::string& msg);
void nu_plan_free(NuPlan& nu);
size_t nu_scratch_bytes_per_image(const NuPlan& nu);
// pix: device float [count][n][n]; polar: device complex [count][n_k][n_psi]; scratch >= count x per-image bytes
void launch_polar_from_pixels(const NuPlan& nu, const float* pix, int64_t count, float2* polar, int n_psi,
                              void* scratch, cudaStream_t s);

}  // namespace ftk
