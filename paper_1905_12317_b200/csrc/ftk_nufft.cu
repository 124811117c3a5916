// Pixel images -> polar Fourier samples: the trapezoid sum of PAPER.md Eq. (Ahattrap), P:302-318,
//   Ahat(k) = sum_{i,j < n} A_ij exp(-i (k_x x_i + k_y y_j)),   x_i = i - n/2,  y_j = j - n/2   (px units, R23)
// on the polar grid k = k_m (cos psi_p, sin psi_p), psi_p = 2 pi p / n_psi, evaluated as a 2-D type-2
// NUFFT (the paper uses FINUFFT).  With modes l = (i - n/2, j - n/2) and "points" k in
// [-pi, pi)^2 this is F(k) = sum_l f_l e^{-i k.l}.  For a kernel phi supported on |u| <= alpha and its
// transform phihat(l) = int phi(u) e^{i u l} du one has e^{-ikl} = (1/phihat(l)) int phi(k - y) e^{-iyl} dy,
// hence F(k) = int phi(k - y) G(y) dy with the 2 pi-periodic G(y) = sum_l (f_l / phihat(l)) e^{-iyl}, and the
// trapezoid rule on the fine grid y_s = h s (h = 2 pi / nf, nf = 2 n) gives
//   F(k) ~ h^2 sum_s phi(k_x - h s_x) phi(k_y - h s_y) G[s],   G[s] = sum_l g_l e^{-2 pi i l s / nf}   (an FFT).
// phi is the "exponential of semicircle" kernel exp(beta (sqrt(1 - (u/alpha)^2) - 1)), alpha = w h / 2,
// beta = 2.30 w (upsampling 2; w = 7 -> ~1e-6 relative error); phihat from Gauss-Legendre in double.
//
// Kernels (per chunk of images):
//   k_nu_rows   : row i of the pixels times corr(i) corr(j), zero-padded to nf at j - n/2 mod nf, FFT over j
//                 -> T [img][i][s_y]                                        (n rows of nf complex)
//   k_nu_cols   : for 16 columns s_y: T[:, s_y] placed at i - n/2 mod nf, FFT over i
//                 -> Gt [img][s_y][s_x] (the fine grid, transposed so the write-out is contiguous)
//   k_nu_interp : per polar target the w x w gather from Gt with separable kernel weights -> [img][m][p]
#include <cmath>
#include <string>
#include <vector>

#include "ftk_fft.cuh"
#include "ftk_internal.cuh"

namespace ftk {

constexpr int NU_RB = 8;    // rows per CTA in k_nu_rows
constexpr int NU_CB = 16;   // columns per CTA in k_nu_cols
constexpr int NU_WMAX = 16;

__global__ void __launch_bounds__(256) k_nu_rows(const float* __restrict__ pix, float2* __restrict__ T, int n, int nf,
                                                 int lognf, const float* __restrict__ corr,
                                                 const float2* __restrict__ twf) {
  extern __shared__ float2 nu_sm[];
  float2* tws = nu_sm + (size_t)NU_RB * nf;
  const int64_t img = blockIdx.x;
  const int i0 = blockIdx.y * NU_RB;
  const int nr = min(NU_RB, n - i0);
  for (int t = threadIdx.x; t < nf / 2; t += blockDim.x) tws[t] = twf[t];
  for (int t = threadIdx.x; t < nr * nf; t += blockDim.x) nu_sm[t] = make_float2(0.f, 0.f);
  __syncthreads();
  const float* src = pix + (img * n + i0) * (int64_t)n;
  for (int t = threadIdx.x; t < nr * n; t += blockDim.x) {
    const int r = t / n, j = t - r * n;
    const float v = src[(int64_t)r * n + j] * corr[i0 + r] * corr[j];
    nu_sm[r * nf + ((j - n / 2 + nf) & (nf - 1))] = make_float2(v, 0.f);
  }
  __syncthreads();
  smem_fft_rows(nu_sm, nr, nf, lognf, tws);
  float2* dst = T + (img * n + i0) * (int64_t)nf;
  for (int t = threadIdx.x; t < nr * nf; t += blockDim.x) dst[t] = nu_sm[t];
}

__global__ void __launch_bounds__(256) k_nu_cols(const float2* __restrict__ T, float2* __restrict__ Gt, int n, int nf,
                                                 int lognf, const float2* __restrict__ twf) {
  extern __shared__ float2 nu_sm[];
  float2* tws = nu_sm + (size_t)NU_CB * nf;
  const int64_t img = blockIdx.x;
  const int c0 = blockIdx.y * NU_CB;
  for (int t = threadIdx.x; t < nf / 2; t += blockDim.x) tws[t] = twf[t];
  for (int t = threadIdx.x; t < NU_CB * nf; t += blockDim.x) nu_sm[t] = make_float2(0.f, 0.f);
  __syncthreads();
  const float2* src = T + img * (int64_t)n * nf + c0;
  for (int t = threadIdx.x; t < n * NU_CB; t += blockDim.x) {
    const int i = t / NU_CB, c = t - i * NU_CB;  // 16 consecutive columns of row i: 128-byte reads
    nu_sm[c * nf + ((i - n / 2 + nf) & (nf - 1))] = src[(int64_t)i * nf + c];
  }
  __syncthreads();
  smem_fft_rows(nu_sm, NU_CB, nf, lognf, tws);
  float2* dst = Gt + (img * nf + c0) * (int64_t)nf;
  for (int t = threadIdx.x; t < NU_CB * nf; t += blockDim.x) dst[t] = nu_sm[t];
}

// phi(u) for |u| <= alpha as a function of the grid offset d = u / h in grid units: z = d / (w / 2)
__device__ __forceinline__ float nu_phi(float d, float half_w, float beta) {
  const float z = d / half_w;
  const float r = 1.f - z * z;
  return r > 0.f ? __expf(beta * (sqrtf(r) - 1.f)) : 0.f;
}

__global__ void __launch_bounds__(256) k_nu_interp(const float2* __restrict__ Gt, float2* __restrict__ polar, int nf,
                                                   int w, float beta, const float* __restrict__ kr, int n_k,
                                                   int n_psi, float h2) {
  const int64_t img = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_k * n_psi) return;
  const int m = t / n_psi, p = t - m * n_psi;
  float sn, cs;
  sincospif(2.f * (float)p / (float)n_psi, &sn, &cs);
  const float inv_h = (float)nf / (2.f * 3.14159265358979323846f);
  const float sx = kr[m] * cs * inv_h, sy = kr[m] * sn * inv_h;  // target in fine-grid units
  const float half_w = 0.5f * (float)w;
  const int x0 = (int)ceilf(sx - half_w), y0 = (int)ceilf(sy - half_w);
  float wx[NU_WMAX], wy[NU_WMAX];
  for (int a = 0; a < w; ++a) {
    wx[a] = nu_phi(sx - (float)(x0 + a), half_w, beta);
    wy[a] = nu_phi(sy - (float)(y0 + a), half_w, beta);
  }
  const float2* G = Gt + img * (int64_t)nf * nf;
  float re = 0.f, im = 0.f;
  for (int b = 0; b < w; ++b) {
    const float2* row = G + (int64_t)((y0 + b) & (nf - 1)) * nf;  // Gt[s_y][s_x]
    float rr = 0.f, ri = 0.f;
    for (int a = 0; a < w; ++a) {
      const float2 g = __ldg(row + ((x0 + a) & (nf - 1)));
      rr = fmaf(wx[a], g.x, rr);
      ri = fmaf(wx[a], g.y, ri);
    }
    re = fmaf(wy[b], rr, re);
    im = fmaf(wy[b], ri, im);
  }
  polar[img * (int64_t)n_k * n_psi + t] = make_float2(h2 * re, h2 * im);
}

int nu_plan_init(NuPlan& nu, int n, const std::vector<double>& k, int w, std::string& msg) {
  nu_plan_free(nu);
  if (n < 2 || (n & (n - 1)) != 0) {
    msg = "pixel front end: n must be a power of two";
    return FTK_EINVAL;
  }
  if (w < 2 || w > NU_WMAX) {
    msg = "pixel front end: kernel width out of range";
    return FTK_EINVAL;
  }
  nu.n = n;
  nu.nf = 2 * n;
  nu.lognf = 0;
  while ((1 << nu.lognf) < nu.nf) nu.lognf++;
  nu.w = w;
  nu.beta = 2.30 * w;
  nu.n_k = (int)k.size();
  const double h = 2.0 * M_PI / nu.nf, alpha = 0.5 * w * h;
  // phihat(l) = alpha int_{-1}^{1} exp(beta (sqrt(1 - t^2) - 1)) cos(alpha l t) dt  (Gauss-Legendre, 256 nodes)
  const int Q = 256;
  std::vector<double> tq(Q), wq(Q);
  for (int i = 0; i < Q; ++i) {  // Newton on P_Q
    double x = std::cos(M_PI * (i + 0.75) / (Q + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int j = 2; j <= Q; ++j) {
        const double p2 = ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / j;
        p0 = p1;
        p1 = p2;
      }
      const double dp = Q * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-16) {
        tq[i] = x;
        wq[i] = 2.0 / ((1.0 - x * x) * dp * dp);
        break;
      }
      tq[i] = x;
      wq[i] = 2.0 / ((1.0 - x * x) * dp * dp);
    }
  }
  std::vector<float> corr(n);
  for (int i = 0; i < n; ++i) {
    const double l = i - n / 2;
    double s = 0;
    for (int q = 0; q < Q; ++q) s += wq[q] * std::exp(nu.beta * (std::sqrt(1.0 - tq[q] * tq[q]) - 1.0)) * std::cos(alpha * l * tq[q]);
    corr[i] = (float)(1.0 / (alpha * s));
  }
  std::vector<float2> twf(nu.nf / 2);
  for (int j = 0; j < nu.nf / 2; ++j) {
    const double ph = -2.0 * M_PI * j / nu.nf;
    twf[j] = make_float2((float)std::cos(ph), (float)std::sin(ph));
  }
  std::vector<float> kr(k.begin(), k.end());
  if (cudaMalloc(&nu.d_corr, n * sizeof(float)) != cudaSuccess || cudaMalloc(&nu.d_twf, twf.size() * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&nu.d_k, kr.size() * sizeof(float)) != cudaSuccess) {
    nu_plan_free(nu);
    msg = "pixel front end: allocation failed";
    return FTK_ENOMEM;
  }
  cudaMemcpy(nu.d_corr, corr.data(), n * sizeof(float), cudaMemcpyHostToDevice);
  cudaMemcpy(nu.d_twf, twf.data(), twf.size() * sizeof(float2), cudaMemcpyHostToDevice);
  cudaMemcpy(nu.d_k, kr.data(), kr.size() * sizeof(float), cudaMemcpyHostToDevice);
  FTK_SMEM_OPTIN(k_nu_rows);
  FTK_SMEM_OPTIN(k_nu_cols);
  nu.ready = true;
  return FTK_OK;
}

void nu_plan_free(NuPlan& nu) {
  cudaFree(nu.d_corr);
  cudaFree(nu.d_twf);
  cudaFree(nu.d_k);
  nu.d_corr = nullptr;
  nu.d_twf = nullptr;
  nu.d_k = nullptr;
  nu.ready = false;
}

size_t nu_scratch_bytes_per_image(const NuPlan& nu) {
  return ((size_t)nu.n * nu.nf + (size_t)nu.nf * nu.nf) * sizeof(float2);
}

void launch_polar_from_pixels(const NuPlan& nu, const float* pix, int64_t count, float2* polar, int n_psi,
                              void* scratch, cudaStream_t s) {
  if (count <= 0) return;
  float2* T = reinterpret_cast<float2*>(scratch);
  float2* Gt = T + (size_t)count * nu.n * nu.nf;
  const size_t sm_rows = ((size_t)NU_RB * nu.nf + nu.nf / 2) * sizeof(float2);
  const size_t sm_cols = ((size_t)NU_CB * nu.nf + nu.nf / 2) * sizeof(float2);
  k_nu_rows<<<dim3((unsigned)count, (nu.n + NU_RB - 1) / NU_RB), 256, sm_rows, s>>>(pix, T, nu.n, nu.nf, nu.lognf,
                                                                                    nu.d_corr, nu.d_twf);
  k_nu_cols<<<dim3((unsigned)count, nu.nf / NU_CB), 256, sm_cols, s>>>(T, Gt, nu.n, nu.nf, nu.lognf, nu.d_twf);
  const double h = 2.0 * M_PI / nu.nf;
  const int tgt = nu.n_k * n_psi;
  k_nu_interp<<<dim3((tgt + 255) / 256, (unsigned)count), 256, 0, s>>>(Gt, polar, nu.nf, nu.w, (float)nu.beta, nu.d_k,
                                                                       nu.n_k, n_psi, (float)(h * h));
}

}  // namespace ftk
