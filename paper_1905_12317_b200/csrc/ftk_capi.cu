// C ABI of the FTK hot path: plan lifetime, loads, the pair-block scheduler behind ftk_align,
// merge and profiling hooks.  See include/ftk.h for the contracts.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ftk_internal.cuh"
#include "ftk_nccl.h"
#include "ftk_plan_math.h"
#include "ftk_tc.cuh"

using namespace ftk;

struct ftk_plan_s {
  PlanMath pm;
  int device = -1, rank = 0, world = 1, engine = 0;
  void* nccl_comm = nullptr;  // caller-owned ncclComm_t (opts.nccl_comm): ftk_align gathers global bests
  ftk_best_t* d_gather = nullptr;  // [world][N_im] all-gathered records
  int64_t gather_cap = 0;
  size_t ws_bytes = (size_t)1 << 30;
  bool ws_user = false;
  std::string err;
  // device constants
  float* d_g = nullptr;
  int* d_ell = nullptr;
  int* d_col = nullptr;
  float* d_Y3 = nullptr;
  float2* d_tw = nullptr;
  int K3p = 0, K3dev = 0, Ke = 0, log2_psi = 0, n_gamma = 0;
  float2* d_twg = nullptr;  // e^{-2 pi i j / n_gamma}, j < n_gamma / 2 (Step-2 FFT)
  int* d_pads = nullptr;
  int npads = 0;
  TcPlan tc;  // tensor-core engine constants (ftk_tc.cu)
  // data
  float2* d_A = nullptr;
  int64_t n_im = 0;
  float2* d_B = nullptr;
  int64_t n_tm_total = 0, n_tm_local = 0, tm_off = 0;
  bool have_images = false, have_templates = false;
  // workspace
  void* d_ws = nullptr;
  size_t ws_size = 0;
  unsigned long long* d_keys = nullptr;
  int64_t keys_cap = 0;
  ftk_best_t* d_best_tmp = nullptr;
  int64_t best_tmp_cap = 0;
  void* d_stage = nullptr;
  size_t stage_bytes = 0;
  // pixel front end (NEXT-2): NUFFT plan and its chunk scratch
  NuPlan nu;
  void* d_nu = nullptr;
  size_t nu_bytes = 0;
  // marginalization partials (G > 1 rep-groups)
  void* d_marg_part = nullptr;
  size_t marg_part_bytes = 0;
  // profiling
  bool prof = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[5];
  size_t ev_used[5] = {0, 0, 0, 0, 0};
};

namespace {

const char* kStatusStr[] = {"FTK_OK",     "FTK_EINVAL", "FTK_ERANGE", "FTK_ENUMERIC", "FTK_ENOMEM",
                            "FTK_ECUDA",  "FTK_ESTATE", "FTK_ECAPACITY", "FTK_ENODEV", "FTK_ENCCL"};

ftk_status_t fail(ftk_plan_t p, ftk_status_t s, const std::string& msg) {
  if (p) p->err = msg;
  return s;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      return fail(plan, e_ == cudaErrorMemoryAllocation ? FTK_ENOMEM : FTK_ECUDA,            \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                        \
    }                                                                                         \
  } while (0)

DevPlan devplan(ftk_plan_t p) {
  DevPlan d;
  d.n_k = p->pm.n_k;
  d.n_psi = p->pm.n_psi;
  d.n_gamma = p->n_gamma;
  d.twg = p->d_twg;
  d.log2_psi = p->log2_psi;
  d.N_t = p->pm.N_t;
  d.H_plus = p->pm.H_plus;
  d.K3 = p->K3dev;
  d.Ke = p->Ke;
  d.npads = p->npads;
  d.pads = p->d_pads;
  d.K3p = p->K3p;
  d.Hs = (p->pm.H_plus + 1) / 2 * 2;
  int lm = 0;
  for (const auto& t : p->pm.terms)
    if (t.ell >= 0) lm = std::max(lm, t.ell);
  d.ell_max = lm;
  d.g = p->d_g;
  d.ell = p->d_ell;
  d.col = p->d_col;
  d.Y3 = p->d_Y3;
  d.tw = p->d_tw;
  return d;
}

void prof_begin(ftk_plan_t p, int c, cudaStream_t s) {
  if (!p->prof) return;
  if (p->ev_used[c] == p->ev[c].size()) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    p->ev[c].push_back({a, b});
  }
  cudaEventRecord(p->ev[c][p->ev_used[c]].first, s);
}
void prof_end(ftk_plan_t p, int c, cudaStream_t s) {
  if (!p->prof) return;
  cudaEventRecord(p->ev[c][p->ev_used[c]].second, s);
  p->ev_used[c]++;
}
void prof_reset(ftk_plan_t p) {
  for (int c = 0; c < 5; ++c) p->ev_used[c] = 0;
}

bool is_device_ptr(const void* ptr) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

template <typename T>
ftk_status_t upload(ftk_plan_t plan, T** dst, const std::vector<T>& src) {
  if (*dst) cudaFree(*dst);
  *dst = nullptr;
  if (src.empty()) return FTK_OK;
  CK(cudaMalloc((void**)dst, src.size() * sizeof(T)));
  CK(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return FTK_OK;
}

}  // namespace

extern "C" {

const char* ftk_status_string(ftk_status_t s) {
  int i = (int)s;
  return (i >= 0 && i <= 9) ? kStatusStr[i] : "FTK_UNKNOWN";
}

int ftk_version(void) { return 100; }

const char* ftk_last_error(ftk_plan_t plan) { return plan ? plan->err.c_str() : ""; }

static ftk_status_t plan_create_impl(int n, double K, double delta_max_px, const double* shifts_xy_px, int N_t,
                                     int n_tau, const double* filters, double eps, const ftk_plan_opts_t* opts,
                                     ftk_plan_t* out) {
  if (!out) return FTK_EINVAL;
  *out = nullptr;
  if (!shifts_xy_px || N_t <= 0 || n_tau < 0 || (n_tau > 0 && !filters)) return FTK_EINVAL;
  if (n_tau > 0 && (long long)N_t * n_tau > (1LL << 30)) return FTK_EINVAL;
  ftk_plan_t plan = new (std::nothrow) ftk_plan_s();
  if (!plan) return FTK_ENOMEM;
  ftk_plan_opts_t o;
  std::memset(&o, 0, sizeof o);
  if (opts) o = *opts;
  PlanMath& pm = plan->pm;
  pm.n = n;
  pm.K_cycles = K;
  pm.delta_max = delta_max_px;
  pm.eps = eps;
  pm.n_k = o.n_k > 0 ? o.n_k : (int)std::lround(K);
  pm.n_psi = o.n_psi > 0 ? o.n_psi : 4 * (int)std::lround(K);
  pm.rule = o.radial_rule;
  pm.svd_nodes = o.svd_nodes > 0 ? o.svd_nodes : 96;
  if (n_tau > 0) {
    // CTF-parameterized kernel (reading R24): virtual shift v = tau * N_t + t, tau-major
    pm.n_tau = n_tau;
    pm.N_base = N_t;
    pm.filt.assign(filters, filters + (size_t)n_tau * pm.n_k);
    pm.N_t = N_t * n_tau;
    pm.shifts.clear();
    for (int ta = 0; ta < n_tau; ++ta) pm.shifts.insert(pm.shifts.end(), shifts_xy_px, shifts_xy_px + 2 * (size_t)N_t);
  } else {
    pm.N_t = N_t;
    pm.shifts.assign(shifts_xy_px, shifts_xy_px + 2 * (size_t)N_t);
  }
  N_t = pm.N_t;
  plan->device = o.device;
  plan->world = o.world > 0 ? o.world : 1;
  plan->rank = o.rank;
  plan->engine = o.engine;
  plan->nccl_comm = o.nccl_comm;
  plan->ws_bytes = o.workspace_bytes ? o.workspace_bytes : ((size_t)1 << 30);
  plan->ws_user = o.workspace_bytes != 0;
  auto bail = [&](ftk_status_t s) {
    ftk_plan_destroy(plan);
    return s;
  };
  if (plan->rank < 0 || plan->rank >= plan->world || (plan->engine != 0 && plan->engine != 1) ||
      (pm.rule != 0 && pm.rule != 1))
    return bail(FTK_EINVAL);
  const int np = pm.n_psi;
  if (np < 64 || np > 1024 || (np & (np - 1)) != 0) return bail(FTK_EINVAL);
  plan->n_gamma = o.n_gamma > 0 ? o.n_gamma : np;
  if (plan->n_gamma < np || plan->n_gamma > 1024 || (plan->n_gamma & (plan->n_gamma - 1)) != 0) return bail(FTK_EINVAL);
  if (plan->n_gamma != np && plan->engine != 0) return bail(FTK_EINVAL);
  if (pm.n_k > 1024) return bail(FTK_EINVAL);
  int st = pm.build();
  if (st != FTK_OK) {
    fprintf(stderr, "ftk_plan_create: %s\n", pm.error.c_str());
    return bail((ftk_status_t)st);
  }
  plan->log2_psi = 0;
  while ((1 << plan->log2_psi) < np) plan->log2_psi++;
  // Step-3 column blocks (see the column map below): even-ell block [0, Ke), odd-ell block [Ke, K3p)
  {
    int n_even = 0, n_odd = 0;
    for (const auto& tm : pm.terms) {
      if (tm.ell > 0 && (tm.ell % 2) == 0) ++n_even;
      if (tm.ell > 0 && (tm.ell % 2) == 1) ++n_odd;
    }
    const int ce = pm.H0 + ((pm.H0 & 1) && n_even > 0 ? 1 : 0) + 2 * n_even;
    plan->Ke = (ce + 15) / 16 * 16;
    plan->K3p = plan->Ke + (2 * n_odd + 15) / 16 * 16;
    plan->K3dev = plan->K3p;
  }
  if (plan->device < 0) {
    *out = plan;
    return FTK_OK;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || plan->device >= ndev) {
    cudaGetLastError();
    return bail(FTK_ENODEV);
  }
  if (cudaSetDevice(plan->device) != cudaSuccess) return bail(FTK_ECUDA);
  if (plan->nccl_comm) {
    std::string msg;
    const int cs = nccl_comm_check(plan->nccl_comm, plan->world, plan->rank, msg);
    if (cs != FTK_OK) {
      fprintf(stderr, "ftk_plan_create: %s\n", msg.c_str());
      return bail((ftk_status_t)cs);
    }
  }
  // ---- device constants: ell >= 0 terms in zeta order
  std::vector<float> g, Y3((size_t)N_t * plan->K3p, 0.f);
  std::vector<int> ell, col;
  // device term order: ell = 0 terms, then even ell > 0, then odd ell (each in zeta order).  Step-3
  // columns: one per ell = 0 term; (Re, Im) pairs of the even ell > 0 terms on even columns; the odd-ell
  // pairs from column Ke (a multiple of 16).  Every group of 8 columns holds whole terms (Step 2 writes
  // column groups) and Y_zeta(-delta) = (-1)^ell Y_zeta(delta) splits X(+-delta) = E(delta) +- O(delta)
  // between the two blocks (the tensor-core Step 3 evaluates half of a symmetric shift list).  The
  // tensor-core engine then moves whole Step-2 blocks (tc_term_order) so that each fits one TMA window.
  std::vector<int> zplus;
  for (int pass = 0; pass < 3; ++pass)
    for (int z = 0; z < pm.H; ++z) {
      const int l = pm.terms[z].ell;
      if ((pass == 0 && l == 0) || (pass == 1 && l > 0 && l % 2 == 0) || (pass == 2 && l % 2 == 1)) zplus.push_back(z);
    }
  std::vector<char> used(plan->K3p, 0);
  int c = 0;
  bool odd_started = false;
  for (int z : zplus) {
    const int l = pm.terms[z].ell;
    if (l % 2 == 1 && !odd_started) {
      c = plan->Ke;
      odd_started = true;
    }
    if (l > 0 && (c & 1)) c += 1;  // pairs on even columns
    ell.push_back(l);
    col.push_back(c);
    used[c] = 1;
    if (l > 0) used[c + 1] = 1;
    for (int m = 0; m < pm.n_k; ++m) g.push_back((float)(2.0 * M_PI * pm.w[m] * pm.G[(size_t)z * pm.n_k + m]));
    for (int t = 0; t < N_t; ++t) {
      const std::complex<double> y = pm.Y[(size_t)t * pm.H + z];
      if (l == 0) {
        Y3[(size_t)t * plan->K3p + c] = (float)y.real();
      } else {
        Y3[(size_t)t * plan->K3p + c] = (float)(2.0 * y.real());
        Y3[(size_t)t * plan->K3p + c + 1] = (float)(-2.0 * y.imag());
      }
    }
    c += (l == 0) ? 1 : 2;
  }
  if (plan->engine == 0) {  // tensor-core engine: term order with every Step-2 block in one TMA window
    std::string msg;
    std::vector<int> perm;
    if (tc_term_order(ell, col, plan->K3p, perm, msg) != FTK_OK) {
      plan->err = msg;
      fprintf(stderr, "ftk_plan_create: %s\n", msg.c_str());
      return bail(FTK_EINVAL);
    }
    std::vector<int> ell2, col2;
    std::vector<float> g2;
    for (int z : perm) {
      ell2.push_back(ell[z]);
      col2.push_back(col[z]);
      g2.insert(g2.end(), g.begin() + (size_t)z * pm.n_k, g.begin() + (size_t)(z + 1) * pm.n_k);
    }
    ell.swap(ell2);
    col.swap(col2);
    g.swap(g2);
  }
  std::vector<int> pads;
  for (int k = 0; k < plan->K3p; ++k)
    if (!used[k]) pads.push_back(k);
  plan->npads = (int)pads.size();
  std::vector<float2> tw(np / 2), twg(plan->n_gamma / 2);
  for (int j = 0; j < np / 2; ++j) {
    const double ph = -2.0 * M_PI * j / np;
    tw[j] = make_float2((float)std::cos(ph), (float)std::sin(ph));
  }
  for (int j = 0; j < plan->n_gamma / 2; ++j) {
    const double ph = -2.0 * M_PI * j / plan->n_gamma;
    twg[j] = make_float2((float)std::cos(ph), (float)std::sin(ph));
  }
  ftk_status_t s;
  if ((s = upload(plan, &plan->d_g, g)) != FTK_OK) return bail(s);
  if ((s = upload(plan, &plan->d_ell, ell)) != FTK_OK) return bail(s);
  if ((s = upload(plan, &plan->d_col, col)) != FTK_OK) return bail(s);
  if ((s = upload(plan, &plan->d_pads, pads)) != FTK_OK) return bail(s);
  if ((s = upload(plan, &plan->d_Y3, Y3)) != FTK_OK) return bail(s);
  if ((s = upload(plan, &plan->d_tw, tw)) != FTK_OK) return bail(s);
  if ((s = upload(plan, &plan->d_twg, twg)) != FTK_OK) return bail(s);
  if (plan->engine == 0) {
    std::string msg;
    int ts = tc_plan_init(plan->tc, pm, g, ell, col, Y3, plan->K3p, plan->Ke, plan->n_gamma, msg);
    if (ts != FTK_OK) {
      plan->err = msg;
      fprintf(stderr, "ftk_plan_create: %s\n", msg.c_str());
      return bail((ftk_status_t)ts);
    }
  }
  *out = plan;
  return FTK_OK;
}

ftk_status_t ftk_plan_create(int n, double K, double delta_max_px, const double* shifts_xy_px, int N_t, double eps,
                             const ftk_plan_opts_t* opts, ftk_plan_t* out) {
  return plan_create_impl(n, K, delta_max_px, shifts_xy_px, N_t, 0, nullptr, eps, opts, out);
}

ftk_status_t ftk_plan_create_ctf(int n, double K, double delta_max_px, const double* shifts_xy_px, int N_t,
                                 int n_tau, const double* filters, double eps, const ftk_plan_opts_t* opts,
                                 ftk_plan_t* out) {
  if (n_tau <= 0) {
    if (out) *out = nullptr;
    return FTK_EINVAL;
  }
  return plan_create_impl(n, K, delta_max_px, shifts_xy_px, N_t, n_tau, filters, eps, opts, out);
}

ftk_status_t ftk_radial_rule(int n, double K, int n_k, int radial_rule, double* k_out, double* w_out) {
  if (n <= 0 || !(K > 0) || n_k <= 0 || n_k > 1024 || (radial_rule != 0 && radial_rule != 1) || !k_out || !w_out)
    return FTK_EINVAL;
  std::vector<double> k, w;
  if (!radial_rule_nodes(n_k, 2.0 * M_PI * K / n, radial_rule, k, w)) return FTK_ENUMERIC;
  std::memcpy(k_out, k.data(), n_k * sizeof(double));
  std::memcpy(w_out, w.data(), n_k * sizeof(double));
  return FTK_OK;
}

void ftk_plan_destroy(ftk_plan_t plan) {
  if (!plan) return;
  if (plan->device >= 0) {
    cudaSetDevice(plan->device);
    cudaFree(plan->d_g);
    cudaFree(plan->d_ell);
    cudaFree(plan->d_col);
    cudaFree(plan->d_pads);
    cudaFree(plan->d_Y3);
    cudaFree(plan->d_tw);
    cudaFree(plan->d_twg);
    cudaFree(plan->d_A);
    cudaFree(plan->d_B);
    cudaFree(plan->d_ws);
    cudaFree(plan->d_keys);
    cudaFree(plan->d_best_tmp);
    cudaFree(plan->d_gather);
    cudaFree(plan->d_stage);
    cudaFree(plan->d_nu);
    cudaFree(plan->d_marg_part);
    nu_plan_free(plan->nu);
    tc_plan_free(plan->tc);
    for (int c = 0; c < 5; ++c)
      for (auto& e : plan->ev[c]) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
      }
  }
  delete plan;
}

ftk_status_t ftk_plan_query(ftk_plan_t plan, ftk_plan_info_t* info) {
  if (!plan || !info) return FTK_EINVAL;
  const PlanMath& pm = plan->pm;
  std::memset(info, 0, sizeof *info);
  info->n = pm.n;
  info->n_k = pm.n_k;
  info->n_psi = pm.n_psi;
  info->N_t = pm.N_t;
  info->H = pm.H;
  info->H_plus = pm.H_plus;
  info->H0 = pm.H0;
  info->K3 = pm.K3;
  info->ell_max = pm.ell_max;
  info->K_cycles = pm.K_cycles;
  info->k_max = pm.k_max;
  info->delta_max = pm.delta_max;
  info->W = pm.W;
  info->eps = pm.eps;
  info->certificate = pm.certificate;
  info->n_images = plan->n_im;
  info->n_templates_total = plan->n_tm_total;
  info->n_templates_local = plan->n_tm_local;
  info->template_offset = plan->tm_off;
  info->engine = plan->engine;
  info->device = plan->device;
  info->rank = plan->rank;
  info->world = plan->world;
  info->K3p = plan->K3p;
  info->n_rep = plan->engine == 0 ? plan->tc.n_rep : plan->pm.N_t;
  info->n_gamma = plan->n_gamma;
  info->n_tau = pm.n_tau;
  info->N_t_base = pm.n_tau > 0 ? pm.N_base : pm.N_t;
  info->s3_cols = plan->engine == 0 ? plan->tc.ncol : plan->pm.N_t;
  info->s3_nch = plan->engine == 0 ? plan->tc.NCH : 0;
  info->s3_groups = plan->engine == 0 ? plan->tc.G : 0;
  info->s3_rtiles = plan->engine == 0 ? plan->tc.NRT : 0;
  return FTK_OK;
}

ftk_status_t ftk_plan_radial(ftk_plan_t plan, double* k, double* w) {
  if (!plan || !k || !w) return FTK_EINVAL;
  std::copy(plan->pm.k.begin(), plan->pm.k.end(), k);
  std::copy(plan->pm.w.begin(), plan->pm.w.end(), w);
  return FTK_OK;
}

ftk_status_t ftk_plan_terms(ftk_plan_t plan, int32_t* ell, int32_t* eta, double* sigma) {
  if (!plan || !ell || !eta || !sigma) return FTK_EINVAL;
  for (int z = 0; z < plan->pm.H; ++z) {
    ell[z] = plan->pm.terms[z].ell;
    eta[z] = plan->pm.terms[z].eta;
    sigma[z] = plan->pm.terms[z].sigma;
  }
  return FTK_OK;
}

ftk_status_t ftk_plan_factors(ftk_plan_t plan, double* G, double* Y) {
  if (!plan || !G || !Y) return FTK_EINVAL;
  std::copy(plan->pm.G.begin(), plan->pm.G.end(), G);
  for (size_t i = 0; i < plan->pm.Y.size(); ++i) {
    Y[2 * i] = plan->pm.Y[i].real();
    Y[2 * i + 1] = plan->pm.Y[i].imag();
  }
  return FTK_OK;
}

static ftk_status_t load_set(ftk_plan_t plan, const void* polar, int64_t first, int64_t count, int is_device,
                             float2* dst, cudaStream_t s) {
  const DevPlan P = devplan(plan);
  const size_t item_bytes = (size_t)P.n_k * P.n_psi * sizeof(float2);
  const float2* src = reinterpret_cast<const float2*>(polar) + first * (int64_t)P.n_k * P.n_psi;
  if (is_device) {
    prof_begin(plan, 0, s);
    launch_ring_fft(src, dst, count, P, s);
    prof_end(plan, 0, s);
    CK(cudaGetLastError());
    return FTK_OK;
  }
  if (!plan->d_stage) {
    plan->stage_bytes = std::max(item_bytes, (size_t)256 << 20);
    CK(cudaMalloc(&plan->d_stage, plan->stage_bytes));
  }
  const int64_t chunk = std::max<int64_t>(1, plan->stage_bytes / item_bytes);
  for (int64_t c0 = 0; c0 < count; c0 += chunk) {
    const int64_t nc = std::min(chunk, count - c0);
    CK(cudaMemcpyAsync(plan->d_stage, src + c0 * (int64_t)P.n_k * P.n_psi, nc * item_bytes, cudaMemcpyHostToDevice, s));
    prof_begin(plan, 0, s);
    launch_ring_fft(reinterpret_cast<float2*>(plan->d_stage), dst + c0 * (int64_t)P.n_k * P.n_psi, nc, P, s);
    prof_end(plan, 0, s);
    CK(cudaGetLastError());
  }
  return FTK_OK;
}

// Pixel images [first, first + count) -> polar samples (NUFFT, Eq. Ahattrap) -> either the caller's polar
// buffer (fb == nullptr) or, through the ring FFT, FB coefficients at fb.  Chunked through plan->d_nu.
static ftk_status_t pixels_chunked(ftk_plan_t plan, const float* pixels, int64_t first, int64_t count, int is_device,
                                   float2* polar_out, float2* fb, cudaStream_t s) {
  const DevPlan P = devplan(plan);
  if (!plan->nu.ready) {
    std::string msg;
    const int st = nu_plan_init(plan->nu, plan->pm.n, plan->pm.k, 7, msg);
    if (st != FTK_OK) return fail(plan, (ftk_status_t)st, msg);
  }
  const int n = plan->pm.n;
  const size_t pix_bytes = (size_t)n * n * sizeof(float);
  const size_t polar_bytes = (size_t)P.n_k * P.n_psi * sizeof(float2);
  const size_t per = nu_scratch_bytes_per_image(plan->nu) + (fb ? polar_bytes : 0) + (is_device ? 0 : pix_bytes);
  int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(count, std::max<size_t>(per, (size_t)512 << 20) / per));
  if (const char* e = std::getenv("FTK_NU_CHUNK"))  // tests: force small chunks (ragged chunk boundaries)
    chunk = std::max<int64_t>(1, std::min<int64_t>(chunk, std::atoll(e)));
  if (plan->nu_bytes < (size_t)chunk * per) {
    cudaFree(plan->d_nu);
    plan->d_nu = nullptr;
    plan->nu_bytes = 0;
    CK(cudaMalloc(&plan->d_nu, (size_t)chunk * per));
    plan->nu_bytes = (size_t)chunk * per;
  }
  uint8_t* base = reinterpret_cast<uint8_t*>(plan->d_nu);
  void* scratch = base;
  float2* pol_tmp = reinterpret_cast<float2*>(base + (size_t)chunk * nu_scratch_bytes_per_image(plan->nu));
  float* pix_tmp = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(pol_tmp) + (fb ? (size_t)chunk * polar_bytes : 0));
  for (int64_t c0 = 0; c0 < count; c0 += chunk) {
    const int64_t nc = std::min(chunk, count - c0);
    const float* src = pixels + (first + c0) * (int64_t)n * n;
    if (!is_device) {
      CK(cudaMemcpyAsync(pix_tmp, src, nc * pix_bytes, cudaMemcpyHostToDevice, s));
      src = pix_tmp;
    }
    float2* pol = fb ? pol_tmp : polar_out + c0 * (int64_t)P.n_k * P.n_psi;
    prof_begin(plan, 0, s);
    launch_polar_from_pixels(plan->nu, src, nc, pol, P.n_psi, scratch, s);
    if (fb) launch_ring_fft(pol, fb + c0 * (int64_t)P.n_k * P.n_psi, nc, P, s);
    prof_end(plan, 0, s);
    CK(cudaGetLastError());
  }
  return FTK_OK;
}

static ftk_status_t load_images_any(ftk_plan_t plan, const void* polar_c64, int64_t N, int is_device, void* stream,
                                    bool pixels) {
  if (!plan) return FTK_EINVAL;
  if (plan->device < 0) return fail(plan, FTK_ESTATE, "host-only plan");
  if (!polar_c64 || N <= 0) return fail(plan, FTK_EINVAL, "ftk_load_images: null pointer or N <= 0");
  CK(cudaSetDevice(plan->device));
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = (size_t)N * plan->pm.n_k * plan->pm.n_psi * sizeof(float2);
  if (N != plan->n_im) {
    cudaFree(plan->d_A);
    plan->d_A = nullptr;
    CK(cudaMalloc(&plan->d_A, bytes));
  }
  plan->n_im = N;
  ftk_status_t st = pixels ? pixels_chunked(plan, reinterpret_cast<const float*>(polar_c64), 0, N, is_device, nullptr,
                                            plan->d_A, s)
                           : load_set(plan, polar_c64, 0, N, is_device, plan->d_A, s);
  if (st != FTK_OK) return st;
  if (plan->engine == 0) {
    std::string msg;
    int ts = tc_prepare_images(plan->tc, plan->d_A, N, devplan(plan), s, msg);
    if (ts != FTK_OK) return fail(plan, (ftk_status_t)ts, msg);
  }
  plan->have_images = true;
  return FTK_OK;
}

static ftk_status_t load_templates_any(ftk_plan_t plan, const void* polar_c64, int64_t N_total, int is_device,
                                       void* stream, bool pixels) {
  if (!plan) return FTK_EINVAL;
  if (plan->device < 0) return fail(plan, FTK_ESTATE, "host-only plan");
  if (!polar_c64 || N_total <= 0) return fail(plan, FTK_EINVAL, "ftk_load_templates: null pointer or N <= 0");
  CK(cudaSetDevice(plan->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t lo = (int64_t)plan->rank * N_total / plan->world;
  const int64_t hi = (int64_t)(plan->rank + 1) * N_total / plan->world;
  const int64_t nl = hi - lo;
  const double flat_max = (double)N_total * plan->pm.N_t * plan->n_gamma;
  if (flat_max > 4294967295.0)
    return fail(plan, FTK_ECAPACITY, "N_templates * N_t * n_gamma exceeds the 32-bit argmax index");
  if (nl != plan->n_tm_local) {
    cudaFree(plan->d_B);
    plan->d_B = nullptr;
    if (nl > 0) CK(cudaMalloc(&plan->d_B, (size_t)nl * plan->pm.n_k * plan->pm.n_psi * sizeof(float2)));
  }
  plan->n_tm_total = N_total;
  plan->n_tm_local = nl;
  plan->tm_off = lo;
  if (nl > 0) {
    ftk_status_t st = pixels ? pixels_chunked(plan, reinterpret_cast<const float*>(polar_c64), lo, nl, is_device,
                                              nullptr, plan->d_B, s)
                             : load_set(plan, polar_c64, lo, nl, is_device, plan->d_B, s);
    if (st != FTK_OK) return st;
    if (plan->engine == 0) {
      std::string msg;
      int ts = tc_prepare_templates(plan->tc, plan->d_B, nl, devplan(plan), s, msg);
      if (ts != FTK_OK) return fail(plan, (ftk_status_t)ts, msg);
    }
  }
  plan->have_templates = true;
  return FTK_OK;
}

ftk_status_t ftk_load_images(ftk_plan_t plan, const void* polar_c64, int64_t N, int is_device, void* stream) {
  return load_images_any(plan, polar_c64, N, is_device, stream, false);
}
ftk_status_t ftk_load_templates(ftk_plan_t plan, const void* polar_c64, int64_t N_total, int is_device, void* stream) {
  return load_templates_any(plan, polar_c64, N_total, is_device, stream, false);
}
ftk_status_t ftk_load_images_pixels(ftk_plan_t plan, const float* pixels, int64_t N, int is_device, void* stream) {
  return load_images_any(plan, pixels, N, is_device, stream, true);
}
ftk_status_t ftk_load_templates_pixels(ftk_plan_t plan, const float* pixels, int64_t N_total, int is_device,
                                       void* stream) {
  return load_templates_any(plan, pixels, N_total, is_device, stream, true);
}

ftk_status_t ftk_polar_from_pixels(ftk_plan_t plan, const float* pixels, int64_t N, int is_device, void* out_c64,
                                   void* stream) {
  if (!plan) return FTK_EINVAL;
  if (plan->device < 0) return fail(plan, FTK_ESTATE, "host-only plan");
  if (!pixels || !out_c64 || N <= 0) return fail(plan, FTK_EINVAL, "ftk_polar_from_pixels: null pointer or N <= 0");
  if (!is_device_ptr(out_c64)) return fail(plan, FTK_EINVAL, "ftk_polar_from_pixels: out must be a device pointer");
  CK(cudaSetDevice(plan->device));
  return pixels_chunked(plan, pixels, 0, N, is_device, reinterpret_cast<float2*>(out_c64), nullptr,
                        (cudaStream_t)stream);
}

ftk_status_t ftk_fb_coeffs(ftk_plan_t plan, int which, int64_t first, int64_t count, void* out_c64, void* stream) {
  if (!plan || !out_c64) return FTK_EINVAL;
  const float2* src = which == 0 ? plan->d_A : plan->d_B;
  const int64_t n = which == 0 ? plan->n_im : plan->n_tm_local;
  if (!src || first < 0 || count < 0 || first + count > n) return fail(plan, FTK_EINVAL, "ftk_fb_coeffs: range");
  CK(cudaSetDevice(plan->device));
  launch_fb_export(src, first, count, plan->pm.n_k, plan->pm.n_psi, reinterpret_cast<float2*>(out_c64),
                   (cudaStream_t)stream);
  CK(cudaGetLastError());
  return FTK_OK;
}

static ftk_status_t ensure_ws(ftk_plan_t plan, size_t bytes) {
  if (plan->ws_size >= bytes) return FTK_OK;
  cudaFree(plan->d_ws);
  plan->d_ws = nullptr;
  plan->ws_size = 0;
  CK(cudaMalloc(&plan->d_ws, bytes));
  CK(cudaMemset(plan->d_ws, 0, bytes));
  plan->ws_size = bytes;
  return FTK_OK;
}

// Run Steps 1-3 on one pair block with the selected engine.
static ftk_status_t run_block(ftk_plan_t plan, const PairBlock& pb, unsigned long long* img_keys,
                              unsigned long long* pair_keys, float* land, cudaStream_t s) {
  const DevPlan P = devplan(plan);
  if (plan->engine == 1) {
    float2* Zhat = reinterpret_cast<float2*>(plan->d_ws);
    float* Z3 = reinterpret_cast<float*>(Zhat + (size_t)pb.count * P.H_plus * P.n_psi);
    prof_begin(plan, 1, s);
    launch_step1_simt(plan->d_A, plan->d_B, Zhat, pb, P, s);
    prof_end(plan, 1, s);
    prof_begin(plan, 2, s);
    launch_step2_simt(Zhat, Z3, pb, P, s);
    prof_end(plan, 2, s);
    prof_begin(plan, 3, s);
    launch_step3_simt(Z3, pb, P, (int)plan->tm_off, img_keys, pair_keys, (int)plan->n_tm_local, land, s);
    prof_end(plan, 3, s);
  } else {
    std::string msg;
    int ts = tc_run_block(plan->tc, pb, P, plan->d_A, plan->d_B, plan->d_ws, plan->ws_size, (int)plan->tm_off, img_keys, pair_keys,
                          (int)plan->n_tm_local, land, s, plan->prof ? &prof_begin_tc : nullptr, plan, msg);
    if (ts != FTK_OK) return fail(plan, (ftk_status_t)ts, msg);
  }
  CK(cudaGetLastError());
  return FTK_OK;
}

static size_t bytes_per_pair(ftk_plan_t plan) {
  const DevPlan P = devplan(plan);
  if (plan->engine == 1) return (size_t)P.H_plus * P.n_psi * sizeof(float2) + (size_t)P.K3p * P.n_psi * sizeof(float);
  return tc_bytes_per_pair(plan->tc, P);
}

// All pair blocks of the (images x local templates) job through run_block (workspace-sized blocks).
static ftk_status_t run_blocks(ftk_plan_t plan, unsigned long long* img_keys, unsigned long long* pair_keys,
                               float* landscape, cudaStream_t s) {
  const DevPlan P = devplan(plan);
  const int64_t NI = plan->n_im, NJ = plan->n_tm_local;
  if (NJ > 0) {
    const size_t per = bytes_per_pair(plan);
    size_t wsb = plan->ws_bytes;
    if (!plan->ws_user && plan->engine == 0) {
      // tensor-core engine: large pair blocks amortize the generated Step-1 operand; take up to half of
      // the free device memory, at most 24 GiB
      size_t fr = 0, tot = 0;
      CK(cudaMemGetInfo(&fr, &tot));
      wsb = std::min<size_t>((size_t)24 << 30, (fr + plan->ws_size) / 2);
      wsb = std::max<size_t>(wsb, (size_t)1 << 30);
    }
    int64_t cap = (int64_t)(wsb / per);
    if (cap < 1) cap = 1;
    if (cap > (1 << 24)) cap = 1 << 24;
    int64_t nj = std::min<int64_t>(NJ, cap);
    int64_t ni = std::max<int64_t>(1, std::min<int64_t>(NI, cap / nj));
    ftk_status_t st = tc_block_shape(plan->tc, P, plan->engine, NI, NJ, cap, ni, nj, landscape != nullptr);
    if (st != FTK_OK) return fail(plan, st, "block shape");
    // landscape rows are addressed as [image][template]: every block must span the full template range
    // (checked after the engine's block shape, which may narrow nj)
    if (landscape && nj < NJ)
      return fail(plan, FTK_ECAPACITY, "landscape output needs workspace for a full template row");
    st = ensure_ws(plan, (size_t)(ni * nj) * per + 4096);
    if (st != FTK_OK) return st;
    for (int64_t i0 = 0; i0 < NI; i0 += ni) {
      for (int64_t j0 = 0; j0 < NJ; j0 += nj) {
        PairBlock pb;
        pb.i0 = (int)i0;
        pb.ni = (int)std::min(ni, NI - i0);
        pb.j0 = (int)j0;
        pb.nj = (int)std::min(nj, NJ - j0);
        pb.li = pb.lj = nullptr;
        pb.count = pb.ni * pb.nj;
        float* land = landscape ? landscape + (size_t)i0 * NJ * P.N_t * P.n_gamma : nullptr;
        st = run_block(plan, pb, img_keys, pair_keys, land, s);
        if (st != FTK_OK) return st;
      }
    }
  }
  return FTK_OK;
}

ftk_status_t ftk_align(ftk_plan_t plan, ftk_best_t* best, ftk_best_t* pair_best, float* landscape,
                       int64_t landscape_capacity, void* stream) {
  if (!plan || !best) return FTK_EINVAL;
  if (plan->device < 0) return fail(plan, FTK_ESTATE, "host-only plan");
  if (!plan->have_images || !plan->have_templates)
    return fail(plan, FTK_ESTATE, "ftk_align called before ftk_load_images and ftk_load_templates");
  CK(cudaSetDevice(plan->device));
  cudaStream_t s = (cudaStream_t)stream;
  const DevPlan P = devplan(plan);
  const int64_t NI = plan->n_im, NJ = plan->n_tm_local;
  if (landscape && landscape_capacity < NI * NJ * P.N_t * (int64_t)P.n_gamma)
    return fail(plan, FTK_ECAPACITY, "landscape buffer too small");
  if (plan->keys_cap < NI * (pair_best ? NJ + 1 : 1)) {
    cudaFree(plan->d_keys);
    plan->d_keys = nullptr;
    plan->keys_cap = NI * (NJ + 1);
    CK(cudaMalloc(&plan->d_keys, plan->keys_cap * sizeof(unsigned long long)));
  }
  unsigned long long* img_keys = plan->d_keys;
  unsigned long long* pair_keys = pair_best ? plan->d_keys + NI : nullptr;
  CK(cudaMemsetAsync(plan->d_keys, 0, NI * (pair_best ? NJ + 1 : 1) * sizeof(unsigned long long), s));
  {
    const ftk_status_t st = run_blocks(plan, img_keys, pair_keys, landscape, s);
    if (st != FTK_OK) return st;
  }
  const bool host_out = !is_device_ptr(best);
  const bool gather = plan->nccl_comm != nullptr;  // world = 1 too (the collective path is then a copy)
  if (plan->best_tmp_cap < NI) {
    cudaFree(plan->d_best_tmp);
    plan->d_best_tmp = nullptr;
    CK(cudaMalloc(&plan->d_best_tmp, NI * sizeof(ftk_best_t)));
    plan->best_tmp_cap = NI;
  }
  prof_begin(plan, 4, s);
  launch_finalize(img_keys, NI, P.N_t, P.n_gamma, (host_out || gather) ? plan->d_best_tmp : best, s);
  if (pair_best) launch_finalize(pair_keys, NI * NJ, P.N_t, P.n_gamma, pair_best, s);
  prof_end(plan, 4, s);
  CK(cudaGetLastError());
  if (gather) {
    // shard merge: all-gather the N_im x 16 B records of every rank over NVLink, then the
    // deterministic device merge (max value, ties -> smallest (template, shift, rot)) into the output
    if (plan->gather_cap < NI * plan->world) {
      cudaFree(plan->d_gather);
      plan->d_gather = nullptr;
      plan->gather_cap = 0;
      CK(cudaMalloc(&plan->d_gather, (size_t)NI * plan->world * sizeof(ftk_best_t)));
      plan->gather_cap = NI * plan->world;
    }
    std::string msg;
    const int gs = nccl_allgather_bests(plan->nccl_comm, plan->d_best_tmp, plan->d_gather, NI, s, msg);
    if (gs != FTK_OK) return fail(plan, (ftk_status_t)gs, msg);
    if (host_out) {
      launch_merge(plan->d_gather, plan->world, NI, plan->d_best_tmp, s);
    } else {
      launch_merge(plan->d_gather, plan->world, NI, best, s);
    }
    CK(cudaGetLastError());
  }
  if (host_out) {
    CK(cudaMemcpyAsync(best, plan->d_best_tmp, NI * sizeof(ftk_best_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return FTK_OK;
}

ftk_status_t ftk_align_marginal(ftk_plan_t plan, double tau, float* log_marginal, void* stream) {
  if (!plan || !log_marginal) return FTK_EINVAL;
  if (!(tau > 0.0) || !std::isfinite(tau)) return fail(plan, FTK_EINVAL, "tau must be positive and finite");
  if (plan->device < 0) return fail(plan, FTK_ESTATE, "host-only plan");
  if (!plan->have_images || !plan->have_templates)
    return fail(plan, FTK_ESTATE, "ftk_align_marginal called before ftk_load_images and ftk_load_templates");
  if (plan->engine != 0) return fail(plan, FTK_EINVAL, "the marginalization epilogue runs on the tensor-core engine");
  if (!is_device_ptr(log_marginal)) return fail(plan, FTK_EINVAL, "log_marginal must be a device pointer");
  CK(cudaSetDevice(plan->device));
  cudaStream_t s = (cudaStream_t)stream;
  plan->tc.marg = log_marginal;
  plan->tc.marg_scale = (float)(1.4426950408889634 / tau);
  plan->tc.marg_part = nullptr;
  plan->tc.marg_np = plan->n_im * plan->n_tm_local;
  // partial (max, sum) sets merged by tc_marg_finalize: k_step3_tc with G > 1 rep-groups writes one per
  // group; the fused k_step23 one per (group, CTA of the pair) (each CTA sees half of the rotations)
  const DevPlan P0 = devplan(plan);
  plan->tc.marg_sets = (tc_s23_eligible(plan->tc, P0) || tc_s3v2_eligible(plan->tc, P0))
                           ? 2 * plan->tc.s23_G
                           : (plan->tc.G > 1 ? plan->tc.G : 0);
  if (plan->tc.marg_sets > 0 && plan->tc.marg_np > 0) {
    const size_t need = (size_t)plan->tc.marg_sets * plan->tc.marg_np * sizeof(float2);
    if (plan->marg_part_bytes < need) {
      cudaFree(plan->d_marg_part);
      plan->d_marg_part = nullptr;
      plan->marg_part_bytes = 0;
      CK(cudaMalloc(&plan->d_marg_part, need));
      plan->marg_part_bytes = need;
    }
    plan->tc.marg_part = reinterpret_cast<float2*>(plan->d_marg_part);
  }
  ftk_status_t st = run_blocks(plan, nullptr, nullptr, nullptr, s);
  if (st == FTK_OK) tc_marg_finalize(plan->tc, s);
  plan->tc.marg = nullptr;
  plan->tc.marg_part = nullptr;
  plan->tc.marg_scale = 0.f;
  if (st != FTK_OK) return st;
  CK(cudaGetLastError());
  return FTK_OK;
}

ftk_status_t ftk_landscape_pairs(ftk_plan_t plan, const int32_t* img_idx, const int32_t* tpl_idx, int n_pairs,
                                 float* out, int64_t out_capacity, void* stream) {
  if (!plan || !img_idx || !tpl_idx || !out || n_pairs <= 0) return FTK_EINVAL;
  if (plan->device < 0) return fail(plan, FTK_ESTATE, "host-only plan");
  if (!plan->have_images || !plan->have_templates) return fail(plan, FTK_ESTATE, "load images and templates first");
  CK(cudaSetDevice(plan->device));
  cudaStream_t s = (cudaStream_t)stream;
  const DevPlan P = devplan(plan);
  const int64_t land_pp = (int64_t)P.N_t * P.n_gamma;
  if (out_capacity < (int64_t)n_pairs * land_pp)
    return fail(plan, FTK_ECAPACITY, "ftk_landscape_pairs: out holds fewer than n_pairs * N_t * n_gamma floats");
  // indices: host or device arrays; validated on the host (an out-of-range index would address memory
  // outside the loaded sets)
  std::vector<int32_t> hi(n_pairs), hj(n_pairs);
  CK(cudaMemcpyAsync(hi.data(), img_idx, n_pairs * sizeof(int32_t), cudaMemcpyDefault, s));
  CK(cudaMemcpyAsync(hj.data(), tpl_idx, n_pairs * sizeof(int32_t), cudaMemcpyDefault, s));
  CK(cudaStreamSynchronize(s));
  for (int k = 0; k < n_pairs; ++k)
    if (hi[k] < 0 || hi[k] >= plan->n_im || hj[k] < 0 || hj[k] >= plan->n_tm_local)
      return fail(plan, FTK_EINVAL, "ftk_landscape_pairs: pair index out of range");
  const size_t per = bytes_per_pair(plan);
  if (plan->engine == 0) {
    ftk_status_t st = ensure_ws(plan, (size_t)128 * per + 4096);
    if (st != FTK_OK) return st;
    std::string msg;
    const int ts = tc_landscape_pairs(plan->tc, P, plan->d_B, hi.data(), hj.data(), n_pairs, plan->n_im,
                                      (int)plan->tm_off, (int)plan->n_tm_local, plan->d_ws, out, s, msg);
    if (ts != FTK_OK) return fail(plan, (ftk_status_t)ts, msg);
    return FTK_OK;
  }
  // SIMT engine: explicit pair blocks through run_block (device copies of the indices)
  int64_t cap = std::max<int64_t>(1, (int64_t)(plan->ws_bytes / per));
  const int64_t chunk = std::min<int64_t>(cap, n_pairs);
  ftk_status_t st = ensure_ws(plan, (size_t)chunk * per + 4096 + (size_t)2 * n_pairs * sizeof(int32_t));
  if (st != FTK_OK) return st;
  int32_t* d_idx = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(plan->d_ws) + (size_t)chunk * per + 4096);
  CK(cudaMemcpyAsync(d_idx, hi.data(), n_pairs * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_idx + n_pairs, hj.data(), n_pairs * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  for (int64_t p0 = 0; p0 < n_pairs; p0 += chunk) {
    PairBlock pb;
    pb.i0 = pb.j0 = 0;
    pb.ni = pb.nj = 1;
    pb.li = d_idx + p0;
    pb.lj = d_idx + n_pairs + p0;
    pb.count = (int)std::min<int64_t>(chunk, n_pairs - p0);
    st = run_block(plan, pb, nullptr, nullptr, out + p0 * land_pp, s);
    if (st != FTK_OK) return st;
  }
  CK(cudaStreamSynchronize(s));  // the host index copies must outlive the asynchronous uploads
  return FTK_OK;
}

ftk_status_t ftk_merge_bests(const ftk_best_t* gathered, int world, int64_t N_im, ftk_best_t* out, void* stream) {
  if (!gathered || !out || world <= 0 || N_im < 0) return FTK_EINVAL;
  launch_merge(gathered, world, N_im, out, (cudaStream_t)stream);
  return cudaGetLastError() == cudaSuccess ? FTK_OK : FTK_ECUDA;
}

ftk_status_t ftk_merge_bests_host(const ftk_best_t* gathered, int world, int64_t N_im, ftk_best_t* out) {
  if (!gathered || !out || world <= 0 || N_im < 0) return FTK_EINVAL;
  for (int64_t i = 0; i < N_im; ++i) {
    ftk_best_t b = gathered[i];
    for (int r = 1; r < world; ++r)
      if (best_better(gathered[(int64_t)r * N_im + i], b)) b = gathered[(int64_t)r * N_im + i];
    out[i] = b;
  }
  return FTK_OK;
}

ftk_status_t ftk_nccl_unique_id(void* id_out) {
  if (!id_out) return FTK_EINVAL;
  std::string msg;
  const int st = nccl_unique_id(id_out, msg);
  if (st != FTK_OK) fprintf(stderr, "ftk_nccl_unique_id: %s\n", msg.c_str());
  return (ftk_status_t)st;
}

ftk_status_t ftk_nccl_comm_create(const void* id, int world, int rank, int device, void** comm_out) {
  if (!id || !comm_out || world <= 0 || rank < 0 || rank >= world) return FTK_EINVAL;
  *comm_out = nullptr;
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return FTK_ENODEV;
  }
  std::string msg;
  const int st = nccl_comm_create(id, world, rank, comm_out, msg);
  if (st != FTK_OK) fprintf(stderr, "ftk_nccl_comm_create: %s\n", msg.c_str());
  return (ftk_status_t)st;
}

ftk_status_t ftk_nccl_comm_destroy(void* comm) { return (ftk_status_t)nccl_comm_destroy(comm); }

ftk_status_t ftk_tc_selftest(int device, double* err_ts, double* err_ss) {
  if (!err_ts || !err_ss) return FTK_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return FTK_ENODEV;
  std::string msg;
  int st = tc_selftest(err_ts, err_ss, msg);
  if (st != FTK_OK) fprintf(stderr, "ftk_tc_selftest: %s\n", msg.c_str());
  return (ftk_status_t)st;
}

ftk_status_t ftk_set_profiling(ftk_plan_t plan, int enabled) {
  if (!plan) return FTK_EINVAL;
  plan->prof = enabled != 0;
  prof_reset(plan);
  return FTK_OK;
}

ftk_status_t ftk_kernel_times(ftk_plan_t plan, double* ms, int64_t* launches) {
  if (!plan || !ms || !launches) return FTK_EINVAL;
  if (plan->device >= 0) CK(cudaSetDevice(plan->device));
  for (int c = 0; c < 5; ++c) {
    double tot = 0;
    for (size_t k = 0; k < plan->ev_used[c]; ++k) {
      float v = 0;
      CK(cudaEventSynchronize(plan->ev[c][k].second));
      CK(cudaEventElapsedTime(&v, plan->ev[c][k].first, plan->ev[c][k].second));
      tot += v;
    }
    ms[c] = tot;
    launches[c] = (int64_t)plan->ev_used[c];
  }
  return FTK_OK;
}

}  // extern "C"

// profiling callback used by the tensor-core engine (class c, begin/end)
void prof_begin_tc(void* plan_v, int cls, int end, cudaStream_t s) {
  ftk_plan_t p = reinterpret_cast<ftk_plan_t>(plan_v);
  if (end)
    prof_end(p, cls, s);
  else
    prof_begin(p, cls, s);
}
