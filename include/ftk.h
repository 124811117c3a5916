/*
 * ftk.h -- C ABI of the B200-native FTK alignment hot path.
 *
 * Method: Rangan, Spivak, Andén, Barnett, "Factorization of the translation kernel for
 * fast rigid image alignment" (arXiv:1905.12317).  "P:n" = line n of the paper text
 * with its section / equation label.
 *
 * What is computed (Eq. Xtrunc P:492-496 evaluated by Eq. fbk3): for every image A_i
 * and template B_j, the bandlimited inner products
 *     X_ij(delta_t, gamma_r) = < R_gamma T_delta A_i , B_j >_{Omega_K}      (Eq. Xdg)
 * over all N_t user shifts delta_t and all n_psi rotations gamma_r = 2 pi r / n_psi, using the
 * Fourier-Bessel representation (Eq. aqkcalc) and the eps-truncated operator SVD of the
 * translation kernel (Eqs. Jsvd/svdtrunc).  Per image the library returns the maximal
 * value and its (template, shift, rotation) (the consistency check of P:1324); small cases may
 * also request every per-pair maximum or the full landscape.
 *
 * Units and conventions
 *   - Lengths in pixels, frequencies in rad/px.  K is given in cycles per image width (the
 *     BASELINE.json configs use K = n/2, i.e. Nyquist): k_max = 2 pi K / n.
 *   - Input images/templates are polar Fourier samples  Ahat(k_m, psi_p)  with the sign convention
 *     Ahat(k) = int A(x) exp(-i k.x) dx (Eq. Ahat), k_m from ftk_plan_radial(),
 *     psi_p = 2 pi p / n_psi.  Layout: complex64 (re, im float pairs), [N][n_k][n_psi], psi fastest.
 *   - Images are assumed REAL (Hermitian samples: Ahat(k, psi + pi) = conj Ahat(k, psi)); the
 *     library uses the exact symmetry of DESIGN.md reading R13 to evaluate only ell >= 0 terms.
 *   - Shift index t = position in the caller's shift list; rotation index r <-> gamma_r.
 *     X(delta, gamma) rotates/translates the IMAGE: a planted image T_d0 R_g0 B peaks at
 *     (-d0, -g0).  Values are Re X in the bandlimited convention (no (2 pi)^-2 prefactor).
 *   - Ties in the argmax resolve to the smallest (template, shift, rotation) (lexicographic).
 *
 * Ownership: load calls COPY the caller's buffers; outputs go to caller-allocated buffers; the plan
 * owns its plan factors, Fourier-Bessel arrays and workspace.  A plan is not thread-safe; distinct
 * plans are independent.  Nothing throws across the ABI: every call returns an ftk_status_t and a
 * message is kept in ftk_last_error(plan).
 *
 * Multi-GPU: every rank creates a plan with opts.rank/opts.world and calls the same sequence with
 * the same arguments.  Rank r keeps templates [floor(r N/W), floor((r+1) N/W)); ftk_align reports
 * GLOBAL template indices.  With opts.nccl_comm set (an NCCL communicator of the `world` ranks, e.g.
 * from ftk_nccl_comm_create), ftk_align itself all-gathers the per-image records over NVLink/NVSwitch
 * (one ncclAllGather of N_im x 16 B per rank) and merges them on the device with the same tie-break, so
 * every rank returns the GLOBAL bests.  Without a communicator ftk_align returns this rank's shard-local
 * bests and the caller may gather them itself and reduce with ftk_merge_bests().
 */
#ifndef FTK_H_
#define FTK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ftk_plan_s* ftk_plan_t;   /* opaque */

typedef enum {
  FTK_OK = 0,
  FTK_EINVAL = 1,      /* bad argument (null pointer, non-positive size, unsupported n_psi, ...) */
  FTK_ERANGE = 2,      /* a shift lies outside the disc ||delta|| <= delta_max (Omega_D) */
  FTK_ENUMERIC = 3,    /* plan construction failed a numerical self-check (quadrature, SVD, energy) */
  FTK_ENOMEM = 4,      /* host or device allocation failed */
  FTK_ECUDA = 5,       /* CUDA runtime error (message holds cudaGetErrorString) */
  FTK_ESTATE = 6,      /* wrong call order (e.g. ftk_align before both loads; host-only plan) */
  FTK_ECAPACITY = 7,   /* an optional output buffer is too small, or an index does not fit */
  FTK_ENODEV = 8,      /* no CUDA device / device ordinal invalid */
  FTK_ENCCL = 9        /* NCCL unavailable or an NCCL call failed (message holds ncclGetErrorString) */
} ftk_status_t;

typedef struct {
  int n_k;              /* radial quadrature nodes; 0 -> round(K)  (configs: n_k = K) */
  int n_psi;            /* angles per ring; 0 -> 4 round(K); power of two, 64..1024 */
  int radial_rule;      /* 0 = Gauss-Legendre x k dk (configs), 1 = Gauss-Jacobi(0,1) (paper P:483-490) */
  int device;           /* CUDA ordinal; -1 = host-only plan: plan math + queries, no device memory */
  int rank, world;      /* template shard of this process; world <= 0 is treated as 1 */
  int engine;           /* 0 = tcgen05 fp16x3 tensor-core path (default; each operand scaled by a power of two
                           and split into two fp16 halves, three products, fp32 accumulation: measured
                           |dX| <= 6.2e-7 ||A|| ||B|| against the float64 oracle; Step 2 at
                           n_gamma = n_psi = 512 as a radix-8 register stage plus a DFT-64 fp16x3 GEMM, else a
                           shared-memory FFT), 1 = SIMT fp32 reference kernels.
                           Engine 0 needs n_k a multiple of 16 (<= 128), n_psi a multiple of 64 and a Step-3
                           width K3p <= 224 (K3 = 2 H_plus - H0 plus block padding; plain configs <= 128, wide
                           CTF plans up to 224), else ftk_plan_create returns FTK_EINVAL (use engine 1) */
  int svd_nodes;        /* Nystrom nodes per axis for the operator SVD; 0 -> 96 */
  size_t workspace_bytes;  /* pair-block workspace; 0 -> 1 GiB */
  int n_gamma;          /* rotations gamma_r = 2 pi r / n_gamma; 0 -> n_psi.  n_gamma > n_psi evaluates Step 2
                           as the zero-padded trigonometric sum (DESIGN reading R21); power of two,
                           n_psi <= n_gamma <= 1024, engine 0 only (engine 1 -> FTK_EINVAL) */
  void* nccl_comm;      /* NULL, or an ncclComm_t of `world` ranks in which this process is `rank` (checked
                           at plan creation, FTK_EINVAL on mismatch): ftk_align then returns global bests on
                           every rank (see "Multi-GPU" above).  Not owned by the plan. */
} ftk_plan_opts_t;

/* One per-image (or per-pair) result, 16 bytes. */
typedef struct {
  float value;               /* Re X at the maximum */
  int32_t template_idx;      /* GLOBAL template index (-1 if no template was seen) */
  int32_t shift_idx;         /* index into the caller's shift list */
  int32_t rot_idx;           /* r, gamma_r = 2 pi r / n_gamma (n_gamma = n_psi unless opts.n_gamma is set) */
} ftk_best_t;

typedef struct {
  int n, n_k, n_psi, N_t;
  int H;                     /* total retained terms, both signs of ell */
  int H_plus;                /* retained terms with ell >= 0 (the ones the device evaluates) */
  int H0;                    /* retained terms with ell = 0 */
  int K3;                    /* Step-3 contraction length 2 H_plus - H0 (reading R13) */
  int ell_max;               /* largest |ell| with a retained term */
  double K_cycles, k_max, delta_max, W, eps;
  double certificate;        /* max |F - F^SVD| over (sampled shifts) x (k_m) x (psi_p) */
  int64_t n_images, n_templates_total, n_templates_local, template_offset;
  int engine, device, rank, world;
  int K3p;                   /* device Step-3 width (K3 + block padding; multiple of 16 for engine 0) */
  int n_rep;                 /* engine 0: representative shifts (+-delta pairs share one E/O column pair) */
  int s3_cols;               /* engine 0: Step-3 GEMM N over all rep-groups (n_rep + padding) */
  int s3_nch;                /* engine 0: Step-3 chunk width (MMA N) */
  int s3_groups;             /* engine 0: rep-groups (Y slices resident in shared memory) */
  int s3_rtiles;             /* engine 0: 128-row rotation tiles per pair (MMA M) */
  int n_gamma;               /* rotations per (pair, shift): gamma_r = 2 pi r / n_gamma */
  int n_tau;                 /* CTF plans (ftk_plan_create_ctf): number of filters; 0 for plain plans */
  int N_t_base;              /* the caller's shift count; N_t = N_t_base * max(n_tau, 1) shift entries */
} ftk_plan_info_t;

/* Build the plan (host, double precision, untimed per P:1321): radial rule, per-ell operator SVD of
 * J_ell(delta k) (Nystrom on Gauss-Jacobi(0,1) nodes with a one-sided Jacobi SVD), eps truncation
 * Sigma > eps, global relabel, G_zeta(k_m) and Y_zeta(delta_t) (Eq. svdtrunc), and their
 * device copies.  shifts_xy_px: host [N_t][2] doubles.  Errors: FTK_EINVAL, FTK_ERANGE (any
 * ||delta_t|| > delta_max_px * (1 + 1e-12)), FTK_ENUMERIC, FTK_ENODEV, FTK_ENOMEM, FTK_ECUDA.
 * On error *out is NULL. */
ftk_status_t ftk_plan_create(int n, double K, double delta_max_px, const double* shifts_xy_px,
                             int N_t, double eps, const ftk_plan_opts_t* opts, ftk_plan_t* out);

/* The plan's radial rule without building a plan (host only): k_m, w_m for n_k nodes on [0, k_max],
 * k_max = 2 pi K / n rad/px (reading R1), radial_rule as in ftk_plan_opts_t (sum w = k_max^2/2).
 * k_out, w_out: caller-allocated host double[n_k].  Used to evaluate CTF filters on the nodes before
 * ftk_plan_create_ctf.  Errors: FTK_EINVAL (bad argument), FTK_ENUMERIC. */
ftk_status_t ftk_radial_rule(int n, double K, int n_k, int radial_rule, double* k_out, double* w_out);

/* CTF-parameterized factorized kernel (Sec. 6 "Other 2D kernels"; SURVEY 8(f)
 * NEXT-4; DESIGN reading R24).  The translation kernel times a family of radial filters (contrast
 * transfer functions, one per defocus tau) is factorized as
 *     F(delta, k) c_tau(|k|) ~= sum_zeta Y_zeta(delta, tau) G_zeta(k),   G_zeta(k) = G_zeta(|k|) e^{i ell psi},
 * per Bessel order ell by one SVD over rows (x_i, tau) (Gauss-Jacobi(0,1) nodes in x = K|delta|, weight 1
 * per tau) and columns k_m (the plan's radial rule, weight w_m); Sigma > eps kept.  Alignment then
 * evaluates X(delta_t, gamma_r, tau) = <R_gamma T_delta A, c_tau B> for every filter: the same Steps 1-3
 * with the shift list replaced by the n_tau * N_t "virtual shifts" v = tau * N_t + t (tau-major), so
 * ftk_best_t.shift_idx, landscapes and marginals index v.
 * filters: host double[n_tau][n_k], the real filter values c_tau(k_m) at this plan's radial nodes (see
 * ftk_radial_rule; any real radial filter — the library does not fix a CTF model).  Other arguments and
 * errors as ftk_plan_create; FTK_EINVAL also for n_tau <= 0, filters == NULL, non-finite filter values. */
ftk_status_t ftk_plan_create_ctf(int n, double K, double delta_max_px, const double* shifts_xy_px, int N_t,
                                 int n_tau, const double* filters, double eps, const ftk_plan_opts_t* opts,
                                 ftk_plan_t* out);

void ftk_plan_destroy(ftk_plan_t plan);

ftk_status_t ftk_plan_query(ftk_plan_t plan, ftk_plan_info_t* info);

/* Host copies of plan quantities (caller-allocated host arrays).
 *   radial: k[n_k], w[n_k]                       (sum_m w_m g(k_m) ~ int_0^K g(k) k dk)
 *   terms : ell[H], eta[H] (0-based), sigma[H]   (zeta order: Sigma desc, |ell| asc, ell>0 first, eta asc)
 *   factors: G[H][n_k] = Sigma_zeta V_zeta(k_m) ; Y[N_t][H][2] = (re, im) of Y_zeta(delta_t)   (px units) */
ftk_status_t ftk_plan_radial(ftk_plan_t plan, double* k, double* w);
ftk_status_t ftk_plan_terms(ftk_plan_t plan, int32_t* ell, int32_t* eta, double* sigma);
ftk_status_t ftk_plan_factors(ftk_plan_t plan, double* G, double* Y);

/* Load polar samples and compute their Fourier-Bessel coefficients on the device (ring FFT kernel,
 * Eq. aqkcalc).  polar_c64: [N][n_k][n_psi] complex64, host (is_device = 0; any host memory,
 * pinned is faster) or device (is_device = 1).  stream: cudaStream_t or NULL.  Images: all N are
 * kept.  Templates: N_total is the global count; this rank keeps its shard.  Re-loading replaces the
 * previous set.  Errors: FTK_ESTATE on a host-only plan, FTK_EINVAL, FTK_ENOMEM, FTK_ECUDA. */
ftk_status_t ftk_load_images(ftk_plan_t plan, const void* polar_c64, int64_t N, int is_device, void* stream);
ftk_status_t ftk_load_templates(ftk_plan_t plan, const void* polar_c64, int64_t N_total, int is_device, void* stream);

/* Pixel front end (PAPER.md Sec. "Conversion of discrete input images to the Fourier
 * domain", Eq. Ahattrap, evaluated with a 2-D type-2 NUFFT as in P:531-541):
 *   Ahat(k_m, psi_p) = sum_{i,j < n} A[i][j] exp(-i k_m ((i - n/2) cos psi_p + (j - n/2) sin psi_p))
 * in pixel units (the paper's box [-1, 1]^2 with dx = 2/n, rescaled so that dx = 1 px; R23),
 * psi_p = 2 pi p / n_psi, k_m = the plan's radial nodes (rad/px).  NUFFT: upsampling 2, exponential-of-
 * semicircle kernel of width 7 (relative error ~1e-6 of sum |A|), fp32 arithmetic.
 *   pixels : float32 [N][n][n] (i slow, j fast), n = the plan's image size; host (is_device = 0, copied
 *            in chunks) or device (is_device = 1).  The caller keeps ownership.
 *   ftk_polar_from_pixels: out_c64 = device complex64 [N][n_k][n_psi] (the layout ftk_load_* takes).
 *   ftk_load_images_pixels / ftk_load_templates_pixels: same as ftk_load_images / ftk_load_templates
 *            from pixels (templates: N_total global, this rank keeps its shard); the polar samples are
 *            not materialized beyond one chunk.
 * Errors: FTK_EINVAL (null pointer, N <= 0, n not a power of two, out not a device pointer),
 * FTK_ESTATE (host-only plan), FTK_ENOMEM, FTK_ECUDA.  Asynchronous on `stream`. */
ftk_status_t ftk_polar_from_pixels(ftk_plan_t plan, const float* pixels, int64_t N, int is_device, void* out_c64,
                                   void* stream);
ftk_status_t ftk_load_images_pixels(ftk_plan_t plan, const float* pixels, int64_t N, int is_device, void* stream);
ftk_status_t ftk_load_templates_pixels(ftk_plan_t plan, const float* pixels, int64_t N_total, int is_device,
                                       void* stream);

/* Copy Fourier-Bessel coefficients a(k_m; q) of loaded items [first, first+count) to out_c64
 * (device, [count][n_k][n_psi] complex64, q fastest, q cyclic).  which: 0 images, 1 local templates. */
ftk_status_t ftk_fb_coeffs(ftk_plan_t plan, int which, int64_t first, int64_t count, void* out_c64, void* stream);

/* The hot path: Steps 1-3 over all (image, local template) pairs, fused max/argmax.
 *   best      : [N_im] per-image best over this rank's templates (global indices); host or device
 *               pointer (detected); required.
 *   pair_best : nullable, device, [N_im][N_tm_local] per-pair maxima (template_idx global).
 *   landscape : nullable, device, float [N_im][N_tm_local][N_t][n_gamma] = Re X; landscape_capacity is its
 *               element count (FTK_ECAPACITY if smaller, or if the workspace cannot hold a block spanning
 *               all local templates).
 * With opts.nccl_comm, `best` holds the GLOBAL bests on every rank (all-gather + device merge on `stream`;
 * every rank must call ftk_align); pair_best and landscape stay rank-local.
 * The call is asynchronous on `stream` for device outputs; it synchronizes `stream` when `best` is
 * a host pointer.  Errors: FTK_ESTATE (missing load / host-only plan), FTK_ECAPACITY, FTK_ECUDA,
 * FTK_ENCCL. */
ftk_status_t ftk_align(ftk_plan_t plan, ftk_best_t* best, ftk_best_t* pair_best, float* landscape,
                       int64_t landscape_capacity, void* stream);

/* Marginalization epilogue (the Bayesian use of the whole landscape, PAPER.md
 * P:73-74 "an integral of a probability distribution over shifts and angles is used to marginalize
 * the likelihood"): Steps 1-3 as in ftk_align, with the Step-3 epilogue replaced by
 *   log_marginal[i][j] = log sum_{t < N_t, r < n_gamma} exp(X_ij(delta_t, gamma_r) / tau)
 * (uniform weights on the caller's shift list and the rotation grid; add log of the prior weights
 * outside).  tau > 0 (units of X), finite, else FTK_EINVAL.  log_marginal: device float
 * [N_im][N_tm_local] (j = local template index; rank r's block starts at its template offset),
 * caller-allocated, fully overwritten.  Accuracy: |delta L| <= max |delta X| / tau + fp32 rounding.
 * Tensor-core engine only (FTK_EINVAL on engine 1).  Asynchronous on `stream`.  Errors: FTK_EINVAL,
 * FTK_ESTATE (missing load / host-only plan), FTK_ECUDA. */
ftk_status_t ftk_align_marginal(ftk_plan_t plan, double tau, float* log_marginal, void* stream);

/* Full landscapes for selected pairs (sampled parity at large configs): X_ij(delta_t, gamma_r) of Eq. fbk3
 * for the pairs (img_idx[k], tpl_idx[k]).  img_idx / tpl_idx: int32 [n_pairs], host or device
 * (template index LOCAL to this rank); out: device float [n_pairs][N_t][n_gamma], out_capacity = its
 * element count (FTK_ECAPACITY if < n_pairs * N_t * n_gamma).  Engine 0 runs the production kernels
 * (k_step1_tc over the pair's 128-image tile, the plan's Step-2 kernel, k_step3_tc with landscape output).  Errors:
 * FTK_EINVAL (null pointer, n_pairs <= 0, an index out of range), FTK_ESTATE, FTK_ECAPACITY, FTK_ECUDA.
 * Synchronizes `stream` once (index validation); the kernels are asynchronous on it. */
ftk_status_t ftk_landscape_pairs(ftk_plan_t plan, const int32_t* img_idx, const int32_t* tpl_idx, int n_pairs,
                                 float* out, int64_t out_capacity, void* stream);

/* Deterministic merge of per-rank results: out[i] = best of gathered[r][i] over r (max value, ties ->
 * smallest (template, shift, rot)).  Device pointers; gathered: [world][N_im].  The _host variant
 * does the same on host arrays (no device needed). */
ftk_status_t ftk_merge_bests(const ftk_best_t* gathered, int world, int64_t N_im, ftk_best_t* out, void* stream);
ftk_status_t ftk_merge_bests_host(const ftk_best_t* gathered, int world, int64_t N_im, ftk_best_t* out);

/* Kernel timing hooks for bench.py: when enabled, ftk_align records CUDA events on its stream around
 * each kernel launch; ftk_kernel_times returns, per kernel class (0 load-FFT, 1 step1, 2 step2, 3 step3,
 * 4 finalize), the summed milliseconds and launch counts of the last ftk_align/ftk_load_* calls. */
ftk_status_t ftk_set_profiling(ftk_plan_t plan, int enabled);
ftk_status_t ftk_kernel_times(ftk_plan_t plan, double* ms /*[5]*/, int64_t* launches /*[5]*/);

/* Hardware self-test of the tensor-core primitives (one 128x64x32 bf16 tcgen05.mma with A from TMEM and
 * one with A from shared memory, K-major, plus one with an MN-major B operand) against a host reference: writes the max
 * absolute errors (expected ~1e-6, fp32 accumulation of exactly representable bf16 products). */
ftk_status_t ftk_tc_selftest(int device, double* err_ts, double* err_ss);

/* NCCL communicator helpers (libnccl.so.2 is loaded at run time; FTK_ENCCL if absent).  The usual
 * bootstrap: rank 0 calls ftk_nccl_unique_id, broadcasts the 128 bytes (any channel: torch.distributed,
 * MPI, a file), every rank calls ftk_nccl_comm_create with cudaSetDevice already pointing at its GPU (or
 * passes `device` >= 0), and passes the communicator in ftk_plan_opts_t.nccl_comm.  The caller owns the
 * communicator (ftk_nccl_comm_destroy after the plans that use it).  Errors: FTK_EINVAL (null pointer,
 * bad rank/world), FTK_ENODEV, FTK_ENCCL. */
ftk_status_t ftk_nccl_unique_id(void* id_out /* 128 bytes */);
ftk_status_t ftk_nccl_comm_create(const void* id /* 128 bytes */, int world, int rank, int device, void** comm_out);
ftk_status_t ftk_nccl_comm_destroy(void* comm);

const char* ftk_last_error(ftk_plan_t plan);   /* never NULL; "" when no error */
const char* ftk_status_string(ftk_status_t s);
int ftk_version(void);                          /* 100 * major + minor */

#ifdef __cplusplus
}
#endif
#endif  /* FTK_H_ */
