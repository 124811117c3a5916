// Tensor-core (tcgen05, fp16x3 split with power-of-two scaling) engine of the FTK hot path.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "ftk_internal.cuh"
#include "ftk_plan_math.h"

namespace ftk {

// Step-2 work blocks: 1 or 2 consecutive 8-column word groups of the Step-3 operand holding <= 8 terms
struct S2BlockTable {
  int nb;
  int zs[16], ze[16];  // term range of block b (device term order)
  int g0[16], ng[16];  // first word group, number of groups
  int used[16];        // words (bit grp * 4 + w) written by some term
  int lone[16];        // terms (bit z - zs) with ell = 0 and no neighbour in their word
};

// Step 2 on the tensor cores (k_step2_tc, n_gamma = n_psi = 512): per Step-2 block, one slot per Step-3 operand
// word (word group grp, word w -> slot 4 grp + w).  kind 0: no term (the word is zero); kind 1: an ell > 0 term at
// window column e1, cyclic shift ell (word = (Re Z, Im Z)); kind 2: ell = 0 terms at window columns e1 (low half)
// and e2 (high half), either may be absent (-1), transformed together as x_e1 + i x_e2 (both Z are real).
// info = kind | e1 << 4 | e2 << 8 | ell << 16 (window columns 0..7, 15 = absent); mask: bits of the word kept;
// needmask[b]: some word of block b keeps only one half (a lone ell = 0 term)
struct S2TSlotTable {
  uint32_t info[16][8];
  uint32_t mask[16][8];
  int needmask[16];
};

struct TcPlan {
  static constexpr int MAXG = 16;  // max rep-groups (Y slices) of Step 3
  bool ready = false;
  int K3p = 0;          // Step-3 contraction length padded to a multiple of 16
  int n_rep = 0;        // representative shifts (+-delta pairs share one column pair E/O)
  int Ke = 0;           // even-ell column block length
  // Step 3 (k_step3_tc): columns = representative shifts in rep-groups of nch[g] chunks of NCH
  int NCH = 0, G = 0, NRT = 0, ncol = 0, NS = 1;  // NS: Step-3 staging ring depth
  int g_col0[MAXG] = {0}, g_nch[MAXG] = {0};
  long long g_yoff[MAXG] = {0};
  int* d_colrep = nullptr;
  int* d_colpart = nullptr;
  uint8_t* d_colfast = nullptr;
  uint8_t* d_Ysm = nullptr;   // per group: shared-memory image of Y3 hi/lo (B operand)
  size_t s3_smem = 0;
  // Step 1 operands
  uint8_t* d_Aop = nullptr;    // images, fp16 hi/lo split (scaled), Step-1 K-major tiles [p][tile][kchunk][part]...
  size_t aop_bytes = 0;
  int NIT = 0, KCH = 64, NKCH = 0;
  S2BlockTable s2_blocks;     // Step-2 work blocks
  float2* d_s2tw = nullptr;  // Step-2 four-step twiddle tables
  // k_step2_tc (tensor-core Step 2, n = 512): DFT-64 matrix as the TMEM A operand ([128 rows][64 hi + 64 lo words]),
  // radix-8 twiddles [64 a][8 c], per-block slot table; s2tc: 1 when this plan runs it (FTK_S2TC != 0, n = 512)
  uint32_t* d_s2F = nullptr;
  float2* d_s2w = nullptr;
  S2TSlotTable s2t;
  int s2tc = 0;
  int s1cg2 = 0;  // (opt-in FTK_S1CG2=1) k_step1_cg2: CTA pairs, half of every image stage per SM
  int64_t n_tm = 0;
  // fp16x3 power-of-two operand scaling (ftk_tc.cu header): per-item maxima of the loaded images / local templates
  // (x = max |Re|, |Im| of the FB coefficients, y = their Frobenius norm), gmax = max |g_zeta(k_m)|, eY = the
  // exponent of the Step-3 Y3 operand
  float2* d_ast = nullptr;  // images: (max |Re|, |Im|, ||a||_F) per item
  float2* d_bst = nullptr;  // local templates, likewise
  int64_t ast_cap = 0, bst_cap = 0;
  float gmax = 0.f;
  int eY = 0;
  int num_sms = 148;
  bool sync_debug = false;
  // FTK_POISON=<byte> (tests, an initcheck / racecheck stand-in): before every pair block the workspace, and before
  // every Steps 1-3 launch the shared memory and TMEM of every SM, are filled with this byte (-1: off)
  int poison = -1;
  // FTK_ONLY_STEP=1|2|3 (power / clock experiments only; results are garbage): run just that step's kernel
  int only_step = 0;
  int only_primed = 0;  // blocks run so far under FTK_ONLY_STEP (the first one runs every step)
  // Step-3 epilogue of the next tc_run_block calls: marg == nullptr -> max / argmax (MODE 0); else the
  // marginalization epilogue (MODE 1) writes log sum exp(X / tau) per pair to marg[i][j], marg_scale =
  // log2(e) / tau
  float* marg = nullptr;
  float marg_scale = 0.f;
  // G > 1 rep-groups: each group's CTAs see only part of the shifts, so MODE 1 writes per-group base-2
  // (max, sum) partials to marg_part[group][i][j] (marg_np = N_im x n_tm_local) and tc_marg_finalize
  // merges them into marg
  float2* marg_part = nullptr;
  int64_t marg_np = 0;
  int marg_sets = 0;  // partial sets merged by tc_marg_finalize (G for k_step3_tc, 2 G' for k_step23)
  // fused Steps 2 + 3 (ftk_s23.cu, k_step23): CTA pairs, rep-groups of its own (each CTA holds half of a
  // group's Y image), FFT length F = n / D per rotation tile
  bool s23_ready = false;   // fused Steps 2 + 3 (opt-in, FTK_S23=1)
  bool s3v2_ready = false;  // Step-3-only CTA-pair kernel (opt-in, FTK_S3V2=1)
  size_t s3v2_smem = 0;
  int s3v2_NRT = 0;
  int s23_G = 0, s23_nch = 0, s23_NCH = 0, s23_F = 0, s23_D = 0, s23_ncol = 0;
  int s23_col0[MAXG] = {0};
  long long s23_yoff[MAXG] = {0};
  long long s23_yhalf = 0;
  int* d_s23_colrep = nullptr;
  int* d_s23_colpart = nullptr;
  uint8_t* d_s23_colfast = nullptr;
  uint8_t* d_s23_Ysm = nullptr;
  float2* d_s23_tw = nullptr;
  size_t s23_smem = 0;
};

typedef void (*prof_cb_t)(void* plan, int cls, int end, cudaStream_t s);

// fused Steps 2 + 3 (ftk_s23.cu).  tc_s23_init leaves s23_ready false (no error) for shapes it does not cover
// (n_gamma != n_psi, n_psi outside {128, 256, 512}, Y halves that do not fit); those run k_step2_fft + k_step3_tc.
int tc_s23_init(TcPlan& tc, int n_psi, int n_gamma, const std::vector<int>& rep, const std::vector<int>& partner,
                const std::vector<float>& Y3, int K3p, bool fused, std::string& msg);
void tc_s23_free(TcPlan& tc);
bool tc_s23_eligible(const TcPlan& tc, const DevPlan& P);
bool tc_s3v2_eligible(const TcPlan& tc, const DevPlan& P);
// Step 3 on the CTA-pair kernel from k_step2_fft's operand images (same contract as launch_step3_tc)
int launch_step3_cg2(const TcPlan& tc, const uint8_t* Zop, const PairBlock& pb, const DevPlan& P, int tm_off,
                     unsigned long long* img_keys, unsigned long long* pair_keys, int n_tm_local, float* land,
                     cudaStream_t s);
int launch_step23(const TcPlan& tc, const float2* Zhat, const PairBlock& pb, const DevPlan& P, int tm_off,
                  unsigned long long* img_keys, unsigned long long* pair_keys, int n_tm_local, float* land,
                  cudaStream_t s);

// log-sum-exp merge of the G rep-group partials of ftk_align_marginal (see TcPlan::marg_part)
void tc_marg_finalize(const TcPlan& tc, cudaStream_t s);

int s2_block_table(const std::vector<int>& ell, const std::vector<int>& col, int K3p, S2BlockTable& t,
                   std::string& msg);
// Device term order for the tensor-core engine (see ftk_tc.cu); perm[new z] = old z.
int tc_term_order(const std::vector<int>& ell, const std::vector<int>& col, int K3p, std::vector<int>& perm,
                  std::string& msg);
int tc_plan_init(TcPlan& tc, const PlanMath& pm, const std::vector<float>& g, const std::vector<int>& ell,
                 const std::vector<int>& col, const std::vector<float>& Y3, int K3p, int Ke, int n_gamma,
                 std::string& msg);
void tc_plan_free(TcPlan& tc);
int tc_prepare_images(TcPlan& tc, const float2* fb, int64_t n, const DevPlan& P, cudaStream_t s, std::string& msg);
int tc_prepare_templates(TcPlan& tc, const float2* fb, int64_t n, const DevPlan& P, cudaStream_t s, std::string& msg);
size_t tc_bytes_per_pair(const TcPlan& tc, const DevPlan& P);
ftk_status_t tc_block_shape(const TcPlan& tc, const DevPlan& P, int engine, int64_t NI, int64_t NJ, int64_t cap,
                            int64_t& ni, int64_t& nj, bool full_rows = false);
int tc_selftest(double* err_ts, double* err_ss, std::string& msg);
// ftk_landscape_pairs on the tensor-core engine (production Step-1/2/3 kernels on minimal blocks); h_img /
// h_tpl: host copies of the pair indices (validated by the caller); ws >= 128 pairs of tc_bytes_per_pair
int tc_landscape_pairs(TcPlan& tc, const DevPlan& P, const float2* B, const int32_t* h_img, const int32_t* h_tpl,
                       int n_pairs, int64_t n_im, int tm_off, int n_tm_local, void* ws, float* out, cudaStream_t s,
                       std::string& msg);
int tc_run_block(TcPlan& tc, const PairBlock& pb, const DevPlan& P, const float2* A, const float2* B, void* ws,
                 size_t ws_size, int tm_off,
                 unsigned long long* img_keys, unsigned long long* pair_keys, int n_tm_local, float* land,
                 cudaStream_t s, prof_cb_t prof, void* plan, std::string& msg);

// fill ws (if non-null) and every SM's shared memory and TMEM with the byte tc.poison (no-op when off)
void tc_poison(const TcPlan& tc, void* ws, size_t ws_bytes, cudaStream_t s);

}  // namespace ftk

void prof_begin_tc(void* plan_v, int cls, int end, cudaStream_t s);
