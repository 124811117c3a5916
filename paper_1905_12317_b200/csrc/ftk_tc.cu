// Tensor-core (tcgen05) engine of the FTK hot path, fp16x3 split arithmetic with power-of-two operand scaling.
//
// Step 3 (PAPER.md Eq. fbk3; real form of DESIGN.md reading R13):
//   X_p(t, r) = sum_k Z3_p[r][k] Y3[t][k],  k < K3 = 2 H_plus - H0,  then max/argmax over (t, r).
// Every operand x is scaled by a power of two into fp16's range and split x = hi + lo in fp16; the product is
// hi*hi + hi*lo + lo*hi with fp32 accumulation in TMEM and the scale removed exactly afterwards (DESIGN.md
// section 6 "fp16x3": 22 significant bits per operand, the accuracy of 3xTF32 at the bf16 MMA rate).
// fp16x3 scaling (all exponents from f16_scale_exp, x 2^e in (2^13, 2^14]):
//   Step-1 image operand  a_i      x 2^{e(amax_i)}            amax_i = max |Re|, |Im| of image i's FB coefficients
//   Step-1 generated operand c_j   x 2^{e(gmax bmax_j)}       gmax = max |g_zeta(k_m)|, bmax_j likewise for template j
//   Step-1 output Zhat'            left scaled: pair (i, j)'s block is Zhat' 2^{e_a(i) + e_c(j)} (one factor per
//                                  pair), which Step 2 folds into its own Z scale (no epilogue work)
//   Step-3 operand Z (pair i, j)   x 2^{e(gmax |a_i| |b_j|)}  |.| = Frobenius norm over (m, p); bounds |Z| by
//                                  |Z_zeta(r)| <= sum_{m,p} |a(m,p)| |g_zeta(m)| |b(m,p+ell)| <= gmax |a| |b|
//                                  (Cauchy-Schwarz; the shift p -> p + ell permutes the modes)
//   Step-3 operand Y3              x 2^{eY}, eY = e(max |Y3|) (plan constant)
//   Step-3 results                 x 2^{-(e_Z + eY)} per pair before keys / landscapes / log-marginals
//
// Kernel k_step3_tc (one CTA per SM, persistent).  GEMM orientation: M = 128 rotations r (one "r-tile"
// of the pair's operand Z3, the A operand, held in TMEM), N = a chunk of NCH representative shifts
// (the B operand Y3, resident in shared memory for the whole kernel), K = K3p.  Shifts are taken in
// +-delta pairs: Y_zeta(-delta) = (-1)^ell Y_zeta(delta), so with the K columns split by the parity of
// ell (even block [0, Ke), odd block [Ke, K3p)) X(+delta) = E + O and X(-delta) = E - O with
// E = Z_even Y_even, O = Z_odd Y_odd accumulated separately: half the shifts, same K.
// Representative shifts are split into rep-groups whose Y image fits in shared memory; CTA b serves
// group b % G for a contiguous range of pairs (G = 1 at the BASELINE configs c2, c3, c5).
//   * warp 1 (one lane): producer -- per (pair, r-tile) one bulk copy of the Step-2 operand image (fp16
//     hi/lo, canonical K-major core matrices) into a shared-memory staging ring.
//   * warp 0 (one elected lane): per r-tile 2 x K3p/16 tcgen05.cp.128x256b staging -> TMEM A slot, then
//     per chunk 3 x K3p/16 tcgen05.mma M128 x NCH x K16 (A = Z r-tile from TMEM, B = Y chunk from SMEM)
//     into the E / O accumulators of one of two TMEM buffers, the k-steps unrolled at compile time
//     (s3_mma_loop<KS>).  cp and mma execute in issue order, so the A slots need no barriers.
//   * warps 2-9: epilogue -- per chunk, tcgen05.ld of this warp's E and O columns into registers in two
//     phases (columns [0, 16) first, the rest loaded while those are reduced) and release of the TMEM
//     buffer; per thread the running max of E + |O| = max(E + O, E - O) and its 8-column group
//     (branch-free over all-fast half chunks); per pair the partial records go to the resolver through
//     shared memory (no CTA-wide barrier).  MODE 1 replaces the max by a log-sum-exp (marginalization).
//   * warp 10: resolver -- merges the 8 partial records, recomputes the 16 E / O sums of the pair's
//     winning group in fp32 from the same fp16 operands to recover the exact (shift, sign), one
//     packed-key atomicMax per pair.
// TMEM columns: D buffers [0, 4 NCH) (E, O of buffer 0 then 1), A slots [4 NCH, 4 NCH + 2 K3p).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "ftk_fft.cuh"
#include "ftk_sm100.cuh"
#include "ftk_tc.cuh"
#include "ftk_tc_dev.cuh"

namespace ftk {
using namespace sm100;

// Diagnostics (wait-cycle counters, FTK_S1_TRACE / FTK_S3_TRACE, FTK_S3_DBG) are compiled in only with
// -DFTK_DIAG=1 (build.py: FTK_DIAG=1 in the environment): clock reads and runtime checks inside the MMA
// and epilogue loops measurably slow them down.
#ifndef FTK_DIAG
#define FTK_DIAG 0
#endif
constexpr bool kDiag = FTK_DIAG != 0;
#ifndef FTK_S1_HINT
#define FTK_S1_HINT 2
#endif
// Step-1 L2 cache policies: bit 1 (default): image-operand stages evict_last (the 8 modes in flight stay
// L2-resident under the Zhat' write stream: c3 Step 1 -14 %, c3 x 2 defoci -5 %, c5 unchanged);
// bit 0: Zhat' stores evict_first (c3 +8-13 %, rejected); bit 2: template rows evict_last (experiment)
constexpr int kS1Hint = FTK_S1_HINT;
__device__ __forceinline__ long long diag_clock() {
  if constexpr (kDiag) return clock64();
  return 0;
}

constexpr int S3_WARPS = 11;
constexpr int S3_THREADS = S3_WARPS * 32;
constexpr int S3_MAXG = TcPlan::MAXG;
constexpr int S3_MAXNS = 4;

struct S3Params {
  const uint8_t* Zop;     // per pair: [r-tile][part][row/8][K3p/8][8 rows x 16 B] fp16x2 words (Step 2 output)
  const uint8_t* Ysm;     // per group: shared-memory image [part][rep/8][K3p/8][8 rows x 16 B]
  const int* colrep;      // [ncol_total] shift index of the representative (+delta); -1: padding column
  const int* colpart;     // [ncol_total] shift index of -delta; -1: none
  const uint8_t* colfast; // [ncol_total / 8] 1 if all 8 columns are paired, non-padding
  PairBlock pb;
  int n, K3p, Ke, N_t, NRT, NCH, G, NS;
  int g_col0[S3_MAXG], g_nch[S3_MAXG];
  long long g_yoff[S3_MAXG];
  int tm_off, n_tm_local;
  unsigned long long* img_keys;
  unsigned long long* pair_keys;
  float* land;
  float* marg;     // MODE 1: [N_im][n_tm_local] log sum_{t,r} exp(X / tau)
  float2* marg_part;  // MODE 1 with G > 1: [G][N_im][n_tm_local] base-2 (max, sum) partials
  long long marg_np;
  float msc;       // MODE 1: log2(e) / tau
  const float2* ast;  // fp16x3 scaling (see the file header): per image / local template maxima
  const float2* bst;
  float gmax;
  int eY;
  int dbg;         // FTK_S3_DBG (diagnostics): bit 0 skips the epilogue arithmetic, bit 1 the TMEM drain (timing only)
  unsigned long long* trace;  // nullable (FTK_S3_TRACE=1): wait / busy cycle counters of CTA 0
};

struct S3Smem {
  uint64_t y_bar;
  uint64_t st_full[S3_MAXNS], st_empty[S3_MAXNS];
  uint64_t d_full[2], d_empty[2];
  uint64_t red_full[2], red_empty[2];
  uint32_t tmem_base;
  float red_v[2][8], red_ve[2][8];
  uint32_t red_k[2][8], red_fe[2][8];
};
static_assert(sizeof(S3Smem) <= 512, "S3Smem must fit below the column metadata");

__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint4& v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
// SMEM -> TMEM: 128 rows x 32 bytes (two K-adjacent canonical core matrices per 8-row group)
__device__ __forceinline__ void tc_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

struct S3MmaArgs {
  uint32_t tmem, acol0, ybase, sbase, ypart, rt_part, SBO;
  int NCH, nch, NRT, NS, K3p, ke_steps, p_begin, p_end;
  S3Smem* S;
  unsigned long long* trace;  // CTA 0 only (FTK_S3_TRACE): per-chunk timestamps
};

// Step-3 MMA issue loop (one thread): per (pair, r-tile) the A slot copies (tcgen05.cp, in order with the
// MMAs), per chunk 3 x KS MMAs M128 x NCH x K16 into E (k-steps < ke) / O.  KS = K3p / 16 at compile time
// (KS = 0: runtime loop, for unusual widths).  tr: total, stage-wait and D-buffer-wait cycles.
template <int KS, bool TR>
__device__ __forceinline__ void s3_mma_loop(const S3MmaArgs& a, long long (&tr)[3]) {
  S3Smem& S = *a.S;
  const uint32_t idesc = idesc_f16_f32(128, a.NCH);
  const int ksteps = KS > 0 ? KS : a.K3p / 16, halfk = a.K3p / 2, ke = a.ke_steps;
  uint32_t g_a = 0, g_d = 0;
  const long long tr0 = diag_clock();
  for (int p = a.p_begin; p < a.p_end; ++p) {
    for (int T = 0; T < a.NRT; ++T, ++g_a) {
      const int ab = g_a & 1, s = g_a % a.NS;
      long long t1 = diag_clock();
      mbar_wait(&S.st_full[s], (g_a / a.NS) & 1);
      tr[1] += diag_clock() - t1;
      tc_fence_after();
      const uint32_t a_hi0 = a.tmem + a.acol0 + (uint32_t)(ab * a.K3p);
      // staging -> TMEM A slot (after the MMAs that last read this slot: in-order tensor pipe)
      const uint32_t src = a.sbase + (uint32_t)s * 2u * a.rt_part;
      for (int part = 0; part < 2; ++part)
        for (int j = 0; j < ksteps; ++j)
          tc_cp_128x256b(a_hi0 + (uint32_t)(part * halfk + 8 * j),
                         smem_desc_kmajor_noswz(src + part * a.rt_part + j * 256, 128, a.SBO));
      tc_commit(&S.st_empty[s]);
      for (int c = 0; c < a.nch; ++c, ++g_d) {
        const int db = g_d & 1;
        t1 = diag_clock();
        mbar_wait(&S.d_empty[db], ((g_d >> 1) & 1) ^ 1);
        tr[2] += diag_clock() - t1;
        tc_fence_after();
        if constexpr (TR) {  // (FTK_S3_TRACE) compile-time: a runtime branch here slows the MMA issue
          if (g_d < 64) a.trace[16 + 4 * g_d] = diag_clock();
        }
        const uint32_t dE = a.tmem + (uint32_t)(db * 2 * a.NCH), dO = dE + (uint32_t)a.NCH;
        const uint32_t bch = a.ybase + (uint32_t)(c * (a.NCH / 8)) * a.SBO;
        const uint64_t bh0 = smem_desc_kmajor_noswz(bch, 128, a.SBO);
        const uint64_t bl0 = smem_desc_kmajor_noswz(bch + a.ypart, 128, a.SBO);
        if constexpr (KS > 0) {
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const uint32_t d = ks >= ke ? dO : dE;
            const uint32_t acc0 = (ks == 0 || ks == ke) ? 0u : 1u;
            const uint32_t a_hi = a_hi0 + (uint32_t)(ks * 8), a_lo = a_hi + (uint32_t)halfk;
            mma_f16_ts(d, a_hi, bh0 + (uint64_t)(ks * 16), idesc, acc0);  // +256 B per k-step
            mma_f16_ts(d, a_hi, bl0 + (uint64_t)(ks * 16), idesc, 1u);
            mma_f16_ts(d, a_lo, bh0 + (uint64_t)(ks * 16), idesc, 1u);
          }
        } else {
          for (int ks = 0; ks < ksteps; ++ks) {
            const uint32_t d = ks >= ke ? dO : dE;
            const uint32_t acc0 = (ks == 0 || ks == ke) ? 0u : 1u;
            const uint32_t a_hi = a_hi0 + (uint32_t)(ks * 8), a_lo = a_hi + (uint32_t)halfk;
            mma_f16_ts(d, a_hi, bh0 + (uint64_t)(ks * 16), idesc, acc0);
            mma_f16_ts(d, a_hi, bl0 + (uint64_t)(ks * 16), idesc, 1u);
            mma_f16_ts(d, a_lo, bh0 + (uint64_t)(ks * 16), idesc, 1u);
          }
        }
        tc_commit(&S.d_full[db]);
        if constexpr (TR) {
          if (g_d < 64) a.trace[16 + 4 * g_d + 1] = diag_clock();
        }
      }
    }
  }
  tr[0] = diag_clock() - tr0;
}

// MODE 0: fused max / argmax (the north-star epilogue).  MODE 1: marginalization epilogue (SURVEY 8(f)
// NEXT-3; the Bayesian use of the full landscape): per pair
//   L = log sum_{t, r} exp(X(delta_t, gamma_r) / tau),
// accumulated per thread as a base-2 running (max, scaled sum) and merged per warp and per pair.
template <int MODE>
__global__ void __launch_bounds__(S3_THREADS, 1) k_step3_tc(S3Params P) {
  extern __shared__ __align__(1024) uint8_t s3_raw[];
  S3Smem& S = *reinterpret_cast<S3Smem*>(s3_raw);
  int* s_rep = reinterpret_cast<int*>(s3_raw + 512);  // [ncol_g] then s_part, s_fast, s_fastc
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = P.n, K3p = P.K3p, NCH = P.NCH, NRT = P.NRT, NS = P.NS;
  const int G = P.G, grp = blockIdx.x % G;
  const int nch = P.g_nch[grp], ncol = nch * NCH, col0 = P.g_col0[grp];
  int* s_part = s_rep + ncol;
  uint8_t* s_fast = reinterpret_cast<uint8_t*>(s_part + ncol);
  uint8_t* s_fastc = s_fast + ncol / 8;  // [nch * 2]: leading columns of a half chunk in fast groups
  const uint32_t meta_bytes = ((uint32_t)ncol * 8u + (uint32_t)ncol / 8u + 2u * (uint32_t)nch + 512u + 1023u) & ~1023u;
  uint8_t* ys = s3_raw + 1024 + meta_bytes;                        // Y image of this group
  const uint32_t ypart = (uint32_t)ncol * (uint32_t)K3p * 2u;       // bytes of one fp16 part
  const uint32_t rt_part = 128u * (uint32_t)K3p * 2u;              // one part of an r-tile image
  uint8_t* stg = ys + ((2u * ypart + 1023u) & ~1023u);              // staging ring: NS r-tile images
  const uint32_t SBO = (uint32_t)K3p * 16u;                         // bytes between 8-row groups
  const size_t pair_bytes = (size_t)NRT * 2 * rt_part;
  if (threadIdx.x == 0) {
    mbar_init(&S.y_bar, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&S.st_full[i], 1);
      mbar_init(&S.st_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.d_full[i], 1);
      mbar_init(&S.d_empty[i], 8);
      mbar_init(&S.red_full[i], 8);
      mbar_init(&S.red_empty[i], 1);
    }
    fence_barrier_init();
  }
  for (int c = threadIdx.x; c < ncol; c += blockDim.x) {
    s_rep[c] = __ldg(P.colrep + col0 + c);
    s_part[c] = __ldg(P.colpart + col0 + c);
  }
  for (int c = threadIdx.x; c < ncol / 8; c += blockDim.x) s_fast[c] = __ldg(P.colfast + col0 / 8 + c);
  for (int hc = threadIdx.x; hc < 2 * nch; hc += blockDim.x) {  // leading fast columns of each half chunk
    int nf = 0;
    if (P.Ke < K3p)
      for (int c8 = hc * (NCH / 2); c8 < (hc + 1) * (NCH / 2) && __ldg(P.colfast + (col0 + c8) / 8) != 0; c8 += 8) nf += 8;
    s_fastc[hc] = (uint8_t)nf;
  }
  if (warp == 0) tmem_alloc<512>(&S.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  const uint32_t acol0 = 4u * (uint32_t)NCH;
  // pair range of this CTA (CTAs of one group split the pairs)
  const int cpg = gridDim.x / G;  // CTAs per group (grid is a multiple of G)
  const int cig = blockIdx.x / G;
  const int count = P.pb.count;
  const int per = (count + cpg - 1) / cpg;
  const int p_begin = min(count, cig * per);
  const int p_end = min(count, p_begin + per);

  if (warp == 0) {
    // ---------------- Y image of the group -> SMEM (once); then A copies + MMAs, all from one elected
    // lane.  The k-step loop is unrolled at compile time (s3_mma_loop<KS>): a runtime-trip-count loop
    // around tcgen05.mma measured ~500 extra cycles per chunk (scripts/micro_s3.cu).
    if (elect_one()) {
      const uint32_t ybytes = 2u * ypart;
      mbar_arrive_expect_tx(&S.y_bar, ybytes);
      const uint8_t* ysrc = P.Ysm + P.g_yoff[grp];
      for (uint32_t o = 0; o < ybytes; o += 32768u) {
        const uint32_t b = min(32768u, ybytes - o);
        bulk_g2s(ys + o, ysrc + o, b, &S.y_bar);
      }
      mbar_wait(&S.y_bar, 0);
      S3MmaArgs a{tmem, acol0, smem_u32(ys), smem_u32(stg), ypart, rt_part, SBO, NCH, nch, NRT, NS, K3p, P.Ke / 16,
                  p_begin, p_end, &S, (P.trace && blockIdx.x == 0) ? P.trace : nullptr};
      long long tr[3] = {0, 0, 0};
      if (a.trace) {
        s3_mma_loop<0, true>(a, tr);
      } else {
        switch (K3p / 16) {
          case 2: s3_mma_loop<2, false>(a, tr); break;
          case 3: s3_mma_loop<3, false>(a, tr); break;
          case 4: s3_mma_loop<4, false>(a, tr); break;
          case 5: s3_mma_loop<5, false>(a, tr); break;
          case 6: s3_mma_loop<6, false>(a, tr); break;
          case 7: s3_mma_loop<7, false>(a, tr); break;
          case 8: s3_mma_loop<8, false>(a, tr); break;
          case 9: s3_mma_loop<9, false>(a, tr); break;    // K3p > 128: CTF plans
          case 10: s3_mma_loop<10, false>(a, tr); break;
          case 11: s3_mma_loop<11, false>(a, tr); break;
          case 12: s3_mma_loop<12, false>(a, tr); break;
          case 13: s3_mma_loop<13, false>(a, tr); break;
          case 14: s3_mma_loop<14, false>(a, tr); break;
          default: s3_mma_loop<0, false>(a, tr); break;
        }
      }
      if (P.trace && blockIdx.x == 0) {
        P.trace[0] = tr[0];
        P.trace[1] = tr[1];
        P.trace[2] = tr[2];
        P.trace[3] = p_end - p_begin;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- producer: one bulk copy per (pair, r-tile) into the staging ring
    if (lane == 0) {
      uint32_t g_a = 0;
      for (int p = p_begin; p < p_end; ++p) {
        const uint8_t* zp = P.Zop + (size_t)p * pair_bytes;
        for (int T = 0; T < NRT; ++T, ++g_a) {
          const int s = g_a % NS;
          mbar_wait(&S.st_empty[s], ((g_a / NS) & 1) ^ 1);
          mbar_arrive_expect_tx(&S.st_full[s], 2u * rt_part);
          const uint8_t* src = zp + (size_t)T * 2 * rt_part;
          uint8_t* dst = stg + (size_t)s * 2 * rt_part;
          for (uint32_t o = 0; o < 2u * rt_part; o += 32768u) bulk_g2s(dst + o, src + o, min(32768u, 2u * rt_part - o), &S.st_full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp <= 9) {
    // ---------------- epilogue: 8 warps, two per TMEM lane quarter, each half of the chunk's columns.
    // Per chunk the warp's E / O columns (hw <= 40 each) are drained to registers and the TMEM buffer is
    // released at once.  Paired columns: X = max(E + O, E - O) = E + |O| per 8-column group, and per
    // thread only the best value and its group are tracked (branch-free); the resolver recovers the
    // exact (shift, sign).  Groups with padding / unpaired shifts, and landscape output, take the exact
    // path.
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int ew = warp - 2;        // 0..7
    const int h = ew >> 2;          // 0 or 1
    const int hw = NCH / 2;         // columns per epilogue warp (multiple of 8, <= 40)
    const bool has_odd = P.Ke < K3p;
    uint32_t g_d = 0, it = 0;
    long long tr_e = 0, tr_x = 0;
    for (int p = p_begin; p < p_end; ++p, ++it) {
      float bvf = -INFINITY;        // fast record: best E + |O| ...
      uint32_t bkf = 0xffffffffu;   // ... and its key (T << 24 | column << 7 | row)
      float bve = -INFINITY;        // exact record (slow groups)
      uint32_t bfe = 0xffffffffu;
      float mrun = -INFINITY, srun = 0.f;  // MODE 1: running base-2 log-sum-exp of X log2(e) / tau
      float* land_p = P.land ? P.land + (size_t)p * P.N_t * n : nullptr;
      float unsc = 1.f;  // this pair's fp16x3 unscale factor (values are X 2^pe, unsc = 2^-pe); MODE 0 needs it
      if (MODE == 1 || land_p) {  // only for landscapes (the resolver unscales the keys)
        int pi_, pj_;
        pair_of(P.pb, p, pi_, pj_);
        unsc = pow2f_wide(-(z_exp(__ldg(P.ast + pi_), __ldg(P.bst + pj_), P.gmax) + P.eY));
      }
      const float msc_p = P.msc * unsc;  // MODE 1: log2(e) / tau in scaled units
      for (int T = 0; T < NRT; ++T) {
        const int r = T * 128 + row;
        const bool active = T * 128 + q * 32 < n;  // warp-uniform: lane quarters beyond n_psi idle
        for (int c = 0; c < nch; ++c, ++g_d) {
          const int db = g_d & 1;
          long long te = diag_clock();
          if (kDiag && (P.dbg & 4)) {  // (diagnostics) one poller + named barrier
            if (warp == 2) mbar_wait(&S.d_full[db], (g_d >> 1) & 1);
            named_bar(3, 256);
          } else {
            mbar_wait(&S.d_full[db], (g_d >> 1) & 1);  // every epilogue warp (suspending try_wait)
          }
          tr_e += diag_clock() - te;
          te = diag_clock();
          tc_fence_after();
          const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(db * 2 * NCH + h * hw);
          const int clb = c * NCH + h * hw;  // first column of this warp's half chunk
          const int nfast = land_p ? 0 : (int)s_fastc[c * 2 + h];
          uint32_t e01[32], e2[8], o01[32], o2[8];
          uint32_t* e0 = e01;
          uint32_t* e1 = e01 + 16;
          uint32_t* o0 = o01;
          uint32_t* o1 = o01 + 16;
          if (!has_odd) {
#pragma unroll
            for (int k = 0; k < 16; ++k) o0[k] = o1[k] = 0u;
#pragma unroll
            for (int k = 0; k < 8; ++k) o2[k] = 0u;
          }
          // MODE 0 (fast groups): per 8-column group, the best E + |O| = max(X(+delta), X(-delta)) and its
          // group key; slow groups (padding / unpaired shifts / landscape output) take the exact path
          const uint32_t kb = ((uint32_t)T << 24) | ((uint32_t)clb << 7) | (uint32_t)row;
          auto grp0 = [&](auto G) {
            constexpr int g8 = decltype(G)::value;
            if (MODE != 0 || !active || (kDiag && (P.dbg & 1)) || 8 * g8 >= hw) return;
            uint32_t e[8], o[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              e[k] = g8 < 2 ? e0[8 * g8 + k] : (g8 < 4 ? e1[8 * (g8 - 2) + k] : e2[k]);
              o[k] = g8 < 2 ? o0[8 * g8 + k] : (g8 < 4 ? o1[8 * (g8 - 2) + k] : o2[k]);
            }
            if (8 * g8 < nfast) {
              float v[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(e[k]) + fabsf(__uint_as_float(o[k]));
              const float m = fmaxf(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])), fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7])));
              const bool upd = m > bvf;
              bvf = upd ? m : bvf;
              bkf = upd ? kb + ((uint32_t)(8 * g8) << 7) : bkf;
            } else if (r < n) {
              const int cl = clb + 8 * g8;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const int tp = s_rep[cl + k], tm = s_part[cl + k];
                if (tp < 0) continue;
                const float ev = __uint_as_float(e[k]), ov = __uint_as_float(o[k]);
                const float xp = ev + ov;
                const uint32_t fp = (uint32_t)tp * (uint32_t)n + (uint32_t)r;
                if (better(xp, fp, bve, bfe)) {
                  bve = xp;
                  bfe = fp;
                }
                if (land_p) land_p[(size_t)tp * n + r] = xp * unsc;
                if (tm >= 0) {
                  const float xm = ev - ov;
                  const uint32_t fm = (uint32_t)tm * (uint32_t)n + (uint32_t)r;
                  if (better(xm, fm, bve, bfe)) {
                    bve = xm;
                    bfe = fm;
                  }
                  if (land_p) land_p[(size_t)tm * n + r] = xm * unsc;
                }
              }
            }
          };
          // all-fast half chunks (the common case): branch-free over the groups [G0, G1) so the FADD / max
          // chains of different groups interleave; the serial compare-select only per group maximum
          const bool allfast = MODE == 0 && active && !(kDiag && (P.dbg & 1)) && nfast >= hw;
          auto fast_range = [&](auto G0, auto G1) {
            constexpr int g0 = decltype(G0)::value, g1 = decltype(G1)::value;
            float m[5];
#pragma unroll
            for (int g8 = g0; g8 < g1; ++g8) {
              float v[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const uint32_t ek = g8 < 2 ? e0[8 * g8 + k] : (g8 < 4 ? e1[8 * (g8 - 2) + k] : e2[k]);
                const uint32_t ok = g8 < 2 ? o0[8 * g8 + k] : (g8 < 4 ? o1[8 * (g8 - 2) + k] : o2[k]);
                v[k] = __uint_as_float(ek) + fabsf(__uint_as_float(ok));
              }
              m[g8] = fmaxf(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])), fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7])));
            }
#pragma unroll
            for (int g8 = g0; g8 < g1; ++g8) {
              const bool upd = m[g8] > bvf;
              bvf = upd ? m[g8] : bvf;
              bkf = upd ? kb + ((uint32_t)(8 * g8) << 7) : bkf;
            }
          };
          auto phase1 = [&]() {
            if (allfast && hw >= 16) {
              fast_range(std::integral_constant<int, 0>{}, std::integral_constant<int, 2>{});
            } else if (allfast) {
              fast_range(std::integral_constant<int, 0>{}, std::integral_constant<int, 1>{});
            } else {
              grp0(std::integral_constant<int, 0>{});
              grp0(std::integral_constant<int, 1>{});
            }
          };
          auto phase2 = [&]() {
            if (allfast && hw == 40) {
              fast_range(std::integral_constant<int, 2>{}, std::integral_constant<int, 5>{});
            } else if (allfast && hw == 32) {
              fast_range(std::integral_constant<int, 2>{}, std::integral_constant<int, 4>{});
            } else if (allfast && hw == 24) {
              fast_range(std::integral_constant<int, 2>{}, std::integral_constant<int, 3>{});
            } else if (!(allfast && hw <= 16)) {
              grp0(std::integral_constant<int, 2>{});
              grp0(std::integral_constant<int, 3>{});
              grp0(std::integral_constant<int, 4>{});
            }
          };
          // two-phase drain: columns [0, 16) first; the rest is loaded while MODE 0 processes them
          // (tcgen05.wait::ld waits for all of a thread's loads; the empty asm "+r" ties each register to
          // the wait so no use is scheduled before it)
          const bool ld = active && !(kDiag && (P.dbg & 2));
          if (ld) {
            tmem_ld16(base, *reinterpret_cast<uint32_t(*)[16]>(e0));
            if (has_odd) tmem_ld16(base + NCH, *reinterpret_cast<uint32_t(*)[16]>(o0));
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 16; ++k) asm volatile("" : "+r"(e0[k]), "+r"(o0[k]));
            if (hw > 16) {
              tmem_ld16(base + 16, *reinterpret_cast<uint32_t(*)[16]>(e1));
              if (has_odd) tmem_ld16(base + NCH + 16, *reinterpret_cast<uint32_t(*)[16]>(o1));
            }
            if (hw > 32) {
              tmem_ld8(base + 32, e2);
              if (has_odd) tmem_ld8(base + NCH + 32, o2);
            }
          }
          phase1();
          if (ld) {
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 16; ++k) asm volatile("" : "+r"(e1[k]), "+r"(o1[k]));
#pragma unroll
            for (int k = 0; k < 8; ++k) asm volatile("" : "+r"(e2[k]), "+r"(o2[k]));
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.d_empty[db]);
          tr_x += diag_clock() - te;
          phase2();
          // MODE 1, all-fast half chunks: branch-free over NG compile-time groups
          auto marg_fast = [&](auto NGc) {
            constexpr int NG = decltype(NGc)::value;
            float cmk[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) cmk[k] = -INFINITY;
#pragma unroll
            for (int g8 = 0; g8 < NG; ++g8)
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float ev = __uint_as_float(g8 < 2 ? e0[8 * g8 + k] : (g8 < 4 ? e1[8 * (g8 - 2) + k] : e2[k]));
                const float ov = __uint_as_float(g8 < 2 ? o0[8 * g8 + k] : (g8 < 4 ? o1[8 * (g8 - 2) + k] : o2[k]));
                cmk[k] = fmaxf(cmk[k], ev + fabsf(ov));
              }
            float cm = fmaxf(fmaxf(fmaxf(cmk[0], cmk[1]), fmaxf(cmk[2], cmk[3])),
                             fmaxf(fmaxf(cmk[4], cmk[5]), fmaxf(cmk[6], cmk[7])));
            cm *= msc_p;
            if (cm > mrun) {
              srun *= ex2_approx(mrun - cm);
              mrun = cm;
            }
            const float nm = -mrun, sc = msc_p;
            float sk[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) sk[k] = 0.f;
#pragma unroll
            for (int g8 = 0; g8 < NG; ++g8)
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float ev = __uint_as_float(g8 < 2 ? e0[8 * g8 + k] : (g8 < 4 ? e1[8 * (g8 - 2) + k] : e2[k]));
                const float ov = __uint_as_float(g8 < 2 ? o0[8 * g8 + k] : (g8 < 4 ? o1[8 * (g8 - 2) + k] : o2[k]));
                sk[k] += ex2_approx(fmaf(ev + ov, sc, nm)) + ex2_approx(fmaf(ev - ov, sc, nm));
              }
            srun += ((sk[0] + sk[1]) + (sk[2] + sk[3])) + ((sk[4] + sk[5]) + (sk[6] + sk[7]));
          };
          bool marg_done = false;
          if (MODE == 1 && active && nfast >= hw) {
            marg_done = true;
            switch (hw >> 3) {
              case 5: marg_fast(std::integral_constant<int, 5>{}); break;
              case 4: marg_fast(std::integral_constant<int, 4>{}); break;
              case 3: marg_fast(std::integral_constant<int, 3>{}); break;
              case 2: marg_fast(std::integral_constant<int, 2>{}); break;
              case 1: marg_fast(std::integral_constant<int, 1>{}); break;
              default: marg_done = false; break;
            }
          }
          if (MODE == 1 && active && !marg_done) {
            // pass 1: the chunk's maximum of X = max(E + O, E - O) = E + |O| over valid columns (the
            // group test is warp-uniform: fast groups have 8 paired, non-padding columns)
            float cmk[8];  // per-k partial maxima (short dependency chains)
#pragma unroll
            for (int k = 0; k < 8; ++k) cmk[k] = -INFINITY;
#pragma unroll
            for (int g8 = 0; g8 < 5; ++g8) {
              if (8 * g8 >= hw) break;
              const int cl = clb + 8 * g8;
              float ev[8], ov[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                ev[k] = __uint_as_float(g8 < 2 ? e0[8 * g8 + k] : (g8 < 4 ? e1[8 * (g8 - 2) + k] : e2[k]));
                ov[k] = __uint_as_float(g8 < 2 ? o0[8 * g8 + k] : (g8 < 4 ? o1[8 * (g8 - 2) + k] : o2[k]));
              }
              if (s_fast[cl >> 3]) {
#pragma unroll
                for (int k = 0; k < 8; ++k) cmk[k] = fmaxf(cmk[k], ev[k] + fabsf(ov[k]));
              } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  if (s_rep[cl + k] >= 0) cmk[k] = fmaxf(cmk[k], ev[k] + ov[k]);
                  if (s_part[cl + k] >= 0) cmk[k] = fmaxf(cmk[k], ev[k] - ov[k]);
                }
              }
            }
            float cm = fmaxf(fmaxf(fmaxf(cmk[0], cmk[1]), fmaxf(cmk[2], cmk[3])),
                             fmaxf(fmaxf(cmk[4], cmk[5]), fmaxf(cmk[6], cmk[7])));
            if (cm != -INFINITY) {
              cm *= msc_p;
              if (cm > mrun) {
                srun *= ex2_approx(mrun - cm);
                mrun = cm;
              }
              // pass 2: sum of 2^(X log2(e) / tau - m) over both signs of delta (per-k partial sums)
              float sk[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) sk[k] = 0.f;
              const float nm = -mrun, sc = msc_p;
#pragma unroll
              for (int g8 = 0; g8 < 5; ++g8) {
                if (8 * g8 >= hw) break;
                const int cl = clb + 8 * g8;
                float ev[8], ov[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  ev[k] = __uint_as_float(g8 < 2 ? e0[8 * g8 + k] : (g8 < 4 ? e1[8 * (g8 - 2) + k] : e2[k]));
                  ov[k] = __uint_as_float(g8 < 2 ? o0[8 * g8 + k] : (g8 < 4 ? o1[8 * (g8 - 2) + k] : o2[k]));
                }
                if (s_fast[cl >> 3]) {
#pragma unroll
                  for (int k = 0; k < 8; ++k) {
                    // X(+delta) log2(e) / tau - m and X(-delta) log2(e) / tau - m
                    sk[k] += ex2_approx(fmaf(ev[k] + ov[k], sc, nm)) + ex2_approx(fmaf(ev[k] - ov[k], sc, nm));
                  }
                } else {
#pragma unroll
                  for (int k = 0; k < 8; ++k) {
                    if (s_rep[cl + k] >= 0) sk[k] += ex2_approx(fmaf(ev[k] + ov[k], sc, nm));   // else padding
                    if (s_part[cl + k] >= 0) sk[k] += ex2_approx(fmaf(ev[k] - ov[k], sc, nm));  // else no -delta
                  }
                }
              }
              srun += ((sk[0] + sk[1]) + (sk[2] + sk[3])) + ((sk[4] + sk[5]) + (sk[6] + sk[7]));
            }
          }
        }
      }
      // per-pair reduction over the warp; the resolver merges the 8 warps' records
      if (MODE == 1) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float m2 = __shfl_xor_sync(0xffffffffu, mrun, o);
          const float s2 = __shfl_xor_sync(0xffffffffu, srun, o);
          lse2_merge(mrun, srun, m2, s2);
        }
        bvf = mrun;
        bve = srun;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        if (MODE == 1) break;
        const float v2 = __shfl_xor_sync(0xffffffffu, bvf, o);
        const uint32_t k2 = __shfl_xor_sync(0xffffffffu, bkf, o);
        if (better(v2, k2, bvf, bkf)) {
          bvf = v2;
          bkf = k2;
        }
        const float v3 = __shfl_xor_sync(0xffffffffu, bve, o);
        const uint32_t f3 = __shfl_xor_sync(0xffffffffu, bfe, o);
        if (better(v3, f3, bve, bfe)) {
          bve = v3;
          bfe = f3;
        }
      }
      const int rb = it & 1;
      if (lane == 0) {
        mbar_wait(&S.red_empty[rb], ((it >> 1) & 1) ^ 1);  // slot consumed by the resolver (pair it - 2)
        S.red_v[rb][ew] = bvf;
        S.red_k[rb][ew] = bkf;
        S.red_ve[rb][ew] = bve;
        S.red_fe[rb][ew] = bfe;
        mbar_arrive(&S.red_full[rb]);
      }
      __syncwarp();
    }
    if (P.trace && blockIdx.x == 0 && lane == 0 && warp == 2) {
      P.trace[4] = tr_e;
      P.trace[5] = tr_x;
    }
  } else {
    // ---------------- resolver (warp 10): merge the 8 partial records; exact (shift, sign) of the pair's
    // winning group by recomputing its 16 E / O sums from the same fp16 hi/lo operands (fp32 on CUDA
    // cores); merge with the exact record; one packed-key atomicMax per pair.
    uint32_t it = 0;
    for (int p = p_begin; p < p_end; ++p, ++it) {
      const int rb = it & 1;
      int pi_r, pj_r;
      pair_of(P.pb, p, pi_r, pj_r);
      const float2 st_a = __ldg(P.ast + pi_r), st_b = __ldg(P.bst + pj_r);  // fp16x3 stats, loaded early
      mbar_wait_lazy(&S.red_full[rb], (it >> 1) & 1, 200);
      if (MODE == 1) {
        float m = S.red_v[rb][0], sm = S.red_ve[rb][0];
        for (int w = 1; w < 8; ++w) lse2_merge(m, sm, S.red_v[rb][w], S.red_ve[rb][w]);
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&S.red_empty[rb]);
          int i, j;
          pair_of(P.pb, p, i, j);
          const size_t ij = (size_t)i * P.n_tm_local + j;
          if (P.marg_part)
            P.marg_part[(size_t)grp * (size_t)P.marg_np + ij] = make_float2(m, sm);
          else
            P.marg[ij] = (m + log2f(sm)) * 0.6931471805599453f;
        }
        __syncwarp();
        continue;
      }
      float v = S.red_v[rb][0], ve = S.red_ve[rb][0];
      uint32_t key = S.red_k[rb][0], fe = S.red_fe[rb][0];
      for (int w = 1; w < 8; ++w) {
        if (better(S.red_v[rb][w], S.red_k[rb][w], v, key)) {
          v = S.red_v[rb][w];
          key = S.red_k[rb][w];
        }
        if (better(S.red_ve[rb][w], S.red_fe[rb][w], ve, fe)) {
          ve = S.red_ve[rb][w];
          fe = S.red_fe[rb][w];
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.red_empty[rb]);
      float bv = ve;
      uint32_t bf = fe;
      if (key != 0xffffffffu) {
        const int T = (int)(key >> 24), cl = (int)((key >> 7) & 0x1ffffu), rrow = (int)(key & 127u);
        const int r = T * 128 + rrow;
        // row rrow of the pair's r-tile image: word w at (rrow / 8) SBO + (w / 4) 128 + (rrow % 8) 16 + (w % 4) 4
        const uint8_t* zrow = P.Zop + (size_t)p * pair_bytes + (size_t)T * 2 * rt_part + (size_t)(rrow >> 3) * SBO +
                              (rrow & 7) * 16;
        float es[8], os[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) es[k] = os[k] = 0.f;
        const __half* yh = reinterpret_cast<const __half*>(ys);
        const __half* yl = yh + (size_t)ncol * K3p;
        for (int kk = lane; kk < K3p; kk += 32) {
          const size_t zo = (size_t)(kk >> 3) * 128 + (kk & 7) * 2;
          const float zh = __half2float(*reinterpret_cast<const __half*>(zrow + zo));
          const float zl = __half2float(*reinterpret_cast<const __half*>(zrow + rt_part + zo));
          const bool even = kk < P.Ke;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int cc = cl + k;
            const size_t yo = (size_t)(cc >> 3) * (K3p / 8) * 64 + (size_t)(kk >> 3) * 64 + (cc & 7) * 8 + (kk & 7);
            const float a = __half2float(yh[yo]), b = __half2float(yl[yo]);
            const float pr = fmaf(zh, a, fmaf(zh, b, zl * a));
            if (even)
              es[k] += pr;
            else
              os[k] += pr;
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            es[k] += __shfl_xor_sync(0xffffffffu, es[k], o);
            os[k] += __shfl_xor_sync(0xffffffffu, os[k], o);
          }
        // the winning column (ties -> smaller flat index); the value reported is the tensor-core one
        float bx = -INFINITY;
        uint32_t bfl = 0xffffffffu;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float x = es[k] + fabsf(os[k]);
          const int t = os[k] >= 0.f ? s_rep[cl + k] : s_part[cl + k];
          const uint32_t f = (uint32_t)t * (uint32_t)n + (uint32_t)r;
          if (better(x, f, bx, bfl)) {
            bx = x;
            bfl = f;
          }
        }
        if (better(v, bfl, bv, bf)) {
          bv = v;
          bf = bfl;
        }
      }
      if (lane == 0 && bf != 0xffffffffu) {
        int i, j;
        pair_of(P.pb, p, i, j);
        const uint32_t tt2 = bf / (uint32_t)n, rr = bf - tt2 * (uint32_t)n;
        const uint32_t gflat = ((uint32_t)(P.tm_off + j) * (uint32_t)P.N_t + tt2) * (uint32_t)n + rr;
        const int pe = z_exp(st_a, st_b, P.gmax) + P.eY;
        const unsigned long long kk = pack_key(bv * pow2f_wide(-pe), gflat);  // fp16x3 scale removed (exact)
        if (P.img_keys) atomicMax(&P.img_keys[i], kk);
        if (P.pair_keys) atomicMax(&P.pair_keys[(size_t)i * P.n_tm_local + j], kk);
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

static size_t s3_smem_bytes(int ncol, int K3p, int NS) {
  const size_t meta = (((size_t)ncol * 8 + ncol / 8) + 2 * (size_t)(ncol / 16) + 512 + 1023) & ~(size_t)1023;
  const size_t y = ((size_t)ncol * K3p * 4 + 1023) & ~(size_t)1023;
  return 1024 + meta + y + (size_t)NS * 128 * K3p * 4;
}


// ---------------------------------------------------------------- Step 1 (tensor cores)
// Form B of Eq. (fbk3) Step 1 (P:836 with p = q - ell): for each image mode p
//   Zhat'_{ij,zeta}(p) = sum_m a_i(m, p) c_{j zeta}(m),  c = g_zeta(m) conj b_j(m, p + ell_zeta),  g = 2 pi w G,
// so that Zhat_zeta(q) = Zhat'_zeta(q - ell) and Step 2 applies e^{-i ell gamma_r} after the FFT.
// Real GEMM per p with K' = 2 n_k:  rows (j, zeta, part) of the GENERATED operand c (A, in TMEM):
//   Re-row = [c_r | -c_i],  Im-row = [c_i | c_r];  columns = images, B = [a_r | a_i] (pre-split, SMEM).
// Output Zhat' [pair][p][Hs] complex (pair = il * nj + jl within the block; Hs = H_plus rounded up to even, the
// pad slot written as zero so that every 32-byte sector of a row is written in full).
constexpr int S1_THREADS = 18 * 32;  // 0 producer, 1 MMA, 2-9 generators, 10-17 epilogue
constexpr int S1_STAGES = 4;

struct S1Params {
  const uint8_t* Aop;   // image operand: [p][image tile][kchunk][part][16][KCH/8][128 B]
  const float2* B;      // template FB coefficients [j][q][m] (local templates)
  const float* g;       // [H_plus][n_k]
  const int* ell;       // [H_plus]
  float2* Zhat;         // [pair][p][Hs]
  int i0, ni, j0, nj;   // block (i0 multiple of 128)
  int n, n_k, Hp, Hs, KCH, NKCH, NIT;  // NIT = image tiles per mode in Aop
  int F, NCT;           // F = nj * Hs flattened (j, zeta slot) columns (pad slots written as zeros), NCT = ceil(F / 64)
  const float2* ast;    // fp16x3 scaling (file header): image maxima [N_im], local template maxima [n_tm_local]
  const float2* bst;
  float gmax;           // max |g_zeta(k_m)|
  unsigned long long* trace;  // nullable (FTK_S1_TRACE=1): wait cycle counters of CTA 0
};

// Unit order: u -> (mode p, column tile ct) with p = 8 p_hi + p_lo, p_lo fastest, then ct, then p_hi.
// The ~148 units in flight then share 8 image-operand modes (L2-resident) and write 8 consecutive
// p-rows of each of their pairs' Zhat' rows together (contiguous runs merged in L2).
#ifndef FTK_S1_PLO
#define FTK_S1_PLO 8
#endif
__device__ __forceinline__ void s1_unit(int u, int NCT, int& p, int& ct) {
  constexpr int PLO = FTK_S1_PLO;
  const int p_lo = u % PLO, rest = u / PLO;
  ct = rest % NCT;
  p = (rest / NCT) * PLO + p_lo;
}
// Processing order of the K' chunks of one image tile: with two generation rounds (NKCH % 4 == 0) all chunks
// of round 0 first, then round 1, so that round 0 of the next unit can be generated during the last tile's
// round-1 MMAs (and round 1 during the first tile's round-0 MMAs)
__host__ __device__ __forceinline__ int s1_chunk_of(int i, int nkch) {
  if (nkch % 4 != 0) return i;
  const int hq = nkch / 2, qq = nkch / 4;
  const int j = i < hq ? i : i - hq;
  return (j / qq) * hq + (i < hq ? 0 : qq) + (j % qq);
}


constexpr int S1_MAXST = 8;  // stage barriers (CTA pair: 8 half-size stages)
struct S1Smem {
  uint64_t st_full[S1_MAXST], st_empty[S1_MAXST];
  uint64_t a_full[2], a_empty[2];  // per generation round (see s1_rounds)
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};

struct S1MmaArgs {
  uint32_t tmem, sbase, stage_bytes, part_bytes, SBO;
  int KCH, NKCH, nk, units, nit, ubeg, ustep;
  S1Smem* S;
};

// Step-1 MMA issue loop (one thread): per unit the generated A operand (TMEM) against every image tile,
// per stage KS = KCH / 16 k-steps x 3 fp16 products (compile-time unrolled: a runtime loop around
// tcgen05.mma costs ~500 cycles per stage, scripts/micro_s3.cu).  tr: total, A-wait, acc-wait, stage-wait.
// NK = NKCH at compile time (1, 2, 4; 0 = runtime): the k-chunk loop is then unrolled, which avoids the
// per-iteration cost of a runtime loop around tcgen05.mma (see the Step-3 note in DESIGN.md).
// CG2: the CTA pair's MMAs (M = 256: this CTA's 128 generated rows and the peer's; each CTA holds half of the
// 128-image stage), issued by the even CTA, committed to both CTAs' barriers.
template <int KS, int NK, bool CG2>
__device__ __forceinline__ uint32_t s1_mma_loop(const S1MmaArgs& a, long long (&tr)[4]) {
  constexpr int NST = CG2 ? 8 : S1_STAGES;
  S1Smem& S = *a.S;
  const uint32_t idesc = idesc_f16_f32(CG2 ? 256 : 128, 128);
  auto mma = [&](uint32_t d, uint32_t at, uint64_t bd, uint32_t acc) {
    if constexpr (CG2)
      mma_f16_ts_cg2(d, at, bd, idesc, acc);
    else
      mma_f16_ts(d, at, bd, idesc, acc);
  };
  auto commit = [&](uint64_t* bar) {
    if constexpr (CG2)
      tc_commit_cg2(bar);
    else
      tc_commit(bar);
  };
  uint32_t g_st = 0, g_acc = 0, g_u = 0;
  const long long tr0 = diag_clock();
  // generation rounds: R = 2 when the K' chunks split by radial halves (NKCH % 4 == 0): round r fills the
  // chunks kc with (kc mod NKCH/2) in [r NKCH/4, (r+1) NKCH/4), i.e. m in [r n_k/2, (r+1) n_k/2)
  const int nkch = NK > 0 ? NK : a.NKCH;
  const int R = (nkch % 4 == 0) ? 2 : 1;
  const int hq = nkch / 2, qq = nkch / 4;
  auto round_of = [&](int kc) { return R == 2 ? ((kc % hq) >= qq ? 1 : 0) : 0; };
  for (int u = a.ubeg; u < a.units; u += a.ustep, ++g_u) {
    bool got0 = false, got1 = false;
    for (int t = 0; t < a.nit; ++t, ++g_acc) {
      const int ab = g_acc & 1;
      long long t1 = diag_clock();
      mbar_wait(&S.acc_empty[ab], ((g_acc >> 1) & 1) ^ 1);
      tr[2] += diag_clock() - t1;
      tc_fence_after();
      const uint32_t d = a.tmem + 256 + (uint32_t)(ab * 128);
      auto chunk = [&](const int i) {  // i: processing index, kc: the K' chunk
        const int kc = s1_chunk_of(i, nkch);
        const int s = g_st % NST;
          const int rr = round_of(kc);
          if (rr == 0 ? !got0 : !got1) {  // the generated operand chunk of this round (first tile of a unit)
            t1 = diag_clock();
            mbar_wait(&S.a_full[rr], g_u & 1);
            tr[1] += diag_clock() - t1;
            tc_fence_after();
            if (rr == 0) got0 = true; else got1 = true;
          }
          t1 = diag_clock();
          mbar_wait(&S.st_full[s], (g_st / NST) & 1);
          tr[3] += diag_clock() - t1;
          tc_fence_after();
          const uint32_t st = a.sbase + s * a.stage_bytes;
          const uint64_t bh0 = smem_desc_kmajor_noswz(st, 128, a.SBO);
          const uint64_t bl0 = smem_desc_kmajor_noswz(st + a.part_bytes, 128, a.SBO);
          const uint32_t a_hi0 = a.tmem + (uint32_t)(kc * (KS * 8));
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const uint32_t a_hi = a_hi0 + (uint32_t)(ks * 8);
            const uint32_t a_lo = a_hi + (uint32_t)a.nk;
            const uint32_t acc = (i > 0 || ks > 0) ? 1u : 0u;
            mma(d, a_hi, bh0 + (uint64_t)(ks * 16), acc);  // +256 B per k-step
            mma(d, a_hi, bl0 + (uint64_t)(ks * 16), 1u);
            mma(d, a_lo, bh0 + (uint64_t)(ks * 16), 1u);
          }
          commit(&S.st_empty[s]);
          // last tile: a round's chunks are free once its last stage has been read
          if (t == a.nit - 1 && (i == nkch - 1 || (R == 2 && i == hq - 1)))
            commit(&S.a_empty[R == 1 ? 0 : (i == nkch - 1 ? 1 : 0)]);
          ++g_st;
      };
      if constexpr (NK > 0) {
#pragma unroll
        for (int kc = 0; kc < NK; ++kc) chunk(kc);
      } else {
        for (int kc = 0; kc < nkch; ++kc) chunk(kc);
      }
      commit(&S.acc_full[ab]);
    }
  }
  tr[0] = diag_clock() - tr0;
  return g_u;
}

// NKC: the k-chunk count at compile time (4: n_k = 128, the c5 shape; 0: runtime), a separate instance so
// that the unrolled MMA loop does not change the register allocation of the other shapes.
// CG2 (k_step1_cg2, opt-in FTK_S1CG2=1): a CTA pair (cluster of 2, cta_group::2) runs two adjacent column tiles
// of one mode as one M = 256 GEMM: each CTA generates its 128 rows into its own TMEM and loads HALF of every
// 128-image stage (64 images, 16 KB), so the image bytes each SM receives per tile halve; the even CTA issues
// the MMAs, a relay thread of the odd CTA forwards its stage completions, and the generators / epilogues of
// both CTAs arrive on the even CTA's barriers.
template <int NKC, bool CG2>
__device__ __forceinline__ void s1_body(const S1Params& P) {
  constexpr int NST = CG2 ? 8 : S1_STAGES;
  extern __shared__ __align__(1024) uint8_t s1_raw[];
  S1Smem& S = *reinterpret_cast<S1Smem*>(s1_raw);
  uint8_t* stages = s1_raw + 1024;                                   // NST x stage_bytes
  const uint32_t stage_bytes = (CG2 ? 64u : 128u) * P.KCH * 4u;      // hi + lo (this CTA's images)
  const uint32_t part_bytes = stage_bytes / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = P.n, nk = P.n_k;
  const uint32_t h = CG2 ? cluster_rank() : 0u;
  // units: (mode p, column tile ct); CTA pair: unit pairs (p, 2 ctp + h)
  const int NCTu = CG2 ? (P.NCT + 1) / 2 : P.NCT;
  const int units = n * NCTu;
  const int ubeg = CG2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ustep = CG2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  auto unit_of = [&](int u, int& p, int& ct) {
    s1_unit(u, NCTu, p, ct);
    if constexpr (CG2) ct = 2 * ct + (int)h;
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&S.st_full[i], (CG2 && h == 0) ? 2 : 1);  // CTA pair: + the odd CTA's relayed completion
      mbar_init(&S.st_empty[i], 1);
    }
    for (int r = 0; r < 2; ++r) {
      mbar_init(&S.a_full[r], CG2 ? 16 : 8);
      mbar_init(&S.a_empty[r], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.acc_full[i], 1);
      mbar_init(&S.acc_empty[i], CG2 ? 16 : 256);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG2)
      tmem_alloc_cg2<512>(&S.tmem_base);
    else
      tmem_alloc<512>(&S.tmem_base);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG2) cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  const int it0 = P.i0 / 128;
  const int nit = (P.ni + 127) / 128;

  if (warp == 0) {
    // ---------------- bulk-copy producer of image operand stages (CTA pair: this CTA's 64 images of each)
    if (lane == 0) {
      uint32_t g_st = 0;
      for (int u = ubeg; u < units; u += ustep) {
        int p, ct_unused;
        unit_of(u, p, ct_unused);
        for (int t = 0; t < nit; ++t) {
          for (int ci = 0; ci < P.NKCH; ++ci, ++g_st) {
            const int kc = s1_chunk_of(ci, P.NKCH);
            const int s = g_st % NST;
            mbar_wait(&S.st_empty[s], ((g_st / NST) & 1) ^ 1);
            const uint8_t* src = P.Aop + (((size_t)p * P.NIT + it0 + t) * P.NKCH + kc) * (size_t)(128u * P.KCH * 4u);
            mbar_arrive_expect_tx(&S.st_full[s], stage_bytes);
            if constexpr (CG2) {
              // the stage's [part][16 row groups][KCH/8][128 B]: this CTA's row groups [8 h, 8 h + 8) of each part
              for (int pt = 0; pt < 2; ++pt)
                bulk_g2s_hint(stages + s * stage_bytes + pt * part_bytes,
                              src + (size_t)pt * (128u * P.KCH * 2u) + (size_t)h * part_bytes, part_bytes,
                              &S.st_full[s], l2_policy_evict_last());
            } else if constexpr ((kS1Hint & 2) != 0) {
              bulk_g2s_hint(stages + s * stage_bytes, src, stage_bytes, &S.st_full[s], l2_policy_evict_last());
            } else {
              bulk_g2s(stages + s * stage_bytes, src, stage_bytes, &S.st_full[s]);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (h == 0) {
      // ---------------- MMA issuer (one elected lane; the k-steps of a stage unrolled at compile time)
      if (elect_one()) {
        S1MmaArgs a{tmem, smem_u32(stages), stage_bytes, part_bytes, (uint32_t)(P.KCH / 8) * 128u, P.KCH,
                    P.NKCH, nk, units, nit, ubeg, ustep, &S};
        long long tr[4] = {0, 0, 0, 0};
        uint32_t g_u = 0;
        if (P.KCH == 64) {
          g_u = s1_mma_loop<4, NKC, CG2>(a, tr);
        } else {
          g_u = s1_mma_loop<2, 0, CG2>(a, tr);
        }
        if (P.trace && blockIdx.x == 0) {
          P.trace[0] = tr[0];
          P.trace[1] = tr[1];
          P.trace[2] = tr[2];
          P.trace[3] = tr[3];
          P.trace[4] = g_u;
        }
      }
    } else if (CG2 && lane == 0) {
      // ---------------- relay (odd CTA): this CTA's stage completions -> the even CTA's stage barriers
      uint32_t g_st = 0;
      const int per_unit = nit * P.NKCH;
      for (int u = ubeg; u < units; u += ustep)
        for (int i = 0; i < per_unit; ++i, ++g_st) {
          const int s = g_st % NST;
          mbar_wait(&S.st_full[s], (g_st / NST) & 1);
          mbar_arrive_cluster(mapa_shared(&S.st_full[s], 0));
        }
    }
    __syncwarp();
  } else if (warp < 10) {
    // ---------------- generators of the template x G operand (A, TMEM columns [0, 2 n_k)); 8 warps: two
    // per TMEM lane quarter, each half of the radial nodes m; loads issued two 16-node steps at a time
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int c = row >> 1, part = row & 1;
    const int mh = (warp - 2) >> 2;  // radial half
    const uint32_t base = tmem + ((uint32_t)(q * 32) << 16);
    const int half = nk / 2;  // u32 columns per K' half
    // generation rounds (as in s1_mma_loop): R = 2 -> round r covers m in [r n_k/2, (r+1) n_k/2), each warp of
    // the quarter pair a quarter of n_k; R = 1 -> each warp half of n_k (n_k < 32: a half would be
    // narrower than one 16-node STTM step; the first-half warps do all nodes)
    const int R = (P.NKCH % 4 == 0) ? 2 : 1;
    const uint64_t pol_b = (kS1Hint & 4) ? l2_policy_evict_last() : 0;
    uint32_t a_full_cl[2] = {0u, 0u};
    if constexpr (CG2) {
      a_full_cl[0] = mapa_shared(&S.a_full[0], 0);
      a_full_cl[1] = mapa_shared(&S.a_full[1], 0);
    }
    uint32_t g_u = 0;
    for (int u = ubeg; u < units; u += ustep, ++g_u) {
      int p, ct;
      unit_of(u, p, ct);
      const int f = ct * 64 + c;
      int jl = 0, z = 0;
      if (f < P.F) {
        jl = f / P.Hs;
        z = f - jl * P.Hs;
      }
      // slots z >= Hp (the Zhat' row padding, Hs > Hp) get zero operand rows, so the epilogue writes whole
      // rows: a never-written slot leaves a partial 32-byte sector in every row, which L2 must complete by a
      // DRAM read-modify-write (that made Step 1 2x slower whenever Hs > Hp)
      const bool valid = f < P.F && z < P.Hp;
      const int qt = valid ? ((p + __ldg(P.ell + z)) & (n - 1)) : 0;
      // fp16x3 operand scale of this row's template (folded into g: (g 2^e) b = (g b) 2^e exactly)
      const float gsc = pow2f(valid ? s1_gen_exp(P.bst, P.gmax, P.j0 + jl) : 0);
      const float2* brow = P.B + ((size_t)(P.j0 + jl) * n + qt) * nk;
      const float* grow = P.g + (size_t)z * nk;
      for (int rnd = 0; rnd < R; ++rnd) {
      int m_beg, m_end;
      if (R == 2) {
        m_beg = rnd * half + mh * (nk / 4);
        m_end = m_beg + nk / 4;
      } else {
        m_beg = nk >= 32 ? mh * half : 0;
        m_end = nk >= 32 ? m_beg + half : (mh == 0 ? nk : 0);
      }
      mbar_wait(&S.a_empty[rnd], (g_u & 1) ^ 1);
      tc_fence_after();
#ifndef FTK_S1_GEN16
#define FTK_S1_GEN16 1
#endif
      // 16 radial nodes per step (one STTM group each): fewer loads in flight than two steps at a time, no
      // register spills at the 96-register cap
      for (int m0 = m_beg; m0 < m_end; m0 += FTK_S1_GEN16 ? 16 : 32) {
        constexpr int NS2 = FTK_S1_GEN16 ? 1 : 2;
        float4 bb[NS2][8];
        float2 gg[NS2][8];
#pragma unroll
        for (int s2 = 0; s2 < NS2; ++s2)
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int m = m0 + 16 * s2 + 2 * e;
            const bool ok = valid && m < m_end;
            if constexpr ((kS1Hint & 4) != 0)
              bb[s2][e] = ok ? ldg_f4_hint(reinterpret_cast<const float4*>(brow + m), pol_b) : make_float4(0.f, 0.f, 0.f, 0.f);
            else
              bb[s2][e] = ok ? __ldg(reinterpret_cast<const float4*>(brow + m)) : make_float4(0.f, 0.f, 0.f, 0.f);
            gg[s2][e] = ok ? mul2(make_float2(gsc, gsc), __ldg(reinterpret_cast<const float2*>(grow + m)))
                           : make_float2(0.f, 0.f);
          }
#pragma unroll
        for (int s2 = 0; s2 < NS2; ++s2) {
          if (m0 + 16 * s2 >= m_end) break;
          uint32_t h1[8], l1[8], h2[8], l2[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            // c = g conj(b) for nodes m, m + 1: one packed multiply each
            const float2 c0 = mul2(make_float2(gg[s2][e].x, gg[s2][e].x), make_float2(bb[s2][e].x, -bb[s2][e].y));
            const float2 c1 = mul2(make_float2(gg[s2][e].y, gg[s2][e].y), make_float2(bb[s2][e].z, -bb[s2][e].w));
            const float cr0 = c0.x, ci0 = c0.y, cr1 = c1.x, ci1 = c1.y;
            // Re-row: [c_r | -c_i],  Im-row: [c_i | c_r]  (branch-free)
            split2_f16(part ? ci0 : cr0, part ? ci1 : cr1, h1[e], l1[e]);
            split2_f16(part ? cr0 : -ci0, part ? cr1 : -ci1, h2[e], l2[e]);
          }
          const uint32_t col = (uint32_t)((m0 + 16 * s2) / 2);
          tmem_st8(base + col, h1);
          tmem_st8(base + half + col, h2);
          tmem_st8(base + nk + col, l1);
          tmem_st8(base + nk + half + col, l2);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG2)
          mbar_arrive_cluster(a_full_cl[rnd]);
        else
          mbar_arrive(&S.a_full[rnd]);
      }
      }
    }
  } else {
    // ---------------- epilogue: accumulator [128 rows (j,zeta,part)] x [128 images] -> Zhat', straight from
    // TMEM to global memory (no shared-memory staging: shared-memory bandwidth is taken by the MMA operand
    // reads and the stage copies).  Lane pairs (2c, 2c + 1) hold the Re / Im rows of complex column c: one
    // shuffle per two images turns them into an (Re, Im) float2 for image e (even lane) and e + 1 (odd lane),
    // so each store instruction writes two 128-byte row segments.
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int ew = warp - 10;  // 0..7
    const int eh = ew >> 2;    // image half of the TMEM columns this warp drains
    const bool odd = lane & 1;
    uint32_t acc_empty_cl[2] = {0u, 0u};
    if constexpr (CG2) {
      acc_empty_cl[0] = mapa_shared(&S.acc_empty[0], 0);
      acc_empty_cl[1] = mapa_shared(&S.acc_empty[1], 0);
    }
    uint32_t g_acc = 0;
    for (int u = ubeg; u < units; u += ustep) {
      int p, ct;
      unit_of(u, p, ct);
      const int f = ct * 64 + (row >> 1);  // this lane's complex column (template jl, slot z)
      const bool cval = f < P.F;           // pad slots included (zero rows)
      const int jl = cval ? f / P.Hs : 0, z = f - jl * P.Hs;
      // Zhat'[pair (il, jl)][p][z] = Zhat + (il nj + jl) n Hs + p Hs + z
      const size_t coff = ((size_t)jl * n + p) * P.Hs + z;
      const size_t istride = (size_t)P.nj * n * P.Hs;
      for (int t = 0; t < nit; ++t, ++g_acc) {
        const int ab = g_acc & 1;
        mbar_wait(&S.acc_full[ab], (g_acc >> 1) & 1);
        tc_fence_after();
        const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + 256 + (uint32_t)(ab * 128);
#pragma unroll 1
        for (int c0 = 64 * eh; c0 < 64 * eh + 64; c0 += 32) {
          uint32_t r[32];
          tmem_ld16(base + c0, *reinterpret_cast<uint32_t(*)[16]>(r));
          tmem_ld16(base + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(r + 16));
          tmem_wait_ld();
          if (c0 + 32 == 64 * eh + 64) {  // this warp's last columns are in registers: release the buffer
            tc_fence_before();
            if constexpr (CG2) {
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(acc_empty_cl[ab]);
            } else {
              mbar_arrive(&S.acc_empty[ab]);
            }
          }
          const int ibase = t * 128 + c0;  // local image index of r[0]
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            // even lane: (Re, Im) of image e; odd lane: (Re, Im) of image e + 1
            const float send = __uint_as_float(odd ? r[e] : r[e + 1]);
            const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
            const float2 v = odd ? make_float2(recv, __uint_as_float(r[e + 1])) : make_float2(__uint_as_float(r[e]), recv);
            const int il = ibase + e + (odd ? 1 : 0);
            if (cval && il < P.ni) P.Zhat[(size_t)il * istride + coff] = v;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG2) cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG2)
      tmem_dealloc_cg2<512>(tmem);
    else
      tmem_dealloc<512>(tmem);
  }
}

template <int NKC>
__global__ void __maxnreg__(96) k_step1_tc(S1Params P) {
  s1_body<NKC, false>(P);
}
template <int NKC>
__global__ void __cluster_dims__(2, 1, 1) __maxnreg__(96) k_step1_cg2(S1Params P) {
  s1_body<NKC, true>(P);
}

static size_t s1_smem_bytes(const TcPlan& tc) { return 1024 + (size_t)S1_STAGES * 128 * tc.KCH * 4; }

// Image operand prep: FB a[i][q][m] -> scaled fp16 hi/lo canonical K-major tiles (B operand of Step 1).
__global__ void k_prep_image_op(const float2* __restrict__ fb, uint8_t* __restrict__ Aop, int NI, int NIT, int n,
                                int nk, int KCH, int NKCH, const float2* __restrict__ ast) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int groups = (2 * nk) / 8;  // 8-element k' groups per row
  const int64_t total = (int64_t)NIT * 128 * n * groups;
  if (tid >= total) return;
  const int gk = (int)(tid % groups);
  int64_t rest = tid / groups;
  const int i = (int)(rest % (NIT * 128));
  const int p = (int)(rest / (NIT * 128));
  const int k0 = gk * 8;
  float v[8];
  const float asc = pow2f(i < NI ? s1_img_exp(ast, i) : 0);  // fp16x3 operand scale of image i
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int kp = k0 + e;
    float x = 0.f;
    if (i < NI) {
      const float2 a = fb[((size_t)i * n + p) * nk + (kp < nk ? kp : kp - nk)];
      x = (kp < nk ? a.x : a.y) * asc;
    }
    v[e] = x;
  }
  uint4 h, l;
  split2_f16(v[0], v[1], h.x, l.x);
  split2_f16(v[2], v[3], h.y, l.y);
  split2_f16(v[4], v[5], h.z, l.z);
  split2_f16(v[6], v[7], h.w, l.w);
  const int it = i / 128, ii = i % 128, kch = k0 / KCH, kk = k0 % KCH;
  const size_t stage_bytes = 128u * KCH * 4u;
  uint8_t* st = Aop + (((size_t)p * NIT + it) * NKCH + kch) * stage_bytes;
  const size_t off = (size_t)(ii / 8) * (KCH / 8) * 128 + (kk / 8) * 128 + (ii % 8) * 16;
  *reinterpret_cast<uint4*>(st + off) = h;
  *reinterpret_cast<uint4*>(st + 128u * KCH * 2u + off) = l;
}

// Step 2 for the tensor-core engine (Eq. fbk3 Step 2, Form B):
//   Z_zeta(r) = e^{-2 pi i ell r / n} sum_p Zhat'_zeta(p) e^{-2 pi i p r / n},   (q = p + ell)
// read from Zhat' [pair][p][Hs] (Form B, written by k_step1_tc); written as the Step-3 A operand rows
// (real columns of reading R13), scaled fp16 hi/lo packed in 32-bit words (two K columns per word), per (pair,
// r-tile, part) the canonical K-major core-matrix image [row/8][word group][8 rows x 16 B] that k_step3_tc
// bulk-copies and tcgen05.cp-s into TMEM.
// Work item = (pair, Step-2 block of <= 8 terms in one aligned 8-term window); persistent CTAs; the item's
// input window arrives by 2-D TMA; one warp per term.
// FFT: four-step decomposition n = 32 E, p = a + 32 b (a = lane), r = c + E d:
//   (A) per lane an E-point DFT over b in registers, (B) twiddle w_n^{a c}, (C) a 32-point radix-2
//   DIF across the warp with shfl_xor (output index d lands on lane bitrev5(d)).
// Output words are staged per (group, part, word) in padded rows (index r + r / E: conflict-free) and
// written out as contiguous 2 KB row blocks.
using S2Blocks = S2BlockTable;
// w_32^k = e^{-2 pi i k / 32}, k < 32 (Step 2's (B2) twiddles for L = 2, read with compile-time indices)
__constant__ float2 c_w32[32];

template <int E>
__global__ void __launch_bounds__(256, (E >= 16 ? 3 : 4)) k_step2_fft(uint8_t* __restrict__ Zop,
                                                      int npair, DevPlan P, S2Blocks B, PairBlock pb,
                                                      const float2* __restrict__ ast, const float2* __restrict__ bst,
                                                      float gmax,
                                                      const float2* __restrict__ twtab,
                                                      const __grid_constant__ CUtensorMap zmap) {
  extern __shared__ __align__(1024) uint8_t s2raw[];
  constexpr int n = 32 * E;  // FFT length = n_gamma (>= n_psi; zero-padded input, reading R21)
  constexpr int LOG = (E == 32) ? 5 : (E == 16) ? 4 : (E == 8 ? 3 : (E == 4 ? 2 : 1));
  constexpr int RS = n + n / E;  // padded staging row (words): index r + r / E
  const int n_in = P.n_psi;     // input rows (cyclic q)
  // [rows: n_in x S2_SMAX complex][stg: 16 x RS words; also the warps' n-slot transpose scratch][mbarrier]
  float2* rows = reinterpret_cast<float2*>(s2raw);
  const size_t rows_bytes = (size_t)n_in * S2_SMAX * 8;
  uint32_t* stg = reinterpret_cast<uint32_t*>(s2raw + rows_bytes);
  uint64_t* bar = reinterpret_cast<uint64_t*>(stg + 16 * RS);
  // warp index made provably warp-uniform (shfl from lane 0) so the shuffles below sit in convergent code
  const int lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  // transpose scratch: 8 warps x E rows of (32 + L) complex (row padding L makes both the row-wise stores and
  // the strided loads conflict-free and the indices compile-time offsets); 8 E (32 + L) complex = 16 RS words
  constexpr int SROW = 32 + 32 / E;
  float2* scr = reinterpret_cast<float2*>(stg) + warp * E * SROW;
  const int total = npair * B.nb;
  const int NWG = P.K3p / 8, NRT = (n + 127) / 128;

  // 32 = L x E: the 32-point DFT over the lane index runs as an E-point register DFT and an L-point
  // DIF across L lanes (log2 L shuffle stages)
  constexpr int L = 32 / E;
  constexpr int LL = (L == 16) ? 4 : (L == 8) ? 3 : (L == 4) ? 2 : (L == 2) ? 1 : 0;
  float2 wc[LL > 0 ? LL : 1];  // stage twiddle of this lane (1 on the upper lanes of each butterfly)
#pragma unroll
  for (int s = 0; s < LL; ++s) {
    const int h = (L / 2) >> s;
    wc[s] = (lane & h) ? tw_full(P.twg, (lane & (h - 1)) * ((L / 2) / h) * (n / L), n) : make_float2(1.f, 0.f);
  }
  int gq = 0;  // L-point DIF output index of this lane: bit-reversed lane % L
#pragma unroll
  for (int bb = 0; bb < LL; ++bb) gq |= (((lane % L) >> bb) & 1) << (LL - 1 - bb);
  // (B) twiddles w_n^{a c} (a = lane, c < E) and (B2) twiddles w_32^{h d'} (h = lane % L, d' < E), both
  // [c][lane] (plan-time tables, L1-resident)
  const float2* __restrict__ twB = twtab;
  const float2* __restrict__ twC = twtab + E * 32;
  auto rv = [](int i) {
    int r = 0;
#pragma unroll
    for (int bb = 0; bb < LOG; ++bb) r |= ((i >> bb) & 1) << (LOG - 1 - bb);
    return r;
  };

  // contiguous item range per CTA (the blocks of one pair back to back)
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int i_beg = blockIdx.x * per;
  const int i_end = min(total, i_beg + per);
  // input: the aligned 8-term window [zs & ~1, +8) holding the block's terms, for the pair's n_psi rows of
  // Zhat' [pair][p][Hs] (Form B), as 2-D TMA boxes (8 x 256, zero fill beyond Hs) into the swizzled [p][8]
  // row buffer.  A box must start on a 16-byte boundary (an odd 8-byte column start faults); the device
  // term order (tc_term_order) puts every block inside one such window.
  auto issue = [&](int it) {
    const int bi = it % B.nb, pi2 = it / B.nb;
    if (threadIdx.x == 0) {
      const int box = n_in < 256 ? n_in : 256;
      mbar_arrive_expect_tx(bar, (uint32_t)n_in * 64u);
      for (int k = 0; k < n_in; k += box)
        tma_load_2d(s2raw + (size_t)k * 64, &zmap, B.zs[bi] & ~1, pi2 * n_in + k, bar);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (i_beg < i_end) issue(i_beg);
  uint32_t phase = 0;
  for (int item = i_beg; item < i_end; ++item) {
    const int b = item % B.nb, pr = item / B.nb;
    const int zs = B.zs[b], nz = B.ze[b] - zs, g0 = B.g0[b];
    // fp16x3 statistics of the item's pair and this warp's term (ell, Step-3 column), loaded before the
    // row wait so that their latency overlaps it
    float2 st_a, st_b;
    {
      int pi_, pj_;
      pair_of(pb, pr, pi_, pj_);
      st_a = __ldg(ast + pi_);
      st_b = __ldg(bst + pj_);
    }
    const int zz = warp;
    const bool act = zz < nz;
    int l = 0, col = 0;
    if (act) {
      l = __ldg(P.ell + zs + zz);
      col = __ldg(P.col + zs + zz);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    // ---- each warp takes one term: load its row (cyclic shift by ell, zero padding to n)
    float2 x[E];
    if (act) {
      const int e = (zs & 1) + zz;  // window column of this term
      auto at = [&](int p) { return rows[s2_slot(p, e)]; };
      // Form B: Z(r) w^{ell r} = DFT of the cyclically shifted row Zhat'(q - ell) (reading R5)
      if (n_in == n) {
        const int q0 = (lane - l) & (n - 1);
#pragma unroll
        for (int bb = 0; bb < E; ++bb) x[bb] = at((q0 + 32 * bb) & (n - 1));
      } else {
        // n_gamma > n_psi: zero-padded signed frequencies, Nyquist split (reading R21)
        const int Qh = n_in >> 1;
#pragma unroll
        for (int bb = 0; bb < E; ++bb) {
          const int qp = lane + 32 * bb;
          const int qc = qp < Qh ? qp : (qp > n - Qh ? qp - n + n_in : Qh);
          const float wgt = (qp < Qh || qp > n - Qh) ? 1.f : ((qp == Qh || qp == n - Qh) ? 0.5f : 0.f);
          const int src = (qc - l) & (n_in - 1);
          const float2 v = at(src);
          x[bb] = mul2(make_float2(wgt, wgt), v);
        }
      }
    }
    __syncthreads();  // the row buffer is free: prefetch the next item while this one is transformed
    if (item + 1 < i_end) issue(item + 1);
    if (act) {
      dft_regs<E>(x);  // (A) E-point DFT over b (p = a + 32 b, a = lane): natural order in x[rv(c)]
#pragma unroll
      for (int c = 1; c < E; ++c) x[rv(c)] = cmulf(x[rv(c)], __ldg(twB + c * 32 + lane));  // (B) x_c *= w_n^{a c}
      // (T) the 32-point DFT over a: transpose through this warp's scratch (slot c*32 + (a + c) % 32) so
      //     that lane (c = lane / L, h = lane % L) holds a = L i + h, i < E; then (A2) an E-point DFT over i
      //     in registers, (B2) twiddle w_32^{h d'}, (C2) an L-point DIF across the L lanes of each c.
#pragma unroll
      for (int c = 0; c < E; ++c) scr[c * SROW + lane] = x[rv(c)];
      __syncwarp();
      {
        const int cq = lane / L, hq = lane % L;
#pragma unroll
        for (int i = 0; i < E; ++i) x[i] = scr[cq * SROW + L * i + hq];
      }
      dft_regs<E>(x);  // (A2): natural order in x[rv(d')]
      if constexpr (L > 1) {
        if constexpr (L == 2) {  // (B2) w_32^{(lane % 2) d'}: 1 on even lanes, a constant-bank value on odd lanes
          const bool oddl = lane & 1;
#pragma unroll
          for (int dd = 1; dd < E; ++dd) {
            const float2 t = cmulf(x[rv(dd)], c_w32[dd]);
            x[rv(dd)] = oddl ? t : x[rv(dd)];
          }
        } else {
#pragma unroll
          for (int dd = 1; dd < E; ++dd) x[rv(dd)] = cmulf(x[rv(dd)], __ldg(twC + dd * 32 + lane));  // (B2)
        }
#pragma unroll
        for (int s = 0; s < LL; ++s) {  // (C2) L-point DIF across lanes (branch-free butterfly)
          const int h = (L / 2) >> s;
          const float sg = (lane & h) ? -1.f : 1.f;  // upper lane: x + x', lower lane: (x' - x) w
#pragma unroll
          for (int c = 0; c < E; ++c) {
            const float px = __shfl_xor_sync(0xffffffffu, x[c].x, h);
            const float py = __shfl_xor_sync(0xffffffffu, x[c].y, h);
            x[c] = cmulf(fma2(make_float2(sg, sg), x[c], make_float2(px, py)), wc[s]);
          }
        }
      }
    }
    __syncthreads();  // all transposes done: the staging area is free
    if (act) {
      // lane holds Z(r), r = cq + E (d' + E g) in x[rv(d')], cq = lane / L, g = bitrev_L(lane % L)
      // stage: ell > 0 -> word (Re, Im) of this term; ell = 0 -> one 16-bit half of a word shared with
      // the neighbouring ell = 0 term (a term without a neighbour writes the whole word, upper half 0)
      const int kl = col - 8 * g0;  // 0..15 within the block
      const int grp = kl >> 3, w = (kl & 7) >> 1;
      const float zsc = zhat_to_z_scale(st_a, st_b, gmax);  // fp16x3: Zhat' scale -> Z scale
      const bool lone = (B.lone[b] >> zz) & 1;
      uint32_t* shi = stg + (size_t)((grp * 2 + 0) * 4 + w) * RS;
      uint32_t* slo = stg + (size_t)((grp * 2 + 1) * 4 + w) * RS;
      const int pbase = lane / L + (E * E + E) * gq;  // padded index pi(r) = r + r / E
#pragma unroll
      for (int dd = 0; dd < E; ++dd) {
        const int pi = pbase + (E + 1) * dd;
        const float2 a0 = mul2(make_float2(zsc, zsc), x[rv(dd)]);
        if (l > 0) {
          uint32_t hh, ll;
          split2_f16(a0.x, a0.y, hh, ll);
          shi[pi] = hh;
          slo[pi] = ll;
        } else if (lone) {
          uint32_t hh, ll;
          split2_f16(a0.x, 0.f, hh, ll);
          shi[pi] = hh;
          slo[pi] = ll;
        } else {
          const __half hb = __float2half_rn(a0.x);
          const __half lb = __float2half_rn(a0.x - __half2float(hb));
          reinterpret_cast<__half*>(shi + pi)[kl & 1] = hb;
          reinterpret_cast<__half*>(slo + pi)[kl & 1] = lb;
        }
      }
    }
    __syncthreads();
    // ---- write out the block's word groups as core-matrix rows; words no term writes are zero.
    //      Thread = (row, part): per (group, r-tile) one 16-byte store; 8-row runs are contiguous 128 B.
    {
      const int ng = B.ng[b];
      const uint32_t used = (uint32_t)B.used[b];  // bit grp * 4 + w
      const int row = threadIdx.x & 127, part = threadIdx.x >> 7;
      uint8_t* dst = Zop + (size_t)pr * NRT * 128 * P.K3p * 4 + (size_t)g0 * 128 + (size_t)part * NWG * 2048 +
                     (size_t)(row >> 3) * NWG * 128 + (row & 7) * 16;
      for (int grp = 0; grp < ng; ++grp) {
        const uint32_t um = used >> (grp * 4);
        const uint32_t* sp = stg + (size_t)((grp * 2 + part) * 4) * RS;
#pragma unroll
        for (int T = 0; T < (n + 127) / 128; ++T) {
          const int r = T * 128 + row;
          uint4 v = make_uint4(0u, 0u, 0u, 0u);
          if (r < n) {
            const int pi = r + r / E;
            v.x = (um & 1u) ? sp[pi] : 0u;
            v.y = (um & 2u) ? sp[RS + pi] : 0u;
            v.z = (um & 4u) ? sp[2 * RS + pi] : 0u;
            v.w = (um & 8u) ? sp[3 * RS + pi] : 0u;
          }
          *reinterpret_cast<uint4*>(dst + (size_t)T * 2 * NWG * 2048 + (size_t)grp * 128) = v;
        }
      }
    }
    __syncthreads();  // the staging area becomes transpose scratch again
  }
}

static size_t step2_smem(int n_in, int n) {  // n_in = n_psi input rows, n = n_gamma >= n_in FFT length
  const int E = n / 32;
  return (size_t)n_in * S2_SMAX * 8 + (size_t)16 * (n + n / E) * 4 + 16;
}

static CUtensorMapL2promotion s2_l2_promotion() {  // FTK_S2_L2PROMO = 0 / 64 / 128 / 256 (diagnostics)
  const char* e = std::getenv("FTK_S2_L2PROMO");
  const int v = e ? std::atoi(e) : 64;  // 64: 17 % less DRAM read than 128 at c5, same time
  return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                          : v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
}

// Zhat' [pair][p][Hs] as a 2-D tensor of 8-byte elements (rows = pair * n_psi + p), 8 x 256 boxes,
// 64-byte swizzle (the layout s2_slot() reads)
static int make_zmap(CUtensorMap* m, const float2* Zhat, int npair, const DevPlan& P) {
  PFN_encodeTiled enc = get_encode_tiled();
  if (!enc) return FTK_ECUDA;
  const cuuint64_t dims[2] = {(cuuint64_t)P.Hs, (cuuint64_t)npair * P.n_psi};
  const cuuint64_t strides[1] = {(cuuint64_t)P.Hs * 8};
  const cuuint32_t box[2] = {8u, (cuuint32_t)(P.n_psi < 256 ? P.n_psi : 256)};
  const cuuint32_t es[2] = {1u, 1u};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<float2*>(Zhat), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, s2_l2_promotion(),
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? FTK_OK : FTK_ECUDA;
}

static int launch_step2_fft(const TcPlan& tc, const float2* Zhat, uint8_t* Zop, int npair, const PairBlock& pb,
                            const DevPlan& P, cudaStream_t s) {
  S2Blocks B;
  std::memcpy(&B, &tc.s2_blocks, sizeof B);
  alignas(64) CUtensorMap zmap;
  std::memset(&zmap, 0, sizeof zmap);
  if (make_zmap(&zmap, Zhat, npair, P) != FTK_OK) return FTK_ECUDA;
  if (tc.sync_debug)
    fprintf(stderr, "step2: Zhat %p (mod 256 = %d) Hs %d npair %d n_psi %d n_gamma %d smem %zu grid %d\n", (const void*)Zhat,
            (int)((uintptr_t)Zhat & 255), P.Hs, npair, P.n_psi, P.n_gamma, step2_smem(P.n_psi, P.n_gamma),
            B.nb * npair < 2 * tc.num_sms ? B.nb * npair : 2 * tc.num_sms);
  const size_t smem = step2_smem(P.n_psi, P.n_gamma);
  const int items = B.nb * npair;
  auto run = [&](auto kern) {
    int occ = 2;  // resident CTAs per SM (registers <= 80 at E <= 16; shared memory decides)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
    occ = std::max(1, std::min(occ, 4));
    dim3 grid(items < occ * tc.num_sms ? items : occ * tc.num_sms);
    kern<<<grid, 256, smem, s>>>(Zop, npair, P, B, pb, tc.d_ast, tc.d_bst, tc.gmax, tc.d_s2tw, zmap);
  };
  switch (P.n_gamma) {
    case 64: run(k_step2_fft<2>); break;
    case 128: run(k_step2_fft<4>); break;
    case 256: run(k_step2_fft<8>); break;
    case 512: run(k_step2_fft<16>); break;
    default: run(k_step2_fft<32>); break;
  }
  return FTK_OK;
}

// ---------------------------------------------------------------- Step 2 on the tensor cores (n_gamma = n_psi = 64 R)
// The same Z as k_step2_fft (Eq. fbk3 Step 2, Form B: x(q) = Zhat'(q - ell), reading R5), by the
// four-step split q = a + 64 b (a < 64, b < R), r = c + R d (c < R, d < 64), n = 64 R, R = 2, 4, 8:
//   Z(c + R d) = sum_a w64^{a d} T(a, c),   T(a, c) = w_n^{a c} sum_b x(a + 64 b) w_R^{b c}     (w_m = e^{-2 pi i / m})
// * T on the CUDA cores: per (slot, a) an R-point register DFT and R - 1 twiddles, scaled into Z's fp16x3 range (the
//   bound of the file header holds for every partial sum of the DFT), split into fp16 hi / lo and stored as the B
//   operand: MN-major (N = (slot, c), K = (Re | Im, a)), canonical core matrices, one stage per block.
// * The DFT-64 over a as ONE GEMM D[(d, Re|Im)][(slot, c)] = F64 . T, F64 = the real 128 x 128 form of
//   [w64^{a d}] (rows m = 2 d + Re|Im, columns k = Re|Im * 64 + a) as fp16 hi / lo, resident in TMEM as the A
//   operand for the whole kernel: 3 x 8 tcgen05.mma M128 N(8 R) K16 per block (fp16x3; N = 4 R for blocks of
//   one word group when 4 R >= 16).
// * Epilogue from TMEM: lane (d, Re) forms the hi words, lane (d, Im) the lo words of rows R d + c of the Step-3
//   operand (one shuffle per two values exchanges the halves), staged 128B-swizzled in shared memory and written
//   by one 5-D TMA store per word group.  Slot s of a block is Step-3 word s (group s / 4, word s % 4): an ell > 0
//   term (Re Z, Im Z), or two ell = 0 terms transformed together as x_1 + i x_2 (their Z are real for real images,
//   reading R13: Re -> low half, Im -> high half).
// Warps: 0 TMA producer (8-term Zhat' windows, NR-deep ring), 1 MMA issuer, 2-9 builders (T -> B operand,
// NB-deep ring), 10-17 epilogue (two TMEM accumulators).  Buffers are sized for R = 8.
constexpr int S2T_THREADS = 18 * 32;
constexpr int S2T_NR = 3, S2T_NB = 2, S2T_NO = 2;  // rows ring, B-operand ring, output staging buffers
constexpr uint32_t S2T_ROWS_BYTES = 512u * 8u * 8u;  // one block window: n <= 512 rows x 8 terms, complex fp32
constexpr uint32_t S2T_BOP_PART = 8u * 2048u;        // one part (hi or lo) of a B stage: <= 8 N-cores x 16 K-cores x 128 B
constexpr uint32_t S2T_BOP_BYTES = 2u * S2T_BOP_PART;
constexpr uint32_t S2T_OUT_BYTES = 2u * 16384u;       // epilogue staging of one block: <= 2 word groups x 16 KB
constexpr size_t S2T_SMEM = (size_t)S2T_NR * S2T_ROWS_BYTES + (size_t)S2T_NB * S2T_BOP_BYTES + S2T_NO * S2T_OUT_BYTES + 512;

struct S2TParams {
  uint8_t* Zop;
  int npair, NWG, K3p, dbg;
  PairBlock pb;
  const float2* ast;
  const float2* bst;
  float gmax;
  const uint32_t* F;  // [128 rows][64 hi words, 64 lo words]
  const float2* tw;   // [64 a][8] w_n^{a c}, c < R
  S2BlockTable B;
  S2TSlotTable sl;
};
struct S2TMeta {  // per rows stage, written by the producer before the TMA is armed
  float zsc;
  int bi;
};

template <int NC>
__device__ __forceinline__ void tmem_ld_x(uint32_t taddr, uint32_t (&r)[NC]) {  // 32 lanes x NC columns
  if constexpr (NC == 4)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
  else if constexpr (NC == 2)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
  else
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(taddr));
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
template <int R>
__device__ __forceinline__ void sts_bytes(uint8_t* p, const uint32_t (&w)[R / 2]) {  // 2 R bytes
  if constexpr (R == 8)
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  else if constexpr (R == 4)
    *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
  else
    *reinterpret_cast<uint32_t*>(p) = w[0];
}

template <int R>
__global__ void __launch_bounds__(S2T_THREADS, 1) k_step2_tc(const __grid_constant__ S2TParams P,
                                                            const __grid_constant__ CUtensorMap zmap,
                                                            const __grid_constant__ CUtensorMap omap) {
  constexpr int n = 64 * R, NRT = n / 128, H = R / 2;  // H: c values per epilogue warp half
  constexpr int LOGR = R == 8 ? 3 : (R == 4 ? 2 : 1);
  extern __shared__ __align__(1024) uint8_t s2traw[];
  uint8_t* rows_base = s2traw;
  uint8_t* bop_base = s2traw + S2T_NR * S2T_ROWS_BYTES;
  uint8_t* out_base = bop_base + S2T_NB * S2T_BOP_BYTES;  // NO x (2 groups x [T][part 2][row group 16][128 B])
  uint64_t* bars = reinterpret_cast<uint64_t*>(out_base + S2T_NO * S2T_OUT_BYTES);
  uint64_t* rows_full = bars;
  uint64_t* rows_empty = bars + S2T_NR;
  uint64_t* bop_full = bars + 2 * S2T_NR;
  uint64_t* bop_empty = bop_full + S2T_NB;
  uint64_t* d_full = bop_empty + S2T_NB;
  uint64_t* d_empty = d_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + 2);
  S2TMeta* meta = reinterpret_cast<S2TMeta*>(tmem_slot + 2);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int nb = P.B.nb;
  const int total = P.npair * nb;
  const int per = (total + gridDim.x - 1) / gridDim.x;
  const int i_beg = blockIdx.x * per;
  const int nit = max(0, min(total, i_beg + per) - i_beg);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S2T_NR; ++i) {
      mbar_init(rows_full + i, 1);
      mbar_init(rows_empty + i, 8);
    }
    for (int i = 0; i < S2T_NB; ++i) {
      mbar_init(bop_full + i, 8);
      mbar_init(bop_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(d_full + i, 1);
      mbar_init(d_empty + i, 8);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // columns [0, 128): two accumulators; [128, 192): F hi; [192, 256): F lo
  if (warp >= 2 && warp <= 9) {      // F64 into TMEM: two builder warps per lane quarter, 64 columns each
    const int q = warp & 3, hh = (warp - 2) >> 2;
    const uint32_t* src = P.F + (size_t)(q * 32 + lane) * 128 + hh * 64;
    const uint32_t dst = tmem + ((uint32_t)(q * 32) << 16) + 128u + (uint32_t)hh * 64u;
#pragma unroll 1
    for (int c0 = 0; c0 < 64; c0 += 16) {
      uint32_t v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = __ldg(src + c0 + k);
      tmem_st16(dst + c0, v);
    }
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    // ---------------- TMA producer: the block's aligned 8-term window of the pair's n Zhat' rows, plus the
    // item's metadata (block, Zhat' -> Z scale) for the builders
    if (lane == 0) {
      int bi = i_beg % nb, pr = i_beg / nb;
      for (int k = 0; k < nit; ++k) {
        const int st = k % S2T_NR;
        int pi_, pj_;
        pair_of(P.pb, pr, pi_, pj_);
        const float zsc = zhat_to_z_scale(__ldg(P.ast + pi_), __ldg(P.bst + pj_), P.gmax);
        mbar_wait(rows_empty + st, ((k / S2T_NR) & 1) ^ 1);
        meta[st].zsc = zsc;
        meta[st].bi = bi;
        uint8_t* dst = rows_base + st * S2T_ROWS_BYTES;
        mbar_arrive_expect_tx(rows_full + st, (uint32_t)n * 64u);
#pragma unroll
        for (int r0 = 0; r0 < n; r0 += 256)
          tma_load_2d(dst + r0 * 64, &zmap, P.B.zs[bi] & ~1, pr * n + r0, rows_full + st);
        if (++bi == nb) {
          bi = 0;
          ++pr;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer: D[db] = F64 . T (fp16x3: Fhi Thi + Fhi Tlo + Flo Thi), 8 k-steps
    if (lane == 0) {
      // B MN-major; blocks of one word group (slots 0-3) run N = 4 R where that is a valid MMA width
      constexpr int NF = 8 * R, NH = 4 * R >= 16 ? 4 * R : 8 * R;
      const uint32_t idescF = idesc_f16_f32(128, NF) | (1u << 16), idescH = idesc_f16_f32(128, NH) | (1u << 16);
      int bi = i_beg % nb;
      for (int k = 0; k < nit; ++k) {
        const int sb = k % S2T_NB, db = k & 1;
        const uint32_t idesc = P.B.ng[bi] > 1 ? idescF : idescH;
        if (++bi == nb) bi = 0;
        mbar_wait(bop_full + sb, (k / S2T_NB) & 1);
        mbar_wait(d_empty + db, ((k >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t bh = smem_u32(bop_base + sb * S2T_BOP_BYTES), bl = bh + S2T_BOP_PART;
        const uint32_t d = tmem + (uint32_t)db * 64u, fh = tmem + 128u, fl = tmem + 192u;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint64_t dh = smem_desc_kmajor_noswz(bh + ks * 256, 128, 2048);
          const uint64_t dl = smem_desc_kmajor_noswz(bl + ks * 256, 128, 2048);
          mma_f16_ts(d, fh + ks * 8, dh, idesc, ks > 0 ? 1u : 0u);
          mma_f16_ts(d, fh + ks * 8, dl, idesc, 1u);
          mma_f16_ts(d, fl + ks * 8, dh, idesc, 1u);
        }
        tc_commit(bop_empty + sb);
        tc_commit(d_full + db);
      }
    }
    __syncwarp();
  } else if (warp <= 9) {
    // ---------------- builders: thread (a, slots 2 s0 and 2 s0 + 1) -> T(a, c), c < R, as B-operand rows
    const int bt = threadIdx.x - 64;
    const int a = bt & 63, s0 = bt >> 6;  // warp-uniform slot pair
    float2 tw[R];
#pragma unroll
    for (int c = 1; c < R; ++c) tw[c] = __ldg(P.tw + a * 8 + c);
    auto rv = [](int i) {
      int r = 0;
#pragma unroll
      for (int bb = 0; bb < LOGR; ++bb) r |= ((i >> bb) & 1) << (LOGR - 1 - bb);
      return r;
    };
    const int swa = (a >> 1) & 3;  // the row swizzle term of rows a + 64 b (independent of b)
    for (int k = 0; k < nit; ++k) {
      const int st = k % S2T_NR, sb = k % S2T_NB;
      mbar_wait(rows_full + st, (k / S2T_NR) & 1);
      const float zsc = meta[st].zsc;
      const int bi = meta[st].bi;
      const bool half = P.B.ng[bi] == 1 && 4 * R >= 16;  // N = 4 R block: slots 4-7 are not read
      uint32_t info[2];
      info[0] = P.sl.info[bi][2 * s0];
      info[1] = P.sl.info[bi][2 * s0 + 1];
      const float2* rows = reinterpret_cast<const float2*>(rows_base + st * S2T_ROWS_BYTES);
      float2 x[2][R];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int kind = info[u] & 3, e1 = (info[u] >> 4) & 15, e2 = (info[u] >> 8) & 15, el = (int)(info[u] >> 16);
        if (kind == 1) {
          // complex index of (row q0 + 64 b mod n, column e1): ((q0 + 64 b) * 8 + swizzled column) mod 8 n
          const int q0 = (a - el) & (n - 1);
          const int base = q0 * 8 + ((((e1 >> 1) ^ (q0 >> 1)) & 3) << 1) + (e1 & 1);
#pragma unroll
          for (int b = 0; b < R; ++b) x[u][b] = rows[(base + 512 * b) & (8 * n - 1)];
        } else if (kind == 2) {
          const int c1 = a * 8 + ((((e1 >> 1) ^ swa) & 3) << 1) + (e1 & 1);
          const int c2 = a * 8 + ((((e2 >> 1) ^ swa) & 3) << 1) + (e2 & 1);
#pragma unroll
          for (int b = 0; b < R; ++b) {
            const float2 r1 = e1 < 15 ? rows[c1 + 512 * b] : make_float2(0.f, 0.f);
            const float2 r2 = e2 < 15 ? rows[c2 + 512 * b] : make_float2(0.f, 0.f);
            x[u][b] = make_float2(r1.x - r2.y, r1.y + r2.x);  // x_1 + i x_2
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(rows_empty + st);
      // the pair's Zhat' -> Z scale folded into the twiddles
      float2 tz[R];
      tz[0] = make_float2(zsc, zsc);
#pragma unroll
      for (int c = 1; c < R; ++c) tz[c] = mul2(make_float2(zsc, zsc), tw[c]);
      mbar_wait(bop_empty + sb, ((k / S2T_NB) & 1) ^ 1);
      uint8_t* bop = bop_base + sb * S2T_BOP_BYTES;
      if (!(half && s0 >= 2)) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          // MN-major core (n / 8, k / 8), row k % 8, element n % 8; N index = slot R + c, K = a (Re), 64 + a (Im)
          const int nn = (2 * s0 + u) * R;
          const uint32_t off = (uint32_t)(nn >> 3) * 2048u + (uint32_t)a * 16u + (uint32_t)(nn & 7) * 2u;
          uint32_t hr[H], lr[H], hi_[H], li_[H];
          if ((info[u] & 3) == 0 || (P.dbg & 1)) {  // no term: a zero column block (the word stays zero)
#pragma unroll
            for (int j = 0; j < H; ++j) hr[j] = lr[j] = hi_[j] = li_[j] = 0u;
          } else {
            dft_regs<R>(x[u]);  // natural order in x[rv(c)]
            float2 T[R];
            T[0] = mul2(tz[0], x[u][rv(0)]);
#pragma unroll
            for (int c = 1; c < R; ++c) T[c] = cmulf(x[u][rv(c)], tz[c]);
#pragma unroll
            for (int j = 0; j < H; ++j) {
              split2_f16(T[2 * j].x, T[2 * j + 1].x, hr[j], lr[j]);
              split2_f16(T[2 * j].y, T[2 * j + 1].y, hi_[j], li_[j]);
            }
          }
          sts_bytes<R>(bop + off, hr);
          sts_bytes<R>(bop + off + 1024u, hi_);
          sts_bytes<R>(bop + S2T_BOP_PART + off, lr);
          sts_bytes<R>(bop + S2T_BOP_PART + off + 1024u, li_);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(bop_full + sb);
    }
  } else {
    // ---------------- epilogue: lane quarter q, columns c in [H h, H h + H) of every slot
    const int ew = warp - 10, q = warp & 3, h = ew >> 2;
    const int ri = lane & 1;  // 0: the Re row of this d (writes hi words), 1: the Im row (lo words)
    const int dd = q * 16 + (lane >> 1);
    // word (c) = (Re, Im) halves: Re lane keeps its hi halves and receives the Im lane's hi halves; the Im
    // lane keeps its lo halves and receives the Re lane's lo halves
    const uint32_t sel0 = ri ? 0x1054u : 0x5410u, sel1 = ri ? 0x3276u : 0x7632u;
    const bool issuer = (warp == 10 && lane == 0);
    int bi = i_beg % nb, pr = i_beg / nb;
    for (int k = 0; k < nit; ++k) {
      const int db = k & 1;
      mbar_wait(d_full + db, (k >> 1) & 1);
      tc_fence_after();
      uint32_t v[8][H];
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)db * 64u + (uint32_t)(H * h);
      const int ng = P.B.ng[bi];
#pragma unroll
      for (int s = 0; s < 4; ++s) tmem_ld_x<H>(base + (uint32_t)(R * s), v[s]);
      if (ng > 1) {
#pragma unroll
        for (int s = 4; s < 8; ++s) tmem_ld_x<H>(base + (uint32_t)(R * s), v[s]);
      }
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d_empty + db);
      uint32_t w[8][H];
#pragma unroll
      for (int s = 0; s < 8; ++s) {
#pragma unroll
        for (int j = 0; j < H; j += 2) {
          uint32_t hh, ll;
          // values c and c + 1 packed in one f16x2 word (H = 1: one value, the high half unused)
          const float v1 = H > 1 ? __uint_as_float(v[s][(j + 1) % H]) : 0.f;
          split2_f16(__uint_as_float(v[s][j]), v1, hh, ll);
          const uint32_t kk = ri ? ll : hh;
          const uint32_t rr = __shfl_xor_sync(0xffffffffu, ri ? hh : ll, 1);
          w[s][j] = prmt(kk, rr, sel0);
          if constexpr (H > 1) w[s][j + 1] = prmt(kk, rr, sel1);
        }
      }
      if (P.sl.needmask[bi]) {
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint32_t m = P.sl.mask[bi][s];
#pragma unroll
          for (int ci = 0; ci < H; ++ci) w[s][ci] &= m;
        }
      }
      // the staging buffer of item k - NO must have been read by its TMA store
      if (issuer) bulk_wait_group_read<S2T_NO - 1>();
      named_bar(1, 256);
      uint8_t* stg = out_base + (k % S2T_NO) * S2T_OUT_BYTES;
#pragma unroll
      for (int grp = 0; grp < 2; ++grp) {
        if (grp >= ng) break;
#pragma unroll
        for (int ci = 0; ci < H; ++ci) {
          // row r = R d + c of the pair's n rows: r-tile r / 128, row group (r / 8) % 16, row r % 8; staging
          // [T][part][row group][128 B] with the 16-byte chunk index XOR (row group & 7) (TMA 128B swizzle)
          const int r = R * dd + H * h + ci, rg = (r >> 3) & 15;
          *reinterpret_cast<uint4*>(stg + grp * 16384 + ((((r >> 7) * 2 + ri) * 16 + rg) << 7) +
                                    (((r & 7) ^ (rg & 7)) << 4)) =
              make_uint4(w[4 * grp][ci], w[4 * grp + 1][ci], w[4 * grp + 2][ci], w[4 * grp + 3][ci]);
        }
      }
      fence_proxy_async_smem();
      named_bar(1, 256);
      if (issuer && !(P.dbg & 2)) {
        for (int grp = 0; grp < ng; ++grp)
          tma_store_5d(&omap, out_base + (k % S2T_NO) * S2T_OUT_BYTES + grp * 16384, 0, P.B.g0[bi] + grp, 0, 0,
                       pr * NRT);
        bulk_commit_group();
      }
      if (++bi == nb) {
        bi = 0;
        ++pr;
      }
    }
    if (issuer) bulk_wait_group<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

static int launch_step2_tc(const TcPlan& tc, const float2* Zhat, uint8_t* Zop, int npair, const PairBlock& pb,
                           const DevPlan& P, cudaStream_t s) {
  S2TParams prm;
  std::memset(&prm, 0, sizeof prm);
  prm.Zop = Zop;
  prm.npair = npair;
  prm.NWG = P.K3p / 8;
  prm.K3p = P.K3p;
  prm.pb = pb;
  prm.ast = tc.d_ast;
  prm.bst = tc.d_bst;
  prm.gmax = tc.gmax;
  prm.F = tc.d_s2F;
  prm.tw = tc.d_s2w;
  {
    const char* dg = std::getenv("FTK_S2TC_DBG");  // (timing experiments: 1 skips the builders' arithmetic, 2 the stores)
    prm.dbg = dg ? std::atoi(dg) : 0;
  }
  std::memcpy(&prm.B, &tc.s2_blocks, sizeof prm.B);
  std::memcpy(&prm.sl, &tc.s2t, sizeof prm.sl);
  alignas(64) CUtensorMap zmap;
  std::memset(&zmap, 0, sizeof zmap);
  if (make_zmap(&zmap, Zhat, npair, P) != FTK_OK) return FTK_ECUDA;
  const int NRT = P.n_psi / 128;
  // Step-3 operand as a 5-D tensor of 32-bit words: (word in a 128-byte core row group, word group, row group
  // of the r-tile, part, pair x r-tile); one (NRT x 4 KB) box per (item, word group), 128-byte swizzle
  alignas(64) CUtensorMap omap;
  std::memset(&omap, 0, sizeof omap);
  {
    PFN_encodeTiled enc = get_encode_tiled();
    if (!enc) return FTK_ECUDA;
    const cuuint64_t NWG = (cuuint64_t)(P.K3p / 8);
    const cuuint64_t dims[5] = {32, NWG, 16, 2, (cuuint64_t)npair * NRT};
    const cuuint64_t strides[4] = {128, NWG * 128, NWG * 2048, NWG * 4096};
    const cuuint32_t box[5] = {32, 1, 16, 2, (cuuint32_t)NRT};
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    if (enc(&omap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, Zop, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return FTK_ECUDA;
  }
  const int items = tc.s2_blocks.nb * npair;
  const int grid = items < tc.num_sms ? items : tc.num_sms;
  switch (P.n_psi) {
    case 128: k_step2_tc<2><<<grid, S2T_THREADS, S2T_SMEM, s>>>(prm, zmap, omap); break;
    case 256: k_step2_tc<4><<<grid, S2T_THREADS, S2T_SMEM, s>>>(prm, zmap, omap); break;
    default: k_step2_tc<8><<<grid, S2T_THREADS, S2T_SMEM, s>>>(prm, zmap, omap); break;
  }
  return FTK_OK;
}

// Step 2 dispatch: the tensor-core kernel where the plan enabled it (n_gamma = n_psi = 512), else the CUDA-core FFT
static int launch_step2(const TcPlan& tc, const float2* Zhat, uint8_t* Zop, int npair, const PairBlock& pb,
                        const DevPlan& P, cudaStream_t s) {
  if (tc.s2tc) return launch_step2_tc(tc, Zhat, Zop, npair, pb, P, s);
  return launch_step2_fft(tc, Zhat, Zop, npair, pb, P, s);
}

// ---------------------------------------------------------------- single-MMA self-test
// D = A * B^T with A [128 x 32] (TS: from TMEM; SS: from SMEM), B [N=64 x 32] from SMEM, bf16 inputs.
__global__ void __launch_bounds__(128, 1) k_tc_selftest(const float* A, const float* B, float* D_ts, float* D_ss,
                                                       float* D_mn) {
  __shared__ __align__(1024) uint8_t sa[128 * 32 * 2];
  __shared__ __align__(1024) uint8_t sb[64 * 32 * 2];
  __shared__ __align__(1024) uint8_t sbm[64 * 32 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int K = 32;
  // canonical K-major no-swizzle: core (row/8, k/8) at (row/8)*SBO + (k/8)*128, SBO = (K/8)*128
  const uint32_t SBO = (K / 8) * 128;
  for (int idx = tid; idx < 128 * K; idx += 128) {
    const int m = idx / K, k = idx % K;
    __nv_bfloat16 v = __float2bfloat16_rn(A[idx]);
    *reinterpret_cast<__nv_bfloat16*>(sa + (m / 8) * SBO + (k / 8) * 128 + (m % 8) * 16 + (k % 8) * 2) = v;
  }
  for (int idx = tid; idx < 64 * K; idx += 128) {
    const int nn = idx / K, k = idx % K;
    __nv_bfloat16 v = __float2bfloat16_rn(B[idx]);
    *reinterpret_cast<__nv_bfloat16*>(sb + (nn / 8) * SBO + (k / 8) * 128 + (nn % 8) * 16 + (k % 8) * 2) = v;
    // MN-major canonical: core (n/8, k/8) at (n/8)*SBO + (k/8)*128, inside: row k%8 (16 B), element n%8
    *reinterpret_cast<__nv_bfloat16*>(sbm + (nn / 8) * SBO + (k / 8) * 128 + (k % 8) * 16 + (nn % 8) * 2) = v;
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  // A -> TMEM columns [0, 16): packed bf16 pairs (k even in the low half)
  {
    const uint32_t base = tm + ((uint32_t)(warp * 32) << 16);
    uint32_t r16[16];
    for (int j = 0; j < 16; ++j) {
      __nv_bfloat162 h = __floats2bfloat162_rn(A[tid * K + 2 * j], A[tid * K + 2 * j + 1]);
      r16[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    tmem_st16(base, r16);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, 64);
    for (int ks = 0; ks < 2; ++ks) {
      const uint64_t bd = smem_desc_kmajor_noswz(smem_u32(sb) + ks * 256, 128, SBO);
      const uint64_t ad = smem_desc_kmajor_noswz(smem_u32(sa) + ks * 256, 128, SBO);
      const uint64_t bm = smem_desc_kmajor_noswz(smem_u32(sbm) + ks * 256, 128, SBO);
      mma_f16_ts(tm + 64, tm + ks * 8, bd, idesc, ks > 0);
      mma_f16_ss(tm + 128, ad, bd, idesc, ks > 0);
      mma_f16_ts(tm + 192, tm + ks * 8, bm, idesc_bf16_f32_bmn(128, 64), ks > 0);
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const uint32_t base = tm + ((uint32_t)(warp * 32) << 16);
  for (int c0 = 0; c0 < 64; c0 += 16) {
    uint32_t r16[16];
    tmem_ld16(base + 64 + c0, r16);
    tmem_wait_ld();
    for (int e = 0; e < 16; ++e) D_ts[tid * 64 + c0 + e] = __uint_as_float(r16[e]);
    tmem_ld16(base + 128 + c0, r16);
    tmem_wait_ld();
    for (int e = 0; e < 16; ++e) D_ss[tid * 64 + c0 + e] = __uint_as_float(r16[e]);
    tmem_ld16(base + 192 + c0, r16);
    tmem_wait_ld();
    for (int e = 0; e < 16; ++e) D_mn[tid * 64 + c0 + e] = __uint_as_float(r16[e]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tm);
  }
}

static float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

int tc_selftest(double* err_ts, double* err_ss, std::string& msg) {
  const int M = 128, N = 64, K = 32;
  std::vector<float> A(M * K), B(N * K), Dts(M * N), Dss(M * N), Dmn(M * N);
  uint32_t s = 12345;
  auto rnd = [&]() {
    s = s * 1664525u + 1013904223u;
    return ((s >> 8) & 0xffff) / 32768.0f - 1.0f;
  };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  float *dA, *dB, *dT, *dS, *dM;
  if (cudaMalloc(&dA, A.size() * 4) || cudaMalloc(&dB, B.size() * 4) || cudaMalloc(&dT, Dts.size() * 4) ||
      cudaMalloc(&dS, Dss.size() * 4) || cudaMalloc(&dM, Dmn.size() * 4)) {
    msg = "selftest alloc";
    return FTK_ENOMEM;
  }
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  k_tc_selftest<<<1, 128>>>(dA, dB, dT, dS, dM);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    msg = std::string("selftest kernel: ") + cudaGetErrorString(e);
    return FTK_ECUDA;
  }
  cudaMemcpy(Dts.data(), dT, Dts.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(Dss.data(), dS, Dss.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(Dmn.data(), dM, Dmn.size() * 4, cudaMemcpyDeviceToHost);
  cudaFree(dM);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dT);
  cudaFree(dS);
  double mt = 0, ms = 0;
  for (int m = 0; m < M; ++m)
    for (int nn = 0; nn < N; ++nn) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)bf16r(A[m * K + k]) * (double)bf16r(B[nn * K + k]);
      mt = std::max(mt, std::fabs(ref - Dts[m * N + nn]));
      ms = std::max(ms, std::max(std::fabs(ref - Dss[m * N + nn]), std::fabs(ref - Dmn[m * N + nn])));
    }
  *err_ts = mt;
  *err_ss = ms;
  return FTK_OK;
}

// ---------------------------------------------------------------- engine plumbing
// Step-2 work blocks: 1 or 2 consecutive word groups (8 Step-3 columns each) holding <= 8 whole terms,
// each a contiguous range of the device term order.
int s2_block_table(const std::vector<int>& ell, const std::vector<int>& col, int K3p, S2BlockTable& t,
                   std::string& msg) {
  std::memset(&t, 0, sizeof t);
  const int ngroups = K3p / 8;
  std::vector<int> tg(ngroups, 0);
  for (int z = 0; z < (int)col.size(); ++z) {
    tg[col[z] / 8]++;
    if (ell[z] > 0 && (col[z] & 1)) {
      msg = "tensor-core engine: an ell > 0 term on an odd column";
      return FTK_EINVAL;
    }
  }
  int nb = 0;
  for (int g = 0; g < ngroups;) {
    const int ng = (g + 1 < ngroups && tg[g] + tg[g + 1] <= 8) ? 2 : 1;
    if (nb >= 16 || tg[g] > 8) {
      msg = "tensor-core engine: unsupported Step-2 block structure";
      return FTK_EINVAL;
    }
    int zs = -1, ze = -1;
    for (int z = 0; z < (int)col.size(); ++z)
      if (col[z] / 8 >= g && col[z] / 8 < g + ng) {
        if (zs < 0) zs = z;
        if (ze >= 0 && z != ze) {
          msg = "tensor-core engine: Step-2 block terms not contiguous";
          return FTK_EINVAL;
        }
        ze = z + 1;
      }
    if (zs < 0) zs = ze = 0;
    int used = 0, lone = 0;
    for (int z = zs; z < ze; ++z) {
      const int kl = col[z] - 8 * g;
      used |= 1 << (kl >> 1);
      if (ell[z] == 0) {
        bool nbr = false;
        for (int z2 = zs; z2 < ze; ++z2) nbr = nbr || (z2 != z && ell[z2] == 0 && col[z2] == (col[z] ^ 1));
        if (!nbr) lone |= 1 << (z - zs);
      }
    }
    t.zs[nb] = zs;
    t.ze[nb] = ze;
    t.g0[nb] = g;
    t.ng[nb] = ng;
    t.used[nb] = used;
    t.lone[nb] = lone;
    ++nb;
    g += ng;
  }
  t.nb = nb;
  return FTK_OK;
}

// Device term order for the tensor-core engine: the blocks of s2_block_table moved as units so that each
// lies in one aligned 8-term window [zs & ~1, (zs & ~1) + 8) of a Zhat' row (a 2-D TMA box must start on a
// 16-byte boundary), i.e. a block starting at an odd term index holds <= 7 terms.  Greedy in block order
// (Step 1 writes runs of consecutive terms: the closer to the column order, the fewer split runs), taking
// the first remaining block that fits the current parity; if that gets stuck, even-sized blocks first,
// then the odd ones (alternating parities, <= 7 terms each).  perm[new z] = old z.
int tc_term_order(const std::vector<int>& ell, const std::vector<int>& col, int K3p, std::vector<int>& perm,
                  std::string& msg) {
  S2BlockTable t;
  if (s2_block_table(ell, col, K3p, t, msg) != FTK_OK) return FTK_EINVAL;
  const int nb = t.nb;
  std::vector<int> order;
  std::vector<bool> done(nb, false);
  int S = 0;
  for (int k = 0; k < nb; ++k) {
    int pick = -1;
    for (int bi = 0; bi < nb && pick < 0; ++bi)
      if (!done[bi] && (!(S & 1) || t.ze[bi] - t.zs[bi] <= 7)) pick = bi;
    if (pick < 0) break;
    done[pick] = true;
    order.push_back(pick);
    S += t.ze[pick] - t.zs[pick];
  }
  if ((int)order.size() < nb) {
    order.clear();
    for (int pass = 0; pass < 2; ++pass)
      for (int bi = 0; bi < nb; ++bi)
        if (((t.ze[bi] - t.zs[bi]) & 1) == pass) order.push_back(bi);
  }
  perm.clear();
  for (int bi : order)
    for (int z = t.zs[bi]; z < t.ze[bi]; ++z) perm.push_back(z);
  if (perm.size() != col.size()) {
    msg = "tensor-core engine: Step-2 blocks do not cover the terms";
    return FTK_EINVAL;
  }
  return FTK_OK;
}

int tc_plan_init(TcPlan& tc, const PlanMath& pm, const std::vector<float>& g, const std::vector<int>& ell,
                 const std::vector<int>& col, const std::vector<float>& Y3, int K3p, int Ke, int n_gamma,
                 std::string& msg) {
  tc_plan_free(tc);
  // TMEM: two A slots (K3p columns each) + two D buffers of E and O (4 NCH columns) <= 512, NCH >= 16.
  // K3p <= 128 keeps NCH >= 64 (full-rate MMAs); wider contractions (CTF plans) run with narrower chunks.
  if (K3p % 16 != 0 || K3p > 224) {
    msg = "tensor-core engine: Step-3 width " + std::to_string(K3p) + " (K3 = 2 H_plus - H0 = " +
          std::to_string(pm.K3) + " plus block padding) exceeds 224 (use engine=1)";
    return FTK_EINVAL;
  }
  if (pm.n_psi % 64 != 0 || pm.n_psi > 1024) {
    msg = "tensor-core engine: n_psi must be a multiple of 64 and <= 1024";
    return FTK_EINVAL;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&tc.num_sms, cudaDevAttrMultiProcessorCount, dev);
  tc.K3p = K3p;
  tc.Ke = Ke;
  // representative shifts: delta_t paired with delta_t' = -delta_t (X(-delta) = E - O); the rest alone
  std::vector<int> rep, partner;
  {
    std::vector<char> taken(pm.N_t, 0);
    for (int t = 0; t < pm.N_t; ++t) {
      if (taken[t]) continue;
      taken[t] = 1;
      int mate = -1;
      const double x = pm.shifts[2 * t], y = pm.shifts[2 * t + 1];
      if (x != 0.0 || y != 0.0) {
        for (int u = t + 1; u < pm.N_t; ++u)
          if (!taken[u] && (pm.n_tau == 0 || u / pm.N_base == t / pm.N_base) &&  // same filter (CTF)
              std::fabs(pm.shifts[2 * u] + x) <= 1e-12 * (1.0 + std::fabs(x)) &&
              std::fabs(pm.shifts[2 * u + 1] + y) <= 1e-12 * (1.0 + std::fabs(y))) {
            mate = u;
            taken[u] = 1;
            break;
          }
      }
      rep.push_back(t);
      partner.push_back(mate);
    }
  }
  {  // columns: paired representatives first (fast epilogue groups), unpaired ones last
    std::vector<int> r2, p2;
    for (int pass = 0; pass < 2; ++pass)
      for (size_t i = 0; i < rep.size(); ++i)
        if ((partner[i] >= 0) == (pass == 0)) {
          r2.push_back(rep[i]);
          p2.push_back(partner[i]);
        }
    rep.swap(r2);
    partner.swap(p2);
  }
  tc.n_rep = (int)rep.size();
  tc.NRT = (n_gamma + 127) / 128;
  // Step-3 chunk width NCH (N of the MMA): TMEM holds two D buffers (E and O, 2 NCH columns each) and
  // two A slots (K3p columns each); a rep-group's Y image must fit in shared memory.
  const int nmax = std::min(256, ((512 - 2 * K3p) / 4) / 16 * 16);
  if (nmax < 16) {
    msg = "tensor-core engine: K3p too large for the Step-3 TMEM layout";
    return FTK_EINVAL;
  }
  const size_t smem_cap = 232448;  // 227 KB opt-in dynamic shared memory per block
  int rg = 0;
  for (int G = 1;; ++G) {
    if (G > TcPlan::MAXG) {
      msg = "tensor-core engine: shift list too long for the Step-3 rep-groups";
      return FTK_EINVAL;
    }
    rg = (tc.n_rep + G - 1) / G;
    const int nch = (rg + nmax - 1) / nmax;
    const int NCH = ((rg + nch - 1) / nch + 15) / 16 * 16;
    if (s3_smem_bytes(nch * NCH, K3p, 1) <= smem_cap) {
      tc.G = G;
      tc.NCH = NCH;
      for (int g = 0; g < G; ++g) tc.g_nch[g] = nch;
      // staging ring depth: as many r-tile images as fit (1..4)
      tc.NS = 1;
      while (tc.NS < 4 && s3_smem_bytes(nch * NCH, K3p, tc.NS + 1) <= smem_cap) ++tc.NS;
      break;
    }
  }
  const int ncol_g = tc.g_nch[0] * tc.NCH;
  tc.ncol = tc.G * ncol_g;
  std::vector<int> colrep(tc.ncol, -1), colpart(tc.ncol, -1);
  std::vector<uint8_t> colfast(tc.ncol / 8, 0);
  const size_t ygroup = (size_t)4 * ncol_g * K3p;
  std::vector<uint16_t> yimg(ygroup / 2 * tc.G, 0);
  {  // fp16x3 scale constants (file header)
    float ym = 0.f;
    for (float y : Y3) ym = std::max(ym, std::fabs(y));
    tc.eY = f16_scale_exp(ym);
    float gm = 0.f;
    for (float x : g) gm = std::max(gm, std::fabs(x));
    tc.gmax = gm;
  }
  for (int g = 0; g < tc.G; ++g) {
    tc.g_col0[g] = g * ncol_g;
    tc.g_yoff[g] = (long long)(g * ygroup);
    for (int c = 0; c < ncol_g; ++c) {
      const int rr = g * rg + c;
      if (c >= rg || rr >= tc.n_rep) continue;
      colrep[g * ncol_g + c] = rep[rr];
      colpart[g * ncol_g + c] = partner[rr];
      const int t = rep[rr];
      for (int k = 0; k < K3p; ++k) {
        const float x = std::ldexp(Y3[(size_t)t * K3p + k], tc.eY);  // fp16x3: scaled, split in fp16
        const __half hi = __float2half_rn(x);
        const __half lo = __float2half_rn(x - __half2float(hi));
        const size_t off = (size_t)(c / 8) * (K3p / 8) * 64 + (size_t)(k / 8) * 64 + (c % 8) * 8 + (k % 8);
        std::memcpy(&yimg[g * ygroup / 2 + off], &hi, 2);
        std::memcpy(&yimg[g * ygroup / 2 + (size_t)ncol_g * K3p + off], &lo, 2);
      }
    }
  }
  for (int c8 = 0; c8 < tc.ncol / 8; ++c8) {
    bool f = true;
    for (int k = 0; k < 8; ++k) f = f && colrep[c8 * 8 + k] >= 0 && colpart[c8 * 8 + k] >= 0;
    colfast[c8] = f ? 1 : 0;
  }
  if (cudaMalloc(&tc.d_colrep, tc.ncol * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&tc.d_colpart, tc.ncol * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&tc.d_colfast, colfast.size() + 16) != cudaSuccess ||
      cudaMalloc(&tc.d_Ysm, yimg.size() * 2) != cudaSuccess) {
    msg = "tensor-core engine: allocation failed";
    return FTK_ENOMEM;
  }
  cudaMemcpy(tc.d_colrep, colrep.data(), tc.ncol * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemcpy(tc.d_colpart, colpart.data(), tc.ncol * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemcpy(tc.d_colfast, colfast.data(), colfast.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(tc.d_Ysm, yimg.data(), yimg.size() * 2, cudaMemcpyHostToDevice);
  tc.s3_smem = s3_smem_bytes(ncol_g, K3p, tc.NS);
  {  // fused Steps 2 + 3 (ftk_s23.cu): opt-in (FTK_S23=1).  Measured slower than the separate k_step2_fft +
     // k_step3_tc at c5 ("Fused Step 2+3"), so the default stays with the separate kernels
    const char* e23 = std::getenv("FTK_S23");
    const int st = tc_s23_init(tc, pm.n_psi, n_gamma, rep, partner, Y3, K3p, e23 && e23[0] == '1', msg);
    if (st != FTK_OK) return st;
  }
  FTK_SMEM_OPTIN((k_step3_tc<0>));
  FTK_SMEM_OPTIN((k_step3_tc<1>));
  if (pm.n_k % 16 != 0 || pm.n_k > 128) {
    msg = "tensor-core engine: n_k must be a multiple of 16 and <= 128";
    return FTK_EINVAL;
  }
  tc.KCH = (2 * pm.n_k) % 64 == 0 ? 64 : 32;
  tc.NKCH = 2 * pm.n_k / tc.KCH;
  FTK_SMEM_OPTIN((k_step1_tc<0>));
  FTK_SMEM_OPTIN((k_step1_tc<4>));
  FTK_SMEM_OPTIN((k_step1_cg2<0>));
  FTK_SMEM_OPTIN((k_step1_cg2<4>));
  {
    const char* e1 = std::getenv("FTK_S1CG2");  // (opt-in) the CTA-pair Step 1
    tc.s1cg2 = (e1 && std::atoi(e1) != 0) ? 1 : 0;
  }
  // Step-2 blocks (s2_block_table); the device term order (tc_term_order, applied in ftk_capi.cu) puts
  // every block's terms in one aligned 8-term window of a Zhat' row (one TMA box)
  {
    if (s2_block_table(ell, col, K3p, tc.s2_blocks, msg) != FTK_OK) return FTK_EINVAL;
    for (int bi = 0; bi < tc.s2_blocks.nb; ++bi)
      if ((tc.s2_blocks.zs[bi] & 1) + tc.s2_blocks.ze[bi] - tc.s2_blocks.zs[bi] > 8) {
        msg = "tensor-core engine: a Step-2 block does not fit its 8-term window (term order)";
        return FTK_EINVAL;
      }
    {  // Step-2 twiddle tables: [c][a] w_n^{a c} and [d'][a] w_32^{(a % L) d'}, E = n / 32, L = 32 / E
      const int n = n_gamma, E = n / 32, L = 32 / E;
      std::vector<float2> tw((size_t)2 * E * 32);
      for (int c = 0; c < E; ++c)
        for (int a = 0; a < 32; ++a) {
          const double ph1 = -2.0 * M_PI * (double)((a * c) % n) / n;
          const double ph2 = -2.0 * M_PI * (double)(((a % L) * c) % 32) / 32.0;
          tw[(size_t)c * 32 + a] = make_float2((float)std::cos(ph1), (float)std::sin(ph1));
          tw[(size_t)E * 32 + c * 32 + a] = make_float2((float)std::cos(ph2), (float)std::sin(ph2));
        }
      if (cudaMalloc(&tc.d_s2tw, tw.size() * sizeof(float2)) != cudaSuccess) {
        msg = "tensor-core engine: allocation failed";
        return FTK_ENOMEM;
      }
      cudaMemcpy(tc.d_s2tw, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice);
      float2 w32[32];
      for (int k = 0; k < 32; ++k) {
        const double ph = -2.0 * M_PI * k / 32.0;
        w32[k] = make_float2((float)std::cos(ph), (float)std::sin(ph));
      }
      cudaMemcpyToSymbol(c_w32, w32, sizeof w32);  // (per device: plan creation runs on the plan's device)
    }
    const int sm2 = (int)step2_smem(pm.n_psi, n_gamma);
    // k_step2_tc tables (n_gamma = n_psi = 64 R, R = 2, 4, 8): F64 real form, radix-R twiddles, per-block word slots
    tc.s2tc = 0;
    if ((pm.n_psi == 128 || pm.n_psi == 256 || pm.n_psi == 512) && n_gamma == pm.n_psi) {
      const char* e2 = std::getenv("FTK_S2TC");
      // default: on at n = 512 (c5: Step 2 -23 %), off below (at n = 256 / 128 the N = 32 / 16 MMAs leave it slower
      // than k_step2_fft: c3 Step 2 41.7 vs 37.4 ms); FTK_S2TC=1 forces it on, FTK_S2TC=0 off
      const int want = e2 ? std::atoi(e2) : (pm.n_psi == 512 ? 1 : 0);
      std::memset(&tc.s2t, 0, sizeof tc.s2t);
      for (int bi = 0; bi < tc.s2_blocks.nb; ++bi) {
        int kind[8] = {0}, e1[8], e2[8], el[8] = {0};
        for (int sl = 0; sl < 8; ++sl) e1[sl] = e2[sl] = 15;
        const int zs = tc.s2_blocks.zs[bi], g0 = tc.s2_blocks.g0[bi];
        for (int z = zs; z < tc.s2_blocks.ze[bi]; ++z) {
          const int kl = col[z] - 8 * g0, sl = kl >> 1, e = (zs & 1) + (z - zs);
          if (kl < 0 || kl >= 16 || e > 7) {
            msg = "tensor-core engine: Step-2 slot table";
            return FTK_EINVAL;
          }
          if (ell[z] > 0) {
            kind[sl] = 1;
            e1[sl] = e;
            el[sl] = ell[z];
          } else {
            kind[sl] = 2;
            if (kl & 1)
              e2[sl] = e;
            else
              e1[sl] = e;
          }
        }
        for (int sl = 0; sl < 8; ++sl) {
          tc.s2t.info[bi][sl] = (uint32_t)kind[sl] | ((uint32_t)e1[sl] << 4) | ((uint32_t)e2[sl] << 8) |
                                ((uint32_t)el[sl] << 16);
          const uint32_t m = kind[sl] == 2 ? ((e1[sl] < 15 ? 0x0000FFFFu : 0u) | (e2[sl] < 15 ? 0xFFFF0000u : 0u))
                                           : 0xFFFFFFFFu;
          tc.s2t.mask[bi][sl] = m;
          if (m != 0xFFFFFFFFu) tc.s2t.needmask[bi] = 1;
        }
      }
      std::vector<uint32_t> F((size_t)128 * 128);
      for (int m = 0; m < 128; ++m) {
        const int d = m >> 1, ro = m & 1;
        for (int kk = 0; kk < 128; kk += 2) {
          uint16_t hw[2], lw[2];
          for (int u = 0; u < 2; ++u) {
            const int k = kk + u, ri = k >> 6, a = k & 63;
            const double ph = 2.0 * M_PI * (double)((a * d) % 64) / 64.0;
            const double v = ro == 0 ? (ri == 0 ? std::cos(ph) : std::sin(ph)) : (ri == 0 ? -std::sin(ph) : std::cos(ph));
            const __half hh = __float2half_rn((float)v);
            const __half ll = __float2half_rn((float)(v - (double)__half2float(hh)));
            hw[u] = *reinterpret_cast<const uint16_t*>(&hh);
            lw[u] = *reinterpret_cast<const uint16_t*>(&ll);
          }
          F[(size_t)m * 128 + kk / 2] = (uint32_t)hw[0] | ((uint32_t)hw[1] << 16);
          F[(size_t)m * 128 + 64 + kk / 2] = (uint32_t)lw[0] | ((uint32_t)lw[1] << 16);
        }
      }
      std::vector<float2> w8((size_t)64 * 8);
      const int nn = pm.n_psi;
      for (int a = 0; a < 64; ++a)
        for (int c = 0; c < 8; ++c) {
          const double ph = -2.0 * M_PI * (double)((a * c) % nn) / (double)nn;
          w8[(size_t)a * 8 + c] = make_float2((float)std::cos(ph), (float)std::sin(ph));
        }
      if (cudaMalloc(&tc.d_s2F, F.size() * 4) != cudaSuccess || cudaMalloc(&tc.d_s2w, w8.size() * 8) != cudaSuccess) {
        msg = "tensor-core engine: allocation failed";
        return FTK_ENOMEM;
      }
      cudaMemcpy(tc.d_s2F, F.data(), F.size() * 4, cudaMemcpyHostToDevice);
      cudaMemcpy(tc.d_s2w, w8.data(), w8.size() * 8, cudaMemcpyHostToDevice);
      FTK_SMEM_OPTIN(k_step2_tc<2>);
      FTK_SMEM_OPTIN(k_step2_tc<4>);
      FTK_SMEM_OPTIN(k_step2_tc<8>);
      tc.s2tc = want != 0 ? 1 : 0;
    }
    FTK_SMEM_OPTIN((k_step2_fft<2>));
    FTK_SMEM_OPTIN((k_step2_fft<4>));
    FTK_SMEM_OPTIN((k_step2_fft<8>));
    FTK_SMEM_OPTIN((k_step2_fft<16>));
    FTK_SMEM_OPTIN((k_step2_fft<32>));
  }
  const char* sdbg = std::getenv("FTK_SYNC_DEBUG");
  tc.sync_debug = sdbg && sdbg[0] == '1';
  const char* pz = std::getenv("FTK_POISON");
  tc.poison = (pz && pz[0]) ? (int)(std::strtol(pz, nullptr, 0) & 0xFF) : -1;
  const char* os_ = std::getenv("FTK_ONLY_STEP");
  tc.only_step = os_ ? std::atoi(os_) : 0;
  if (tc.only_step < 0 || tc.only_step > 3) tc.only_step = 0;
  if (tc.sync_debug)
    for (int bi = 0; bi < tc.s2_blocks.nb; ++bi)
      fprintf(stderr, "s2 block %d: terms [%d,%d) groups %d+%d used %x lone %x\n", bi, tc.s2_blocks.zs[bi],
              tc.s2_blocks.ze[bi], tc.s2_blocks.g0[bi], tc.s2_blocks.ng[bi], tc.s2_blocks.used[bi],
              tc.s2_blocks.lone[bi]);
  tc.ready = true;
  return FTK_OK;
}

void tc_plan_free(TcPlan& tc) {
  tc_s23_free(tc);
  cudaFree(tc.d_s2tw);
  tc.d_s2tw = nullptr;
  cudaFree(tc.d_s2F);
  tc.d_s2F = nullptr;
  cudaFree(tc.d_s2w);
  tc.d_s2w = nullptr;
  cudaFree(tc.d_Ysm);
  cudaFree(tc.d_colrep);
  cudaFree(tc.d_colpart);
  cudaFree(tc.d_colfast);
  cudaFree(tc.d_Aop);
  cudaFree(tc.d_ast);
  cudaFree(tc.d_bst);
  tc.d_ast = tc.d_bst = nullptr;
  tc.ast_cap = tc.bst_cap = 0;
  tc.d_Ysm = nullptr;
  tc.d_colrep = tc.d_colpart = nullptr;
  tc.d_colfast = nullptr;
  tc.d_Aop = nullptr;
  tc.aop_bytes = 0;
  tc.ready = false;
}

// fp16x3 scaling: out[i] = (max over item i's FB coefficients of max(|Re|, |Im|), Frobenius norm of item i's
// coefficients, rounded up by 2^-20 so that it bounds the exact norm), one CTA of 256 threads per item
__global__ void k_item_stats(const float2* __restrict__ fb, int64_t per_item, float2* __restrict__ out) {
  const float2* x = fb + (size_t)blockIdx.x * per_item;
  float m = 0.f, q = 0.f;
  for (int64_t k = threadIdx.x; k < per_item; k += blockDim.x) {
    const float2 v = x[k];
    m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    q = fmaf(v.x, v.x, fmaf(v.y, v.y, q));
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    q += __shfl_xor_sync(0xffffffffu, q, o);
  }
  __shared__ float wm[8], wq[8];
  if ((threadIdx.x & 31) == 0) {
    wm[threadIdx.x >> 5] = m;
    wq[threadIdx.x >> 5] = q;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    m = wm[0];
    double qq = wq[0];
    for (int w = 1; w < 8; ++w) {
      m = fmaxf(m, wm[w]);
      qq += wq[w];
    }
    out[blockIdx.x] = make_float2(m, (float)(sqrt(qq) * (1.0 + 0x1p-20)));
  }
}

static int item_stats(const float2* fb, int64_t n, int64_t per_item, float2*& d_out, int64_t& cap, cudaStream_t s,
                      std::string& msg) {
  if (n > cap) {
    cudaFree(d_out);
    d_out = nullptr;
    cap = 0;
    if (cudaMalloc(&d_out, (size_t)n * sizeof(float2)) != cudaSuccess) {
      cudaGetLastError();
      msg = "tensor-core engine: scale table allocation failed";
      return FTK_ENOMEM;
    }
    cap = n;
  }
  if (n > 0) k_item_stats<<<(unsigned)n, 256, 0, s>>>(fb, per_item, d_out);
  return FTK_OK;
}

int tc_prepare_images(TcPlan& tc, const float2* fb, int64_t n_im, const DevPlan& P, cudaStream_t s, std::string& msg) {
  tc.NIT = (int)((n_im + 127) / 128);
  const size_t bytes = (size_t)P.n_psi * tc.NIT * 128 * (2 * P.n_k) * 4;
  if (bytes != tc.aop_bytes) {
    cudaFree(tc.d_Aop);
    tc.d_Aop = nullptr;
    tc.aop_bytes = 0;
    if (cudaMalloc(&tc.d_Aop, bytes) != cudaSuccess) {
      cudaGetLastError();
      msg = "tensor-core engine: image operand allocation failed";
      return FTK_ENOMEM;
    }
    tc.aop_bytes = bytes;
  }
  if (item_stats(fb, n_im, (int64_t)P.n_k * P.n_psi, tc.d_ast, tc.ast_cap, s, msg) != FTK_OK) return FTK_ENOMEM;
  const int64_t total = (int64_t)tc.NIT * 128 * P.n_psi * (2 * P.n_k / 8);
  k_prep_image_op<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(fb, tc.d_Aop, (int)n_im, tc.NIT, P.n_psi, P.n_k,
                                                                   tc.KCH, tc.NKCH, tc.d_ast);
  return cudaGetLastError() == cudaSuccess ? FTK_OK : FTK_ECUDA;
}
int tc_prepare_templates(TcPlan& tc, const float2* fb, int64_t n_tm, const DevPlan& P, cudaStream_t s,
                         std::string& msg) {
  if (item_stats(fb, n_tm, (int64_t)P.n_k * P.n_psi, tc.d_bst, tc.bst_cap, s, msg) != FTK_OK) return FTK_ENOMEM;
  return cudaGetLastError() == cudaSuccess ? FTK_OK : FTK_ECUDA;
}

size_t tc_bytes_per_pair(const TcPlan& tc, const DevPlan& P) {
  if (tc_s23_eligible(tc, P)) return (size_t)P.Hs * P.n_psi * sizeof(float2);  // fused: Zhat' only
  return (size_t)P.Hs * P.n_psi * sizeof(float2) + (size_t)tc.NRT * 128 * P.K3p * 4;
}

ftk_status_t tc_block_shape(const TcPlan&, const DevPlan&, int engine, int64_t NI, int64_t NJ, int64_t cap,
                            int64_t& ni, int64_t& nj, bool full_rows) {
  if (engine != 0) return FTK_OK;
  // image rows in multiples of 128 (Step-1 N tiles); as many as the workspace allows, up to 2048
  int64_t ni_t = std::min<int64_t>((NI + 127) / 128 * 128, 2048);
  if (full_rows) {
    // landscape output: every block spans all NJ templates, so the image rows shrink instead
    while (ni_t > 128 && ni_t * NJ > cap) ni_t -= 128;
    if (NI <= 128) ni_t = NI;
    ni = std::min<int64_t>(ni_t, NI);
    nj = ni_t * NJ <= cap ? NJ : std::max<int64_t>(1, cap / std::max<int64_t>(ni_t, 1));
    return (ni < NI && ni % 128 != 0) ? FTK_EINVAL : FTK_OK;
  }
  while (ni_t > 128 && ni_t * 1 > cap) ni_t -= 128;
  if (NI <= 128) ni_t = NI;
  ni = std::min<int64_t>(ni_t, NI);
  nj = std::max<int64_t>(1, std::min<int64_t>(NJ, cap / std::max<int64_t>(ni_t, 1)));
  if (ni < NI && ni % 128 != 0) return FTK_EINVAL;
  return FTK_OK;
}

void launch_step3_tc(const TcPlan& tc, const uint8_t* Zop, const PairBlock& pb, const DevPlan& P, int tm_off,
                     unsigned long long* img_keys, unsigned long long* pair_keys, int n_tm_local, float* land,
                     cudaStream_t s) {
  S3Params prm;
  std::memset(&prm, 0, sizeof prm);
  prm.Zop = Zop;
  prm.Ysm = tc.d_Ysm;
  prm.colrep = tc.d_colrep;
  prm.colpart = tc.d_colpart;
  prm.colfast = tc.d_colfast;
  prm.pb = pb;
  prm.n = P.n_gamma;
  prm.K3p = P.K3p;
  prm.Ke = P.Ke;
  prm.N_t = P.N_t;
  prm.NRT = tc.NRT;
  prm.NCH = tc.NCH;
  prm.G = tc.G;
  prm.NS = tc.NS;
  for (int g = 0; g < tc.G; ++g) {
    prm.g_col0[g] = tc.g_col0[g];
    prm.g_nch[g] = tc.g_nch[g];
    prm.g_yoff[g] = tc.g_yoff[g];
  }
  prm.tm_off = tm_off;
  prm.n_tm_local = n_tm_local;
  prm.img_keys = img_keys;
  prm.pair_keys = pair_keys;
  prm.land = land;
  int cpg = tc.num_sms / tc.G;
  if (cpg > pb.count) cpg = pb.count;
  if (cpg < 1) cpg = 1;
  static unsigned long long* d_trace = nullptr;  // diagnostics: FTK_S3_TRACE=1 prints CTA 0's counters
  const char* tenv = kDiag ? std::getenv("FTK_S3_TRACE") : nullptr;  // needs a -DFTK_DIAG=1 build
  if (tenv && tenv[0] == '1') {
    if (!d_trace) cudaMalloc(&d_trace, (16 + 4 * 64 + 64) * sizeof(unsigned long long));
    cudaMemsetAsync(d_trace, 0, (16 + 4 * 64 + 64) * sizeof(unsigned long long), s);
    prm.trace = d_trace;
  }
  {
    const char* e = std::getenv("FTK_S3_DBG");
    prm.dbg = e ? std::atoi(e) : 0;
  }
  prm.marg = tc.marg;
  prm.marg_part = tc.marg_part;
  prm.marg_np = tc.marg_np;
  prm.msc = tc.marg_scale;
  prm.ast = tc.d_ast;
  prm.bst = tc.d_bst;
  prm.gmax = tc.gmax;
  prm.eY = tc.eY;
  if (tc.marg)
    k_step3_tc<1><<<cpg * tc.G, S3_THREADS, tc.s3_smem, s>>>(prm);
  else
    k_step3_tc<0><<<cpg * tc.G, S3_THREADS, tc.s3_smem, s>>>(prm);
  if (prm.trace) {
    unsigned long long h[16 + 4 * 64 + 64];
    cudaMemcpyAsync(h, d_trace, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "s3trace pairs=%llu total=%llu mma_wait_stage=%llu mma_wait_dempty=%llu epi_wait_dfull=%llu "
            "epi_drain=%llu\n", h[3], h[0], h[1], h[2], h[4], h[5]);
    // per-chunk MMA issue timeline of CTA 0 (issue duration, interval to the next chunk's issue)
    for (int c = 0; c < 63; ++c) {
      const unsigned long long* t = h + 16 + 4 * c;
      if (!t[0] || !t[4]) break;
      fprintf(stderr, "s3chunk %d: issue %lld  next-issue %lld\n", c, (long long)(t[1] - t[0]), (long long)(t[4] - t[0]));
    }
    if (h[16] && h[16 + 4 * 62]) fprintf(stderr, "s3chunk avg issue interval chunks 0..62: %lld\n", (long long)(h[16 + 4 * 62] - h[16]) / 62);

  }
}

__global__ void k_marg_finalize(const float2* __restrict__ part, int G, long long np, float* __restrict__ out) {
  const long long ij = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (ij >= np) return;
  float m = -INFINITY, sm = 0.f;
  for (int g = 0; g < G; ++g) {
    const float2 v = part[(size_t)g * np + ij];
    lse2_merge(m, sm, v.x, v.y);
  }
  out[ij] = (m + log2f(sm)) * 0.6931471805599453f;
}

void tc_marg_finalize(const TcPlan& tc, cudaStream_t s) {
  if (!tc.marg_part || tc.marg_np <= 0 || tc.marg_sets <= 0) return;
  k_marg_finalize<<<(unsigned)((tc.marg_np + 255) / 256), 256, 0, s>>>(tc.marg_part, tc.marg_sets, tc.marg_np, tc.marg);
}

void launch_step1_tc(const TcPlan& tc, const float2* B, float2* Zhat, const PairBlock& pb, const DevPlan& P,
                     cudaStream_t s) {
  S1Params prm;
  prm.Aop = tc.d_Aop;
  prm.B = B;
  prm.g = P.g;
  prm.ell = P.ell;
  prm.Zhat = Zhat;
  prm.i0 = pb.i0;
  prm.ni = pb.ni;
  prm.j0 = pb.j0;
  prm.nj = pb.nj;
  prm.n = P.n_psi;
  prm.n_k = P.n_k;
  prm.Hp = P.H_plus;
  prm.Hs = P.Hs;
  prm.KCH = tc.KCH;
  prm.NKCH = tc.NKCH;
  prm.NIT = tc.NIT;
  prm.F = pb.nj * P.Hs;  // (template, slot) columns, pad slots included
  prm.NCT = (prm.F + 63) / 64;
  prm.ast = tc.d_ast;
  prm.bst = tc.d_bst;
  prm.gmax = tc.gmax;
  const int units = P.n_psi * prm.NCT;
  const int grid = units < tc.num_sms ? units : tc.num_sms;
  static unsigned long long* d_trace = nullptr;  // diagnostics: FTK_S1_TRACE=1 prints CTA 0's counters
  const char* tenv = kDiag ? std::getenv("FTK_S1_TRACE") : nullptr;  // needs a -DFTK_DIAG=1 build
  prm.trace = nullptr;
  if (tenv && tenv[0] == '1') {
    if (!d_trace) cudaMalloc(&d_trace, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(d_trace, 0, 16 * sizeof(unsigned long long), s);
    prm.trace = d_trace;
  }
  if (tc.s1cg2) {  // CTA pairs over unit pairs (opt-in FTK_S1CG2=1)
    const int upairs = P.n_psi * ((prm.NCT + 1) / 2);
    const int ncl = std::max(1, std::min(upairs, tc.num_sms / 2));
    if (tc.KCH == 64 && tc.NKCH == 4)
      k_step1_cg2<4><<<2 * ncl, S1_THREADS, s1_smem_bytes(tc), s>>>(prm);
    else
      k_step1_cg2<0><<<2 * ncl, S1_THREADS, s1_smem_bytes(tc), s>>>(prm);
  } else if (tc.KCH == 64 && tc.NKCH == 4)
    k_step1_tc<4><<<grid, S1_THREADS, s1_smem_bytes(tc), s>>>(prm);
  else
    k_step1_tc<0><<<grid, S1_THREADS, s1_smem_bytes(tc), s>>>(prm);
  if (prm.trace) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, d_trace, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "s1trace units=%llu total=%llu mma_wait_a=%llu mma_wait_acc=%llu mma_wait_stage=%llu\n", h[4],
            h[0], h[1], h[2], h[3]);
  }
}

// FTK_POISON (tests): one CTA per SM takes all of the SM's dynamic shared memory and all 512 TMEM columns and
// fills both with the byte pattern, so that a later kernel that reads shared memory or TMEM it did not write
// (a missing accumulate-reset, a stale stage, a race on a buffer hand-off) sees the pattern instead of zeros or a
// previous launch's values.  With 0x7B the pattern is a large finite value in fp32 (1.3e36) and fp16 (61280),
// so a stray read cannot hide inside a max as a NaN would; 0xFF gives NaNs.
__global__ void __launch_bounds__(128, 1) k_poison_onchip(uint32_t word, int smem_bytes) {
  extern __shared__ __align__(16) uint8_t praw[];
  __shared__ uint32_t taddr;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&taddr);
  uint4* p4 = reinterpret_cast<uint4*>(praw);
  for (int i = threadIdx.x; i < smem_bytes / 16; i += blockDim.x) p4[i] = make_uint4(word, word, word, word);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = word;
  const uint32_t base = taddr + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < 512; c += 16) tmem_st16(base + c, v);
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(taddr);
  }
}

void tc_poison(const TcPlan& tc, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (tc.poison < 0) return;
  const uint32_t b = (uint32_t)tc.poison & 0xFFu;
  if (ws && ws_bytes) cudaMemsetAsync(ws, (int)b, ws_bytes, s);
  FTK_SMEM_OPTIN(k_poison_onchip);
  int dev = 0, mx = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int smem = (mx - 1024) / 16 * 16;  // the static taddr word + reserve; one CTA per SM
  k_poison_onchip<<<tc.num_sms, 128, smem, s>>>(b * 0x01010101u, smem);
}

int tc_run_block(TcPlan& tc, const PairBlock& pb, const DevPlan& P, const float2* A, const float2* B, void* ws,
                 size_t ws_bytes, int tm_off, unsigned long long* img_keys, unsigned long long* pair_keys, int n_tm_local,
                 float* land, cudaStream_t s, prof_cb_t prof, void* plan, std::string& msg) {
  if (!tc.ready) {
    msg = "tensor-core engine not initialized";
    return FTK_ESTATE;
  }
  float2* Zhat = reinterpret_cast<float2*>(ws);
  uint8_t* Zop = reinterpret_cast<uint8_t*>(Zhat + (size_t)pb.count * P.Hs * P.n_psi);
  if (pb.li) {
    msg = "tensor-core engine: explicit pair lists go through tc_landscape_pairs";
    return FTK_EINVAL;
  }
  tc_poison(tc, ws, ws_bytes, s);
  // (experiment) the plan's first block runs all steps so the workspace holds real Zhat' / Zop; later blocks run
  // only FTK_ONLY_STEP's kernel on that data
  if (tc.only_step && tc.only_primed++ > 0) {
    if (prof) prof(plan, tc.only_step, 0, s);
    if (tc.only_step == 1) launch_step1_tc(tc, B, Zhat, pb, P, s);
    if (tc.only_step == 2) launch_step2(tc, Zhat, Zop, pb.count, pb, P, s);
    if (tc.only_step == 3) launch_step3_tc(tc, Zop, pb, P, tm_off, img_keys, pair_keys, n_tm_local, land, s);
    if (prof) prof(plan, tc.only_step, 1, s);
    return cudaGetLastError() == cudaSuccess ? FTK_OK : FTK_ECUDA;
  }
  {
    if (prof) prof(plan, 1, 0, s);
    launch_step1_tc(tc, B, Zhat, pb, P, s);
    if (prof) prof(plan, 1, 1, s);
    if (tc.sync_debug) {
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) {
        msg = std::string("Step 1: ") + cudaGetErrorString(e);
        return FTK_ECUDA;
      }
    }
    tc_poison(tc, nullptr, 0, s);
    if (tc_s23_eligible(tc, P)) {  // fused Steps 2 + 3: Zhat' -> keys
      if (prof) prof(plan, 3, 0, s);
      const int st = launch_step23(tc, Zhat, pb, P, tm_off, img_keys, pair_keys, n_tm_local, land, s);
      if (prof) prof(plan, 3, 1, s);
      if (st != FTK_OK) {
        msg = "fused Step 2+3: launch failed (tensor map or configuration)";
        return FTK_ECUDA;
      }
      if (tc.sync_debug) {
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
          msg = std::string("Steps 2+3: ") + cudaGetErrorString(e);
          return FTK_ECUDA;
        }
      }
      return FTK_OK;
    }
    if (prof) prof(plan, 2, 0, s);
    if (launch_step2(tc, Zhat, Zop, pb.count, pb, P, s) != FTK_OK) {
      msg = "Step 2: tensor map encoding failed";
      return FTK_ECUDA;
    }
    if (prof) prof(plan, 2, 1, s);
  }
  if (tc.sync_debug) {  // FTK_SYNC_DEBUG=1: attribute an asynchronous fault to its step
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      msg = std::string("Steps 1-2: ") + cudaGetErrorString(e);
      return FTK_ECUDA;
    }
  }
  tc_poison(tc, nullptr, 0, s);
  if (prof) prof(plan, 3, 0, s);
  if (tc_s3v2_eligible(tc, P)) {
    if (launch_step3_cg2(tc, Zop, pb, P, tm_off, img_keys, pair_keys, n_tm_local, land, s) != FTK_OK) {
      msg = "Step 3 (CTA pair): launch failed";
      return FTK_ECUDA;
    }
  } else {
    launch_step3_tc(tc, Zop, pb, P, tm_off, img_keys, pair_keys, n_tm_local, land, s);
  }
  if (prof) prof(plan, 3, 1, s);
  if (tc.sync_debug) {
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      msg = std::string("Step 3: ") + cudaGetErrorString(e);
      return FTK_ECUDA;
    }
  }
  return FTK_OK;
}

// ftk_landscape_pairs on the tensor-core engine: the production kernels on minimal blocks.  Pairs are
// grouped by (128-image tile, template); per group one k_step1_tc launch over the tile x 1 template (the
// Step-1 instance and block structure ftk_align runs), then per requested pair k_step2_fft (Form B) and
// k_step3_tc on that single pair with landscape output (the exact epilogue path).
int tc_landscape_pairs(TcPlan& tc, const DevPlan& P, const float2* B, const int32_t* h_img, const int32_t* h_tpl,
                       int n_pairs, int64_t n_im, int tm_off, int n_tm_local, void* ws, float* out, cudaStream_t s,
                       std::string& msg) {
  if (!tc.ready) {
    msg = "tensor-core engine not initialized";
    return FTK_ESTATE;
  }
  std::vector<int> order(n_pairs);
  for (int k = 0; k < n_pairs; ++k) order[k] = k;
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    const long long ka = (long long)(h_img[a] / 128) * n_tm_local + h_tpl[a];
    const long long kb = (long long)(h_img[b] / 128) * n_tm_local + h_tpl[b];
    return ka != kb ? ka < kb : a < b;
  });
  float2* Zhat = reinterpret_cast<float2*>(ws);
  uint8_t* Zop = reinterpret_cast<uint8_t*>(Zhat + (size_t)128 * P.Hs * P.n_psi);
  const size_t land_pp = (size_t)P.N_t * P.n_gamma;
  for (int a = 0; a < n_pairs;) {
    const int tile = h_img[order[a]] / 128, j = h_tpl[order[a]];
    int b = a;
    while (b < n_pairs && h_img[order[b]] / 128 == tile && h_tpl[order[b]] == j) ++b;
    PairBlock pb1;
    pb1.i0 = tile * 128;
    pb1.ni = (int)std::min<int64_t>(128, n_im - pb1.i0);
    pb1.j0 = j;
    pb1.nj = 1;
    pb1.li = pb1.lj = nullptr;
    pb1.count = pb1.ni;
    tc_poison(tc, ws, (size_t)128 * P.Hs * P.n_psi * sizeof(float2) + (size_t)tc_bytes_per_pair(tc, P), s);
    launch_step1_tc(tc, B, Zhat, pb1, P, s);
    for (int c = a; c < b; ++c) {
      const int k = order[c], i = h_img[k];
      const float2* zp = Zhat + (size_t)(i - pb1.i0) * P.n_psi * P.Hs;
      if (tc_s23_eligible(tc, P)) {  // the fused kernel on this one pair
        PairBlock pb3;
        pb3.i0 = i;
        pb3.ni = 1;
        pb3.j0 = j;
        pb3.nj = 1;
        pb3.li = pb3.lj = nullptr;
        pb3.count = 1;
        if (launch_step23(tc, zp, pb3, P, tm_off, nullptr, nullptr, n_tm_local, out + (size_t)k * land_pp, s) != FTK_OK) {
          msg = "fused Step 2+3: launch failed";
          return FTK_ECUDA;
        }
        continue;
      }
      PairBlock pb3;
      pb3.i0 = i;
      pb3.ni = 1;
      pb3.j0 = j;
      pb3.nj = 1;
      pb3.li = pb3.lj = nullptr;
      pb3.count = 1;
      tc_poison(tc, Zop, (size_t)tc_bytes_per_pair(tc, P) - (size_t)P.Hs * P.n_psi * sizeof(float2), s);
      if (launch_step2(tc, zp, Zop, 1, pb3, P, s) != FTK_OK) {
        msg = "Step 2: tensor map encoding failed";
        return FTK_ECUDA;
      }
      tc_poison(tc, nullptr, 0, s);
      if (tc_s3v2_eligible(tc, P)) {
        if (launch_step3_cg2(tc, Zop, pb3, P, tm_off, nullptr, nullptr, n_tm_local, out + (size_t)k * land_pp, s) !=
            FTK_OK) {
          msg = "Step 3 (CTA pair): launch failed";
          return FTK_ECUDA;
        }
      } else {
        launch_step3_tc(tc, Zop, pb3, P, tm_off, nullptr, nullptr, n_tm_local, out + (size_t)k * land_pp, s);
      }
    }
    a = b;
  }
  return cudaGetLastError() == cudaSuccess ? FTK_OK : FTK_ECUDA;
}

}  // namespace ftk
