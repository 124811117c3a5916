// Fused Steps 2 + 3 of the tensor-core engine (PAPER.md Eq. fbk3):
//   Z_zeta(gamma_r) = sum_q Zhat_zeta(q) e^{-i q gamma_r}          (Step 2, Form B: Zhat(q) = Zhat'(q - ell))
//   X(delta_t, gamma_r) = sum_k Z3[r][k] Y3[t][k]                   (Step 3, real form of reading R13)
// with the fused max / argmax (MODE 0) or log-sum-exp (MODE 1) epilogue, so that neither Z nor X ever
// reaches HBM: the kernel reads Step 1's Zhat' and writes per-image keys.
//
// CTA pair (cluster of 2, tcgen05 cta_group::2).  Both CTAs of a cluster work on the same pair; CTA h
// owns the rotations r = D i + c with c = 2 s + h (tile s < NT = D / 2, row i < F = n / D, n = n_psi =
// n_gamma).  Decimation in frequency over q = q1 + F j:
//   Z(D i + c) = sum_{q1 < F} w_F^{q1 i} y_c(q1),   y_c(q1) = w_n^{q1 c} sum_{j < D} w_D^{j c} Zhat(q1 + F j),
// one F-point FFT per (term, tile): each CTA transforms only its own rotations (no exchange), from the full
// input window of the term.  A "unit" is (pair, tile s); the cluster runs the units of its pair range in
// order, the two CTAs in lock step.  One tcgen05.mma M = 256 covers both CTAs' 128-row tiles (rows >= F
// unused), N = NCH representative shifts (B = Y3 chunk, its NCH/2 columns of each chunk resident in each
// CTA's shared memory: half of the Y image per SM), K = K3p in fp16x3 (hi*hi + hi*lo + lo*hi, scaled operands).
//
// Warp roles (20 warps):
//   0-7    FFT: two groups of 4 warps, one per input slot; each warp two terms of a Step-2 block (16 lanes
//          each): y_c from the input window, F-point FFT (V-point register DFTs around a transpose, one or
//          two shuffle stages), fp16 hi/lo split (scaled) into the staging area [part][word][row]
//   8      Y image load at start, then idle
//   9      merge: the 8 epilogue records -> packed-key atomicMax (or the MODE-1 partial)
//   10     TMA producer: per (unit, Step-2 block) the block's 8-term window of Zhat', n/2 rows per CTA,
//          multicast to both CTAs of the cluster (each CTA receives all n rows)
//   11-18  epilogue: per chunk the E / O accumulators (tcgen05.ld in 16-column batches, pipelined), E + |O|
//          max with the exact (shift, sign) resolved in-branch on a new maximum (carried over one image's
//          templates); after a unit's last chunk the staged A operand of unit u + 2 is copied into the
//          freed TMEM slot (tcgen05.st)
//   19     TMEM allocation (both CTAs); in the even CTA one elected lane issues all MMAs of the pair
// (the issue arbiter favours higher warp ids: the tensor-core critical path gets the highest)
// TMEM (per CTA, 512 columns): D buffers [0, 4 NCH) (E and O of buffer 0, then 1), A slots
// [4 NCH, 4 NCH + 2 K3p) (hi words then lo words, K3p / 2 each).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "ftk_tc.cuh"
#include "ftk_tc_dev.cuh"

namespace ftk {

#ifndef FTK_DIAG
#define FTK_DIAG 0
#endif
constexpr bool kDiag23 = FTK_DIAG != 0;  // wait-cycle counters of cluster 0 (FTK_S23_TRACE=1, -DFTK_DIAG=1 builds)
__device__ __forceinline__ long long clk23() {
  if constexpr (kDiag23) return clock64();
  return 0;
}
// TMA prefetch of a tile into L2 (no shared-memory destination)
__device__ __forceinline__ void tma_prefetch_2d(const void* tmap, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(tmap), "r"(x), "r"(y) : "memory");
}

constexpr int S23_WARPS = 20;
// warp roles, ordered by scheduler priority (the issue arbiter favours higher warp ids): FFT warps lowest,
// the epilogue and the MMA issuer (the tensor-core critical path) highest
// (warpgroups are homogeneous for setmaxnreg: [0, 8) FFT, [8, 12) control, [12, 20) epilogue)
constexpr int kWEpiFft = 8;   // warps [0, 8): FFT (two groups of 4, one per input slot)
constexpr int kWY = 8;        // Y image load, then idle
constexpr int kWMerge = 9;    // per-record merge + atomics
constexpr int kWTma = 10;     // TMA producer
constexpr int kWMma = 11;     // TMEM allocation + MMA issue (even CTA)
constexpr int kWEpi = 12;     // warps [12, 20): epilogue (lane quarter warp % 4, two warps per quarter)
// register budget: the CTA's pool is what it launched with (640 threads x 96); FFT warps drop to 72 and
// control warps to 56 so that the epilogue can take 128 (it drains a whole half chunk, 2 x 48 columns,
// in one TMEM round trip): 256 x 72 + 128 x 56 + 256 x 128 <= 640 x 96
constexpr int kRegFft = 72, kRegCtl = 56, kRegEpi = 128;
static_assert(256 * kRegFft + 128 * kRegCtl + 256 * kRegEpi <= 640 * 96, "register pool");
constexpr int S23_THREADS = S23_WARPS * 32;
constexpr int S23_NIN = 2;  // input window slots

struct S23Smem {
  uint64_t in_full[S23_NIN], in_empty[S23_NIN];
  uint64_t stg_full, stg_empty;
  uint64_t a_full[2];   // even CTA: both CTAs' epilogue warps (16)
  uint64_t d_full[2];   // each CTA: the pair's commit
  uint64_t d_empty[2];  // even CTA: both CTAs' epilogue warps (16)
  uint64_t red_full[2], red_empty[2];
  uint64_t y_bar;
  uint32_t tmem_base;
  float red_v[2][8], red_s[2][8];
  uint32_t red_f[2][8];
};
static_assert(sizeof(S23Smem) <= 1024, "S23Smem");

// FFT geometry: F = 16 V points per (term, tile), V values per lane, two terms per FFT warp (16 lanes each);
// staging row index pi(i) = i + V (i / V^2) (conflict-free FFT writes), row stride RS = 16 (mod 32) words
__host__ __device__ constexpr int s23_rs(int V) {
  if (V == 0) return 0;
  return ((16 * V + V * (16 / V - 1) + 15) / 32) * 32 + 16 >= 16 * V + V * (16 / V - 1)
             ? ((16 * V + V * (16 / V - 1) + 15) / 32) * 32 + 16
             : ((16 * V + V * (16 / V - 1) + 15) / 32) * 32 + 48;
}
// shared-memory layout (host and device)
struct S23Layout {
  uint32_t meta, ys, inb, stg, scr, total;
};
__host__ __device__ inline S23Layout s23_layout(int ncol, int nch, int NCH, int K3p, int n, int V) {
  S23Layout L;
  auto up = [](uint32_t x) { return (x + 1023u) & ~1023u; };
  L.meta = 1024;
  const uint32_t meta_bytes = (uint32_t)ncol * 8u + (uint32_t)ncol / 8u + 2u * (uint32_t)nch + 64u;
  L.ys = up(L.meta + meta_bytes);
  const uint32_t ybytes = 2u * (uint32_t)nch * (uint32_t)(NCH / 2) * (uint32_t)K3p * 2u;
  if (V == 0) {  // Step-3 only (operand tiles from k_step2_fft): two staging slots of one r-tile image (hi + lo)
    L.inb = L.stg = up(L.ys + ybytes);
    L.scr = L.total = up(L.stg + 2u * 2u * 128u * (uint32_t)K3p * 2u);
    return L;
  }
  L.inb = up(L.ys + ybytes);
  L.stg = up(L.inb + (uint32_t)S23_NIN * (uint32_t)n * 64u);
  L.scr = up(L.stg + 2u * (uint32_t)(K3p / 2) * (uint32_t)s23_rs(V) * 4u);
  // transpose scratch: 8 FFT warps x 2 terms x V rows x (16 + R) complex
  L.total = up(L.scr + 8u * 2u * (uint32_t)V * (uint32_t)(16 + 16 / V) * 8u);
  return L;
}

struct S23Params {
  const uint8_t* Ysm;  // per (group, CTA half): [part][chunk][NCH/2 rows][K3p] canonical K-major core matrices
  const int* colrep;   // [ncol_total] shift of the representative (+delta); -1 padding
  const int* colpart;  // [ncol_total] shift of -delta; -1 none
  const uint8_t* colfast;
  const int* ell;      // [H_plus] device term order
  const int* col;      // [H_plus] Step-3 column of the term
  const float2* twn;   // [n/2] e^{-2 pi i j / n}
  const float2* twA;   // [16][V] w_F^{a k1}, then [R][V] w_16^{a0 m} (four-step twiddles of the F-point FFT)
  S2BlockTable B;
  PairBlock pb;
  int n, F, D, NT;
  int K3p, Ke, N_t, NCH, G, nch;
  int g_col0[TcPlan::MAXG];
  long long g_yoff[TcPlan::MAXG];
  long long yhalf;  // bytes of one CTA half of a group's Y image
  int tm_off, n_tm_local;
  unsigned long long* img_keys;
  unsigned long long* pair_keys;
  float* land;
  float2* marg_part;  // MODE 1: [2 G][N_im][n_tm_local] base-2 (max, sum) partials
  long long marg_np;
  float msc;          // MODE 1: log2(e) / tau
  const float2* ast;  // fp16x3 scaling (ftk_tc.cu header): image / local template maxima, 
  const float2* bst;  // Y3 exponent
  float gmax;
  int eY;
  unsigned long long* trace;  // diagnostics (kDiag23): [cta of cluster 0][16] cycle counters
  const void* zdbg;           // diagnostics: base of the block's Zhat' (FTK_S23_DBG bit 2)
  int Hs;
  const uint8_t* Zop;         // ZS: k_step2_fft's r-tile images [pair][r-tile][part][128 x K3p fp16]
  int NRT;                    // ZS: r-tiles per pair
  int dbg;                    // diagnostics (kDiag23, FTK_S23_DBG): bit 0 skips the FFT arithmetic, bit 1 the
                              // epilogue arithmetic (timing experiments; results are wrong by design)
};

// Step-3 MMAs of one chunk over the CTA pair (one thread of the even CTA): 3 x KS fp16 products M256 x NCH x K16
template <int KS>
__device__ __forceinline__ void s23_chunk_mmas(uint32_t dE, uint32_t dO, uint32_t a_hi0, uint32_t halfk, uint64_t bh0,
                                               uint64_t bl0, uint32_t idesc, int ke, int ksteps) {
  if constexpr (KS > 0) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const uint32_t d = ks >= ke ? dO : dE;
      const uint32_t acc0 = (ks == 0 || ks == ke) ? 0u : 1u;
      const uint32_t a_hi = a_hi0 + (uint32_t)(ks * 8), a_lo = a_hi + halfk;
      mma_f16_ts_cg2(d, a_hi, bh0 + (uint64_t)(ks * 16), idesc, acc0);
      mma_f16_ts_cg2(d, a_hi, bl0 + (uint64_t)(ks * 16), idesc, 1u);
      mma_f16_ts_cg2(d, a_lo, bh0 + (uint64_t)(ks * 16), idesc, 1u);
    }
  } else {
    for (int ks = 0; ks < ksteps; ++ks) {
      const uint32_t d = ks >= ke ? dO : dE;
      const uint32_t acc0 = (ks == 0 || ks == ke) ? 0u : 1u;
      const uint32_t a_hi = a_hi0 + (uint32_t)(ks * 8), a_lo = a_hi + halfk;
      mma_f16_ts_cg2(d, a_hi, bh0 + (uint64_t)(ks * 16), idesc, acc0);
      mma_f16_ts_cg2(d, a_hi, bl0 + (uint64_t)(ks * 16), idesc, 1u);
      mma_f16_ts_cg2(d, a_lo, bh0 + (uint64_t)(ks * 16), idesc, 1u);
    }
  }
}

struct S23MmaArgs {
  uint32_t tmem, acol0, ybase, ypart, chunk_bytes, SBO;
  int NCH, nch, K3p, ke, U;
  S23Smem* S;
  unsigned long long* tr;  // diagnostics: [0] total, [1] a_full waits, [2] d_empty waits
};

template <int KS>
__device__ __forceinline__ void s23_mma_loop(const S23MmaArgs& a) {
  S23Smem& S = *a.S;
  const uint32_t idesc = idesc_f16_f32(256, a.NCH);
  const uint32_t halfk = (uint32_t)a.K3p / 2u;
  uint32_t g_d = 0;
  long long w_a = 0, w_d = 0;
  const long long t_0 = clk23();
  for (int u = 0; u < a.U; ++u) {
    const int slot = u & 1;
    long long t1 = clk23();
    mbar_wait_cluster(&S.a_full[slot], (uint32_t)(u >> 1) & 1u);
    w_a += clk23() - t1;
    tc_fence_after();
    const uint32_t a_hi0 = a.tmem + a.acol0 + (uint32_t)(slot * a.K3p);
    for (int c = 0; c < a.nch; ++c, ++g_d) {
      const int db = g_d & 1;
      t1 = clk23();
      mbar_wait_cluster(&S.d_empty[db], ((g_d >> 1) & 1u) ^ 1u);
      w_d += clk23() - t1;
      tc_fence_after();
      const uint32_t dE = a.tmem + (uint32_t)(db * 2 * a.NCH), dO = dE + (uint32_t)a.NCH;
      const uint32_t bch = a.ybase + (uint32_t)c * a.chunk_bytes;
      const uint64_t bh0 = smem_desc_kmajor_noswz(bch, 128, a.SBO);
      const uint64_t bl0 = smem_desc_kmajor_noswz(bch + a.ypart, 128, a.SBO);
      s23_chunk_mmas<KS>(dE, dO, a_hi0, halfk, bh0, bl0, idesc, a.ke, a.K3p / 16);
      tc_commit_cg2(&S.d_full[db]);
    }
  }
  if (kDiag23 && a.tr) {
    a.tr[0] = clk23() - t_0;
    a.tr[1] = w_a;
    a.tr[2] = w_d;
  }
}

// Does the epilogue emit a record after pair p?  Per pair for MODE 1, for per-pair maxima and for explicit
// pair lists; otherwise (MODE 0, per-image keys only) once per run of consecutive pairs with the same image.
__device__ __forceinline__ bool s23_flush(const S23Params& P, int MODE, int p, int p_end, int i) {
  if (MODE != 0 || P.pair_keys || P.pb.li || p + 1 >= p_end) return true;
  int i2, j2;
  pair_of(P.pb, p + 1, i2, j2);
  return i2 != i;
}

template <int MODE, int V, int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(S23_THREADS, 1)
    k_step23(const __grid_constant__ S23Params P, const __grid_constant__ CUtensorMap zmap) {
  extern __shared__ __align__(1024) uint8_t sraw[];
  S23Smem& S = *reinterpret_cast<S23Smem*>(sraw);
  // V = 0: Step 3 only -- the A operand arrives as k_step2_fft's r-tile images (canonical K-major core matrices)
  // and CTA h of the pair takes r-tile T = 2 s + h of unit s; V > 0: the fused FFT (F-point per tile)
  constexpr bool ZS = V == 0;
  constexpr int F = ZS ? 128 : 16 * V;  // rows per tile
  constexpr int VV = ZS ? 8 : V;
  constexpr int R = 16 / VV;            // lanes per column group after the transpose
  constexpr int LR = (R == 4) ? 2 : 1;
  constexpr int RS = s23_rs(V);         // staging row stride (words)
  constexpr int SR = 16 + R;            // transpose scratch row (complex)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t h = cluster_rank();
  const int n = ZS ? P.n : F * D, K3p = P.K3p, NCH = P.NCH, nch = P.nch;
  const int NT = ZS ? P.NT : D / 2;
  const uint32_t rt_part = 128u * (uint32_t)K3p * 2u;  // ZS: bytes of one part of an r-tile image
  const int G = P.G;
  const int cl = blockIdx.x >> 1;    // cluster index
  const int ncl = gridDim.x >> 1;
  const int grp = cl % G;
  const int ncol = nch * NCH, col0 = P.g_col0[grp];
  const S23Layout LY = s23_layout(ncol, nch, NCH, K3p, n, V);
  int* s_rep = reinterpret_cast<int*>(sraw + LY.meta);
  int* s_part = s_rep + ncol;
  uint8_t* s_fast = reinterpret_cast<uint8_t*>(s_part + ncol);
  uint8_t* s_fastc = s_fast + ncol / 8;
  uint8_t* ys = sraw + LY.ys;
  uint8_t* inb = sraw + LY.inb;
  uint32_t* stg = reinterpret_cast<uint32_t*>(sraw + LY.stg);
  const int KW = K3p / 2;  // words per part of a row
  // pair range of this cluster (clusters of one group split the block's pairs evenly)
  const int cpg = ncl / G, cig = cl / G;
  const int count = P.pb.count;
  const int p_begin = (int)((long long)cig * count / cpg);
  const int p_end = (int)((long long)(cig + 1) * count / cpg);
  const int U = (p_end - p_begin) * NT;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S23_NIN; ++i) {
      mbar_init(&S.in_full[i], 1);
      mbar_init(&S.in_empty[i], 8);  // fused: the slot's 4 FFT warps in each CTA; ZS: the 8 epilogue warps
    }
    mbar_init(&S.stg_full, 8);
    mbar_init(&S.stg_empty, 8);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.a_full[i], 16);
      mbar_init(&S.d_full[i], 1);
      mbar_init(&S.d_empty[i], 16);
      mbar_init(&S.red_full[i], 8);
      mbar_init(&S.red_empty[i], 1);
    }
    mbar_init(&S.y_bar, 1);
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
  // staging starts zeroed: words no term writes (padding columns, the unused half of a lone ell = 0 word)
  // stay zero for the whole kernel
  if (!ZS)
    for (int w = threadIdx.x; w < 2 * KW * RS; w += blockDim.x) stg[w] = 0u;
  if (warp == kWMma) tmem_alloc_cg2<512>(&S.tmem_base);
  if (warp == kWY && lane == 0) {  // this CTA's half of the group's Y image
    const uint32_t yb = (uint32_t)P.yhalf;
    mbar_arrive_expect_tx(&S.y_bar, yb);
    const uint8_t* src = P.Ysm + P.g_yoff[grp] + (long long)h * P.yhalf;
    for (uint32_t o = 0; o < yb; o += 32768u) bulk_g2s(ys + o, src + o, min(32768u, yb - o), &S.y_bar);
    mbar_wait(&S.y_bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // barriers initialized, TMEM allocated, Y halves resident in both CTAs
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  const uint32_t acol0 = 4u * (uint32_t)NCH;
  unsigned long long* tr = (kDiag23 && P.trace && cl == 0) ? P.trace + 16 * h : nullptr;

  if (warp == kWMma) {
    // ---------------- MMA issue (even CTA): all K-steps unrolled at compile time per chunk
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
    if (h == 0 && elect_one()) {
      S23MmaArgs a{tmem, acol0, smem_u32(ys), (uint32_t)nch * (uint32_t)(NCH / 2) * (uint32_t)K3p * 2u,
                   (uint32_t)(NCH / 2) * (uint32_t)K3p * 2u, (uint32_t)K3p * 16u, NCH, nch, K3p, P.Ke / 16, U, &S,
                   tr};
      switch (K3p / 16) {
        case 2: s23_mma_loop<2>(a); break;
        case 3: s23_mma_loop<3>(a); break;
        case 4: s23_mma_loop<4>(a); break;
        case 5: s23_mma_loop<5>(a); break;
        case 6: s23_mma_loop<6>(a); break;
        case 7: s23_mma_loop<7>(a); break;
        case 8: s23_mma_loop<8>(a); break;
        default: s23_mma_loop<0>(a); break;
      }
    }
    __syncwarp();
  } else if (warp == kWTma) {
    // ---------------- TMA producer: the block's 8-term window, this CTA's n/2 rows, multicast to both CTAs
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
    if (lane == 0 && ZS) {
      // r-tile images of k_step2_fft (one contiguous hi + lo image per (pair, r-tile)) into the staging ring
      for (int u = 0; u < U; ++u) {
        const int slot = u & 1;
        const int p = p_begin + u / NT, T = 2 * (u % NT) + (int)h;
        mbar_wait(&S.in_empty[slot], ((uint32_t)(u >> 1) & 1u) ^ 1u);
        if (T < P.NRT) {
          const uint32_t bytes = 2u * rt_part;
          mbar_arrive_expect_tx(&S.in_full[slot], bytes);
          const uint8_t* src = P.Zop + ((size_t)p * P.NRT + T) * bytes;
          uint8_t* dst = reinterpret_cast<uint8_t*>(stg) + (size_t)slot * bytes;
          for (uint32_t o = 0; o < bytes; o += 32768u) bulk_g2s(dst + o, src + o, min(32768u, bytes - o), &S.in_full[slot]);
        } else {
          mbar_arrive(&S.in_full[slot]);  // no such r-tile (odd NRT): the rows stay inactive
        }
      }
    } else if (lane == 0) {
      uint32_t g = 0;
      const int half = n / 2;
      long long w_e = 0;
      for (int u = 0; u < U; ++u) {
        const int p = p_begin + u / NT;
        if (u % NT == 0 && p + 1 < p_end)  // the next pair's windows into L2 while this pair is loaded
          for (int b = 0; b < P.B.nb; ++b) tma_prefetch_2d(&zmap, P.B.zs[b] & ~1, (p + 1) * n + (int)h * half);
        for (int b = 0; b < P.B.nb; ++b, ++g) {
          const int slot = g % S23_NIN;
          const long long t1 = clk23();
          mbar_wait(&S.in_empty[slot], ((g / S23_NIN) & 1u) ^ 1u);
          w_e += clk23() - t1;
          mbar_arrive_expect_tx(&S.in_full[slot], (uint32_t)n * 64u);
          if (kDiag23 && (P.dbg & 4))  // timing experiment: contiguous 1-D bulk copies of the same size
            bulk_g2s_mc(inb + (size_t)slot * n * 64 + (size_t)h * half * 64,
                        reinterpret_cast<const uint8_t*>(P.zdbg) + (size_t)p * n * P.Hs * 8 + (size_t)(b % 6) * n * 64 / 2 +
                            (size_t)h * half * 32,
                        (uint32_t)half * 64u, &S.in_full[slot], (uint16_t)3);
          else
          tma_load_2d_mc(inb + (size_t)slot * n * 64 + (size_t)h * half * 64, &zmap, P.B.zs[b] & ~1,
                         p * n + (int)h * half, &S.in_full[slot], (uint16_t)3);
        }
      }
      if (tr) tr[9] = w_e;
    }
    __syncwarp();
  } else if (warp == kWMerge) {
    // ---------------- merge: the 8 epilogue warps' records of each pair
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
    uint32_t it = 0;
    for (int p = p_begin; p < p_end; ++p) {
      int i, j;
      pair_of(P.pb, p, i, j);
      if (!s23_flush(P, MODE, p, p_end, i)) continue;
      const int rb = it & 1;
      mbar_wait_lazy(&S.red_full[rb], (it >> 1) & 1, 200);
      ++it;
      if (lane == 0) {
        if (MODE == 1) {
          float m = S.red_v[rb][0], sm = S.red_s[rb][0];
          for (int w = 1; w < 8; ++w) lse2_merge(m, sm, S.red_v[rb][w], S.red_s[rb][w]);
          mbar_arrive(&S.red_empty[rb]);
          const size_t ij = (size_t)i * P.n_tm_local + j;
          P.marg_part[(size_t)(grp * 2 + (int)h) * (size_t)P.marg_np + ij] = make_float2(m, sm);
        } else {
          float v = S.red_v[rb][0];
          uint32_t f = S.red_f[rb][0];
          for (int w = 1; w < 8; ++w)
            if (better(S.red_v[rb][w], S.red_f[rb][w], v, f)) {
              v = S.red_v[rb][w];
              f = S.red_f[rb][w];
            }
          mbar_arrive(&S.red_empty[rb]);
          if (f != 0xffffffffu) {
            // f: global flat index (template, shift, rot); v is in pair p's fp16x3 units (exact rescale)
            const int pe = z_exp(__ldg(P.ast + i), __ldg(P.bst + j), P.gmax) + P.eY;
            const unsigned long long key = pack_key(v * pow2f_wide(-pe), f);
            if (P.img_keys) atomicMax(&P.img_keys[i], key);
            if (P.pair_keys) atomicMax(&P.pair_keys[(size_t)i * P.n_tm_local + j], key);
          }
        }
      }
      __syncwarp();
    }
  } else if (warp >= kWEpi && warp < kWEpi + 8) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegEpi));
    // ---------------- epilogue (two warps per TMEM lane quarter, each half of a chunk's columns)
    const int q = warp & 3;
    const int ew = warp - kWEpi;
    const int eh = ew >> 2;
    const int row = q * 32 + lane;         // tile row i
    const int hw = NCH / 2;                // columns per warp (multiple of 8)
    const bool has_odd = P.Ke < K3p;
    const bool active_f = q * 32 < F;      // warp-uniform: rows >= F are padding
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t a_full_cl0 = mapa_shared(&S.a_full[0], 0), a_full_cl1 = mapa_shared(&S.a_full[1], 0);
    const uint32_t d_empty_cl0 = mapa_shared(&S.d_empty[0], 0), d_empty_cl1 = mapa_shared(&S.d_empty[1], 0);
    const int wq = KW / 2;                 // words per part this warp copies: [eh wq, (eh + 1) wq)
    const int pi_row = row + V * (row / (V * V));
    auto copy_stage_zs = [&](int v) {
      // ZS: the r-tile image of unit v (staging slot v & 1, canonical K-major core matrices [part][row/8]
      // [K3p/8][8 rows x 16 B]) -> TMEM A slot v & 1, 4 words (one 16-byte core row) per tcgen05.st
      const int slot = v & 1;
      const uint8_t* img = reinterpret_cast<const uint8_t*>(stg) + (size_t)slot * 2 * rt_part +
                           (size_t)(row >> 3) * (K3p * 16) + (row & 7) * 16;
#pragma unroll 1
      for (int part = 0; part < 2; ++part)
#pragma unroll 1
        for (int w0 = eh * wq; w0 < (eh + 1) * wq; w0 += 4) {
          const uint4 v4 = *reinterpret_cast<const uint4*>(img + (size_t)part * rt_part + (w0 / 4) * 128);
          asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(
                           lane_base + acol0 + (uint32_t)(slot * K3p + part * KW + w0)),
                       "r"(v4.x), "r"(v4.y), "r"(v4.z), "r"(v4.w)
                       : "memory");
        }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_cluster(slot ? a_full_cl1 : a_full_cl0);
        mbar_arrive(&S.in_empty[slot]);
      }
    };
    auto copy_stage = [&](int slot) {
      // staging [part][word][RS] -> TMEM A slot (this warp's 32 rows, half of the words of each part)
      const bool ok = row < F;
#pragma unroll 1
      for (int part = 0; part < 2; ++part)
#pragma unroll 1
        for (int w0 = eh * wq; w0 < (eh + 1) * wq; w0 += 4) {
          uint4 v;
          const uint32_t* sp = stg + (size_t)(part * KW + w0) * RS + pi_row;
          v.x = ok ? sp[0] : 0u;
          v.y = ok ? sp[RS] : 0u;
          v.z = ok ? sp[2 * RS] : 0u;
          v.w = ok ? sp[3 * RS] : 0u;
          asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(
                           lane_base + acol0 + (uint32_t)(slot * K3p + part * KW + w0)),
                       "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                       : "memory");
        }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_cluster(slot ? a_full_cl1 : a_full_cl0);
        mbar_arrive(&S.stg_empty);
      }
    };
    // prologue: units 0 and 1 into both A slots
    for (int u0 = 0; u0 < 2 && u0 < U; ++u0) {
      if (ZS) {
        mbar_wait(&S.in_full[u0 & 1], 0u);
        copy_stage_zs(u0);
      } else {
        mbar_wait(&S.stg_full, (uint32_t)u0 & 1u);
        copy_stage(u0 & 1);
      }
    }
    uint32_t g_d = 0, pit = 0;
    long long w_df = 0, w_sf = 0, w_ld = 0, w_cp = 0, w_pr = 0, w_rl = 0;
    const long long t_e0 = clk23();
    float bv = -INFINITY;          // MODE 0: best value of this thread's rows in the current pair
    uint32_t bf = 0xffffffffu;     //         and its flat index t n + r
    float mrun = -INFINITY, srun = 0.f;  // MODE 1: running base-2 log-sum-exp of X log2(e) / tau
    int pe_prev = 0;
    for (int u = 0; u < U; ++u) {
      const int pl = u / NT, s = u - pl * NT;
      const int p = p_begin + pl;
      const int crot = 2 * s + (int)h;
      // rotation of this thread's row: fused r = D i + c; ZS r = 128 T + i (T = the r-tile, rows beyond n idle)
      const uint32_t r = ZS ? (uint32_t)(128 * crot + row) : (uint32_t)(D * row + crot);
      const bool active = ZS ? (128 * crot + q * 32 < n) : active_f;
      float* land_p = P.land ? P.land + (size_t)p * P.N_t * n : nullptr;
      int pi_img, pj_tm;
      pair_of(P.pb, p, pi_img, pj_tm);
      // fp16x3: this pair's results are X 2^pe; a MODE-0 record carried over from the previous pair of the same
      // image is rescaled (exactly) into this pair's units
      const int pe = z_exp(__ldg(P.ast + pi_img), __ldg(P.bst + pj_tm), P.gmax) + P.eY;
      if (s == 0) {
        if (MODE == 0 && bv != -INFINITY) bv *= pow2f_wide(pe - pe_prev);
        pe_prev = pe;
      }
      const float unsc = pow2f_wide(-pe);
      const float msc_p = P.msc * unsc;
      // flat indices are global ((template, shift) major, rotation minor): the running best of MODE 0 is
      // carried over the consecutive templates of one image unless per-pair maxima are requested
      const uint32_t fbase = (uint32_t)(P.tm_off + pj_tm) * (uint32_t)P.N_t;
      for (int c = 0; c < nch; ++c, ++g_d) {
        const int db = g_d & 1;
        long long t1 = clk23();
        mbar_wait(&S.d_full[db], (g_d >> 1) & 1u);
        w_df += clk23() - t1;
        tc_fence_after();
        const uint32_t base = lane_base + (uint32_t)(db * 2 * NCH + eh * hw);
        const int clb = c * NCH + eh * hw;
        const int nfast = land_p ? 0 : (int)s_fastc[c * 2 + eh];
        auto release = [&]() {
          const long long t5 = clk23();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(db ? d_empty_cl1 : d_empty_cl0);
          w_rl += clk23() - t5;
        };
        // the warp's whole half chunk (hw <= 48 columns of E and of O) in one TMEM round trip, then the D
        // buffer is released and the registers reduced
        uint32_t e[48], o[48];
        t1 = clk23();
        if (active) {
          tmem_ld16(base, *reinterpret_cast<uint32_t(*)[16]>(e));
          if (has_odd) tmem_ld16(base + NCH, *reinterpret_cast<uint32_t(*)[16]>(o));
          if (hw >= 32) {
            tmem_ld16(base + 16, *reinterpret_cast<uint32_t(*)[16]>(e + 16));
            if (has_odd) tmem_ld16(base + NCH + 16, *reinterpret_cast<uint32_t(*)[16]>(o + 16));
          } else if (hw >= 24) {
            tmem_ld8(base + 16, *reinterpret_cast<uint32_t(*)[8]>(e + 16));
            if (has_odd) tmem_ld8(base + NCH + 16, *reinterpret_cast<uint32_t(*)[8]>(o + 16));
          }
          if (hw >= 48) {
            tmem_ld16(base + 32, *reinterpret_cast<uint32_t(*)[16]>(e + 32));
            if (has_odd) tmem_ld16(base + NCH + 32, *reinterpret_cast<uint32_t(*)[16]>(o + 32));
          } else if (hw >= 40) {
            tmem_ld8(base + 32, *reinterpret_cast<uint32_t(*)[8]>(e + 32));
            if (has_odd) tmem_ld8(base + NCH + 32, *reinterpret_cast<uint32_t(*)[8]>(o + 32));
          }
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 48; ++k) asm volatile("" : "+r"(e[k]), "+r"(o[k]));  // no use before the wait
        }
        w_ld += clk23() - t1;
        release();
        if (!has_odd) {
#pragma unroll
          for (int k = 0; k < 48; ++k) o[k] = 0u;
        }
        const long long t4 = clk23();
        if (active && !(kDiag23 && (P.dbg & 2))) {
#pragma unroll
          for (int g8 = 0; g8 < 6; ++g8) {
            if (8 * g8 >= hw) break;
            const int cl = clb + 8 * g8;
            const bool fast = 8 * g8 < nfast;
            if (MODE == 0) {
              if (fast) {
                float v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(e[8 * g8 + k]) + fabsf(__uint_as_float(o[8 * g8 + k]));
                const float m = fmaxf(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])), fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7])));
                if (kDiag23 && (P.dbg & 8)) {  // timing experiment: track the value only
                  bv = fmaxf(bv, m);
                } else if (m >= bv) {  // rare: resolve the exact (shift, sign) of a new maximum
#pragma unroll
                  for (int k = 0; k < 8; ++k) {
                    if (v[k] != m) continue;
                    const float ov = __uint_as_float(o[8 * g8 + k]);
                    const int tp = s_rep[cl + k], tm = s_part[cl + k];
                    const int t = (ov > 0.f || (ov == 0.f && tp < tm)) ? tp : tm;
                    const uint32_t f = (fbase + (uint32_t)t) * (uint32_t)n + r;
                    if (better(m, f, bv, bf)) {
                      bv = m;
                      bf = f;
                    }
                  }
                }
              } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  const int tp = s_rep[cl + k], tm = s_part[cl + k];
                  if (tp < 0) continue;
                  const float ev = __uint_as_float(e[8 * g8 + k]), ov = __uint_as_float(o[8 * g8 + k]);
                  const float xp = ev + ov;
                  const uint32_t fp = (fbase + (uint32_t)tp) * (uint32_t)n + r;
                  if (better(xp, fp, bv, bf)) {
                    bv = xp;
                    bf = fp;
                  }
                  if (land_p && row < F) land_p[(size_t)tp * n + r] = xp * unsc;
                  if (tm >= 0) {
                    const float xm = ev - ov;
                    const uint32_t fm = (fbase + (uint32_t)tm) * (uint32_t)n + r;
                    if (better(xm, fm, bv, bf)) {
                      bv = xm;
                      bf = fm;
                    }
                    if (land_p && row < F) land_p[(size_t)tm * n + r] = xm * unsc;
                  }
                }
              }
            } else {
              // MODE 1: online log-sum-exp over both signs of delta (valid columns only)
              float cm = -INFINITY;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float ev = __uint_as_float(e[8 * g8 + k]), ov = __uint_as_float(o[8 * g8 + k]);
                if (fast) {
                  cm = fmaxf(cm, ev + fabsf(ov));
                } else {
                  if (s_rep[cl + k] >= 0) cm = fmaxf(cm, ev + ov);
                  if (s_part[cl + k] >= 0) cm = fmaxf(cm, ev - ov);
                }
              }
              if (cm != -INFINITY) {
                cm *= msc_p;
                if (cm > mrun) {
                  srun *= ex2_approx(mrun - cm);
                  mrun = cm;
                }
                const float nm = -mrun, sc = msc_p;
                float sk = 0.f;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  const float ev = __uint_as_float(e[8 * g8 + k]), ov = __uint_as_float(o[8 * g8 + k]);
                  if (fast) {
                    sk += ex2_approx(fmaf(ev + ov, sc, nm)) + ex2_approx(fmaf(ev - ov, sc, nm));
                  } else {
                    if (s_rep[cl + k] >= 0) sk += ex2_approx(fmaf(ev + ov, sc, nm));
                    if (s_part[cl + k] >= 0) sk += ex2_approx(fmaf(ev - ov, sc, nm));
                  }
                }
                srun += sk;
              }
            }
          }
        }
        if (kDiag23 && (P.dbg & 2) && active) bv = fmaxf(bv, __uint_as_float(e[0]) + __uint_as_float(o[0]));
        w_pr += clk23() - t4;
      }
      // unit u's MMAs are complete (its last chunk's commit arrived): refill its A slot with unit u + 2
      if (u + 2 < U) {
        const long long t1 = clk23();
        if (ZS)
          mbar_wait(&S.in_full[u & 1], (uint32_t)((u + 2) >> 1) & 1u);
        else
          mbar_wait(&S.stg_full, (uint32_t)(u + 2) & 1u);
        w_sf += clk23() - t1;
        const long long t2 = clk23();
        if (ZS)
          copy_stage_zs(u + 2);
        else
          copy_stage(u & 1);
        w_cp += clk23() - t2;
      }
      if (s == NT - 1 && s23_flush(P, MODE, p, p_end, pi_img)) {
        // record of this warp (per pair, or per run of one image's templates) -> merge warp
        if (MODE == 1) {
#pragma unroll
          for (int o2 = 16; o2 > 0; o2 >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, mrun, o2);
            const float s2 = __shfl_xor_sync(0xffffffffu, srun, o2);
            lse2_merge(mrun, srun, m2, s2);
          }
        } else {
#pragma unroll
          for (int o2 = 16; o2 > 0; o2 >>= 1) {
            const float v2 = __shfl_xor_sync(0xffffffffu, bv, o2);
            const uint32_t f2 = __shfl_xor_sync(0xffffffffu, bf, o2);
            if (better(v2, f2, bv, bf)) {
              bv = v2;
              bf = f2;
            }
          }
        }
        const int rb = pit & 1;
        if (lane == 0) {
          mbar_wait(&S.red_empty[rb], ((pit >> 1) & 1u) ^ 1u);
          S.red_v[rb][ew] = MODE == 1 ? mrun : bv;
          S.red_s[rb][ew] = srun;
          S.red_f[rb][ew] = bf;
          mbar_arrive(&S.red_full[rb]);
        }
        __syncwarp();
        ++pit;
        bv = -INFINITY;
        bf = 0xffffffffu;
        mrun = -INFINITY;
        srun = 0.f;
      }
    }
    if (tr && warp == kWEpi && lane == 0) {
      tr[3] = clk23() - t_e0;
      tr[4] = w_df;
      tr[5] = w_sf;
      tr[11] = w_ld;
      tr[12] = w_cp;
      tr[15] = w_pr;
      tr[2 + 16 * 0] = tr[2];  // (kept)
      tr[0 + 16 * 0] = tr[0];
      if (h == 1) tr[1] = w_rl;
    }
  } else if (warp == kWY) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
  } else if (warp < kWEpiFft) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegFft));
    if constexpr (!ZS) {
    // ---------------- FFT warps: two terms of each Step-2 block per warp, one per 16-lane half.
    // F-point DFT of y_c over q1 = a + 16 b (a = lane % 16, b < V):
    //   (A) V-point DFT over b in registers, twiddle w_F^{a k1};  (T) transpose through the warp's scratch so
    //   that lane (k1, a0) holds a = R a1 + a0, a1 < V;  (A2) V-point DFT over a1, twiddle w_16^{a0 m};
    //   (C) R-point DIF across the R lanes of each k1 (log2 R shuffle stages).
    // Output row i = k1 + V (m + V m2), m2 = bitrev_R(a0), in x[rv(m)].
    const int fg = warp >> 2, fw = warp & 3;  // group fg takes the blocks of input slot fg
    const int tau = lane >> 4, a = lane & 15;
    const int k1g = a / R, a0 = a % R;
    const int m2 = (R == 4) ? (((a0 & 1) << 1) | (a0 >> 1)) : a0;
    float2* scr = reinterpret_cast<float2*>(sraw + LY.scr) + (warp * 2 + tau) * V * SR;
    const uint32_t in_empty_cl0 = mapa_shared(&S.in_empty[0], h ^ 1u), in_empty_cl1 = mapa_shared(&S.in_empty[1], h ^ 1u);
    const float2* __restrict__ twa = P.twA + a * V;             // w_F^{a k1}   (L1-resident tables)
    const float2* __restrict__ tw16 = P.twA + 16 * V + a0 * V;  // w_16^{a0 m}
    float2 wcr[LR];  // twiddles of the R-point DIF stages (1 on the lower lanes)
#pragma unroll
    for (int st = 0; st < LR; ++st) {
      const int hh = (R / 2) >> st;
      wcr[st] = make_float2(1.f, 0.f);
      if (R == 4 && hh == 2 && (a0 & 2) && (a0 & 1)) wcr[st] = make_float2(0.f, -1.f);  // w_4^1
    }
    auto rv = [](int i) {
      constexpr int LOGV = (V == 8) ? 3 : 2;
      int rr = 0;
#pragma unroll
      for (int bb = 0; bb < LOGV; ++bb) rr |= ((i >> bb) & 1) << (LOGV - 1 - bb);
      return rr;
    };
    uint32_t g = 0;
    long long w_se = 0, w_if = 0, w_cb = 0, w_ff = 0;
    const long long t_f0 = clk23();
    for (int u = 0; u < U; ++u) {
      const int s = u % NT;
      const int crot = 2 * s + (int)h;
      float zsc;  // fp16x3: this pair's Zhat' scale -> its Z scale
      {
        int pi_, pj_;
        pair_of(P.pb, p_begin + u / NT, pi_, pj_);
        zsc = zhat_to_z_scale(__ldg(P.ast + pi_), __ldg(P.bst + pj_), P.gmax);  // Zhat' arrives in Step 1's scale
      }
      // per unit: w_n^{q1 c} for this lane's q1 = a + 16 b, and the radix-D combination constants
      float2 tu[V];
#pragma unroll
      for (int b = 0; b < V; ++b) tu[b] = tw_full(P.twn, ((a + 16 * b) * crot) & (n - 1), n);
      const float sg = (crot & 1) ? -1.f : 1.f;                       // w_D^{(D/2) c} = (-1)^c
      const float2 rho = (crot & 3) == 0 ? make_float2(1.f, 0.f) : (crot & 3) == 1 ? make_float2(0.f, -1.f)
                        : (crot & 3) == 2 ? make_float2(-1.f, 0.f) : make_float2(0.f, 1.f);  // D = 4: (-i)^c
      long long t1 = clk23();
      mbar_wait(&S.stg_empty, ((uint32_t)u & 1u) ^ 1u);
      w_se += clk23() - t1;
      for (int b = 0; b < P.B.nb; ++b, ++g) {
        const int slot = g % S23_NIN;
        if (slot != fg) continue;
        t1 = clk23();
        mbar_wait(&S.in_full[slot], (g / S23_NIN) & 1u);
        w_if += clk23() - t1;
        const int zs = P.B.zs[b], nz = P.B.ze[b] - zs;
        const int zz = 2 * fw + tau;
        const bool act = zz < nz;
        const int zc = act ? zz : 0;
        int l = 0, cc = 0;
        if (nz > 0) {
          l = __ldg(P.ell + zs + zc);
          cc = __ldg(P.col + zs + zc);
        }
        const int e = (zs & 1) + zc;  // window column
        // y_c(q1) = w_n^{q1 c} sum_j w_D^{j c} Zhat'(q1 + F j - ell)  (Form B shift, reading R5).  The rows
        // q1 + F j - ell = p0 + 16 (b + V j) share one 64B-swizzle phase (multiples of 16 apart)
        long long t3 = clk23();
        if (kDiag23 && (P.dbg & 1)) {  // timing experiment: no FFT arithmetic
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&S.in_empty[slot]);
            mbar_arrive_cluster(slot ? in_empty_cl1 : in_empty_cl0);
          }
          continue;
        }
        const int p0 = (a - l) & (n - 1);
        const int swz = ((((e >> 1) ^ (p0 >> 1)) & 3) << 1) | (e & 1);
        const float2* rows = reinterpret_cast<const float2*>(inb + (size_t)slot * n * 64) + swz;
        float2 x[V];
#pragma unroll
        for (int b = 0; b < V; ++b) {
          auto at = [&](int m) { return rows[((p0 + 16 * m) & (n - 1)) * 8]; };
          float2 y;
          if (D == 2) {
            y = fma2(make_float2(sg, sg), at(b + V), at(b));
          } else {
            const float2 t1a = fma2(make_float2(sg, sg), at(b + 2 * V), at(b));
            const float2 t2a = fma2(make_float2(sg, sg), at(b + 3 * V), at(b + V));
            y = add2(t1a, cmulf(rho, t2a));
          }
          x[b] = cmulf(y, tu[b]);
        }
        __syncwarp();
        if (lane == 0) {  // this CTA is done reading the slot: release it in both CTAs (multicast refill)
          mbar_arrive(&S.in_empty[slot]);
          mbar_arrive_cluster(slot ? in_empty_cl1 : in_empty_cl0);
        }
        w_cb += clk23() - t3;
        t3 = clk23();
        dft_regs<V>(x);  // (A): X[a, k1] at x[rv(k1)]
#pragma unroll
        for (int k = 1; k < V; ++k) x[rv(k)] = cmulf(x[rv(k)], __ldg(twa + k));
#pragma unroll
        for (int k = 0; k < V; ++k) scr[k * SR + a] = x[rv(k)];  // (T)
        __syncwarp();
#pragma unroll
        for (int a1 = 0; a1 < V; ++a1) x[a1] = scr[k1g * SR + R * a1 + a0];
        __syncwarp();
        dft_regs<V>(x);  // (A2): Y[m] at x[rv(m)]
#pragma unroll
        for (int m = 1; m < V; ++m) x[rv(m)] = cmulf(x[rv(m)], __ldg(tw16 + m));
#pragma unroll
        for (int st = 0; st < LR; ++st) {  // (C)
          const int hh = (R / 2) >> st;
          const float sgn = (a0 & hh) ? -1.f : 1.f;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const float px = __shfl_xor_sync(0xffffffffu, x[v].x, hh);
            const float py = __shfl_xor_sync(0xffffffffu, x[v].y, hh);
            x[v] = fma2(make_float2(sgn, sgn), x[v], make_float2(px, py));
            if (R == 4 && st == 0) x[v] = cmulf(x[v], wcr[0]);
          }
        }
        w_ff += clk23() - t3;
        if (act && !(kDiag23 && (P.dbg & 16))) {
          // stage: ell > 0 -> word (Re, Im); ell = 0 -> one fp16 half of a word (the other: a neighbour or zero)
          const int W = cc >> 1;
          uint32_t* shi = stg + (size_t)W * RS;
          uint32_t* slo = stg + (size_t)(KW + W) * RS;
#pragma unroll
          for (int m = 0; m < V; ++m) {
            const int i = k1g + V * m + V * V * m2;
            const int pi = i + V * m2;
            const float2 a0v = mul2(make_float2(zsc, zsc), x[rv(m)]);
            if (l > 0) {
              uint32_t hh2, ll2;
              split2_f16(a0v.x, a0v.y, hh2, ll2);
              shi[pi] = hh2;
              slo[pi] = ll2;
            } else {
              const __half hb = __float2half_rn(a0v.x);
              const __half lb = __float2half_rn(a0v.x - __half2float(hb));
              reinterpret_cast<__half*>(shi + pi)[cc & 1] = hb;
              reinterpret_cast<__half*>(slo + pi)[cc & 1] = lb;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.stg_full);
    }
    if (tr && warp == 0 && lane == 0) {
      tr[6] = clk23() - t_f0;
      tr[7] = w_se;
      tr[8] = w_if;
      tr[10] = U;
      tr[13] = w_cb;
      tr[14] = w_ff;
    }
    }  // !ZS
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == kWMma) {
    tc_fence_after();
    tmem_dealloc_cg2<512>(tmem);
  }
}

// ---------------------------------------------------------------- host side
bool tc_s23_eligible(const TcPlan& tc, const DevPlan& P) { return tc.s23_ready && P.n_gamma == P.n_psi; }
bool tc_s3v2_eligible(const TcPlan& tc, const DevPlan&) { return tc.s3v2_ready; }

// Plan-time setup of the CTA-pair Step-3 kernels (k_step23): the Step-3-only variant (operand tiles from
// k_step2_fft, any n_gamma) whenever its layout fits, and the fused Step 2+3 variant (n_gamma = n_psi in
// {128, 256, 512}) when requested (fused = true) and its larger shared-memory layout fits with the same
// rep-groups.  Leaves both off (no error) for shapes they do not cover: k_step3_tc then runs.
int tc_s23_init(TcPlan& tc, int n_psi, int n_gamma, const std::vector<int>& rep, const std::vector<int>& partner,
                const std::vector<float>& Y3, int K3p, bool fused, std::string& msg) {
  tc.s23_ready = tc.s3v2_ready = false;
  const int n = n_psi;
  const bool fused_shape = fused && n_gamma == n_psi && (n_psi == 128 || n_psi == 256 || n_psi == 512);
  const int F = std::min(128, n / 2), D = std::max(2, n / std::max(F, 1)), V = F / 16;
  // TMEM: two D buffers (E + O, NCH columns each) + two A slots (K3p columns) <= 512; NCH multiple of 16
  // (the epilogue drains a half chunk of up to 48 columns per warp: NCH <= 96)
  const int nmax = std::min(96, ((512 - 2 * K3p) / 4) / 16 * 16);
  if (nmax < 32) return FTK_OK;
  const size_t smem_cap = 232448;
  const int n_rep = (int)rep.size();
  int G = 0, nch = 0, NCH = 0;
  for (int g = 1; g <= TcPlan::MAXG; ++g) {
    const int rg = (n_rep + g - 1) / g;
    const int c = (rg + nmax - 1) / nmax;
    const int w = ((rg + c - 1) / c + 15) / 16 * 16;
    const S23Layout LY = s23_layout(c * w, c, w, K3p, n_gamma, 0);
    if (LY.total <= smem_cap) {
      G = g;
      nch = c;
      NCH = w;
      break;
    }
  }
  if (G == 0) return FTK_OK;
  const bool fused_fits = fused_shape && s23_layout(nch * NCH, nch, NCH, K3p, n, V).total <= smem_cap;
  const int rg = (n_rep + G - 1) / G;
  const int ncol_g = nch * NCH;
  tc.s23_G = G;
  tc.s23_nch = nch;
  tc.s23_NCH = NCH;
  tc.s23_F = F;
  tc.s23_D = D;
  tc.s23_ncol = G * ncol_g;
  std::vector<int> colrep(tc.s23_ncol, -1), colpart(tc.s23_ncol, -1);
  std::vector<uint8_t> colfast(tc.s23_ncol / 8 + 16, 0);
  // Y image per (group, half): [part][chunk][NCH/2 rows][K3p] canonical K-major (core = 8 rows x 16 B)
  const int hr = NCH / 2;
  const size_t half_elems = (size_t)2 * nch * hr * K3p;  // fp16 elements (both parts)
  tc.s23_yhalf = (long long)half_elems * 2;
  std::vector<uint16_t> yimg((size_t)G * 2 * half_elems, 0);
  for (int g = 0; g < G; ++g) {
    tc.s23_col0[g] = g * ncol_g;
    tc.s23_yoff[g] = (long long)g * 2 * tc.s23_yhalf;
    for (int c = 0; c < ncol_g; ++c) {
      const int rr = g * rg + c;
      if (c >= rg || rr >= n_rep) continue;
      colrep[g * ncol_g + c] = rep[rr];
      colpart[g * ncol_g + c] = partner[rr];
      const int t = rep[rr];
      const int chunk = c / NCH, within = c % NCH, hh = within / hr, rrow = within % hr;
      for (int k = 0; k < K3p; ++k) {
        const float x = std::ldexp(Y3[(size_t)t * K3p + k], tc.eY);  // fp16x3 (see ftk_tc.cu header)
        const __half hi = __float2half_rn(x);
        const __half lo = __float2half_rn(x - __half2float(hi));
        const size_t core = (size_t)chunk * hr * K3p + (size_t)(rrow / 8) * (K3p / 8) * 64 + (size_t)(k / 8) * 64 +
                            (rrow % 8) * 8 + (k % 8);
        const size_t hbase = ((size_t)g * 2 + hh) * half_elems;
        std::memcpy(&yimg[hbase + core], &hi, 2);
        std::memcpy(&yimg[hbase + (size_t)nch * hr * K3p + core], &lo, 2);
      }
    }
  }
  for (int c8 = 0; c8 < tc.s23_ncol / 8; ++c8) {
    bool f = true;
    for (int k = 0; k < 8; ++k) f = f && colrep[c8 * 8 + k] >= 0 && colpart[c8 * 8 + k] >= 0;
    colfast[c8] = f ? 1 : 0;
  }
  // four-step twiddles of the F-point FFT (F = 16 V, R = 16 / V): [a < 16][k1 < V] w_F^{a k1}, [a0 < R][m < V] w_16^{a0 m}
  const int R = 16 / V;
  std::vector<float2> tw((size_t)16 * V + (size_t)R * V), twh;
  for (int a = 0; a < 16; ++a)
    for (int k = 0; k < V; ++k) {
      const double ph = -2.0 * M_PI * (double)((a * k) % F) / F;
      tw[(size_t)a * V + k] = make_float2((float)std::cos(ph), (float)std::sin(ph));
    }
  for (int a0 = 0; a0 < R; ++a0)
    for (int m = 0; m < V; ++m) {
      const double ph = -2.0 * M_PI * (double)((a0 * m) % 16) / 16.0;
      tw[(size_t)16 * V + (size_t)a0 * V + m] = make_float2((float)std::cos(ph), (float)std::sin(ph));
    }
  if (cudaMalloc(&tc.d_s23_colrep, colrep.size() * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&tc.d_s23_colpart, colpart.size() * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&tc.d_s23_colfast, colfast.size()) != cudaSuccess ||
      cudaMalloc(&tc.d_s23_Ysm, yimg.size() * 2) != cudaSuccess ||
      cudaMalloc(&tc.d_s23_tw, tw.size() * sizeof(float2)) != cudaSuccess) {
    msg = "fused Step 2+3: allocation failed";
    return FTK_ENOMEM;
  }
  cudaMemcpy(tc.d_s23_colrep, colrep.data(), colrep.size() * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemcpy(tc.d_s23_colpart, colpart.data(), colpart.size() * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemcpy(tc.d_s23_colfast, colfast.data(), colfast.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(tc.d_s23_Ysm, yimg.data(), yimg.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(tc.d_s23_tw, tw.data(), tw.size() * sizeof(float2), cudaMemcpyHostToDevice);
  tc.s3v2_smem = s23_layout(ncol_g, nch, NCH, K3p, n_gamma, 0).total;
  tc.s23_smem = fused_fits ? s23_layout(ncol_g, nch, NCH, K3p, n, V).total : 0;
  tc.s3v2_NRT = (n_gamma + 127) / 128;
  FTK_SMEM_OPTIN((k_step23<0, 8, 4>));
  FTK_SMEM_OPTIN((k_step23<0, 8, 2>));
  FTK_SMEM_OPTIN((k_step23<0, 4, 2>));
  FTK_SMEM_OPTIN((k_step23<1, 8, 4>));
  FTK_SMEM_OPTIN((k_step23<1, 8, 2>));
  FTK_SMEM_OPTIN((k_step23<1, 4, 2>));
  FTK_SMEM_OPTIN((k_step23<0, 0, 2>));
  FTK_SMEM_OPTIN((k_step23<1, 0, 2>));
  tc.s23_ready = fused_fits;
  {  // opt-in (FTK_S3V2=1): bit-identical to k_step3_tc but measured 2x slower at c5 (with
     // two TMEM D buffers the cross-CTA release chain is longer than one chunk's MMAs)
    const char* e = std::getenv("FTK_S3V2");
    tc.s3v2_ready = e && e[0] == '1';
  }
  return FTK_OK;
}

void tc_s23_free(TcPlan& tc) {
  cudaFree(tc.d_s23_colrep);
  cudaFree(tc.d_s23_colpart);
  cudaFree(tc.d_s23_colfast);
  cudaFree(tc.d_s23_Ysm);
  cudaFree(tc.d_s23_tw);
  tc.d_s23_colrep = tc.d_s23_colpart = nullptr;
  tc.d_s23_colfast = nullptr;
  tc.d_s23_Ysm = nullptr;
  tc.d_s23_tw = nullptr;
  tc.s23_ready = tc.s3v2_ready = false;
}

// One launch of k_step23: zs = false -> fused Steps 2 + 3 from Zhat'; zs = true -> Step 3 only from k_step2_fft's
// r-tile images Zop.
static int launch_cg2(const TcPlan& tc, bool zs, const float2* Zhat, const uint8_t* Zop, const PairBlock& pb,
                      const DevPlan& P, int tm_off, unsigned long long* img_keys, unsigned long long* pair_keys,
                      int n_tm_local, float* land, cudaStream_t s) {
  const int n = zs ? P.n_gamma : P.n_psi;
  // fused: Zhat' [pair][p][Hs] as a 2-D tensor of 8-byte elements (rows = pair * n + p), boxes of 8 terms x n/2
  // rows, 64-byte swizzle (the layout s2_slot() reads)
  alignas(64) CUtensorMap zmap;
  std::memset(&zmap, 0, sizeof zmap);
  if (!zs) {
    PFN_encodeTiled enc = get_encode_tiled();
    if (!enc) return FTK_ECUDA;
    const cuuint64_t dims[2] = {(cuuint64_t)P.Hs, (cuuint64_t)pb.count * n};
    const cuuint64_t strides[1] = {(cuuint64_t)P.Hs * 8};
    const cuuint32_t box[2] = {8u, (cuuint32_t)(n / 2)};
    const cuuint32_t es[2] = {1u, 1u};
    if (enc(&zmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<float2*>(Zhat), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return FTK_ECUDA;
  }
  S23Params prm;
  std::memset(&prm, 0, sizeof prm);
  prm.Ysm = tc.d_s23_Ysm;
  prm.colrep = tc.d_s23_colrep;
  prm.colpart = tc.d_s23_colpart;
  prm.colfast = tc.d_s23_colfast;
  prm.ell = P.ell;
  prm.col = P.col;
  prm.twn = P.twg;
  prm.twA = tc.d_s23_tw;
  std::memcpy(&prm.B, &tc.s2_blocks, sizeof prm.B);
  prm.pb = pb;
  prm.n = n;
  prm.F = tc.s23_F;
  prm.D = tc.s23_D;
  prm.NT = zs ? (tc.s3v2_NRT + 1) / 2 : tc.s23_D / 2;
  prm.Zop = Zop;
  prm.NRT = tc.s3v2_NRT;
  prm.K3p = P.K3p;
  prm.Ke = P.Ke;
  prm.N_t = P.N_t;
  prm.NCH = tc.s23_NCH;
  prm.G = tc.s23_G;
  prm.nch = tc.s23_nch;
  for (int g = 0; g < tc.s23_G; ++g) {
    prm.g_col0[g] = tc.s23_col0[g];
    prm.g_yoff[g] = tc.s23_yoff[g];
  }
  prm.yhalf = tc.s23_yhalf;
  prm.tm_off = tm_off;
  prm.n_tm_local = n_tm_local;
  prm.img_keys = img_keys;
  prm.pair_keys = pair_keys;
  prm.land = land;
  prm.marg_part = tc.marg ? tc.marg_part : nullptr;
  prm.marg_np = tc.marg_np;
  prm.msc = tc.marg_scale;
  prm.ast = tc.d_ast;
  prm.bst = tc.d_bst;
  prm.gmax = tc.gmax;
  prm.eY = tc.eY;
  if (kDiag23) {
    const char* e = std::getenv("FTK_S23_DBG");
    prm.dbg = e ? std::atoi(e) : 0;
    prm.zdbg = Zhat;
    prm.Hs = P.Hs;
  }
  static unsigned long long* d_trace = nullptr;  // diagnostics: FTK_S23_TRACE=1 prints cluster 0's counters
  const char* tenv = kDiag23 ? std::getenv("FTK_S23_TRACE") : nullptr;
  if (tenv && tenv[0] == '1') {
    if (!d_trace) cudaMalloc(&d_trace, 32 * sizeof(unsigned long long));
    cudaMemsetAsync(d_trace, 0, 32 * sizeof(unsigned long long), s);
    prm.trace = d_trace;
  }
  // clusters: a multiple of G, at most one CTA per SM, at most one cluster per pair of the block
  int ncl = tc.num_sms / 2;
  ncl = std::min(ncl, pb.count * tc.s23_G);
  ncl = std::max(tc.s23_G, ncl / tc.s23_G * tc.s23_G);
  const dim3 grid(2 * ncl);
  const size_t smem = zs ? tc.s3v2_smem : tc.s23_smem;
  const int V = tc.s23_F / 16, D = tc.s23_D;
  auto go = [&](auto kern) { kern<<<grid, S23_THREADS, smem, s>>>(prm, zmap); };
  if (zs) {
    if (tc.marg) go(k_step23<1, 0, 2>);
    else go(k_step23<0, 0, 2>);
  } else if (tc.marg) {
    if (V == 8 && D == 4) go(k_step23<1, 8, 4>);
    else if (V == 8) go(k_step23<1, 8, 2>);
    else go(k_step23<1, 4, 2>);
  } else {
    if (V == 8 && D == 4) go(k_step23<0, 8, 4>);
    else if (V == 8) go(k_step23<0, 8, 2>);
    else go(k_step23<0, 4, 2>);
  }
  if (prm.trace) {
    unsigned long long hb[32];
    cudaMemcpyAsync(hb, d_trace, sizeof hb, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    for (int c = 0; c < 2; ++c) {
      const unsigned long long* t = hb + 16 * c;
      fprintf(stderr, "s23trace cta%d units=%llu mma: total %llu wait_a %llu wait_d %llu | epi: total %llu wait_dfull %llu "
              "wait_stg %llu ld+wait %llu copy %llu | fft: total %llu wait_stg_empty %llu wait_in %llu combine %llu fft %llu | "
              "tma wait_empty %llu | process %llu release(cta1) %llu\n",
              c, t[10], t[0], t[1], t[2], t[3], t[4], t[5], t[11], t[12], t[6], t[7], t[8], t[13], t[14], t[9], t[15], t[1]);
    }
  }
  return cudaGetLastError() == cudaSuccess ? FTK_OK : FTK_ECUDA;
}

int launch_step23(const TcPlan& tc, const float2* Zhat, const PairBlock& pb, const DevPlan& P, int tm_off,
                  unsigned long long* img_keys, unsigned long long* pair_keys, int n_tm_local, float* land,
                  cudaStream_t s) {
  return launch_cg2(tc, false, Zhat, nullptr, pb, P, tm_off, img_keys, pair_keys, n_tm_local, land, s);
}

int launch_step3_cg2(const TcPlan& tc, const uint8_t* Zop, const PairBlock& pb, const DevPlan& P, int tm_off,
                     unsigned long long* img_keys, unsigned long long* pair_keys, int n_tm_local, float* land,
                     cudaStream_t s) {
  return launch_cg2(tc, true, nullptr, Zop, pb, P, tm_off, img_keys, pair_keys, n_tm_local, land, s);
}

}  // namespace ftk
