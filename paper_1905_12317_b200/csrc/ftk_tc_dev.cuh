// Device helpers shared by the tensor-core kernels (ftk_tc.cu, ftk_s23.cu): log-sum-exp merges, the
// lexicographic argmax comparison, TMEM loads, the Step-2 row-buffer swizzle, packed fp32x2 complex
// arithmetic and the in-register radix-2 DFT of the four-step FFT; CTA-pair (cta_group::2) primitives;
// the driver entry point of cuTensorMapEncodeTiled.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ftk_sm100.cuh"

namespace ftk {
using namespace sm100;

// fp16x3 operand scales of the tensor-core engine (ftk_tc.cu header).  ast / bst: per image / local template
// (x = max |Re|, |Im| of the FB coefficients, y = Frobenius norm); gmax = max |g_zeta(k_m)|.
// Step-1 image operand exponent and generated-operand exponent:
__device__ __forceinline__ int s1_img_exp(const float2* ast, int i) { return f16_scale_exp(__ldg(ast + i).x); }
__device__ __forceinline__ int s1_gen_exp(const float2* bst, float gmax, int j) {
  return f16_scale_exp(gmax * __ldg(bst + j).x);
}
// Step-3 Z operand exponent of pair (i, j) from its statistics a = ast[i], b = bst[j]: |Z| <= gmax |a_i| |b_j|
// (Cauchy-Schwarz over (m, p))
__device__ __forceinline__ int z_exp(float2 a, float2 b, float gmax) { return f16_scale_exp(gmax * a.y * b.y); }
// Step 1 stores pair (i, j)'s Zhat' block x 2^{s1_img_exp + s1_gen_exp}; Step 2 (and the fused kernel) move it to
// Z's scale with one exact factor
__device__ __forceinline__ float zhat_to_z_scale(float2 a, float2 b, float gmax) {
  return pow2f_wide(z_exp(a, b, gmax) - f16_scale_exp(a.x) - f16_scale_exp(gmax * b.x));
}

__device__ __forceinline__ float ex2_approx(float x) {  // 2^x, one MUFU op (2^-inf = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// (m, s) pairs of a scaled log-sum-exp in base 2: value = m + log2(s); m = -inf means "empty"
__device__ __forceinline__ void lse2_merge(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  if (mn != -INFINITY) {
    s = s * ex2_approx(m - mn) + s2 * ex2_approx(m2 - mn);
    m = mn;
  }
}

__device__ __forceinline__ bool better(float v, uint32_t f, float bv, uint32_t bf) {
  return v > bv || (v == bv && f < bf);
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
// Step-2 row buffer: [p][8 terms] complex (64-byte rows) in the TMA SWIZZLE_64B layout: the 16-byte
// chunk c of row p sits at chunk c ^ ((p >> 1) & 3), which makes the warps' column reads conflict-free.
constexpr int S2_SMAX = 8;
__device__ __forceinline__ int s2_slot(int p, int zz) {  // complex index of (row p, term zz < 8)
  return p * 8 + ((((zz >> 1) ^ (p >> 1)) & 3) << 1) + (zz & 1);
}

// packed fp32x2 arithmetic (sm_100a FADD2 / FFMA2: one instruction for both components)
__device__ __forceinline__ unsigned long long f2_u64(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 u64_f2(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u64(a)), "l"(f2_u64(b)));
  return u64_f2(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u64(a)), "l"(f2_u64(b)));
  return u64_f2(d);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_u64(a)), "l"(f2_u64(b)), "l"(f2_u64(c)));
  return u64_f2(d);
}

__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u64(a)), "l"(f2_u64(b)));
  return u64_f2(d);
}
// complex a * b as two packed instructions: t = (a.x b.x, a.x b.y), then (b.y, b.x) * (-a.y, a.y) + t.  In
// this operand order ptxas folds the broadcast, swap and sign into FMUL2 / FFMA2 operand modifiers (no MOVs;
// the scalar form takes 2 FMUL + 2 FFMA)
__device__ __forceinline__ float2 cmulf(float2 a, float2 b) {
  const float2 t = mul2(make_float2(a.x, a.x), b);
  return fma2(make_float2(b.y, b.x), make_float2(-a.y, a.y), t);
}
__device__ __forceinline__ float2 tw_full(const float2* tw, int j, int n) {  // e^{-2 pi i j / n}, 0 <= j < n
  const float2 w = __ldg(tw + (j & (n / 2 - 1)));
  return j < n / 2 ? w : make_float2(-w.x, -w.y);
}

// w_32^m = e^{-2 pi i m / 32}, m = 0..31 (cos, -sin): compile-time constants for the in-register DFTs
__device__ constexpr float kW32c[32] = {
    1.f, 0.98078528f, 0.92387953f, 0.83146961f, 0.70710678f, 0.55557023f, 0.38268343f, 0.19509032f,
    0.f, -0.19509032f, -0.38268343f, -0.55557023f, -0.70710678f, -0.83146961f, -0.92387953f, -0.98078528f,
    -1.f, -0.98078528f, -0.92387953f, -0.83146961f, -0.70710678f, -0.55557023f, -0.38268343f, -0.19509032f,
    0.f, 0.19509032f, 0.38268343f, 0.55557023f, 0.70710678f, 0.83146961f, 0.92387953f, 0.98078528f};
__device__ constexpr float kW32s[32] = {
    0.f, -0.19509032f, -0.38268343f, -0.55557023f, -0.70710678f, -0.83146961f, -0.92387953f, -0.98078528f,
    -1.f, -0.98078528f, -0.92387953f, -0.83146961f, -0.70710678f, -0.55557023f, -0.38268343f, -0.19509032f,
    0.f, 0.19509032f, 0.38268343f, 0.55557023f, 0.70710678f, 0.83146961f, 0.92387953f, 0.98078528f,
    1.f, 0.98078528f, 0.92387953f, 0.83146961f, 0.70710678f, 0.55557023f, 0.38268343f, 0.19509032f};

// x * w_32^m for a compile-time m (after unrolling): the trivial rotations cost no multiplies
__device__ __forceinline__ float2 cmul_w32(float2 x, int m) {
  m &= 31;
  if (m == 0) return x;
  if (m == 8) return make_float2(x.y, -x.x);
  if (m == 16) return make_float2(-x.x, -x.y);
  if (m == 24) return make_float2(-x.y, x.x);
  const float c = kW32c[m], sn = kW32s[m];
  // x c + (-x.y, x.x) sn: FMUL2 + FFMA2 with the constants as immediates (no MOVs; scalar form: 4 ops)
  return fma2(make_float2(sn, sn), make_float2(-x.y, x.x), mul2(make_float2(c, c), x));
}

template <int E>
__device__ __forceinline__ void dft_regs(float2 (&x)[E]) {
  // radix-2 DIT over E <= 32 points with compile-time twiddles; x is addressed in bit-reversed order
  // through rv() (a compile-time renaming), so the natural-order result ends up in x[rv(c)].
  constexpr int LOG = (E == 32) ? 5 : (E == 16) ? 4 : (E == 8 ? 3 : (E == 4 ? 2 : 1));
  auto rv = [](int i) {
    int r = 0;
#pragma unroll
    for (int bb = 0; bb < LOG; ++bb) r |= ((i >> bb) & 1) << (LOG - 1 - bb);
    return r;
  };
#pragma unroll
  for (int s = 1; s < E; s *= 2) {
#pragma unroll
    for (int blk = 0; blk < E; blk += 2 * s) {
#pragma unroll
      for (int j = 0; j < s; ++j) {
        const float2 u = x[rv(blk + j)], v = cmul_w32(x[rv(blk + j + s)], j * (32 / (2 * s)));
        x[rv(blk + j)] = add2(u, v);
        x[rv(blk + j + s)] = sub2(u, v);
      }
    }
  }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PFN_encodeTiled get_encode_tiled() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}



// ---------------------------------------------------------------- CTA pair (cluster of 2, cta_group::2)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared-memory variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// arrive on an mbarrier given by its shared::cluster address (local or peer CTA).  Default semantics
// (release, CTA scope), as in CUTLASS's cluster barriers: the data these barriers order is TMEM / shared
// memory handed between the tensor and async proxies (tcgen05 fences, mbarrier transactions).  A
// cluster-scope release / acquire would emit MEMBAR.GPU / CCTL.IVALL (an L1 invalidation) per call.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cl_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }
// 2-D TMA tile load multicast to the CTAs of ctamask (same shared-memory offset and mbarrier offset in each)
__device__ __forceinline__ void tma_load_2d_mc(void* dst_smem, const void* tmap, int x, int y, uint64_t* bar,
                                               uint16_t ctamask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst_smem)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(ctamask)
      : "memory");
}
// 1-D bulk copy global -> shared, multicast to the CTAs of ctamask (same offsets), complete_tx on each CTA's mbarrier
__device__ __forceinline__ void bulk_g2s_mc(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                            uint16_t ctamask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "h"(ctamask)
      : "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc_cg2(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc_cg2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS));
}
// D[tmem] (+)= A[tmem] * B[smem]^T over the CTA pair: M = 256 (128 rows of A / D in each CTA's TMEM), B's N
// columns split N/2 per CTA (same shared-memory offset).  Issued by one thread of the even CTA.
__device__ __forceinline__ void mma_f16_ts_cg2(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit of the pair's MMAs: one arrival on the mbarrier at this offset in both CTAs
__device__ __forceinline__ void tc_commit_cg2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

}  // namespace ftk
