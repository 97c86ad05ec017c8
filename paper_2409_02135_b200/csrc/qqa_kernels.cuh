// qqa_kernels.cuh -- sm_100a kernels of the PQQA hot path (see include/qqa.h).
//
// Layout in HBM (one GPU holds S_local replicas of all n variables):
//   theta, m, v, p[2]  float [B][NR][SB]  replica-blocked: the S_p = B*SB local
//                      replicas are split into B column blocks of SB (a multiple
//                      of 8 = one 32-byte sector); NR = n + 1 rows per block, row
//                      n of p is all zeros (target of CSR padding entries).
//                      Row i of block b is read as SB contiguous floats by every
//                      neighbour of i -- the SpMM gather of north_star.
//   c[2]               float [n]       shift of the replica statistics
//   sums[3]            int64 [2][n]    sum_s D and sum_s D2 (fixed point 2^40)
//   colidx_pad         int32           CSR with every row padded to a multiple of
//                                      4 entries with the sentinel n (one int4 load
//                                      fetches 4 neighbour indices)
//   X                  uint32 [n][W]   rounded replicas, W = ceil(S_local/32)
//
// Work item = (block b, variable i). The step walks b in the outer loop and i
// in a grid-stride inner loop, so while the grid sweeps block b only that
// block's p (NR*SB*4 bytes, chosen <= 64 MB) is being gathered and it stays
// resident in the 126 MB L2.
//
// Lane mapping: one lane owns 8 consecutive replicas (one 256-bit access,
// ld/st.global.v8.f32, new on sm_100); LANES lanes cover an item's SB replicas
// (VPL 8-vectors per lane when SB > 256).
//
// Arithmetic: the fp32 contract of DESIGN.md §3. Every contract operation is
// written with an explicit round-to-nearest intrinsic: separate roundings as
// __fadd_rn / __fmul_rn / __fdiv_rn (which nvcc never contracts into an FMA; the
// file is also compiled with -fmad=false), and the multiply-adds the contract
// fuses as explicit __fmaf_rn (one rounding, C's fmaf in DESIGN.md §3: the
// exp / ln / cos Horner steps, the gradient, AdamW and the noise add). Adding a
// padding entry adds +0.0f to a sum that is never -0.0f (p >= 0, q starts at
// +0), which leaves it unchanged.
#pragma once
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include "qqa_sigdiv.cuh"

namespace qqa {

enum : int { kMIS = 0, kMAXCUT = 1, kMAXCLIQUE = 2, kCOLORING = 3, kMAXCLIQUE_SPARSE = 4 };
// Step-kernel mode (template): bit 0 = clamp map (Eq. 11),
// bit 1 = Langevin noise (Eq. 9 / 11), bit 2 = the printed clique relaxation on
// the original graph (per-replica column sums enter the objective), bit 3 = edge weights
// (q_i = sum_j w_ij p_j as fl(q + fl(w p)) in CSR order; MIS and Max-Cut).
enum : int { kModeClamp = 1, kModeNoise = 2, kModeSparseClique = 4, kModeWeighted = 8 };

// Kernels with VPL >= 2 vectors per lane (S_p > 256, e.g. c4's S = 512) gather each round of 4 neighbour
// rows as two halves of 2 rows, which takes them from 121 to 80 registers and 2 to 3 CTAs per SM
// (c4: 137.4 -> 128.1 us per step, same CSR-order adds; profiles/r2_ab_c4_half_rounds.txt).
#ifndef QQA_VPL2_HALF
#define QQA_VPL2_HALF 1        // 0: the round-1 gather (4 rows x VPL vectors in registers)
#endif
#ifndef QQA_VPL2_MINB
#define QQA_VPL2_MINB 3        // min CTAs per SM of the VPL = 2 kernels (2 with QQA_VPL2_HALF=0; VPL = 4: 2)
#endif
#ifndef QQA_GATHER_U
#define QQA_GATHER_U 4         // neighbour rows in flight per lane (multiple of 4)
#endif
#ifndef QQA_STEP_MIN_BLOCKS
#define QQA_STEP_MIN_BLOCKS 4  // 4 x 256 threads per SM when VPL = 1: <= 64 registers per thread
#endif

// ----------------------------------------------------------- contract math
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }

// exp(-a) for 0 <= a <= 87: a = k ln2 + r (Cody-Waite), exp(r) by the degree-7
// Taylor polynomial in Horner form, times 2^k built from bits. Reduction and Horner steps are
// explicit fused multiply-adds (__fmaf_rn == C fmaf, one rounding; DESIGN.md §3 item 2).
__device__ __forceinline__ float exp_neg_c(float a) {
  const float x = -a;
  const float kf = rintf(fmul(x, 1.44269504088896341f));
  const float r = __fmaf_rn(-kf, 1.428606765330187e-6f, __fmaf_rn(-kf, 0.693145751953125f, x));
  float P = 1.0f / 5040.0f;
  P = __fmaf_rn(P, r, 1.0f / 720.0f);
  P = __fmaf_rn(P, r, 1.0f / 120.0f);
  P = __fmaf_rn(P, r, 1.0f / 24.0f);
  P = __fmaf_rn(P, r, 1.0f / 6.0f);
  P = __fmaf_rn(P, r, 0.5f);
  P = __fmaf_rn(P, r, 1.0f);
  P = __fmaf_rn(P, r, 1.0f);
  return fmul(P, __int_as_float((static_cast<int>(kf) + 127) << 23));
}

// p = sigmoid(theta): 1/(1+E) for theta >= 0, E/(1+E) otherwise, E = exp(-|theta|).
__device__ __forceinline__ float sigmoid_c(float th) {
  const float a = fabsf(th);
  const float Ec = exp_neg_c(fminf(a, 87.0f));     // evaluated unconditionally (no branch)
  const float E = (a > 87.0f) ? 0.0f : Ec;
  const float den = fadd(1.0f, E);
  return sig_div((th >= 0.0f) ? 1.0f : E, den);   // one division (the numerator is selected, not the quotient);
                                                  // = __fdiv_rn for every reachable operand (qqa_sigdiv.cuh)
}

// Clamp(w) into [0, 1]; NaN and -0 map to +0 (non-finite is flagged first).
__device__ __forceinline__ float clamp01(float w) { return (w > 0.0f) ? ((w < 1.0f) ? w : 1.0f) : 0.0f; }

// ln(u), u in (0, 1]: u = 2^e m, m in [sqrt(1/2), sqrt(2)), f = m - 1 (exact),
// s = f/(2+f), ln m = 2 s (1 + s^2/3 + s^4/5 + s^6/7 + s^8/9), ln u = (e ln2_hi + ln m) + e ln2_lo.
__device__ __forceinline__ float ln_c(float u) {
  const uint32_t b = __float_as_uint(u);
  int e = (int)((b >> 23) & 0xffu) - 127;
  float m = __uint_as_float((b & 0x007fffffu) | 0x3f800000u);
  if (m > 1.41421356f) { m = fmul(m, 0.5f); e = e + 1; }
  const float f = fsub(m, 1.0f);
  const float sv = sig_div(f, fadd(2.0f, f));   // divisor in [1.70, 2.42]: = __fdiv_rn for every f (qqa_sigdiv.cuh)
  const float z = fmul(sv, sv);
  float P = 1.0f / 9.0f;   // Horner steps as __fmaf_rn (== C fmaf)
  P = __fmaf_rn(P, z, 1.0f / 7.0f);
  P = __fmaf_rn(P, z, 1.0f / 5.0f);
  P = __fmaf_rn(P, z, 1.0f / 3.0f);
  P = __fmaf_rn(P, z, 1.0f);
  const float lnm = fmul(2.0f, fmul(sv, P));
  const float ef = (float)e;
  return fadd(fadd(fmul(ef, 0.693145751953125f), lnm), fmul(ef, 1.428606765330187e-6f));
}

// cos(2 pi x) and sin(2 pi x), x in [0, 1): quadrant k = rint(4x), a = (4x - k) pi/2 in
// [-pi/4, pi/4], Taylor cos a (to a^8) / sin a (to a^9).
__device__ __forceinline__ void cossin2pi_c(float x, float& cs, float& sn) {
  const float y = fmul(4.0f, x);
  const float k = rintf(y);
  const float r = fsub(y, k);
  const float a = fmul(r, 1.57079632679489662f);
  const float a2 = fmul(a, a);
  float C = 1.0f / 40320.0f;   // Horner steps as __fmaf_rn (== C fmaf)
  C = __fmaf_rn(C, a2, -(1.0f / 720.0f));
  C = __fmaf_rn(C, a2, 1.0f / 24.0f);
  C = __fmaf_rn(C, a2, -0.5f);
  C = __fmaf_rn(C, a2, 1.0f);
  float Sn = 1.0f / 362880.0f;
  Sn = __fmaf_rn(Sn, a2, -(1.0f / 5040.0f));
  Sn = __fmaf_rn(Sn, a2, 1.0f / 120.0f);
  Sn = __fmaf_rn(Sn, a2, -(1.0f / 6.0f));
  Sn = __fmaf_rn(Sn, a2, 1.0f);
  Sn = fmul(Sn, a);
  const int q = ((int)k) & 3;
  cs = (q == 0) ? C : (q == 1) ? -Sn : (q == 2) ? -C : Sn;
  sn = (q == 0) ? Sn : (q == 1) ? C : (q == 2) ? -Sn : -C;
}

// Replica mean / population STD of one variable from its fixed-point sums.
__device__ __forceinline__ void finalize_stats(float c, long long sD, long long sD2, double S,
                                               float& mu, float& sd) {
  const double md = __ddiv_rn(__dmul_rn(__ll2double_rn(sD), 0x1p-40), S);
  mu = __double2float_rn(__dadd_rn((double)c, md));
  const double ex2 = __ddiv_rn(__dmul_rn(__ll2double_rn(sD2), 0x1p-40), S);
  const double var = __dsub_rn(ex2, __dmul_rn(md, md));
  sd = __double2float_rn(__dsqrt_rn(var > 0.0 ? var : 0.0));
}

// Fixed-point terms of one replica value: D = rint((p-c) 2^40), D2 = rint(fl((p-c)^2) 2^40).
__device__ __forceinline__ void stat_terms(float p, float c, long long& D, long long& D2) {
  const float d = fsub(p, c);
  D = __float2ll_rn(fmul(d, 0x1p40f));
  D2 = __float2ll_rn(fmul(fmul(d, d), 0x1p40f));
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Two independent N(0,1) from one hash by Box-Muller: u1 = (h>>40 + 1) 2^-24 in (0,1],
// u2 = ((h>>16) & 0xFFFFFF) 2^-24 in [0,1), r = sqrt(-2 ln u1); zc = r cos(2 pi u2), zs = r sin(2 pi u2).
__device__ __forceinline__ void gauss_pair_c(uint64_t h, float& zc, float& zs) {
  const float u1 = fmul(__ull2float_rn((h >> 40) + 1ull), 0x1p-24f);
  const float u2 = fmul(__ull2float_rn((h >> 16) & 0xFFFFFFull), 0x1p-24f);
  const float r = __fsqrt_rn(fmul(-2.0f, ln_c(u1)));
  float c, sn;
  cossin2pi_c(u2, c, sn);
  zc = fmul(r, c);
  zs = fmul(r, sn);
}

// The noise of global replica sg from the row key rk: replicas pair up (sg even, sg + 1) on
// mix64(rk + sg_even); the even one takes the cos half, the odd one the sin half (reading R24).
__device__ __forceinline__ float noise_of(unsigned long long rk, int sg) {
  float zc, zs;
  gauss_pair_c(mix64(rk + (unsigned long long)(sg & ~1)), zc, zs);
  return (sg & 1) ? zs : zc;
}

// ------------------------------------------------------ 256-bit accesses
struct V8 {
  float f[8];
};

// acc += b on 8 floats as 4 packed FADD2 (sm_100 add.rn.f32x2: per component exactly __fadd_rn).
// Only pure add chains use packed ops: ptxas 12.9 contracts mul.rn.f32x2 -> add.rn.f32x2 into FFMA2
// even with -fmad=false, which would break the contract.
__device__ __forceinline__ void add8(V8& acc, const V8& b) {
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const float2 r = __fadd2_rn(make_float2(acc.f[k], acc.f[k + 1]), make_float2(b.f[k], b.f[k + 1]));
    acc.f[k] = r.x;
    acc.f[k + 1] = r.y;
  }
}

__device__ __forceinline__ V8 zero8() {
  V8 r;
#pragma unroll
  for (int k = 0; k < 8; ++k) r.f[k] = 0.0f;
  return r;
}

#define QQA_V8_OUT(r) "=f"(r.f[0]), "=f"(r.f[1]), "=f"(r.f[2]), "=f"(r.f[3]), \
                      "=f"(r.f[4]), "=f"(r.f[5]), "=f"(r.f[6]), "=f"(r.f[7])
#define QQA_V8_IN(v) "f"(v.f[0]), "f"(v.f[1]), "f"(v.f[2]), "f"(v.f[3]), \
                     "f"(v.f[4]), "f"(v.f[5]), "f"(v.f[6]), "f"(v.f[7])

// L2 policies (compile-time; measured in profiles/r1_design_iterations.md):
//   QQA_GATHER_POLICY 0: gathered p rows evict_last, 1: evict_normal, 2: evict_last + L1::no_allocate,
//                     3: ld.global.cg (L2 only) evict_last
//   QQA_PNEXT_POLICY  0: p_next stored evict_normal, 1: evict_last (next step's gather source),
//                     2: evict_first (streamed like theta / m / v)
//   QQA_INDEX_POLICY  0: CSR indices through the default path, 1: streamed (L1::no_allocate, L2 evict_first),
//                     2: L1-allocating, L2 evict_first
#ifndef QQA_GATHER_POLICY
#define QQA_GATHER_POLICY 0
#endif
#ifndef QQA_PNEXT_POLICY
#define QQA_PNEXT_POLICY 0
#endif
#ifndef QQA_INDEX_POLICY
#define QQA_INDEX_POLICY 0
#endif
// 1: the sigmoid step recomputes its own p row as sigmoid(theta) instead of reading p_cur
// (bit-identical; saves N S 4 mostly L2-missing bytes per step but costs more issue than it
// saves on c5, so off -- profiles/r1_design_iterations.md). Under clamp p == theta is reused.
#ifndef QQA_RECOMPUTE_P
#define QQA_RECOMPUTE_P 0
#endif
// 1: the next round's CSR indices are loaded before this round's gathers in every kernel (software
// pipeline; the non-FULL kernels always do, see step_item; the FULL ones do not: r1 and r2 measurements)
#ifndef QQA_IDX_PIPELINE
#define QQA_IDX_PIPELINE 0
#endif

// Gathered p rows: read-only during the step, reused by every neighbour.
__device__ __forceinline__ V8 ld8_gather(const float* ptr) {
  V8 r;
#if QQA_GATHER_POLICY == 1
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : QQA_V8_OUT(r) : "l"(ptr));
#elif QQA_GATHER_POLICY == 2
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : QQA_V8_OUT(r) : "l"(ptr));
#elif QQA_GATHER_POLICY == 3
  asm volatile("ld.global.cg.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : QQA_V8_OUT(r) : "l"(ptr));
#else
  asm volatile("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : QQA_V8_OUT(r) : "l"(ptr));
#endif
  return r;
}

// Four CSR indices (read once per step).
__device__ __forceinline__ int4 ld_idx4(const int* ptr) {
#if QQA_INDEX_POLICY == 1
  int4 r;   // evict-first policy via an L2 cache hint (the qualifier form needs 256-bit accesses)
  asm volatile("{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
               " ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], pol;\n}"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr));
  return r;
#elif QQA_INDEX_POLICY == 2
  int4 r;   // L2 evict_first (the CSR streams through L2 once per replica block) but L1-allocating
  asm volatile("{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
               " ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], pol;\n}"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr));
  return r;
#else
  return __ldg(reinterpret_cast<const int4*>(ptr));
#endif
}
// theta / m / v: read once and written once per step -> first out of L2, bypass L1.
__device__ __forceinline__ V8 ld8_stream(const float* ptr) {
  V8 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : QQA_V8_OUT(r) : "l"(ptr));
  return r;
}
__device__ __forceinline__ void st8_stream(float* ptr, const V8& v) {
  asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "l"(ptr), QQA_V8_IN(v) : "memory");
}
// p_next: gathered by the next step -> normal priority.
__device__ __forceinline__ void st8(float* ptr, const V8& v) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(ptr), QQA_V8_IN(v) : "memory");
}
__device__ __forceinline__ void st8_pnext(float* ptr, const V8& v) {
#if QQA_PNEXT_POLICY == 1
  asm volatile("st.global.L2::evict_last.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(ptr), QQA_V8_IN(v) : "memory");
#elif QQA_PNEXT_POLICY == 2
  st8_stream(ptr, v);
#else
  st8(ptr, v);
#endif
}
__device__ __forceinline__ V8 ld8(const float* ptr) {
  V8 r;
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : QQA_V8_OUT(r) : "l"(ptr));
  return r;
}

// Staged state (k_step_st): the next item's theta / m / v / p vectors are copied global -> shared memory
// with cp.async (no registers held while in flight) during the current item's update, so their DRAM
// latency is hidden. Shared layout [4 vectors][2 halves][blockDim] of 16 bytes: thread t's 16-byte halves
// are consecutive across the warp (conflict-free LDS.128).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// the streamed theta / m / v: L2 evict_first, as ld8_stream (they would otherwise push gathered p rows out)
__device__ __forceinline__ void cp_async16_ef(uint32_t dst, const void* src) {
  asm volatile("{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
               " cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, pol;\n}" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void stage_v8(const float4* smem, int vec, const float* src) {
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  if (vec < 3) {   // theta, m, v
    cp_async16_ef(base + (uint32_t)(((2 * vec + 0) * nt + t) * 16), src);
    cp_async16_ef(base + (uint32_t)(((2 * vec + 1) * nt + t) * 16), src + 4);
  } else {         // p: part of the gathered block
    cp_async16(base + (uint32_t)(((2 * vec + 0) * nt + t) * 16), src);
    cp_async16(base + (uint32_t)(((2 * vec + 1) * nt + t) * 16), src + 4);
  }
}
__device__ __forceinline__ V8 unstage_v8(const float4* smem, int vec) {
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  const float4 a = smem[(2 * vec + 0) * nt + t], b = smem[(2 * vec + 1) * nt + t];
  V8 r;
  r.f[0] = a.x; r.f[1] = a.y; r.f[2] = a.z; r.f[3] = a.w; r.f[4] = b.x; r.f[5] = b.y; r.f[6] = b.z; r.f[7] = b.w;
  return r;
}

// The per-step part of a step launch: buffers of this step and its scalars.
// (A member of the kernel parameters for the launch-per-step kernel, so it stays in the
// constant bank; a register copy per step in the persistent kernel.)
struct StepVar {
  const float* p_cur;                   // [B][NR][SB]
  float* p_next;
  long long* sums_next;                 // [2][n] this rank's sums; zero on entry when B > 1
  long long* sums_zero;                 // [2][n] buffer of the step after next (zeroed here), B > 1
  float kt, st, rt;                     // -2 alpha gamma_t, lr/(1-b1^t), 1/sqrt(1-b2^t) (host double -> float)
  unsigned long long nkey;              // noise key of (t, row 0): nbase + t n S_total (binary) / + offset (K-ary)
  int rev;                              // 1: sweep the replica blocks in reverse (serpentine order over steps,
                                        // so a step starts on the block whose p the previous step wrote last)
};

// ------------------------------------------------------------ parameters
struct StepParams {
  const int* __restrict__ rowptr;       // [n+1]   original CSR (degree for Max-Cut)
  const int* __restrict__ rowptr_pad;   // [n+1]   multiples of 4
  const int* __restrict__ colidx_pad;   // padded CSR, sentinel n
  const float* __restrict__ w_pad;      // edge weights aligned with colidx_pad (0 on padding), weighted mode
  const float* __restrict__ wdeg;       // [n] weighted degree sum_j w_ij in CSR order, weighted Max-Cut
  StepVar var;                          // this step: p_cur / p_next [B][NR][SB], sums, scalars
  float* __restrict__ theta;
  float* __restrict__ m;
  float* __restrict__ v;
  const float2* __restrict__ ms;        // [n] (mu_i, STD_i) of the current p (k_finalize)
  const long long* __restrict__ colsum; // [S_p] sum_k rint(p_ks 2^40) of the current p (printed clique only)
  int* __restrict__ flag;               // bit 0: non-finite theta
  int n, SB, B, S_local;
  int off;                              // replica_offset: global index of local replica 0 (noise pairing)
  int row_begin, row_end;               // rows [row_begin, row_end) of this launch (comm overlap chunks)
  double S_total;
  int problem, alpha;
  float lam, comm, b1, c1, b2, c2, eps;
  float at;                             // 1 - lr wd (host double -> float)
  float ns;                             // Langevin scale sqrt(2 lr T) (host double -> float)
  unsigned long long S_total_u;         // key stride per row
  int blo, bhi;                         // replica blocks [blo, bhi) of a segmented-gather launch (k_seg_*)
};

// Gradient (Eq. 6/7/10 + App. D), AdamW, optional Langevin noise and
// the map for one element. MODE bit 0: clamp (the parameter th is p itself, no
// chain factor, p = Clamp(th)); otherwise p = sigmoid(th). Returns p_next; bad
// is set when the pre-map parameter is non-finite.
// The communication coefficient of a row, kc_i = -alpha_c / STD_i (0 if STD_i < 1e-6, reading R6): computed
// once per row (one division), so the per-element term of Eq. 10 is one fused multiply-add.
__device__ __forceinline__ float comm_coef(float comm, float sd) { return (sd >= 1e-6f) ? fdiv(-comm, sd) : 0.0f; }

// aux: the constant term of the objective gradient, -1 (MIS / clique-on-complement) or -deg_i (Max-Cut),
// with ok = lambda or 2 (obj_coefs); the replica's column sum T (printed clique relaxation).
template <int MODE>
__device__ __forceinline__ float update_element(const StepParams& P, const StepVar& V, float q, float ok, float aux,
                                                float pi, float mu, float kc, float& th, float& mm, float& vv,
                                                float xi, bool& bad) {
  const float e = __fmaf_rn(2.0f, pi, -1.0f);                         // 2p - 1 (2p is exact: = fl(fl(2p) - 1))
  float ep = e;
  for (int a = 2; a < P.alpha; ++a) ep = fmul(ep, e);                 // (2p-1)^(alpha-1)
  // __fmaf_rn(a, b, c) = one fused multiply-add (one rounding), C's fmaf
  // aux: the degree (Max-Cut) or the replica's column sum T (printed clique relaxation)
  // MIS / clique-on-complement: fma(lambda, q, -1); Max-Cut: fma(2, q, -deg) -- the operands (ok, oc) are
  // selected once per item by the caller (obj_coefs), the same single rounding either way
  const float obj = (MODE & kModeSparseClique) ? __fmaf_rn(P.lam, fsub(fsub(aux, 0.5f), q), -1.0f)
                                               : __fmaf_rn(ok, q, aux);
  // (obj - 2 alpha gamma (2p-1)^(alpha-1)) + (p - mu) kc: entropy and communication terms fused
  const float gp = __fmaf_rn(fsub(pi, mu), kc, __fmaf_rn(V.kt, ep, obj));
  const float g = (MODE & kModeClamp) ? gp                             // sensitive transition: d/dp
                                      : fmul(gp, fmul(pi, fsub(1.0f, pi)));  // chain rule through sigmoid
  const float t1 = fmul(th, P.at);                                    // decoupled weight decay
  mm = __fmaf_rn(P.b1, mm, fmul(P.c1, g));
  vv = __fmaf_rn(P.b2, vv, fmul(fmul(P.c2, g), g));
  const float den = __fmaf_rn(__fsqrt_rn(vv), V.rt, P.eps);
  float w = __fmaf_rn(-V.st, fdiv(mm, den), t1);
  if (MODE & kModeNoise) w = __fmaf_rn(P.ns, xi, w);                    // + sqrt(2 lr T) xi
  bad |= !isfinite(w);
  if (MODE & kModeClamp) {
    th = clamp01(w);
    return th;
  }
  th = w;
  return sigmoid_c(w);
}

// Per-element constant term of the objective gradient: oc (-1, or -deg_i for Max-Cut), or the replica's
// column sum T_s = (float)((double)C_s 2^-40) of the printed clique relaxation.
template <int MODE>
__device__ __forceinline__ float aux_of(const StepParams& P, float oc, int s) {
  if (!(MODE & kModeSparseClique)) return oc;
  return __double2float_rn(__dmul_rn(__ll2double_rn(__ldg(P.colsum + s)), 0x1p-40));
}

// (ok, oc) of obj = fma(ok, q, oc): (lambda, -1) for MIS / clique-on-complement, (2, -deg_i) for Max-Cut.
__device__ __forceinline__ void obj_coefs(const StepParams& P, float degf, float& ok, float& oc) {
  const bool cut = P.problem == kMAXCUT;
  ok = cut ? 2.0f : P.lam;
  oc = cut ? -degf : -1.0f;
}

// Fire-and-forget int64 add (exact, order-free). Inline PTX so the front end does not wrap it in its
// warp-aggregation prologue (MATCH / REDUX / VOTEU per call): the callers' lanes never share an address.
__device__ __forceinline__ void red_add_s64(long long* p, long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"((unsigned long long)v) : "memory");
}

// Reduce the group's fixed-point partial sums and publish them for variable i.
template <int LANES>
__device__ __forceinline__ void publish_sums(long long sD, long long sD2, unsigned gmask, int lane, int i, int b,
                                             int n, int B, long long* __restrict__ sums,
                                             long long* __restrict__ zero) {
#pragma unroll
  for (int off = LANES / 2; off > 0; off >>= 1) {
    sD += __shfl_xor_sync(gmask, sD, off, LANES);
    sD2 += __shfl_xor_sync(gmask, sD2, off, LANES);
  }
  if (lane == 0) {
    if (B == 1) {
      sums[i] = sD;
      sums[n + i] = sD2;
    } else {  // blocks of one variable meet here: exact, order-free integer atomics
      red_add_s64(sums + i, sD);
      red_add_s64(sums + n + i, sD2);
    }
    if (b == 0 && zero) { zero[i] = 0; zero[n + i] = 0; }
  }
}

template <int LANES>
__device__ __forceinline__ unsigned group_mask() {
  return (LANES == 32) ? 0xffffffffu : (((1u << LANES) - 1u) << ((threadIdx.x & 31) & ~(LANES - 1)));
}

#ifndef QQA_INST_ONLY   // non-template kernels: compiled once, in qqa.cu
// K0: per-variable replica mean / STD of the current p, once per step:
// (mu_i, STD_i) from the shift c_i and the (all-rank) fixed-point sums; the
// shift of the next step's sums is mu_i (written to c_next).
__global__ void k_finalize(const float* __restrict__ c_cur, const long long* __restrict__ sums, int n,
                           double S_total, float2* __restrict__ ms, float* __restrict__ c_next) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float mu, sd;
    finalize_stats(c_cur[i], sums[i], sums[n + i], S_total, mu, sd);
    ms[i] = make_float2(mu, sd);
    c_next[i] = mu;
  }
}

// K-ary: (mu, kc) per (variable, colour), kc = -alpha_c / STD (0 if STD < 1e-6): the Eq. 10 coefficient
// computed once per (i, k) and step instead of a division per element (reading R6).
__global__ void k_finalize_kc(const float* __restrict__ c_cur, const long long* __restrict__ sums, int n,
                              double S_total, float comm, float2* __restrict__ ms, float* __restrict__ c_next) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float mu, sd;
    finalize_stats(c_cur[i], sums[i], sums[n + i], S_total, mu, sd);
    ms[i] = make_float2(mu, comm_coef(comm, sd));
    c_next[i] = mu;
  }
}

#endif  // QQA_INST_ONLY

// K2: the fused step. Per item (b, i): gather q = A p over block b (4 neighbour
// rows in flight per lane, CSR-order adds; the first row initialises the sum,
// which equals 0 + row exactly since p >= +0), gradient + AdamW + sigmoid for
// the block's replicas with (mu_i, STD_i) from k_finalize, then the fixed-point
// sums of p_next (shuffles; atomics across blocks).
// One work item (replica block b, variable i) of the step: gather, update, statistics.
// FULL: every lane holds a vector of the block (SB / 8 == LANES * VPL), so the gather needs no
// per-lane guard (a compile-time variant; measured 1.7 % on c5).
// QIN (segmented gather): the sum continues a partial sum stored in the item's p_next row by the
// previous source segments; a row's neighbours ascend, so segments of ascending source ranges add them in
// CSR order and the bits equal the one-pass gather. SKIP: sentinel entries (column n, the zero row) issue no
// load (exactly +0 added). Both are compile-time: the default kernels' code is unchanged by them (SASS
// compared).
template <int LANES, int VPL, int MODE, bool FULL = false, bool STAGE = false, bool QIN = false, bool SKIP = false>
__device__ __forceinline__ void step_item(const StepParams& P, const StepVar& V, int b, int i, int lane,
                                          unsigned gmask, float mu, float sd, bool& bad, bool force_atomic = false,
                                          long long* sums_dst = nullptr, long long* zero_dst = nullptr,
                                          const float4* stage = nullptr, int nb = -1, int ni = -1,
                                          int slot_stride = 0) {
      const int SB8 = P.SB >> 3;
      const size_t blk = (size_t)b * ((size_t)P.n + 1) * P.SB;     // float offset of block b
      const float* __restrict__ pc = V.p_cur + blk;
      // ---- gather q_i over block b
      V8 acc[VPL];
      if constexpr (QIN) {   // segmented gather: continue the partial sum stored in the item's p_next row
#pragma unroll
        for (int w = 0; w < VPL; ++w) {
          const int col8 = lane + w * LANES;
          acc[w] = (FULL || col8 < SB8) ? ld8_stream(V.p_next + blk + (size_t)i * P.SB + col8 * 8) : zero8();
        }
      }
      const int e0 = __ldg(P.rowptr_pad + i), e1 = __ldg(P.rowptr_pad + i + 1);
      constexpr int U = (VPL == 1) ? QQA_GATHER_U : 4;   // neighbour rows in flight per lane
      // Index loads of round k+1 issued before round k's gathers: measured faster for the non-FULL shapes
      // (the ER batches c2 / t1, S_p = 104: -3.6 % / -2.1 %) and neutral or slower for the FULL ones (c3 +0.4 %,
      // c5 ±0.3 %; profiles/r2_ab_index_pipeline.txt), so it is compiled into the non-FULL kernels only.
      constexpr bool kIdxPipe = QQA_IDX_PIPELINE || !FULL;
      // The indices of round k+1 are loaded before the gathers of round k (software pipeline), so
      // each round waits for one memory latency, not an index load followed by the gathers.
      // Rows are padded to multiples of 4 (not of U): past the row end the sentinel row n is read.
      int4 nxt[U / 4];
#pragma unroll
      for (int u4 = 0; u4 < U / 4; ++u4)
        nxt[u4] = (e0 + 4 * u4 < e1) ? ld_idx4(P.colidx_pad + e0 + 4 * u4) : make_int4(P.n, P.n, P.n, P.n);
#if QQA_VPL2_HALF
      if constexpr (VPL >= 2 && !(MODE & kModeWeighted)) {
        // wide rows (VPL >= 2 vectors per lane): each round of 4 neighbours is gathered as two halves of 2
        // rows, so only 2 x VPL vectors are held in registers (same CSR-order adds)
        for (int e = e0; e < e1; e += 4) {
          const int js[4] = {nxt[0].x, nxt[0].y, nxt[0].z, nxt[0].w};
#pragma unroll
          for (int h = 0; h < 4; h += 2) {
            V8 buf[2][VPL];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int w = 0; w < VPL; ++w) {
                const int col8 = lane + w * LANES;
                const int col8c = (FULL || col8 < SB8) ? col8 : SB8 - 1;   // idle lanes: a duplicate, unused
                buf[u][w] = (!SKIP || js[h + u] != P.n) ? ld8_gather(pc + (size_t)js[h + u] * P.SB + col8c * 8)
                                                        : zero8();
              }
            if (h == 2) nxt[0] = (e + 4 < e1) ? ld_idx4(P.colidx_pad + e + 4) : make_int4(P.n, P.n, P.n, P.n);
#pragma unroll
            for (int w = 0; w < VPL; ++w) {
              if (!QIN && e == e0 && h == 0) acc[w] = buf[0][w]; else add8(acc[w], buf[0][w]);
              add8(acc[w], buf[1][w]);
            }
          }
        }
      } else
#endif
      for (int e = e0; e < e1; e += U) {
        int js[U];
#pragma unroll
        for (int u4 = 0; u4 < U / 4; ++u4) {
          js[4 * u4] = nxt[u4].x; js[4 * u4 + 1] = nxt[u4].y; js[4 * u4 + 2] = nxt[u4].z; js[4 * u4 + 3] = nxt[u4].w;
        }
        if constexpr (kIdxPipe) {
#pragma unroll
          for (int u4 = 0; u4 < U / 4; ++u4)
            nxt[u4] = (e + U + 4 * u4 < e1) ? ld_idx4(P.colidx_pad + e + U + 4 * u4) : make_int4(P.n, P.n, P.n, P.n);
        }
        V8 buf[U][VPL];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int w = 0; w < VPL; ++w) {
            const int col8 = lane + w * LANES;
            // lanes past the block's last vector (non-FULL shapes) load the last vector again (same sectors as
            // its owner, no extra traffic) instead of zeros: no zeroing or predication per load; their sums
            // are never used (the update skips them)
            const int col8c = (FULL || col8 < SB8) ? col8 : SB8 - 1;
            buf[u][w] = (!SKIP || js[u] != P.n) ? ld8_gather(pc + (size_t)js[u] * P.SB + col8c * 8) : zero8();
          }
        if constexpr (!kIdxPipe) {
#pragma unroll
          for (int u4 = 0; u4 < U / 4; ++u4)
            nxt[u4] = (e + U + 4 * u4 < e1) ? ld_idx4(P.colidx_pad + e + U + 4 * u4) : make_int4(P.n, P.n, P.n, P.n);
        }
        if (MODE & kModeWeighted) {   // q = fl(q + fl(w p)) in CSR order from +0 (padding: w = 0, p = 0)
          float wt[U];
#pragma unroll
          for (int u = 0; u < U; u += 4) {
            const float4 w4 = (u == 0 || e + u < e1) ? __ldg(reinterpret_cast<const float4*>(P.w_pad + e + u))
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            wt[u] = w4.x; wt[u + 1] = w4.y; wt[u + 2] = w4.z; wt[u + 3] = w4.w;
          }
          if (!QIN && e == e0) {
#pragma unroll
            for (int w = 0; w < VPL; ++w) acc[w] = zero8();
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int w = 0; w < VPL; ++w)
#pragma unroll
              for (int k = 0; k < 8; ++k) acc[w].f[k] = fadd(acc[w].f[k], fmul(wt[u], buf[u][w].f[k]));
        } else {
          if (!QIN && e == e0) {
#pragma unroll
            for (int w = 0; w < VPL; ++w) acc[w] = buf[0][w];
          } else {
#pragma unroll
            for (int w = 0; w < VPL; ++w) add8(acc[w], buf[0][w]);
          }
#pragma unroll
          for (int u = 1; u < U; ++u)
#pragma unroll
            for (int w = 0; w < VPL; ++w) add8(acc[w], buf[u][w]);
        }
      }
      if (!QIN && e0 == e1) {
#pragma unroll
        for (int w = 0; w < VPL; ++w) acc[w] = zero8();
      }

      const float degf = (P.problem != kMAXCUT) ? 0.0f
                         : (MODE & kModeWeighted) ? __ldg(P.wdeg + i)
                                                  : (float)(__ldg(P.rowptr + i + 1) - __ldg(P.rowptr + i));

      // ---- gradient, AdamW, (noise), map, statistics of p_next
      const float kc = comm_coef(P.comm, sd);   // once per item: -alpha_c / STD_i
      float ok, oc;
      obj_coefs(P, degf, ok, oc);
      long long sD = 0, sD2 = 0;
      const unsigned long long rkey = V.nkey + (unsigned long long)i * P.S_total_u;  // noise key of (t, i, replica 0)
#pragma unroll
      for (int w = 0; w < VPL; ++w) {
        const int col8 = lane + w * LANES;
        if (!FULL && col8 >= SB8) continue;
        const size_t at = blk + (size_t)i * P.SB + col8 * 8;
        V8 th, mm, vv, pp;
        if constexpr (STAGE) {   // this item's state was staged into shared memory during the previous item
          cp_async_wait_all();
          th = unstage_v8(stage, 0);
          mm = unstage_v8(stage, 1);
          vv = unstage_v8(stage, 2);
          if (!(MODE & kModeClamp)) pp = unstage_v8(stage, 3);
          if (nb >= 0) {         // stage the next item's (nb, ni) while this one updates
            const size_t an = (size_t)nb * ((size_t)P.n + 1) * P.SB + (size_t)ni * P.SB + col8 * 8;
            stage_v8(stage, 0, P.theta + an);
            stage_v8(stage, 1, P.m + an);
            stage_v8(stage, 2, P.v + an);
            if (!(MODE & kModeClamp)) stage_v8(stage, 3, V.p_cur + an);
          }
          cp_async_commit();
        } else {
          th = ld8_stream(P.theta + at);
          mm = ld8_stream(P.m + at);
          vv = ld8_stream(P.v + at);
        }
        if (STAGE && !(MODE & kModeClamp)) {
          // pp staged above
        } else if (MODE & kModeClamp) {
          pp = th;                                    // clamp map: the parameter is p
        } else if (QQA_RECOMPUTE_P) {
#pragma unroll
          for (int k = 0; k < 8; ++k) pp.f[k] = sigmoid_c(th.f[k]);   // == p_cur (same contract function)
        } else {
          pp = ld8(V.p_cur + at);
        }
        V8 pn = pp;
        const int s0 = b * P.SB + col8 * 8;          // local replica index of element 0
        if (s0 + 8 <= P.S_local && (!(MODE & kModeNoise) || ((P.off + s0) & 1) == 0)) {
#pragma unroll
          for (int k = 0; k < 8; k += 2) {            // a replica pair shares one noise hash (cos / sin halves)
            float z0 = 0.0f, z1 = 0.0f;
            if (MODE & kModeNoise) gauss_pair_c(mix64(rkey + (unsigned long long)(P.off + s0 + k)), z0, z1);
            pn.f[k] = update_element<MODE>(P, V, acc[w].f[k], ok, aux_of<MODE>(P, oc, s0 + k), pp.f[k], mu, kc,
                                           th.f[k], mm.f[k], vv.f[k], z0, bad);
            pn.f[k + 1] = update_element<MODE>(P, V, acc[w].f[k + 1], ok, aux_of<MODE>(P, oc, s0 + k + 1),
                                               pp.f[k + 1], mu, kc, th.f[k + 1], mm.f[k + 1], vv.f[k + 1], z1, bad);
            long long D, D2;
            stat_terms(pn.f[k], mu, D, D2);
            sD += D; sD2 += D2;
            stat_terms(pn.f[k + 1], mu, D, D2);
            sD += D; sD2 += D2;
          }
        } else {   // ragged last vector (padding is never updated), or an odd shard offset under noise
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (s0 + k < P.S_local) {
              const float z = (MODE & kModeNoise) ? noise_of(rkey, P.off + s0 + k) : 0.0f;
              pn.f[k] = update_element<MODE>(P, V, acc[w].f[k], ok, aux_of<MODE>(P, oc, s0 + k), pp.f[k], mu, kc,
                                             th.f[k], mm.f[k], vv.f[k], z, bad);
              long long D, D2;
              stat_terms(pn.f[k], mu, D, D2);
              sD += D; sD2 += D2;
            }
          }
        }
        st8_stream(P.theta + at, th);
        st8_stream(P.m + at, mm);
        st8_stream(P.v + at, vv);
        st8_pnext(V.p_next + at, pn);
      }
      if (slot_stride > 0)   // owner-slotted exchange: plain stores into this rank's slot at the owner (B = 1)
        publish_sums<LANES>(sD, sD2, gmask, lane, i, b, slot_stride, 1, sums_dst, nullptr);
      else if (force_atomic)   // fused exchange: the owner's buffers (atomics across ranks and blocks)
        publish_sums<LANES>(sD, sD2, gmask, lane, i, b, P.n, 2, sums_dst, zero_dst);
      else
        publish_sums<LANES>(sD, sD2, gmask, lane, i, b, P.n, P.B, V.sums_next, V.sums_zero);
}

template <int LANES, int VPL, int MODE, bool FULL>
__global__ void __launch_bounds__(256, (VPL >= 4 ? 2 : VPL >= 2 ? QQA_VPL2_MINB : QQA_STEP_MIN_BLOCKS)) k_step(const StepParams P) {
  const int lane = threadIdx.x & (LANES - 1);
  const unsigned gmask = group_mask<LANES>();
  const int group = (int)((blockIdx.x * blockDim.x + threadIdx.x) / LANES);
  const int ngroups = (int)((gridDim.x * blockDim.x) / LANES);
  bool bad = false;
  for (int bb = 0; bb < P.B; ++bb) {
    const int b = P.var.rev ? P.B - 1 - bb : bb;
    for (int i = P.row_begin + group; i < P.row_end; i += ngroups) {
      const float2 msi = P.ms[i];
      step_item<LANES, VPL, MODE, FULL>(P, P.var, b, i, lane, gmask, msi.x, msi.y, bad);
    }
  }
  if (bad) atomicOr(P.flag, 1);
}

// Segmented gather (round 2): the sources j of block b are split into KS ascending ranges
// (segments) small enough to stay in L2 while the grid sweeps all rows; launch (b, k) adds segment k's
// neighbours of every row i to the partial q_i kept in the item's p_next row (written only by this step's
// last pass of (b, i), by the same lane). k_seg_gather: segments 0..KS-2 (FIRST: segment 0 starts the
// sum); k_step_seg: the last segment followed by the whole update of k_step. The rows' neighbours are
// strictly ascending, so the adds happen in CSR order: bit-identical to k_step (test_gpu_segmented.py).
// VPL = 1, FULL shapes, unweighted modes 0-3; blocks [blo, bhi) of one launch.
// One item of a partial pass with the NEXT item's row bounds and first index quad loaded while this item
// gathers (a gather-only pass is bound by the rowptr -> index -> row chain, not by bandwidth; ncu r2).
// The sum starts from +0 (or the stored partial): 0 + x == x for the p >= +0 values added.
template <int LANES, bool QIN>
__device__ __forceinline__ V8 seg_gather_item(const StepParams& P, const StepVar& V, size_t blk, int i, int lane,
                                              int e0, int e1, int4 nxt, int in, int& e0n, int& e1n, int4& nxtn) {
  const float* __restrict__ pc = V.p_cur + blk;
  const int4 sent = make_int4(P.n, P.n, P.n, P.n);
  V8 acc = QIN ? ld8_stream(V.p_next + blk + (size_t)i * P.SB + lane * 8) : zero8();
  const bool more = in < P.row_end;
  if (more) { e0n = __ldg(P.rowptr_pad + in); e1n = __ldg(P.rowptr_pad + in + 1); }
  for (int e = e0; e < e1; e += 4) {
    const int js[4] = {nxt.x, nxt.y, nxt.z, nxt.w};
    V8 buf[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) buf[u] = (js[u] != P.n) ? ld8_gather(pc + (size_t)js[u] * P.SB + lane * 8) : zero8();
    nxt = (e + 4 < e1) ? ld_idx4(P.colidx_pad + e + 4) : sent;
    if (e == e0) nxtn = (more && e0n < e1n) ? ld_idx4(P.colidx_pad + e0n) : sent;
#pragma unroll
    for (int u = 0; u < 4; ++u) add8(acc, buf[u]);
  }
  if (e0 == e1) nxtn = (more && e0n < e1n) ? ld_idx4(P.colidx_pad + e0n) : sent;
  return acc;
}

template <int LANES, bool FIRST>
__global__ void __launch_bounds__(256, QQA_STEP_MIN_BLOCKS) k_seg_gather(const StepParams P) {
  const int lane = threadIdx.x & (LANES - 1);
  const int group = (int)((blockIdx.x * blockDim.x + threadIdx.x) / LANES);
  const int ngroups = (int)((gridDim.x * blockDim.x) / LANES);
  const int4 sent = make_int4(P.n, P.n, P.n, P.n);
  for (int b = P.blo; b < P.bhi; ++b) {
    const size_t blk = (size_t)b * ((size_t)P.n + 1) * P.SB;
    int i = P.row_begin + group, e0 = 0, e1 = 0;
    int4 nxt = sent;
    if (i < P.row_end) {
      e0 = __ldg(P.rowptr_pad + i);
      e1 = __ldg(P.rowptr_pad + i + 1);
      if (e0 < e1) nxt = ld_idx4(P.colidx_pad + e0);
    }
    while (i < P.row_end) {
      const int in = i + ngroups;
      int e0n = 0, e1n = 0;
      int4 nxtn = sent;
      const V8 acc = seg_gather_item<LANES, !FIRST>(P, P.var, blk, i, lane, e0, e1, nxt, in, e0n, e1n, nxtn);
      st8_stream(P.var.p_next + blk + (size_t)i * P.SB + lane * 8, acc);
      i = in; e0 = e0n; e1 = e1n; nxt = nxtn;
    }
  }
}

template <int LANES, int MODE>
__global__ void __launch_bounds__(256, QQA_STEP_MIN_BLOCKS) k_step_seg(const StepParams P) {
  const int lane = threadIdx.x & (LANES - 1);
  const unsigned gmask = group_mask<LANES>();
  const int group = (int)((blockIdx.x * blockDim.x + threadIdx.x) / LANES);
  const int ngroups = (int)((gridDim.x * blockDim.x) / LANES);
  bool bad = false;
  for (int b = P.blo; b < P.bhi; ++b) {
    for (int i = P.row_begin + group; i < P.row_end; i += ngroups) {
      const float2 msi = P.ms[i];
      step_item<LANES, 1, MODE, true, false, true, true>(P, P.var, b, i, lane, gmask, msi.x, msi.y, bad);
    }
  }
  if (bad) atomicOr(P.flag, 1);
}

// k_step with the staged state (VPL = 1, FULL): the same items in the same order; item k+1's theta / m / v / p
// are in flight in shared memory (cp.async) while item k updates and item k+1 gathers. Bit-identical to k_step.
// Opt-in (QQA_STAGE=1): measured slower than k_step on c5 (873 / 935 vs 812 / 813 us per step at SB = 32 / 16),
// the shared memory it needs is L1 the in-flight gathers no longer get.
template <int LANES, int MODE>
__global__ void __launch_bounds__(256, QQA_STEP_MIN_BLOCKS) k_step_st(const StepParams P) {
  extern __shared__ float4 stage_smem[];
  const int lane = threadIdx.x & (LANES - 1);
  const unsigned gmask = group_mask<LANES>();
  const int group = (int)((blockIdx.x * blockDim.x + threadIdx.x) / LANES);
  const int ngroups = (int)((gridDim.x * blockDim.x) / LANES);
  bool bad = false;
  // item sequence: block passes bb = 0..B-1 (block b = rev ? B-1-bb : bb), rows row_begin + group + k ngroups
  auto blk_of = [&](int bb) { return P.var.rev ? P.B - 1 - bb : bb; };
  int bb = 0, i = P.row_begin + group;
  if (i >= P.row_end) bb = P.B;   // no rows for this group
  if (bb < P.B) {
    const size_t a0 = (size_t)blk_of(bb) * ((size_t)P.n + 1) * P.SB + (size_t)i * P.SB + lane * 8;
    stage_v8(stage_smem, 0, P.theta + a0);
    stage_v8(stage_smem, 1, P.m + a0);
    stage_v8(stage_smem, 2, P.v + a0);
    if (!(MODE & kModeClamp)) stage_v8(stage_smem, 3, P.var.p_cur + a0);
    cp_async_commit();
  }
  while (bb < P.B) {
    int nbb = bb, ni = i + ngroups;
    if (ni >= P.row_end) { nbb = bb + 1; ni = P.row_begin + group; }
    const float2 msi = P.ms[i];
    step_item<LANES, 1, MODE, true, true>(P, P.var, blk_of(bb), i, lane, gmask, msi.x, msi.y, bad, false, nullptr,
                                          nullptr, stage_smem, nbb < P.B ? blk_of(nbb) : -1, ni);
    bb = nbb;
    i = ni;
  }
  if (bad) atomicOr(P.flag, 1);
}

// ---------------------------------------------- fused statistics exchange (G GPUs, no NCCL per step)
// Each rank owns a contiguous range of rows of the int64 statistic sums. In the step epilogue every
// rank adds its replicas' fixed-point terms of row i straight into row i of the OWNER's buffer (peer
// memory over NVLink, `atomicAdd` performed at the owner), so the exchange overlaps the step tile by
// tile; the next step reads row i's total from the owner (one 16-byte peer load per row) and finalizes
// (mu_i, STD_i) in registers. Step boundaries are a flag barrier in peer memory: the last CTA of a
// rank's step kernel (ticket counter) releases +1 into every rank's arrival counter, and a step
// kernel starts once its own counter reaches G x (barriers so far). The sums are exact integers, so
// the result is bit-identical to the NCCL all-reduce path and to one GPU.
constexpr int kMaxRanks = 8;
struct XParams {
  long long* peer_cur[kMaxRanks];       // every rank's sums buffer of this step (owner rows hold totals)
  long long* peer_next[kMaxRanks];      // every rank's sums buffer of the next step (zeroed owner rows)
  long long* zero;                      // this rank's buffer two steps ahead (owned rows zeroed here)
  unsigned long long* flag;             // this rank's arrival counter
  unsigned long long* peer_flag[kMaxRanks];
  unsigned int* ticket;                 // this rank's CTA ticket (0 between launches)
  const float* c_cur;                   // shift of the current sums (every rank keeps all rows)
  float* c_next;
  float2* ms;                           // [n] (mu, STD) of this step, written by the kernel's own pre-pass
  unsigned long long expect;            // arrivals to wait for = G x barriers before this step
  int rank, G, rows_per_rank;
  // owner-slotted exchange (k_step_xs): owner r keeps slots [2 parities][G writers][2][rpr] and totals [2][rpr]
  long long* slot_w[kMaxRanks];         // owner r's slot of THIS rank for this step's partials: [2][rpr]
  const long long* slot_r;              // this rank's slots of the previous step's partials: [G][2][rpr]
  long long* totals[kMaxRanks];         // owner r's totals [2][rpr] of the current statistics
};

__device__ __forceinline__ void x_wait_until(const XParams& X, unsigned long long expect, int* err) {
  if (threadIdx.x == 0) {
    long long spins = 0;
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(X.flag) : "memory");
      if (v >= expect) break;
      __nanosleep(128);
      if (++spins > (1ll << 25)) { atomicOr(err, 4); break; }   // a peer never arrived: report, do not hang
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void x_wait(const XParams& X, int* err) { x_wait_until(X, X.expect, err); }

__device__ __forceinline__ void x_arrive_all(const XParams& X) {
  __threadfence_system();
  for (int r = 0; r < X.G; ++r)
    asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(X.peer_flag[r]) : "memory");
}

// The last of the rank's ncta CTAs (ticket) releases this rank's arrival into every rank's counter.
__device__ __forceinline__ void x_signal(const XParams& X, unsigned ncta) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();   // this CTA's peer additions, ordered before the ticket
    const unsigned t = atomicAdd(X.ticket, 1u);
    if (t == ncta - 1) {
      *X.ticket = 0;
      x_arrive_all(X);
    }
  }
}

// One step of one rank with the fused exchange, run by the rank's CTAs cta = 0..ncta-1 (a k_step_x
// launch: blockIdx.x of gridDim.x; the one-GPU emulation k_step_x_emul: a slice of one cooperative grid).
template <int LANES, int VPL, int MODE, bool FULL>
__device__ __forceinline__ void step_x_body(const StepParams& P, const XParams& X, int cta, int ncta) {
  const int lane = threadIdx.x & (LANES - 1);
  const unsigned gmask = group_mask<LANES>();
  const int group = (int)((cta * blockDim.x + threadIdx.x) / LANES);
  const int ngroups = (int)((ncta * blockDim.x) / LANES);
  x_wait(X, P.flag);
  // Pre-pass: lane 0 of each group finalizes (mu_i, STD_i) of the group's own rows from the owners' totals
  // (the k_finalize arithmetic) into ms / c_next. The loads of all rows are independent, so their latency
  // (remote at G > 1) overlaps; the main loop then reads one float2 per item as k_step does. A 128-byte
  // line of ms holds rows of consecutive groups of this CTA, so the CTA barrier orders every write before
  // any read (c5's G = 8 shard at one rank: 148.3 -> 146.8 us per step).
  for (int i = P.row_begin + group; i < P.row_end; i += ngroups) {
    if (lane == 0) {
      const long long* sc = X.peer_cur[min(i / X.rows_per_rank, X.G - 1)];
      float mu, sd;
      finalize_stats(X.c_cur[i], sc[i], sc[P.n + i], P.S_total, mu, sd);
      X.ms[i] = make_float2(mu, sd);
      X.c_next[i] = mu;
    }
  }
  __syncthreads();
  bool bad = false;
  for (int bb = 0; bb < P.B; ++bb) {
    const int b = P.var.rev ? P.B - 1 - bb : bb;
    for (int i = P.row_begin + group; i < P.row_end; i += ngroups) {
      const int own = min(i / X.rows_per_rank, X.G - 1);
      const float2 msi = __ldcg(X.ms + i);
      step_item<LANES, VPL, MODE, FULL>(P, P.var, b, i, lane, gmask, msi.x, msi.y, bad, true, X.peer_next[own],
                                  (own == X.rank) ? X.zero : nullptr);
    }
  }
  if (bad) atomicOr(P.flag, 1);
  x_signal(X, (unsigned)ncta);
}

template <int LANES, int VPL, int MODE, bool FULL>
__global__ void __launch_bounds__(256, (VPL >= 4 ? 2 : VPL >= 2 ? QQA_VPL2_MINB : QQA_STEP_MIN_BLOCKS)) k_step_x(const StepParams P, const XParams X) {
  step_x_body<LANES, VPL, MODE, FULL>(P, X, (int)blockIdx.x, (int)gridDim.x);
}

// Owner-slotted exchange (no remote atomics; one replica block): every rank STORES its replicas' partial
// (sum D, sum D^2) of row i into its own slot at the row's owner (coalesced 8-byte stores, a warp writes
// contiguous rows); after a barrier the owner sums the G slots of its rows into totals; after a second
// barrier every rank reads row i's totals from the owner and finalizes. Slots are double-buffered by step
// parity and fully rewritten every step (nothing to zero). Bit-identical to the other exchanges (exact
// integer sums). The mid-kernel barrier needs every CTA of every rank resident: cooperative launch.
template <int LANES, int VPL, int MODE, bool FULL>
__device__ __forceinline__ void step_xs_body(const StepParams& P, const XParams& X, int cta, int ncta) {
  const int lane = threadIdx.x & (LANES - 1);
  const unsigned gmask = group_mask<LANES>();
  const int group = (int)((cta * blockDim.x + threadIdx.x) / LANES);
  const int ngroups = (int)((ncta * blockDim.x) / LANES);
  const int rpr = X.rows_per_rank;
  x_wait(X, P.flag);   // every rank's partials of the previous step are in the slots
  {                    // owner rows: totals = sum over the G writers' slots
    const int r0 = X.rank * rpr, own_n = max(0, min(rpr, P.n - r0));
    const int tid = cta * (int)blockDim.x + (int)threadIdx.x, nt = ncta * (int)blockDim.x;
    long long* tot = X.totals[X.rank];
    for (int k = tid; k < own_n; k += nt) {
      long long s0 = 0, s1 = 0;
      for (int q = 0; q < X.G; ++q) {
        s0 += __ldcg(X.slot_r + ((size_t)q * 2 + 0) * rpr + k);
        s1 += __ldcg(X.slot_r + ((size_t)q * 2 + 1) * rpr + k);
      }
      tot[k] = s0;
      tot[rpr + k] = s1;
    }
  }
  x_signal(X, (unsigned)ncta);
  x_wait_until(X, X.expect + (unsigned long long)X.G, P.flag);   // every owner's totals are written
  for (int i = P.row_begin + group; i < P.row_end; i += ngroups) {   // (mu, STD) of the group's rows
    if (lane == 0) {
      const int own = min(i / rpr, X.G - 1);
      const long long* tt = X.totals[own];
      const int k = i - own * rpr;
      float mu, sd;
      finalize_stats(X.c_cur[i], __ldcg(tt + k), __ldcg(tt + rpr + k), P.S_total, mu, sd);
      X.ms[i] = make_float2(mu, sd);
      X.c_next[i] = mu;
    }
  }
  __syncthreads();
  bool bad = false;
  for (int i = P.row_begin + group; i < P.row_end; i += ngroups) {
    const int own = min(i / rpr, X.G - 1);
    const float2 msi = __ldcg(X.ms + i);
    step_item<LANES, VPL, MODE, FULL>(P, P.var, 0, i, lane, gmask, msi.x, msi.y, bad, false,
                                      X.slot_w[own] - (size_t)own * rpr, nullptr, nullptr, -1, -1, rpr);
  }
  if (bad) atomicOr(P.flag, 1);
  x_signal(X, (unsigned)ncta);
}

template <int LANES, int VPL, int MODE, bool FULL>
__global__ void __launch_bounds__(256, (VPL >= 4 ? 2 : VPL >= 2 ? QQA_VPL2_MINB : QQA_STEP_MIN_BLOCKS)) k_step_xs(const StepParams P, const XParams X) {
  step_xs_body<LANES, VPL, MODE, FULL>(P, X, (int)blockIdx.x, (int)gridDim.x);
}

// One-GPU emulation of G ranks running the fused exchange CONCURRENTLY (test of the barrier / atomics
// protocol, qqa_exchange_emulate): one cooperative launch whose grid is G slices of cta_per_rank CTAs;
// slice r runs rank r's k_step_x body for steps 0..nsteps-1 with its own parameters, so ranks really
// wait on one another's arrivals (all CTAs are co-resident). Per (step j, rank r): P = base[r] with
// var = var[j G + r], X = xp[j G + r]. The gathered p rows and peer sums of step j were written by other
// CTAs during step j-1 of this same launch; x_wait's acquire load invalidates the SM's L1 (SASS
// CCTL.IVALL) before any of them is read, as the grid barrier of the persistent k_run does.
struct XEmulParams {
  const StepParams* base;   // [G]
  const StepVar* var;       // [nsteps][G]
  const XParams* xp;        // [nsteps][G]
  int G, nsteps, cta_per_rank;
  int slotted;              // 1: the owner-slotted exchange (step_xs_body)
};

template <int LANES, int VPL, int MODE, bool FULL>
__global__ void __launch_bounds__(256, (VPL >= 4 ? 2 : VPL >= 2 ? QQA_VPL2_MINB : QQA_STEP_MIN_BLOCKS)) k_step_x_emul(const XEmulParams E) {
  const int r = (int)blockIdx.x / E.cta_per_rank, cta = (int)blockIdx.x % E.cta_per_rank;
  if (r >= E.G) return;
  for (int j = 0; j < E.nsteps; ++j) {
    StepParams P = E.base[r];
    P.var = E.var[(size_t)j * E.G + r];
    const XParams X = E.xp[(size_t)j * E.G + r];
    if (E.slotted)
      step_xs_body<LANES, VPL, MODE, FULL>(P, X, cta, E.cta_per_rank);
    else
      step_x_body<LANES, VPL, MODE, FULL>(P, X, cta, E.cta_per_rank);
  }
}

#ifndef QQA_INST_ONLY
// One barrier arrival of this rank (after the initial statistics, outside a step kernel).
__global__ void k_x_arrive(const XParams X) {
  if (threadIdx.x == 0 && blockIdx.x == 0) x_arrive_all(X);
}
// Owner-slotted exchange, initial statistics: this rank's partial sums [2][n] -> its slot at every owner.
__global__ void k_xs_scatter(const XParams X, int n, const long long* __restrict__ part) {
  const int rpr = X.rows_per_rank;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int own = min(i / rpr, X.G - 1);
    X.slot_w[own][i - own * rpr] = part[i];
    X.slot_w[own][rpr + i - own * rpr] = part[n + i];
  }
}
// Owner-slotted exchange: the current statistics (sum of the G writers' slots at each row's owner, parity of
// slot_r) -> a local [2][n] copy (qqa_get_stats); waits for the barrier that ends the last step first.
__global__ void k_xs_gather(const XParams X, int n, int par, long long* __restrict__ out, int* err) {
  x_wait(X, err);
  const int rpr = X.rows_per_rank;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int own = min(i / rpr, X.G - 1);
    const long long* s = X.totals[own] - 2 * (size_t)X.G * 2 * rpr;   // owner's slot base (totals follow the slots)
    long long s0 = 0, s1 = 0;
    for (int q = 0; q < X.G; ++q) {
      s0 += __ldcg(s + (((size_t)par * X.G + q) * 2 + 0) * rpr + (i - own * rpr));
      s1 += __ldcg(s + (((size_t)par * X.G + q) * 2 + 1) * rpr + (i - own * rpr));
    }
    out[i] = s0;
    out[n + i] = s1;
  }
}

// Owner rows of the current sums -> a local [2][n] copy (qqa_get_stats). Waits for the barrier that
// ends the last step first: until every rank has arrived, peers may still be adding into owner rows.
__global__ void k_x_gather(const XParams X, int n, long long* __restrict__ out, int* err) {
  x_wait(X, err);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const long long* sc = X.peer_cur[min(i / X.rows_per_rank, X.G - 1)];
    out[i] = sc[i];
    out[n + i] = sc[n + i];
  }
}
#endif

// Persistent form for small / L2-resident problems (one replica block, one GPU): ONE
// cooperative launch runs nsteps annealing steps with a grid barrier between them. A
// group owns the same variables every step, so (mu_i, STD_i) come from the sums the
// group itself published the step before (the k_finalize arithmetic, in registers) and
// only the gather needs the barrier. Buffers rotate exactly as the launch-per-step path
// does (p, c ping-pong; sums mod 3) and the per-step scalars come from a host-filled
// table sched[j] = (k_t, s_t, r_t, 0) of step t = t0 + j + 1, so both paths are
// bit-identical.
struct RunParams {
  StepParams P;                         // invariants (var and ms unused)
  const float4* __restrict__ sched;     // [nsteps]
  float* c[2];                          // shift of the statistics, ping-pong
  long long* sums[3];                   // [2][n] rotating
  float* p[2];
  unsigned long long nbase;             // noise stream base; key of (t, i, s) = nbase + (t n + i) S_total + s_even
  long long t0;                         // Adam steps taken before this launch
  int nsteps, cur0, scur0;
  double S_total;
  int rows_cta;                         // k_run_cluster: rows per CTA of the cluster
};

// CT (CTA threads): 1024 = one CTA per SM (32 warps) owning a CONTIGUOUS row range, so an SM
// gathers from a compact part of p (for a batch of small instances: about one instance, whose p
// rows largely stay in that SM's L1; c2 69.8 -> 57.8 us/step); 256 = 4 CTAs per SM with rows
// strided over the grid (kernels needing > 64 registers, or too little work to fill every SM).
// CT = 256 with one vector per lane runs 3 CTAs per SM (up to 85 registers: no constant reloads or spills in
// the update), measured faster than 4 x 64 registers on single-instance L2-resident problems (c3 22.8 -> 19.8
// us per step, profiles/r2_ab_run256_minb.txt).
#ifndef QQA_RUN256_MINB
#define QQA_RUN256_MINB 3
#endif
template <int LANES, int VPL, int MODE, int CT, bool FULL>
__global__ void __launch_bounds__(CT, (CT >= 512 ? 1 : (VPL >= 4 ? 2 : VPL >= 2 ? QQA_VPL2_MINB : QQA_RUN256_MINB)))
    k_run(const RunParams R) {
  namespace cg = cooperative_groups;
  const StepParams& P = R.P;
  const int lane = threadIdx.x & (LANES - 1);
  const unsigned gmask = group_mask<LANES>();
  int group, ngroups, row1;
  if (CT >= 512) {   // one CTA per SM owning contiguous rows
    const int rows_cta = (P.n + (int)gridDim.x - 1) / (int)gridDim.x;   // contiguous rows of this CTA
    const int row0 = (int)blockIdx.x * rows_cta;
    row1 = min(P.n, row0 + rows_cta);
    group = row0 + (int)(threadIdx.x / LANES);
    ngroups = (int)(blockDim.x / LANES);
  } else {
    row1 = P.n;
    group = (int)((blockIdx.x * blockDim.x + threadIdx.x) / LANES);
    ngroups = (int)((gridDim.x * blockDim.x) / LANES);
  }
  bool bad = false;
  for (int j = 0; j < R.nsteps; ++j) {
    const int a = (R.cur0 + j) & 1, sa = (R.scur0 + j) % 3, sb = (R.scur0 + j + 1) % 3;
    const float4 sc = R.sched[j];
    const unsigned long long t = (unsigned long long)(R.t0 + j + 1);
    const StepVar V{R.p[a], R.p[a ^ 1], R.sums[sb], nullptr, sc.x, sc.y, sc.z,
                    R.nbase + t * (unsigned long long)P.n * P.S_total_u};
    const long long* __restrict__ sc_cur = R.sums[sa];
    for (int i = group; i < row1; i += ngroups) {
      float mu, sd;
      finalize_stats(R.c[a][i], sc_cur[i], sc_cur[P.n + i], R.S_total, mu, sd);
      if (lane == 0) R.c[a ^ 1][i] = mu;
      step_item<LANES, VPL, MODE, FULL>(P, V, 0, i, lane, gmask, mu, sd, bad);
    }
    cg::this_grid().sync();
  }
  if (bad) atomicOr(P.flag, 1);
}

// Tiny problems (c1: n S_p = 4096): the whole anneal in ONE thread-block cluster, all state in
// shared memory. CTA r of the cluster owns rows [r R, (r+1) R) (R = rows_cta): their theta / m / v,
// both p buffers, shift and fixed-point sums live in its shared memory; a neighbour row owned by
// another CTA is read through distributed shared memory (mapa). Per step: the CTA finalizes its
// rows' (mu, STD), __syncthreads, one thread per element gathers (CSR order, skipping the trailing
// sentinel entries: + 0 leaves the sum unchanged), updates and adds its fixed-point terms into the
// row's sums (shared int64 atomics: exact, order-free), then one cluster barrier publishes p_next.
// No global memory traffic between the first load and the final write-back, no grid barrier.
// Same buffers in and out as k_run (p / c ping-pong, sums mod 3), bit-identical.
// Threads per CTA of the one-cluster anneal: 512 (up to 128 registers) measured faster than 1024 (64) and 256
// on c1 (2.2 vs 2.4 / 2.5 us per step, profiles/r2_ab_cluster_ct.txt); the element loops stride by blockDim.
#ifndef QQA_CLUSTER_CT
#define QQA_CLUSTER_CT 512
#endif
template <int MODE>
__global__ void __launch_bounds__(QQA_CLUSTER_CT, 1) k_run_cluster(const RunParams R) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const StepParams& P = R.P;
  const int RC = R.rows_cta, SP = P.SB, S = P.S_local, n = P.n;   // RC a power of two
  const int rsh = __ffs(RC) - 1;
  const int r0 = (int)cl.block_rank() * RC;
  const int nr = max(0, min(RC, n - r0));
  const int tid = threadIdx.x, nt = blockDim.x;
  extern __shared__ float4 smem_f4[];
  float* sth = reinterpret_cast<float*>(smem_f4);      // [RC][SP] each
  float* smm = sth + (size_t)RC * SP;
  float* svv = smm + (size_t)RC * SP;
  float* spb[2] = {svv + (size_t)RC * SP, svv + 2 * (size_t)RC * SP};
  long long* ssum = reinterpret_cast<long long*>(svv + 3 * (size_t)RC * SP);   // [2 buffers][2][RC]
  float* sc = reinterpret_cast<float*>(ssum + 4 * (size_t)RC);                // [RC]
  float2* sms = reinterpret_cast<float2*>(sc + ((RC + 1) & ~1));              // [RC]
  {
    const float* pg = R.p[R.cur0 & 1];
    for (int e = tid; e < nr * SP; e += nt) {
      const size_t g = (size_t)r0 * SP + e;
      sth[e] = P.theta[g]; smm[e] = P.m[g]; svv[e] = P.v[g]; spb[0][e] = pg[g];
    }
    const long long* sg = R.sums[R.scur0];
    for (int r = tid; r < nr; r += nt) {
      sc[r] = R.c[R.cur0 & 1][r0 + r];
      ssum[r] = sg[r0 + r];
      ssum[RC + r] = sg[n + r0 + r];
    }
  }
  cl.sync();
  bool bad = false;
  for (int j = 0; j < R.nsteps; ++j) {
    const float4 sch = R.sched[j];
    const unsigned long long t = (unsigned long long)(R.t0 + j + 1);
    const StepVar V{nullptr, nullptr, nullptr, nullptr, sch.x, sch.y, sch.z,
                    R.nbase + t * (unsigned long long)n * P.S_total_u};
    long long* scur = ssum + (size_t)(j & 1) * 2 * RC;
    long long* snext = ssum + (size_t)((j + 1) & 1) * 2 * RC;
    for (int r = tid; r < nr; r += nt) {   // (mu_i, STD_i) of the current p; shift of the next sums
      float mu, sd;
      finalize_stats(sc[r], scur[r], scur[RC + r], R.S_total, mu, sd);
      sms[r] = make_float2(mu, comm_coef(P.comm, sd));   // (mu_i, kc_i)
      sc[r] = mu;
      snext[r] = 0;
      snext[RC + r] = 0;
    }
    __syncthreads();
    const float* pc = spb[j & 1];
    float* pn = spb[(j + 1) & 1];
    // S a power of two <= 32: a row's S elements are S adjacent lanes of one warp (nt is a multiple
    // of 32), so its fixed-point terms are shuffle-reduced and stored by one lane; else atomics.
    const bool lanes_row = (S & (S - 1)) == 0 && S <= 32;
    for (int base = 0; base < nr * S; base += nt) {
      const int e = base + tid;
      const bool live = e < nr * S;
      const int r = live ? e / S : 0, s = e - r * S, i = r0 + r;
      long long D = 0, D2 = 0;
      if (live) {
        float q = 0.0f;   // CSR order, 4 neighbour rows per round (DSMEM loads first, then the adds);
                          // the sentinel n of the row padding contributes +0, which leaves q unchanged
        for (int k = __ldg(P.rowptr_pad + i), k1 = __ldg(P.rowptr_pad + i + 1); k < k1; k += 4) {
          const int4 j4 = __ldg(reinterpret_cast<const int4*>(P.colidx_pad + k));
          const int js[4] = {j4.x, j4.y, j4.z, j4.w};
          float vals[4];
  #pragma unroll
          for (int u = 0; u < 4; ++u)
            vals[u] = (js[u] < n) ? cl.map_shared_rank(pc, js[u] >> rsh)[(size_t)(js[u] & (RC - 1)) * SP + s] : 0.0f;
  #pragma unroll
          for (int u = 0; u < 4; ++u) q = fadd(q, vals[u]);
        }
        const int at = r * SP + s;
        const float degf = (P.problem == kMAXCUT) ? (float)(__ldg(P.rowptr + i + 1) - __ldg(P.rowptr + i)) : 0.0f;
        const float z = (MODE & kModeNoise) ? noise_of(V.nkey + (unsigned long long)i * P.S_total_u, P.off + s) : 0.0f;
        float th = sth[at], mm = smm[at], vv = svv[at];
        const float pi = (MODE & kModeClamp) ? th : pc[at];
        const float2 st = sms[r];
        float ok, oc;
        obj_coefs(P, degf, ok, oc);
        const float pv = update_element<MODE>(P, V, q, ok, oc, pi, st.x, st.y, th, mm, vv, z, bad);
        sth[at] = th; smm[at] = mm; svv[at] = vv; pn[at] = pv;
        stat_terms(pv, st.x, D, D2);
      }
      if (lanes_row) {
        for (int off = S / 2; off > 0; off >>= 1) {
          D += __shfl_xor_sync(0xffffffffu, D, off, S);
          D2 += __shfl_xor_sync(0xffffffffu, D2, off, S);
        }
        if (live && s == 0) { snext[r] = D; snext[RC + r] = D2; }
      } else if (live) {
        atomicAdd(reinterpret_cast<unsigned long long*>(snext + r), (unsigned long long)D);
        atomicAdd(reinterpret_cast<unsigned long long*>(snext + RC + r), (unsigned long long)D2);
      }
    }
    cl.sync();   // p_next of every CTA written; every read of p_cur done
  }
  {  // write back in the k_run buffer convention
    const int cf = (R.cur0 + R.nsteps) & 1;
    float* pg = R.p[cf];
    const float* pl = spb[R.nsteps & 1];
    for (int e = tid; e < nr * SP; e += nt) {
      const size_t g = (size_t)r0 * SP + e;
      P.theta[g] = sth[e]; P.m[g] = smm[e]; P.v[g] = svv[e]; pg[g] = pl[e];
    }
    long long* sg = R.sums[(R.scur0 + R.nsteps) % 3];
    const long long* sl = ssum + (size_t)(R.nsteps & 1) * 2 * RC;
    for (int r = tid; r < nr; r += nt) {
      R.c[cf][r0 + r] = sc[r];
      sg[r0 + r] = sl[r];
      sg[n + r0 + r] = sl[RC + r];
    }
  }
  if (bad) atomicOr(P.flag, 1);
}

// Shared memory of k_run_cluster for rows_cta rows of SP columns.
__host__ __device__ inline size_t cluster_smem_bytes(int rows_cta, int SP) {
  return (size_t)rows_cta * SP * 5 * sizeof(float) + (size_t)rows_cta * 4 * sizeof(long long) +
         (size_t)((rows_cta + 1) & ~1) * sizeof(float) + (size_t)rows_cta * sizeof(float2);
}

// ------------------------------------------------------------------- K1
struct InitParams {
  float* theta; float* m; float* v; float* p0; float* p1;   // [B][NR][SB]
  float* c; long long* sums;            // c[n], sums[2][n]: this rank's sums (zero on entry)
  int n, SB, B, S_local, S_total, replica_offset;
  uint64_t base;                        // mix64(seed)
  double lo, hi;
  int use_given;                        // 1: keep theta/m/v (set_state), recompute p and stats
  const float* c_given;                 // shift per row (NULL -> 1/2)
  int clamp;                            // map = clamp: the parameter is p, p_0 = 1/2 + U(lo, hi), p = theta
};

// theta_0 = lo + (hi - lo) k 2^-24, k = top 24 bits of mix64(mix64(seed) + i S_total + s_global);
// clamp map: p_0 = theta_0 = 1/2 + (lo + (hi - lo) k 2^-24), the sum in double, rounded once.
template <int LANES, int VPL>
__global__ void __launch_bounds__(256) k_init(const InitParams P) {
  const int lane = threadIdx.x & (LANES - 1);
  const unsigned gmask = group_mask<LANES>();
  const int group = (int)((blockIdx.x * blockDim.x + threadIdx.x) / LANES);
  const int ngroups = (int)((gridDim.x * blockDim.x) / LANES);
  const int SB8 = P.SB >> 3;
  const size_t NR = (size_t)P.n + 1;
  for (int b = 0; b < P.B; ++b) {
    const size_t blk = (size_t)b * NR * P.SB;
    for (int i = group; i < P.n; i += ngroups) {
      const float ci = P.c_given ? P.c_given[i] : 0.5f;
      long long sD = 0, sD2 = 0;
#pragma unroll
      for (int w = 0; w < VPL; ++w) {
        const int col8 = lane + w * LANES;
        if (col8 >= SB8) continue;
        const size_t at = blk + (size_t)i * P.SB + col8 * 8;
        V8 th = P.use_given ? ld8(P.theta + at) : zero8();
        V8 pp;
        const int s0 = b * P.SB + col8 * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int s = s0 + k;
          float t = 0.0f;
          if (s < P.S_local) {
            if (P.use_given) {
              t = th.f[k];
            } else {
              const uint64_t key = P.base + (uint64_t)i * (uint64_t)P.S_total + (uint64_t)(P.replica_offset + s);
              const uint64_t kk = mix64(key) >> 40;
              const double x = __dadd_rn(P.lo, __dmul_rn(__dmul_rn(__dsub_rn(P.hi, P.lo), (double)kk), 0x1p-24));
              t = __double2float_rn(P.clamp ? __dadd_rn(0.5, x) : x);
            }
          }
          th.f[k] = t;
          pp.f[k] = P.clamp ? t : sigmoid_c(t);
          if (s < P.S_local) {
            long long D, D2;
            stat_terms(pp.f[k], ci, D, D2);
            sD += D; sD2 += D2;
          }
        }
        st8(P.theta + at, th);
        if (!P.use_given) {
          st8(P.m + at, zero8());
          st8(P.v + at, zero8());
        }
        st8(P.p0 + at, pp);
        st8(P.p1 + at, pp);
      }
      publish_sums<LANES>(sD, sD2, gmask, lane, i, b, P.n, P.B, P.sums, nullptr);
      if (lane == 0 && b == 0) P.c[i] = ci;
    }
  }
}

#ifndef QQA_INST_ONLY   // non-template kernels: compiled once, in qqa.cu
// --------------------------------------------------------- graph checks
// Original CSR: bit 1: column out of range, bit 2: row not strictly ascending
// (unsorted / duplicate), bit 3: self-loop, bit 4: asymmetric (j's row lacks i).
// bit 5: edge between two instances of a batch (group_of_row[i] != group_of_row[j]).
// bit 6: asymmetric weights (w_ij != w_ji bitwise) or a non-finite weight.
__global__ void k_validate(const int* __restrict__ rowptr, const int* __restrict__ colidx, int n,
                           const int* __restrict__ gor, const float* __restrict__ w, int* __restrict__ flag) {
  int bad = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int e0 = rowptr[i], e1 = rowptr[i + 1];
    int prev = -1;
    for (int e = e0; e < e1; ++e) {
      const int j = colidx[e];
      if (j < 0 || j >= n) { bad |= 2; continue; }
      if (j <= prev) bad |= 4;
      if (j == i) bad |= 8;
      if (gor && gor[j] != gor[i]) bad |= 32;
      prev = j;
      int lo = rowptr[j], hi = rowptr[j + 1];
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (colidx[mid] < i) lo = mid + 1; else hi = mid;
      }
      if (lo >= rowptr[j + 1] || colidx[lo] != i) bad |= 16;
      else if (w && (__float_as_uint(w[lo]) != __float_as_uint(w[e]) || !isfinite(w[e]))) bad |= 64;
    }
  }
  if (bad) atomicOr(flag, bad);
}

// Row-padded copy of the CSR: row i occupies [rowptr_pad[i], rowptr_pad[i+1]),
// a multiple of 4 entries, the tail filled with the sentinel n (zero row of p).
// (weights: w_pad aligned with colidx_pad, 0 on padding; wdeg[i] = ((0 + w_1) + w_2) + ... in CSR order)
__global__ void k_pad_csr(const int* __restrict__ rowptr, const int* __restrict__ colidx,
                          const int* __restrict__ rowptr_pad, int* __restrict__ colidx_pad, int n,
                          const float* __restrict__ w, float* __restrict__ w_pad, float* __restrict__ wdeg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int e0 = rowptr[i], e1 = rowptr[i + 1], f0 = rowptr_pad[i], f1 = rowptr_pad[i + 1];
    for (int k = 0; k < f1 - f0; ++k) colidx_pad[f0 + k] = (e0 + k < e1) ? colidx[e0 + k] : n;
    if (w) {
      float d = 0.0f;
      for (int k = 0; k < f1 - f0; ++k) {
        const float x = (e0 + k < e1) ? w[e0 + k] : 0.0f;
        w_pad[f0 + k] = x;
        if (e0 + k < e1) d = fadd(d, x);
      }
      wdeg[i] = d;
    }
  }
}

// ---------------------------------------------------------------- K3/K4/K5
// K3: X[i][w] bit l = (theta of local replica 32w+l >= thr) for 32w+l < S_local
// (Theta(0)=1; thr = 0 for the sigmoid map, 1/2 for clamp where theta
// holds p); theta is [B][n+1][SB].
__global__ void k_pack(const float* __restrict__ theta, uint32_t* __restrict__ X, int n, int SB,
                       int S_local, int W, float thr) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long it = warp; it < (long long)n * W; it += nwarps) {
    const int i = (int)(it / W), w = (int)(it % W);
    const int s = w * 32 + lane;
    bool x = false;
    if (s < S_local) {
      const int b = s / SB, col = s - b * SB;
      x = theta[((size_t)b * (n + 1) + i) * SB + col] >= thr;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, x);
    if (lane == 0) X[it] = word;
  }
}

// K4: per-(instance, replica) integer counts; lane = replica bit of word w; each
// undirected edge once (j > i). Warp k takes word k % W and the contiguous row
// chunk [c CH, (c+1) CH), c = k / W; its partial counts are flushed (u64 atomics:
// exact, order-free) whenever the instance of the row changes (rows of one
// instance are contiguous) and at the end.
// counts[s][g][3] = (size, violations, cut), s local (the caller offsets the pointer).
// Weighted graphs (G = 1): wsums[s][2] += (sum of rint(w 2^24) over violated edges, over cut edges).
__global__ void k_eval(const int* __restrict__ rowptr, const int* __restrict__ colidx,
                       const uint32_t* __restrict__ X, const int* __restrict__ gor, int n, int W, int R, int CH,
                       int S_local, int G, unsigned long long* __restrict__ counts,
                       const float* __restrict__ wts, unsigned long long* __restrict__ wsums) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= W * R) return;
  const int w = warp % W;
  const int s = w * 32 + lane;
  const int i0 = (warp / W) * CH, i1 = min(n, i0 + CH);
  unsigned long long size = 0, viol = 0, cut = 0;
  long long wv = 0, wc = 0;
  int cur = (gor && i0 < n) ? gor[i0] : 0;
  auto flush = [&](int g) {
    if (s < S_local && (size | viol | cut)) {
      unsigned long long* c = counts + ((size_t)s * G + g) * 3;
      atomicAdd(c + 0, size);
      atomicAdd(c + 1, viol);
      atomicAdd(c + 2, cut);
    }
    size = viol = cut = 0;
  };
  for (int i = i0; i < i1; ++i) {
    if (gor) {
      const int g = gor[i];
      if (g != cur) { flush(cur); cur = g; }
    }
    const uint32_t bi = (X[(size_t)i * W + w] >> lane) & 1u;
    size += bi;
    const int e1 = rowptr[i + 1];
    for (int e = rowptr[i]; e < e1; ++e) {
      const int j = colidx[e];
      if (j <= i) continue;
      const uint32_t bj = (X[(size_t)j * W + w] >> lane) & 1u;
      viol += bi & bj;
      cut += bi ^ bj;
      if (wts) {
        const long long Wt = __float2ll_rn(fmul(__ldg(wts + e), 0x1p24f));
        wv += (bi & bj) ? Wt : 0;
        wc += (bi ^ bj) ? Wt : 0;
      }
    }
  }
  flush(cur);
  if (wts && s < S_local && (wv | wc)) {
    atomicAdd(wsums + 2 * (size_t)s + 0, (unsigned long long)wv);
    atomicAdd(wsums + 2 * (size_t)s + 1, (unsigned long long)wc);
  }
}

// Totals over instances: tot[s][c] = sum_g counts[s][g][c] (the energy of the union graph).
__global__ void k_sum_groups(const long long* __restrict__ counts, int S_total, int G, long long* __restrict__ tot) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < 3 * S_total; k += gridDim.x * blockDim.x) {
    const int s = k / 3, c = k - 3 * s;
    long long a = 0;
    for (int g = 0; g < G; ++g) a += counts[((size_t)s * G + g) * 3 + c];
    tot[k] = a;
  }
}

// K5: energies of all S_total replicas and argmin (lowest index on ties). One CTA
// per instance g = blockIdx.x: counts of replica s at counts[s stride + 3 g],
// energy[g][S_total], best[g], best_e[g] (stride = 3 G; G = 1 for the totals).
// (wsums [S_total][2], weighted graphs: the energy uses the weight sums instead of the edge counts)
__global__ void k_argmin(const long long* __restrict__ counts, int stride, int S_total, int problem, double lam,
                         double* __restrict__ energy, int* __restrict__ best, double* __restrict__ best_e,
                         const long long* __restrict__ wsums) {
  __shared__ double se[32];
  __shared__ int si[32];
  counts += 3 * (size_t)blockIdx.x;
  energy += (size_t)blockIdx.x * S_total;
  best += blockIdx.x;
  best_e += blockIdx.x;
  double be = 0.0;
  int bi = -1;
  for (int s = threadIdx.x; s < S_total; s += blockDim.x) {
    const long long* c = counts + (size_t)s * stride;
    const double viol = wsums ? __dmul_rn((double)wsums[2 * s], 0x1p-24) : (double)c[1];
    const double cut = wsums ? __dmul_rn((double)wsums[2 * s + 1], 0x1p-24) : (double)c[2];
    const double e = (problem == kMAXCUT)     ? -cut
                     : (problem == kCOLORING) ? (double)c[1]                  // conflicts
                                              : __dadd_rn(-(double)c[0], __dmul_rn(lam, viol));
    energy[s] = e;
    if (bi < 0 || e < be) { be = e; bi = s; }
  }
  // warp reduce (energy, index) with lowest index on ties
  for (int off = 16; off > 0; off >>= 1) {
    const double oe = __shfl_down_sync(0xffffffffu, be, off);
    const int oi = __shfl_down_sync(0xffffffffu, bi, off);
    if (oi >= 0 && (bi < 0 || oe < be || (oe == be && oi < bi))) { be = oe; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { se[threadIdx.x >> 5] = be; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = (blockDim.x + 31) >> 5;
    be = (threadIdx.x < nw) ? se[threadIdx.x] : 0.0;
    bi = (threadIdx.x < nw) ? si[threadIdx.x] : -1;
    for (int off = 16; off > 0; off >>= 1) {
      const double oe = __shfl_down_sync(0xffffffffu, be, off);
      const int oi = __shfl_down_sync(0xffffffffu, bi, off);
      if (oi >= 0 && (bi < 0 || oe < be || (oe == be && oi < bi))) { be = oe; bi = oi; }
    }
    if (threadIdx.x == 0) { *best = bi; *best_e = be; }
  }
}

// Printed clique relaxation: per-replica column sums C_s = sum_k rint(p_ks 2^40) (exact int64,
// order-free) of p [B][n+1][SB]. The grid-stride step T is a multiple of S_p, so a thread
// always sums the same column c = tid mod S_p and adds its partial once. out must be zero.
__global__ void k_colsum(const float* __restrict__ p, int n, int SB, int S_p, int S_local, int T,
                         unsigned long long* __restrict__ out) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= T) return;
  const int c = tid % S_p, b = c / SB, col = c - b * SB;
  if (c >= S_local) return;
  const float* __restrict__ base = p + (size_t)b * ((size_t)n + 1) * SB + col;
  long long acc = 0;
  for (long long e = tid; e < (long long)n * S_p; e += T) {
    const int r = (int)(e / S_p);
    acc += __float2ll_rn(fmul(__ldg(base + (size_t)r * SB), 0x1p40f));
  }
  if (acc) atomicAdd(out + c, (unsigned long long)acc);
}

// Printed clique relaxation evaluated on the ORIGINAL graph: k_eval's (size, edges inside x, cut)
// become the complement's (size, non-adjacent pairs inside x, non-adjacent pairs across x).
__global__ void k_clique_counts(long long* __restrict__ counts, int S, long long n) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    const long long sz = counts[3 * s];
    counts[3 * s + 1] = sz * (sz - 1) / 2 - counts[3 * s + 1];
    counts[3 * s + 2] = sz * (n - sz) - counts[3 * s + 2];
  }
}

// Loopback exchange (emulated shards on one device): acc += x over len int64 entries.
__global__ void k_add_i64(long long* __restrict__ acc, const long long* __restrict__ x, long long len) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < len; k += (long long)gridDim.x * blockDim.x)
    acc[k] += x[k];
}

// x of one local replica as bytes.
__global__ void k_extract(const uint32_t* __restrict__ X, int n, int W, int s_local, uint8_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = (uint8_t)((X[(size_t)i * W + (s_local >> 5)] >> (s_local & 31)) & 1u);
}

// Batch: row i gets x of its instance's best replica best[gor[i]] if this rank
// holds it ([off, off + S_local)), else 0 (ranks are then summed: one owner per row).
__global__ void k_extract_groups(const uint32_t* __restrict__ X, const int* __restrict__ gor,
                                 const int* __restrict__ best, int n, int W, int off, int S_local,
                                 uint8_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int s = best[gor[i]] - off;
    out[i] = (s >= 0 && s < S_local) ? (uint8_t)((X[(size_t)i * W + (s >> 5)] >> (s & 31)) & 1u) : (uint8_t)0;
  }
}

#endif  // QQA_INST_ONLY

// ======================================================== K-ary (NEXT-4)
// Graph colouring with K <= KP colours (App. B, map P:672-676, energy
// P:745-750). Layout: P[2] (ping-pong), m, v float [n][S][KP] -- replica s of
// variable i is KP contiguous floats (the K colour probabilities, padding = 0);
// statistics per (i, k): c / ms [n][K], sums int64 [2][n K]. One thread owns a
// (variable, replica) pair with all its colours in registers; a group of L lanes
// (L = min(32, pow2 >= S)) covers the replicas of one variable (replica r =
// lane + L v). The parameter is P itself: AdamW with dR/dP, (+ noise), then
// P = Clamp(P') / sum_k Clamp(P'_k) (uniform 1/K if every clamp is 0).
struct StepKParams {
  const int* __restrict__ rowptr;
  const int* __restrict__ colidx;
  const float* __restrict__ p_cur;      // [n][S][KP]
  float* __restrict__ p_next;
  float* __restrict__ m;
  float* __restrict__ v;
  const float2* __restrict__ ms;        // [n][K] (mu, STD) of the current P
  long long* __restrict__ sums_next;    // [2][n K]; zero on entry when S > L (chunk atomics)
  long long* __restrict__ sums_zero;    // [2][n K] buffer of the step after next (zeroed here)
  int* __restrict__ flag;
  int n, S, K, L;
  int kgrad;                            // 1: gradient through the map, g - <g, p> (reading R33)
  int cmaj;                             // 1: items ordered chunk-major (all variables of replica chunk 0, then
                                        // chunk 1, ...): while the grid sweeps one chunk only that chunk's
                                        // lines of P are gathered (n L KP 4 bytes), which can stay in L2
  float Kf, comm, b1, c1, b2, c2, eps, unif;   // unif = (float)(1/K)
  int alpha;
  float kt, at, st, rt, ns;
  unsigned long long nkey;              // nbase + t n K S_total + replica_offset
  unsigned long long S_total_u;
};

template <int KP>
__device__ __forceinline__ void ld_colours(const float* ptr, float (&x)[KP]) {
#pragma unroll
  for (int k = 0; k < KP; k += 4) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(ptr + k));
    x[k] = t.x; x[k + 1] = t.y; x[k + 2] = t.z; x[k + 3] = t.w;
  }
}
template <int KP>
__device__ __forceinline__ void st_colours(float* ptr, const float (&x)[KP]) {
#pragma unroll
  for (int k = 0; k < KP; k += 4) *reinterpret_cast<float4*>(ptr + k) = make_float4(x[k], x[k + 1], x[k + 2], x[k + 3]);
}

// P = Clamp(w) / Z, Z = ((c_0 + c_1) + c_2) + ... (K colours; padding stays 0).
template <int KP>
__device__ __forceinline__ void normalize_colours(float (&w)[KP], int K, float unif) {
  float Z = 0.0f;
#pragma unroll
  for (int k = 0; k < KP; ++k)
    if (k < K) Z = fadd(Z, clamp01(w[k]));
#pragma unroll
  for (int k = 0; k < KP; ++k) w[k] = (k < K) ? ((Z > 0.0f) ? fdiv(clamp01(w[k]), Z) : unif) : 0.0f;
}

// Work item = (variable i, replica chunk c): a group of L lanes (L a power of two
// in [4, 32], so a group lies inside one warp) takes replicas c L + lane. The
// fixed-point sums of a chunk are reduced by shuffles within the group and, with
// several chunks, meet in global u64 atomics (exact, order-free); chunk 0 zeroes
// the variable's entries of the buffer used two steps later.
#ifndef QQA_KARY_MINB
#define QQA_KARY_MINB 3      // min CTAs per SM for k_step_K, KP > 8 (measured: q13 0.141 -> 0.098 ms at 3)
#endif
#ifndef QQA_KARY_U_WIDE
#define QQA_KARY_U_WIDE 2    // neighbour rows in flight per lane for KP > 8
#endif
#ifndef QQA_KARY_REDUX
#define QQA_KARY_REDUX 0     // 1: k_step_K statistics of 32-lane groups by redux.sync on 32-bit halves (measured:
                             // q13 with k_step_K 97.5 -> 90.7 us, but k8 603 -> 607 us from the extra code: off)
#endif
#ifndef QQA_KARY_MINB_NARROW
#define QQA_KARY_MINB_NARROW 4   // min CTAs per SM for k_step_K, KP <= 8
#endif
// FK: K == KP (no padding colours), so the per-colour K tests compile away.
template <int KP, int MODE, bool FK = false>
__global__ void __launch_bounds__(256, (KP > 8 ? QQA_KARY_MINB : QQA_KARY_MINB_NARROW)) k_step_K(const StepKParams P) {
  constexpr int U = (KP <= 8) ? 4 : QQA_KARY_U_WIDE;     // neighbour rows in flight per lane
  const int L = P.L;
  const int lane = threadIdx.x & (L - 1);
  const int gl = threadIdx.x / L;
  const int groups_cta = blockDim.x / L;
  const int nch = (P.S + L - 1) / L;
  const long long items = (long long)P.n * nch;
  bool bad = false;
  // item it = (chunk-major) ch n + i, or (row-major) i nch + ch; the pair is advanced by the grid stride with
  // one quotient / remainder per thread instead of a 64-bit division per item
  const long long it0 = (long long)blockIdx.x * groups_cta + gl, stride = (long long)gridDim.x * groups_cta;
  const long long inner = P.cmaj ? P.n : nch;             // the fast-moving index's range
  const int sq = (int)(stride / inner), sr = (int)(stride % inner);
  int outer_ix = (int)(it0 / inner), inner_ix = (int)(it0 % inner);
  // warp-uniform trip count: the warp's groups hold consecutive items (it0 - wg is its first), so every lane
  // runs the same iterations and the statistics shuffles take the full mask (no per-call mask match); a
  // group past the end (valid = false) only joins the shuffles with zeros
  const long long wg = (threadIdx.x & 31) / L;
  for (long long it = it0; it - wg < items; it += stride) {
    const bool valid = it < items;
    const int i = P.cmaj ? inner_ix : outer_ix;
    const int ch = P.cmaj ? outer_ix : inner_ix;
    inner_ix += sr;
    outer_ix += sq;
    if (inner_ix >= inner) { inner_ix -= (int)inner; ++outer_ix; }
    const int r = ch * L + lane;
    const bool live = valid && r < P.S;
    float w[KP];                                          // the replica's new P (0 on idle lanes)
#pragma unroll
    for (int k = 0; k < KP; ++k) w[k] = 0.0f;
    if (live) {
      const int e0 = __ldg(P.rowptr + i), e1 = __ldg(P.rowptr + i + 1);
      // q_k = sum_{j in N(i)} p_j[r][k] in CSR order (U rows loaded before the adds)
      float q[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) q[k] = 0.0f;
      int e = e0;
      for (; e + U <= e1; e += U) {
        float pj[U][KP];
#pragma unroll
        for (int u = 0; u < U; ++u) ld_colours<KP>(P.p_cur + ((size_t)__ldg(P.colidx + e + u) * P.S + r) * KP, pj[u]);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < KP; k += 2) {   // packed FADD2 (pure add chain, see add8)
            const float2 r = __fadd2_rn(make_float2(q[k], q[k + 1]), make_float2(pj[u][k], pj[u][k + 1]));
            q[k] = r.x;
            q[k + 1] = r.y;
          }
      }
      for (; e < e1; ++e) {
        float pj[KP];
        ld_colours<KP>(P.p_cur + ((size_t)__ldg(P.colidx + e) * P.S + r) * KP, pj);
#pragma unroll
        for (int k = 0; k < KP; ++k) q[k] = fadd(q[k], pj[k]);
      }
      const unsigned long long rkey = P.nkey + (unsigned long long)i * (unsigned long long)P.K * P.S_total_u;
      const size_t at = ((size_t)i * P.S + r) * KP;
      float mm[KP], vv2[KP];
      ld_colours<KP>(P.p_cur + at, w);
      ld_colours<KP>(P.m + at, mm);
      ld_colours<KP>(P.v + at, vv2);
#pragma unroll
      for (int k = 0; k < KP; ++k) {              // g_k = dR/dp_k (into q[k])
        if (!FK && k >= P.K) continue;
        const float pi = w[k];
        const float2 st = P.ms[(size_t)i * P.K + k];          // (mu, kc) of (i, k), k_finalize_kc
        const float e = fsub(fmul(P.Kf, pi), 1.0f);
        float ep = e;
        for (int a = 2; a < P.alpha; ++a) ep = fmul(ep, e);            // (K p - 1)^(alpha-1)
        q[k] = __fmaf_rn(fsub(pi, st.x), st.y, __fmaf_rn(P.kt, ep, q[k]));   // (q + entropy) + comm, fused
      }
      if (P.kgrad) {                              // through the map: g - <g, p>, <g, p> in colour order
        float gb = 0.0f;
#pragma unroll
        for (int k = 0; k < KP; ++k)
          if (FK || k < P.K) gb = fadd(gb, fmul(q[k], w[k]));
#pragma unroll
        for (int k = 0; k < KP; ++k) q[k] = fsub(q[k], gb);
      }
      float xi = 0.0f, xi_odd = 0.0f;              // colours pair up (k even, k + 1) on one noise hash
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        if (!FK && k >= P.K) continue;
        if (MODE & kModeNoise) {
          if ((k & 1) == 0)
            gauss_pair_c(mix64(rkey + (unsigned long long)k * P.S_total_u + (unsigned long long)r), xi, xi_odd);
          else
            xi = xi_odd;
        }
        const float pi = w[k];
        const float g = q[k];
        const float t1 = fmul(pi, P.at);
        mm[k] = __fmaf_rn(P.b1, mm[k], fmul(P.c1, g));
        vv2[k] = __fmaf_rn(P.b2, vv2[k], fmul(fmul(P.c2, g), g));
        const float den = __fmaf_rn(__fsqrt_rn(vv2[k]), P.rt, P.eps);
        float x = __fmaf_rn(-P.st, fdiv(mm[k], den), t1);
        if (MODE & kModeNoise) x = __fmaf_rn(P.ns, xi, x);
        bad |= !isfinite(x);
        w[k] = x;
      }
      normalize_colours<KP>(w, FK ? KP : P.K, P.unif);
      st_colours<KP>(P.m + at, mm);
      st_colours<KP>(P.v + at, vv2);
      st_colours<KP>(P.p_next + at, w);
    }
    // fixed-point statistics of the new P per colour: shuffle-reduce over the group's replicas
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (!FK && k >= P.K) continue;
      const size_t ik = (size_t)i * P.K + k, nk = (size_t)P.n * P.K;
      long long D = 0, D2 = 0;
      if (live) stat_terms(w[k], P.ms[ik].x, D, D2);
      if (QQA_KARY_REDUX && L == 32) {
        // whole-warp groups: exact sums of D, D2 as two 32-bit halves, one redux.sync each. |p - c| <= 1
        // bounds |D|, D2 by 2^40, so hi = D >> 24 (|hi| <= 2^16) and lo = D mod 2^24 summed over 32 lanes
        // fit 32 bits, and D = hi 2^24 + lo recombines exactly. (Measured: a win with the full mask, q13's
        // k_step_K 97.5 -> 90.7 us; with 8-lane group masks the redux is far slower than the shuffles, k8
        // 604 -> 803 us, so only 32-lane groups could take it; QQA_KARY_REDUX.)
        const int dh = __reduce_add_sync(0xffffffffu, (int)(D >> 24));
        const unsigned dl = __reduce_add_sync(0xffffffffu, (unsigned)(D & 0xFFFFFF));
        const int eh = __reduce_add_sync(0xffffffffu, (int)(D2 >> 24));
        const unsigned el = __reduce_add_sync(0xffffffffu, (unsigned)(D2 & 0xFFFFFF));
        D = (long long)dh * (1ll << 24) + (long long)dl;
        D2 = (long long)eh * (1ll << 24) + (long long)el;
      } else {
        for (int off = L / 2; off > 0; off >>= 1) {
          D += __shfl_xor_sync(0xffffffffu, D, off, L);
          D2 += __shfl_xor_sync(0xffffffffu, D2, off, L);
        }
      }
      if (valid && lane == (k & (L - 1))) {
        if (nch == 1) {
          P.sums_next[ik] = D;
          P.sums_next[nk + ik] = D2;
        } else {
          red_add_s64(P.sums_next + ik, D);
          red_add_s64(P.sums_next + nk + ik, D2);
          if (ch == 0) { P.sums_zero[ik] = 0; P.sums_zero[nk + ik] = 0; }
        }
      }
    }
  }
  if (bad) atomicOr(P.flag, 1);
}

// K-ary step with colour quads (KP = 12 / 16; small graphs with many replicas, e.g. queen13-13 at
// S = 1000): a thread owns 4 colours (one float4) of one replica, the 4 lanes of a replica hold its
// colours, a warp covers 8 replicas. Four times the threads of k_step_K per (variable, replica) and a
// quarter of the registers, so many more gathers are in flight. Same arithmetic: CSR-order float4
// gather, the per-colour update, the normaliser Z summed in colour order by passing the running sum
// from lane to lane, per-colour statistics reduced over the warp's 8 replicas (u64 atomics across
// chunks). Bit-identical to k_step_K.
// KP = 8 runs the same kernel with 2 lanes per replica (2 quads): a warp then holds two work items
// (two variables of one 8-replica chunk), 16 lanes each.
constexpr int kQuadReps = 8;   // replicas per work item (chunk)
template <int KP> __host__ __device__ constexpr int quad_lanes() { return KP <= 8 ? 2 : 4; }   // lanes per replica
template <int KP> __host__ __device__ constexpr int quad_reps() { return 32 / quad_lanes<KP>(); }   // replicas per warp
#ifndef QQA_KQ_U
#define QQA_KQ_U 4               // neighbour rows in flight per lane (measured: 4 at 5 CTAs/SM)
#endif
#ifndef QQA_KQ_MINB
#define QQA_KQ_MINB 5
#endif
template <int KP, int MODE>
__global__ void __launch_bounds__(256, QQA_KQ_MINB) k_step_Kq(const StepKParams P) {
  constexpr int U = QQA_KQ_U;                            // neighbour rows in flight per lane
  constexpr int NQ = KP / 4;                             // quads holding colours (2, 3 or 4)
  constexpr int LPR = quad_lanes<KP>(), REPS = kQuadReps, IL = LPR * REPS, IPW = 32 / IL;   // IPW items per warp
  const int lane = threadIdx.x & 31;
  const int sub = lane / IL, li = lane & (IL - 1);      // item of the warp, lane within the item
  const int rq = li / LPR, q = li & (LPR - 1);          // replica in the chunk, colour quad
  const int warps_cta = blockDim.x >> 5;
  const int nch = (P.S + REPS - 1) / REPS;
  const long long items = (long long)P.n * nch;
  bool bad = false;
  for (long long itw = (long long)blockIdx.x * warps_cta + (threadIdx.x >> 5); itw * IPW < items;
       itw += (long long)gridDim.x * warps_cta) {       // warp-uniform trip count: shuffles take the full mask
    const long long it = itw * IPW + sub;
    int i = 0, ch = P.S;                                 // past the end: no live replica
    if (it < items) {
      if (P.cmaj) { ch = (int)(it / P.n); i = (int)(it - (long long)ch * P.n); }
      else { i = (int)(it / nch); ch = (int)(it - (long long)i * nch); }
    }
    const int r = ch * REPS + rq;
    const bool rep = r < P.S;                            // a live replica (all LPR lanes)
    const bool live = rep && q < NQ;                     // ... and a quad holding colours
    const int k0 = 4 * q;
    float w[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    float cl4[4] = {0.0f, 0.0f, 0.0f, 0.0f};             // Clamp(w) of this quad's colours
    float mm[4], vv2[4];
    float qv[4] = {0.0f, 0.0f, 0.0f, 0.0f};             // q, then the gradient g of this quad's colours
    size_t at = 0;
    if (live) {
      const int e0 = __ldg(P.rowptr + i), e1 = __ldg(P.rowptr + i + 1);
      float4 qa = make_float4(0.0f, 0.0f, 0.0f, 0.0f);   // q_k = sum_j p_j[r][k], CSR order
      const float* base = P.p_cur + (size_t)r * KP + k0;
      int e = e0;
      for (; e + U <= e1; e += U) {
        float4 pj[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          pj[u] = __ldg(reinterpret_cast<const float4*>(base + (size_t)__ldg(P.colidx + e + u) * P.S * KP));
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float2 lo = __fadd2_rn(make_float2(qa.x, qa.y), make_float2(pj[u].x, pj[u].y));
          const float2 hi = __fadd2_rn(make_float2(qa.z, qa.w), make_float2(pj[u].z, pj[u].w));
          qa = make_float4(lo.x, lo.y, hi.x, hi.y);
        }
      }
      for (; e < e1; ++e) {
        const float4 pj = __ldg(reinterpret_cast<const float4*>(base + (size_t)__ldg(P.colidx + e) * P.S * KP));
        qa = make_float4(fadd(qa.x, pj.x), fadd(qa.y, pj.y), fadd(qa.z, pj.z), fadd(qa.w, pj.w));
      }
      qv[0] = qa.x; qv[1] = qa.y; qv[2] = qa.z; qv[3] = qa.w;
      at = ((size_t)i * P.S + r) * KP + k0;
      const float4 w4 = *reinterpret_cast<const float4*>(P.p_cur + at);
      const float4 m4 = *reinterpret_cast<const float4*>(P.m + at);
      const float4 v4 = *reinterpret_cast<const float4*>(P.v + at);
      w[0] = w4.x; w[1] = w4.y; w[2] = w4.z; w[3] = w4.w;
      mm[0] = m4.x; mm[1] = m4.y; mm[2] = m4.z; mm[3] = m4.w;
      vv2[0] = v4.x; vv2[1] = v4.y; vv2[2] = v4.z; vv2[3] = v4.w;
#pragma unroll
      for (int c = 0; c < 4; ++c) {               // g_k = dR/dp_k (into qv[c])
        const int k = k0 + c;
        if (k >= P.K) continue;
        const float pi = w[c];
        const float2 st = P.ms[(size_t)i * P.K + k];          // (mu, kc) of (i, k), k_finalize_kc
        const float e1f = fsub(fmul(P.Kf, pi), 1.0f);
        float ep = e1f;
        for (int a = 2; a < P.alpha; ++a) ep = fmul(ep, e1f);          // (K p - 1)^(alpha-1)
        qv[c] = __fmaf_rn(fsub(pi, st.x), st.y, __fmaf_rn(P.kt, ep, qv[c]));   // (q + entropy) + comm, fused
      }
    }
    // through the map (reading R33): g - <g, p>, <g, p> summed in colour order -- the running sum
    // passes from quad to quad as the normaliser's does below
    if (P.kgrad) {
      float gb = 0.0f;
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq) {
        if (q == qq && live)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (k0 + c < P.K) gb = fadd(gb, fmul(qv[c], w[c]));
        gb = __shfl_sync(0xffffffffu, gb, (lane & ~(LPR - 1)) + qq);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) qv[c] = fsub(qv[c], gb);
    }
    if (live) {
      const unsigned long long rkey = P.nkey + (unsigned long long)i * (unsigned long long)P.K * P.S_total_u;
      float xi = 0.0f, xi_odd = 0.0f;                    // colours pair up (k even, k + 1) on one noise hash
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int k = k0 + c;
        if (k >= P.K) continue;
        if (MODE & kModeNoise) {
          if ((c & 1) == 0)
            gauss_pair_c(mix64(rkey + (unsigned long long)k * P.S_total_u + (unsigned long long)r), xi, xi_odd);
          else
            xi = xi_odd;
        }
        const float pi = w[c];
        const float g = qv[c];
        const float t1 = fmul(pi, P.at);
        mm[c] = __fmaf_rn(P.b1, mm[c], fmul(P.c1, g));
        vv2[c] = __fmaf_rn(P.b2, vv2[c], fmul(fmul(P.c2, g), g));
        const float den = __fmaf_rn(__fsqrt_rn(vv2[c]), P.rt, P.eps);
        float x = __fmaf_rn(-P.st, fdiv(mm[c], den), t1);
        if (MODE & kModeNoise) x = __fmaf_rn(P.ns, xi, x);
        bad |= !isfinite(x);
        w[c] = x;
        cl4[c] = clamp01(x);
      }
    }
    // Z = ((c_0 + c_1) + c_2) + ... over the K colours in order: the running sum passes from quad to quad
    float Z = 0.0f;
#pragma unroll
    for (int qq = 0; qq < NQ; ++qq) {
      if (q == qq)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (k0 + c < P.K) Z = fadd(Z, cl4[c]);
      Z = __shfl_sync(0xffffffffu, Z, (lane & ~(LPR - 1)) + qq);
    }
    if (live) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        w[c] = (k0 + c < P.K) ? ((Z > 0.0f) ? fdiv(cl4[c], Z) : P.unif) : 0.0f;
      *reinterpret_cast<float4*>(P.m + at) = make_float4(mm[0], mm[1], mm[2], mm[3]);
      *reinterpret_cast<float4*>(P.v + at) = make_float4(vv2[0], vv2[1], vv2[2], vv2[3]);
      *reinterpret_cast<float4*>(P.p_next + at) = make_float4(w[0], w[1], w[2], w[3]);
    }
    // fixed-point statistics per colour: reduce over the warp's replicas (lanes of the same quad)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int k = k0 + c;
      long long D = 0, D2 = 0;
      if (live && k < P.K) stat_terms(w[c], P.ms[(size_t)i * P.K + k].x, D, D2);
#pragma unroll
      for (int off = LPR; off < IL; off <<= 1) {
        D += __shfl_xor_sync(0xffffffffu, D, off);
        D2 += __shfl_xor_sync(0xffffffffu, D2, off);
      }
      if (rq == 0 && q < NQ && k < P.K && it < items) {
        const size_t ik = (size_t)i * P.K + k, nk = (size_t)P.n * P.K;
        if (nch == 1) {
          P.sums_next[ik] = D;
          P.sums_next[nk + ik] = D2;
        } else {
          red_add_s64(P.sums_next + ik, D);
          red_add_s64(P.sums_next + nk + ik, D2);
          if (ch == 0) { P.sums_zero[ik] = 0; P.sums_zero[nk + ik] = 0; }
        }
      }
    }
  }
  if (bad) atomicOr(P.flag, 1);
}

// K1 for K-ary: W_0 = 1/K + U(lo, hi) keyed (seed, i K + k, global s), P_0 = normalise(W_0),
// m = v = 0; or (use_given) P_0 as given. Sums of P_0 with shift c (1/K or c_given), u64 atomics.
struct InitKParams {
  float* p0; float* p1; float* m; float* v;
  float* c; long long* sums;            // c[n K], sums[2][n K] (zero on entry)
  int n, S, K, S_total, replica_offset;
  uint64_t base;
  double lo, hi;
  float unif;
  int use_given;
  const float* c_given;
};

template <int KP>
__global__ void __launch_bounds__(256) k_init_K(const InitKParams P) {
  const long long total = (long long)P.n * P.S;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < total;
       it += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(it / P.S), r = (int)(it % P.S);
    const size_t at = (size_t)it * KP;
    float w[KP];
    if (P.use_given) {
      ld_colours<KP>(P.p0 + at, w);
    } else {
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        w[k] = 0.0f;
        if (k < P.K) {
          const uint64_t key = P.base + ((uint64_t)i * (uint64_t)P.K + (uint64_t)k) * (uint64_t)P.S_total +
                               (uint64_t)(P.replica_offset + r);
          const uint64_t kk = mix64(key) >> 40;
          const double u = __dadd_rn(P.lo, __dmul_rn(__dmul_rn(__dsub_rn(P.hi, P.lo), (double)kk), 0x1p-24));
          w[k] = __double2float_rn(__dadd_rn(__ddiv_rn(1.0, (double)P.K), u));
        }
      }
      normalize_colours<KP>(w, P.K, P.unif);
      float z[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) z[k] = 0.0f;
      st_colours<KP>(P.p0 + at, w);
      st_colours<KP>(P.m + at, z);
      st_colours<KP>(P.v + at, z);
    }
    st_colours<KP>(P.p1 + at, w);
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (k >= P.K) continue;
      const size_t ik = (size_t)i * P.K + k;
      const float ci = P.c_given ? P.c_given[ik] : P.unif;
      long long D, D2;
      stat_terms(w[k], ci, D, D2);
      atomicAdd(reinterpret_cast<unsigned long long*>(P.sums + ik), (unsigned long long)D);
      atomicAdd(reinterpret_cast<unsigned long long*>(P.sums + (size_t)P.n * P.K + ik), (unsigned long long)D2);
      if (r == 0) P.c[ik] = ci;
    }
  }
}

// K3 for K-ary: X8[i][s] = argmax_k P[i][s][k] (lowest k on ties).
template <int KP>
__global__ void k_pack_K(const float* __restrict__ Pm, uint8_t* __restrict__ X8, int n, int S, int K) {
  const long long total = (long long)n * S;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < total;
       it += (long long)gridDim.x * blockDim.x) {
    float w[KP];
    ld_colours<KP>(Pm + (size_t)it * KP, w);
    int b = 0;
#pragma unroll
    for (int k = 1; k < KP; ++k)
      if (k < K && w[k] > w[b]) b = k;
    X8[it] = (uint8_t)b;
  }
}

#ifndef QQA_INST_ONLY   // non-template kernels: compiled once, in qqa.cu
// K4 for K-ary: conflicts per replica; lane = replica 32 w + lane, warp k takes word k % W and the
// row chunk [c CH, (c+1) CH), c = k / W. counts[s][3] = (0, conflicts, |E| - conflicts) (the last
// term is added by the host-known |E| in k_conflicts_finish).
__global__ void k_eval_K(const int* __restrict__ rowptr, const int* __restrict__ colidx,
                         const uint8_t* __restrict__ X8, int n, int S, int W, int R, int CH,
                         unsigned long long* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= W * R) return;
  const int s = (warp % W) * 32 + lane;
  if (s >= S) return;
  const int i0 = (warp / W) * CH, i1 = min(n, i0 + CH);
  unsigned long long conf = 0;
  for (int i = i0; i < i1; ++i) {
    const uint8_t xi = X8[(size_t)i * S + s];
    const int e1 = rowptr[i + 1];
    for (int e = rowptr[i]; e < e1; ++e) {
      const int j = colidx[e];
      if (j > i) conf += (X8[(size_t)j * S + s] == xi);
    }
  }
  if (conf) atomicAdd(counts + 3 * (size_t)s + 1, conf);
}

__global__ void k_conflicts_finish(long long* __restrict__ counts, int S, long long n_edges) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x)
    counts[3 * s + 2] = n_edges - counts[3 * s + 1];
}

__global__ void k_extract_K(const uint8_t* __restrict__ X8, int n, int S, int s_local, uint8_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = X8[(size_t)i * S + s_local];
}

#endif  // QQA_INST_ONLY

}  // namespace qqa
