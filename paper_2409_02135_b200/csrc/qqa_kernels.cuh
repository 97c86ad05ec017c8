// qqa_kernels.cuh -- sm_100a kernels of the PQQA hot path (see include/qqa.h).
//
// Layout in HBM (one GPU holds S_local replicas of all n variables):
//   theta, m, v, p[2]  float [n][S_p], S_p = S_local rounded up to 8 (one 32-B
//                      sector); row i of p is read as S_p contiguous floats by
//                      every neighbour of i -- the SpMM gather (north_star).
//   c[2]               float [n]       shift of the replica statistics
//   sums[2]            int64 [2][n]    sum_s D and sum_s D2 (fixed point 2^40)
//   X                  uint32 [n][W]   rounded replicas, W = ceil(S_local/32)
//
// Arithmetic: the fp32 contract of DESIGN.md §3. Every contract operation is
// written with an explicit round-to-nearest intrinsic (__fadd_rn, __fmul_rn,
// ...), which nvcc never contracts into FMA, and the file is compiled with
// -fmad=false as a second guard.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace qqa {

enum : int { kMIS = 0, kMAXCUT = 1, kMAXCLIQUE = 2 };

// ----------------------------------------------------------- contract math
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }

// exp(-a) for 0 <= a <= 87: a = k ln2 + r (Cody-Waite), exp(r) by the degree-7
// Taylor polynomial in Horner form, times 2^k built from bits.
__device__ __forceinline__ float exp_neg_c(float a) {
  const float x = -a;
  const float kf = rintf(fmul(x, 1.44269504088896341f));
  const float r = fsub(fsub(x, fmul(kf, 0.693145751953125f)), fmul(kf, 1.428606765330187e-6f));
  float P = 1.0f / 5040.0f;
  P = fadd(fmul(P, r), 1.0f / 720.0f);
  P = fadd(fmul(P, r), 1.0f / 120.0f);
  P = fadd(fmul(P, r), 1.0f / 24.0f);
  P = fadd(fmul(P, r), 1.0f / 6.0f);
  P = fadd(fmul(P, r), 0.5f);
  P = fadd(fmul(P, r), 1.0f);
  P = fadd(fmul(P, r), 1.0f);
  return fmul(P, __int_as_float((static_cast<int>(kf) + 127) << 23));
}

// p = sigmoid(theta): 1/(1+E) for theta >= 0, E/(1+E) otherwise, E = exp(-|theta|).
__device__ __forceinline__ float sigmoid_c(float th) {
  const float a = fabsf(th);
  const float E = (a > 87.0f) ? 0.0f : exp_neg_c(a);
  const float den = fadd(1.0f, E);
  return (th >= 0.0f) ? fdiv(1.0f, den) : fdiv(E, den);
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

__device__ __forceinline__ float comp(const float4& v, int k) {
  return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w;
}
__device__ __forceinline__ void set_comp(float4& v, int k, float x) {
  if (k == 0) v.x = x; else if (k == 1) v.y = x; else if (k == 2) v.z = x; else v.w = x;
}

// L2 cache policies (createpolicy): the theta/m/v streams are read and written
// once per step -> evict_first, so that the gathered p rows, reused by every
// neighbour, stay resident (evict_last).
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ float4 ld_stream(const float4* ptr, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_stream(float4* ptr, const float4& v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(ptr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ float4 ld_gather(const float4* ptr, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(ptr), "l"(pol));
  return r;
}

// ------------------------------------------------------------ parameters
struct StepParams {
  const int* __restrict__ rowptr;       // [n+1]
  const int* __restrict__ colidx;       // [nnz]
  const float* __restrict__ p_cur;      // [n][S_p]
  float* __restrict__ p_next;           // [n][S_p]
  float* __restrict__ theta;            // [n][S_p]
  float* __restrict__ m;
  float* __restrict__ v;
  const float* __restrict__ c_cur;      // [n]
  const long long* __restrict__ sums_cur;  // [2][n] (reduced over ranks)
  float* __restrict__ c_next;
  long long* __restrict__ sums_next;    // [2][n] (this rank's partial)
  int* __restrict__ flag;               // bit 0: non-finite theta
  int n, S_p4, S_local;
  double S_total;
  int problem, alpha;
  float lam, comm, b1, c1, b2, c2, eps;
  float kt, at, st, rt;                 // per-step scalars (host double -> float)
};

// One lane group of LANES lanes owns one variable i at a time; lane l holds the
// float4 columns l, l+LANES, ... (VPL of them). Gather: the group loads up to
// LANES neighbour indices with one coalesced load, broadcasts them with
// shuffles, and issues U neighbour-row loads before consuming them -- the sum
// itself is sequential in CSR order (contract).
template <int LANES, int VPL>
__device__ __forceinline__ void gather_row(const StepParams& P, int i, int lane, unsigned gmask,
                                           uint64_t pol, float4 (&acc)[VPL]) {
  constexpr int U = (VPL >= 8) ? 1 : (VPL >= 4 ? 2 : (VPL >= 2 ? 4 : 8));
  const float4* __restrict__ p4 = reinterpret_cast<const float4*>(P.p_cur);
  const int e0 = __ldg(P.rowptr + i), e1 = __ldg(P.rowptr + i + 1);
#pragma unroll
  for (int w = 0; w < VPL; ++w) acc[w] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int eb = e0; eb < e1; eb += LANES) {
    const int cnt = min(LANES, e1 - eb);
    const int myj = (lane < cnt) ? __ldg(P.colidx + eb + lane) : 0;
    for (int k0 = 0; k0 < cnt; k0 += U) {
      float4 buf[U][VPL];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = __shfl_sync(gmask, myj, (k0 + u) & (LANES - 1), LANES);
        if (k0 + u < cnt) {
          const float4* row = p4 + (size_t)j * P.S_p4;
#pragma unroll
          for (int w = 0; w < VPL; ++w) {
            const int col = lane + w * LANES;
            buf[u][w] = (col < P.S_p4) ? ld_gather(row + col, pol) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (k0 + u < cnt) {
#pragma unroll
          for (int w = 0; w < VPL; ++w) {
            acc[w].x = fadd(acc[w].x, buf[u][w].x);
            acc[w].y = fadd(acc[w].y, buf[u][w].y);
            acc[w].z = fadd(acc[w].z, buf[u][w].z);
            acc[w].w = fadd(acc[w].w, buf[u][w].w);
          }
        }
      }
    }
  }
}

// Gradient (Eq. 6/7/10 + App. D), AdamW and sigmoid for one element.
__device__ __forceinline__ float update_element(const StepParams& P, float q, float degf, float pi,
                                                float mu, float sd, float& th, float& mm, float& vv) {
  const float e = fsub(fmul(2.0f, pi), 1.0f);
  float ep = e;
  for (int a = 2; a < P.alpha; ++a) ep = fmul(ep, e);                 // (2p-1)^(alpha-1)
  const float ent = fmul(P.kt, ep);                                   // -2 alpha gamma (2p-1)^(alpha-1)
  const float obj = (P.problem == kMAXCUT) ? fsub(fmul(2.0f, q), degf)   // -deg + 2q
                                           : fsub(fmul(P.lam, q), 1.0f); // -1 + lambda q
  const float com = (sd >= 1e-6f) ? fmul(-P.comm, fdiv(fsub(pi, mu), sd)) : 0.0f;
  const float gp = fadd(fadd(obj, ent), com);
  const float g = fmul(gp, fmul(pi, fsub(1.0f, pi)));                 // chain rule through sigmoid
  float t1 = fmul(th, P.at);                                          // decoupled weight decay
  mm = fadd(fmul(P.b1, mm), fmul(P.c1, g));
  vv = fadd(fmul(P.b2, vv), fmul(fmul(P.c2, g), g));
  const float den = fadd(fmul(__fsqrt_rn(vv), P.rt), P.eps);
  th = fsub(t1, fmul(P.st, fdiv(mm, den)));
  return sigmoid_c(th);
}

// K2: the fused step. Per variable i (one lane group): gather q = A p, finalize
// mu_i / STD_i from the previous step's sums, gradient + AdamW + sigmoid for all
// local replicas, then this rank's fixed-point sums of p_next (warp shuffles).
template <int LANES, int VPL>
__global__ void __launch_bounds__(256) k_step(const StepParams P) {
  const int lane = threadIdx.x & (LANES - 1);
  const unsigned gmask = (LANES == 32) ? 0xffffffffu
                                       : (((1u << LANES) - 1u) << ((threadIdx.x & 31) & ~(LANES - 1)));
  const int group = (blockIdx.x * blockDim.x + threadIdx.x) / LANES;
  const int ngroups = (gridDim.x * blockDim.x) / LANES;
  const float4* __restrict__ pc4 = reinterpret_cast<const float4*>(P.p_cur);
  float4* __restrict__ pn4 = reinterpret_cast<float4*>(P.p_next);
  float4* __restrict__ th4 = reinterpret_cast<float4*>(P.theta);
  float4* __restrict__ m4 = reinterpret_cast<float4*>(P.m);
  float4* __restrict__ v4 = reinterpret_cast<float4*>(P.v);
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_gather = policy_evict_last();
  bool bad = false;

  for (int i = group; i < P.n; i += ngroups) {
    float4 acc[VPL];
    gather_row<LANES, VPL>(P, i, lane, gmask, pol_gather, acc);

    float mu, sd;
    finalize_stats(P.c_cur[i], P.sums_cur[i], P.sums_cur[P.n + i], P.S_total, mu, sd);
    const float degf = (float)(__ldg(P.rowptr + i + 1) - __ldg(P.rowptr + i));

    long long sD = 0, sD2 = 0;
#pragma unroll
    for (int w = 0; w < VPL; ++w) {
      const int col = lane + w * LANES;
      if (col >= P.S_p4) continue;
      const size_t at = (size_t)i * P.S_p4 + col;
      float4 th = ld_stream(th4 + at, pol_stream);
      float4 mm = ld_stream(m4 + at, pol_stream);
      float4 vv = ld_stream(v4 + at, pol_stream);
      const float4 pp = pc4[at];
      float4 pn = pp;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (col * 4 + k >= P.S_local) continue;   // padding: never updated, no stats
        float t = comp(th, k), a = comp(mm, k), b = comp(vv, k);
        const float np = update_element(P, comp(acc[w], k), degf, comp(pp, k), mu, sd, t, a, b);
        bad |= !isfinite(t);
        set_comp(th, k, t); set_comp(mm, k, a); set_comp(vv, k, b); set_comp(pn, k, np);
        long long D, D2;
        stat_terms(np, mu, D, D2);
        sD += D; sD2 += D2;
      }
      st_stream(th4 + at, th, pol_stream);
      st_stream(m4 + at, mm, pol_stream);
      st_stream(v4 + at, vv, pol_stream);
      pn4[at] = pn;
    }
#pragma unroll
    for (int off = LANES / 2; off > 0; off >>= 1) {
      sD += __shfl_xor_sync(gmask, sD, off, LANES);
      sD2 += __shfl_xor_sync(gmask, sD2, off, LANES);
    }
    if (lane == 0) {
      P.sums_next[i] = sD;
      P.sums_next[P.n + i] = sD2;
      P.c_next[i] = mu;
    }
  }
  if (bad) atomicOr(P.flag, 1);
}

// ------------------------------------------------------------------- K1
struct InitParams {
  float* theta; float* m; float* v; float* p0; float* p1;
  float* c; long long* sums;            // c[n], sums[2][n]: this rank's partial
  int n, S_p4, S_local, S_total, replica_offset;
  uint64_t base;                        // mix64(seed)
  double lo, hi;
  int use_given;                        // 1: keep theta/m/v (set_state), recompute p and stats
  const float* c_given;                 // shift per row (NULL -> 1/2)
};

// theta_0 = lo + (hi - lo) k 2^-24, k = top 24 bits of mix64(mix64(seed) + i S_total + s).
template <int LANES, int VPL>
__global__ void __launch_bounds__(256) k_init(const InitParams P) {
  const int lane = threadIdx.x & (LANES - 1);
  const unsigned gmask = (LANES == 32) ? 0xffffffffu
                                       : (((1u << LANES) - 1u) << ((threadIdx.x & 31) & ~(LANES - 1)));
  const int group = (blockIdx.x * blockDim.x + threadIdx.x) / LANES;
  const int ngroups = (gridDim.x * blockDim.x) / LANES;
  for (int i = group; i < P.n; i += ngroups) {
    const float ci = P.c_given ? P.c_given[i] : 0.5f;
    long long sD = 0, sD2 = 0;
#pragma unroll
    for (int w = 0; w < VPL; ++w) {
      const int col = lane + w * LANES;
      if (col >= P.S_p4) continue;
      const size_t at = (size_t)i * P.S_p4 + col;
      float4 th, pp;
      float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
      th = P.use_given ? reinterpret_cast<float4*>(P.theta)[at] : zero;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int s = col * 4 + k;
        float t = 0.0f;
        if (s < P.S_local) {
          if (P.use_given) {
            t = comp(th, k);
          } else {
            const uint64_t key = P.base + (uint64_t)i * (uint64_t)P.S_total + (uint64_t)(P.replica_offset + s);
            const uint64_t kk = mix64(key) >> 40;
            const double x = __dadd_rn(P.lo, __dmul_rn(__dmul_rn(__dsub_rn(P.hi, P.lo), (double)kk), 0x1p-24));
            t = __double2float_rn(x);
          }
        }
        set_comp(th, k, t);
        const float pv = sigmoid_c(t);
        set_comp(pp, k, pv);
        if (s < P.S_local) {
          long long D, D2;
          stat_terms(pv, ci, D, D2);
          sD += D; sD2 += D2;
        }
      }
      reinterpret_cast<float4*>(P.theta)[at] = th;
      if (!P.use_given) {
        reinterpret_cast<float4*>(P.m)[at] = zero;
        reinterpret_cast<float4*>(P.v)[at] = zero;
      }
      reinterpret_cast<float4*>(P.p0)[at] = pp;
      reinterpret_cast<float4*>(P.p1)[at] = pp;
    }
#pragma unroll
    for (int off = LANES / 2; off > 0; off >>= 1) {
      sD += __shfl_xor_sync(gmask, sD, off, LANES);
      sD2 += __shfl_xor_sync(gmask, sD2, off, LANES);
    }
    if (lane == 0) {
      P.sums[i] = sD;
      P.sums[P.n + i] = sD2;
      P.c[i] = ci;
    }
  }
}

// --------------------------------------------------------- graph checks
// bit 1: column out of range, bit 2: unsorted / duplicate, bit 3: self-loop,
// bit 4: asymmetric (j's row lacks i).
__global__ void k_validate(const int* __restrict__ rowptr, const int* __restrict__ colidx, int n,
                           int* __restrict__ flag) {
  int bad = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int e0 = rowptr[i], e1 = rowptr[i + 1];
    int prev = -1;
    for (int e = e0; e < e1; ++e) {
      const int j = colidx[e];
      if (j < 0 || j >= n) { bad |= 2; continue; }
      if (j <= prev) bad |= 4;
      if (j == i) bad |= 8;
      prev = j;
      int lo = rowptr[j], hi = rowptr[j + 1];
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (colidx[mid] < i) lo = mid + 1; else hi = mid;
      }
      if (lo >= rowptr[j + 1] || colidx[lo] != i) bad |= 16;
    }
  }
  if (bad) atomicOr(flag, bad);
}

// ---------------------------------------------------------------- K3/K4/K5
// K3: X[i][w] bit b = (theta[i][32w+b] >= 0) for 32w+b < S_local  (Theta(0)=1)
__global__ void k_pack(const float* __restrict__ theta, uint32_t* __restrict__ X, int n, int S_p,
                       int S_local, int W) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long it = warp; it < (long long)n * W; it += nwarps) {
    const int i = (int)(it / W), w = (int)(it % W);
    const int s = w * 32 + lane;
    const bool x = (s < S_local) && (theta[(size_t)i * S_p + s] >= 0.0f);
    const uint32_t word = __ballot_sync(0xffffffffu, x);
    if (lane == 0) X[it] = word;
  }
}

// K4: per-replica integer counts; lane = replica bit of word w; each undirected
// edge once (j > i). Warps 0..W*R-1: warp k takes word k % W and rows k / W, +R, ...
// counts[s][3] = (size, violations, cut), unsigned 64-bit atomics (exact, order-free).
__global__ void k_eval(const int* __restrict__ rowptr, const int* __restrict__ colidx,
                       const uint32_t* __restrict__ X, int n, int W, int R, int S_local,
                       unsigned long long* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= W * R) return;
  const int w = warp % W;
  unsigned long long size = 0, viol = 0, cut = 0;
  for (int i = warp / W; i < n; i += R) {
    const uint32_t bi = (X[(size_t)i * W + w] >> lane) & 1u;
    size += bi;
    const int e1 = rowptr[i + 1];
    for (int e = rowptr[i]; e < e1; ++e) {
      const int j = colidx[e];
      if (j <= i) continue;
      const uint32_t bj = (X[(size_t)j * W + w] >> lane) & 1u;
      viol += bi & bj;
      cut += bi ^ bj;
    }
  }
  const int s = w * 32 + lane;
  if (s < S_local && (size | viol | cut)) {
    atomicAdd(counts + 3 * s + 0, size);
    atomicAdd(counts + 3 * s + 1, viol);
    atomicAdd(counts + 3 * s + 2, cut);
  }
}

// K5: energies of all S_total replicas and argmin (lowest index on ties). One CTA.
__global__ void k_argmin(const long long* __restrict__ counts, int S_total, int problem, double lam,
                         double* __restrict__ energy, int* __restrict__ best, double* __restrict__ best_e) {
  __shared__ double se[32];
  __shared__ int si[32];
  double be = 0.0;
  int bi = -1;
  for (int s = threadIdx.x; s < S_total; s += blockDim.x) {
    const double e = (problem == kMAXCUT)
                         ? -(double)counts[3 * s + 2]
                         : __dadd_rn(-(double)counts[3 * s + 0], __dmul_rn(lam, (double)counts[3 * s + 1]));
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

// x of one local replica as bytes.
__global__ void k_extract(const uint32_t* __restrict__ X, int n, int W, int s_local, uint8_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = (uint8_t)((X[(size_t)i * W + (s_local >> 5)] >> (s_local & 31)) & 1u);
}

}  // namespace qqa
