// Exhaustive check of qqa::sig_div (paper_2409_02135_b200/csrc/qqa_sigdiv.cuh) against __fdiv_rn over the
// sigmoid's operands: every fp32 E in [0, 1] (bit patterns 0 .. 0x3F800000), den = fl(1 + E), num in {1, E};
// and ln_c's: f = m - 1 over every mantissa m (halved above sqrt(2)), den = fl(2 + f).
// Prints "sigdiv: <checked> checked, <mismatches> mismatches" (and the first few mismatches).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#include "qqa_sigdiv.cuh"

__global__ void check(uint32_t lo, uint32_t hi, unsigned long long* bad, uint32_t* first) {
  for (uint64_t b = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= hi; b += (uint64_t)gridDim.x * blockDim.x) {
    const float E = __uint_as_float((uint32_t)b);
    const float den = __fadd_rn(1.0f, E);
    const float a1 = qqa::sig_div(1.0f, den), r1 = __fdiv_rn(1.0f, den);
    const float a2 = qqa::sig_div(E, den), r2 = __fdiv_rn(E, den);
    if (__float_as_uint(a1) != __float_as_uint(r1) || __float_as_uint(a2) != __float_as_uint(r2)) {
      const unsigned long long k = atomicAdd(bad, 1ull);
      if (k < 8) first[k] = (uint32_t)b;
    }
  }
}

// ln_c's s = f / (2 + f): every mantissa m of [1, 2), halved above sqrt(2) as ln_c does.
__global__ void check_ln(unsigned long long* bad, uint32_t* first) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < (1u << 23); b += gridDim.x * blockDim.x) {
    float m = __uint_as_float(b | 0x3f800000u);
    if (m > 1.41421356f) m = __fmul_rn(m, 0.5f);
    const float f = __fsub_rn(m, 1.0f);
    const float den = __fadd_rn(2.0f, f);
    if (__float_as_uint(qqa::sig_div(f, den)) != __float_as_uint(__fdiv_rn(f, den))) {
      const unsigned long long k = atomicAdd(bad, 1ull);
      if (k < 8) first[k] = b;
    }
  }
}

int main() {
  unsigned long long* bad; uint32_t* first;
  cudaMalloc(&bad, sizeof(*bad)); cudaMalloc(&first, 8 * sizeof(uint32_t));
  cudaMemset(bad, 0, sizeof(*bad)); cudaMemset(first, 0, 8 * sizeof(uint32_t));
  const uint32_t lo = 0u, hi = 0x3F800000u;   // +0 .. 1.0f
  check<<<148 * 8, 256>>>(lo, hi, bad, first);
  check_ln<<<148 * 8, 256>>>(bad, first);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("sigdiv: CUDA error\n"); return 2; }
  unsigned long long nb = 0; uint32_t f[8];
  cudaMemcpy(&nb, bad, sizeof(nb), cudaMemcpyDeviceToHost);
  cudaMemcpy(f, first, sizeof(f), cudaMemcpyDeviceToHost);
  printf("sigdiv: %llu checked, %llu mismatches\n", (unsigned long long)(hi - lo) + 1ull + (1ull << 23), nb);
  for (unsigned long long k = 0; k < nb && k < 8; ++k) {
    float E; memcpy(&E, &f[k], 4);
    printf("  E = %a (0x%08x)\n", E, f[k]);
  }
  return nb == 0 ? 0 : 1;
}
