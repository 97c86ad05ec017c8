// L2 -> SM gather throughput probe (design evidence for DESIGN.md §4/§5, not product code).
// Every item gathers DEG = 20 random rows of R bytes (R/32 lanes per row, one 256-bit load per lane, like
// k_step's replica-contiguous rows) from a working set of X MB, 4 rows in flight per lane, and sums them.
// With X = 16 MB every row is an L2 hit after the first touch: the time is the L2 -> SM rate for R-byte
// rows, the ceiling of the gather of a step kernel whose block of p is L2-resident.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw l2bw.cu ; ./l2bw [X_MB]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

struct V8 { float f[8]; };
__device__ __forceinline__ V8 ldg(const float* p) {
  V8 r;
  asm volatile("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.f[0]), "=f"(r.f[1]), "=f"(r.f[2]), "=f"(r.f[3]), "=f"(r.f[4]), "=f"(r.f[5]), "=f"(r.f[6]),
                 "=f"(r.f[7]) : "l"(p));
  return r;
}

template <int LANES>
__global__ void __launch_bounds__(256, 4) gather(const float* __restrict__ g, uint32_t rows, uint32_t items,
                                                  uint32_t seed, float* out) {
  const int lane = threadIdx.x & (LANES - 1);
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) / LANES;
  const uint32_t ngrp = gridDim.x * blockDim.x / LANES;
  float acc = 0.f;
  for (uint32_t it = grp; it < items; it += ngrp) {
    uint32_t h = hash32(it * 2654435761u + seed);
#pragma unroll 1
    for (int e = 0; e < 20; e += 4) {
      V8 b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        h = hash32(h + u + 1);
        b[u] = ldg(g + (size_t)(h % rows) * (LANES * 8) + lane * 8);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += b[u].f[k];
    }
  }
  if (acc == 12345.678f) out[0] = acc;
}

template <int LANES>
double run(const float* g, size_t X, float* out, int sms) {
  const uint32_t rows = (uint32_t)(X / (LANES * 32));
  const uint32_t items = (uint32_t)((5.12e9 / 20) / (LANES * 32));   // 5.12 GB of gathered rows, as c5
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<LANES><<<sms * 4, 256>>>(g, rows, items, 1, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) gather<LANES><<<sms * 4, 256>>>(g, rows, items, 7 + r, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = 5.0 * items * 20.0 * LANES * 32;
  printf("row %4d B, X %4zu MB: %.3f ms per 5.12 GB -> %6.0f GB/s of gathered rows\n", LANES * 32, X >> 20,
         ms / 5, bytes / (ms * 1e-3) / 1e9);
  return bytes / (ms * 1e-3);
}

int main(int argc, char** argv) {
  const size_t X = (size_t)(argc > 1 ? atoi(argv[1]) : 16) << 20;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *g, *out;
  cudaMalloc(&g, X);
  cudaMalloc(&out, 4);
  cudaMemset(g, 0, X);
  for (int rep = 0; rep < 2; ++rep) {
    run<1>(g, X, out, sms);
    run<2>(g, X, out, sms);
    run<4>(g, X, out, sms);
    run<8>(g, X, out, sms);
    run<16>(g, X, out, sms);
    run<32>(g, X, out, sms);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
