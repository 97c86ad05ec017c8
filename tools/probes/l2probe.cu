// L2 capacity probe (design evidence for DESIGN.md §4, not product code): random 32-byte gathers over a
// working set of X MB from every SM, alone (mode 0) or interleaved with c5-like streaming traffic
// (mode 1: per gathered row, read 4 and write 4 x 32 B of a separate 1 GB buffer with evict_first hints,
// the theta / m / v / p traffic of k_step). ncu's dram__bytes / lts__ hit rate / fabric sectors per X
// say whether the 126 MB L2 holds X (one copy per line) or only ~63 MB (a copy per die).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2probe l2probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

struct V8 { float f[8]; };
__device__ __forceinline__ V8 ldg_last(const float* p) {
  V8 r;
  asm volatile("ld.global.nc.L2::evict_last.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.f[0]), "=f"(r.f[1]), "=f"(r.f[2]), "=f"(r.f[3]), "=f"(r.f[4]), "=f"(r.f[5]), "=f"(r.f[6]),
                 "=f"(r.f[7]) : "l"(p));
  return r;
}
__device__ __forceinline__ V8 ldg_first(const float* p) {
  V8 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.f[0]), "=f"(r.f[1]), "=f"(r.f[2]), "=f"(r.f[3]), "=f"(r.f[4]), "=f"(r.f[5]), "=f"(r.f[6]),
                 "=f"(r.f[7]) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_first(float* p, const V8& v) {
  asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "l"(p), "f"(v.f[0]), "f"(v.f[1]), "f"(v.f[2]), "f"(v.f[3]), "f"(v.f[4]), "f"(v.f[5]), "f"(v.f[6]),
                  "f"(v.f[7]) : "memory");
}

// rows: X / 32 B rows; items: total (row-item) count; each item gathers 20 random rows (like degree 20)
__global__ void __launch_bounds__(256, 4) probe(const float* __restrict__ g, uint32_t rows, float* stream,
                                                 uint64_t stream_rows, uint32_t items, int mode, uint32_t seed,
                                                 float* out) {
  float acc = 0.f;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  // mode >= 2: the SMs are split in two halves by smid (split 0: smid < 74, 1: smid even, 2: (smid/2) even,
  // 3: (smid/4) even...); each half gathers only from its own half of the rows (a disjoint X/2 set)
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const int split = mode - 2;
  const uint32_t half = (split < 0) ? 0u
                        : (split == 0) ? (smid < 74u ? 0u : 1u) : ((smid >> (split - 1)) & 1u);
  const uint32_t rows_eff = (split < 0) ? rows : rows / 2;
  for (uint32_t it = tid; it < items; it += nt) {
    V8 a{};
#pragma unroll 4
    for (int k = 0; k < 20; ++k) {
      const uint32_t r = hash32(it * 20u + k + seed) % rows_eff + half * rows_eff;
      const V8 v = ldg_last(g + (size_t)r * 8);
#pragma unroll
      for (int q = 0; q < 8; ++q) a.f[q] += v.f[q];
    }
    if (mode == 1) {   // streams: 4 reads + 4 writes of 32 B per item, sequential over a separate buffer
      const uint64_t s = ((uint64_t)it * 4) % (stream_rows - 4);
      V8 t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) t[u] = ldg_first(stream + (s + u) * 8);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int q = 0; q < 8; ++q) t[u].f[q] += a.f[q];
        stg_first(stream + (s + u) * 8 + (size_t)0, t[u]);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += a.f[q];
  }
  if (acc == 123.456f) out[0] = acc;
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int mbs[] = {16, 32, 48, 64, 80, 96, 112, 128, 160};
  float *g, *stream, *out;
  const size_t gmax = (size_t)160 << 20, sbytes = (size_t)1 << 30;
  cudaMalloc(&g, gmax); cudaMalloc(&stream, sbytes); cudaMalloc(&out, 64);
  cudaMemset(g, 0, gmax); cudaMemset(stream, 0, sbytes);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t items = 1u << 23;   // 8.4M items x 20 gathers x 32 B = 5.4 GB gathered
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mb : mbs) {
    const uint32_t rows = (uint32_t)(((size_t)mb << 20) / 32);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      probe<<<sms * 4, 256>>>(g, rows, stream, sbytes / 32, items, mode, 1234u * rep, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("mode %d X %3d MB: %.3f ms, gathered %.2f GB -> %.0f GB/s of gathers\n", mode, mb, ms,
                           items * 20.0 * 32 / 1e9, items * 20.0 * 32 / 1e6 / ms);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
