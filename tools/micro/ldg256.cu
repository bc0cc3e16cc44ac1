// Microbenchmark: per-lane random 128 B record reads (BVH-node-like access)
// with 8 x LDG.128 vs 4 x LDG.256 (sm_100a); prints time per variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld256(const float4 *p, float4 &a, float4 &b) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                 "=f"(b.w)
               : "l"(p));
}

template <int MODE>
__global__ void k(const float4 *__restrict__ nodes, uint32_t n_nodes, int iters,
                  float *__restrict__ out) {
  uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 1u;
  float acc = 0.f;
  uint32_t idx = x % n_nodes;
  for (int it = 0; it < iters; ++it) {
    const float4 *p = nodes + 8 * (size_t)idx;
    float4 r[8];
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __ldg(p + j);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) ld256(p + 2 * j, r[2 * j], r[2 * j + 1]);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += r[j].x + r[j].y + r[j].z + r[j].w;
    acc += s;
    // next index depends on the data (a dependent chain like traversal)
    x = x * 1664525u + 1013904223u + (__float_as_uint(s) & 1u);
    idx = x % n_nodes;
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const uint32_t n_nodes = (16u << 20) / 128;  // 16 MB working set
  float4 *nodes;
  float *out;
  cudaMalloc(&nodes, (size_t)n_nodes * 128);
  cudaMemset(nodes, 0, (size_t)n_nodes * 128);
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 128, blocks = sms * 12, iters = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(nodes, n_nodes, iters, out);
      else k<1><<<blocks, threads>>>(nodes, n_nodes, iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double recs = (double)blocks * threads * iters;
      printf("mode %s: %.3f ms, %.2f G records/s, %.1f GB/s\n", mode ? "4xLDG.256" : "8xLDG.128",
             ms, recs / ms / 1e6, recs * 128 / ms / 1e6);
    }
  }
  return 0;
}
