// Microbenchmark (tooling, not product): random 4-byte gather rate from an
// L2-resident 16.8 MB table when the CTA also holds a large shared-memory
// allocation (the hub table leaves ~28 KB of L1 for global loads).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)
__global__ void fill_idx(uint32_t* idx, size_t m, uint32_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < m; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = 12345 + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    idx[i] = (uint32_t)(z % n);
  }
}
template <int MODE, int PER>
__global__ void gather(const uint32_t* __restrict__ idx, size_t m, const int* __restrict__ tab, int* out) {
  extern __shared__ int sm[];
  if (threadIdx.x == 0 && out == nullptr) sm[0] = 1;
  int acc = 0x7fffffff;
  const size_t stride = (size_t)gridDim.x * blockDim.x * PER;
  for (size_t i = (blockIdx.x * (size_t)blockDim.x) * PER + threadIdx.x; i < m; i += stride) {
    uint32_t c[PER]; int v[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) c[j] = idx[i + j * blockDim.x];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (MODE == 0) v[j] = __ldg(tab + c[j]);
      else if (MODE == 1) v[j] = __ldcg(tab + c[j]);
      else if (MODE == 2) asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v[j]) : "l"(tab + c[j]));
      else asm volatile("ld.global.relaxed.gpu.b32 %0, [%1];" : "=r"(v[j]) : "l"(tab + c[j]));
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) acc = min(acc, v[j]);
  }
  if (acc == -12345) out[0] = acc + sm[0];
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  size_t m = 64ull << 20;
  uint32_t n = 1u << 22;
  uint32_t* idx; int* tab; int* out;
  CK(cudaMalloc(&idx, m * 4 + (1 << 20))); CK(cudaMalloc(&tab, (size_t)n * 4)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(tab, 0, (size_t)n * 4));
  fill_idx<<<4096, 256>>>(idx, m + (1 << 18), n); CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"ldg(nc)", "ldcg", "nc.no_allocate", "relaxed.gpu"};
  for (int smem : {0, 32 * 1024, 64 * 1024, 100 * 1024, 132 * 1024, 164 * 1024, 180 * 1024, 196 * 1024, 212 * 1024, 224 * 1024})
    for (int mode = 0; mode < 2; ++mode)
      for (int per : {8}) {
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          auto launch = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            cudaEventRecord(e0);
            kern<<<p.multiProcessorCount, 1024, smem>>>(idx, m, tab, out);
            cudaEventRecord(e1);
          };
          if (per == 4) { if (mode == 0) launch(gather<0, 4>); else if (mode == 1) launch(gather<1, 4>); else if (mode == 2) launch(gather<2, 4>); else launch(gather<3, 4>); }
          else { if (mode == 0) launch(gather<0, 8>); else if (mode == 1) launch(gather<1, 8>); else if (mode == 2) launch(gather<2, 8>); else launch(gather<3, 8>); }
          CK(cudaDeviceSynchronize());
          float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        printf("smem %3d KB  %-15s per %d: %.3f ms  %.1f Ggather/s\n", smem >> 10, names[mode], per, best, m / best * 1e-6);
      }
  return 0;
}
