// Microbenchmark (tooling, not product): random 4-byte gather throughput on B200
// from tables of various sizes, to size the FastSV phase-H design.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void fill_idx(uint32_t* idx, size_t m, uint32_t n, uint64_t seed, int skew) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < m; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    uint32_t v;
    if (skew) { // crude power law: square of uniform concentrates near 0, then scatter by hash
      double u = (double)(z >> 11) * (1.0 / 9007199254740992.0);
      uint64_t r = (uint64_t)(u * u * u * n);
      uint64_t h = r * 0x9E3779B97F4A7C15ull; v = (uint32_t)((h >> 20) % n);
      v = (uint32_t)((r * 2654435761ull) % n);
    } else v = (uint32_t)(z % n);
    idx[i] = v;
  }
}
template <int MODE>
__global__ void gather(const uint4* __restrict__ idx4, size_t m4, const int* __restrict__ tab, int* out) {
  int acc = 0x7fffffff;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < m4; i += (size_t)gridDim.x * blockDim.x) {
    uint4 c;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(c.x),"=r"(c.y),"=r"(c.z),"=r"(c.w) : "l"(idx4 + i));
    int a,b,d,e;
    if (MODE == 0) { a = __ldg(tab + c.x); b = __ldg(tab + c.y); d = __ldg(tab + c.z); e = __ldg(tab + c.w); }
    else if (MODE == 1) { a = __ldcg(tab + c.x); b = __ldcg(tab + c.y); d = __ldcg(tab + c.z); e = __ldcg(tab + c.w); }
    else { a = (int)c.x; b = (int)c.y; d = (int)c.z; e = (int)c.w; }
    acc = min(acc, min(min(a, b), min(d, e)));
  }
  if (acc == -12345) out[0] = acc;
}
int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int l2 = 0; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  int maxPersist = 0; cudaDeviceGetAttribute(&maxPersist, cudaDevAttrMaxPersistingL2CacheSize, dev);
  printf("dev %s SMs %d L2 %d MB maxPersistL2 %d MB smemPerBlockOptin %zu\n", p.name, p.multiProcessorCount, l2 >> 20, maxPersist >> 20, p.sharedMemPerBlockOptin);
  size_t m = 128ull << 20;  // 128M gathers (RMAT-22 m_dir ~ 128M)
  uint32_t* idx; int* tab; int* out;
  CK(cudaMalloc(&idx, m * 4)); CK(cudaMalloc(&tab, (size_t)1 << 31)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(tab, 0, (size_t)1 << 31));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  uint32_t sizes[] = {1u << 16, 1u << 20, 1u << 22, 1u << 24, 1u << 26, 1u << 28};
  for (int skew = 0; skew < 2; ++skew)
  for (uint32_t n : sizes) {
    fill_idx<<<4096, 256>>>(idx, m, n, 12345, skew); CK(cudaDeviceSynchronize());
    for (int mode = 0; mode < 3; ++mode) {
      for (int bs : {256}) for (int gm : {8, 16}) {
        int grid = p.multiProcessorCount * gm;
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
          cudaEventRecord(e0);
          if (mode == 0) gather<0><<<grid, bs>>>((const uint4*)idx, m / 4, tab, out);
          else if (mode == 1) gather<1><<<grid, bs>>>((const uint4*)idx, m / 4, tab, out);
          else gather<2><<<grid, bs>>>((const uint4*)idx, m / 4, tab, out);
          cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
          float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        printf("skew %d table %6u K entries (%7.1f MB) mode %s grid %d: %.3f ms  %.1f Ggather/s  idx-stream %.0f GB/s\n",
          skew, n >> 10, n * 4.0 / 1e6, mode == 0 ? "nc " : mode == 1 ? "cg " : "none", grid, best, m / best / 1e6, m * 4.0 / best / 1e6);
      }
    }
  }
  return 0;
}
