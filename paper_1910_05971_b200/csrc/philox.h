// Counter-based PRNG shared by the host generators and (later) device-side
// generators: Philox-4x32-10 (Salmon et al., SC'11). Pure function of
// (key, counter), so every edge of a synthetic graph is reproducible from
// its index alone and generation parallelises without shared state.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define FSV_HD __host__ __device__ __forceinline__
#else
#define FSV_HD static inline
#endif

typedef struct { uint32_t v[4]; } fsv_u32x4;

FSV_HD uint32_t fsv_mulhilo32(uint32_t a, uint32_t b, uint32_t* hi) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  return (uint32_t)p;
}

// counter = (c0, c1, c2, c3), key = (k0, k1)
FSV_HD fsv_u32x4 fsv_philox4x32(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, hi1;
    uint32_t lo0 = fsv_mulhilo32(M0, c0, &hi0);
    uint32_t lo1 = fsv_mulhilo32(M1, c2, &hi1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0; k1 += W1;
  }
  fsv_u32x4 out;
  out.v[0] = c0; out.v[1] = c1; out.v[2] = c2; out.v[3] = c3;
  return out;
}

// Stream ids separate the independent random sequences of one generator so
// that e.g. the RMAT quadrant draws and the id permutation never overlap.
enum {
  FSV_STREAM_RMAT = 1,
  FSV_STREAM_PERM = 2,
  FSV_STREAM_GRID = 3,
  FSV_STREAM_TREE_SIZE = 4,
  FSV_STREAM_TREE_PARENT = 5,
  FSV_STREAM_TREE_EXTRA = 6,
  FSV_STREAM_GNM = 7
};

// Four 32-bit uniforms for (seed, stream, index hi/lo, word-group).
FSV_HD fsv_u32x4 fsv_draw4(uint64_t seed, uint32_t stream, uint64_t index, uint32_t group) {
  return fsv_philox4x32((uint32_t)index, (uint32_t)(index >> 32), group, stream,
                        (uint32_t)seed, (uint32_t)(seed >> 32));
}

// Uniform integer in [0, range) by Lemire's multiply-shift (range < 2^32).
FSV_HD uint32_t fsv_bounded(uint32_t r, uint32_t range) {
  return (uint32_t)(((uint64_t)r * (uint64_t)range) >> 32);
}
