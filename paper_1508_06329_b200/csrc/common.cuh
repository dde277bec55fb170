// common.cuh -- shared device helpers for the sm_100a chordality kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/chordal_b200.h"

#define CH_FULL 0xFFFFFFFFu

namespace chordal {

// splitmix64 / mix64 (reference _bitops.py:43-57) -- the seeded-arbitration
// tie key of parallel/engine.py:47-53.
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t mix64_3(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t h = splitmix64(a);
    h = splitmix64(h ^ b);
    return splitmix64(h ^ c);
}

// mix64(crc32("current"), 0): the "current" cell hash of engine.py:69-70.
// crc32("current") is computed on the host (capi.cu) and folded here.
__host__ __device__ __forceinline__ uint64_t current_cell(uint32_t crc_current) {
    return splitmix64(splitmix64((uint64_t)crc_current) ^ 0ULL);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ uint32_t mask_below(int b) {  // bits [0, b), b in [0,32]
    return b >= 32 ? CH_FULL : ((1u << b) - 1u);
}

__device__ __forceinline__ int highest_bit(uint32_t x) { return 31 - __clz(x); }

}  // namespace chordal

// Status helpers used by the C-ABI layer.
#define CH_LAUNCH_CHECK()                                  \
    do {                                                   \
        cudaError_t _e = cudaGetLastError();               \
        if (_e != cudaSuccess) return CHORDAL_ECUDA;       \
    } while (0)
