// philox.cuh -- numpy's Philox4x64-10 bit generator and the Generator draws
// the reference's seeded features use (rng.py:18-21: key = mix64(seed,
// crc32(label)), counter starting at 0 and incremented before each block).
//   next64 / next32  numpy's random_next64 / next_uint32 (the low then the high
//                    half of a 64-bit output, buffered across calls as the bit
//                    generator does);
//   bounded          random_bounded_uint64 for ranges < 2^32 - 1 (Lemire's
//                    32-bit rejection) -- Generator.integers.
#pragma once
#include "common.cuh"

namespace chordal {

struct U4 {
    uint64_t v[4];
};

__device__ __forceinline__ U4 philox4x64_10(uint64_t c0, uint64_t key) {
    uint64_t c[4] = {c0, 0, 0, 0};
    uint64_t k0 = key, k1 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c[0];
        uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c[0]);
        uint64_t lo1 = 0xCA5A826395121157ULL * c[2];
        uint64_t hi1 = __umul64hi(0xCA5A826395121157ULL, c[2]);
        uint64_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
        k0 += 0x9E3779B97F4A7C15ULL;
        k1 += 0xBB67AE8584CAA73BULL;
    }
    U4 out;
    out.v[0] = c[0]; out.v[1] = c[1]; out.v[2] = c[2]; out.v[3] = c[3];
    return out;
}

struct PhiloxStream {
    uint64_t key, ctr;
    uint64_t b0, b1, b2, b3;
    int pos;
    bool has32;
    uint32_t u32;

    __device__ explicit PhiloxStream(uint64_t k) : key(k), ctr(0), b0(0), b1(0), b2(0), b3(0), pos(4), has32(false), u32(0) {}

    __device__ uint64_t next64() {
        if (pos >= 4) {
            ++ctr;
            U4 b = philox4x64_10(ctr, key);
            b0 = b.v[0]; b1 = b.v[1]; b2 = b.v[2]; b3 = b.v[3];
            pos = 0;
        }
        uint64_t x = pos == 0 ? b0 : pos == 1 ? b1 : pos == 2 ? b2 : b3;
        ++pos;
        return x;
    }
    __device__ uint32_t next32() {
        if (has32) {
            has32 = false;
            return u32;
        }
        uint64_t x = next64();
        has32 = true;
        u32 = (uint32_t)(x >> 32);
        return (uint32_t)x;
    }
    // random_bounded_uint64(off, rng) for 0 <= rng < 2^32 - 1 (inclusive range)
    __device__ uint64_t bounded(uint64_t off, uint64_t rng) {
        if (rng == 0) return off;
        const uint32_t excl = (uint32_t)rng + 1u;
        uint64_t m = (uint64_t)next32() * excl;
        uint32_t left = (uint32_t)m;
        if (left < excl) {
            const uint32_t th = (0xFFFFFFFFu - (uint32_t)rng) % excl;
            while (left < th) {
                m = (uint64_t)next32() * excl;
                left = (uint32_t)m;
            }
        }
        return off + (m >> 32);
    }
};

}  // namespace chordal
