// gen.cu -- device-side, bit-exact replay of the reference's dense generator.
//
// gen_dense_random(n, p, seed) (generate.py:32-56) draws one uniform double
// per ordered cell of each 1024-row block, row-major, from the Philox4x64-10
// stream keyed by mix64(seed, crc32("dense-random")) (rng.py:18-21), keeps
// the strict upper triangle (cols > row) and mirrors it.  Because the blocks
// are consecutive full rows, draw number k = u*n + v decides edge {u, v},
// u < v.  numpy's Philox increments its 256-bit counter before producing
// each 4-word block, so block c = k/4 + 1, word k%4; the double is
// (x >> 11) * 2^-53 (numpy random_standard_uniform).
//
// Kernel 1 writes every row word (upper-triangle bits only); kernel 2 ORs in
// the mirrored lower triangle with a 32x32 ballot bit-transpose per warp.
#include "common.cuh"

namespace chordal {

namespace {

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

__device__ __forceinline__ uint64_t dense_key(long long seed, uint32_t crc) {
    // mix64(seed, crc32("dense-random")) -- _bitops.py:51-57
    return splitmix64(splitmix64((uint64_t)seed) ^ (uint64_t)crc);
}

}  // namespace

// One thread per (graph, row u, 32-bit word w).
__global__ void gen_dense_upper_kernel(uint8_t *__restrict__ adj, long long batch, int n, int stride,
                                       double p, long long seed0, long long seed_step, uint32_t crc) {
    const int words = stride >> 2;
    const long long total = batch * (long long)n * words;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(t % words);
        const long long r = t / words;
        const int u = (int)(r % n);
        const long long b = r / n;
        uint32_t bits = 0;
        const int v0 = 32 * w;
        if (v0 + 31 > u && v0 < n) {
            const uint64_t key = dense_key(seed0 + b * seed_step, crc);
            const int vlo = max(v0, u + 1), vhi = min(v0 + 32, n);
            long long k = (long long)u * n + vlo;
            const long long kend = (long long)u * n + vhi;
            while (k < kend) {
                U4 blk = philox4x64_10((uint64_t)(k >> 2) + 1, key);
                for (int j = (int)(k & 3); j < 4 && k < kend; ++j, ++k) {
                    double d = (double)(blk.v[j] >> 11) * (1.0 / 9007199254740992.0);
                    if (d < p) bits |= 1u << ((int)(k - (long long)u * n) - v0);
                }
            }
        }
        reinterpret_cast<uint32_t *>(adj + r * stride)[w] = bits;
    }
}

// One warp per 32x32 lower tile (I >= J) of one graph: rows 32I+c, word J
// receive bit r = A[32J + r][32I + c] (upper triangle, written by kernel 1).
__global__ void gen_mirror_kernel(uint8_t *__restrict__ adj, long long batch, int n, int stride) {
    const int lane = threadIdx.x & 31;
    const int RB = (n + 31) >> 5;
    const long long tiles = (long long)RB * (RB + 1) / 2;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarp = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long t = gw; t < batch * tiles; t += nwarp) {
        const long long b = t / tiles;
        long long k = t % tiles;
        // tile index k -> (I, J) with 0 <= J <= I
        int I = (int)((sqrt(8.0 * (double)k + 1.0) - 1.0) * 0.5);
        while ((long long)I * (I + 1) / 2 > k) --I;
        while ((long long)(I + 1) * (I + 2) / 2 <= k) ++I;
        const int J = (int)(k - (long long)I * (I + 1) / 2);
        uint8_t *g = adj + b * (long long)n * stride;
        const int srow = 32 * J + lane;
        uint32_t src = srow < n ? reinterpret_cast<const uint32_t *>(g + (long long)srow * stride)[I] : 0u;
        uint32_t mine = 0;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            uint32_t bal = __ballot_sync(CH_FULL, (src >> c) & 1u);
            if (lane == c) mine = bal;
        }
        const int drow = 32 * I + lane;
        if (drow < n && mine) {
            // each destination word has exactly one writer; on the diagonal
            // tile this warp is also the only reader of the word (read above)
            uint32_t *dst = reinterpret_cast<uint32_t *>(g + (long long)drow * stride) + J;
            *dst |= mine;
        }
    }
}

int launch_gen_dense_random(uint8_t *adj, int64_t batch, int64_t n, int64_t stride, double p,
                            int64_t seed0, int64_t seed_step, uint32_t crc, cudaStream_t stream) {
    const int threads = 256;
    long long total = batch * n * (stride >> 2);
    long long blocks = (total + threads - 1) / threads;
    if (blocks > 148LL * 64) blocks = 148LL * 64;
    gen_dense_upper_kernel<<<(int)blocks, threads, 0, stream>>>(adj, batch, (int)n, (int)stride, p, seed0,
                                                                seed_step, crc);
    CH_LAUNCH_CHECK();
    const long long RB = (n + 31) / 32;
    long long warps = batch * RB * (RB + 1) / 2;
    long long mblocks = (warps * 32 + threads - 1) / threads;
    if (mblocks > 148LL * 64) mblocks = 148LL * 64;
    gen_mirror_kernel<<<(int)mblocks, threads, 0, stream>>>(adj, batch, (int)n, (int)stride);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal
