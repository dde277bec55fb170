// dense_util.cu -- small device helpers of the dense entry points: positions
// from an order (VertexOrdering.pos0, graph.py:224-230), the relabelling used to
// replay the reference's seeded array tie-break (search.py:535-541), and fill.
#include "common.cuh"

namespace chordal {

__global__ void positions_kernel(const int32_t *__restrict__ order, int n, int32_t *__restrict__ pos) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        pos[order[i]] = i;
}

int launch_positions(const int32_t *order, int64_t n, int32_t *pos, cudaStream_t stream) {
    if (n <= 0) return CHORDAL_OK;
    int blocks = (int)((n + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    positions_kernel<<<blocks, 256, 0, stream>>>(order, (int)n, pos);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal

namespace chordal {

// Relabel: out[r] bit s = adj[perm[r]][perm[s]].  Used to replay the
// reference's seeded array tie-break (search.py:535-541: ties go to the
// earliest vertex of a Philox permutation) with the ascending kernel.
__global__ void permute_dense_kernel(const uint8_t *__restrict__ adj, int n, long long stride,
                                     const int32_t *__restrict__ perm, uint8_t *__restrict__ out) {
    const int words = (int)(stride >> 2);
    const long long total = (long long)n * words;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(t / words), w = (int)(t % words);
        uint32_t bits = 0;
        if (32 * w < n) {
            const uint32_t *row = reinterpret_cast<const uint32_t *>(adj + (long long)__ldg(perm + r) * stride);
            const int hi = min(32, n - 32 * w);
            for (int j = 0; j < hi; ++j) {
                int u = __ldg(perm + 32 * w + j);
                bits |= ((__ldg(row + (u >> 5)) >> (u & 31)) & 1u) << j;
            }
        }
        reinterpret_cast<uint32_t *>(out + (long long)r * stride)[w] = bits;
    }
}

int launch_permute_dense(const uint8_t *adj, int64_t n, int64_t stride, const int32_t *perm, uint8_t *out,
                         cudaStream_t stream) {
    if (n <= 0) return CHORDAL_OK;
    long long total = n * (stride >> 2);
    long long blocks = (total + 255) / 256;
    if (blocks > 148LL * 32) blocks = 148LL * 32;
    permute_dense_kernel<<<(int)blocks, 256, 0, stream>>>(adj, (int)n, stride, perm, out);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal

namespace chordal {

__global__ void fill_i32_kernel(int32_t *__restrict__ p, long long n, int32_t value) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = value;
}

int launch_fill_i32(int32_t *p, int64_t n, int32_t value, cudaStream_t stream) {
    if (n <= 0) return CHORDAL_OK;
    long long blocks = (n + 255) / 256;
    if (blocks > 148LL * 8) blocks = 148LL * 8;
    fill_i32_kernel<<<(int)blocks, 256, 0, stream>>>(p, n, value);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal

namespace chordal {

// Host rows arrive as one flat copy with pitch src_pitch (< stride, e.g. the
// reference's ceil(n/8)-byte packing): spread them to the device pitch, the
// first nb = ceil(n/8) bytes of each row copied and the rest of the row zeroed.
// (A pitched cudaMemcpy2D from pageable memory costs ~0.45 ms at n = 1000 --
// it is staged row by row -- against ~19 us for the flat copy plus this kernel.)
__global__ void spread_rows_kernel(const uint8_t *__restrict__ src, long long src_pitch, int n, int nb,
                                   long long stride, uint32_t *__restrict__ dst) {
    const long long words = stride >> 2, total = (long long)n * words;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long r = t / words;
        const int b0 = 4 * (int)(t - r * words);
        const uint8_t *row = src + r * src_pitch;
        uint32_t w = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (b0 + j < nb) w |= (uint32_t)__ldg(row + b0 + j) << (8 * j);
        dst[t] = w;
    }
}

// rows rows of nb vertex bytes (ceil(n/8)); a batch passes all its graphs' rows at once
int launch_spread_rows(const uint8_t *src, int64_t src_pitch, int64_t rows, int64_t nb, int64_t stride,
                       uint8_t *dst, cudaStream_t stream) {
    if (rows <= 0) return CHORDAL_OK;
    const long long total = rows * (stride >> 2);
    long long blocks = (total + 255) / 256;
    if (blocks > 148LL * 16) blocks = 148LL * 16;
    spread_rows_kernel<<<(int)blocks, 256, 0, stream>>>(src, src_pitch, (int)rows, (int)nb, stride,
                                                        reinterpret_cast<uint32_t *>(dst));
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal
