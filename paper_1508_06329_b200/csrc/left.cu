// left.cu -- left neighbourhoods and parents under an ordering.
//
// Replaces left_neighborhoods (graph.py:284-302): LN(v) = N(v) restricted to
// the vertices placed before v, parent(v) = the member of LN(v) with the
// greatest position (-1 when LN(v) is empty).  The same quantities are what
// the reference's list scan builds in its scan 1 (peo.py:106-121), so the
// kernels also return |LN(v)| and deg(v): the host reconstructs ScanStats'
// read count from them in O(n) (peo.py:100-149).
//
// Dense rows: one warp per vertex v (grid-stride), lane l takes 32-bit words
// l, l+32, ...; every set bit u is kept iff pos[u] < pos[v] (one gather per
// neighbour, eight in flight per lane).  The masked words are written to a
// row of the same pitch (LN rows, optional), the kept count and max position
// are reduced over the warp.  Bytes per vertex: its row (read) + its LN row
// (written) + deg(v) 4-byte pos gathers.
// CSR: one warp per vertex over its index slice, same reductions.
#include "common.cuh"

namespace chordal {

namespace {

__device__ __forceinline__ void warp_reduce(int &best, int &cnt, int &deg) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        best = max(best, __shfl_xor_sync(CH_FULL, best, d));
        cnt += __shfl_xor_sync(CH_FULL, cnt, d);
        deg += __shfl_xor_sync(CH_FULL, deg, d);
    }
}

}  // namespace

__global__ void __launch_bounds__(256)
left_dense_kernel(const uint8_t *__restrict__ adj, int n, long long stride, const int32_t *__restrict__ order,
                  const int32_t *__restrict__ pos, uint8_t *__restrict__ ln_rows, int32_t *__restrict__ parent,
                  int32_t *__restrict__ ln_size, int32_t *__restrict__ deg) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int words = (int)(stride >> 2);  // whole pitch: padding words are copied as zero
    for (int v = gw; v < n; v += nwarps) {
        const int pv = __ldg(pos + v);
        const uint32_t *row = reinterpret_cast<const uint32_t *>(adj + (long long)v * stride);
        uint32_t *out = ln_rows ? reinterpret_cast<uint32_t *>(ln_rows + (long long)v * stride) : nullptr;
        int best = -1, cnt = 0, dg = 0;
        for (int w = lane; w < words; w += 32) {
            uint32_t x = __ldg(row + w);
            dg += __popc(x);
            uint32_t keep = 0;
            while (x) {  // up to eight position lookups in flight
                int b[8], pu[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    b[j] = x ? __ffs(x) - 1 : -1;
                    x &= x - 1;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) pu[j] = b[j] >= 0 ? __ldg(pos + 32 * w + b[j]) : 0x7FFFFFFF;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (pu[j] < pv) {
                        keep |= 1u << b[j];
                        best = max(best, pu[j]);
                    }
                }
            }
            cnt += __popc(keep);
            if (out) out[w] = keep;
        }
        warp_reduce(best, cnt, dg);
        if (lane == 0) {
            if (parent) parent[v] = best >= 0 ? __ldg(order + best) : -1;
            if (ln_size) ln_size[v] = cnt;
            if (deg) deg[v] = dg;
        }
    }
}

__global__ void __launch_bounds__(256)
left_csr_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices, int n,
                const int32_t *__restrict__ order, const int32_t *__restrict__ pos, int32_t *__restrict__ parent,
                int32_t *__restrict__ ln_size) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int v = gw; v < n; v += nwarps) {
        const int pv = __ldg(pos + v);
        const long long a = __ldg(indptr + v), e = __ldg(indptr + v + 1);
        int best = -1, cnt = 0, dg = 0;
        for (long long i = a + lane; i < e; i += 32) {
            const int pu = __ldg(pos + __ldg(indices + i));
            if (pu < pv) {
                ++cnt;
                best = max(best, pu);
            }
        }
        warp_reduce(best, cnt, dg);
        if (lane == 0) {
            if (parent) parent[v] = best >= 0 ? __ldg(order + best) : -1;
            if (ln_size) ln_size[v] = cnt;
        }
    }
}

static int grid_for(int64_t n) {
    int64_t blocks = (n * 32 + 255) / 256;
    const int64_t cap = 148LL * 16;
    if (blocks > cap) blocks = cap;
    return (int)(blocks < 1 ? 1 : blocks);
}

int launch_left_dense(const uint8_t *adj, int64_t n, int64_t stride, const int32_t *order, const int32_t *pos,
                      uint8_t *ln_rows, int32_t *parent, int32_t *ln_size, int32_t *deg, cudaStream_t s) {
    if (n == 0) return CHORDAL_OK;
    left_dense_kernel<<<grid_for(n), 256, 0, s>>>(adj, (int)n, stride, order, pos, ln_rows, parent, ln_size, deg);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

int launch_left_csr(const int64_t *indptr, const int32_t *indices, int64_t n, const int32_t *order,
                    const int32_t *pos, int32_t *parent, int32_t *ln_size, cudaStream_t s) {
    if (n == 0) return CHORDAL_OK;
    left_csr_kernel<<<grid_for(n), 256, 0, s>>>(indptr, indices, (int)n, order, pos, parent, ln_size);
    CH_LAUNCH_CHECK();
    return CHORDAL_OK;
}

}  // namespace chordal
